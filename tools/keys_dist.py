"""Keys-only u32 sort throughput at 2^28 over key distributions (uniform,
AND-of-q entropy reduction, all-equal, presorted).  python tools/keys_dist.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2206_01784_b200 import DeviceSorter, KeyGenSpec, generate_keys

tag = os.environ.get("TAG", "lib")
n = 1 << 28
s = DeviceSorter(n, torch.uint32)
out = torch.empty(n, dtype=torch.uint32, device="cuda")
cases = [("q=1", lambda: generate_keys(KeyGenSpec(q=1, seed=0, n=n), device="cuda")),
         ("q=4", lambda: generate_keys(KeyGenSpec(q=4, seed=0, n=n), device="cuda")),
         ("q=16", lambda: generate_keys(KeyGenSpec(q=16, seed=0, n=n), device="cuda")),
         ("all-equal", lambda: torch.full((n,), 0xABACADAE, dtype=torch.int64, device="cuda").to(torch.uint32)),
         ("presorted", lambda: torch.sort(generate_keys(KeyGenSpec(q=1, seed=0, n=n), device="cuda").to(torch.int64))[0].to(torch.uint32))]
for name, make in cases:
    keys = make()
    for _ in range(3):
        s(keys, out, stats=False)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0.record()
    for _ in range(10):
        s(keys, out, stats=False)
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / 10
    print(f"{tag} {name:10s} {ms:7.3f} ms {n / ms / 1e6:7.2f} GKey/s", flush=True)
    del keys
