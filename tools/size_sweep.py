"""Sort throughput (GKey/s) of u32 keys-only over a range of sizes with the
current library (ONESWEEP_B200_LIB selects a variant).  python tools/size_sweep.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2206_01784_b200 import DeviceSorter, KeyGenSpec, generate_keys

tag = os.environ.get("TAG", "lib")
for lg in (20, 22, 24, 25, 26, 27, 28):
    n = 1 << lg
    keys = generate_keys(KeyGenSpec(q=1, seed=0, n=n), device="cuda")
    out = torch.empty_like(keys)
    s = DeviceSorter(n, torch.uint32)
    for _ in range(5):
        s(keys, out, stats=False)
    steps = max(10, (1 << 30) // n)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0.record()
    for _ in range(steps):
        s(keys, out, stats=False)
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / steps
    print(f"{tag} 2^{lg} {ms * 1e3:9.1f} us {n / ms / 1e6:7.2f} GKey/s", flush=True)
