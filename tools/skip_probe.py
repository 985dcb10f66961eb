"""Sort throughput on inputs with trivial digit places (pass skipping,
PassRoute) at 2^28 keys: ONESWEEP_B200_NO_SKIP=1 gives the fixed schedule.
usage: python tools/skip_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2206_01784_b200 import DeviceSorter, KeyGenSpec, generate_keys

n = 1 << 28
tag = "fixed" if os.environ.get("ONESWEEP_B200_NO_SKIP", "0") != "0" else "routed"
u32 = generate_keys(KeyGenSpec(q=1, seed=0, n=n), device="cuda")
u64 = generate_keys(KeyGenSpec(q=1, seed=1, n=n, key_bits=64), device="cuda")

def low(t, bits):  # keep the low bits (torch's CUDA AND skips the unsigned dtypes)
    s = {4: torch.int32, 8: torch.int64}[t.element_size()]
    return (t.view(s) & ((1 << bits) - 1)).view(t.dtype)


cases = {
    "u32 keys < 2^24": (low(u32, 24), None),
    "u32 keys < 2^16": (low(u32, 16), None),
    "u32 all-equal + u32 values": (torch.full((n,), 0x2BACADAE, dtype=torch.int32, device="cuda").view(torch.uint32),
                                   torch.arange(n, device="cuda").to(torch.int32)),
    "u64 keys < 2^32 + u32 values": (low(u64, 32), torch.arange(n, device="cuda").to(torch.int32)),
    "u64 keys < 2^32": (low(u64, 32), None),
    "u32 uniform (no trivial place)": (u32, None),
}
for name, (k, v) in cases.items():
    k = k.contiguous()
    ok = torch.empty_like(k)
    ov = None if v is None else torch.empty_like(v)
    s = DeviceSorter(n, k.dtype, 0 if v is None else v.element_size())
    for _ in range(3):
        s(k, ok, v, ov, stats=False)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(5):
        s(k, ok, v, ov, stats=False)
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / 5
    print(f"{tag:6s} {name:32s} {ms:7.3f} ms {n / ms / 1e6:7.2f} GKey/s", flush=True)
