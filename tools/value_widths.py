"""Sort throughput for every (key, value) width pair at 2^28 keys (uniform
keys, arange payload): the drop-in takes any value width, and numpy's
default arange payload is int64.  usage: python tools/value_widths.py [n]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2206_01784_b200 import DeviceSorter, KeyGenSpec, generate_keys

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 28
for kbits, kdt in ((32, torch.uint32), (64, torch.uint64)):
    keys = generate_keys(KeyGenSpec(q=1, seed=0, n=n, key_bits=kbits), device="cuda")
    for vb, vdt in ((0, None), (1, torch.uint8), (2, torch.int16), (4, torch.int32), (8, torch.int64)):
        vals = None if vdt is None else torch.arange(n, device="cuda").to(vdt)
        ok = torch.empty_like(keys)
        ov = None if vals is None else torch.empty_like(vals)
        s = DeviceSorter(n, kdt, vb)
        for _ in range(3):
            s(keys, ok, vals, ov, stats=False)
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        steps = 5
        t0.record()
        for _ in range(steps):
            s(keys, ok, vals, ov, stats=False)
        t1.record()
        torch.cuda.synchronize()
        ms = t0.elapsed_time(t1) / steps
        passes = kbits // 8
        gb = (n * (kbits // 8) * (1 + 2 * passes) + 2 * passes * n * vb) / 1e9
        print(f"u{kbits} keys + {vb}-byte values: {n / ms / 1e6:6.2f} GKey/s  {ms:7.2f} ms  "
              f"{gb / (ms * 1e-3):6.0f} GB/s (alg.)  tile {s.tile}", flush=True)
        del vals, ov, ok
    del keys
    torch.cuda.empty_cache()
