"""Reduce-then-scan ablation: the device rts_sort
(3n element transfers per place) against Onesweep (2n per place + one
histogram read) on the same keys, with per-phase CUDA-event times.
    python tools/bench_rts.py [--n 268435456] [--steps 10] [--pairs]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2206_01784_b200 import DeviceRtsSorter, DeviceSorter, KeyGenSpec, generate_keys


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 28)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--pairs", action="store_true")
    a = ap.parse_args()
    n = a.n
    keys = generate_keys(KeyGenSpec(q=1, seed=0, n=n), device="cuda")
    vals = torch.arange(n, dtype=torch.int32, device="cuda").view(torch.uint32) if a.pairs else None
    vb = 4 if a.pairs else 0
    ko = torch.empty_like(keys)
    vo = torch.empty_like(vals) if a.pairs else None
    stream = torch.cuda.current_stream()
    out = {"n": n, "pairs": a.pairs}

    rts = DeviceRtsSorter(n, torch.uint32, vb)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3 * rts.passes + 1)]
    for e in ev:  # torch creates the CUDA event on first record
        e.record(stream)
    for _ in range(a.warmup):
        rts(keys, ko, vals, vo)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0.record(stream)
    for i in range(a.steps):
        rts(keys, ko, vals, vo, events=ev if i == a.steps - 1 else None)
    t1.record(stream)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / a.steps
    ref = torch.sort(keys.to(torch.int64) & 0xFFFFFFFF, stable=True)
    ok = torch.equal(ko.to(torch.int64) & 0xFFFFFFFF, ref.values)
    up = [ev[3 * k].elapsed_time(ev[3 * k + 1]) * 1e3 for k in range(rts.passes)]
    pre = [ev[3 * k + 1].elapsed_time(ev[3 * k + 2]) * 1e3 for k in range(rts.passes)]
    down = [ev[3 * k + 2].elapsed_time(ev[3 * k + 3]) * 1e3 for k in range(rts.passes)]
    out["rts"] = {"ms": ms, "gkeys": n / ms / 1e6, "upsweep_us": up, "prefix_us": pre,
                  "downsweep_us": down, "sorted_ok": bool(ok),
                  "element_transfers": f"{3 * rts.passes}n"}

    one = DeviceSorter(n, torch.uint32, vb)
    for _ in range(a.warmup):
        one(keys, ko, vals, vo, stats=False)
    torch.cuda.synchronize()
    t0.record(stream)
    for _ in range(a.steps):
        one(keys, ko, vals, vo, stats=False)
    t1.record(stream)
    torch.cuda.synchronize()
    ms1 = t0.elapsed_time(t1) / a.steps
    out["onesweep"] = {"ms": ms1, "gkeys": n / ms1 / 1e6,
                       "element_transfers": f"{2 * one.passes + 1}n"}
    out["onesweep_speedup"] = ms / ms1
    print(json.dumps(out))


if __name__ == "__main__":
    main()
