"""Device throughput of the BASELINE configs other than the bench headline
(C2): C1, C3 (pairs, several key distributions) and C4 (64-bit keys).

Each line: GKey/s over `--steps` sorts of resident data (CUDA events on the
sort's stream), the per-pass binning time of the last timed sort, and the
fraction of the HBM roofline (1 + 2p) n (kb + vb) bytes.  Measurement tool
only; bench.py stays the driver contract.
    python tools/bench_configs.py [--n 268435456] [--steps 10] [--only C3]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2206_01784_b200 import DeviceSorter, KeyGenSpec, _native, generate_keys

PEAK = 6547.5


def peak():
    try:
        with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                               "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return PEAK


def run(name, keys, vals, key_dtype, steps, warmup):
    n = keys.numel()
    vb = 0 if vals is None else vals.element_size()
    s = DeviceSorter(n, key_dtype, vb)
    ko = torch.empty_like(keys)
    vo = None if vals is None else torch.empty_like(vals)
    L = _native.load()
    passes = s.passes
    stream = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(passes + 2)]
    for e in ev:
        e.record(stream)
    for _ in range(warmup):
        s(keys, ko, vals, vo, stats=False)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0.record(stream)
    for _ in range(steps - 1):
        s(keys, ko, vals, vo, stats=False)
    handles = (_native._vp * (passes + 2))(*[e.cuda_event for e in ev])
    _native.check(L.os_sort_events(
        keys.data_ptr(), ko.data_ptr(), None if vals is None else vals.data_ptr(),
        None if vo is None else vo.data_ptr(), n, s.spec.type_id, vb, 8, 0, s.spec.bits,
        s.tile, 0, s.ws.data_ptr(), s.ws.numel(), None, handles, passes + 2,
        stream.cuda_stream), "os_sort_events")
    t1.record(stream)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / steps
    kb = keys.element_size()
    pass_us = [ev[1 + k].elapsed_time(ev[2 + k]) * 1e3 for k in range(passes)]
    alg = (1 + 2 * passes) * n * (kb + vb) - n * vb  # histogram reads keys only
    line = {"config": name, "n": n, "key_bytes": kb, "val_bytes": vb, "tile": s.tile,
            "gkeys": n / ms / 1e6, "ms": ms, "hist_us": ev[0].elapsed_time(ev[1]) * 1e3,
            "pass_us": [round(x, 1) for x in pass_us],
            "pass_frac_hbm": round(2 * n * (kb + vb) / (sum(pass_us) / passes * 1e-6) / 1e9 / peak(), 3),
            "sort_frac_hbm": round(alg / (ms * 1e-3) / 1e9 / peak(), 3)}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 28)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    n = a.n
    dev = torch.device("cuda")
    cfgs = []
    cfgs.append(("C1 16M u32 keys", lambda: (generate_keys(KeyGenSpec(q=1, seed=0, n=1 << 24), device=dev), None, torch.uint32)))
    cfgs.append(("C2 u32 keys", lambda: (generate_keys(KeyGenSpec(q=1, seed=0, n=n), device=dev), None, torch.uint32)))
    for q in (1, 2, 4, 8, 16):
        cfgs.append((f"C3 u32 pairs q={q}", lambda q=q: (
            generate_keys(KeyGenSpec(q=q, seed=0, n=n), device=dev),
            torch.arange(n, dtype=torch.int32, device=dev).view(torch.uint32), torch.uint32)))
    cfgs.append(("C3 u32 pairs all-equal", lambda: (
        torch.full((n,), 0xABACADAE, dtype=torch.int64, device=dev).to(torch.uint32),
        torch.arange(n, dtype=torch.int32, device=dev).view(torch.uint32), torch.uint32)))
    cfgs.append(("C3 u32 pairs presorted", lambda: (
        torch.sort(generate_keys(KeyGenSpec(q=1, seed=0, n=n), device=dev).view(torch.int32) ^ (-2**31))[0].__xor__(-2**31).view(torch.uint32),
        torch.arange(n, dtype=torch.int32, device=dev).view(torch.uint32), torch.uint32)))
    for dt in (torch.uint64, torch.int64, torch.float64):
        cfgs.append((f"C4 {str(dt).split('.')[1]} keys + u32 values", lambda dt=dt: (
            generate_keys(KeyGenSpec(q=1, seed=0, n=n, key_bits=64), device=dev).view(dt),
            torch.arange(n, dtype=torch.int32, device=dev).view(torch.uint32), dt)))
    cfgs.append(("C5 single-GPU 2^31 u32 keys (8 strips)", lambda: (
        generate_keys(KeyGenSpec(q=1, seed=0, n=1 << 31), device=dev), None, torch.uint32)))
    for name, make in cfgs:
        if a.only and not any(s in name for s in a.only.split(",")):
            continue
        keys, vals, dt = make()
        run(name, keys, vals, dt, a.steps, a.warmup)
        del keys, vals
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
