"""Does replaying a sort as a CUDA graph shorten it?  Times `steps` plain
DeviceSorter sorts against `steps` replays of the same sort captured in a
torch.cuda.CUDAGraph (CUDA events; same buffers).  usage: python tools/graph_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2206_01784_b200 import DeviceSorter, KeyGenSpec, generate_keys


def timed(fn, steps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(steps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) * 1e3 / steps


for n in (1 << 22, 1 << 24, 1 << 26, 1 << 28):
    keys = generate_keys(KeyGenSpec(q=1, seed=0, n=n), device="cuda")
    out = torch.empty_like(keys)
    srt = DeviceSorter(n, keys.dtype)
    for _ in range(3):
        srt(keys, out, stats=False)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        with torch.cuda.graph(g, stream=side):
            srt(keys, out, stream=side, stats=False)
    torch.cuda.synchronize()
    steps = 50 if n <= 1 << 24 else 20
    plain = timed(lambda: srt(keys, out, stats=False), steps)
    graph = timed(g.replay, steps)
    ok = torch.equal(out.view(torch.int32).to(torch.int64) & 0xFFFFFFFF,
                     torch.sort(keys.view(torch.int32).to(torch.int64) & 0xFFFFFFFF).values)
    print(f"n=2^{n.bit_length() - 1}: plain {plain:8.1f} us  graph {graph:8.1f} us  "
          f"({n / plain / 1e3:6.1f} vs {n / graph / 1e3:6.1f} GKey/s) sorted={ok}", flush=True)
    del keys, out, srt, g
    torch.cuda.empty_cache()
