"""Per-tile timeline of one binning pass of the C2 sort (os_debug_trace).

Prints the distribution of each phase and how late predecessors publish L
relative to a tile's look-back start -- the quantity that decides whether
the decoupled look-back waits.  Usage: python tools/trace_diag.py [pass] [n]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2206_01784_b200 import DeviceSorter, KeyGenSpec, _native, generate_keys

pas = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 28
keys = generate_keys(KeyGenSpec(q=1, seed=0, n=n), device="cuda")
out = torch.empty_like(keys)
s = DeviceSorter(n, torch.uint32, graphs=False)  # the trace pointer is set per launch
for _ in range(3):
    s(keys, out, stats=False)
tiles = (n + s.tile - 1) // s.tile
buf = torch.zeros(tiles * 8, dtype=torch.int64, device="cuda")
L = _native.load()
L.os_debug_trace(buf.data_ptr(), pas)
s(keys, out, stats=False)
torch.cuda.synchronize()
L.os_debug_trace(None, -1)
t = buf.view(tiles, 8).cpu().numpy().astype(np.int64)
t0 = t[:, 0].min()
claim, staged, lpub, reord, gpub, end, sm = (t[:, i] - (t0 if i < 6 else 0) for i in range(7))
dur = end.max()
print(f"pass {pas}: {tiles} tiles, span {dur/1e3:.1f} us, timer resolution ~{np.diff(np.unique(claim))[:50].min() if len(np.unique(claim))>1 else -1} ns")


def q(name, x):
    p = np.percentile(x, [5, 25, 50, 75, 95, 99])
    print(f"{name:34s} mean {x.mean():8.0f}  p5 {p[0]:7.0f} p25 {p[1]:7.0f} p50 {p[2]:7.0f} p75 {p[3]:7.0f} p95 {p[4]:7.0f} p99 {p[5]:7.0f}")


# record layout (binning.cu): 0 claim, 1 staged, 2 L published, 3 reorder done
# (look-back start), 4 G published (digit 0), 5 done
q("claim -> keys staged (TMA)", staged - claim)
q("staged -> L published (rank+cnt)", lpub - staged)
q("L -> reorder done", reord - lpub)
q("reorder done -> G (look-back)", gpub - reord)
q("G -> done (scatter)", end - gpub)
q("claim -> done", end - claim)
lb_start = reord
# how much later than us did our predecessor publish L (positive = we waited)
lag = lpub[:-1] - lb_start[1:]
q("pred L - own look-back start", lag)
print(f"fraction of tiles whose predecessor's L came after their look-back start: {(lag > 0).mean():.3f}")
# G frontier: for each tile, distance back to the newest predecessor whose G was
# published before this tile's look-back started
order = np.argsort(gpub)
gsorted = gpub[order]
dist = []
for i in range(1000, tiles, max(1, tiles // 4000)):
    start = lb_start[i]
    # predecessors with G before start
    cand = np.nonzero(gpub[max(0, i - 512):i] <= start)[0]
    dist.append(i - (max(0, i - 512) + cand.max()) if len(cand) else 512)
q("distance to newest G at look-back start", np.array(dist, dtype=np.float64))
rate = tiles / (dur / 1e3)
print(f"tile rate {rate:.1f} tiles/us; resident blocks ~{np.mean([(claim <= x).sum() - (end <= x).sum() for x in np.linspace(dur*0.2, dur*0.8, 50)]):.0f}")


# look-back duration by tile index: the first wave of resident blocks has no
# published G below it, so its walks run back towards tile 0
lb = gpub - reord
wave = 148 * 4
for lo, hi in ((0, wave // 4), (wave // 4, wave // 2), (wave // 2, wave), (wave, 2 * wave), (2 * wave, tiles)):
    if lo < min(hi, tiles):
        q(f"look-back, tiles [{lo},{min(hi, tiles)})", lb[lo:min(hi, tiles)])
