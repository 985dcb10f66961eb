import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2206_01784_b200 import global_histograms, radix_plan, onesweep_sort
rng = np.random.default_rng(1)
for n in [1000, 100_001, 3_000_000]:
    k = rng.integers(0, 2**64, size=n, dtype=np.uint64)
    h = global_histograms(k, radix_plan(64, 8))
    want = np.stack([np.bincount((k >> np.uint64(8*p)) & np.uint64(255), minlength=256) for p in range(8)])
    print(n, np.array_equal(np.asarray(h.counts), want), flush=True)
