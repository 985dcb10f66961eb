"""Look-back diagnostics: run C2 sorts with device stats and report per-tile
look-back rounds and not-ready waits."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_01784_b200 import DeviceSorter, KeyGenSpec, generate_keys
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 28
keys = generate_keys(KeyGenSpec(q=1, seed=0, n=n), device="cuda")
out = torch.empty_like(keys)
s = DeviceSorter(n, torch.uint32)
for _ in range(3):
    s(keys, out)
s.stats.zero_()
s(keys, out)
torch.cuda.synchronize()
fast, reads, tiles, waits, rounds = s.stats.tolist()
digits = 256
print(f"lib={os.environ.get('ONESWEEP_B200_LIB','default')} tiles={tiles} rounds/digit-tile={rounds/tiles/digits:.2f} "
      f"waits/digit-tile={waits/tiles/digits:.2f} reads/digit-tile={reads/tiles/digits:.1f}")
