import time, torch, numpy as np, sys
sys.path.insert(0, '/root/repo')
from paper_2206_01784_b200 import onesweep_sort, generate_keys, KeyGenSpec
n = 1 << 28
k = generate_keys(KeyGenSpec(q=1, seed=0, n=n), device='cuda')
h = torch.empty(n, dtype=torch.uint32, pin_memory=True); h.copy_(k); torch.cuda.synchronize()
hn = h.numpy()
for _ in range(2): onesweep_sort(hn)
d = torch.empty(n, dtype=torch.uint32, device='cuda')
o = torch.empty(n, dtype=torch.uint32, pin_memory=True)
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
    o.copy_(d, non_blocking=True); torch.cuda.synchronize(); t2 = time.perf_counter()
    r = onesweep_sort(hn); t3 = time.perf_counter()
    print(f"H2D {1e3*(t1-t0):.2f} ms ({4*n/(t1-t0)/1e9:.1f} GB/s)  D2H {1e3*(t2-t1):.2f} ms ({4*n/(t2-t1)/1e9:.1f} GB/s)  e2e {1e3*(t3-t2):.2f} ms")
# both directions at once
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize(); t0 = time.perf_counter()
with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2): o.copy_(k, non_blocking=True)
torch.cuda.synchronize(); t1 = time.perf_counter()
print(f"bidirectional 2 GB: {1e3*(t1-t0):.2f} ms")
