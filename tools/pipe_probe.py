"""SortPipeline depth sweep and raw PCIe copy bandwidths (H2D, D2H, both at
once) for 1 GiB of u32 keys.  python tools/pipe_probe.py"""
import sys, time, torch
sys.path.insert(0, "/root/repo")
from paper_2206_01784_b200 import SortPipeline, KeyGenSpec, generate_keys
n = 1 << 28
keys_h = generate_keys(KeyGenSpec(q=1, seed=0, n=n), device="cuda").cpu().pin_memory()
for depth in (2, 3, 4):
    pipe = SortPipeline(n, torch.uint32, depth=depth)
    outs = [torch.empty(n, dtype=torch.uint32, pin_memory=True) for _ in range(depth)]
    for j in range(2 * depth):  # every slot's graph captured before timing
        pipe.submit(keys_h, outs[j % depth])
    pipe.synchronize()
    steps = 12
    t0 = time.perf_counter()
    for j in range(steps):
        pipe.submit(keys_h, outs[j % depth])
    pipe.synchronize()
    dt = (time.perf_counter() - t0) / steps
    print("depth", depth, "ms/step", round(dt * 1e3, 2), "GKey/s", round(n / dt / 1e9, 2))
    del pipe, outs
    torch.cuda.empty_cache()
# raw copy bandwidths
d = torch.empty(n, dtype=torch.uint32, device="cuda")
torch.cuda.synchronize(); t0 = time.perf_counter(); d.copy_(keys_h, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
print("H2D GB/s", round(n * 4 / (t1 - t0) / 1e9, 1))
o = torch.empty(n, dtype=torch.uint32, pin_memory=True)
torch.cuda.synchronize(); t0 = time.perf_counter(); o.copy_(d, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
print("D2H GB/s", round(n * 4 / (t1 - t0) / 1e9, 1))
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
d2 = torch.empty_like(d)
torch.cuda.synchronize(); t0 = time.perf_counter()
with torch.cuda.stream(s1): d2.copy_(keys_h, non_blocking=True)
with torch.cuda.stream(s2): o.copy_(d, non_blocking=True)
torch.cuda.synchronize(); t1 = time.perf_counter()
print("both directions at once: ms", round((t1 - t0) * 1e3, 1), "aggregate GB/s", round(2 * n * 4 / (t1 - t0) / 1e9, 1))
