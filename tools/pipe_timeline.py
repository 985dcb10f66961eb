"""SortPipeline timeline: CUDA events around every upload, sort and download
of a run of 1 GiB steps, to see where the overlap breaks.
python tools/pipe_timeline.py [depth] [warmup_submits]"""
import sys
import time

import torch

sys.path.insert(0, "/root/repo")
from paper_2206_01784_b200 import KeyGenSpec, SortPipeline, generate_keys

depth = int(sys.argv[1]) if len(sys.argv) > 1 else 4
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 2 * depth
n = 1 << 28
keys_h = generate_keys(KeyGenSpec(q=1, seed=0, n=n), device="cuda").cpu().pin_memory()
pipe = SortPipeline(n, torch.uint32, depth=depth)
outs = [torch.empty(n, dtype=torch.uint32, pin_memory=True) for _ in range(depth)]
for j in range(warm):
    pipe.submit(keys_h, outs[j % depth])
pipe.synchronize()

# the same submit sequence with timing events on each stream
ev = lambda: torch.cuda.Event(enable_timing=True)
steps = 24
marks = []
origin = ev()
origin.record(pipe.s_h2d)
t0 = time.perf_counter()
host_submit = []
for j in range(steps):
    slot = pipe.i % pipe.depth
    a, b, c, d, e, f = ev(), ev(), ev(), ev(), ev(), ev()
    if pipe.free[slot] is not None:
        pipe.s_h2d.wait_event(pipe.free[slot])
    a.record(pipe.s_h2d)
    h0 = time.perf_counter()
    # same work as SortPipeline.submit, events interleaved
    with torch.cuda.stream(pipe.s_h2d):
        pipe.in_k[slot].copy_(keys_h, non_blocking=True)
        up = torch.cuda.Event()
        up.record(pipe.s_h2d)
    b.record(pipe.s_h2d)
    pipe.s_sort.wait_event(up)
    c.record(pipe.s_sort)
    pipe.sorter(pipe.in_k[slot], pipe.out_k[slot], stream=pipe.s_sort, stats=False)
    done = torch.cuda.Event()
    done.record(pipe.s_sort)
    d.record(pipe.s_sort)
    pipe.s_d2h.wait_event(done)
    e.record(pipe.s_d2h)
    with torch.cuda.stream(pipe.s_d2h):
        outs[j % depth].copy_(pipe.out_k[slot], non_blocking=True)
        free = torch.cuda.Event()
        free.record(pipe.s_d2h)
    f.record(pipe.s_d2h)
    pipe.free[slot] = free
    pipe.i += 1
    host_submit.append((time.perf_counter() - h0) * 1e3)
    marks.append((a, b, c, d, e, f))
pipe.synchronize()
wall = (time.perf_counter() - t0) * 1e3
print(f"depth {depth} warm {warm}: {wall / steps:.2f} ms/step wall; host submit ms max {max(host_submit):.2f}")
print("step  h2d[start,end]   sort[start,end]   d2h[start,end]  (ms from origin)")
for j, m in enumerate(marks):
    t = [origin.elapsed_time(x) for x in m]
    print(f"{j:3d}  {t[0]:8.1f} {t[1]:8.1f}  {t[2]:8.1f} {t[3]:8.1f}  {t[4]:8.1f} {t[5]:8.1f}   "
          f"h2d {t[1]-t[0]:5.1f} d2h {t[5]-t[4]:5.1f}")
