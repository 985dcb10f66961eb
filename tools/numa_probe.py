"""Host NUMA topology of the GPU box and the PCIe copy bandwidth of pinned
buffers first-touched from each NUMA node (the e2e leg's bound).
python tools/numa_probe.py"""
import glob, os, subprocess, time
import torch

def cpulist(s):
    out = []
    for part in s.strip().split(","):
        if not part:
            continue
        a, _, b = part.partition("-")
        out += list(range(int(a), int(b or a) + 1))
    return out

nodes = {}
for p in sorted(glob.glob("/sys/devices/system/node/node[0-9]*")):
    nodes[int(p.rsplit("node", 1)[1])] = cpulist(open(p + "/cpulist").read())
print("numa nodes:", {k: (v[0], v[-1], len(v)) for k, v in nodes.items()})
print("process affinity:", len(os.sched_getaffinity(0)), "cpus")
bus = torch.cuda.get_device_properties(0).pci_bus_id if hasattr(torch.cuda.get_device_properties(0), "pci_bus_id") else None
try:
    q = subprocess.run(["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader"], capture_output=True, text=True).stdout.split()
    print("nvidia-smi bus ids:", q)
    for b in q:
        b2 = b.lower()[4:] if len(b) > 12 else b.lower()
        for cand in glob.glob("/sys/bus/pci/devices/*"):
            if cand.endswith(b2[-7:]):
                print(" ", b, "numa_node", open(cand + "/numa_node").read().strip(),
                      "local_cpulist", open(cand + "/local_cpulist").read().strip())
except Exception as e:  # noqa: BLE001
    print("bus probe failed:", e)
print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout[:1500])

n = 1 << 28
d_in = torch.empty(n, dtype=torch.uint32, device="cuda")
d_out = torch.zeros(n, dtype=torch.uint32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
orig = os.sched_getaffinity(0)

def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best

for node, cpus in nodes.items():
    cpus = [c for c in cpus if c in orig]
    if not cpus:
        continue
    os.sched_setaffinity(0, cpus)
    # fresh host buffers, first-touched on this node (numpy + cudaHostRegister,
    # so the caching host allocator cannot hand back another node's pages)
    import numpy as np
    a = np.ones(n, dtype=np.uint32); b = np.zeros(n, dtype=np.uint32)
    ha = torch.from_numpy(a); hb = torch.from_numpy(b)
    rt = torch.cuda.cudart()
    rt.cudaHostRegister(ha.data_ptr(), n * 4, 0); rt.cudaHostRegister(hb.data_ptr(), n * 4, 0)
    h2d = timed(lambda: d_in.copy_(ha, non_blocking=True))
    d2h = timed(lambda: hb.copy_(d_out, non_blocking=True))
    def both():
        with torch.cuda.stream(s1): d_in.copy_(ha, non_blocking=True)
        with torch.cuda.stream(s2): hb.copy_(d_out, non_blocking=True)
    dup = timed(both)
    print(f"node {node} ({len(cpus)} cpus): H2D {n*4/h2d/1e9:.1f} GB/s  D2H {n*4/d2h/1e9:.1f} GB/s  "
          f"duplex {2*n*4/dup/1e9:.1f} GB/s ({dup*1e3:.1f} ms for 1 GiB each way)")
    rt.cudaHostUnregister(ha.data_ptr()); rt.cudaHostUnregister(hb.data_ptr())
    del a, b, ha, hb
os.sched_setaffinity(0, orig)
