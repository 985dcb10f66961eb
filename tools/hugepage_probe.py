"""Does the page size behind pinned host buffers change PCIe copy rates?
(The GPU box is a KVM guest: DMA goes through the IOMMU, and 4 KiB pages
mean many more IOTLB entries than 2 MiB pages.)  Times 1 GiB H2D, D2H and
both at once for cudaHostAlloc'd buffers (torch pin_memory) and for
mmap'd buffers advised MADV_HUGEPAGE / MADV_NOHUGEPAGE and then
cudaHostRegister'd.  python tools/hugepage_probe.py"""
import ctypes
import mmap
import time

import numpy as np
import torch

print("THP enabled:", open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())
print("THP defrag:", open("/sys/kernel/mm/transparent_hugepage/defrag").read().strip())
rt = ctypes.CDLL("libcudart.so.12")
n = 1 << 28
nb = n * 4
d_in = torch.empty(n, dtype=torch.uint32, device="cuda")
d_out = torch.ones(n, dtype=torch.uint32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def anon_huge():
    for line in open("/proc/self/smaps_rollup"):
        if line.startswith("AnonHugePages"):
            return line.split()[1] + " kB"
    return "?"


def rates(hin, hout):
    def timed(fn):
        best = 1e9
        for _ in range(3):
            torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        return best
    h2d = timed(lambda: d_in.copy_(hin, non_blocking=True))
    d2h = timed(lambda: hout.copy_(d_out, non_blocking=True))

    def both():
        with torch.cuda.stream(s1):
            d_in.copy_(hin, non_blocking=True)
        with torch.cuda.stream(s2):
            hout.copy_(d_out, non_blocking=True)
    dup = timed(both)
    return f"H2D {nb / h2d / 1e9:5.1f} GB/s  D2H {nb / d2h / 1e9:5.1f} GB/s  both {dup * 1e3:5.1f} ms"


def mapped(advice):
    mm = mmap.mmap(-1, nb + (2 << 20), flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    mm.madvise(advice)
    a = np.frombuffer(mm, dtype=np.uint8)
    off = (-a.ctypes.data) % (2 << 20)  # 2 MiB aligned start
    a = a[off:off + nb].view(np.uint32)
    a[:] = 1  # first touch
    t = torch.from_numpy(a)
    assert rt.cudaHostRegister(ctypes.c_void_p(t.data_ptr()), ctypes.c_size_t(nb), 0) == 0
    return mm, t


for rep in range(2):
    hin = torch.empty(n, dtype=torch.uint32, pin_memory=True); hin.fill_(1)
    hout = torch.empty(n, dtype=torch.uint32, pin_memory=True); hout.fill_(0)
    print(f"[{rep}] cudaHostAlloc (torch pin_memory):   {rates(hin, hout)}")
    del hin, hout
    for name, adv in (("MADV_HUGEPAGE", mmap.MADV_HUGEPAGE), ("MADV_NOHUGEPAGE", mmap.MADV_NOHUGEPAGE)):
        m1, hin = mapped(adv)
        m2, hout = mapped(adv)
        print(f"[{rep}] mmap + {name:15s} + register: {rates(hin, hout)}   AnonHugePages {anon_huge()}")
        rt.cudaHostUnregister(ctypes.c_void_p(hin.data_ptr())); rt.cudaHostUnregister(ctypes.c_void_p(hout.data_ptr()))
        del hin, hout
        m1.close(); m2.close()
