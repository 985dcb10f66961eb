"""Batch sorting from host memory with the transfers overlapped.

`onesweep_sort` on a host array is synchronous: upload, sort, download, one
after the other, and the two PCIe copies dominate (the sort of 256M keys is
~3 ms, each 1 GiB copy ~20 ms).  A user sorting a stream of host arrays can
instead submit them to a `SortPipeline`: step i's upload, step i-1's sort
and step i-2's download run concurrently on three CUDA streams (PCIe is full
duplex, the copy engines and the SMs are separate), with `depth` device
buffer sets rotating between them.  Every step still moves its input host ->
device and its result device -> host; only the overlap differs.
"""

from __future__ import annotations

from .binning import DeviceSorter


class SortPipeline:
    """Overlapped H2D / sort / D2H of equal-sized host batches.

    submit(keys_host, keys_out_host[, values_host, values_out_host]) enqueues
    one stable sort; host tensors should be pinned for the copies to be
    asynchronous.  synchronize() waits for everything submitted so far."""

    def __init__(self, n: int, key_dtype, val_dtype=None, depth: int = 2, device=None):
        import torch

        self.n = int(n)
        self.device = torch.device(device or "cuda")
        vb = torch.empty(0, dtype=val_dtype).element_size() if val_dtype is not None else 0
        self.sorter = DeviceSorter(self.n, key_dtype, vb, device=self.device)
        self.depth = int(depth)
        mk = lambda dt: [torch.empty(self.n, dtype=dt, device=self.device) for _ in range(self.depth)]
        self.in_k, self.out_k = mk(key_dtype), mk(key_dtype)
        self.in_v = mk(val_dtype) if val_dtype is not None else None
        self.out_v = mk(val_dtype) if val_dtype is not None else None
        self.s_h2d = torch.cuda.Stream(self.device)
        self.s_sort = torch.cuda.Stream(self.device)
        self.s_d2h = torch.cuda.Stream(self.device)
        self.free = [None] * self.depth  # event: the slot's last download is done
        self.i = 0

    def submit(self, keys_host, keys_out_host, values_host=None, values_out_host=None):
        import torch

        slot = self.i % self.depth
        self.i += 1
        has_v = values_host is not None
        if has_v != (self.in_v is not None):
            raise ValueError("values must be given iff the pipeline was built with val_dtype")
        if self.free[slot] is not None:
            self.s_h2d.wait_event(self.free[slot])
        with torch.cuda.stream(self.s_h2d):
            self.in_k[slot].copy_(keys_host, non_blocking=True)
            if has_v:
                self.in_v[slot].copy_(values_host, non_blocking=True)
            up = torch.cuda.Event()
            up.record(self.s_h2d)
        self.s_sort.wait_event(up)
        self.sorter(self.in_k[slot], self.out_k[slot], self.in_v[slot] if has_v else None,
                    self.out_v[slot] if has_v else None, stream=self.s_sort, stats=False)
        done = torch.cuda.Event()
        done.record(self.s_sort)
        self.s_d2h.wait_event(done)
        with torch.cuda.stream(self.s_d2h):
            keys_out_host.copy_(self.out_k[slot], non_blocking=True)
            if has_v:
                values_out_host.copy_(self.out_v[slot], non_blocking=True)
            free = torch.cuda.Event()
            free.record(self.s_d2h)
        self.free[slot] = free

    def synchronize(self):
        for s in (self.s_h2d, self.s_sort, self.s_d2h):
            s.synchronize()
