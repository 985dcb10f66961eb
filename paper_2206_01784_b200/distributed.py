"""Multi-GPU sharded Onesweep: MSD top-digit splitter + all-to-all exchange +
local Onesweep per GPU.  The reference has no multi-GPU path;
this follows the plan there.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).  Rank g
holds a contiguous shard of the global input (rank order = input order).

1. each rank counts the top digit of its encoded keys (os_msd_histogram);
2. all_gather of the G x 256 u64 count table -- every rank then knows every
   (source, bin) count and computes the same plan locally, no second round;
3. plan_split assigns each destination a contiguous range of whole bins
   holding ~N/G keys;
4. os_msd_partition stably partitions the shard into G contiguous send
   segments (one binning pass whose digit is the destination);
5. all_to_all_single exchanges the segments; received data is concatenated in
   source-rank order, so equal keys arrive in (source rank, source position)
   order -- the global input order -- and stability is preserved;
6. a full-width local Onesweep sorts what arrived.

Every rank ends up with a contiguous slice of the global stable order:
concatenating the outputs in rank order equals the stable sort of the
concatenated inputs.  Whole-bin splitting balances uniform keys; under heavy
skew one destination receives the largest bin.

The exchange uses device tensors with NCCL; with any other backend (gloo in
the CPU tests) it is staged through host memory.
"""

from __future__ import annotations

import numpy as np

from . import _native
from ._device import workspace
from .keycodec import spec_for_dtype

SPLIT_DIGIT_BITS = 8


def plan_split(table: np.ndarray, parts: int) -> list[int]:
    """Destination bin boundaries from the all-gathered (G, radix) count table.

    Returns bin_lo of length parts+1 with bin_lo[0] = 0, bin_lo[parts] = radix,
    non-decreasing; destination g receives bins [bin_lo[g], bin_lo[g+1]).
    Boundary g is the bin edge whose prefix count is closest to g*N/parts."""
    table = np.asarray(table, dtype=np.uint64)
    radix = table.shape[1]
    per_bin = table.sum(axis=0, dtype=np.uint64).astype(np.float64)
    before = np.concatenate([[0.0], np.cumsum(per_bin)])  # before[k] = keys in bins < k
    total = before[-1]
    bounds = [0]
    for g in range(1, parts):
        target = total * g / parts
        k = int(np.argmin(np.abs(before - target)))  # first minimiser: the smaller edge
        bounds.append(max(k, bounds[-1]))
    bounds.append(radix)
    return bounds


def exchange_counts(table: np.ndarray, bin_lo: list[int], rank: int) -> tuple[list[int], list[int]]:
    """(send counts per destination, receive counts per source) for `rank`."""
    table = np.asarray(table, dtype=np.uint64)
    parts = len(bin_lo) - 1
    send = [int(table[rank, bin_lo[g]:bin_lo[g + 1]].sum()) for g in range(parts)]
    recv = [int(table[s, bin_lo[rank]:bin_lo[rank + 1]].sum()) for s in range(table.shape[0])]
    return send, recv


class DeviceOps:
    """The three device steps, through the C ABI."""

    def top_histogram(self, keys, spec, digit_bits: int):
        import torch

        hist = torch.empty(1 << digit_bits, dtype=torch.uint64, device=keys.device)
        _native.check(
            _native.load().os_msd_histogram(_native.ptr(keys), keys.numel(), spec.type_id, digit_bits,
                                            spec.bits, _native.ptr(hist), _native.stream_handle()),
            "msd_histogram",
        )
        return hist

    def partition(self, keys, values, spec, digit_bits: int, bin_lo: list[int], send: list[int]):
        import torch

        dev = keys.device
        parts = len(bin_lo) - 1
        lo = torch.tensor(bin_lo, dtype=torch.int32, device=dev)
        seg = torch.tensor(np.concatenate([[0], np.cumsum(send)[:-1]]).astype(np.int64),
                           dtype=torch.int64, device=dev)
        out_k = torch.empty_like(keys)
        out_v = torch.empty_like(values) if values is not None else None
        L = _native.load()
        ws = workspace(L.os_msd_partition_workspace_bytes(keys.numel()), dev)
        vb = 0 if values is None else values.element_size()
        _native.check(
            L.os_msd_partition(_native.ptr(keys), _native.ptr(out_k), _native.ptr(values),
                               _native.ptr(out_v), keys.numel(), spec.type_id, vb, digit_bits,
                               spec.bits, _native.ptr(lo), parts, _native.ptr(seg),
                               _native.ptr(ws), ws.numel(), _native.stream_handle()),
            "msd_partition",
        )
        return out_k, out_v

    def local_sort(self, keys, values):
        from .binning import onesweep_sort

        return onesweep_sort(keys, values) if values is not None else (onesweep_sort(keys), None)


def _all_to_all(t, send: list[int], recv: list[int], group):
    """Variable all-to-all of a 1-D tensor; bytes on the wire, any dtype."""
    import torch
    import torch.distributed as dist

    es = t.element_size()
    backend = dist.get_backend(group)
    src = t.contiguous().view(torch.uint8)
    if backend != "nccl":
        src = src.cpu()
    out = torch.empty(sum(recv) * es, dtype=torch.uint8, device=src.device)
    dist.all_to_all_single(out, src, [r * es for r in recv], [s * es for s in send], group=group)
    if out.device != t.device:
        out = out.to(t.device)
    return out.view(t.dtype)


def sharded_sort(keys, values=None, group=None, *, ops=None, digit_bits: int = SPLIT_DIGIT_BITS,
                 return_plan: bool = False):
    """Stable sort of the global array whose rank-order concatenation is
    `keys` over all ranks of `group`.  Returns this rank's contiguous slice
    of the sorted output (and values)."""
    import torch
    import torch.distributed as dist

    ops = ops or DeviceOps()
    spec = spec_for_dtype(keys.dtype)
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if values is not None and values.shape != keys.shape:
        raise ValueError("values must have the same length as keys")

    hist = ops.top_histogram(keys, spec, digit_bits)
    backend = dist.get_backend(group)
    h64 = hist.view(torch.int64)
    if backend != "nccl":
        h64 = h64.cpu()
    gathered = [torch.empty_like(h64) for _ in range(world)]
    dist.all_gather(gathered, h64, group=group)
    table = torch.stack(gathered).cpu().numpy().view(np.uint64)
    bin_lo = plan_split(table, world)
    send, recv = exchange_counts(table, bin_lo, rank)

    part_k, part_v = ops.partition(keys, values, spec, digit_bits, bin_lo, send)
    recv_k = _all_to_all(part_k, send, recv, group)
    recv_v = _all_to_all(part_v, send, recv, group) if values is not None else None
    out_k, out_v = ops.local_sort(recv_k, recv_v)
    result = out_k if values is None else (out_k, out_v)
    if return_plan:
        return result, {"bin_lo": bin_lo, "send": send, "recv": recv}
    return result


class ShardedSorter:
    """Bench helper: a sharded sort of `n` keys per rank."""

    def __init__(self, n: int, key_dtype, device=None, group=None):
        from .keycodec import radix_plan

        self.n = n
        self.group = group
        self.spec = spec_for_dtype(key_dtype)
        self.local_passes = radix_plan(self.spec.bits, 8).passes
        strips = -(-2 * n // (1 << 28))  # receive side may exceed n under skew
        self.launches_per_step = 1 + 1 + 1 + self.local_passes * strips  # msd hist, map, partition, local

    def __call__(self, keys, values=None):
        return sharded_sort(keys, values, self.group)
