"""Upfront digit histograms and their exclusive sums, on the device.

Mirrors onesweep.histogram (histogram.py:24-99).  `global_histograms` launches
the one-read all-places histogram kernel (csrc/histogram.cu); the last block
to finish also writes the per-place exclusive sums, which
`global_bin_offsets` can reuse or recompute with os_exclusive_scan.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from ._device import as_device, from_device, workspace
from .executor import Executor
from .keycodec import RadixConfig


@dataclass(frozen=True)
class GlobalHistogram:
    """(passes, radix) u64 digit counts (histogram.py:24-36)."""

    counts: object  # numpy array or CUDA tensor

    @property
    def passes(self) -> int:
        return self.counts.shape[0]

    @property
    def radix(self) -> int:
        return self.counts.shape[1]


@dataclass(frozen=True)
class GlobalBinOffsets:
    """(passes, radix) exclusive prefix sums (histogram.py:39-46)."""

    offsets: object

    def row(self, place: int):
        return self.offsets[place]


def _scan_rows(counts_dev, rows: int, radix: int):
    import torch

    out = torch.empty((rows, radix), dtype=torch.uint64, device=counts_dev.device)
    _native.check(
        _native.load().os_exclusive_scan(
            _native.ptr(counts_dev), rows, radix, _native.ptr(out), _native.stream_handle()
        ),
        "exclusive_scan",
    )
    return out


def exclusive_sum(counts):
    """out[0] = 0, out[i] = out[i-1] + in[i-1] (histogram.py:49-54), on the device."""
    import torch

    was_tensor = torch.is_tensor(counts)
    arr = counts if was_tensor else np.asarray(counts)
    if not was_tensor and arr.dtype != np.uint64:
        if arr.dtype.kind in "iu" and arr.size and arr.min() < 0:
            raise ValueError("counts must be non-negative")
        arr = arr.astype(np.uint64)
    dev, was_numpy = as_device(arr)
    if dev.dtype != torch.uint64:
        dev = dev.to(torch.int64).view(torch.uint64)
    shape = dev.shape
    flat = dev.reshape(1, -1)
    out = _scan_rows(flat, 1, flat.shape[1]).reshape(shape)
    return from_device(out, was_numpy)


def global_histograms(encoded, cfg: RadixConfig, executor: Executor | None = None,
                      *, begin_bit: int = 0, end_bit: int | None = None) -> GlobalHistogram:
    """Exact digit counts for every place from one read of each key
    (histogram.py:57-91).  `encoded` holds encoded u32/u64 bits."""
    import torch

    dev, was_numpy = as_device(encoded)
    kb = dev.element_size()
    if kb not in (4, 8) or (kb * 8) != cfg.key_bits:
        raise ValueError(f"config is for {cfg.key_bits}-bit keys but got {kb * 8}-bit data")
    end_bit = cfg.key_bits if end_bit is None else end_bit
    passes = -(-(end_bit - begin_bit) // cfg.digit_bits)
    hist = torch.empty((passes, cfg.radix), dtype=torch.uint64, device=dev.device)
    offs = torch.empty_like(hist)
    L = _native.load()
    ws = workspace(L.os_histogram_workspace_bytes(), dev.device)
    n = dev.numel()
    _native.check(
        L.os_histogram(_native.ptr(dev), n, kb, _native.CODEC_NONE, cfg.digit_bits, begin_bit, end_bit,
                       _native.ptr(hist), _native.ptr(offs), _native.ptr(ws), ws.numel(),
                       _native.stream_handle()),
        "histogram",
    )
    if executor is not None and n:
        executor.ledger_record("histogram", "element_reads", n)
    result = GlobalHistogram(from_device(hist, was_numpy))
    # remember the fused scan so global_bin_offsets need not relaunch
    object.__setattr__(result, "_offsets", offs if not was_numpy else None)
    return result


def global_bin_offsets(hist: GlobalHistogram) -> GlobalBinOffsets:
    """Per-place exclusive sums (histogram.py:94-99)."""
    import torch

    cached = getattr(hist, "_offsets", None)
    if cached is not None:
        return GlobalBinOffsets(cached)
    dev, was_numpy = as_device(hist.counts)
    if dev.dtype != torch.uint64:
        dev = dev.to(torch.int64).view(torch.uint64)
    out = _scan_rows(dev.contiguous(), dev.shape[0], dev.shape[1])
    return GlobalBinOffsets(from_device(out, was_numpy))
