"""Reduce-then-scan comparator sort on the device (the ablation of SURVEY.md
8f rank 4).

`rts_sort` mirrors the reference's `rts_sort(keys, values=None, cfg=None,
executor=None)` (baseline.py:121-173): same output contract as
`onesweep_sort`, but every digit place costs 3n element transfers -- an
upsweep of per-tile histograms (baseline.py:55-73), a digit-major prefix over
that table (baseline.py:76-84) and a downsweep scatter (baseline.py:87-118)
-- where Onesweep's chained scan needs 2n.  On the device the downsweep is the
Onesweep binning kernel with its look-back replaced by a read of the prefix
table (os_rts_sort), so timing the two sorts isolates exactly what the single
pass saves.

`oracle_stable_sort` is the reference's comparator API (baseline.py:27-34:
stable argsort of the encoded keys + gather), kept for drop-in callers such as
the CLI's `verify`.  It is deliberately *not* Onesweep: an independent order
from torch's stable device sort of the encoded keys, so checking a Onesweep
result against it is a real check.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from ._device import as_device, from_device, is_tensor, launch_on, workspace
from ._values import _gather_rows, _index_payload, _payload_width, _rows_as, _val_bytes, _value_rows
from .executor import Executor
from .keycodec import MAX_DEVICE_DIGIT_BITS, radix_plan, spec_for_dtype


class DeviceRtsSorter:
    """Pre-planned device rts sort of n keys (optionally with values)."""

    def __init__(self, n: int, key_dtype, val_bytes: int = 0, device=None):
        import torch

        self.spec = spec_for_dtype(key_dtype)
        self.n = int(n)
        self.val_bytes = int(val_bytes)
        self.passes = self.spec.bits // 8
        L = _native.load()
        nbytes = L.os_rts_sort_workspace_bytes(self.n, self.spec.type_id, self.val_bytes)
        if self.n > 1 and nbytes == 0:
            raise ValueError("invalid rts sort parameters: " + L.os_last_error().decode())
        self.device = torch.device(device or "cuda")
        self.ws = workspace(nbytes, self.device)

    def __call__(self, keys, keys_out, values=None, values_out=None, stream=None, events=None):
        handles = None
        if events is not None:
            handles = (_native._vp * len(events))(*[e.cuda_event for e in events])
        _native.check(
            _native.load().os_rts_sort(
                _native.ptr(keys), _native.ptr(keys_out), _native.ptr(values),
                _native.ptr(values_out), self.n, self.spec.type_id, self.val_bytes,
                _native.ptr(self.ws), self.ws.numel(), handles,
                len(events) if events is not None else 0, _native.stream_handle(stream)),
            "rts_sort",
        )
        return keys_out if values is None else (keys_out, values_out)


def rts_sort(keys, values=None, cfg=None, executor: Executor | None = None):
    """Reduce-then-scan LSD radix sort (baseline.py:121-173): stable, ascending,
    inputs untouched, same container type out as in.  8-bit places; a
    configured digit width > 8 sorts identically (the stable order is unique)."""
    import torch

    to_numpy = not is_tensor(keys)
    if to_numpy:
        keys = np.asarray(keys)
    spec = spec_for_dtype(keys.dtype)  # KeyError for unsupported dtypes
    if cfg is None:
        cfg = radix_plan(spec.bits, 8)
    elif cfg.key_bits != spec.bits:
        raise ValueError(
            f"config is for {cfg.key_bits}-bit keys but got {spec.bits}-bit {spec.name}"
        )
    if executor is None:
        executor = Executor()
    if values is not None:
        if not is_tensor(values):
            values = np.asarray(values)
        if tuple(values.shape) != tuple(keys.shape):
            raise ValueError("values must have the same length as keys")
    n = keys.numel() if is_tensor(keys) else int(keys.size)
    if n <= 1:  # baseline.py:151-153
        sk = keys.clone() if is_tensor(keys) else keys.copy()
        if values is None:
            return sk
        return sk, (values.clone() if is_tensor(values) else values.copy())
    dk, _ = as_device(keys)
    vb = _val_bytes(values)
    wide = values is not None and not _payload_width(vb)
    if wide:  # values wider than 8 bytes ride as an index payload
        dv, vb = _index_payload(n, dk.device)
    else:
        dv = as_device(values)[0] if values is not None else None
    ok = torch.empty_like(dk)
    ov = torch.empty_like(dv) if dv is not None else None
    sorter = DeviceRtsSorter(n, dk.dtype, vb, device=dk.device)
    launch_on(executor.stream, (dk, ok, dv, ov, sorter.ws),
              lambda s: sorter(dk, ok, dv, ov, stream=s))
    # the configured plan's algorithmic traffic, 3n per place (baseline.py:70,
    # 116-117); the device always runs 8-bit places (same output)
    for _ in range(cfg.passes):
        executor.ledger_record("upsweep", "element_reads", n)
        executor.ledger_record("downsweep", "element_reads", n)
        executor.ledger_record("downsweep", "element_writes", n)
    executor.device_element_ops += 3 * sorter.passes * n
    sk = from_device(ok, to_numpy)
    if values is None:
        return sk
    if wide:
        return sk, _rows_as(_gather_rows(_value_rows(values, dk.device), ov, vb), values, to_numpy)
    return sk, from_device(ov, to_numpy and not is_tensor(values))


@dataclass(frozen=True)
class BlockHistogramTable:
    """(tiles, radix) per-tile digit counts of one digit place
    (baseline.py:37-48)."""

    counts: np.ndarray

    @property
    def tiles(self) -> int:
        return self.counts.shape[0]

    @property
    def radix(self) -> int:
        return self.counts.shape[1]


def _rts_width(cfg) -> int:
    if cfg.digit_bits > MAX_DEVICE_DIGIT_BITS:
        raise ValueError(f"the device rts passes run digit widths <= {MAX_DEVICE_DIGIT_BITS}, "
                         f"got {cfg.digit_bits}")
    return cfg.digit_bits


def rts_upsweep(encoded, place: int, cfg, executor: Executor | None = None) -> BlockHistogramTable:
    """First data pass of the comparator (baseline.py:55-73): per-tile digit
    counts of already-encoded keys, n element reads, on the device
    (csrc/rts.cu rts_upsweep_kernel via os_rts_upsweep)."""
    import torch

    executor = executor or Executor()
    width = _rts_width(cfg)
    dk, _ = as_device(encoded)
    n = dk.numel()
    tiles = -(-n // cfg.tile_size)
    counts = torch.zeros(max(tiles * cfg.radix, 1), dtype=torch.int32, device=dk.device)
    L = _native.load()
    launch_on(executor.stream, (dk, counts), lambda s: _native.check(
        L.os_rts_upsweep(_native.ptr(dk), n, dk.element_size(), _native.CODEC_NONE,
                         cfg.digit_shift(place), width, cfg.tile_size, _native.ptr(counts),
                         _native.stream_handle(s)), "rts_upsweep"))
    if n:
        executor.ledger_record("upsweep", "element_reads", n)
    table = counts[: tiles * cfg.radix].view(torch.uint32).cpu().numpy().astype(np.int64)
    return BlockHistogramTable(table.reshape(tiles, cfg.radix))


def rts_block_prefix(table: BlockHistogramTable) -> np.ndarray:
    """Exclusive prefix over the digit-major linearisation of the table
    (baseline.py:76-84): entry [tile, digit] is the absolute output start of
    that tile's digit run.  Device scan (os_rts_block_prefix)."""
    import torch

    counts = np.asarray(table.counts)
    tiles, radix = counts.shape
    if tiles == 0:
        return np.zeros((0, radix), dtype=np.int64)
    if counts.min(initial=0) < 0 or counts.max(initial=0) >= 1 << 32:
        raise ValueError("tile counts must fit in 32 bits")
    dc, _ = as_device(np.ascontiguousarray(counts.astype(np.uint32)))
    out = torch.empty(tiles * radix, dtype=torch.int64, device=dc.device)
    L = _native.load()
    ws = workspace(L.os_rts_prefix_workspace_bytes(tiles, radix), dc.device)
    _native.check(L.os_rts_block_prefix(_native.ptr(dc), tiles, radix, _native.ptr(out), _native.ptr(ws),
                                        ws.numel(), _native.stream_handle(None)), "rts_block_prefix")
    return out.cpu().numpy().reshape(tiles, radix)


def rts_downsweep(encoded, place: int, offsets, out, cfg, executor: Executor | None = None,
                  values=None, out_values=None) -> None:
    """Second data pass (baseline.py:87-118): stable scatter of every tile
    seeded by its row of `offsets` (n reads + n writes).  The device kernel is
    the Onesweep binning kernel with the look-back replaced by the table
    (os_rts_downsweep).  Numpy outputs are updated in place."""
    import torch

    executor = executor or Executor()
    width = _rts_width(cfg)
    dk, _ = as_device(encoded)
    n = dk.numel()
    if n == 0:
        return
    kb = dk.element_size()
    off = offsets if is_tensor(offsets) else np.ascontiguousarray(np.asarray(offsets, dtype=np.int64))
    doff, _ = as_device(off)
    if doff.numel() != (-(-n // cfg.tile_size)) * cfg.radix:
        raise ValueError("offsets must have one row of radix run starts per tile")
    ok, _ = as_device(out)
    dv = ov = None
    vb = 0
    if values is not None:
        dv, _ = as_device(values)
        ov, _ = as_device(out_values)
        vb = dv.element_size()
    L = _native.load()
    ws = workspace(L.os_rts_downsweep_workspace_bytes(), dk.device)
    launch_on(executor.stream, (dk, doff, ok, dv, ov, ws), lambda s: _native.check(
        L.os_rts_downsweep(_native.ptr(dk), _native.ptr(ok), _native.ptr(dv), _native.ptr(ov), n, kb, vb,
                           cfg.digit_shift(place), width, _native.ptr(doff), cfg.tile_size,
                           _native.CODEC_NONE, _native.CODEC_NONE, _native.ptr(ws), ws.numel(),
                           _native.stream_handle(s)), "rts_downsweep"))
    executor.ledger_record("downsweep", "element_reads", n)
    executor.ledger_record("downsweep", "element_writes", n)
    for dst, dev in ((out, ok), (out_values, ov)):
        if dst is None:
            continue
        if is_tensor(dst):
            if dst.data_ptr() != dev.data_ptr():
                dst.copy_(dev)
        else:
            np.copyto(dst, from_device(dev, True).view(np.asarray(dst).dtype))


def oracle_stable_sort(keys, values=None):
    """Stable ascending sort by encoded key order (baseline.py:27-34), by an
    independent path: torch.sort(stable=True) of the encoded keys widened to
    int64 in the same order, then a gather.  Same container type out as in."""
    import torch

    from .keycodec import encode_array

    to_numpy = not is_tensor(keys)
    if to_numpy:
        keys = np.asarray(keys)
    spec_for_dtype(keys.dtype)  # KeyError for unsupported dtypes
    dk, _ = as_device(keys)
    enc = encode_array(dk)
    if enc.element_size() == 4:
        order_key = enc.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    else:  # unsigned 64-bit order as signed: flip the top bit
        order_key = enc.view(torch.int64) ^ (-(1 << 63))
    order = torch.sort(order_key, stable=True).indices
    sk = from_device(_take(dk, order), to_numpy)
    if values is None:
        return sk
    vnp = not is_tensor(values)
    if not _payload_width(_val_bytes(values)):  # e.g. complex128, structured dtypes
        rows = _gather_rows(_value_rows(values, dk.device), order, 8)
        return sk, _rows_as(rows, values, vnp)
    dv, _ = as_device(np.asarray(values) if vnp else values)
    return sk, from_device(_take(dv, order), vnp)


def _take(t, order):
    """t[order] by bit pattern (CUDA has no gather for the unsigned dtypes)."""
    import torch

    signed = {1: torch.int8, 2: torch.int16, 4: torch.int32, 8: torch.int64}[t.element_size()]
    return t.view(signed)[order].view(t.dtype)
