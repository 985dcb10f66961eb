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

import numpy as np

from . import _native
from ._device import as_device, from_device, is_tensor, launch_on, workspace
from .executor import Executor
from .keycodec import radix_plan, spec_for_dtype


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
    dv = as_device(values)[0] if values is not None else None
    vb = 0 if values is None else dv.element_size()
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
    return sk, from_device(ov, to_numpy and not is_tensor(values))


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
    dv, _ = as_device(np.asarray(values) if vnp else values)
    return sk, from_device(_take(dv, order), vnp)


def _take(t, order):
    """t[order] by bit pattern (CUDA has no gather for the unsigned dtypes)."""
    import torch

    signed = {1: torch.int8, 2: torch.int16, 4: torch.int32, 8: torch.int64}[t.element_size()]
    return t.view(signed)[order].view(t.dtype)
