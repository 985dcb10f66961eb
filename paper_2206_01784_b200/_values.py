"""Value payloads of any width.

The reference reorders values of any numpy dtype (binning.py:301-304; the
scatter kernels move whole elements, _kernels.py:85-128).  Widths of 1, 2, 4
and 8 bytes ride through the binning passes; any other width (complex128,
structured or byte-string dtypes) travels as a 4- or 8-byte index payload and
is gathered once at the end by the os_gather_rows kernel.
"""

from __future__ import annotations

import numpy as np

from . import _native
from ._device import from_device, is_tensor


def _val_bytes(values) -> int:
    """Value width in bytes.  Widths 1, 2, 4 and 8 ride through the passes
    themselves; any other width (complex128, structured or byte-string
    dtypes: the reference reorders values of any dtype, binning.py:301-304)
    travels as a 4- or 8-byte index payload and is gathered once at the end
    (os_gather_rows)."""
    if values is None:
        return 0
    vb = values.element_size() if is_tensor(values) else values.dtype.itemsize
    if vb <= 0:
        raise ValueError("values must have a non-zero element size")
    return vb


def _payload_width(vb: int) -> bool:
    return vb in (1, 2, 4, 8)


def _index_payload(n: int, device):
    """arange(n) as the u32 (or, past 2^32 elements, u64) index payload."""
    import torch

    if n < (1 << 32):
        return torch.arange(n, dtype=torch.int64, device=device).to(torch.int32).view(torch.uint32), 4
    return torch.arange(n, dtype=torch.int64, device=device).view(torch.uint64), 8


def _value_rows(values, device):
    """Device byte tensor of shape (n, width) holding `values` (any dtype)."""
    import torch

    if is_tensor(values):
        t = values.contiguous().to(device)
        return t.view(torch.uint8).reshape(t.numel(), -1) if t.numel() else \
            torch.empty((0, t.element_size()), dtype=torch.uint8, device=device)
    arr = np.ascontiguousarray(values)
    rows = arr.view(np.uint8).reshape(arr.size, arr.dtype.itemsize)
    return torch.from_numpy(rows).to(device)


def _gather_rows(rows, index, index_bytes: int, stream=None):
    """rows[index] on the device through os_gather_rows (a fresh tensor)."""
    import torch

    out = torch.empty_like(rows)
    n, width = rows.shape
    _native.check(
        _native.load().os_gather_rows(_native.ptr(rows), _native.ptr(index), index_bytes,
                                      _native.ptr(out), n, width,
                                      _native.stream_handle(stream)),
        "gather_rows",
    )
    return out


def _rows_as(rows, like, to_numpy: bool):
    """Gathered byte rows back in the container and dtype of `like`."""
    import torch

    if is_tensor(like):
        return rows.reshape(-1).view(like.dtype).reshape(like.shape)
    host = from_device(rows, True)
    return np.ascontiguousarray(host).view(np.asarray(like).dtype).reshape(np.asarray(like).shape)
