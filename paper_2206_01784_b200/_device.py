"""Buffer plumbing: numpy <-> CUDA tensors, workspace tensors.

torch is used only for device memory, streams and host<->device copies; every
byte of sort work runs in the sm_100a library.
"""

from __future__ import annotations

import numpy as np

_NP_TO_TORCH = None


def _np_to_torch_dtype(dt):
    import torch

    global _NP_TO_TORCH
    if _NP_TO_TORCH is None:
        _NP_TO_TORCH = {
            np.dtype(np.uint8): torch.uint8,
            np.dtype(np.int8): torch.int8,
            np.dtype(np.uint16): torch.uint16,
            np.dtype(np.int16): torch.int16,
            np.dtype(np.float16): torch.float16,
            np.dtype(np.uint32): torch.uint32,
            np.dtype(np.int32): torch.int32,
            np.dtype(np.float32): torch.float32,
            np.dtype(np.uint64): torch.uint64,
            np.dtype(np.int64): torch.int64,
            np.dtype(np.float64): torch.float64,
            np.dtype(np.bool_): torch.bool,
        }
    return _NP_TO_TORCH[np.dtype(dt)]


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("onesweep_b200 needs a CUDA device (sm_100a); there is no CPU path")
    return torch


def is_tensor(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return torch.is_tensor(x)


def as_device(x, device=None):
    """Return (contiguous CUDA tensor, was_numpy)."""
    torch = require_cuda()
    if torch.is_tensor(x):
        if not x.is_cuda:
            return x.contiguous().to(device or "cuda", non_blocking=False), False
        return x.contiguous(), False
    arr = np.ascontiguousarray(np.asarray(x))
    t = torch.from_numpy(arr) if arr.size else torch.empty(0, dtype=_np_to_torch_dtype(arr.dtype))
    return t.to(device or "cuda"), True


def from_device(t, to_numpy: bool):
    """Device tensor -> numpy.  Large results land in pinned (page-locked)
    host memory from torch's caching host allocator, so the D2H copy runs at
    full PCIe/NVLink-C2C rate."""
    if not to_numpy:
        return t
    import torch

    if t.numel() * t.element_size() >= (1 << 20):
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return h.numpy()
    return t.cpu().numpy()


def workspace(nbytes: int, device):
    import torch

    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)


def launch_on(stream, tensors, launch) -> None:
    """Run `launch(stream)` ordered against the current stream.

    The inputs, outputs and workspace in `tensors` were allocated (and the
    inputs uploaded) on the current stream.  When the caller names another
    stream, that stream first waits for the current one, the tensors are
    marked as used on it (so the caching allocator cannot hand them out while
    the kernels still run), and the current stream then waits for the sort,
    so a later read or download on it sees the result."""
    import torch

    cur = torch.cuda.current_stream()
    if stream is None or stream == cur:
        launch(cur)
        return
    stream.wait_stream(cur)
    launch(stream)
    for t in tensors:
        if t is not None:
            t.record_stream(stream)
    cur.wait_stream(stream)
