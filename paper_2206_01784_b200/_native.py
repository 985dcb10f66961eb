"""ctypes binding of the sm_100a C-ABI library (include/onesweep_b200.h).

The library is built in-tree (``make`` or ``__graft_entry__.build()``) into
``paper_2206_01784_b200/_lib/libonesweep_b200.so``.  There is no fallback: if
the library is missing every entry point raises NativeLibraryMissing, and a
CUDA device is required for any data-moving call.
"""

from __future__ import annotations

import ctypes
import os
import threading

LIB_PATH = os.environ.get(
    "ONESWEEP_B200_LIB",
    os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libonesweep_b200.so"),
)

OS_OK = 0
OS_ERR_ARG = 1
OS_ERR_KEYTYPE = 2
OS_ERR_CUDA = 3
OS_ERR_WORKSPACE = 4

KEY_TYPE_IDS = {"u32": 0, "u64": 1, "i32": 2, "i64": 3, "f32": 4, "f64": 5}
CODEC_NONE, CODEC_SIGNED, CODEC_FLOAT_ENC, CODEC_FLOAT_DEC = 0, 1, 2, 3

# Every symbol declared in include/onesweep_b200.h, with (restype, argtypes).
_vp = ctypes.c_void_p
_sz = ctypes.c_size_t
_i = ctypes.c_int
_u64 = ctypes.c_ulonglong
SIGNATURES = {
    "os_version": (ctypes.c_char_p, []),
    "os_last_error": (ctypes.c_char_p, []),
    "os_max_digit_bits": (_i, []),
    "os_stream_check": (_i, [_vp]),
    "os_tile_capacity": (_i, [_i, _i]),
    "os_encode": (_i, [_vp, _vp, _sz, _i, _vp]),
    "os_decode": (_i, [_vp, _vp, _sz, _i, _vp]),
    "os_gather_rows": (_i, [_vp, _vp, _i, _vp, _sz, _sz, _vp]),
    "os_keygen": (_i, [_vp, _sz, _i, _i, _u64, _u64, _vp]),
    "os_histogram_workspace_bytes": (_sz, []),
    "os_histogram": (_i, [_vp, _sz, _i, _i, _i, _i, _i, _vp, _vp, _vp, _sz, _vp]),
    "os_exclusive_scan": (_i, [_vp, _i, _i, _vp, _vp]),
    "os_partition_status_words": (_sz, [_sz, _i, _i, _sz]),
    "os_partition_workspace_bytes": (_sz, [_sz, _i, _i, _sz]),
    "os_partition_workspace_bytes_kv": (_sz, [_sz, _i, _i, _i, _i, _sz]),
    "os_partition_pass": (_i, [_vp, _vp, _vp, _vp, _sz, _i, _i, _i, _i, _vp, _vp, _i, _i, _i, _sz,
                               _vp, _vp, _sz, _vp, _vp]),
    "os_sort_workspace_bytes": (_sz, [_sz, _i, _i, _i, _i, _i, _i, _sz]),
    "os_sort_route_words": (_i, [_vp, _sz, _i, _i, _i, _i, _i, _i, _sz, _vp, _i, _vp]),
    "os_sort": (_i, [_vp, _vp, _vp, _vp, _sz, _i, _i, _i, _i, _i, _i, _sz, _vp, _sz, _vp, _vp]),
    "os_sort_events": (_i, [_vp, _vp, _vp, _vp, _sz, _i, _i, _i, _i, _i, _i, _sz, _vp, _sz, _vp,
                            ctypes.POINTER(_vp), _i, _vp]),
    "os_debug_trace": (_i, [_vp, _i]),
    "os_msd_histogram": (_i, [_vp, _sz, _i, _i, _i, _vp, _vp]),
    "os_msd_partition_workspace_bytes": (_sz, [_sz]),
    "os_msd_partition": (_i, [_vp, _vp, _vp, _vp, _sz, _i, _i, _i, _i, _vp, _i, _vp, _vp, _sz, _vp]),
    "os_msd_partition_p2p": (_i, [_vp, _vp, _vp, _vp, _sz, _i, _i, _i, _i, _vp, _i, _vp, _vp, _sz, _vp]),
    "os_rts_sort_workspace_bytes": (_sz, [_sz, _i, _i]),
    "os_rts_sort": (_i, [_vp, _vp, _vp, _vp, _sz, _i, _i, _vp, _sz, _vp, _i, _vp]),
    "os_rts_upsweep": (_i, [_vp, _sz, _i, _i, _i, _i, _i, _vp, _vp]),
    "os_rts_prefix_workspace_bytes": (_sz, [_sz, _i]),
    "os_rts_block_prefix": (_i, [_vp, _sz, _i, _vp, _vp, _sz, _vp]),
    "os_rts_downsweep_workspace_bytes": (_sz, []),
    "os_rts_downsweep": (_i, [_vp, _vp, _vp, _vp, _sz, _i, _i, _i, _i, _vp, _i, _i, _i, _vp, _sz, _vp]),
}


class NativeLibraryMissing(RuntimeError):
    """The sm_100a library has not been built; there is no CPU fallback."""


_lock = threading.Lock()
_lib: ctypes.CDLL | None = None


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeLibraryMissing(
                    f"{LIB_PATH} not found: build it with `make` or __graft_entry__.build() "
                    "(the sort has no CPU fallback)"
                )
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


# ONESWEEP_B200_SYNC_CHECK=1: after every successful call, synchronise the
# device and raise on an asynchronous kernel fault at the call that caused it
# (debug mode; calls are otherwise asynchronous on their stream).
SYNC_CHECK = os.environ.get("ONESWEEP_B200_SYNC_CHECK", "0") not in ("", "0")


def check(rc: int, what: str = "") -> None:
    """Map an os_status onto the reference's exception classes."""
    if rc == OS_OK and SYNC_CHECK:
        rc = load().os_stream_check(None)  # NULL stream: legacy default, waits for all
        what = f"{what} (asynchronous)" if what else "asynchronous"
    if rc == OS_OK:
        return
    msg = load().os_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc in (OS_ERR_ARG, OS_ERR_WORKSPACE):
        raise ValueError(text)
    if rc == OS_ERR_KEYTYPE:
        raise KeyError(text)
    raise RuntimeError(text)


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None passes NULL)."""
    return None if t is None else t.data_ptr()


def stream_handle(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
