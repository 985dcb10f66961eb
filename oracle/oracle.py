"""TEST INFRASTRUCTURE ONLY -- ctypes front end of the CPU oracle.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this module, and only as the checker or
the CPU baseline.  The product package never imports it.

It wraps oracle/liboracle.so (a C restatement of the reference package
`onesweep`, see onesweep_oracle.c for per-function file:line citations) and
adds numpy restatements for the two semantics the reference does not have:
begin/end-bit sorts and the multi-GPU sharded sort.

Parity of the restatement is pinned by tests/test_oracle.py against
tests/golden/reference_golden.npz, which tests/golden/make_golden.py produced
by running the reference itself.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

KEY_TYPES = {"u32": 0, "u64": 1, "i32": 2, "i64": 3, "f32": 4, "f64": 5}
DTYPE_NAMES = {
    np.dtype(np.uint32): "u32",
    np.dtype(np.uint64): "u64",
    np.dtype(np.int32): "i32",
    np.dtype(np.int64): "i64",
    np.dtype(np.float32): "f32",
    np.dtype(np.float64): "f64",
}

_lib = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        vp, sz, i, u64p = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p
        L.or_encode.argtypes = [vp, vp, sz, i]
        L.or_decode.argtypes = [vp, vp, sz, i]
        L.or_keygen.argtypes = [vp, sz, i, i, ctypes.c_uint64, ctypes.c_uint64]
        L.or_keygen.restype = None
        L.or_exclusive_sum.argtypes = [vp, sz, vp]
        L.or_exclusive_sum.restype = None
        L.or_histogram.argtypes = [vp, sz, i, i, i, i, vp]
        L.or_histogram.restype = None
        L.or_wlms_rank.argtypes = [vp, sz, i, vp, vp]
        L.or_wlms_rank.restype = None
        L.or_partition_pass.argtypes = [vp, vp, vp, vp, sz, i, i, i, i, i, vp, vp, sz, sz, vp,
                                        u64p, u64p, i]
        L.or_sort.argtypes = [vp, vp, vp, vp, sz, i, i, i, i, i, sz, sz, i, u64p, u64p]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def key_type_of(dtype) -> str:
    try:
        return DTYPE_NAMES[np.dtype(dtype)]
    except KeyError:
        raise KeyError(f"unsupported key dtype {np.dtype(dtype)!r}") from None


def uint_view(a: np.ndarray) -> np.ndarray:
    return a.view(np.uint32 if a.dtype.itemsize == 4 else np.uint64)


def encode(keys: np.ndarray) -> np.ndarray:
    keys = np.ascontiguousarray(keys)
    out = np.empty(keys.shape, dtype=np.uint32 if keys.dtype.itemsize == 4 else np.uint64)
    lib().or_encode(_p(keys), _p(out), keys.size, KEY_TYPES[key_type_of(keys.dtype)])
    return out


def decode(enc: np.ndarray, key_type: str) -> np.ndarray:
    enc = np.ascontiguousarray(enc)
    out = np.empty_like(enc)
    lib().or_decode(_p(enc), _p(out), enc.size, KEY_TYPES[key_type])
    dt = {"u32": np.uint32, "u64": np.uint64, "i32": np.int32, "i64": np.int64,
          "f32": np.float32, "f64": np.float64}[key_type]
    return out.view(dt)


def keygen(n: int, q: int, seed: int, key_bits: int = 32, first: int = 0) -> np.ndarray:
    out = np.empty(n, dtype=np.uint32 if key_bits == 32 else np.uint64)
    lib().or_keygen(_p(out), n, key_bits, q, seed & 0xFFFFFFFFFFFFFFFF, first)
    return out


def exclusive_sum(counts: np.ndarray) -> np.ndarray:
    c = np.ascontiguousarray(counts, dtype=np.uint64)
    out = np.empty_like(c)
    lib().or_exclusive_sum(_p(c), c.size, _p(out))
    return out


def histogram(enc: np.ndarray, digit_bits: int, begin_bit: int = 0, end_bit: int | None = None) -> np.ndarray:
    enc = np.ascontiguousarray(enc)
    kbits = enc.dtype.itemsize * 8
    end_bit = kbits if end_bit is None else end_bit
    passes = -(-(end_bit - begin_bit) // digit_bits)
    out = np.empty((passes, 1 << digit_bits), dtype=np.uint64)
    lib().or_histogram(_p(enc), enc.size, enc.dtype.itemsize, digit_bits, begin_bit, end_bit, _p(out))
    return out


def bin_offsets(hist: np.ndarray) -> np.ndarray:
    return np.stack([exclusive_sum(row) for row in hist]) if hist.size else hist.copy()


def wlms_rank(digits: np.ndarray, digit_bits: int):
    d = np.ascontiguousarray(digits, dtype=np.uint32)
    ranks = np.empty(d.size, dtype=np.uint32)
    counts = np.empty(1 << digit_bits, dtype=np.uint32)
    lib().or_wlms_rank(_p(d), d.size, digit_bits, _p(ranks), _p(counts))
    return counts, ranks


def partition_pass(src, dst, shift, digit_bits, base, src_vals=None, dst_vals=None,
                   tile=4096, strip=1 << 28, width=None, threads=1, want_status=False):
    """Returns (carry u64[radix], fast_tiles, status words or None)."""
    radix = 1 << digit_bits
    width = digit_bits if width is None else width
    base = np.ascontiguousarray(base, dtype=np.uint64)
    carry = np.empty(radix, dtype=np.uint64)
    n = src.size
    tiles_total = sum(-(-min(strip, n - lo) // tile) for lo in range(0, n, strip))
    status = np.zeros(tiles_total * radix, dtype=np.uint32) if want_status else None
    fast = ctypes.c_uint64(0)
    ops = ctypes.c_uint64(0)
    vb = 0 if src_vals is None else src_vals.dtype.itemsize
    lib().or_partition_pass(_p(src), _p(dst), _p(src_vals), _p(dst_vals), n, src.dtype.itemsize, vb,
                            shift, digit_bits, width, _p(base), _p(carry), tile, strip, _p(status),
                            ctypes.byref(fast), ctypes.byref(ops), threads)
    return carry, fast.value, status


def sort(keys: np.ndarray, values: np.ndarray | None = None, digit_bits: int = 8, begin_bit: int = 0,
         end_bit: int | None = None, tile: int = 4096, strip: int = 1 << 28, threads: int = 1):
    """The reference's onesweep_sort restated in C (plus begin/end bits)."""
    keys = np.ascontiguousarray(keys)
    kt = key_type_of(keys.dtype)
    end_bit = keys.dtype.itemsize * 8 if end_bit is None else end_bit
    out = np.empty_like(keys)
    vout = None
    vb = 0
    if values is not None:
        values = np.ascontiguousarray(values)
        vout = np.empty_like(values)
        vb = values.dtype.itemsize
    fast = ctypes.c_uint64(0)
    ops = ctypes.c_uint64(0)
    rc = lib().or_sort(_p(keys), _p(out), _p(values), _p(vout), keys.size, KEY_TYPES[kt], vb,
                       digit_bits, begin_bit, end_bit, tile, strip, threads, ctypes.byref(fast),
                       ctypes.byref(ops))
    if rc:
        raise RuntimeError(f"or_sort failed with {rc}")
    sort.last_fast_path_tiles = fast.value
    return out if values is None else (out, vout)


sort.last_fast_path_tiles = 0


# -- numpy restatements for semantics the reference lacks ------------------


def stable_sort_bits(keys: np.ndarray, values=None, begin_bit: int = 0, end_bit: int | None = None):
    """argsort(((enc >> b) & mask), stable) -- begin/end-bit oracle
    (CUB convention; baseline.py:27-34 generalised)."""
    enc = encode(keys)
    kbits = enc.dtype.itemsize * 8
    end_bit = kbits if end_bit is None else end_bit
    width = end_bit - begin_bit
    mask = (1 << width) - 1
    sub = (enc >> enc.dtype.type(begin_bit)) & enc.dtype.type(mask)
    order = np.argsort(sub, kind="stable")
    if values is None:
        return keys[order]
    return keys[order], np.asarray(values)[order]


def sharded_sort(shards: list[np.ndarray], values: list[np.ndarray] | None = None):
    """Oracle for the multi-GPU sort: stable sort of concat(shards in rank
    order); returns the full sorted keys (and values)."""
    keys = np.concatenate(shards)
    order = np.argsort(encode(keys), kind="stable")
    if values is None:
        return keys[order]
    return keys[order], np.concatenate(values)[order]
