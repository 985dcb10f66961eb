"""Seeded random sweep over the drop-in's input space, bit-exact against the
CPU oracle's stable sort on the encoded (begin, end) bit range
(oracle.stable_sort_bits, the reference's baseline.py:27-34 ordering
generalised; its twiddle follows keycodec.py).

Each case draws a key dtype, a size (edge sizes around warps and tiles, and
random sizes up to a few million), a key distribution (uniform, narrow ranges
that make the device skip places, few distinct values, presorted, reversed,
all-equal, raw float bit patterns with NaNs / infinities / signed zeros), a
value payload (none, 1 to 16 bytes, structured and byte-string rows), a bit
range, a digit width and tile size, and host (numpy) or device (torch)
containers.  FUZZ_CASES / FUZZ_SEED scale and reseed the sweep."""

from __future__ import annotations

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = int(os.environ.get("FUZZ_CASES", "160"))
SEED = int(os.environ.get("FUZZ_SEED", "20261017"))

KEY_DTYPES = [np.uint32, np.uint64, np.int32, np.int64, np.float32, np.float64]
VAL_DTYPES = [None, None, np.uint8, np.int16, np.uint32, np.int64, np.float64, np.complex128,
              np.dtype([("a", "<i4"), ("b", "<f8")]), np.dtype("S5")]
TORCH_OK = {np.uint32, np.uint64, np.int32, np.int64, np.float32, np.float64}
TORCH_VAL_OK = {np.uint8, np.int16, np.int64, np.float64}


def _uint(dt):
    return np.uint32 if np.dtype(dt).itemsize == 4 else np.uint64


def _keys(rng, dt, n, dist):
    u = _uint(dt)
    bits = np.dtype(u).itemsize * 8
    raw = rng.integers(0, 2**63, size=n, dtype=np.uint64, endpoint=False)
    raw = (raw << np.uint64(1)) ^ rng.integers(0, 2, size=n, dtype=np.uint64)
    raw = raw.astype(u) if bits == 32 else raw
    if dist == "uniform" or dist == "floatbits":
        k = raw
    elif dist == "narrow":  # a few low bits vary: most places are skipped
        k = raw & u((1 << int(rng.integers(1, 20))) - 1)
    elif dist == "high":  # only the top byte varies
        k = (raw >> u(bits - 8)) << u(bits - 8)
    elif dist == "few":
        k = rng.choice(raw[: max(1, min(n, 5))], size=n) if n else raw
    elif dist == "equal":
        k = np.full(n, raw[0] if n else 0, dtype=u)
    elif dist == "sorted":
        k = np.sort(raw)
    elif dist == "reversed":
        k = np.sort(raw)[::-1].copy()
    else:
        raise AssertionError(dist)
    k = np.ascontiguousarray(k.astype(u))
    if np.dtype(dt).kind == "f" and dist != "floatbits":
        # genuine floats with the special values mixed in
        f = rng.standard_normal(n).astype(dt) * dt(1e3)
        sp = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, -np.nan], dtype=dt)
        m = rng.random(n) < 0.1
        f[m] = rng.choice(sp, size=int(m.sum()))
        return f
    return k.view(dt)


def _values(rng, vdt, n):
    if vdt is None:
        return None
    vdt = np.dtype(vdt)
    b = rng.integers(0, 256, size=n * vdt.itemsize, dtype=np.uint8)
    return b.view(vdt)


def _case(rng, i):
    dt = KEY_DTYPES[int(rng.integers(len(KEY_DTYPES)))]
    kb = np.dtype(dt).itemsize * 8
    edges = [0, 1, 2, 31, 32, 33, 1023, 1024, 4095, 4097, 6143, 8191, 8193, 10239, 10241, 20481]
    r = rng.random()
    if r < 0.3:
        n = edges[int(rng.integers(len(edges)))]
    elif r < 0.9:
        n = int(rng.integers(1, 300_000))
    else:
        n = int(rng.integers(300_000, 3_000_000))
    dists = ["uniform", "narrow", "high", "few", "equal", "sorted", "reversed"]
    if np.dtype(dt).kind == "f":
        dists += ["floatbits", "floatbits"]
    dist = dists[int(rng.integers(len(dists)))]
    vdt = VAL_DTYPES[int(rng.integers(len(VAL_DTYPES)))]
    if rng.random() < 0.7:
        begin, end = 0, kb
    else:
        begin = int(rng.integers(0, kb - 1))
        end = int(rng.integers(begin + 1, kb + 1))
    digit_bits = [8, 8, 8, 8, 4, 6, 7, 11, 16][int(rng.integers(9))]
    tile = [None, None, 64, 1000, 4096, 7777][int(rng.integers(6))]
    strip = [None, None, None, 9000, 65536][int(rng.integers(5))]
    on_device = bool(rng.random() < 0.4) and dt in TORCH_OK and (vdt is None or vdt in TORCH_VAL_OK)
    return dict(i=i, dt=dt, n=n, dist=dist, vdt=vdt, begin=begin, end=end,
                digit_bits=digit_bits, tile=tile, strip=strip, on_device=on_device)


def _cases():
    rng = np.random.default_rng(SEED)
    return [_case(rng, i) for i in range(CASES)]


@pytest.mark.parametrize("case", _cases(), ids=lambda c: f"{c['i']}-{np.dtype(c['dt']).name}-{c['n']}-{c['dist']}")
def test_fuzz(cuda, oracle, case):
    import torch

    from paper_2206_01784_b200 import onesweep_sort, radix_plan

    rng = np.random.default_rng(SEED * 1000 + case["i"])
    dt, n = case["dt"], case["n"]
    keys = _keys(rng, dt, n, case["dist"])
    vals = _values(rng, case["vdt"], n)
    kbits = np.dtype(dt).itemsize * 8
    cfg = None
    if case["digit_bits"] != 8 or case["tile"] is not None or case["strip"] is not None:
        extra = {}
        if case["tile"] is not None:
            extra["tile_size"] = case["tile"]
        if case["strip"] is not None:
            extra["strip_size"] = case["strip"]
        cfg = radix_plan(kbits, case["digit_bits"], **extra)
    want = oracle.stable_sort_bits(keys, vals, case["begin"], case["end"])
    want_k, want_v = (want, None) if vals is None else want
    kw = dict(cfg=cfg, begin_bit=case["begin"], end_bit=case["end"])
    if case["on_device"]:
        tk = torch.from_numpy(keys.view(np.int32 if kbits == 32 else np.int64).copy())
        tk = tk.view(getattr(torch, np.dtype(dt).name)).cuda()
        tv = torch.from_numpy(vals.copy()).cuda() if vals is not None else None
        got = onesweep_sort(tk, tv, **kw)
        got_k, got_v = (got, None) if vals is None else got
        assert got_k.device.type == "cuda"
        got_k = got_k.cpu().view(torch.int32 if kbits == 32 else torch.int64).numpy().view(dt)
        got_v = got_v.cpu().numpy() if got_v is not None else None
    else:
        got = onesweep_sort(keys, vals, **kw)
        got_k, got_v = (got, None) if vals is None else got
        assert isinstance(got_k, np.ndarray) and got_k.dtype == keys.dtype
    u = _uint(dt)
    assert np.array_equal(np.asarray(got_k).view(u), want_k.view(u)), case
    if vals is not None:
        assert got_v.dtype == vals.dtype
        assert np.array_equal(np.ascontiguousarray(got_v).view(np.uint8),
                              np.ascontiguousarray(want_v).view(np.uint8)), case


@pytest.mark.parametrize("case", [c for c in _cases() if c["begin"] == 0 and c["end"] == np.dtype(c["dt"]).itemsize * 8][::4],
                         ids=lambda c: f"{c['i']}-{np.dtype(c['dt']).name}-{c['n']}-{c['dist']}")
def test_fuzz_rts(cuda, oracle, case):
    """The reduce-then-scan comparator (baseline.py:121-173) over the same draws."""
    from paper_2206_01784_b200 import radix_plan, rts_sort

    rng = np.random.default_rng(SEED * 1000 + case["i"])
    dt, n = case["dt"], case["n"]
    keys = _keys(rng, dt, n, case["dist"])
    vals = _values(rng, case["vdt"], n)
    cfg = radix_plan(np.dtype(dt).itemsize * 8, case["digit_bits"])
    want = oracle.stable_sort_bits(keys, vals)
    want_k, want_v = (want, None) if vals is None else want
    got = rts_sort(keys, vals, cfg=cfg)
    got_k, got_v = (got, None) if vals is None else got
    u = _uint(dt)
    assert np.array_equal(got_k.view(u), want_k.view(u)), case
    if vals is not None:
        assert np.array_equal(np.ascontiguousarray(got_v).view(np.uint8),
                              np.ascontiguousarray(want_v).view(np.uint8)), case
