"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba \
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Writes tests/golden/reference_golden.npz.  The fixtures pin the CPU oracle
(oracle/) and, transitively, the GPU path: every array in the file is an
output of /root/reference/pkg/src/onesweep on the stored inputs.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.dont_write_bytecode = True
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba")
REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from onesweep import (  # noqa: E402
    CounterMatrix,
    Executor,
    KeyGenSpec,
    encode_array,
    generate_keys,
    global_bin_offsets,
    global_histograms,
    onesweep_sort,
    oracle_stable_sort,
    partition_pass,
    radix_plan,
)
from onesweep.binning import StripCarry, process_tile, wlms_rank  # noqa: E402
from onesweep.keycodec import extract_digits  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_golden.npz")

DTYPES = {
    "u32": np.uint32,
    "u64": np.uint64,
    "i32": np.int32,
    "i64": np.int64,
    "f32": np.float32,
    "f64": np.float64,
}


def special_bits(name: str) -> np.ndarray:
    """Edge patterns per key type: zeros, sign, extremes, NaN/inf payloads."""
    bits = 64 if name.endswith("64") else 32
    u = np.uint64 if bits == 64 else np.uint32
    sign = 1 << (bits - 1)
    full = (1 << bits) - 1
    pats = [0, 1, sign, sign - 1, sign + 1, full, full - 1]
    if name == "f32":
        pats += [0x7F800000, 0xFF800000, 0x7FC00000, 0xFFC00000, 0x3F800000, 0xBF800000, 0x00000001]
    if name == "f64":
        pats += [0x7FF0000000000000, 0xFFF0000000000000, 0x7FF8000000000000, 0xFFF8000000000000,
                 0x3FF0000000000000, 0xBFF0000000000000, 1]
    return np.array(pats, dtype=u)


def main() -> None:
    g: dict[str, np.ndarray] = {}
    rng = np.random.default_rng(2206_01784)

    # -- keygen (keygen.py:63-76)
    for q, kbits, seed in [(1, 32, 0), (2, 32, 7), (3, 32, 1234), (4, 64, 3), (8, 32, 11), (16, 64, 5)]:
        g[f"keygen_q{q}_k{kbits}_s{seed}"] = generate_keys(KeyGenSpec(q=q, seed=seed, n=2048, key_bits=kbits))

    # -- codec (keycodec.py:184-212)
    for name, dt in DTYPES.items():
        bits = 64 if name.endswith("64") else 32
        u = np.uint64 if bits == 64 else np.uint32
        raw = np.concatenate([special_bits(name), rng.integers(0, 2**bits, size=1000, dtype=np.uint64).astype(u)])
        g[f"codec_{name}_in"] = raw
        g[f"codec_{name}_enc"] = encode_array(raw.view(dt))

    # -- histograms (histogram.py:57-99)
    for kbits, d in [(32, 8), (32, 5), (32, 3), (64, 8), (64, 6)]:
        u = np.uint32 if kbits == 32 else np.uint64
        keys = rng.integers(0, 2**kbits, size=5000, dtype=np.uint64).astype(u)
        cfg = radix_plan(kbits, d)
        hist = global_histograms(keys, cfg, Executor(workers=2))
        g[f"hist_k{kbits}_d{d}_in"] = keys
        g[f"hist_k{kbits}_d{d}_counts"] = hist.counts
        g[f"hist_k{kbits}_d{d}_offsets"] = global_bin_offsets(hist).offsets

    # -- WLMS (binning.py:57-68)
    for i, d in enumerate([1, 2, 3, 5, 8, 8]):
        digits = rng.integers(0, 1 << d, size=int(rng.integers(1, 33)))
        counts, ranks = wlms_rank(digits, d)
        g[f"wlms_{i}_d"] = np.array([d])
        g[f"wlms_{i}_digits"] = digits
        g[f"wlms_{i}_counts"] = counts
        g[f"wlms_{i}_ranks"] = ranks

    # -- CounterMatrix final words after a sequential pass (lookback.py:63-169)
    cfg = radix_plan(32, 4, tile_size=64)
    keys = rng.integers(0, 2**32, size=1000, dtype=np.uint32)
    digits = extract_digits(keys, 1, cfg)
    offs = np.zeros(cfg.radix, dtype=np.uint64)
    np.cumsum(np.bincount(digits, minlength=cfg.radix)[:-1], dtype=np.uint64, out=offs[1:])
    tiles = -(-keys.size // cfg.tile_size)
    cm = CounterMatrix(tiles, cfg.radix)
    out = np.zeros_like(keys)
    for t in range(tiles):
        lo, hi = t * cfg.tile_size, min((t + 1) * cfg.tile_size, keys.size)
        process_tile(t, keys[lo:hi], out, 1, offs, cm, cfg)
    g["counters_in"] = keys
    g["counters_offsets"] = offs
    g["counters_words"] = cm.words.copy()
    g["counters_out"] = out

    # -- partition passes (binning.py:218-275), including strip carries
    for tag, kbits, d, place, tile, strip, with_vals in [
        ("p8", 32, 8, 1, 256, 1 << 28, True),
        ("p5", 32, 5, 2, 100, 1000, False),
        ("p3", 64, 3, 7, 37, 333, True),
        ("p8s", 64, 8, 6, 512, 2048, True),
    ]:
        u = np.uint32 if kbits == 32 else np.uint64
        cfg = radix_plan(kbits, d, tile_size=tile, strip_size=strip)
        src = rng.integers(0, 2**kbits, size=4000, dtype=np.uint64).astype(u)
        vals = np.arange(src.size, dtype=np.uint64) * 3 + 1 if with_vals else None
        digits = extract_digits(src, place, cfg)
        base = np.zeros(cfg.radix, dtype=np.uint64)
        np.cumsum(np.bincount(digits, minlength=cfg.radix)[:-1], dtype=np.uint64, out=base[1:])
        dst = np.zeros_like(src)
        dvals = None if vals is None else np.zeros_like(vals)
        ex = Executor(workers=2)
        carry = partition_pass(src, dst, place, base, cfg, ex, vals, dvals)
        g[f"pass_{tag}_meta"] = np.array([kbits, d, place, tile, strip, int(with_vals)])
        g[f"pass_{tag}_src"] = src
        g[f"pass_{tag}_base"] = base
        g[f"pass_{tag}_dst"] = dst
        g[f"pass_{tag}_carry"] = carry.offsets
        g[f"pass_{tag}_fast"] = np.array([ex.ledger_snapshot().fast_path_tiles])
        if vals is not None:
            g[f"pass_{tag}_vals"] = vals
            g[f"pass_{tag}_dvals"] = dvals
        # chained halves through a StripCarry (test_binning.py:272-291)
        half = src.size // 2
        h = np.zeros_like(src)
        c1 = partition_pass(src[:half], h, place, base, cfg, Executor(workers=1))
        assert isinstance(c1, StripCarry)
        c2 = partition_pass(src[half:], h, place, c1, cfg, Executor(workers=1))
        g[f"pass_{tag}_halves"] = h
        g[f"pass_{tag}_carry_half"] = c1.offsets
        g[f"pass_{tag}_carry_full"] = c2.offsets

    # -- full sorts (binning.py:278-337) incl. signed/float twiddling and payloads
    for name, dt in DTYPES.items():
        bits = 64 if name.endswith("64") else 32
        u = np.uint64 if bits == 64 else np.uint32
        raw = np.concatenate([special_bits(name), special_bits(name),
                              rng.integers(0, 2**bits, size=3000, dtype=np.uint64).astype(u)])
        rng.shuffle(raw)
        keys = raw.view(dt)
        vals = np.arange(keys.size, dtype=np.uint32)
        for d in (8, 5):
            cfg = radix_plan(bits, d, tile_size=512)
            sk, sv = onesweep_sort(keys, vals, cfg, Executor(workers=2))
            ok, ov = oracle_stable_sort(keys, vals)
            assert np.array_equal(sk.view(u), ok.view(u)) and np.array_equal(sv, ov)
            g[f"sort_{name}_d{d}_keys"] = sk.view(u)
            g[f"sort_{name}_d{d}_vals"] = sv
        g[f"sort_{name}_in"] = raw

    # distributions (C3 shapes, small): q bands, all-equal, presorted, few distinct
    dist = {
        "q2": generate_keys(KeyGenSpec(q=2, seed=1, n=6000)),
        "q8": generate_keys(KeyGenSpec(q=8, seed=2, n=6000)),
        "q16": generate_keys(KeyGenSpec(q=16, seed=3, n=6000)),
        "equal": np.full(8192, 0xABACADAE, dtype=np.uint32),
        "presorted": np.sort(generate_keys(KeyGenSpec(q=1, seed=4, n=6000))),
        "dups": rng.integers(0, 8, size=6000, dtype=np.uint32),
    }
    for tag, keys in dist.items():
        cfg = radix_plan(32, 8, tile_size=512)
        ex = Executor(workers=2)
        sk, sv = onesweep_sort(keys, np.arange(keys.size, dtype=np.uint32), cfg, ex)
        snap = ex.ledger_snapshot()
        g[f"dist_{tag}_in"] = keys
        g[f"dist_{tag}_keys"] = sk
        g[f"dist_{tag}_vals"] = sv
        g[f"dist_{tag}_ledger"] = np.array(
            [snap.element_reads, snap.element_writes, snap.copy_ops, snap.fast_path_tiles]
        )

    # odd pass count (d=7 -> 5 passes) ledger incl. the parity copy
    keys = rng.integers(0, 2**32, size=5000, dtype=np.uint32)
    ex = Executor(workers=2)
    sk = onesweep_sort(keys, cfg=radix_plan(32, 7, tile_size=512), executor=ex)
    snap = ex.ledger_snapshot()
    g["odd_in"] = keys
    g["odd_keys"] = sk
    g["odd_ledger"] = np.array([snap.element_ops, snap.copy_ops])

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays, {os.path.getsize(OUT)} bytes")


if __name__ == "__main__":
    main()
