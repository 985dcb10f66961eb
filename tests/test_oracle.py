"""CPU: pin the oracle (oracle/) to the reference.

Every golden array was produced by the reference package itself
(tests/golden/make_golden.py); the known-answer constants are the reference
tests' own (cited per test)."""

from __future__ import annotations

import numpy as np
import pytest

DT = {"u32": np.uint32, "u64": np.uint64, "i32": np.int32, "i64": np.int64,
      "f32": np.float32, "f64": np.float64}


def test_keygen_matches_reference(golden, oracle):
    for key in [k for k in golden if k.startswith("keygen_")]:
        _, q, kb, s = key.split("_")
        want = golden[key]
        got = oracle.keygen(want.size, int(q[1:]), int(s[1:]), int(kb[1:]))
        assert np.array_equal(got, want), key


@pytest.mark.parametrize("name", list(DT))
def test_codec_matches_reference(golden, oracle, name):
    raw = golden[f"codec_{name}_in"]
    enc = oracle.encode(raw.view(DT[name]))
    assert np.array_equal(enc, golden[f"codec_{name}_enc"])
    back = oracle.decode(enc, name)
    assert np.array_equal(back.view(raw.dtype), raw)


def test_codec_known_answers(oracle):
    # test_keycodec.py:46-52, 76-90
    e = lambda v, t: int(oracle.encode(np.array([v], dtype=DT[t]))[0])  # noqa: E731
    assert e(-1, "i32") == 0x7FFFFFFF
    assert e(-(2**31), "i32") == 0
    assert e(2**31 - 1, "i32") == 0xFFFFFFFF
    assert e(-1, "i64") == 0x7FFFFFFFFFFFFFFF
    assert e(-0.0, "f32") == 0x7FFFFFFF
    assert e(0.0, "f32") == 0x80000000
    pos_nan = e(np.uint32(0x7FC00000).view(np.float32), "f32")
    neg_nan = e(np.uint32(0xFFC00000).view(np.float32), "f32")
    assert pos_nan > e(np.inf, "f32") and neg_nan < e(-np.inf, "f32")


def test_exclusive_sum_known_answers(oracle):
    # test_histogram.py:32-38
    assert oracle.exclusive_sum(np.array([8, 6, 7, 5, 3, 0, 9, 2])).tolist() == [0, 8, 14, 21, 26, 29, 29, 38]
    assert oracle.exclusive_sum(np.array([0, 1, 1, 0])).tolist() == [0, 0, 1, 2]


@pytest.mark.parametrize("kbits,d", [(32, 8), (32, 5), (32, 3), (64, 8), (64, 6)])
def test_histogram_matches_reference(golden, oracle, kbits, d):
    keys = golden[f"hist_k{kbits}_d{d}_in"]
    hist = oracle.histogram(keys, d)
    assert np.array_equal(hist, golden[f"hist_k{kbits}_d{d}_counts"])
    assert np.array_equal(oracle.bin_offsets(hist), golden[f"hist_k{kbits}_d{d}_offsets"])


def test_histogram_worked_example(oracle):
    # test_histogram.py:52-58: <17,8,24,5>, d=3, place 0 -> digit0=2, digit1=1, digit5=1
    h = oracle.histogram(np.array([17, 8, 24, 5], dtype=np.uint32), 3)
    assert h[0, 0] == 2 and h[0, 1] == 1 and h[0, 5] == 1 and h[0].sum() == 4


def test_wlms_matches_reference(golden, oracle):
    for i in range(6):
        d = int(golden[f"wlms_{i}_d"][0])
        counts, ranks = oracle.wlms_rank(golden[f"wlms_{i}_digits"], d)
        assert np.array_equal(counts, golden[f"wlms_{i}_counts"])
        assert np.array_equal(ranks, golden[f"wlms_{i}_ranks"])


def test_wlms_worked_example(oracle):
    # test_binning.py:54-57
    counts, ranks = oracle.wlms_rank(np.array([2, 0, 2, 1]), 2)
    assert counts.tolist() == [1, 1, 2, 0] and ranks.tolist() == [0, 0, 1, 0]


def test_counter_words_match_reference(golden, oracle):
    src = golden["counters_in"]
    dst = np.zeros_like(src)
    carry, fast, status = oracle.partition_pass(src, dst, 4, 4, golden["counters_offsets"], tile=64,
                                                want_status=True, threads=4)
    assert np.array_equal(dst, golden["counters_out"])
    assert np.array_equal(status.reshape(golden["counters_words"].shape), golden["counters_words"])


@pytest.mark.parametrize("tag", ["p8", "p5", "p3", "p8s"])
@pytest.mark.parametrize("threads", [1, 4])
def test_partition_pass_matches_reference(golden, oracle, tag, threads):
    kbits, d, place, tile, strip, with_vals = (int(x) for x in golden[f"pass_{tag}_meta"])
    src = golden[f"pass_{tag}_src"]
    dst = np.zeros_like(src)
    sv = golden.get(f"pass_{tag}_vals") if with_vals else None
    dv = np.zeros_like(sv) if with_vals else None
    carry, fast, _ = oracle.partition_pass(src, dst, place * d, d, golden[f"pass_{tag}_base"], sv, dv,
                                           tile=tile, strip=strip, threads=threads)
    assert np.array_equal(dst, golden[f"pass_{tag}_dst"])
    assert np.array_equal(carry, golden[f"pass_{tag}_carry"])
    assert fast == int(golden[f"pass_{tag}_fast"][0])
    if with_vals:
        assert np.array_equal(dv, golden[f"pass_{tag}_dvals"])
    # two halves chained through a StripCarry (test_binning.py:272-291)
    half = src.size // 2
    h = np.zeros_like(src)
    c1, _, _ = oracle.partition_pass(src[:half], h, place * d, d, golden[f"pass_{tag}_base"],
                                     tile=tile, strip=strip, threads=threads)
    c2, _, _ = oracle.partition_pass(src[half:], h, place * d, d, c1, tile=tile, strip=strip,
                                     threads=threads)
    assert np.array_equal(c1, golden[f"pass_{tag}_carry_half"])
    assert np.array_equal(c2, golden[f"pass_{tag}_carry_full"])
    assert np.array_equal(h, golden[f"pass_{tag}_halves"])


def test_partition_worked_example(oracle):
    # test_binning.py:215-223
    src = np.array([17, 8, 24, 5], dtype=np.uint32)
    dst = np.zeros_like(src)
    base = np.zeros(8, dtype=np.uint64)
    base[1], base[5] = 2, 3
    oracle.partition_pass(src, dst, 0, 3, base, tile=4)
    assert dst.tolist() == [8, 24, 17, 5]


@pytest.mark.parametrize("name", list(DT))
@pytest.mark.parametrize("d", [8, 5])
def test_sort_matches_reference(golden, oracle, name, d):
    raw = golden[f"sort_{name}_in"]
    keys = raw.view(DT[name])
    vals = np.arange(keys.size, dtype=np.uint32)
    sk, sv = oracle.sort(keys, vals, digit_bits=d, tile=512, threads=2)
    assert np.array_equal(sk.view(raw.dtype), golden[f"sort_{name}_d{d}_keys"])
    assert np.array_equal(sv, golden[f"sort_{name}_d{d}_vals"])


@pytest.mark.parametrize("tag", ["q2", "q8", "q16", "equal", "presorted", "dups"])
def test_distributions_match_reference(golden, oracle, tag):
    keys = golden[f"dist_{tag}_in"]
    sk, sv = oracle.sort(keys, np.arange(keys.size, dtype=np.uint32), tile=512, threads=3)
    assert np.array_equal(sk, golden[f"dist_{tag}_keys"])
    assert np.array_equal(sv, golden[f"dist_{tag}_vals"])
    assert oracle.sort.last_fast_path_tiles == int(golden[f"dist_{tag}_ledger"][3])


def test_sort_oracle_helpers_agree(oracle):
    rng = np.random.default_rng(0)
    keys = rng.integers(0, 2**32, size=10000, dtype=np.uint32)
    assert np.array_equal(oracle.sort(keys, threads=4), np.sort(keys, kind="stable"))
    # begin/end bit restatement: full range equals the full sort
    assert np.array_equal(oracle.stable_sort_bits(keys), np.sort(keys))
    got = oracle.sort(keys, begin_bit=4, end_bit=20, digit_bits=8)
    assert np.array_equal(got, oracle.stable_sort_bits(keys, begin_bit=4, end_bit=20))
    got = oracle.sort(keys.view(np.int32), begin_bit=3, end_bit=32, digit_bits=7)
    assert np.array_equal(got, oracle.stable_sort_bits(keys.view(np.int32), begin_bit=3))
