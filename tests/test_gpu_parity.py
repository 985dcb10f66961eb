"""GPU parity: the sm_100a path against the reference's golden vectors and
the CPU oracle, bit-exact (integer / byte work: no tolerance)."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DT = {"u32": np.uint32, "u64": np.uint64, "i32": np.int32, "i64": np.int64,
      "f32": np.float32, "f64": np.float64}


def _pkg():
    import paper_2206_01784_b200 as os_b200

    return os_b200


# -- elementwise ------------------------------------------------------------


def test_keygen_matches_reference(cuda, golden):
    from paper_2206_01784_b200 import KeyGenSpec, generate_keys

    for key in [k for k in golden if k.startswith("keygen_")]:
        _, q, kb, s = key.split("_")
        want = golden[key]
        got = generate_keys(KeyGenSpec(q=int(q[1:]), seed=int(s[1:]), n=want.size, key_bits=int(kb[1:])))
        assert np.array_equal(got, want), key


def test_keygen_shards_concatenate(cuda, oracle):
    from paper_2206_01784_b200 import KeyGenSpec, generate_keys

    full = generate_keys(KeyGenSpec(q=3, seed=99, n=10_000))
    a = generate_keys(KeyGenSpec(q=3, seed=99, n=4_000), device="cuda", first_index=0).cpu().numpy()
    b = generate_keys(KeyGenSpec(q=3, seed=99, n=6_000), device="cuda", first_index=4_000).cpu().numpy()
    assert np.array_equal(np.concatenate([a, b]), full)
    assert np.array_equal(full, oracle.keygen(10_000, 3, 99))


@pytest.mark.parametrize("name", list(DT))
def test_codec_matches_reference(cuda, golden, name):
    from paper_2206_01784_b200 import decode_array, encode_array

    raw = golden[f"codec_{name}_in"]
    enc = encode_array(raw.view(DT[name]))
    assert np.array_equal(enc, golden[f"codec_{name}_enc"])
    assert np.array_equal(decode_array(enc, name).view(raw.dtype), raw)


def test_codec_constants(cuda):
    from paper_2206_01784_b200 import decode_key, encode_key

    assert encode_key(-1, "i32") == 0x7FFFFFFF
    assert encode_key(-(2**31), "i32") == 0
    assert encode_key(-1, "i64") == 0x7FFFFFFFFFFFFFFF
    assert encode_key(np.float32(-0.0), "f32") == 0x7FFFFFFF
    assert encode_key(np.float32(0.0), "f32") == 0x80000000
    assert decode_key(0x7FFFFFFF, "i32") == -1
    assert np.signbit(decode_key(0x7FFFFFFF, "f32"))


# -- histogram ----------------------------------------------------------------


@pytest.mark.parametrize("kbits,d", [(32, 8), (32, 5), (32, 3), (64, 8), (64, 6)])
def test_histogram_matches_reference(cuda, golden, kbits, d):
    from paper_2206_01784_b200 import Executor, global_bin_offsets, global_histograms, radix_plan

    keys = golden[f"hist_k{kbits}_d{d}_in"]
    ex = Executor()
    hist = global_histograms(keys, radix_plan(kbits, d), ex)
    assert np.array_equal(hist.counts, golden[f"hist_k{kbits}_d{d}_counts"])
    assert np.array_equal(global_bin_offsets(hist).offsets, golden[f"hist_k{kbits}_d{d}_offsets"])
    assert ex.ledger_snapshot().phase("histogram").element_reads == keys.size
    # the fused last-block scan equals the standalone scan kernel
    import torch

    dev = global_histograms(torch.from_numpy(keys).cuda(), radix_plan(kbits, d))
    assert np.array_equal(global_bin_offsets(dev).offsets.cpu().numpy(),
                          golden[f"hist_k{kbits}_d{d}_offsets"])


def test_histogram_edge_cases(cuda, oracle):
    from paper_2206_01784_b200 import global_histograms, radix_plan

    cfg = radix_plan(32, 8)
    assert not global_histograms(np.empty(0, np.uint32), cfg).counts.any()
    h = global_histograms(np.array([17, 8, 24, 5], dtype=np.uint32), radix_plan(32, 3)).counts
    assert h[0, 0] == 2 and h[0, 1] == 1 and h[0, 5] == 1
    # unaligned start (no 16-byte alignment) + ragged tail, all-equal keys
    rng = np.random.default_rng(5)
    base = rng.integers(0, 2**32, size=100_003, dtype=np.uint32)
    import torch

    t = torch.from_numpy(base).cuda()
    for off in (0, 1, 2, 3):
        got = global_histograms(t[off:], cfg).counts.cpu().numpy()
        assert np.array_equal(got, oracle.histogram(base[off:], 8))
    same = np.full(1 << 20, 0xABACADAE, dtype=np.uint32)
    assert np.array_equal(global_histograms(same, cfg).counts, oracle.histogram(same, 8))


def test_exclusive_sum_known_answers(cuda):
    from paper_2206_01784_b200 import exclusive_sum

    assert exclusive_sum(np.array([8, 6, 7, 5, 3, 0, 9, 2])).tolist() == [0, 8, 14, 21, 26, 29, 29, 38]
    assert exclusive_sum(np.array([0, 1, 1, 0])).tolist() == [0, 0, 1, 2]
    big = np.arange(5000, dtype=np.uint64)
    assert np.array_equal(exclusive_sum(big), np.concatenate([[0], np.cumsum(big)[:-1]]).astype(np.uint64))


# -- partition passes ----------------------------------------------------------


@pytest.mark.parametrize("tag", ["p8", "p5", "p3", "p8s"])
def test_partition_pass_matches_reference(cuda, golden, tag):
    from paper_2206_01784_b200 import Executor, StripCarry, partition_pass, radix_plan

    kbits, d, place, tile, strip, with_vals = (int(x) for x in golden[f"pass_{tag}_meta"])
    cfg = radix_plan(kbits, d, tile_size=tile, strip_size=strip)
    src = golden[f"pass_{tag}_src"]
    dst = np.zeros_like(src)
    sv = golden[f"pass_{tag}_vals"] if with_vals else None
    dv = np.zeros_like(sv) if with_vals else None
    ex = Executor()
    carry = partition_pass(src, dst, place, golden[f"pass_{tag}_base"], cfg, ex, sv, dv)
    assert isinstance(carry, StripCarry)
    assert np.array_equal(dst, golden[f"pass_{tag}_dst"])
    assert np.array_equal(carry.offsets, golden[f"pass_{tag}_carry"])
    if with_vals:
        assert np.array_equal(dv, golden[f"pass_{tag}_dvals"])
    snap = ex.ledger_snapshot()
    assert snap.phase("partition").element_reads == src.size
    assert snap.phase("partition").element_writes == src.size
    assert snap.fast_path_tiles == int(golden[f"pass_{tag}_fast"][0])
    half = src.size // 2
    h = np.zeros_like(src)
    c1 = partition_pass(src[:half], h, place, golden[f"pass_{tag}_base"], cfg)
    c2 = partition_pass(src[half:], h, place, c1, cfg)
    assert np.array_equal(c1.offsets, golden[f"pass_{tag}_carry_half"])
    assert np.array_equal(c2.offsets, golden[f"pass_{tag}_carry_full"])
    assert np.array_equal(h, golden[f"pass_{tag}_halves"])


def test_status_words_match_reference_counter_matrix(cuda, golden):
    # final CounterMatrix of a pass is schedule-independent: every word is
    # G | inclusive prefix (lookback.py:136-142, test_lookback.py:150-160)
    from paper_2206_01784_b200 import partition_pass, radix_plan

    cfg = radix_plan(32, 4, tile_size=64)
    src = golden["counters_in"]
    dst = np.zeros_like(src)
    _, views = partition_pass(src, dst, 1, golden["counters_offsets"], cfg, return_status=True)
    assert len(views) == 1
    assert np.array_equal(views[0].words, golden["counters_words"])
    assert np.array_equal(dst, golden["counters_out"])


def test_partition_worked_example(cuda):
    from paper_2206_01784_b200 import partition_pass, radix_plan

    src = np.array([17, 8, 24, 5], dtype=np.uint32)
    dst = np.zeros_like(src)
    base = np.zeros(8, dtype=np.uint64)
    base[1], base[5] = 2, 3
    partition_pass(src, dst, 0, base, radix_plan(32, 3, tile_size=4))
    assert dst.tolist() == [8, 24, 17, 5]
    # process_tile offset identity (test_binning.py:161-170)
    out = np.zeros(16, dtype=np.uint32)
    base = np.zeros(8, dtype=np.uint64)
    base[0] = 8
    partition_pass(np.array([8, 16, 24], dtype=np.uint32), out, 0, base, radix_plan(32, 3, tile_size=16))
    assert out[8] == 8 and out[9] == 16 and out[10] == 24


# -- full sorts -------------------------------------------------------------------


@pytest.mark.parametrize("name", list(DT))
@pytest.mark.parametrize("d", [8, 5])
def test_sort_matches_reference(cuda, golden, name, d):
    from paper_2206_01784_b200 import Executor, onesweep_sort, radix_plan

    raw = golden[f"sort_{name}_in"]
    keys = raw.view(DT[name])
    vals = np.arange(keys.size, dtype=np.uint32)
    bits = raw.dtype.itemsize * 8
    ex = Executor()
    sk, sv = onesweep_sort(keys, vals, radix_plan(bits, d, tile_size=512), ex)
    assert sk.dtype == keys.dtype
    assert np.array_equal(sk.view(raw.dtype), golden[f"sort_{name}_d{d}_keys"])
    assert np.array_equal(sv, golden[f"sort_{name}_d{d}_vals"])
    p = -(-bits // d)
    assert ex.ledger_snapshot().element_ops == (2 * p + 1) * keys.size  # (2p+1)n
    # keys only, default config (device tile)
    assert np.array_equal(onesweep_sort(keys).view(raw.dtype), golden[f"sort_{name}_d8_keys"])


@pytest.mark.parametrize("tag", ["q2", "q8", "q16", "equal", "presorted", "dups"])
def test_distributions_match_reference(cuda, golden, tag):
    from paper_2206_01784_b200 import Executor, onesweep_sort, radix_plan

    keys = golden[f"dist_{tag}_in"]
    ex = Executor()
    sk, sv = onesweep_sort(keys, np.arange(keys.size, dtype=np.uint32), radix_plan(32, 8, tile_size=512), ex)
    assert np.array_equal(sk, golden[f"dist_{tag}_keys"])
    assert np.array_equal(sv, golden[f"dist_{tag}_vals"])
    snap = ex.ledger_snapshot()
    reads, writes, _copy, fast = (int(x) for x in golden[f"dist_{tag}_ledger"])
    assert snap.element_reads == reads and snap.element_writes == writes
    assert snap.fast_path_tiles == fast  # e.g. all-equal: 4 passes x 16 tiles = 64


def test_odd_pass_count_avoids_parity_copy(cuda, golden):
    # d=7 -> 5 passes.  The reference ledgers 11n + a 2n parity copy
    # (test_binning.py:353-362) and so does the plan's ledger here; the device
    # routes the passes so the last one lands in the output buffer, so the
    # copy never happens on the device (device_element_ops: five 7-bit passes,
    # (2*5+1)n, no copy).
    from paper_2206_01784_b200 import Executor, onesweep_sort, radix_plan

    keys = golden["odd_in"]
    ex = Executor()
    got = onesweep_sort(keys, cfg=radix_plan(32, 7, tile_size=512), executor=ex)
    assert np.array_equal(got, golden["odd_keys"])
    snap = ex.ledger_snapshot()
    assert snap.element_ops == int(golden["odd_ledger"][0]) == 11 * keys.size
    assert snap.copy_ops == 2 * keys.size
    assert ex.device_element_ops == 11 * keys.size


def test_sort_rejects_bad_arguments(cuda):
    from paper_2206_01784_b200 import onesweep_sort, radix_plan

    with pytest.raises(KeyError):
        onesweep_sort(np.zeros(4, dtype=np.float16))
    with pytest.raises(ValueError):
        onesweep_sort(np.zeros(4, dtype=np.uint32), cfg=radix_plan(64, 8))
    with pytest.raises(ValueError):
        onesweep_sort(np.zeros(4, dtype=np.uint32), np.zeros(3, dtype=np.uint32))


def test_sort_pipeline_matches_onesweep_sort(cuda):
    """SortPipeline (overlapped upload / sort / download of host batches)
    returns, for every submitted batch, what onesweep_sort returns."""
    import torch

    from paper_2206_01784_b200 import KeyGenSpec, SortPipeline, generate_keys, onesweep_sort

    n = 1_000_003
    pipe = SortPipeline(n, torch.uint32, torch.uint32, depth=2)
    ins, outs, want = [], [], []
    for seed in range(5):
        k = generate_keys(KeyGenSpec(q=1 + seed % 3, seed=seed, n=n), device="cuda").cpu().pin_memory()
        v = torch.arange(n, dtype=torch.int32).view(torch.uint32).pin_memory()
        ok = torch.empty(n, dtype=torch.uint32).pin_memory()
        ov = torch.empty(n, dtype=torch.uint32).pin_memory()
        pipe.submit(k, ok, v, ov)
        ins.append((k, v))
        outs.append((ok, ov))
    pipe.synchronize()
    for (k, v), (ok, ov) in zip(ins, outs):
        wk, wv = onesweep_sort(k.numpy(), v.numpy())
        assert np.array_equal(ok.numpy(), wk) and np.array_equal(ov.numpy(), wv)


@pytest.mark.parametrize("case", ["all-equal", "q16", "presorted", "two-digits"])
def test_keys_only_uniform_warp_shortcut(cuda, case):
    """Keys-only passes skip the multisplit for warps whose keys share one
    digit (OS_UNIFORM_KEYS): the output must still be the stable sort, for
    inputs where such warps are common, rare, or mixed within a tile."""
    import torch

    from paper_2206_01784_b200 import KeyGenSpec, generate_keys, onesweep_sort

    n = (1 << 24) + 12345
    if case == "all-equal":
        keys = np.full(n, 0xABACADAE, dtype=np.uint32)
    elif case == "q16":
        keys = generate_keys(KeyGenSpec(q=16, seed=3, n=n), device="cuda").cpu().numpy()
    elif case == "presorted":
        keys = np.sort(generate_keys(KeyGenSpec(q=1, seed=4, n=n), device="cuda").cpu().numpy())
    else:  # long runs of one value, then another: uniform and mixed warps
        keys = np.where((np.arange(n) // 5000) % 2 == 0, 0x11223344, 0x11223345).astype(np.uint32)
    got = onesweep_sort(torch.from_numpy(keys).cuda()).cpu().numpy()
    assert np.array_equal(got, np.sort(keys, kind="stable"))
