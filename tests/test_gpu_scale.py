"""GPU parity at scale and on edge cases.

Small and medium sizes compare bit-exactly with the oracle.  At the
BASELINE sizes (16M, 256M) the checks are size-independent properties that
together pin a stable sort uniquely: output sorted by encoded key, output is
the input permuted by the returned index payload, and equal keys keep their
input order."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _stable_sort_np(keys, values=None):
    from oracle import oracle

    order = np.argsort(oracle.encode(keys), kind="stable")
    return keys[order] if values is None else (keys[order], values[order])


@pytest.mark.parametrize("n", [2, 3, 31, 32, 33, 100, 4095, 4096, 4097, 8191, 8192, 8193, 3 * 8192 + 5])
def test_ragged_sizes(cuda, n):
    from paper_2206_01784_b200 import onesweep_sort

    rng = np.random.default_rng(n)
    keys = rng.integers(0, 2**32, size=n, dtype=np.uint32)
    vals = np.arange(n, dtype=np.uint32)
    sk, sv = onesweep_sort(keys, vals)
    wk, wv = _stable_sort_np(keys, vals)
    assert np.array_equal(sk, wk) and np.array_equal(sv, wv)


@pytest.mark.parametrize("offset", [1, 2, 3])
def test_misaligned_inputs_take_the_plain_load_path(cuda, offset):
    import torch

    from paper_2206_01784_b200 import onesweep_sort

    rng = np.random.default_rng(offset)
    base = rng.integers(0, 2**32, size=200_000, dtype=np.uint32)
    bv = np.arange(base.size, dtype=np.uint32)
    tk = torch.from_numpy(base).cuda()[offset:]
    tv = torch.from_numpy(bv).cuda()[offset:]
    sk, sv = onesweep_sort(tk, tv)
    wk, wv = _stable_sort_np(base[offset:], bv[offset:])
    assert np.array_equal(sk.cpu().numpy(), wk) and np.array_equal(sv.cpu().numpy(), wv)
    assert np.array_equal(tk.cpu().numpy(), base[offset:])  # input untouched


@pytest.mark.parametrize("name,dt", [("u64", np.uint64), ("i64", np.int64), ("f64", np.float64),
                                     ("i32", np.int32), ("f32", np.float32)])
@pytest.mark.parametrize("vdt", [None, np.uint8, np.uint16, np.uint32, np.uint64])
def test_key_and_value_widths(cuda, name, dt, vdt):
    from paper_2206_01784_b200 import onesweep_sort

    rng = np.random.default_rng(7)
    bits = np.dtype(dt).itemsize * 8
    raw = rng.integers(0, 2**bits, size=300_001, dtype=np.uint64)
    keys = (raw if bits == 64 else raw.astype(np.uint32)).view(dt)
    if vdt is None:
        got = onesweep_sort(keys)
        assert np.array_equal(got.view(raw.dtype if bits == 64 else np.uint32),
                              _stable_sort_np(keys).view(raw.dtype if bits == 64 else np.uint32))
        return
    vals = rng.integers(0, np.iinfo(vdt).max, size=keys.size, dtype=np.uint64).astype(vdt)
    sk, sv = onesweep_sort(keys, vals)
    wk, wv = _stable_sort_np(keys, vals)
    u = np.uint64 if bits == 64 else np.uint32
    assert np.array_equal(sk.view(u), wk.view(u)) and np.array_equal(sv, wv)


@pytest.mark.parametrize("d", [1, 2, 3, 4, 5, 6, 7, 8])
def test_every_digit_width(cuda, oracle, d):
    from paper_2206_01784_b200 import onesweep_sort, radix_plan

    rng = np.random.default_rng(d)
    keys = rng.integers(0, 2**64, size=50_000, dtype=np.uint64)
    vals = np.arange(keys.size, dtype=np.uint32)
    sk, sv = onesweep_sort(keys, vals, radix_plan(64, d))
    wk, wv = _stable_sort_np(keys, vals)
    assert np.array_equal(sk, wk) and np.array_equal(sv, wv)


def test_wide_digit_configs_sort_identically(cuda):
    # digit_bits > 8 run as 8-bit places: the stable order is unique
    from paper_2206_01784_b200 import onesweep_sort, radix_plan

    keys = np.random.default_rng(0).integers(0, 2**32, size=100_000, dtype=np.uint32)
    assert np.array_equal(onesweep_sort(keys, cfg=radix_plan(32, 11)), np.sort(keys))


@pytest.mark.parametrize("begin,end", [(0, 32), (0, 16), (4, 20), (13, 32), (31, 32), (0, 1), (5, 6)])
def test_begin_end_bits(cuda, oracle, begin, end):
    from paper_2206_01784_b200 import onesweep_sort

    rng = np.random.default_rng(begin * 100 + end)
    keys = rng.integers(0, 2**32, size=70_000, dtype=np.uint32).view(np.int32)
    vals = np.arange(keys.size, dtype=np.uint32)
    sk, sv = onesweep_sort(keys, vals, begin_bit=begin, end_bit=end)
    wk, wv = oracle.stable_sort_bits(keys, vals, begin, end)
    assert np.array_equal(sk, wk) and np.array_equal(sv, wv)
    ok = oracle.sort(keys, begin_bit=begin, end_bit=end, digit_bits=8)
    assert np.array_equal(sk, ok)


def test_begin_end_bits_64(cuda, oracle):
    from paper_2206_01784_b200 import onesweep_sort

    keys = np.random.default_rng(1).standard_normal(60_000)
    for b, e in [(0, 64), (20, 64), (8, 40), (52, 64)]:
        assert np.array_equal(onesweep_sort(keys, begin_bit=b, end_bit=e).view(np.uint64),
                              oracle.stable_sort_bits(keys, None, b, e).view(np.uint64))


def test_tiny_tiles_deep_lookback_chains(cuda, oracle):
    # 32-key tiles: ~30k blocks per pass, look-back walks long L chains
    from paper_2206_01784_b200 import Executor, onesweep_sort, radix_plan

    keys = np.random.default_rng(3).integers(0, 2**32, size=1_000_000, dtype=np.uint32)
    ex = Executor()
    got = onesweep_sort(keys, cfg=radix_plan(32, 8, tile_size=32), executor=ex)
    assert np.array_equal(got, np.sort(keys))
    assert ex.ledger_snapshot().counter_ops > 0


def test_small_strips_chain_carries(cuda, oracle):
    from paper_2206_01784_b200 import onesweep_sort, radix_plan

    keys = np.random.default_rng(4).integers(0, 2**32, size=50_000, dtype=np.uint32)
    vals = np.arange(keys.size, dtype=np.uint64)
    for tile, strip in [(256, 1000), (100, 777), (8192, 4096)]:
        sk, sv = onesweep_sort(keys, vals, radix_plan(32, 8, tile_size=tile, strip_size=strip))
        wk, wv = _stable_sort_np(keys, vals)
        assert np.array_equal(sk, wk) and np.array_equal(sv, wv), (tile, strip)


def test_short_circuit_tile_count(cuda):
    # test_binning.py:375-384: 8192 x 0xABACADAE, tile 512 -> 4 x 16 fast tiles
    from paper_2206_01784_b200 import Executor, onesweep_sort, radix_plan

    keys = np.full(1 << 13, 0xABACADAE, dtype=np.uint32)
    ex = Executor()
    got = onesweep_sort(keys, cfg=radix_plan(32, 8, tile_size=512), executor=ex)
    assert np.array_equal(got, keys)
    assert ex.ledger_snapshot().fast_path_tiles == 4 * 16


def test_heavy_duplicates_stability(cuda):
    from paper_2206_01784_b200 import onesweep_sort

    keys = np.random.default_rng(11).integers(0, 8, size=1_000_000, dtype=np.uint32)
    vals = np.arange(keys.size, dtype=np.uint64)
    gk, gv = onesweep_sort(keys, vals)
    for k in range(8):
        assert (np.diff(gv[gk == k].astype(np.int64)) > 0).all()


def test_torch_in_out_and_determinism(cuda):
    import torch

    from paper_2206_01784_b200 import KeyGenSpec, generate_keys, onesweep_sort

    keys = generate_keys(KeyGenSpec(q=2, seed=5, n=3_000_000), device="cuda")
    before = keys.clone()
    a = onesweep_sort(keys)
    b = onesweep_sort(keys)
    torch.cuda.synchronize()
    assert a.is_cuda and a.dtype == torch.uint32
    assert torch.equal(keys.view(torch.int32), before.view(torch.int32))
    assert np.array_equal(a.cpu().numpy(), b.cpu().numpy())
    assert np.array_equal(a.cpu().numpy(), np.sort(keys.cpu().numpy()))


# -- BASELINE sizes -------------------------------------------------------------


def _check_stable_permutation(keys_in: np.ndarray, keys_out: np.ndarray, idx_out: np.ndarray):
    """sorted + (keys_out == keys_in[idx_out]) + stable  <=>  the unique stable sort."""
    assert (keys_out[1:] >= keys_out[:-1]).all()  # unsigned compare on encoded-order dtypes
    assert np.array_equal(keys_in[idx_out], keys_out)
    same = keys_out[1:] == keys_out[:-1]
    assert (idx_out[1:][same] > idx_out[:-1][same]).all()


@pytest.mark.slow
def test_config1_16M_bit_exact(cuda):
    from paper_2206_01784_b200 import KeyGenSpec, generate_keys, onesweep_sort

    keys = generate_keys(KeyGenSpec(q=1, seed=0, n=1 << 24, key_bits=32))
    got = onesweep_sort(keys)
    assert np.array_equal(got, np.sort(keys))


@pytest.mark.slow
@pytest.mark.parametrize("q", [1, 4, 16])
def test_config3_pairs_256M_properties(cuda, q):
    import torch

    from paper_2206_01784_b200 import KeyGenSpec, generate_keys, onesweep_sort

    n = 1 << 28
    keys = generate_keys(KeyGenSpec(q=q, seed=q, n=n), device="cuda")
    idx = torch.arange(n, dtype=torch.int32, device="cuda").view(torch.uint32)
    sk, sv = onesweep_sort(keys, idx)
    torch.cuda.synchronize()
    k_in = keys.cpu().numpy()
    del keys, idx
    k_out, v_out = sk.cpu().numpy(), sv.cpu().numpy()
    _check_stable_permutation(k_in, k_out, v_out)


@pytest.mark.slow
def test_config2_multi_strip_2e28_plus(cuda):
    # > 2^28 keys: two strips per pass chained by 64-bit carries
    import torch

    from paper_2206_01784_b200 import KeyGenSpec, generate_keys, onesweep_sort

    n = (1 << 28) + 123_457
    keys = generate_keys(KeyGenSpec(q=1, seed=77, n=n), device="cuda")
    out = onesweep_sort(keys)
    torch.cuda.synchronize()
    a = keys.cpu().numpy()
    b = out.cpu().numpy()
    assert (b[1:] >= b[:-1]).all()
    assert np.array_equal(np.bincount(a >> 16, minlength=1 << 16), np.bincount(b >> 16, minlength=1 << 16))
    assert int(a.astype(np.uint64).sum()) == int(b.astype(np.uint64).sum())


@pytest.mark.slow
def test_config4_u64_pairs_signed_float(cuda):
    import torch

    from oracle import oracle
    from paper_2206_01784_b200 import KeyGenSpec, generate_keys, onesweep_sort

    n = 1 << 24
    raw = generate_keys(KeyGenSpec(q=1, seed=9, n=n, key_bits=64), device="cuda")
    idx = torch.arange(n, dtype=torch.int32, device="cuda").view(torch.uint32)
    for dt in (torch.uint64, torch.int64, torch.float64):
        sk, sv = onesweep_sort(raw.view(dt), idx)
        k_in = raw.view(dt).cpu().numpy()
        k_out, v_out = sk.cpu().numpy(), sv.cpu().numpy()
        enc = oracle.encode(k_out)
        assert (enc[1:] >= enc[:-1]).all()
        assert np.array_equal(k_in.view(np.uint64)[v_out], k_out.view(np.uint64))
        same = enc[1:] == enc[:-1]
        assert (v_out[1:][same] > v_out[:-1][same]).all()
