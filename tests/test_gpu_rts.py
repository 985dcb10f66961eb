"""GPU: the reduce-then-scan comparator (os_rts_sort) -- the reference's
rts_sort contract (baseline.py:121-173, pinned by test_baseline.py:158-200)
restated against the oracle, its 3pn ledger, and byte equality with the
Onesweep sort at BASELINE sizes."""

from __future__ import annotations

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", [np.uint32, np.int32, np.float32, np.uint64])
def test_rts_sort_equals_oracle(cuda, dtype):
    from oracle import oracle
    from paper_2206_01784_b200 import rts_sort

    rng = np.random.default_rng(13)
    bits = 64 if dtype == np.uint64 else 32
    raw = rng.integers(0, 2**bits, size=8000, dtype=np.uint64)
    keys = raw.astype(np.uint32).view(dtype) if bits == 32 else raw.view(dtype)
    values = np.arange(keys.size, dtype=np.uint64)
    got_k, got_v = rts_sort(keys, values)
    want_k, want_v = oracle.sort(keys, values)
    assert np.array_equal(got_k.view(np.uint8), want_k.view(np.uint8))
    assert np.array_equal(got_v, want_v)


def test_rts_ledger_is_3pn_and_ratio_holds(cuda):
    from paper_2206_01784_b200 import Executor, onesweep_sort, radix_plan, rts_sort

    n = 20_000
    keys = np.random.default_rng(17).integers(0, 2**32, size=n, dtype=np.uint32)
    cfg = radix_plan(32, 8)
    ex_rts, ex_one = Executor(), Executor()
    a = rts_sort(keys, cfg=cfg, executor=ex_rts)
    b = onesweep_sort(keys, cfg=cfg, executor=ex_one)
    assert np.array_equal(a, b)
    rts_ops = ex_rts.ledger_snapshot().element_ops
    one_ops = ex_one.ledger_snapshot().element_ops
    assert rts_ops == 3 * cfg.passes * n  # 12n
    assert one_ops == (2 * cfg.passes + 1) * n  # 9n


def test_rts_sort_tiny_inputs(cuda):
    from paper_2206_01784_b200 import rts_sort

    assert rts_sort(np.empty(0, dtype=np.uint32)).size == 0
    assert np.array_equal(rts_sort(np.array([7], dtype=np.uint32)), [7])
    assert np.array_equal(rts_sort(np.array([9, 3], dtype=np.int64)), [3, 9])


@pytest.mark.parametrize("n,q,pairs", [(1 << 24, 1, False), (12_345_679, 1, True),
                                       (1 << 22, 16, True), (3_000_001, 4, False)])
def test_rts_matches_onesweep_bytes(cuda, n, q, pairs):
    from paper_2206_01784_b200 import KeyGenSpec, generate_keys, onesweep_sort, rts_sort

    keys = generate_keys(KeyGenSpec(q=q, seed=n, n=n), device="cuda")
    if pairs:
        vals = torch.arange(n, dtype=torch.int32, device="cuda").view(torch.uint32)
        a = rts_sort(keys, vals)
        b = onesweep_sort(keys, vals)
        assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
    else:
        assert torch.equal(rts_sort(keys), onesweep_sort(keys))


def test_rts_all_equal_and_f64_pairs(cuda):
    from oracle import oracle
    from paper_2206_01784_b200 import rts_sort

    keys = np.full(300_000, 0xABACADAE, dtype=np.uint32)
    vals = np.arange(keys.size, dtype=np.uint32)
    k, v = rts_sort(keys, vals)
    assert np.array_equal(k, keys) and np.array_equal(v, vals)
    raw = np.random.default_rng(3).integers(0, 2**64, size=200_000, dtype=np.uint64)
    fk = raw.view(np.float64)
    fv = np.arange(fk.size, dtype=np.uint32)
    got = rts_sort(fk, fv)
    want = oracle.sort(fk, fv)
    assert np.array_equal(got[0].view(np.uint64), want[0].view(np.uint64))
    assert np.array_equal(got[1], want[1])


@pytest.mark.slow
def test_rts_sort_above_one_strip(cuda):
    # n > 2^28: the upsweep and the downsweep must tile every strip alike
    # (a whole-array upsweep left count rows unwritten)
    import torch

    from paper_2206_01784_b200 import KeyGenSpec, generate_keys, rts_sort

    n = (1 << 28) + 70_001
    keys = generate_keys(KeyGenSpec(q=1, seed=21, n=n), device="cuda")
    got = rts_sort(keys)
    want = torch.sort(keys.view(torch.int32).to(torch.int64) & 0xFFFFFFFF, stable=True).values
    assert torch.equal(got.view(torch.int32).to(torch.int64) & 0xFFFFFFFF, want)


@pytest.mark.parametrize("kb,d,tile,n", [(4, 8, 512, 20_000), (4, 3, 100, 3_001), (8, 5, 256, 9_000),
                                          (4, 8, 4096, 4_096), (8, 8, 1000, 12_345)])
def test_rts_building_blocks_match_oracle(cuda, kb, d, tile, n):
    """rts_upsweep / rts_block_prefix / rts_downsweep on the device
    (baseline.py:55-118) against numpy restatements of the reference's
    formulas: per-tile bincount, digit-major exclusive scan, and the stable
    partition (the oracle's partition pass with the same global offsets)."""
    from oracle import oracle
    from paper_2206_01784_b200 import (
        BlockHistogramTable, Executor, radix_plan, rts_block_prefix, rts_downsweep, rts_upsweep)

    rng = np.random.default_rng(n + d)
    dt = np.uint32 if kb == 4 else np.uint64
    keys = rng.integers(0, 2 ** (8 * kb), size=n, dtype=np.uint64).astype(dt)
    cfg = radix_plan(8 * kb, d, tile_size=tile)
    for place in (0, cfg.passes - 1):
        shift = cfg.digit_shift(place)
        digits = ((keys >> dt(shift)) & dt(cfg.radix - 1)).astype(np.int64)
        tiles = -(-n // tile)
        want = np.zeros((tiles, cfg.radix), np.int64)
        for t in range(tiles):
            want[t] = np.bincount(digits[t * tile:(t + 1) * tile], minlength=cfg.radix)
        ex = Executor()
        table = rts_upsweep(keys, place, cfg, ex)
        assert isinstance(table, BlockHistogramTable)
        assert np.array_equal(table.counts, want)
        offsets = rts_block_prefix(table)
        flat = want.T.reshape(-1)
        want_off = (np.cumsum(flat) - flat).reshape(cfg.radix, tiles).T
        assert np.array_equal(offsets, want_off)
        out = np.zeros_like(keys)
        vals = np.arange(n, dtype=np.uint64)
        out_v = np.zeros_like(vals)
        rts_downsweep(keys, place, offsets, out, cfg, ex, vals, out_v)
        base = np.zeros(cfg.radix, np.uint64)
        base[1:] = np.cumsum(want.sum(axis=0))[:-1]
        ref_k, ref_v = np.zeros_like(keys), np.zeros_like(vals)
        oracle.partition_pass(keys, ref_k, shift, d, base, vals, ref_v)
        assert np.array_equal(out, ref_k) and np.array_equal(out_v, ref_v)
        assert ex.ledger_snapshot().phase("upsweep").element_reads == n
        assert ex.ledger_snapshot().phase("downsweep").element_writes == n


def test_process_tile_chain_equals_partition_pass(cuda):
    """Host-driven tiles (binning.py:162-215) through process_tile, chained
    by a host CounterMatrix, place keys exactly as one device partition pass
    and leave the reference's final counter words."""
    from oracle import oracle
    from paper_2206_01784_b200 import CounterMatrix, process_tile, radix_plan

    rng = np.random.default_rng(5)
    n, tile = 5_000, 700
    cfg = radix_plan(32, 6, tile_size=tile)
    keys = rng.integers(0, 2**32, size=n, dtype=np.uint32)
    digits = (keys >> 6) & 63
    base = np.zeros(64, np.uint64)
    base[1:] = np.cumsum(np.bincount(digits, minlength=64))[:-1]
    tiles = -(-n // tile)
    m = CounterMatrix(tiles, cfg.radix)
    out = np.zeros_like(keys)
    carry = np.zeros(64, np.uint64)
    fast = 0
    for t in range(tiles):
        stats = process_tile(t, keys[t * tile:(t + 1) * tile], out, 1, base, m, cfg,
                             carry_out=carry if t == tiles - 1 else None)
        fast += stats.fast_path_tiles
        assert stats.element_reads == min(tile, n - t * tile)
    want = np.zeros_like(keys)
    _, _, words = oracle.partition_pass(keys, want, 6, 6, base, tile=tile, want_status=True)
    assert np.array_equal(out, want)
    assert np.array_equal(m.words.reshape(-1), words)
    assert np.array_equal(carry, base + np.bincount(digits, minlength=64).astype(np.uint64))
