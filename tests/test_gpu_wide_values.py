"""Values of any width (the reference reorders values of any numpy dtype,
binning.py:301-304): widths other than 1/2/4/8 bytes travel through the
passes as an index payload and are gathered once (os_gather_rows).  Checked
against numpy's stable argsort of the encoded keys -- a permutation, so
bit-exact."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rng_values(n, dtype, rng):
    raw = rng.integers(0, 256, size=n * np.dtype(dtype).itemsize, dtype=np.uint8)
    return raw.view(dtype)


def _same(a, b) -> bool:
    """Bit-equal values; structured dtypes field by field (padding bytes carry
    no data and numpy's copies do not preserve them)."""
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    if a.dtype.names:
        return all(_same(a[f], b[f]) for f in a.dtype.names)
    return np.array_equal(a.view(np.uint8), b.view(np.uint8))


def _order(keys):
    from paper_2206_01784_b200 import encode_array

    enc = np.asarray(encode_array(np.asarray(keys)))
    return np.argsort(enc, kind="stable")


STRUCT = np.dtype([("a", "<u4"), ("b", "<f8")])          # 12 bytes, packed
STRUCT_ALIGNED = np.dtype([("a", "<u4"), ("b", "<f8")], align=True)  # 16 bytes


@pytest.mark.parametrize("vdt", [np.complex128, STRUCT, STRUCT_ALIGNED, "S5", "V3", "V24"])
@pytest.mark.parametrize("kdt", [np.uint32, np.int64, np.float32])
@pytest.mark.parametrize("n", [1, 2, 3000, 70001])
def test_onesweep_sort_wide_values(cuda, kdt, vdt, n):
    from paper_2206_01784_b200 import onesweep_sort

    rng = np.random.default_rng(n + np.dtype(vdt).itemsize)
    keys = rng.integers(0, 1 << 20, size=n).astype(kdt)  # duplicates: stability matters
    vals = _rng_values(n, vdt, rng)
    sk, sv = onesweep_sort(keys, vals)
    order = _order(keys)
    assert np.array_equal(sk.view(np.uint8), keys[order].view(np.uint8))
    assert sv.dtype == vals.dtype and sv.shape == vals.shape
    assert _same(sv, vals[order])


def test_onesweep_sort_complex_tensor(cuda):
    import torch

    from paper_2206_01784_b200 import onesweep_sort

    n = 50_000
    g = torch.Generator(device="cpu").manual_seed(5)
    keys = torch.randint(0, 1000, (n,), generator=g, dtype=torch.int32).cuda()
    vals = torch.randn(n, dtype=torch.complex128, generator=g).cuda()
    sk, sv = onesweep_sort(keys, vals)
    order = torch.sort(keys.to(torch.int64), stable=True).indices
    assert torch.equal(sk, keys[order])
    assert sv.dtype == torch.complex128 and torch.equal(sv, vals[order])


def test_partition_pass_wide_values(cuda):
    from paper_2206_01784_b200 import global_bin_offsets, global_histograms, partition_pass, radix_plan

    n = 40_000
    rng = np.random.default_rng(11)
    keys = rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32)
    vals = _rng_values(n, STRUCT, rng)
    cfg = radix_plan(32, 8, 4096)
    offsets = global_bin_offsets(global_histograms(keys, cfg)).row(1)
    dk = np.empty_like(keys)
    dv = np.empty_like(vals)
    partition_pass(keys, dk, 1, offsets, cfg, src_values=vals, dst_values=dv)
    order = np.argsort((keys >> 8) & 0xFF, kind="stable")
    assert np.array_equal(dk, keys[order])
    assert _same(dv, vals[order])


def test_rts_and_oracle_wide_values(cuda):
    from paper_2206_01784_b200 import oracle_stable_sort, rts_sort

    n = 30_000
    rng = np.random.default_rng(3)
    keys = rng.integers(-500, 500, size=n).astype(np.int32)
    vals = _rng_values(n, "V10", rng)
    order = _order(keys)
    for fn in (rts_sort, oracle_stable_sort):
        sk, sv = fn(keys, vals)
        assert np.array_equal(sk, keys[order]), fn.__name__
        assert _same(sv, vals[order]), fn.__name__


@pytest.mark.parametrize("row_bytes", [1, 3, 8, 16, 40])
@pytest.mark.parametrize("index_bytes", [4, 8])
def test_gather_rows_abi(cuda, row_bytes, index_bytes):
    import torch

    from paper_2206_01784_b200 import _native

    n = 10_007
    src = torch.randint(0, 256, (n, row_bytes), dtype=torch.uint8, device="cuda")
    perm = torch.randperm(n, device="cuda")
    idx = perm.to(torch.int32) if index_bytes == 4 else perm
    dst = torch.empty_like(src)
    L = _native.load()
    _native.check(L.os_gather_rows(src.data_ptr(), idx.data_ptr(), index_bytes, dst.data_ptr(), n,
                                   row_bytes, None), "gather_rows")
    torch.cuda.synchronize()
    assert torch.equal(dst, src[perm])
