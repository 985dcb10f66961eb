"""Device-side pass skipping (PassRoute, csrc/common.cuh): a digit place
whose histogram has one bin holding every key is an identity permutation,
so os_sort skips its pass and re-routes the ping-pong so the last sorting
pass still lands in the caller's output (with the key codec applied on the
first sorting pass's load and the last one's store).  Results must be
identical to the unskipped schedule and to the oracle, and every skipped
tile still counts as a one-run tile, as the reference counts them
(binning.py:201-205)."""

from __future__ import annotations

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sorted(keys, values=None):
    from paper_2206_01784_b200 import encode_array

    order = np.argsort(np.asarray(encode_array(np.asarray(keys))), kind="stable")
    return keys[order], (None if values is None else values[order])


CASES = {
    # (trivial places) u32 keys below 2^16: places 2 and 3 skipped (m = 2)
    "u32_low16": lambda r, n: r.integers(0, 1 << 16, n).astype(np.uint32),
    # only byte 1 varies: places 0, 2, 3 skipped (m = 1, odd)
    "u32_byte1": lambda r, n: (r.integers(0, 256, n).astype(np.uint32) << 8) | 0x5A0000A5,
    # all equal: every place trivial, the last pass copies (m = 0)
    "u32_equal": lambda r, n: np.full(n, 0xABACADAE, np.uint32),
    # signed keys with a constant sign and top bytes: codec on the routed passes
    "i32_small": lambda r, n: r.integers(-(1 << 11), 1 << 11, n).astype(np.int32),
    "f32_unit": lambda r, n: r.random(n).astype(np.float32) + np.float32(1.0),
    "f64_unit": lambda r, n: r.random(n) + 1.0,
    "i64_equal": lambda r, n: np.full(n, -42, np.int64),
    "u64_byte3": lambda r, n: (r.integers(0, 256, n).astype(np.uint64) << np.uint64(24)),
}


@pytest.mark.parametrize("case", sorted(CASES))
@pytest.mark.parametrize("with_values", [False, True])
def test_skipped_places_match_stable_sort(cuda, case, with_values):
    from paper_2206_01784_b200 import Executor, onesweep_sort

    r = np.random.default_rng(len(case))
    n = 200_003
    keys = CASES[case](r, n)
    vals = np.arange(n, dtype=np.uint32) if with_values else None
    ex = Executor()
    got = onesweep_sort(keys, vals, executor=ex)
    want_k, want_v = _sorted(keys, vals)
    if with_values:
        assert np.array_equal(got[0].view(np.uint8), want_k.view(np.uint8))
        assert np.array_equal(got[1], want_v)
    else:
        assert np.array_equal(got.view(np.uint8), want_k.view(np.uint8))


def test_multi_strip_and_all_tiles_fast(cuda):
    """small strips (carry chains) with two skipped places; all-equal keys
    count every tile of every pass as a one-run tile"""
    from paper_2206_01784_b200 import Executor, onesweep_sort, radix_plan

    r = np.random.default_rng(7)
    n = 50_000
    keys = r.integers(0, 1 << 16, n).astype(np.uint32)
    vals = np.arange(n, dtype=np.uint64)
    cfg = radix_plan(32, 8, tile_size=1024, strip_size=9_000)
    sk, sv = onesweep_sort(keys, vals, cfg)
    wk, wv = _sorted(keys, vals)
    assert np.array_equal(sk, wk) and np.array_equal(sv, wv)
    eq = np.full(n, 7, np.uint32)
    ex = Executor()
    sk, sv = onesweep_sort(eq, vals, radix_plan(32, 8, tile_size=1000), ex)
    assert np.array_equal(sk, eq) and np.array_equal(sv, vals)
    assert ex.ledger_snapshot().fast_path_tiles == 4 * 50  # 4 passes x 50 tiles


def test_in_place_sort_keeps_fixed_schedule(cuda):
    """keys_out == keys_in: routing is off (a skipped place would flip the
    parity), the even pass count keeps the in-place sort legal"""
    import torch

    from paper_2206_01784_b200 import DeviceSorter

    r = np.random.default_rng(3)
    n = 100_000
    keys_np = r.integers(0, 1 << 16, n).astype(np.uint32)
    keys = torch.from_numpy(keys_np.view(np.int32)).cuda().view(torch.uint32)
    s = DeviceSorter(n, torch.uint32, graphs=False)
    s(keys, keys)
    torch.cuda.synchronize()
    assert np.array_equal(keys.cpu().numpy(), np.sort(keys_np, kind="stable"))


def test_no_skip_switch_gives_same_bytes(cuda, tmp_path):
    """ONESWEEP_B200_NO_SKIP=1 (fixed schedule) and the routed schedule agree"""
    code = (
        "import numpy as np, sys\n"
        "from paper_2206_01784_b200 import onesweep_sort\n"
        "r = np.random.default_rng(1)\n"
        "k = (r.integers(0, 1 << 12, 123_457).astype(np.int64) << 20) - (1 << 31)\n"
        "v = np.arange(k.size, dtype=np.uint16)\n"
        "sk, sv = onesweep_sort(k, v)\n"
        "np.save(sys.argv[1], np.concatenate([sk.view(np.uint8), sv.view(np.uint8)]))\n")
    outs = []
    for flag in ("0", "1"):
        out = tmp_path / f"o{flag}.npy"
        env = dict(os.environ, ONESWEEP_B200_NO_SKIP=flag, PYTHONPATH=ROOT)
        subprocess.run([sys.executable, "-c", code, str(out)], check=True, env=env, cwd=ROOT)
        outs.append(np.load(out))
    assert np.array_equal(outs[0], outs[1])


def test_skipped_places_reported(cuda):
    """DeviceSorter.skipped_places / os_sort_skipped_places and the device
    element count of the ledger follow the plan"""
    import torch

    from paper_2206_01784_b200 import DeviceSorter, Executor, onesweep_sort

    r = np.random.default_rng(5)
    n = 60_000
    cases = [
        (r.integers(0, 1 << 16, n).astype(np.uint32), [False, False, True, True]),
        (np.full(n, 9, np.uint32), [True, True, True, False]),  # the last place runs as the copy
        (r.integers(0, 1 << 20, n).astype(np.int64), [False, False, False, True, True, True, True, False]),
        (r.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32), [False] * 4),
    ]
    for keys, want in cases:
        t = torch.from_numpy(keys).cuda()
        s = DeviceSorter(n, t.dtype, graphs=False)
        out = torch.empty_like(t)
        s(t, out)
        assert s.skipped_places() == want, (keys.dtype, want)
        ex = Executor()
        onesweep_sort(keys, executor=ex)
        assert ex.device_element_ops == (1 + 2 * (len(want) - sum(want))) * n
