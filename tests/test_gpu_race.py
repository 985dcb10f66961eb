"""Race and failure exploration on the device.

The reference explores thread interleavings with a seeded Jitter between the
L publish and the look-back (executor.py:108-121, binning.py:187-193) and makes
waiters abort instead of hanging (lookback.py:176-189).  The B200 equivalents
live in the debug twin of the library, _lib/libonesweep_b200_debug.so
(Makefile DEBUG_FLAGS: -DOS_JITTER=1, 2^16-poll watchdog):

* jitter: pseudo-random __nanosleep (up to 20 us) before the L publish, before
  the look-back and before the G publish, per (tile, digit) -- tiles publish
  out of order and look-backs meet unpublished (N) words.  The parity cases
  below must stay bit-exact against the oracle under it.
* watchdog: ONESWEEP_B200_DEBUG_STALL_TILE=t makes tile t skip its publishes;
  its successors must trap after the spin limit and the call must raise
  RuntimeError (not hang the GPU).

Each case runs in a subprocess (a trapped kernel poisons the CUDA context)."""

from __future__ import annotations

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEBUG_LIB = os.path.join(ROOT, "paper_2206_01784_b200", "_lib", "libonesweep_b200_debug.so")

PARITY = r"""
import sys
import numpy as np
sys.path.insert(0, {root!r})
from oracle import oracle
from paper_2206_01784_b200 import _native, onesweep_sort, partition_pass, radix_plan
assert "debug" in _native.load().os_version().decode(), _native.load().os_version()
rng = np.random.default_rng({seed})
cases = 0
for n, dt, d, tile, strip, vals in [
    (200_000, np.uint32, 8, 256, 1 << 28, False),     # 782 tiles, deep chains
    (150_001, np.uint32, 8, 512, 30_000, True),       # ragged, several strips
    (100_000, np.uint64, 8, 1024, 1 << 28, True),     # 64-bit keys
    (120_000, np.int32, 6, 300, 50_000, True),        # signed, 6-bit digits
    (90_000, np.float64, 8, 0, 1 << 28, False),       # device tile
    (60_000, np.uint32, 8, 64, 1 << 28, False),       # 938 tiny tiles
]:
    bits = np.dtype(dt).itemsize * 8
    raw = rng.integers(0, 2**bits, size=n, dtype=np.uint64)
    keys = (raw if bits == 64 else raw.astype(np.uint32)).view(dt)
    if dt in (np.uint32,) and n == 60_000:
        keys = (keys & 0x0F0F0F0F).astype(dt)          # heavy duplicates
    cfg = radix_plan(bits, d, tile_size=tile or 8192, strip_size=strip)
    v = np.arange(n, dtype=np.uint32) if vals else None
    got = onesweep_sort(keys, v, cfg if tile else None)
    want = oracle.sort(keys, v, digit_bits=d)
    u = np.uint64 if bits == 64 else np.uint32  # bit patterns: NaN keys compare equal
    if vals:
        assert np.array_equal(got[0].view(u), want[0].view(u)) and np.array_equal(got[1], want[1]), (n, dt)
    else:
        assert np.array_equal(got.view(u), want.view(u)), (n, dt)
    cases += 1
# a pass's final status words under jitter equal the sequential CounterMatrix
src = rng.integers(0, 2**32, size=40_000, dtype=np.uint32)
cfg = radix_plan(32, 8, tile_size=128)
dig = (src >> 8) & 0xFF
base = np.zeros(256, np.uint64); np.cumsum(np.bincount(dig, minlength=256)[:-1], out=base[1:])
dst = np.zeros_like(src)
_, views = partition_pass(src, dst, 1, base, cfg, return_status=True)
want_dst = np.zeros_like(src)
_, _, words = oracle.partition_pass(src, want_dst, 8, 8, base, tile=128, want_status=True)
assert np.array_equal(dst, want_dst)
assert np.array_equal(views[0].words.reshape(-1), words)
print("JITTER_PARITY_OK", cases + 1)
"""

STALL = r"""
import sys
import numpy as np
sys.path.insert(0, {root!r})
from paper_2206_01784_b200 import onesweep_sort, radix_plan
keys = np.random.default_rng(0).integers(0, 2**32, size=100_000, dtype=np.uint32)
try:
    onesweep_sort(keys, cfg=radix_plan(32, 8, tile_size=1024))
except RuntimeError as e:
    print("WATCHDOG_TRAPPED", str(e)[:200])
    sys.exit(0)
print("NO_TRAP")
sys.exit(1)
"""


def _run(code: str, env_extra: dict, timeout: int):
    env = dict(os.environ)
    env["ONESWEEP_B200_LIB"] = DEBUG_LIB
    env.update(env_extra)
    return subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                          timeout=timeout, cwd=ROOT)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_parity_under_lookback_jitter(cuda, seed):
    if not os.path.exists(DEBUG_LIB):
        pytest.fail("debug library missing: run `make` (it builds libonesweep_b200_debug.so)")
    r = _run(PARITY.format(root=ROOT, seed=seed), {}, timeout=600)
    assert r.returncode == 0 and "JITTER_PARITY_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]


def test_watchdog_traps_a_stalled_lookback(cuda):
    if not os.path.exists(DEBUG_LIB):
        pytest.fail("debug library missing: run `make`")
    r = _run(STALL.format(root=ROOT), {"ONESWEEP_B200_DEBUG_STALL_TILE": "5",
                                       "ONESWEEP_B200_SYNC_CHECK": "1"}, timeout=300)
    assert r.returncode == 0 and "WATCHDOG_TRAPPED" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]
