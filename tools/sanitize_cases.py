"""Small device sorts for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): keys-only, pairs, 64-bit keys, ragged and misaligned inputs, tiny
tiles, strips, wide digits, the reduce-then-scan ablation and the single-GPU
p2p emulation -- every kernel of the library.  Each case is checked against
the oracle, so a run also proves the results are right under the tool.
usage: compute-sanitizer --tool memcheck python tools/sanitize_cases.py [case...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle  # noqa: E402
from paper_2206_01784_b200 import (  # noqa: E402
    encode_array,
    global_histograms, onesweep_sort, partition_pass, radix_plan, rts_sort)
from paper_2206_01784_b200.distributed import emulate_p2p_sort  # noqa: E402

rng = np.random.default_rng(7)


def eq(a, b, u):
    return np.array_equal(np.asarray(a).view(u), np.asarray(b).view(u))


def case_keys():
    k = rng.integers(0, 2**32, size=40_000, dtype=np.uint32)
    assert eq(onesweep_sort(k), oracle.sort(k), np.uint32)


def case_pairs():
    k = rng.integers(0, 2**32, size=30_001, dtype=np.uint32).view(np.float32)
    v = np.arange(k.size, dtype=np.uint32)
    gk, gv = onesweep_sort(k, v)
    wk, wv = oracle.sort(k, v)
    assert eq(gk, wk, np.uint32) and np.array_equal(gv, wv)


def case_u64():
    k = rng.integers(0, 2**63, size=20_000, dtype=np.int64)
    v = np.arange(k.size, dtype=np.uint32)
    gk, gv = onesweep_sort(k, v)
    wk, wv = oracle.sort(k, v)
    assert eq(gk, wk, np.uint64) and np.array_equal(gv, wv)


def case_ragged_misaligned():
    base = torch.from_numpy(rng.integers(0, 2**32, size=25_003, dtype=np.uint32)).cuda()
    t = base[3:]
    got = onesweep_sort(t).cpu().numpy()
    assert eq(got, oracle.sort(base[3:].cpu().numpy()), np.uint32)


def case_tiny_tiles_strips():
    k = rng.integers(0, 2**32, size=30_000, dtype=np.uint32)
    v = np.arange(k.size, dtype=np.uint64)
    gk, gv = onesweep_sort(k, v, radix_plan(32, 8, tile_size=64, strip_size=7000))
    wk, wv = oracle.sort(k, v)
    assert eq(gk, wk, np.uint32) and np.array_equal(gv, wv)


def case_wide():
    k = rng.integers(0, 2**32, size=20_000, dtype=np.uint32)
    cfg = radix_plan(32, 12, tile_size=1024)
    h = global_histograms(k, cfg)
    assert np.array_equal(h.counts, oracle.histogram(k, 12))
    d = (k >> 12) & 0xFFF
    base = np.zeros(4096, np.uint64)
    np.cumsum(np.bincount(d, minlength=4096)[:-1], out=base[1:])
    dst = np.zeros_like(k)
    partition_pass(k, dst, 1, base, cfg)
    want = np.zeros_like(k)
    oracle.partition_pass(k, want, 12, 12, base)
    assert np.array_equal(dst, want)


def case_rts():
    k = rng.integers(0, 2**32, size=30_000, dtype=np.uint32)
    v = np.arange(k.size, dtype=np.uint32)
    gk, gv = rts_sort(k, v)
    wk, wv = oracle.sort(k, v)
    assert eq(gk, wk, np.uint32) and np.array_equal(gv, wv)


def case_p2p_emulation():
    shards = [torch.from_numpy(rng.integers(0, 2**32, size=m, dtype=np.uint32)).cuda()
              for m in (9000, 7001, 12000)]
    outs, _ = emulate_p2p_sort(shards)
    got = np.concatenate([o.cpu().numpy() for o in outs])
    want = oracle.sort(np.concatenate([s.cpu().numpy() for s in shards]))
    assert eq(got, want, np.uint32)


def case_wide_values():
    k = rng.integers(0, 1 << 12, size=20_000, dtype=np.uint32)
    v = rng.standard_normal(k.size) + 1j * rng.standard_normal(k.size)  # complex128: gathered
    gk, gv = onesweep_sort(k, v)
    order = np.argsort(k, kind="stable")
    assert np.array_equal(gk, k[order]) and np.array_equal(gv, v[order])


def case_value_widths():
    """every (key, value) width geometry: values stashed in TMEM (1/2/8 bytes)"""
    for kdt in (np.uint32, np.int64):
        k = rng.integers(0, 1 << 20, size=20_001).astype(kdt)
        order = np.argsort(np.asarray(encode_array(k)), kind="stable")
        assert np.array_equal(onesweep_sort(k).view(np.uint8), k[order].view(np.uint8))
        for vdt in (np.uint8, np.int16, np.int64):
            v = rng.integers(0, 1 << 7, size=k.size).astype(vdt)
            gk, gv = onesweep_sort(k, v)
            assert np.array_equal(gk.view(np.uint8), k[order].view(np.uint8)) and np.array_equal(gv, v[order])


def case_skipped_places():
    """device-side pass skipping: small-range keys (two places skipped), all-equal pairs
    (every place but the last skipped), small signed 64-bit keys (middle places skipped)"""
    k = rng.integers(0, 1 << 16, size=30_001).astype(np.uint32)
    assert np.array_equal(onesweep_sort(k), np.sort(k, kind="stable"))
    eq = np.full(25_000, 0x1234, np.uint32)
    v = np.arange(eq.size, dtype=np.uint32)
    gk, gv = onesweep_sort(eq, v)
    assert np.array_equal(gk, eq) and np.array_equal(gv, v)
    s = rng.integers(-(1 << 20), 1 << 20, size=20_000).astype(np.int64)
    gk, gv = onesweep_sort(s, v[:s.size])
    order = np.argsort(s, kind="stable")
    assert np.array_equal(gk, s[order]) and np.array_equal(gv, v[:s.size][order])


CASES = {k[5:]: v for k, v in globals().items() if k.startswith("case_")}
for name in (sys.argv[1:] or list(CASES)):
    CASES[name]()
    torch.cuda.synchronize()
    print("case ok:", name, flush=True)
torch.cuda.empty_cache()  # the caching allocator's blocks are not leaks
print("SANITIZE_CASES_OK")
