"""GPU parity at the BASELINE sizes, on exactly the inputs bench.py and
tools/bench_configs.py time.

* C2 (the headline): the bench's own input, 2^28 keys from the reference key
  generator (q=1, seed 0), sorted through DeviceSorter exactly as bench.py
  does, compared byte for byte with the oracle's multi-threaded C port of the
  reference onesweep_sort (oracle/onesweep_oracle.c, pinned to the reference
  by tests/test_oracle.py).
* C3: 2^28 pairs for the distributions the survey names that the 256M
  property test in test_gpu_scale.py does not cover (q=2, q=8, all-equal,
  presorted), keys and values byte for byte against the oracle.
* C4: 2^28 u64 / i64 / f64 keys with a u32 index payload, checked by the
  properties that pin the unique stable sort.
* 1-GPU 2^31 keys (8 strips per pass: the C5 denominator), index payload,
  checked on the device in chunks by the same properties.

The property check (sorted by encoded key + out == in[idx] + idx is a
permutation + idx ascending among equal keys) is equivalent to equality with
the reference's stable sort (binning.py:278-337; the oracle contract of
test_binning.py:315-329)."""

from __future__ import annotations

import os

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

THREADS = max(1, os.cpu_count() or 1)


def _c2_keys(n, q=1, seed=0, bits=32):
    from paper_2206_01784_b200 import KeyGenSpec, generate_keys

    return generate_keys(KeyGenSpec(q=q, seed=seed, n=n, key_bits=bits), device="cuda")


def test_c2_bench_input_bit_exact_vs_oracle(cuda, oracle):
    import torch

    from paper_2206_01784_b200 import DeviceSorter

    n = 1 << 28
    keys = _c2_keys(n)
    out = torch.empty_like(keys)
    sorter = DeviceSorter(n, keys.dtype, 0, 8, device=keys.device)  # bench.py's sorter
    sorter(keys, out)
    torch.cuda.synchronize()
    k_in = keys.cpu().numpy()
    got = out.cpu().numpy()
    del out
    assert np.array_equal(keys.cpu().numpy(), k_in), "input modified"
    want = oracle.sort(k_in, threads=THREADS)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("dist", ["q2", "q8", "all_equal", "presorted"])
def test_c3_pairs_256M_bit_exact_vs_oracle(cuda, oracle, dist):
    import torch

    from paper_2206_01784_b200 import onesweep_sort

    n = 1 << 28
    if dist == "all_equal":  # test_binning.py:377
        keys = torch.full((n,), 0xABACADAE - (1 << 32), dtype=torch.int32, device="cuda").view(torch.uint32)
    elif dist == "presorted":  # np.sort of the q=1 keys
        k = _c2_keys(n)
        keys = onesweep_sort(k)
        del k
    else:
        keys = _c2_keys(n, q=int(dist[1:]), seed=int(dist[1:]))
    idx = torch.arange(n, dtype=torch.int32, device="cuda").view(torch.uint32)
    sk, sv = onesweep_sort(keys, idx)
    torch.cuda.synchronize()
    k_in = keys.cpu().numpy()
    del keys
    got_k, got_v = sk.cpu().numpy(), sv.cpu().numpy()
    del sk, sv
    want_k, want_v = oracle.sort(k_in, np.arange(n, dtype=np.uint32), threads=THREADS)
    assert np.array_equal(got_k, want_k)
    assert np.array_equal(got_v, want_v)


def _device_stable_check(k_in, k_out, idx_out, enc_out, chunk=1 << 27):
    """Chunked on-device check that (k_out, idx_out) is the stable sort of
    k_in.  enc_out(lo, hi) returns int64 whose signed order is the encoded
    (unsigned) key order of k_out[lo:hi]."""
    import torch

    n = k_in.numel()
    iv = torch.int64 if k_in.element_size() == 8 else torch.int32
    kin, kout = k_in.view(iv), k_out.view(iv)
    seen = torch.zeros(n, dtype=torch.uint8, device=k_in.device)
    prev_e = prev_i = None
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        e = enc_out(lo, hi)
        i = idx_out[lo:hi].view(torch.int32).to(torch.int64) & 0xFFFFFFFF
        assert torch.equal(kin[i], kout[lo:hi]), f"out != in[idx] in [{lo}, {hi})"
        seen[i] = 1
        if prev_e is not None:  # include the pair across the chunk boundary
            e = torch.cat([prev_e, e])
            i = torch.cat([prev_i, i])
        assert bool((e[1:] >= e[:-1]).all()), f"not sorted in [{lo}, {hi})"
        same = e[1:] == e[:-1]
        assert bool((i[1:][same] > i[:-1][same]).all()), f"unstable in [{lo}, {hi})"
        prev_e, prev_i = e[-1:].clone(), i[-1:].clone()
        del e, i, same
    assert int(seen.sum(dtype=torch.int64)) == n, "index payload is not a permutation"


@pytest.mark.parametrize("dt", ["u64", "i64", "f64"])
def test_c4_u64_pairs_256M_properties(cuda, oracle, dt):
    import torch

    from paper_2206_01784_b200 import onesweep_sort

    n = 1 << 28
    raw = _c2_keys(n, bits=64)
    tdt = {"u64": torch.uint64, "i64": torch.int64, "f64": torch.float64}[dt]
    keys = raw.view(tdt)
    idx = torch.arange(n, dtype=torch.int32, device="cuda").view(torch.uint32)
    sk, sv = onesweep_sort(keys, idx)
    torch.cuda.synchronize()
    sign = -(1 << 63)

    def enc(x):  # keycodec.py:157-181 on int64 bit patterns, as a signed-order int64
        b = x.view(torch.int64)
        if dt == "u64":
            return b ^ sign
        if dt == "i64":
            return b
        # float: negative -> ~x, else x | sign; then flip back to signed order
        return torch.where(b < 0, ~b, b | sign) ^ sign

    _device_stable_check(keys, sk, sv, lambda lo, hi: enc(sk[lo:hi]))
    # a small exact slice against the oracle as well
    m = 1 << 20
    part_k = keys[:m].cpu().numpy()
    got_k, got_v = onesweep_sort(part_k, np.arange(m, dtype=np.uint32))
    want_k, want_v = oracle.sort(part_k, np.arange(m, dtype=np.uint32), threads=THREADS)
    assert np.array_equal(got_k.view(np.uint64), want_k.view(np.uint64))
    assert np.array_equal(got_v, want_v)


def test_single_gpu_2e31_keys_eight_strips(cuda):
    import torch

    from paper_2206_01784_b200 import onesweep_sort

    n = 1 << 31
    free, _ = torch.cuda.mem_get_info()
    if free < 60 * (1 << 30):
        pytest.skip("needs ~60 GiB of free device memory")
    keys = _c2_keys(n)  # C5's global input on one GPU
    idx = torch.arange(n, dtype=torch.int64, device="cuda").to(torch.int32).view(torch.uint32)
    sk, sv = onesweep_sort(keys, idx)
    torch.cuda.synchronize()
    del idx

    def enc(lo, hi):
        return sk[lo:hi].view(torch.int32).to(torch.int64) & 0xFFFFFFFF

    _device_stable_check(keys, sk, sv, enc)
