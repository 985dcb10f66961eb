"""CPU: the multi-GPU sharded sort's host logic with world_size 2/3 over gloo.

The device steps (top-digit histogram, MSD partition, local Onesweep) are
swapped for oracle-backed stand-ins -- test infrastructure only -- so the
split planning, count exchange, all-to-all and stability argument are
exercised end to end on CPU.  The GPU test (tests/test_gpu_distributed.py)
runs the same orchestration with the real kernels."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


class OracleOps:
    """Test-only CPU stand-ins for distributed.DeviceOps."""

    def top_histogram(self, keys, spec, digit_bits):
        from oracle import oracle

        enc = oracle.encode(keys.numpy())
        top = (enc >> enc.dtype.type(spec.bits - digit_bits)).astype(np.int64)
        return torch.from_numpy(np.bincount(top, minlength=1 << digit_bits).astype(np.int64)).view(torch.uint64)

    def partition(self, keys, values, spec, digit_bits, bin_lo, send):
        from oracle import oracle

        enc = oracle.encode(keys.numpy())
        top = (enc >> enc.dtype.type(spec.bits - digit_bits)).astype(np.int64)
        dest = np.searchsorted(np.asarray(bin_lo[1:-1]), top, side="right")
        order = np.argsort(dest, kind="stable")
        assert np.array_equal(np.bincount(dest, minlength=len(send)), send)
        pk = torch.from_numpy(keys.numpy()[order].copy())
        pv = None if values is None else torch.from_numpy(values.numpy()[order].copy())
        return pk, pv

    def local_sort(self, keys, values):
        from oracle import oracle

        if values is None:
            return torch.from_numpy(oracle.sort(keys.numpy())), None
        k, v = oracle.sort(keys.numpy(), values.numpy())
        return torch.from_numpy(k), torch.from_numpy(v)


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, shards, vals, results):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2206_01784_b200.distributed import sharded_sort

    k = torch.from_numpy(shards[rank])
    v = torch.from_numpy(vals[rank]) if vals is not None else None
    out, plan = sharded_sort(k, v, ops=OracleOps(), return_plan=True)
    if vals is None:
        results[rank] = (out.numpy(), None, plan)
    else:
        results[rank] = (out[0].numpy(), out[1].numpy(), plan)
    dist.barrier()
    dist.destroy_process_group()


def _run(world, shards, vals=None):
    port = _free_port()
    with mp.Manager() as m:
        results = m.dict()
        mp.spawn(_worker, args=(world, port, shards, vals, results), nprocs=world, join=True)
        return [results[r] for r in range(world)]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_sort_equals_global_stable_sort(world):
    from oracle import oracle

    rng = np.random.default_rng(world)
    shards = [rng.integers(0, 2**32, size=int(rng.integers(3000, 6000)), dtype=np.uint32)
              for _ in range(world)]
    vals = []
    start = 0
    for s in shards:
        vals.append(np.arange(start, start + s.size, dtype=np.uint32))
        start += s.size
    res = _run(world, shards, vals)
    got_k = np.concatenate([r[0] for r in res])
    got_v = np.concatenate([r[1] for r in res])
    want_k, want_v = oracle.sharded_sort(shards, vals)
    assert np.array_equal(got_k, want_k)
    assert np.array_equal(got_v, want_v)
    plans = [r[2] for r in res]
    assert all(p["bin_lo"] == plans[0]["bin_lo"] for p in plans)  # same plan on every rank
    sizes = [r[0].size for r in res]
    total = sum(s.size for s in shards)
    assert max(sizes) <= total / world * 1.2  # whole-bin split balances uniform keys


def test_sharded_sort_signed_keys_heavy_duplicates():
    from oracle import oracle

    rng = np.random.default_rng(9)
    shards = [rng.integers(-3, 3, size=2000).astype(np.int64) for _ in range(2)]
    vals = [np.arange(2000, dtype=np.uint64), np.arange(2000, 4000, dtype=np.uint64)]
    res = _run(2, shards, vals)
    got_k = np.concatenate([r[0] for r in res])
    got_v = np.concatenate([r[1] for r in res])
    want_k, want_v = oracle.sharded_sort(shards, vals)
    assert np.array_equal(got_k, want_k) and np.array_equal(got_v, want_v)


def test_plan_split_properties():
    from paper_2206_01784_b200.distributed import exchange_counts, plan_split

    rng = np.random.default_rng(0)
    table = rng.integers(0, 1000, size=(4, 256)).astype(np.uint64)
    lo = plan_split(table, 4)
    assert lo[0] == 0 and lo[-1] == 256 and all(a <= b for a, b in zip(lo, lo[1:]))
    sends = [exchange_counts(table, lo, r)[0] for r in range(4)]
    recvs = [exchange_counts(table, lo, r)[1] for r in range(4)]
    for src in range(4):
        for dst in range(4):
            assert sends[src][dst] == recvs[dst][src]
    assert sum(map(sum, sends)) == int(table.sum())
    # everything in one bin: one destination takes it all, others empty
    skew = np.zeros((2, 256), dtype=np.uint64)
    skew[:, 17] = 100
    lo = plan_split(skew, 2)
    s0, _ = exchange_counts(skew, lo, 0)
    assert sorted(s0) == [0, 100]


def test_p2p_receive_offsets_and_dest_index():
    """Host logic of the fused exchange: source segments are concatenated in
    rank order at each destination, and the u64 destination index reaches the
    peer slot from the local base modulo 2^64 (peer below or above)."""
    from paper_2206_01784_b200.distributed import (exchange_counts, p2p_dest_index, plan_split,
                                                   receive_offsets)

    rng = np.random.default_rng(7)
    world = 4
    table = rng.integers(0, 1000, size=(world, 256)).astype(np.uint64)
    bin_lo = plan_split(table, world)
    for rank in range(world):
        off = receive_offsets(table, bin_lo, rank)
        send, _ = exchange_counts(table, bin_lo, rank)
        for g in range(world):
            # this rank's segment ends where the next source's begins
            nxt = receive_offsets(table, bin_lo, rank + 1)[g] if rank + 1 < world else None
            if nxt is not None:
                assert off[g] + send[g] == nxt
        assert off == [int(table[:rank, bin_lo[g]:bin_lo[g + 1]].sum()) for g in range(world)]
    ptrs = [0x7F0000000000, 0x7E0000001000, 0x7F8000000200, 0x100]
    for eb in (4, 8):
        for rank in range(world):
            off = receive_offsets(table, bin_lo, rank)
            idx = p2p_dest_index(ptrs, ptrs[rank], eb, off)
            for g in range(world):
                assert (ptrs[rank] + int(idx[g]) * eb) % (1 << 64) == ptrs[g] + off[g] * eb
    with pytest.raises(ValueError):
        p2p_dest_index([0x1000, 0x1002], 0x1000, 4, [0, 0])
