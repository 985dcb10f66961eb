"""GPU: the sharded sort with the real kernels (MSD histogram, MSD partition,
local Onesweep) on one B200, two ranks sharing cuda:0 over gloo (the
exchange is staged through host memory; with NCCL it stays on device)."""

from __future__ import annotations

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, shards, vals, results):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2206_01784_b200.distributed import sharded_sort

    k = torch.from_numpy(shards[rank]).cuda()
    v = torch.from_numpy(vals[rank]).cuda() if vals is not None else None
    out = sharded_sort(k, v)
    if vals is None:
        results[rank] = (out.cpu().numpy(), None)
    else:
        results[rank] = (out[0].cpu().numpy(), out[1].cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


def _run(world, shards, vals=None):
    from test_distributed_cpu import _free_port

    port = _free_port()
    with mp.Manager() as m:
        results = m.dict()
        mp.spawn(_worker, args=(world, port, shards, vals, results), nprocs=world, join=True)
        return [results[r] for r in range(world)]


@pytest.mark.parametrize("dtype", [np.uint32, np.float32, np.int64])
def test_sharded_sort_on_device(cuda, dtype):
    from oracle import oracle

    rng = np.random.default_rng(3)
    world = 2
    bits = np.dtype(dtype).itemsize * 8
    shards = []
    for _ in range(world):
        raw = rng.integers(0, 2**bits, size=int(rng.integers(150_000, 250_000)), dtype=np.uint64)
        shards.append((raw.astype(np.uint32) if bits == 32 else raw).view(dtype))
    vals, start = [], 0
    for s in shards:
        vals.append(np.arange(start, start + s.size, dtype=np.uint32))
        start += s.size
    res = _run(world, shards, vals)
    got_k = np.concatenate([r[0] for r in res])
    got_v = np.concatenate([r[1] for r in res])
    want_k, want_v = oracle.sharded_sort(shards, vals)
    u = np.uint32 if bits == 32 else np.uint64
    assert np.array_equal(got_k.view(u), want_k.view(u))
    assert np.array_equal(got_v, want_v)


def test_msd_partition_is_stable_segmentation(cuda):
    from oracle import oracle
    from paper_2206_01784_b200.distributed import DeviceOps
    from paper_2206_01784_b200.keycodec import spec_for_dtype

    rng = np.random.default_rng(5)
    keys = rng.integers(0, 2**32, size=300_001, dtype=np.uint32)
    vals = np.arange(keys.size, dtype=np.uint32)
    ops = DeviceOps()
    spec = spec_for_dtype(np.uint32)
    tk = torch.from_numpy(keys).cuda()
    hist = ops.top_histogram(tk, spec, 8).cpu().numpy()
    assert np.array_equal(hist, np.bincount(keys >> 24, minlength=256))
    bin_lo = [0, 40, 41, 200, 256]
    top = (keys >> 24).astype(np.int64)
    dest = np.searchsorted(np.asarray(bin_lo[1:-1]), top, side="right")
    send = np.bincount(dest, minlength=4).tolist()
    pk, pv = ops.partition(tk, torch.from_numpy(vals).cuda(), spec, 8, bin_lo, send)
    order = np.argsort(dest, kind="stable")
    assert np.array_equal(pk.cpu().numpy(), keys[order])
    assert np.array_equal(pv.cpu().numpy(), vals[order])
