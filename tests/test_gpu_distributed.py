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


def _p2p_case(world, dtype, sizes, q=1, with_values=True, seed=11):
    from oracle import oracle
    from paper_2206_01784_b200.distributed import emulate_p2p_sort

    rng = np.random.default_rng(seed)
    bits = np.dtype(dtype).itemsize * 8
    shards = []
    for n in sizes:
        raw = np.full(n, (1 << bits) - 1, dtype=np.uint64)
        for _ in range(q):  # AND of q words: the keygen's entropy reduction
            raw &= rng.integers(0, 2**bits, size=n, dtype=np.uint64)
        shards.append((raw.astype(np.uint32) if bits == 32 else raw).view(dtype))
    vdt = np.uint32 if bits == 32 else np.uint64
    vals, start = [], 0
    for s in shards:
        vals.append(np.arange(start, start + s.size, dtype=vdt))
        start += s.size
    tk = [torch.from_numpy(s).cuda() for s in shards]
    tv = [torch.from_numpy(v).cuda() for v in vals] if with_values else None
    out, plan = emulate_p2p_sort(tk, tv)
    if with_values:
        got_k = np.concatenate([o[0].cpu().numpy() for o in out])
        got_v = np.concatenate([o[1].cpu().numpy() for o in out])
    else:
        got_k = np.concatenate([o.cpu().numpy() for o in out])
    want_k, want_v = oracle.sharded_sort(shards, vals)
    u = np.uint32 if bits == 32 else np.uint64
    assert np.array_equal(got_k.view(u), want_k.view(u))
    if with_values:
        assert np.array_equal(got_v.astype(np.uint64), want_v.astype(np.uint64))
    # each rank's slice is what the plan said it would receive
    lens = [(o[0] if with_values else o).numel() for o in out]
    assert lens == plan["recv"]


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_p2p_exchange_u32_pairs(cuda, world):
    """Fused partition + peer stores (os_msd_partition_p2p) into separate
    per-rank receive allocations: the destination indices are real
    cross-allocation pointer differences, as with peer-mapped NVLink buffers."""
    rng = np.random.default_rng(world)
    sizes = [int(rng.integers(100_000, 300_000)) for _ in range(world)]
    _p2p_case(world, np.uint32, sizes)


@pytest.mark.parametrize("dtype,q", [(np.int32, 1), (np.float32, 1), (np.uint64, 1),
                                     (np.float64, 1), (np.uint32, 16)])
def test_p2p_exchange_key_types_and_skew(cuda, dtype, q):
    _p2p_case(3, dtype, [200_001, 150_000, 99_999], q=q)


def test_p2p_exchange_keys_only_and_empty_shard(cuda):
    _p2p_case(3, np.uint32, [250_000, 0, 123_457], with_values=False)


def test_p2p_exchange_all_equal_keys_one_destination(cuda):
    """All keys in one top-digit bin: one rank receives everything, the
    others nothing (whole-bin splitting), and stability still holds."""
    from oracle import oracle
    from paper_2206_01784_b200.distributed import emulate_p2p_sort

    shards = [np.full(n, 0xABACADAE, dtype=np.uint32) for n in (70_000, 90_000)]
    vals = [np.arange(70_000, dtype=np.uint32), np.arange(70_000, 160_000, dtype=np.uint32)]
    out, plan = emulate_p2p_sort([torch.from_numpy(s).cuda() for s in shards],
                                 [torch.from_numpy(v).cuda() for v in vals])
    assert sorted(plan["recv"]) == [0, 160_000]
    got_v = np.concatenate([o[1].cpu().numpy() for o in out])
    assert np.array_equal(got_v, oracle.sharded_sort(shards, vals)[1])


def test_p2p_rejects_mixed_widths(cuda):
    from paper_2206_01784_b200.distributed import emulate_p2p_sort

    k = torch.zeros(1000, dtype=torch.uint32, device="cuda")
    v = torch.zeros(1000, dtype=torch.int64, device="cuda")
    with pytest.raises(ValueError):
        emulate_p2p_sort([k, k], [v, v])


def test_p2p_symmetric_memory_plumbing_world1(cuda):
    """The fused exchange's real host plumbing on one GPU: a world-size-1 NCCL
    group, torch symmetric memory (empty / rendezvous / buffer_ptrs /
    barrier) and sharded_sort(exchange="p2p") against onesweep_sort, and the
    ShardedSorter probe selecting p2p (tools/p2p_probe.py, in a subprocess so
    the process group stays private)."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "p2p_probe.py")],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "exchange p2p keys equal True values equal True" in r.stdout
    assert "ShardedSorter exchange: p2p" in r.stdout
