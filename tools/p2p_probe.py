"""Single-GPU probe of the fused p2p exchange's host plumbing: a world-size-1
NCCL group, torch symmetric memory (empty / rendezvous / buffer_ptrs /
barrier) and sharded_sort(exchange="p2p") against onesweep_sort.  Real peer
mappings need >= 2 GPUs; this catches API-level breakage on one.
    python tools/p2p_probe.py"""
import os
import socket
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist


def main():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    from paper_2206_01784_b200 import KeyGenSpec, generate_keys, onesweep_sort
    from paper_2206_01784_b200.distributed import ShardedSorter, sharded_sort

    n = 3_000_017
    k = generate_keys(KeyGenSpec(q=1, seed=5, n=n), device="cuda")
    v = torch.arange(n, dtype=torch.int32, device="cuda").view(torch.uint32)
    (ok, ov), plan = sharded_sort(k, v, exchange="p2p", return_plan=True)
    wk, wv = onesweep_sort(k, v)
    print("exchange", plan["exchange"], "keys equal", torch.equal(ok, wk), "values equal", torch.equal(ov, wv))
    print("ShardedSorter exchange:", ShardedSorter(1 << 20, torch.uint32).exchange)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
