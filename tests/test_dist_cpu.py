"""World-size-2 gloo test of the N>1 bench path (timing max over ranks,
aggregate replica throughput) -- runs on CPU."""

import os

import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1706_09384_b200.dist import max_over_ranks, replica_throughput

    ms_local = 10.0 if rank == 0 else 20.0
    gbps, ms = replica_throughput(ms_local, bytes_per_step=1e9, steps=5, device="cpu")
    q.put((rank, max_over_ranks(rank + 1.5, "cpu"), gbps, ms))
    dist.barrier()
    dist.destroy_process_group()


def test_replica_aggregation_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, mx, gbps, ms in res:
        assert mx == 2.5
        assert ms == 20.0
        # 2 ranks x 5 steps x 1 GB / 20 ms
        assert abs(gbps - 2 * 5 * 1e9 / 0.020 / 1e9) < 1e-9
