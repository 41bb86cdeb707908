"""Multi-GPU path = independent replicas.  The host-side aggregation bench.py
uses under torchrun (max-over-ranks timing, whole-job throughput) is exercised here with the gloo
backend, world_size 2, on CPU."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)
    local_ms = 100.0 * (rank + 1)                       # rank 1 is the slower replica
    value, ms = bench.replica_throughput(units_per_rank=1024, local_ms=local_ms, device=torch.device("cpu"))
    r, lr, w = bench.dist_env()
    q.put((rank, value, ms, r, w))
    bench.barrier()
    dist.destroy_process_group()


def test_replica_aggregation_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, value, ms, r, w in res:
        assert ms == 200.0                               # max over ranks
        assert abs(value - 2 * 1024 / 0.2) < 1e-6        # all units / job time
        assert (r, w) == (rank, 2)
