"""Multi-process host logic of the replica benchmark (world size 2, gloo, CPU):
max-over-ranks time, sum-over-ranks work, every rank solving the same seeded instance
(so the oracle's F* golden is every replica's target)."""
import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from paper_1701_04900_b200 import inputs
    ms, units = bench.reduce_over_ranks(10.0 + 5 * rank, 100.0 * (rank + 1), world, device="cpu")
    P = bench.make_problem(0)
    out[rank] = (ms, units, float(P.b.sum()), P.meta["config_idx"])
    dist.barrier()
    dist.destroy_process_group()


def test_replica_reduction_gloo():
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    for r in range(world):
        ms, units, _, idx = res[r]
        assert ms == 15.0 and units == 300.0 and idx == 0
    assert res[0][2] == res[1][2]  # replicas solve the same seeded instance
