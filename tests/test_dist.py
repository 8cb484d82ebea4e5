"""Multi-process plumbing of the N>1 bench path (replicas; max over ranks),
exercised with the gloo backend, world size 2, on CPU."""
import os

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_14526_b200.dist import max_over_ranks, replica_value
    ms = max_over_ranks(10.0 + rank)
    val = replica_value(steps=4, ms=ms, world=world)
    out[rank] = (ms, val)
    dist.barrier()
    dist.destroy_process_group()


def test_max_over_ranks_gloo():
    world = 2
    port = 29000 + os.getpid() % 1000
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    assert res[0][0] == res[1][0] == 11.0
    assert res[0][1] == pytest.approx(2 * 4 / 0.011)
