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


def _batch_worker(rank, world, port, out):
    """Each rank evaluates its shard of the C5-style batch with the oracle and
    the shard sums are all-reduced, as bench.py --workload C5 does over NCCL."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import numpy as np
    from conftest import ORACLE_LIB
    from paper_2605_14526_b200 import scenes
    from paper_2605_14526_b200.dist import allreduce_loss_grad, shard
    from paper_2605_14526_b200.hd import Library
    lib = Library(ORACLE_LIB)
    sc = lib.scene(scenes.block_scene(dims=(2, 1, 1), frames=2))
    ne = sc.element_count
    young = scenes.c5_young(5, ne, base=5e4)
    mine = shard(5, rank, world)
    b = sc.batch(len(mine), young[mine.start:mine.stop])
    r = b.evaluate(2)
    buf = torch.tensor(np.concatenate([[r["loss"].sum()], r["dl_de"]]), dtype=torch.float64)
    allreduce_loss_grad(buf)
    out[rank] = buf.numpy().tolist()
    dist.barrier()
    dist.destroy_process_group()


def test_batch_shards_allreduce_to_the_full_batch(orc):
    import numpy as np
    from paper_2605_14526_b200 import scenes
    from paper_2605_14526_b200.dist import shard
    assert [list(shard(5, r, 2)) for r in range(2)] == [[0, 1, 2], [3, 4]]
    assert [len(shard(64, r, 8)) for r in range(8)] == [8] * 8
    world = 2
    port = 29500 + os.getpid() % 1000
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_batch_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    assert res[0] == res[1]
    sc = orc.scene(scenes.block_scene(dims=(2, 1, 1), frames=2))
    full = sc.batch(5, scenes.c5_young(5, sc.element_count, base=5e4)).evaluate(2)
    ref = np.concatenate([[full["loss"].sum()], full["dl_de"]])
    np.testing.assert_allclose(res[0], ref, rtol=1e-12, atol=1e-300)
