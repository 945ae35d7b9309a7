"""World-size-2 gloo tests of the multi-GPU host path: leaf sharding + result exchange give the
same merged per-leaf statistics as a single rank."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2410_05534_b200.parallel import allgather_leaf_results, leaf_shard, rewards


def test_leaf_shard_covers_everything():
    for total in (0, 1, 7, 256, 4097):
        for world in (1, 2, 3, 8):
            spans = [leaf_shard(total, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))


def _worker(rank, world, port, costs, status, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s, e = leaf_shard(len(costs), world, rank)
    c, st = allgather_leaf_results(torch.tensor(costs[s:e]), torch.tensor(status[s:e]))
    prev = torch.tensor(costs) + 1.0
    r = rewards(prev, c)
    if rank == 0:
        q.put((c.numpy(), st.numpy(), r.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_allgather_matches_single_rank(world):
    rng = np.random.default_rng(0)
    n = 64 * world
    costs = rng.random(n)
    status = rng.integers(0, 3, n).astype(np.int32)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, world, port, costs, status, q)) for r in range(world)]
    for p in procs:
        p.start()
    c, st, r = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert np.array_equal(c, costs) and np.array_equal(st, status)
    assert np.allclose(r, 1.0)


def _sweep_worker(rank, world, port, seeds, q):
    from paper_2410_05534_b200.parallel import root_parallel_sweep

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # stand-in for optimize_mcts: deterministic per seed
    res, best = root_parallel_sweep(lambda s: (float((s * 37) % 11), [s % 5, s % 3]), seeds)
    q.put((rank, res, best))
    dist.barrier()
    dist.destroy_process_group()


def test_root_parallel_sweep_matches_single_rank():
    """Config 5's 64-seed sweep sharded over 2 ranks equals the single-rank sweep on every rank."""
    from paper_2410_05534_b200.parallel import root_parallel_sweep

    seeds = list(range(64))
    single, best1 = root_parallel_sweep(lambda s: (float((s * 37) % 11), [s % 5, s % 3]), seeds)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29611
    procs = [ctx.Process(target=_sweep_worker, args=(r, 2, port, seeds, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, res, best in outs:
        assert res == single and best == best1, rank
    assert len(single) == 64 and best1[1] == 0.0
