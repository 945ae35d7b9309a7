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


def _search(model, cfg_kw):
    """optimize_mcts with the CPU reference engine (oracle/mcts_ref.py), sharded when a process group
    is up; returns the RunReport as JSON."""
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))
    from make_mcts_golden import RULES, build_input

    from oracle.mcts_ref import ReferenceEngine, import_reference
    from paper_2410_05534_b200.cost_model import CostModelConfig
    from paper_2410_05534_b200.mcts import MctsConfig, optimize_mcts
    from paper_2410_05534_b200.parallel import ShardedEngine

    E, R, X, T = import_reference()
    text = RULES["taso_analog"].read_text()
    eng = ShardedEngine(ReferenceEngine(text, CostModelConfig(), workers=1))
    rep = optimize_mcts(build_input(model, T), R.parse_rules(text), MctsConfig(**cfg_kw), CostModelConfig(),
                        engine=eng)
    return rep.to_json_dict(), eng.exchanged_bytes


def _search_worker(rank, world, port, model, cfg_kw, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rep, nbytes = _search(model, cfg_kw)
    q.put((rank, rep, nbytes))
    dist.barrier()
    dist.destroy_process_group()


def test_leaf_parallel_search_matches_single_rank():
    """the NasRNN search with every batch's expansions and rollouts sharded over two
    ranks (parallel.ShardedEngine, all-gather of the per-leaf rows) returns, on every rank, the
    RunReport of the single-rank search -- same applied-rule trace, costs and final program."""
    from oracle.mcts_ref import reference_available

    if not reference_available():
        pytest.skip("reference not importable")
    cfg_kw = dict(budget=24, batch=8, node_limit=400, seed=0, max_sim_steps=3)
    single, _ = _search("nasrnn", cfg_kw)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + os.getpid() % 200
    procs = [ctx.Process(target=_search_worker, args=(r, 2, port, "nasrnn", cfg_kw, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert single["iterations"], single
    for rank, rep, nbytes in outs:
        assert rep == single, rank
        assert nbytes > 0


def _bench_shard_worker(rank, world, port, q):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    import bench

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    leaves = list(range(37))            # stand-ins: make_batch only indexes the leaf list
    B = 16
    from paper_2410_05534_b200.arena import Batch

    orig = Batch.pack
    Batch.pack = lambda self: {"n_leaves": len(self.leaves)}
    try:
        packed, src = bench.make_batch(leaves, B, rotate=rank * B)
    finally:
        Batch.pack = orig
    # the bench's exchange: per-leaf (root cost, status) all-gathered in rank order
    cost = torch.tensor([float(s) for s in src], dtype=torch.float64)
    stat = torch.tensor(src, dtype=torch.int32)
    c, st = allgather_leaf_results(cost, stat)
    q.put((rank, src, c.tolist(), st.tolist()))
    dist.barrier()
    dist.destroy_process_group()


def test_bench_leaf_shards_and_gather():
    """bench.py --gpus N (C3): rank r takes the contiguous shard [r*B, (r+1)*B) of the global leaf
    sequence and the per-leaf results all-gathered over the ranks are that sequence in order."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29800 + os.getpid() % 100
    procs = [ctx.Process(target=_bench_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    glob = [i % 37 for i in range(32)]
    assert outs[0][1] == glob[:16] and outs[1][1] == glob[16:]
    for _, _, c, st in outs:
        assert st == glob and c == [float(x) for x in glob]
