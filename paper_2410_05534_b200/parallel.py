"""Multi-GPU leaf/seed sharding and the MCTS result exchange.

Leaves of one MCTS batch step (and MCTS seeds) are independent e-graphs, so the data
path shards with no collective: rank r owns the contiguous global leaf range
``leaf_shard(total, world, r)``. The one real exchange is the MCTS update: every rank
needs every leaf's (status, root cost) to backpropagate Eq. 3 rewards,
so per step the per-leaf results are all-gathered (NCCL over NVLink on B200s; gloo in the
CPU tests). Rank-ordered concatenation of contiguous shards is global leaf order, so the
merged statistics are identical at any world size.
"""

from __future__ import annotations


def leaf_shard(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [start, end) share of `total` leaves for `rank` (first ranks take the remainder)."""
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def allgather_leaf_results(root_cost, status, group=None):
    """All-gather equal-size per-rank result tensors; returns tensors in global leaf order."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    out_c = torch.empty(root_cost.numel() * world, dtype=root_cost.dtype, device=root_cost.device)
    out_s = torch.empty(status.numel() * world, dtype=status.dtype, device=status.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out_c, root_cost, group=group)
        dist.all_gather_into_tensor(out_s, status, group=group)
    else:
        dist.all_gather(list(out_c.chunk(world)), root_cost, group=group)
        dist.all_gather(list(out_s.chunk(world)), status, group=group)
    return out_c, out_s


def rewards(prev_cost, new_cost):
    """Eq. 3 per leaf step: max(runtime_{i-1} - runtime_i, 0)."""
    import torch

    return torch.clamp(prev_cost - new_cost, min=0.0)


def root_parallel_sweep(run_seed, seeds, group=None):
    """Root-parallel MCTS sweep (BASELINE config 5: 64 seeds sharded over 8 GPUs).

    Rank r runs ``run_seed(seed) -> (final_cost, trace)`` for its contiguous share of ``seeds``;
    the per-seed results ``(seed, final cost, trace hash)`` are all-gathered (NCCL over NVLink, gloo
    in the CPU tests) so every rank holds the whole sweep in seed order and the same best seed."""
    import hashlib

    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    s, e = leaf_shard(len(seeds), world, rank)
    per = -(-len(seeds) // world)   # padded share so every rank contributes equal-size tensors
    rows = torch.full((per, 3), -1.0, dtype=torch.float64)
    for i, seed in enumerate(seeds[s:e]):
        cost, trace = run_seed(seed)
        h = int.from_bytes(hashlib.blake2b(repr(list(trace)).encode(), digest_size=6).digest(), "big")
        rows[i] = torch.tensor([float(seed), float(cost), float(h)], dtype=torch.float64)
    if world > 1:
        backend = dist.get_backend(group)
        dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
        src = rows.to(dev)
        out = [torch.empty_like(src) for _ in range(world)]
        dist.all_gather(out, src, group=group)
        rows = torch.cat([o.cpu() for o in out])
    res = [(int(r[0]), float(r[1]), int(r[2])) for r in rows.tolist() if r[0] >= 0]
    res.sort()
    best = min(res, key=lambda t: (t[1], t[0])) if res else None
    return res, best


class ShardedEngine:
    """Leaf-parallel MCTS over ranks: wraps one rank's engine so every
    batch of expansions and rollouts is split into contiguous shards, each rank runs its shard on
    its own GPU, and the per-leaf results are all-gathered in rank order (= leaf order). Every rank
    therefore applies the same updates in selection order and holds the same tree; the search's RNG
    is consumed identically everywhere (rollouts carry their own seeds, mcts.py), so the search is
    the single-GPU search. The exchange per batch is the expansion rows (changed, cost, e-nodes,
    e-classes, applicability bits and the child's e-graph, which any rank may expand later -- a device
    engine's snapshot slots are exported to host states for the exchange and imported into every
    rank's own store) and the rollout rewards -- ``torch.distributed.all_gather_object`` over NCCL (gloo in the CPU tests).

    ``evaluate`` / ``final`` / ``initial`` run redundantly on every rank (one e-graph each)."""

    def __init__(self, engine, group=None):
        import torch.distributed as dist

        self.engine = engine
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.exchanged_bytes = 0

    def _gather(self, obj):
        if self.world == 1:
            return [obj]
        import pickle

        import torch.distributed as dist

        out = [None] * self.world
        dist.all_gather_object(out, obj, group=self.group)
        self.exchanged_bytes += sum(len(pickle.dumps(o)) for o in out)
        return out

    def configure(self, cfg):
        if cfg.extraction_cache and self.world > 1:
            raise ValueError("the run-wide extraction cache is per engine: not supported with sharded rollouts")
        if hasattr(self.engine, "configure"):
            self.engine.configure(cfg)

    def initial(self, egraph):
        return self.engine.initial(egraph)

    def evaluate(self, states):
        return self.engine.evaluate(states)

    def final(self, state, method):
        return self.engine.final(state, method)

    def expand(self, states, rules):
        import numpy as np

        s, e = leaf_shard(len(states), self.world, self.rank)
        part = self.engine.expand(states[s:e], list(rules[s:e])) if e > s else None
        dev = self.world > 1 and hasattr(self.engine, "export_states")   # device snapshots travel as host states
        if part is not None and dev:
            part = (self.engine.export_states(part[0]), *part[1:])
        parts = [p for p in self._gather(part) if p is not None]
        kids = [k for p in parts for k in p[0]]
        if dev:
            kids = self.engine.import_states(kids)
        cat = [np.concatenate([p[i] for p in parts]) for i in range(1, 6)]
        return (kids, *cat)

    def simulate(self, states, costs0, allowed, steps, node_limit, seeds):
        import numpy as np

        s, e = leaf_shard(len(states), self.world, self.rank)
        part = (self.engine.simulate(states[s:e], list(costs0[s:e]), allowed[s:e], steps, node_limit, seeds[s:e])
                if e > s else np.zeros(0))
        return np.concatenate(self._gather(part))
