"""Root-parallel MCTS seed sweep (BASELINE config 5), one process per GPU.

    python -m torch.distributed.run --nproc-per-node 8 --master-addr 127.0.0.1 \\
        -m paper_2410_05534_b200.sweep --model nasnet_a --seeds 64

Every rank runs optimize_mcts (mcts.py, device-batched) for its contiguous share of the seeds on
its own GPU; the (seed, final cost, trace hash) rows are all-gathered over NCCL and rank 0 prints
one JSON line with the whole sweep, the best seed and the max-over-ranks wall time.
"""

from __future__ import annotations

import argparse
import json
import os
import time


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="nasnet_a")
    ap.add_argument("--seeds", type=int, default=64)
    ap.add_argument("--budget", type=int, default=128)
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--node-limit", type=int, default=2000)
    ap.add_argument("--sim-steps", type=int, default=10)
    args = ap.parse_args()

    import torch
    import torch.distributed as dist

    from . import analogs, native
    from . import tensor_ir as T
    from .cost_model import CostModelConfig
    from .mcts import MctsConfig, optimize_mcts
    from .parallel import root_parallel_sweep
    from .patterns import load_rules

    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = native.Context(local)
    rules = load_rules("taso_analog")
    cost = CostModelConfig()

    def run_seed(seed):
        from .mcts import DeviceEngine
        from .symtab import SymbolTable

        eg = T.graph_to_egraph(analogs.build_analog(args.model, T.GraphBuilder))
        cfg = MctsConfig(budget=args.budget, node_limit=args.node_limit, seed=seed, batch=args.batch,
                         max_sim_steps=args.sim_steps)
        st = SymbolTable()
        engine = DeviceEngine(rules, st, eg.language, cost, ctx=ctx, method=cfg.main_extractor, headroom=cfg.headroom)
        rep = optimize_mcts(eg, rules, cfg, cost, symtab=st, engine=engine)
        run_seed.initial = rep.original_cost
        return rep.optimized_cost, rep.trace

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res, best = root_parallel_sweep(run_seed, list(range(args.seeds)))
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([wall], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        wall = float(t.item())
    if int(os.environ.get("RANK", "0")) == 0:
        print(json.dumps({"workload": f"{args.model} analog, {args.seeds}-seed root-parallel MCTS sweep",
                          "n_gpus": world, "budget": args.budget, "batch": args.batch, "wall_s": wall,
                          "seeds_per_s": args.seeds / wall, "best": {"seed": best[0], "cost": best[1]},
                          "results": [{"seed": s, "cost": c, "trace_hash": h} for s, c, h in res]}), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
