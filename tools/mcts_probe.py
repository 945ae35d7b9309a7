"""Probe: MCTS on analog models, wall time and costs."""
import sys, time
sys.path.insert(0, ".")
from paper_2410_05534_b200 import analogs
from paper_2410_05534_b200 import tensor_ir as T
from paper_2410_05534_b200.cost_model import CostModelConfig
from paper_2410_05534_b200.mcts import MctsConfig, optimize_mcts
from paper_2410_05534_b200.patterns import load_rules

for model in sys.argv[1:] or ["nasrnn"]:
    eg = T.graph_to_egraph(analogs.build_analog(model, T.GraphBuilder))
    cfg = MctsConfig(budget=128, node_limit=2000, seed=0, batch=64, max_sim_steps=10)
    t = time.time()
    rep = optimize_mcts(eg, load_rules("taso_analog"), cfg, CostModelConfig())
    dt = time.time() - t
    print(f"{model}: cost {rep.original_cost:.6g} -> {rep.optimized_cost:.6g} ({rep.speedup_pct:.2f}% better), "
          f"{len(rep.trace)} rules applied, {dt:.1f}s", flush=True)
