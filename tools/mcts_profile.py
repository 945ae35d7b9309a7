"""Probe: where a device MCTS search spends its wall time (cProfile of optimize_mcts)."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
from paper_2410_05534_b200 import analogs  # noqa: E402
from paper_2410_05534_b200 import tensor_ir as T  # noqa: E402
from paper_2410_05534_b200.cost_model import CostModelConfig  # noqa: E402
from paper_2410_05534_b200.mcts import MctsConfig, optimize_mcts  # noqa: E402
from paper_2410_05534_b200.patterns import load_rules  # noqa: E402

model = sys.argv[1] if len(sys.argv) > 1 else "nasrnn"
budget = int(sys.argv[2]) if len(sys.argv) > 2 else 128
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 32
eg = T.graph_to_egraph(analogs.build_analog(model, T.GraphBuilder))
cfg = MctsConfig(budget=budget, node_limit=2000, seed=0, batch=batch, max_sim_steps=10)
rules = load_rules("taso_analog")
optimize_mcts(T.graph_to_egraph(analogs.build_analog("toy" if False else model, T.GraphBuilder)), rules,
              MctsConfig(budget=4, node_limit=2000, seed=0, batch=4, max_sim_steps=2), CostModelConfig())  # warm
t = time.time()
prof = cProfile.Profile()
prof.enable()
rep = optimize_mcts(eg, rules, cfg, CostModelConfig())
prof.disable()
print(f"{model}: {time.time() - t:.2f}s, {rep.original_cost:.6g} -> {rep.optimized_cost:.6g}, "
      f"{len(rep.trace)} rules", flush=True)
pstats.Stats(prof).sort_stats("tottime").print_stats(30)
