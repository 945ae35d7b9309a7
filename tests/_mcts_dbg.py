import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2410_05534_b200 import analogs
from paper_2410_05534_b200 import tensor_ir as T
from paper_2410_05534_b200.cost_model import CostModelConfig
from paper_2410_05534_b200.mcts import MctsConfig, optimize_mcts, DeviceEngine
from paper_2410_05534_b200.arena import export_state
from paper_2410_05534_b200.symtab import SymbolTable
from paper_2410_05534_b200.patterns import load_rules
rules = load_rules("taso_analog")
for model in ["nasnet_a", "nasrnn"]:
    eg = T.graph_to_egraph(analogs.build_analog(model, T.GraphBuilder))
    st = SymbolTable(); cfg = CostModelConfig()
    eng = DeviceEngine(rules, st, eg.language, cfg)
    s = export_state(eg, st, cfg)
    clean, cost, n, app = eng.evaluate([s])
    print(model, "n", n, "cost", cost, "applicable rules", np.nonzero(app[0])[0].tolist(), flush=True)
    t = time.time()
    r = optimize_mcts(eg, rules, MctsConfig(budget=32, batch=16, seed=0, max_sim_steps=3), cfg)
    print(model, r, time.time() - t, flush=True)
