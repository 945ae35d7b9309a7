"""Probe: every k_apply call of a device MCTS search (NasRNN, budget 128, node limit 2000) with its
batch size, arena headroom, matches / adds of its heaviest leaf and wall time -- the slowest first."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2410_05534_b200 import analogs  # noqa: E402
from paper_2410_05534_b200 import tensor_ir as T  # noqa: E402
from paper_2410_05534_b200 import native  # noqa: E402
from paper_2410_05534_b200.apply import ApplyDriver  # noqa: E402
from paper_2410_05534_b200.cost_model import CostModelConfig  # noqa: E402
from paper_2410_05534_b200.mcts import MctsConfig, optimize_mcts  # noqa: E402
from paper_2410_05534_b200.patterns import load_rules  # noqa: E402

model = sys.argv[1] if len(sys.argv) > 1 else "nasrnn"
calls = []
orig = ApplyDriver.apply
rounds = [0]
orig_b = native.DeviceBatch.apply


def count(self, *a, **k):
    rounds[0] += 1
    return orig_b(self, *a, **k)


native.DeviceBatch.apply = count


def timed(self, rules, *a, **k):
    b = self.pipe.batch
    n0, _ = b.live_counts()
    rounds[0] = 0
    t = time.perf_counter()
    res = orig(self, rules, *a, **k)
    dt = time.perf_counter() - t
    rep = res["report"]
    j = int(np.argmax(rep[:, 0]))
    calls.append((dt, b.n_leaves, int(b.nb[1] - b.nb[0]) - int(n0[0]), int(rep[j, 0]), int(rep[j, 5]), int(n0[j]),
                  int(rules[j]), int(rep[:, 0].sum()), rounds[0]))
    return res


ApplyDriver.apply = timed
eg = T.graph_to_egraph(analogs.build_analog(model, T.GraphBuilder))
cfg = MctsConfig(budget=int(sys.argv[2]) if len(sys.argv) > 2 else 128, node_limit=2000, seed=0, batch=32,
                 max_sim_steps=10)
t = time.time()
rep = optimize_mcts(eg, load_rules("taso_analog"), cfg, CostModelConfig())
print(f"{model}: {time.time() - t:.2f}s, {len(calls)} applies, {sum(c[0] for c in calls):.2f}s in apply")
print("   s   leaves headroom0 max_matches its_adds its_n0 rule total_matches rounds")
for c in sorted(calls, reverse=True)[:25]:
    print(f"{c[0]:6.3f} {c[1]:5d} {c[2]:8d} {c[3]:8d} {c[4]:8d} {c[5]:6d} {c[6]:4d} {c[7]:8d} {c[8]:4d}")
