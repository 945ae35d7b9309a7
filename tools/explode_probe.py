"""Probe: the heaviest k_apply of a device MCTS search (NasRNN: the multi-pattern rule on a ~1.9k-node
leaf, ~41k matches, ~106k added e-nodes), replayed alone on a one-leaf batch with enough headroom and
timed; the last replay runs between cudaProfilerStart/Stop so
    ncu --profile-from-start off -k regex:k_apply -c 1 python tools/explode_probe.py
captures exactly it."""
import os
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_05534_b200 import analogs  # noqa: E402
from paper_2410_05534_b200 import native  # noqa: E402
from paper_2410_05534_b200 import tensor_ir as T  # noqa: E402
from paper_2410_05534_b200.apply import ApplyDriver  # noqa: E402
from paper_2410_05534_b200.cost_model import CostModelConfig  # noqa: E402
from paper_2410_05534_b200.mcts import MctsConfig, optimize_mcts  # noqa: E402
from paper_2410_05534_b200.patterns import load_rules  # noqa: E402

MIN = int(os.environ.get("EXPLODE_MIN_MATCHES", "20000"))
HEAD = int(os.environ.get("EXPLODE_HEADROOM", "262144"))
orig = ApplyDriver.apply


def hook(self, rules, *a, **k):
    res = orig(self, rules, *a, **k)
    rep = res["report"]
    j = int(np.argmax(rep[:, 0]))
    if rep[j, 0] < MIN or res["status"][j] != native.A_OK:
        return res
    pipe, rule = self.pipe, int(rules[j])
    store = native.SnapshotStore(pipe.ctx)
    slot = store.save(pipe.batch, [j])[0]
    print(f"leaf: n={slot.n} U={slot.U} rule {rule}, {rep[j, 0]} matches", flush=True)
    for r in range(3):
        pipe.load_slots(store, [slot], HEAD)
        pipe.rebuild()
        mask = pipe.rule_masks([rule])
        pipe.ematch(mask)
        pipe.ctx.sync()
        if r == 2:
            torch.cuda.profiler.start()
        t = time.perf_counter()
        out = orig(self, np.array([rule], np.uint32), leaf_mask=mask)
        dt = time.perf_counter() - t
        if r == 2:
            torch.cuda.profiler.stop()
        print(f"replay {r}: {dt * 1e3:.1f} ms status {out['status'][0]} report {out['report'][0].tolist()}",
              flush=True)
    os._exit(0)


ApplyDriver.apply = hook
torch.cuda.init()
eg = T.graph_to_egraph(analogs.build_analog("nasrnn", T.GraphBuilder))
optimize_mcts(eg, load_rules("taso_analog"), MctsConfig(budget=128, node_limit=2000, seed=0, batch=32,
                                                        max_sim_steps=10), CostModelConfig())
print("no explosion found")
