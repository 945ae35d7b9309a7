"""Subprocess body of tests/test_gpu_refpatch.py: a seeded rollout on the reference's own objects,
run twice -- with the stock reference, then with refpatch.install (device rebuild / matching /
extraction / apply) -- printing a JSON digest of every step for comparison."""
import hashlib
import json
import random
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
from oracle.mcts_ref import import_reference  # noqa: E402

E, R, X, T = import_reference()
from paper_2410_05534_b200 import analogs, refpatch  # noqa: E402
from paper_2410_05534_b200.cost_model import CostModelConfig, egraph_costs  # noqa: E402


def rollout(model, seed, steps, apply_on_device):
    rules = R.parse_rules((REPO / "paper_2410_05534_b200" / "rules" / "taso_analog.rules").read_text())
    eg = T.graph_to_egraph(analogs.build_analog(model, T.GraphBuilder))
    rng = random.Random(seed)
    rows = []
    for _ in range(steps):
        live = [r for r in rules if 0 < len(R.joint_match(eg, r.sources)) <= 600]
        if not live or eg.size()[0] >= 2000:
            break
        rule = live[rng.randrange(len(live))]
        rep = R.apply_rule(eg, rule, 2000)
        costs = egraph_costs(eg, CostModelConfig())
        ext = []
        for fn in (X.extract_default_greedy, X.extract_ocf_greedy):
            try:
                r = fn(eg, costs)
                ext.append((float(r.total_cost).hex(), sorted((c, n.symbol.name, n.children) for c, n in r.chosen.items())))
            except X.ExtractionError as exc:
                ext.append((type(exc).__name__, str(exc)))
        app = [R.is_rule_applicable(eg, r) for r in rules]
        rows.append({"rule": rule.id, "report": [rep.matches_found, rep.changed, rep.nodes_after, rep.classes_after,
                                                  rep.cycles_filtered, rep.shape_filtered],
                     "dump": hashlib.sha256(eg.dump().encode()).hexdigest(), "extract": ext, "applicable": app})
    return rows


mode = sys.argv[1]
if mode != "stock":
    refpatch.install(E, R, X, apply_rule=(mode == "device_apply"))
out = {m: [rollout(m, s, 6, mode == "device_apply") for s in (0, 1)] for m in ("bert", "nasnet_a")}
print(json.dumps(out))
