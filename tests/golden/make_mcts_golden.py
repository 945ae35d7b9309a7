"""Generate the MCTS-level golden RunReports by running the SPEC MCTS (mcts.optimize_mcts) on the
REFERENCE's own e-graph code (oracle/mcts_ref.ReferenceEngine: esat.rewrite.apply_rule,
is_rule_applicable, esat.extraction.extract_*_greedy, extraction_to_graph, save_graph).

Run in the build container only (needs the reference: /root/reference or baseline/_ref):

    python tests/golden/make_mcts_golden.py <name> [...]     # names: see CASES; 'all' for every case

Writes tests/golden/mcts/<name>.json: the case (model, MCTS config, cost model, rule-file SHA-256),
the RunReport (costs as float.hex, per-iteration rows, rule histogram, final program as the exact
save_graph text) and the generator's own wall time. tests/test_gpu_mcts_parity.py runs the same
case with the device engine and requires an identical RunReport.
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))

RULES = {"taso_analog": REPO / "paper_2410_05534_b200" / "rules" / "taso_analog.rules",
         "toy_math": REPO / "paper_2410_05534_b200" / "rules" / "toy_math.rules"}

# name -> (model, rules, cost mode, MctsConfig kwargs)
CASES = {
    "toy_b1": ("toy", "toy_math", "term", dict(budget=64, node_limit=10, seed=0, batch=1, final_extractor="ocf")),
    "toy_b8": ("toy", "toy_math", "term", dict(budget=64, node_limit=10, seed=1, batch=8, final_extractor="exact")),
    "bert_c1_b1": ("bert", "taso_analog", "analytic", dict(budget=8, node_limit=500, seed=0, batch=1,
                                                          max_sim_steps=4)),
    "bert_c1": ("bert", "taso_analog", "analytic", dict(budget=128, node_limit=500, seed=0, batch=32)),
    # reduced budgets ("a committed reduced budget if runtime forces it"): the reference's
    # apply_rule needs tens of minutes for one application of the #128 / #138-analog multi-pattern
    # rules on a 1-2k-node leaf (28k matches, a would_create_cycle DFS each), so the node limit of
    # these cases keeps the leaves the search explodes from small
    "nasrnn_c2": ("nasrnn", "taso_analog", "analytic", dict(budget=128, node_limit=800, seed=0, batch=32)),
    "nasrnn_c2_cache": ("nasrnn", "taso_analog", "analytic", dict(budget=128, node_limit=800, seed=0, batch=32,
                                                                  extraction_cache=True)),
    "nasrnn_c2_limit2000": ("nasrnn", "taso_analog", "analytic", dict(budget=128, node_limit=2000, seed=0, batch=32)),
    "resnext50_c3": ("resnext50", "taso_analog", "analytic", dict(budget=128, node_limit=1000, seed=0, batch=32)),
    "inception_v3_c4": ("inception_v3", "taso_analog", "analytic", dict(budget=64, node_limit=1000, seed=0,
                                                                        batch=32)),
    "nasnet_a_c5_s0": ("nasnet_a", "taso_analog", "analytic", dict(budget=64, node_limit=1000, seed=0, batch=32)),
    "nasnet_a_c5_s1": ("nasnet_a", "taso_analog", "analytic", dict(budget=64, node_limit=1000, seed=1, batch=32)),
}


def build_input(model: str, T):
    """The case's initial e-graph with the given tensor_ir module (the reference's or ours)."""
    from paper_2410_05534_b200 import analogs

    if model == "toy":
        return T.toy_term_to_egraph(("div", ("mul", "a", 2), 2))
    return T.graph_to_egraph(analogs.build_analog(model, T.GraphBuilder))


def run_case(name: str, workers: int = 8) -> dict:
    from oracle.mcts_ref import ReferenceEngine, import_reference
    from paper_2410_05534_b200.cost_model import CostModelConfig
    from paper_2410_05534_b200.mcts import MctsConfig, optimize_mcts

    E, R, X, T = import_reference()
    model, rules_name, mode, kw = CASES[name]
    text = RULES[rules_name].read_text()
    cfg = MctsConfig(**kw)
    cost = CostModelConfig(mode=mode)
    eng = ReferenceEngine(text, cost, method=cfg.main_extractor, workers=workers)
    t0 = time.time()
    try:
        rep = optimize_mcts(build_input(model, T), R.parse_rules(text), cfg, cost, engine=eng)
    finally:
        eng.close()
    return {"name": name, "model": model, "rules": rules_name,
            "rules_sha256": hashlib.sha256(text.encode()).hexdigest(), "cost_mode": mode,
            "config": {k: getattr(cfg, k) for k in cfg.__dataclass_fields__},
            "report": rep.to_json_dict(), "reference_wall_s": round(time.time() - t0, 1),
            "generator": "tests/golden/make_mcts_golden.py (oracle/mcts_ref.ReferenceEngine)"}


def main():
    names = sys.argv[1:] or ["toy_b1"]
    if names == ["all"]:
        names = list(CASES)
    out = HERE / "mcts"
    out.mkdir(exist_ok=True)
    for nm in names:
        rec = run_case(nm)
        (out / f"{nm}.json").write_text(json.dumps(rec, indent=1, sort_keys=True) + "\n")
        print(nm, rec["reference_wall_s"], "s", rec["report"]["optimized_cost"], len(rec["report"]["iterations"]),
              flush=True)


if __name__ == "__main__":
    main()
