"""MCTS-level parity (the north_star target): ``optimize_mcts`` driven by the device engine must
reproduce the RunReport the same search produces on the REFERENCE's own e-graph code
(tests/golden/mcts/*.json, made by tests/golden/make_mcts_golden.py with oracle/mcts_ref.py):
identical applied-rule trace, per-iteration e-node / e-class counts, main-extractor costs
(float.hex), original / optimized cost and speedup bits, and the final program as the exact
``save_graph`` text."""

import json
from pathlib import Path

import pytest

GOLD = Path(__file__).resolve().parent / "golden" / "mcts"
CASES = sorted(p.stem for p in GOLD.glob("*.json"))


def _run(case: dict) -> dict:
    import sys

    sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))
    from make_mcts_golden import build_input

    from paper_2410_05534_b200 import tensor_ir as T
    from paper_2410_05534_b200.cost_model import CostModelConfig
    from paper_2410_05534_b200.mcts import MctsConfig, optimize_mcts
    from paper_2410_05534_b200.patterns import load_rules

    cfg = MctsConfig(**case["config"])
    rep = optimize_mcts(build_input(case["model"], T), load_rules(case["rules"]), cfg,
                        CostModelConfig(mode=case["cost_mode"]))
    return rep.to_json_dict()


def test_mcts_goldens_present():
    assert {"toy_b1", "toy_b8"} <= set(CASES)
    for name in CASES:
        case = json.loads((GOLD / f"{name}.json").read_text())
        rep = case["report"]
        orig, opt = float.fromhex(rep["original_cost"]), float.fromhex(rep["optimized_cost"])
        assert float.fromhex(rep["speedup_pct"]) == ((orig - opt) / orig * 100.0 if orig else 0.0)
        assert sum(rep["rule_histogram"].values()) == len(rep["iterations"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_device_mcts_equals_reference(name):
    case = json.loads((GOLD / f"{name}.json").read_text())
    got = _run(case)
    want = case["report"]
    assert got["iterations"] == want["iterations"], name
    assert got == want, name
