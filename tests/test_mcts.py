"""MCTS driver: SPEC.md mcts-module examples on the host, and device-batched
searches on the toy fixture and an analog model."""

import math
import random

import pytest


def test_ucb1_spec_examples():
    from paper_2410_05534_b200.mcts import ucb1

    assert ucb1(1, 1, 1, 1) == 1.0
    assert abs(ucb1(10, 4, 16, 1) - (2.5 + math.sqrt(math.log(16) / 4))) < 1e-12
    assert ucb1(5, 1, 2, 0) > ucb1(1, 1, 2, 0)                            # SPEC.md:581 (c = 0)


def test_update_and_best_child_spec_examples():
    from paper_2410_05534_b200.mcts import SearchNode, best_child, update

    root = SearchNode(None, 0.0, 0)
    a, b = SearchNode(None, 0.0, 0, parent=root, rule=0), SearchNode(None, 0.0, 0, parent=root, rule=1)
    root.children = {0: a, 1: b}
    update(a, 1.0)
    update(a, 3.0)
    assert (a.v, a.n) == (4.0, 2) and root.n == 2
    update(b, 3.0)
    assert best_child(root) == 1                                           # SPEC.md:629 (mean 3 > 2)
    b.s = True
    assert best_child(root) == 0
    a.s = True
    assert best_child(root) is None


@pytest.mark.gpu
def test_toy_mcts_reaches_optimum():
    """SPEC AC-1 analog: toy (a*2)/2 with rule set R, node limit 10 -> extracted cost 1 (term `a`)."""
    from paper_2410_05534_b200 import tensor_ir as T
    from paper_2410_05534_b200.cost_model import CostModelConfig
    from paper_2410_05534_b200.mcts import MctsConfig, optimize_mcts
    from paper_2410_05534_b200.patterns import load_rules

    eg = T.toy_term_to_egraph(("div", ("mul", "a", 2), 2))
    cfg = MctsConfig(budget=64, node_limit=10, seed=0, batch=8, headroom=256)
    rep = optimize_mcts(eg, load_rules("toy_math"), cfg, CostModelConfig(mode="term"))
    assert rep.original_cost == 4.0 and rep.optimized_cost == 1.0, rep   # 4 e-nodes (shared `2`) -> `a`
    assert rep.speedup_pct == 75.0


@pytest.mark.gpu
def test_analog_mcts_deterministic_and_improves():
    from paper_2410_05534_b200 import analogs
    from paper_2410_05534_b200 import tensor_ir as T
    from paper_2410_05534_b200.cost_model import CostModelConfig
    from paper_2410_05534_b200.mcts import MctsConfig, optimize_mcts
    from paper_2410_05534_b200.patterns import load_rules

    runs = []
    for _ in range(2):
        eg = T.graph_to_egraph(analogs.build_analog("nasrnn", T.GraphBuilder))
        cfg = MctsConfig(budget=32, node_limit=2000, seed=3, batch=16, max_sim_steps=4)
        rep = optimize_mcts(eg, load_rules("taso_analog"), cfg, CostModelConfig())
        runs.append(rep.to_json_dict())
    assert runs[0] == runs[1]
    assert rep.trace and rep.optimized_cost <= rep.original_cost, runs[0]
    assert rep.final_program is not None


@pytest.mark.gpu
def test_seed_sweep_single_rank():
    """Config 5 structure on one GPU: the sweep's rows equal direct optimize_mcts runs per seed."""
    from paper_2410_05534_b200 import analogs
    from paper_2410_05534_b200 import tensor_ir as T
    from paper_2410_05534_b200.cost_model import CostModelConfig
    from paper_2410_05534_b200.mcts import MctsConfig, optimize_mcts
    from paper_2410_05534_b200.parallel import root_parallel_sweep
    from paper_2410_05534_b200.patterns import load_rules

    rules = load_rules("taso_analog")

    def run(seed):
        eg = T.graph_to_egraph(analogs.build_analog("nasnet_a", T.GraphBuilder))
        cfg = MctsConfig(budget=16, node_limit=2000, seed=seed, batch=8, max_sim_steps=3)
        rep = optimize_mcts(eg, rules, cfg, CostModelConfig())
        return rep.optimized_cost, rep.trace

    res, best = root_parallel_sweep(run, [0, 1])
    direct = [run(0), run(1)]
    assert all(d[1] for d in direct)   # the searches applied rules
    assert [r[1] for r in res] == [d[0] for d in direct]
    assert best[1] == min(d[0] for d in direct)
