"""The drop-in Python API (egraph / rewrite / extraction modules with the reference's names)
driving the device kernels: SPEC known-answer tests and a replay of the reference's own
seeded rollouts (tests/golden) -- same rule sequence, same ApplyReports, same rebuilt
hashcons, same extraction results."""

import random

import pytest

from golden_io import load_group

pytestmark = pytest.mark.gpu

MAX_MATCHES = 600  # tests/golden/make_golden.py


def _api():
    from paper_2410_05534_b200 import egraph, extraction, rewrite, tensor_ir

    return egraph, rewrite, extraction, tensor_ir


def test_toy_spec_kats():
    E, R, X, T = _api()
    eg = T.toy_term_to_egraph(("div", ("mul", "a", 2), 2))
    assert eg.size() == (4, 4)
    rules = R.load_rules("toy_math")
    subs = R.ematch(eg, R.parse_pattern("(mul ?x 2)"))
    assert len(subs) == 1 and eg.classes[subs[0].var("x")].nodes
    assert R.ematch(eg, R.parse_pattern("(div ?x ?x)")) == []
    assert len(R.ematch(eg, R.parse_pattern("?x"))) == 4
    assert not R.is_rule_applicable(eg, rules[2])
    rep = R.apply_rule(eg, rules[0])
    assert rep.changed and eg.size() == (6, 5)
    assert not R.apply_rule(eg, rules[0]).changed
    R.apply_rule(eg, rules[1])
    assert R.is_rule_applicable(eg, rules[2])


def test_congruence_rebuild_kat():
    E, R, X, T = _api()
    eg = E.EGraph(T.TermLanguage())
    a = eg.add(E.ENode(E.Symbol("a", 0)))
    b = eg.add(E.ENode(E.Symbol("b", 0)))
    fa = eg.add(E.ENode(E.Symbol("f", 1), (a,)))
    fb = eg.add(E.ENode(E.Symbol("f", 1), (b,)))
    eg.union(a, b)
    assert eg.rebuild() == 1 and eg.find(fa) == eg.find(fb)
    assert eg.rebuild() == 0


def test_resblock_extraction_kats():
    """resblock-style residual chain: default over-counts shared convs, OCF is exact."""
    E, R, X, T = _api()
    from paper_2410_05534_b200.cost_model import CostModelConfig, egraph_costs

    for k in (1, 2, 3, 4):
        b = T.GraphBuilder()
        x = b.input("x", (1, 8, 16, 16))
        w = b.weight("w", (8, 8, 3, 3))
        for _ in range(k):
            c1 = b.op("conv2d", x, w, stride=1, padding=1, activation="none")
            c2 = b.op("conv2d", c1, w, stride=1, padding=1, activation="none")
            x = b.op("ewadd", c1, c2)
        eg = T.graph_to_egraph(b.build(b.op("relu", x)))
        costs = egraph_costs(eg, CostModelConfig(mode="unit"))
        assert X.extract_default_greedy(eg, costs).total_cost == 2 ** (k + 2) - 3
        assert X.extract_ocf_greedy(eg, costs).total_cost == 3 * k + 1


def _sym_key(st_json, sid):
    name, arity, payload = st_json["symbols"][sid]
    return (name, arity, payload)


@pytest.mark.parametrize("group,model", [("analog_bert", "bert"), ("analog_resnext50", "resnext50"),
                                         ("analog_inception_v3", "inception_v3"), ("analog_nasnet_a", "nasnet_a"),
                                         ("analog_nasrnn", "nasrnn"), ("toy", None)])
def test_replay_reference_rollouts(group, model):
    """Replays make_golden.rollout_cases with the drop-in API and compares every step."""
    E, R, X, T = _api()
    from paper_2410_05534_b200 import analogs
    from paper_2410_05534_b200.cost_model import CostModelConfig, egraph_costs

    g = load_group(group)
    rules = R.load_rules(g["rules"].replace(".rules", ""))
    cfg = CostModelConfig(**g["cost"])
    cases = {c["name"]: c for c in g["cases"]}
    if model is None:
        build = lambda: T.toy_term_to_egraph(("div", ("mul", "a", 2), 2))  # noqa: E731
        label, seeds, steps, limit = "toy", range(6), 12, 40
    else:
        build = lambda: T.graph_to_egraph(analogs.build_analog(model, T.GraphBuilder))  # noqa: E731
        label, seeds, steps, limit = model, (0, 1, 2), 10, 2000
    checked = 0
    for seed in seeds:
        eg = build()
        rng = random.Random(seed)
        for step in range(steps):
            if eg.size()[0] >= limit:
                break
            live = [r for r in rules if 0 < len(R.joint_match(eg, r.sources)) <= MAX_MATCHES]
            if not live:
                break
            rule = live[rng.randrange(len(live))]
            rep = R.apply_rule(eg, rule, limit)
            ref = cases[f"{label}/seed{seed}/step{step}"]
            assert ref["rule"] == rule.id
            assert {k: getattr(rep, k) for k in ref["apply"]} == ref["apply"], (ref["name"], rep)
            gold = ref["rebuild"]
            assert list(eg.size()) == gold["size"]
            got_hc = [(n.symbol.name, n.symbol.arity, repr(n.symbol.payload), list(n.children), c)
                      for n, c in eg.hashcons.items()]
            want_hc = [(*_sym_key(g["symtab"], s), kids, c) for s, kids, c in gold["hashcons"]]
            assert got_hc == want_hc, ref["name"]
            costs = egraph_costs(eg, cfg)
            for method, fn in (("default", X.extract_default_greedy), ("ocf", X.extract_ocf_greedy)):
                exp = ref["extract"][method]
                try:
                    res = fn(eg, costs)
                    got = float(res.total_cost).hex()
                except X.ExtractionError as exc:
                    got = str(exc)
                assert got == exp.get("cost", exp.get("msg")), (ref["name"], method)
            checked += 1
    assert checked > 0


def test_extraction_costs_not_cached_across_calls():
    """Two different cost dicts on the same (unchanged) e-graph, back to back, and a dict edited in
    place: each extraction must use the costs it is given (no identity-keyed cache)."""
    E, R, X, T = _api()
    from paper_2410_05534_b200 import analogs
    from paper_2410_05534_b200.cost_model import CostModelConfig, egraph_costs

    eg = T.graph_to_egraph(analogs.build_analog("nasrnn", T.GraphBuilder))
    unit = X.extract_ocf_greedy(eg, egraph_costs(eg, CostModelConfig(mode="unit"))).total_cost
    flops = X.extract_ocf_greedy(eg, egraph_costs(eg, CostModelConfig(mode="analytic"))).total_cost
    assert unit != flops
    assert X.extract_ocf_greedy(eg, egraph_costs(eg, CostModelConfig(mode="unit"))).total_cost == unit
    costs = egraph_costs(eg, CostModelConfig(mode="unit"))
    base = X.extract_default_greedy(eg, costs).total_cost
    for node in costs:
        costs[node] *= 2.0
    assert X.extract_default_greedy(eg, costs).total_cost == 2.0 * base
