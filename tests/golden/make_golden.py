"""Generate the golden vectors by running the REFERENCE implementation.

Run in the build container only (needs /root/reference):

    python tests/golden/make_golden.py

For every fixture e-graph and seeded rewrite sequence it wraps the reference's
``EGraph.rebuild`` (egraph.py:203) to capture each *dirty* state right before the
rebuild inside ``apply_rule`` (rewrite.py:569), then records what the reference
computes on that state:

* rebuild   -- merge count, new hashcons order, find() of every id, ranks, classes
* ematch    -- ``joint_match`` of every rule's sources (rewrite.py:405), and the
               per-source ``ematch`` counts behind ``is_rule_applicable`` (579)
* extract   -- ``extract_default_greedy`` / ``extract_ocf_greedy``
               (extraction.py:157/229): total cost (float.hex) and chosen nodes,
               or the exception type and message
* apply     -- the ``ApplyReport`` of the application that produced the state

Inputs: the analog graphs of paper_2410_05534_b200/analogs.py, the reference
zoo, the toy term, and random small e-graphs; rules from
paper_2410_05534_b200/rules/. Output: tests/golden/*.json.gz (+ MANIFEST.sha256).
"""

from __future__ import annotations

import gzip
import hashlib
import json
import random
import sys
import time
from pathlib import Path

REF = "/root/reference/pkg/src"
HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, REF)
sys.path.insert(0, str(REPO))

from esat import egraph as E, extraction as X, rewrite as R, tensor_ir as T  # noqa: E402

from paper_2410_05534_b200 import analogs  # noqa: E402
from paper_2410_05534_b200.arena import export_state  # noqa: E402
from paper_2410_05534_b200.cost_model import CostModelConfig, egraph_costs  # noqa: E402
from paper_2410_05534_b200.symtab import SymbolTable  # noqa: E402

RULES_DIR = REPO / "paper_2410_05534_b200" / "rules"
MAX_MATCHES = 600          # explosion guard of the rollout generator (skip the rule)
JOINT_MATCH_NODE_CAP = 1300  # multi-pattern goldens only below this size (reference is quadratic)


class Capture:
    def __init__(self):
        self.on = False
        self.states = []
        self.symtab = None
        self.cfg = None
        orig = E.EGraph.rebuild
        cap = self

        def rebuild(egraph):
            snap = export_state(egraph, cap.symtab, cap.cfg) if cap.on else None
            merges = orig(egraph)
            if snap is not None:
                cap.states.append((snap, merges))
            return merges

        E.EGraph.rebuild = rebuild


CAP = Capture()


def node_rec(symtab, egraph, node):
    return [symtab.intern(node.symbol, egraph.language), list(node.children)]


def rebuild_golden(symtab, eg, merges):
    uf = eg._uf
    return {
        "merges": merges,
        "hashcons": [node_rec(symtab, eg, n) + [c] for n, c in eg.hashcons.items()],
        "find": [uf.find(i) for i in range(len(uf.parent))],
        "rank": list(uf.rank),
        "classes": [[cid, [node_rec(symtab, eg, n) for n in sorted(eg.classes[cid].nodes, key=E.node_sort_key)]]
                    for cid in eg.canonical_class_ids()],
        "root": eg.canonical_root() if eg.root is not None else None,
        "size": list(eg.size()),
    }


def subst_rec(s):
    return [list(s.roots), [[k, v] for k, v in s.vars], [[k, v] for k, v in s.params]]


def ematch_golden(eg, rules):
    out = []
    n_nodes = eg.size()[0]
    for r in rules:
        per_source = [len(R.ematch(eg, s)) for s in r.sources]
        rec = {"rule": r.id, "source_counts": per_source}
        if r.kind == "single" or n_nodes <= JOINT_MATCH_NODE_CAP:
            rec["matches"] = [subst_rec(s) for s in R.joint_match(eg, r.sources)]
        out.append(rec)
    return out


def extract_golden(symtab, eg, costs):
    res = {}
    for method, fn in (("default", X.extract_default_greedy), ("ocf", X.extract_ocf_greedy)):
        try:
            r = fn(eg, costs)
            res[method] = {"cost": float(r.total_cost).hex(),
                           "chosen": [[cid] + node_rec(symtab, eg, n) for cid, n in sorted(r.chosen.items())]}
        except X.ExtractionError as exc:
            res[method] = {"error": type(exc).__name__, "msg": str(exc)}
    return res


def report_rec(rep):
    return {k: getattr(rep, k) for k in ("rule_id", "matches_found", "changed", "nodes_after",
                                         "classes_after", "hit_node_limit", "cycles_filtered",
                                         "shape_filtered")}


def rollout_cases(label, eg, rules, symtab, cfg, seed, steps, node_limit, with_ematch=True):
    """Seeded random rule applications; one case per application that rebuilt."""
    rng = random.Random(seed)
    cases = []
    CAP.symtab, CAP.cfg = symtab, cfg
    for step in range(steps):
        if eg.size()[0] >= node_limit:
            break
        # applicable rules only (MCTS expansion prunes with blacklists), with the
        # explosion guard: a rule whose application would exceed MAX_MATCHES is not drawn
        live = [r for r in rules if 0 < len(R.joint_match(eg, r.sources)) <= MAX_MATCHES]
        if not live:
            break
        rule = live[rng.randrange(len(live))]
        CAP.states.clear()
        CAP.on = True
        rep = R.apply_rule(eg, rule, node_limit)
        CAP.on = False
        (dirty, merges), = CAP.states
        costs = egraph_costs(eg, cfg)
        case = {"name": f"{label}/seed{seed}/step{step}", "rule": rule.id, "apply": report_rec(rep),
                "state": dirty.to_json(), "rebuild": rebuild_golden(symtab, eg, merges),
                "extract": extract_golden(symtab, eg, costs)}
        if with_ematch:
            case["ematch"] = ematch_golden(eg, rules)
        cases.append(case)
    return cases


def initial_case(label, eg_builder, rules, symtab, cfg, with_ematch=True):
    CAP.symtab, CAP.cfg = symtab, cfg
    CAP.states.clear()
    CAP.on = True
    eg = eg_builder()
    CAP.on = False
    (dirty, merges), = CAP.states[-1:]
    costs = egraph_costs(eg, cfg)
    case = {"name": f"{label}/initial", "rule": None, "apply": None, "state": dirty.to_json(),
            "rebuild": rebuild_golden(symtab, eg, merges), "extract": extract_golden(symtab, eg, costs)}
    if with_ematch:
        case["ematch"] = ematch_golden(eg, rules)
    return eg, case


def symtab_json(symtab):
    a = symtab.arrays()
    return {
        "names": symtab.names,
        "values": symtab.values,
        "symbols": [[s.name, s.arity, repr(s.payload)] for s in symtab.symbols],
        "sym_params": [list(p) for p in symtab.params],
        **{k: v.tolist() for k, v in a.items()},   # name/arity/rank/poff/params (flat codes)
    }


def write(name, payload):
    path = HERE / f"{name}.json.gz"
    raw = json.dumps(payload, sort_keys=True, separators=(",", ":")).encode()
    with gzip.GzipFile(path, "wb", mtime=0) as fh:
        fh.write(raw)
    print(f"wrote {path.name}: {len(payload['cases'])} cases, {path.stat().st_size/1e3:.0f} kB", flush=True)


def group_tensor(name, builders, rules_file, cfg, seeds, steps, node_limit):
    rules = R.parse_rules((RULES_DIR / rules_file).read_text())
    symtab = SymbolTable()
    cases = []
    for label, build in builders:
        t0 = time.time()
        for seed in seeds:
            eg, init = initial_case(label, build, rules, symtab, cfg)
            if seed == seeds[0]:
                cases.append(init)
            cases.extend(rollout_cases(label, eg, rules, symtab, cfg, seed, steps, node_limit))
        print(f"  {label}: {time.time()-t0:.1f}s", flush=True)
    write(name, {"rules": rules_file, "cost": cfg.__dict__, "symtab": symtab_json(symtab), "cases": cases})


def random_egraph_cases(n_graphs, seed, keep_plain=300):
    """Random small dirty e-graphs (adds + unions) for rebuild / extraction fuzzing."""
    rng = random.Random(seed)
    symtab = SymbolTable()
    lang = R.TermLanguage()
    cases = []
    cost_of = {}
    for g in range(n_graphs):
        eg = E.EGraph(lang)
        ids = []
        for _ in range(rng.randint(1, 4)):
            ids.append(eg.add(E.ENode(E.Symbol(f"v{rng.randrange(3)}", 0))))
        for _ in range(rng.randint(2, 40)):
            ar = rng.choice((1, 2, 2, 3))
            name = f"f{rng.randrange(4)}" if ar < 3 else "g"
            kids = tuple(rng.choice(ids) for _ in range(ar))
            ids.append(eg.add(E.ENode(E.Symbol(name, ar), kids)))
        eg.root = ids[-1]
        for _ in range(rng.randint(0, 10)):
            eg.union(rng.choice(ids), rng.choice(ids))
        # stale-key adds after unions (hashcons keys computed with a mid-state UF)
        for _ in range(rng.randint(0, 3)):
            kids = tuple(rng.choice(ids) for _ in range(2))
            ids.append(eg.add(E.ENode(E.Symbol(f"f{rng.randrange(4)}", 2), kids)))
            if rng.random() < 0.5:
                eg.union(ids[-1], rng.choice(ids))
        cfg_costs = {}
        dirty = export_state(eg, symtab)
        sym_names = [symtab.symbols[s].name for s in dirty.hc_sym]
        for nm in set(sym_names):
            cost_of.setdefault(nm, rng.choice((0.0, 0.5, 1.0, 2.0, 3.0, 0.1, 0.7)))
        dirty.hc_cost[:] = [cost_of[nm] for nm in sym_names]
        merges = eg.rebuild()
        costs = {n: cost_of[n.symbol.name] for _, n in eg.enodes()}
        ext = extract_golden(symtab, eg, costs)
        interesting = merges > 0 or any("error" in v for v in ext.values())
        if interesting or keep_plain > 0:
            keep_plain -= 0 if interesting else 1
            cases.append({"name": f"random/{seed}/{g}", "rule": None, "apply": None, "state": dirty.to_json(),
                          "rebuild": rebuild_golden(symtab, eg, merges), "extract": ext})
        del cfg_costs
    return symtab, cases


def main():
    t0 = time.time()
    # 1. toy term + rule set R, AST-size costs
    toy_rules = R.parse_rules((RULES_DIR / "toy_math.rules").read_text())
    symtab = SymbolTable()
    cfg = CostModelConfig(mode="term")
    cases = []
    eg, init = initial_case("toy", lambda: T.toy_term_to_egraph(("div", ("mul", "a", 2), 2)), toy_rules, symtab, cfg)
    cases.append(init)
    for seed in range(6):
        eg = T.toy_term_to_egraph(("div", ("mul", "a", 2), 2))
        cases.extend(rollout_cases("toy", eg, toy_rules, symtab, cfg, seed, 12, 40))
    write("toy", {"rules": "toy_math.rules", "cost": cfg.__dict__, "symtab": symtab_json(symtab), "cases": cases})

    # 2. reference zoo with the TASO-analog rules, unit costs
    zoo = [(spec, (lambda s=spec: T.zoo_generate(s).to_egraph()))
           for spec in ("resblock_stack(3)", "mlp(3,16)", "attention_block(8,2)", "inception_cell(3)")]
    group_tensor("zoo", zoo, "taso_analog.rules", CostModelConfig(mode="unit"), seeds=(0, 1), steps=10,
                 node_limit=2000)

    # 3. the five BASELINE config analogs, analytic costs
    for model in analogs.ANALOGS:
        build = lambda m=model: T.graph_to_egraph(analogs.build_analog(m, T.GraphBuilder))
        group_tensor(f"analog_{model}", [(model, build)], "taso_analog.rules", CostModelConfig(),
                     seeds=(0, 1, 2), steps=10, node_limit=2000)

    # 4. random dirty e-graphs (merges during rebuild, cyclic OCF selections, infeasible roots)
    symtab, cases = random_egraph_cases(6000, seed=7)
    write("random", {"rules": None, "cost": None, "symtab": symtab_json(symtab), "cases": cases})

    manifest = "".join(f"{hashlib.sha256(p.read_bytes()).hexdigest()}  {p.name}\n"
                       for p in sorted(HERE.glob("*.json.gz")))
    (HERE / "MANIFEST.sha256").write_text(manifest)
    print(f"done in {time.time()-t0:.0f}s")


if __name__ == "__main__":
    main()
