"""Generate the benchmark leaf sets by running the REFERENCE implementation.

    python tests/golden/make_bench_leaves.py [model ...]

An MCTS simulation applies random rewrite rules to a
snapshot and extracts after every step; every step is one *leaf* of the data-parallel hot
path: the dirty e-graph left by apply_rule's unions (rewrite.py:567-568) goes through
rebuild (rewrite.py:569), all-rule e-matching (next step / blacklists, rewrite.py:579) and
the main extractor. This script replays seeded rollouts with the reference's own
``apply_rule`` and records the dirty state in front of the final rebuild of each rollout:

* model: one of paper_2410_05534_b200/analogs.py; rules: rules/taso_analog.rules
* rollout depth ~ U{1..10} (max simulation depth 10), node limit 2000
* each step draws uniformly among rules with at least one and at most MAX_MATCHES matches
  (applicable rules, as MCTS blacklists prune; the cap guards against one application
  exploding the graph beyond what the reference can replay in reasonable time)

Output: tests/golden/bench_<model>.npz -- packed leaves (arena.py layout) + symbol table +
the reference's OCF and default-greedy root costs for every leaf (parity spot checks).
"""

from __future__ import annotations

import json
import multiprocessing as mp
import random
import sys
import time
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, REF)
sys.path.insert(0, str(REPO))

MAX_MATCHES = 600
NODE_LIMIT = 2000


def rollout(args):
    model, seed = args
    from esat import egraph as E, extraction as X, rewrite as R, tensor_ir as T

    from paper_2410_05534_b200 import analogs
    from paper_2410_05534_b200.arena import export_state
    from paper_2410_05534_b200.cost_model import CostModelConfig, egraph_costs
    from paper_2410_05534_b200.symtab import SymbolTable

    rules = R.parse_rules((REPO / "paper_2410_05534_b200" / "rules" / "taso_analog.rules").read_text())
    cfg = CostModelConfig()
    rng = random.Random(1000003 * seed + 17)
    eg = T.graph_to_egraph(analogs.build_analog(model, T.GraphBuilder))
    depth = rng.randint(1, 10)
    captured = []
    orig = E.EGraph.rebuild
    st = SymbolTable()

    def cap(self):
        captured.append(export_state(self, st, cfg))
        return orig(self)

    last = None
    for _ in range(depth):
        if eg.size()[0] >= NODE_LIMIT:
            break
        live = [r for r in rules if 0 < len(R.joint_match(eg, r.sources)) <= MAX_MATCHES]
        if not live:
            break
        rule = live[rng.randrange(len(live))]
        captured.clear()
        E.EGraph.rebuild = cap
        try:
            R.apply_rule(eg, rule, NODE_LIMIT)
        finally:
            E.EGraph.rebuild = orig
        last = captured[0]
    if last is None:  # no applicable rule: the leaf is the initial graph's own rebuild
        captured.clear()
        E.EGraph.rebuild = cap
        try:
            eg = T.graph_to_egraph(analogs.build_analog(model, T.GraphBuilder))
        finally:
            E.EGraph.rebuild = orig
        last = captured[-1]
    costs = egraph_costs(eg, cfg)
    ocf = X.extract_ocf_greedy(eg, costs).total_cost
    dflt = X.extract_default_greedy(eg, costs).total_cost
    syms = [(s, p) for s, p in zip(st.symbols, st.params)]
    return seed, last, syms, ocf, dflt, eg.size()


def main():
    models = sys.argv[1:] or ["nasrnn"]
    from esat import tensor_ir as T  # noqa: F401  (warm import)

    from paper_2410_05534_b200.arena import Batch
    from paper_2410_05534_b200.symtab import SymbolTable
    from esat import rewrite as R

    import os

    n_leaves = int(os.environ.get("ESAT_BENCH_LEAVES", "256"))   # seeds 0..n-1 (a prefix of a larger set)
    for model in models:
        t0 = time.time()
        with mp.Pool(mp.cpu_count()) as pool:
            res = pool.map(rollout, [(model, s) for s in range(n_leaves)], chunksize=1)
        res.sort(key=lambda r: r[0])
        lang_params = {}
        gst = SymbolTable()

        class _L:  # params already computed by the worker's language
            def node_params(self, symbol):
                return lang_params[(symbol.name, symbol.arity, repr(symbol.payload))]

        lang = _L()
        leaves = []
        for seed, leaf, syms, ocf, dflt, size in res:
            remap = np.zeros(len(syms), np.uint32)
            for i, (s, p) in enumerate(syms):
                lang_params[(s.name, s.arity, repr(s.payload))] = p
                remap[i] = gst.intern(s, lang)
            leaf.hc_sym = remap[leaf.hc_sym]
            leaves.append(leaf)
        packed = Batch(leaves).pack()
        arr = gst.arrays()
        rules_text = (REPO / "paper_2410_05534_b200" / "rules" / "taso_analog.rules").read_text()
        R.parse_rules(rules_text)  # validates
        out = HERE / f"bench_{model}.npz"
        np.savez_compressed(
            out,
            **{k: v for k, v in packed.items() if k != "n_leaves"},
            n_leaves=np.array(packed["n_leaves"]),
            sym_name=arr["name"], sym_arity=arr["arity"], sym_rank=arr["rank"], sym_poff=arr["poff"],
            sym_params=arr["params"],
            meta=np.array(json.dumps({"model": model, "names": gst.names, "values": gst.values,
                                      "symbols": [[s.name, s.arity, repr(s.payload)] for s in gst.symbols],
                                      "max_matches": MAX_MATCHES, "node_limit": NODE_LIMIT})),
            ref_ocf=np.array([r[3] for r in res], np.float64),
            ref_default=np.array([r[4] for r in res], np.float64),
            sizes=np.array([r[5] for r in res], np.int64),
        )
        sz = np.array([r[5][0] for r in res])
        print(f"{model}: {n_leaves} leaves, nodes min/mean/max {sz.min()}/{sz.mean():.0f}/{sz.max()}, "
              f"{out.stat().st_size/1e6:.1f} MB, {time.time()-t0:.0f}s", flush=True)


if __name__ == "__main__":
    main()
