"""TEST INFRASTRUCTURE ONLY -- the CPU reference engine of the MCTS parity tests.

Implements the engine contract of paper_2410_05534_b200/mcts.py (initial / evaluate / expand /
simulate / final) on the REFERENCE's own objects: ``esat.egraph.EGraph`` snapshots
(egraph.py:300-312), ``esat.rewrite.apply_rule`` (rewrite.py:526-573, which rebuilds),
``esat.rewrite.is_rule_applicable`` (rewrite.py:579-589), ``esat.extraction.extract_ocf_greedy`` /
``extract_default_greedy`` (extraction.py:157/229) and, for the final program,
``esat.tensor_ir.extraction_to_graph`` + ``save_graph`` (tensor_ir.py:316-352, 487-504).
``optimize_mcts(..., engine=ReferenceEngine(...))`` is therefore the SPEC MCTS (which the reference
lacks) driven by the reference's e-graph code; tests/golden/make_mcts_golden.py records
its RunReports and tests/test_gpu_mcts_parity.py requires DeviceEngine to reproduce them exactly.

The cost model is SPEC's (cost_model.py, noise 0) -- the reference ships none.

Leaves of one batch are independent, so ``workers > 1`` evaluates them in forked worker processes
(leaf l lives in worker l % workers for a whole rollout); every random draw stays in the parent, in
DeviceEngine's order, so the result does not depend on ``workers``.

Never imported by the product package.
"""

from __future__ import annotations

import math
import multiprocessing as mp
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
REF_PATHS = (REPO / "baseline" / "_ref", Path("/root/reference/pkg/src"))


def import_reference():
    """The reference package (installed into baseline/_ref, or the source tree in the build
    container). Raises ImportError when neither exists."""
    for p in REF_PATHS:
        if (p / "esat").is_dir() and str(p) not in sys.path:
            sys.path.insert(0, str(p))
            break
    from esat import egraph as E, extraction as X, rewrite as R, tensor_ir as T  # noqa: F401

    return E, R, X, T


def reference_available() -> bool:
    try:
        import_reference()
        return True
    except ImportError:
        return False


class _Ops:
    """The per-leaf reference calls (shared by the in-process and worker paths)."""

    def __init__(self, rules_text: str, cost_config, method: str):
        from paper_2410_05534_b200.cost_model import egraph_costs

        self.E, self.R, self.X, self.T = import_reference()
        self.rules = self.R.parse_rules(rules_text)
        self.cfg, self.method = cost_config, method
        self.egraph_costs = egraph_costs

    def extract(self, eg, method=None):
        fn = {"ocf": self.X.extract_ocf_greedy, "default": self.X.extract_default_greedy}[method or self.method]
        try:
            return fn(eg, self.egraph_costs(eg, self.cfg)).total_cost
        except self.X.ExtractionError:
            return math.inf

    def applicable(self, eg):
        return [self.R.is_rule_applicable(eg, r) for r in self.rules]

    def apply(self, eg, rule: int):
        return self.R.apply_rule(eg, self.rules[rule]).changed


def _worker(conn, rules_text, cost_config, method):
    ops = _Ops(rules_text, cost_config, method)
    leaves = {}
    while True:
        msg = conn.recv()
        kind = msg[0]
        if kind == "stop":
            return
        if kind == "load":            # (l, egraph)
            for l, eg in msg[1]:
                leaves[l] = eg
            conn.send(None)
        elif kind == "step":          # [(l, rule, want fingerprint)] -> [(l, cost, n, fingerprint)]
            out = []
            for l, rule, want_fp in msg[1]:
                ops.apply(leaves[l], rule)
                out.append((l, ops.extract(leaves[l]), leaves[l].size()[0], leaves[l].fingerprint() if want_fp else 0))
            conn.send(out)
        elif kind == "expand":        # [(l, egraph, rule)] -> [(l, child, changed, cost, n, c, app)]
            out = []
            for l, eg, rule in msg[1]:
                g = eg.snapshot()
                ch = ops.apply(g, rule)
                n, c = g.size()
                out.append((l, g, ch, ops.extract(g), n, c, ops.applicable(g)))
            conn.send(out)
        elif kind == "drop":
            leaves.clear()
            conn.send(None)


class ReferenceEngine:
    def __init__(self, rules_text: str, cost_config, method: str = "ocf", workers: int = 1):
        self.ops = _Ops(rules_text, cost_config, method)
        self.rules_text, self.cfg, self.method = rules_text, cost_config, method
        self.workers = max(1, int(workers))
        self._pool = None
        self.cache = None

    def configure(self, cfg):
        from paper_2410_05534_b200.mcts import ExtractionCache

        self.method = self.ops.method = cfg.main_extractor
        self.cache = ExtractionCache() if cfg.extraction_cache else None

    # -- worker pool (fork; leaves pinned to workers) ------------------------------------
    def _conns(self):
        if self._pool is None and self.workers > 1:
            ctx = mp.get_context("fork")
            self._pool = []
            for _ in range(self.workers):
                a, b = ctx.Pipe()
                p = ctx.Process(target=_worker, args=(b, self.rules_text, self.cfg, self.method), daemon=True)
                p.start()
                self._pool.append((p, a))
        return [c for _, c in self._pool] if self._pool else None

    def close(self):
        if self._pool:
            for p, c in self._pool:
                c.send(("stop",))
                p.join(timeout=10)
            self._pool = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _scatter(self, kind, items):
        """items: [(l, ...)] -> results in leaf order, computed by worker l % W."""
        conns = self._conns()
        if conns is None:
            return None
        W = len(conns)
        parts = [[] for _ in range(W)]
        for it in items:
            parts[it[0] % W].append(it)
        for w, c in enumerate(conns):
            c.send((kind, parts[w]))
        out = {}
        for c in conns:
            for r in c.recv() or []:
                out[r[0]] = r
        return [out[it[0]] for it in items] if out else []

    # -- engine contract ----------------------------------------------------------------
    def initial(self, egraph):
        return egraph.snapshot()

    def evaluate(self, states):
        clean, cost, n, c, app = [], [], [], [], []
        for s in states:
            g = s.snapshot()
            if g.dirty:
                g.rebuild()
            clean.append(g)
            cost.append(self.ops.extract(g))
            nn, cc = g.size()
            n.append(nn)
            c.append(cc)
            app.append(self.ops.applicable(g))
        return clean, np.array(cost), np.array(n), np.array(c), np.array(app, bool).reshape(len(states), -1)

    def expand(self, states, rules):
        res = self._scatter("expand", [(l, s, int(r)) for l, (s, r) in enumerate(zip(states, rules))])
        if res is None:
            res = []
            for l, (s, r) in enumerate(zip(states, rules)):
                g = s.snapshot()
                ch = self.ops.apply(g, int(r))
                nn, cc = g.size()
                res.append((l, g, ch, self.ops.extract(g), nn, cc, self.ops.applicable(g)))
        kids = [r[1] for r in res]
        return (kids, np.array([r[2] for r in res], bool), np.array([r[3] for r in res], np.float64),
                np.array([r[4] for r in res]), np.array([r[5] for r in res]),
                np.array([r[6] for r in res], bool).reshape(len(states), -1))

    def simulate(self, states, costs0, allowed, steps: int, node_limit: int, seeds):
        """DeviceEngine.simulate's loop, leaf by leaf on reference snapshots (same draws)."""
        import random

        from paper_2410_05534_b200.mcts import rollout_rewards

        L = len(states)
        rngs = [random.Random(sd) for sd in seeds]
        snaps = [s.snapshot() for s in states]
        pooled = self._conns() is not None
        if pooled:
            self._scatter("load", [(l, snaps[l]) for l in range(L)])
        reward = np.zeros(L)
        prev = np.asarray(costs0, np.float64).copy()
        live = np.ones(L, bool)
        for _ in range(steps):
            rules = [None] * L
            for l in range(L):
                if live[l] and allowed[l]:
                    rules[l] = rngs[l].choice(allowed[l])
                else:
                    live[l] = False
            if not live.any():
                break
            cost = np.full(L, math.inf)
            n = np.zeros(L, np.int64)
            fps = np.zeros(L, np.uint64)
            todo = [(l, rules[l], self.cache is not None) for l in range(L) if live[l]]
            if pooled:
                for l, cst, nn, fp in self._scatter("step", todo):
                    cost[l], n[l], fps[l] = cst, nn, fp
            else:
                for l, r, _ in todo:
                    self.ops.apply(snaps[l], r)
                    cost[l], n[l] = self.ops.extract(snaps[l]), snaps[l].size()[0]
                    if self.cache is not None:
                        fps[l] = snaps[l].fingerprint()   # the reference's own WL hash (egraph.py:247)
            if self.cache is not None:
                cost = self.cache.resolve(fps, live, cost)
            rollout_rewards(reward, prev, live, cost)
            live &= n < node_limit
        if pooled:
            for c in self._conns():
                c.send(("drop",))
                c.recv()
        return reward

    def final(self, state, method: str):
        X, T = self.ops.X, self.ops.T
        costs = self.ops.egraph_costs(state, self.cfg)
        fn = {"ocf": X.extract_ocf_greedy, "default": X.extract_default_greedy, "exact": X.extract_exact}[method]
        try:
            res = fn(state, costs)
        except X.ExtractionError:
            return math.inf, None
        if type(state.language).__name__ != "TensorLanguage":
            return res.total_cost, None
        try:
            g = T.extraction_to_graph(state, res)
        except T.GraphFormatError:
            return res.total_cost, None
        with tempfile.TemporaryDirectory() as d:
            path = os.path.join(d, "g.json")
            T.save_graph(g, path)
            return res.total_cost, Path(path).read_text()
