"""TEST INFRASTRUCTURE ONLY -- the reference's own Python timed on the leaf pipeline (bench.py's
cpu_baseline leg): one leaf = ``EGraph.rebuild`` of the dirty state
(egraph.py:203-226), ``joint_match`` of every rule's sources (rewrite.py:405-433) and
``extract_ocf_greedy`` (extraction.py:229-242), on reference objects rebuilt from the arena leaves.

Bounded samples only: the reference is orders of magnitude slower than the C port.
"""

from __future__ import annotations

import ast
import multiprocessing as mp
import os
import time

from .mcts_ref import import_reference

_W = {}


def to_ref_egraph(leaf, symbols, E, T):
    """Reference EGraph of an arena leaf (the dirty hashcons in order + union-find)."""
    syms = _W.get(("syms", id(symbols)))
    if syms is None:
        syms = [E.Symbol(n, a, ast.literal_eval(p) if isinstance(p, str) else p) for n, a, p in symbols]
        _W[("syms", id(symbols))] = syms
    eg = E.EGraph(T.TensorLanguage())
    ko = leaf.hc_koff
    eg.hashcons = {E.ENode(syms[int(leaf.hc_sym[i])], tuple(int(k) for k in leaf.hc_kids[ko[i]:ko[i + 1]])):
                   int(leaf.hc_cid[i]) for i in range(leaf.n)}
    eg._uf.parent = [int(x) for x in leaf.uf_parent]
    eg._uf.rank = [int(x) for x in leaf.uf_rank]
    eg.root = None if leaf.root == 0xFFFFFFFF else int(leaf.root)
    eg.dirty = [0]
    return eg


def leaf_pipeline(leaf, symbols, rules, cfg):
    from paper_2410_05534_b200.cost_model import egraph_costs

    E, R, X, T = import_reference()
    eg = to_ref_egraph(leaf, symbols, E, T)
    eg.rebuild()
    matches = sum(len(R.joint_match(eg, r.sources)) for r in rules)
    try:
        cost = X.extract_ocf_greedy(eg, egraph_costs(eg, cfg)).total_cost
    except X.ExtractionError:
        cost = float("inf")
    return matches, cost


def _init(leaves, symbols, rules_text, cfg):
    E, R, X, T = import_reference()
    _W["job"] = (leaves, symbols, R.parse_rules(rules_text), cfg)


def _run(i):
    leaves, symbols, rules, cfg = _W["job"]
    return leaf_pipeline(leaves[i], symbols, rules, cfg)


def time_reference(leaves, symbols, rules_text, cfg, budget_s: float = 8.0, workers: int = 1) -> dict:
    """Leaves/s of the reference Python on ``leaves`` (cycled) for about ``budget_s`` seconds."""
    _, R, _, _ = import_reference()
    rules = R.parse_rules(rules_text)
    done, t0 = 0, time.perf_counter()
    if workers <= 1:
        while time.perf_counter() - t0 < budget_s:
            leaf_pipeline(leaves[done % len(leaves)], symbols, rules, cfg)
            done += 1
    else:
        ctx = mp.get_context("fork")
        with ctx.Pool(workers, initializer=_init, initargs=(leaves, symbols, rules_text, cfg)) as pool:
            t0 = time.perf_counter()
            it = pool.imap_unordered(_run, (i % len(leaves) for i in range(10 ** 9)), chunksize=1)
            while time.perf_counter() - t0 < budget_s:
                next(it)
                done += 1
            dt = time.perf_counter() - t0
            pool.terminate()
            return {"value": done / dt, "cores": workers, "leaves": done, "seconds": dt}
    dt = time.perf_counter() - t0
    return {"value": done / dt, "cores": 1, "leaves": done, "seconds": dt}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_cores() -> int:
    return len(os.sched_getaffinity(0))
