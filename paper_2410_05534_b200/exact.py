"""Exact (branch-and-bound) extraction for the run's final program.

Host-side restatement of ``extract_exact`` (extraction.py:252-349): one binary choice per e-node,
exactly one node in the root class, the classes a chosen node needs must be chosen, blacklisted
nodes excluded, acyclic. The incumbent is seeded with the OCF greedy selection (extraction.py:292,
here the device's k_extract result when the caller has it) and the bound is the sum of per-class
minimum node costs over the classes still needed. The search order -- needed classes ascending,
candidates in ``node_sort_key`` order, prune on ``bound >= best - 1e-12``, accept on
``cost < best - 1e-12`` -- is the reference's, so the same optimum is returned when several tie.

This runs once per optimization (the paper's final ILP extraction), not per MCTS leaf, so it stays
on the host as the SURVEY ranks it. The class graph is pre-canonicalised once (the reference
re-canonicalises children in every reachability probe).
"""

from __future__ import annotations

import math
import sys

from .egraph import node_sort_key
from .extraction import (CapacityError, ExtractionError, ExtractionResult, InfeasibleExtraction,
                         selection_dag_cost, validate_extraction)


def _reachable_chosen(egraph, chosen: dict) -> dict:
    """extraction.py:106-115."""
    out: dict = {}
    stack = [egraph.canonical_root()]
    while stack:
        cid = egraph.find(stack.pop())
        if cid in out:
            continue
        out[cid] = chosen[cid]
        stack.extend(chosen[cid].children)
    return out


def extract_exact(egraph, costs: dict, blacklist=(), size_bound: int = 5000, seed=None) -> ExtractionResult:
    """Globally minimal unique-node-cost selection (extraction.py:252-349). ``seed`` may carry an
    already computed OCF ExtractionResult; otherwise extract_ocf_greedy runs on the device."""
    if egraph.dirty:
        raise ExtractionError("extraction requires a rebuilt e-graph")
    n_nodes = egraph.size()[0]
    if n_nodes > size_bound:
        raise CapacityError(f"{n_nodes} e-nodes exceeds exact-extraction bound {size_bound}; use a greedy extractor")
    banned = {egraph.canonicalize(n) for n in blacklist}
    root = egraph.canonical_root()
    find = egraph.find
    candidates = {}
    kids_of = {}
    for cid in egraph.canonical_class_ids():
        nodes = [n for n in sorted(egraph.classes[cid].nodes, key=node_sort_key) if n not in banned]
        candidates[cid] = nodes
        for n in nodes:
            kids_of[n] = tuple(dict.fromkeys(find(c) for c in n.children))
    if not candidates[root]:
        raise InfeasibleExtraction("every e-node in the root e-class is blacklisted")
    min_cost = {cid: min((costs[n] for n in nodes), default=math.inf) for cid, nodes in candidates.items()}

    best_cost, best_sel = math.inf, None
    try:
        if seed is None:
            from .extraction import extract_ocf_greedy

            seed = extract_ocf_greedy(egraph, costs)
        seeded = {cid: n for cid, n in seed.chosen.items() if n not in banned}
        if seeded == seed.chosen:
            best_cost = selection_dag_cost(egraph, seed.chosen, costs)
            best_sel = dict(seed.chosen)
    except ExtractionError:
        pass

    chosen: dict = {}

    def reaches(start: int, goal: int) -> bool:
        stack, seen = [start], set()
        while stack:
            cid = stack.pop()
            if cid == goal:
                return True
            if cid in seen or cid not in chosen:
                continue
            seen.add(cid)
            stack.extend(kids_of[chosen[cid]])
        return False

    def search(need: list, cost_so_far: float) -> None:
        nonlocal best_cost, best_sel
        if not need:
            if cost_so_far < best_cost - 1e-12:
                best_cost, best_sel = cost_so_far, dict(chosen)
            return
        bound = cost_so_far + sum(min_cost[c] for c in need)
        if bound >= best_cost - 1e-12:
            return
        cid, rest = need[0], need[1:]
        for node in candidates[cid]:
            kids = kids_of[node]
            if any(reaches(k, cid) for k in kids):
                continue
            chosen[cid] = node
            new_need = [k for k in kids if k not in chosen and k not in rest]
            search(sorted(set(rest) | set(new_need)), cost_so_far + costs[node])
            del chosen[cid]

    old = sys.getrecursionlimit()
    sys.setrecursionlimit(max(old, 2 * len(candidates) + 100))
    try:
        search([root], 0.0)
    finally:
        sys.setrecursionlimit(old)
    if best_sel is None:
        raise InfeasibleExtraction("no acyclic selection satisfies the constraints")
    res = ExtractionResult(best_cost, _reachable_chosen(egraph, best_sel), "exact")
    validate_extraction(egraph, res)
    return res
