"""Batched MCTS over rewrite-rule applications (§4.1).

The search tree lives on the host; every e-graph operation of an iteration batch runs on the
device: expansion applies the sampled rule to a snapshot of the selected node (k_apply, then
k_rebuild), blacklists come from per-source e-matching of the child (is_rule_applicable,
rewrite.py:579-589: a rule is inapplicable as soon as one source has no match), and the
simulations are device-resident random rollouts -- apply, rebuild, extract after every step,
reward Eq. 3 ``r = sum max(cost_{i-1} - cost_i, 0)`` anchored at the child's own extracted cost.

SPEC's concurrency model allows simulations of distinct iterations to run in parallel on
snapshots with the results applied to the tree serially: ``batch`` selections are
made sequentially (a node/rule pair is reserved so one batch never expands it twice), the batch's
expansions and simulations run as one device batch, and the updates are applied in selection
order. ``batch=1`` is the strictly sequential search.
"""

from __future__ import annotations

import math
import random
from dataclasses import dataclass, field

import numpy as np

from . import native
from .apply import ApplyDriver
from .arena import Batch, LeafState
from .pipeline import LeafPipeline

NONE = 0xFFFFFFFF


@dataclass
class MctsConfig:
    budget: int = 128
    c: float = math.sqrt(2.0)
    stop_prob: float = 0.5
    max_sim_steps: int = 10
    node_limit: int = 2000
    seed: int = 0
    main_extractor: str = "ocf"
    batch: int = 32
    headroom: int = 4096


@dataclass
class SearchNode:
    state: LeafState
    cost: float
    n_nodes: int
    v: float = 0.0
    n: int = 0
    s: bool = False
    b: set = field(default_factory=set)
    children: dict = field(default_factory=dict)
    parent: "SearchNode | None" = None
    rule: int | None = None
    pending: set = field(default_factory=set)


def ucb1(v: float, n: int, N: int, c: float) -> float:
    """Eq. 2: v/n + c * sqrt(ln N / n)."""
    return v / n + c * math.sqrt(math.log(N) / n)


def update(node: SearchNode, reward: float) -> None:
    """v += r, n += 1 up to the root."""
    while node is not None:
        node.v += reward
        node.n += 1
        node = node.parent


def best_child(root: SearchNode):
    """Rule of the non-saturated visited child with the highest mean value, ties -> lowest id."""
    best, key = None, None
    for rid in sorted(root.children):
        ch = root.children[rid]
        if ch.s or ch.n == 0:
            continue
        m = ch.v / ch.n
        if key is None or m > key:
            best, key = rid, m
    return best


class DeviceEngine:
    """Batched e-graph operations of the search on the device (one LeafPipeline per batch)."""

    def __init__(self, rules, symtab, language, cost_config, ctx=None, method: str = "ocf", headroom: int = 4096):
        self.ctx = ctx or native.Context(0)
        self.rules, self.symtab, self.language, self.cfg = rules, symtab, language, cost_config
        self.method, self.headroom = method, headroom

    def _open(self, states):
        packed = Batch(states).pack_with_headroom(nodes=self.headroom)
        self.symtab.finalize()
        pipe = LeafPipeline(self.ctx, self.symtab.arrays(), self.rules,
                            lambda nm: self.symtab.name_id(nm, create=False), self.symtab.code, method=self.method,
                            pool_entries_per_node=32)
        b = pipe.load(packed)
        b.set_counts(packed["n_cnt"], packed["u_cnt"])
        drv = ApplyDriver(pipe, self.symtab, self.language, self.cfg)
        return packed, pipe, b, drv

    def _extract(self, pipe, b):
        out = native.extract_with_retry(b, self.method, factor=32)
        cost = out["root_cost"].copy()
        cost[out["status"] != 0] = np.inf
        return cost

    def _clean_states(self, packed, b):
        reb = b.download_rebuild()
        U = b.download_state()["U"]
        out = []
        for l in range(packed["n_leaves"]):
            n0, k0, u0 = (int(packed[k][l]) for k in ("node_base", "kid_base", "id_base"))
            n = int(reb["n"][l])
            koff = reb["hc_koff"][n0 + l:n0 + l + n + 1].copy()
            out.append(LeafState(reb["hc_sym"][n0:n0 + n].copy(), koff, reb["hc_kids"][k0:k0 + int(koff[-1])].copy(),
                                 reb["hc_cid"][n0:n0 + n].copy(), reb["hc_cost"][n0:n0 + n].copy(),
                                 reb["uf_parent"][u0:u0 + int(U[l])].copy(), reb["uf_rank"][u0:u0 + int(U[l])].copy(),
                                 int(packed["root"][l])))
        return out, reb["n"].copy()

    def _applicable(self, pipe, b):
        """[L, R] is_rule_applicable: every source of the rule has a match (rewrite.py:579-589)."""
        pipe.ematch()
        cnt = {}
        for r in pipe.rules:
            for pid in r.pattern_ids:
                if pid not in cnt:
                    cnt[pid] = b.download_matches(pid)[2]
        return np.stack([np.all([cnt[p] > 0 for p in r.pattern_ids], axis=0) for r in pipe.rules], axis=1)

    def evaluate(self, states):
        """Rebuild + extract + applicability of raw states: (clean states, costs, sizes, applicable)."""
        packed, pipe, b, drv = self._open(states)
        pipe.rebuild()
        cost = self._extract(pipe, b)
        clean, n = self._clean_states(packed, b)
        app = self._applicable(pipe, b)
        b.close()
        return clean, cost, n, app

    def expand(self, states, rules):
        """Apply rules[l] to states[l]: (child clean states, changed, costs, sizes, applicable)."""
        packed, pipe, b, drv = self._open(states)
        pipe.rebuild()
        pipe.ematch()
        res = drv.apply(np.asarray(rules, np.uint32))
        ok = res["status"] == native.A_OK
        changed = (res["report"][:, 1] > 0) & ok
        pipe.rebuild()
        cost = self._extract(pipe, b)
        clean, n = self._clean_states(packed, b)
        app = self._applicable(pipe, b)
        b.close()
        return clean, changed, cost, n, app

    def simulate(self, states, costs0, allowed, steps: int, node_limit: int, rng: random.Random):
        """Random rollouts: per step every live leaf applies a uniformly drawn
        allowed rule, rebuilds and extracts; r += max(prev - cost, 0); a failed extraction adds 0."""
        L = len(states)
        packed, pipe, b, drv = self._open(states)
        reward = np.zeros(L)
        prev = np.asarray(costs0, np.float64).copy()
        live = np.ones(L, bool)
        pipe.rebuild()
        for _ in range(steps):
            rules = np.full(L, NONE, np.uint32)
            for l in range(L):
                if live[l] and allowed[l]:
                    rules[l] = rng.choice(allowed[l])
                else:
                    live[l] = False
            if not live.any():
                break
            pipe.ematch()
            res = drv.apply(rules)
            live &= res["status"] == native.A_OK
            pipe.rebuild()
            cost = self._extract(pipe, b)
            good = live & np.isfinite(cost)
            reward[good] += np.maximum(prev[good] - cost[good], 0.0)
            prev[good] = cost[good]
            n = b.download_rebuild()["n"]
            live &= n < node_limit
        b.close()
        return reward


def run_search(root: SearchNode, engine: DeviceEngine, n_rules: int, cfg: MctsConfig, rng: random.Random):
    """N select/expand/simulate/update iterations (Alg. 1 body), batched."""
    done = 0
    while done < cfg.budget:
        picks = []
        while len(picks) < min(cfg.batch, cfg.budget - done) and not root.s:
            node = root
            while True:   # selection
                free = [r for r in range(n_rules)
                        if r not in node.b and r not in node.children and r not in node.pending]
                kids = [ch for _, ch in sorted(node.children.items()) if not ch.s and ch.n > 0]
                stop = rng.random() < cfg.stop_prob
                if free and (stop or not kids):
                    break                      # expand here (progressive widening)
                if not kids:
                    if not node.pending:
                        node.s = True          # nothing left to expand below: saturated
                    node = None
                    break
                N = max(node.n, 1)
                node = max(kids, key=lambda ch: ucb1(ch.v, ch.n, N, cfg.c))
            if node is None:
                done += 1                      # a saturated-expansion iteration (reward 0)
                continue
            rule = rng.choice(free)
            node.pending.add(rule)
            picks.append((node, rule))
        if not picks:
            break
        kids, changed, cost, n, app = engine.expand([p.state for p, _ in picks], [r for _, r in picks])
        sims, anchors, allowed = [], [], []
        for j, (node, rule) in enumerate(picks):
            node.pending.discard(rule)
            ch = SearchNode(kids[j], float(cost[j]), int(n[j]), parent=node, rule=rule)
            node.children[rule] = ch
            if not changed[j]:
                ch.s = True   # the rule cannot change this e-graph: blacklist it here
                node.b.add(rule)
                continue
            ch.b = {r for r in range(n_rules) if not app[j, r]}
            sims.append(j)
            anchors.append(float(cost[j]))
            allowed.append([r for r in range(n_rules) if r not in ch.b])
        rewards = np.zeros(len(picks))
        if sims:
            live_n = [int(n[j]) for j in sims]
            r = engine.simulate([kids[j] for j in sims], anchors,
                                [a if ln < cfg.node_limit else [] for a, ln in zip(allowed, live_n)],
                                cfg.max_sim_steps, cfg.node_limit, rng)
            rewards[sims] = r
        for j, (node, rule) in enumerate(picks):   # updates in selection order
            update(node.children[rule], float(rewards[j]))
            done += 1
    return best_child(root)


def optimize_mcts(egraph, rules, cfg: MctsConfig, cost_config, symtab=None, engine=None):
    """Alg. 1: search, apply the best rule to the root, repeat until saturation or
    the node limit; returns (initial cost, final cost, applied rule ids)."""
    from .arena import export_state
    from .symtab import SymbolTable

    symtab = SymbolTable() if symtab is None else symtab
    language = egraph.language
    state = export_state(egraph, symtab, cost_config)
    engine = engine if engine is not None else DeviceEngine(rules, symtab, language, cost_config, method=cfg.main_extractor,
                                    headroom=cfg.headroom)
    rng = random.Random(cfg.seed)
    (state,), cost, n, app = engine.evaluate([state])
    initial = float(cost[0])
    trace = []
    while int(n[0]) < cfg.node_limit:
        root = SearchNode(state, float(cost[0]), int(n[0]))
        root.b = {r for r in range(len(rules)) if not app[0, r]}
        best = run_search(root, engine, len(rules), cfg, rng)
        if best is None:
            break
        trace.append(best)
        (state,), changed, cost, n, app = engine.expand([state], [best])
        if not changed[0]:
            break
    return initial, float(cost[0]), trace
