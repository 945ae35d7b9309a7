"""Batched MCTS over rewrite-rule applications (§4.1).

The search tree lives on the host; every e-graph operation of an iteration batch is delegated to
an *engine* with four calls (``initial`` / ``evaluate`` / ``expand`` / ``simulate``, plus ``final``
for the run's last extraction). ``DeviceEngine`` runs them on the B200: expansion applies the
sampled rule to a snapshot of the selected node (k_apply, then k_rebuild), blacklists come from
per-source e-matching of the child (is_rule_applicable, rewrite.py:579-589: a rule is
inapplicable as soon as one source has no match), and the simulations are device-resident random
rollouts -- apply, rebuild, extract after every step, reward Eq. 3 ``r = sum max(cost_{i-1} -
cost_i, 0)`` anchored at the child's own extracted cost. The test-only CPU engine
(oracle/mcts_ref.py) runs the same four calls on the reference's own EGraph / apply_rule /
extractors, so ``optimize_mcts`` with either engine must produce the identical RunReport.

SPEC's concurrency model allows simulations of distinct iterations to run in parallel on
snapshots with the results applied to the tree serially: ``batch`` selections are
made sequentially (a node/rule pair is reserved so one batch never expands it twice), the batch's
expansions and simulations run as one engine batch, and the updates are applied in selection
order. ``batch=1`` is the strictly sequential search.

Engine contract (what both engines implement, state objects are engine-private):

    initial(egraph)                     -> state
    evaluate(states)                    -> (clean states, cost f64[L], nodes[L], classes[L], app bool[L,R])
    expand(states, rules)               -> (child states, changed[L], cost, nodes, classes, app)
    simulate(states, cost0, allowed, steps, node_limit, seeds) -> reward f64[L]
    final(state, method)                -> (cost, save_graph JSON text)
    configure(cfg)                      -> None (start of a run: extractor, extraction cache reset)

A failed extraction yields cost ``inf``. In a rollout a step whose extraction failed adds no reward
and leaves the anchor unchanged ("treat that step's improvement as 0"); a step right
after a failed anchor only re-anchors.

Randomness (one seeded stream): selection and expansion draw from the search's
``random.Random(seed)``; each rollout draws its rules from its own ``random.Random(s)`` with ``s``
taken from the search stream (64 bits per simulated leaf, in selection order) -- a rollout's draws
do not depend on its batch-mates, so the leaves of a batch can be simulated on different GPUs
(parallel.ShardedEngine) with results identical to one GPU.
"""

from __future__ import annotations

import math
import random
import time
from collections import Counter
from dataclasses import dataclass, field

import numpy as np

from . import native
from .apply import ApplyDriver
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
    final_extractor: str = "ocf"
    batch: int = 32
    headroom: int = 4096
    # SPEC.md:655 / PAPER §4.3: rollouts reuse extracted costs by e-graph fingerprint (egraph.py:247)
    # for the whole optimization run. Off by default on the device: the WL fingerprint costs more
    # than the extraction it would save there (bench.py `fingerprint` vs `kernel_ms.extract`).
    extraction_cache: bool = False


@dataclass
class SearchNode:
    state: object
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
    exhausted: bool = False   # no rule left to expand anywhere below (selection prunes it)


@dataclass
class RunReport:
    """SPEC.md:685-697 RunReport: costs, speedup, per-iteration rows (rule id, e-nodes, e-classes,
    main-extractor cost) and the rule histogram; ``final_program`` is the optimized program as the
    exact text ``save_graph`` writes (tensor_ir.py:487-504)."""

    original_cost: float
    optimized_cost: float
    speedup_pct: float
    wall_time_s: float
    iterations: list
    rule_histogram: dict
    final_program: str | None
    final_extractor: str = "ocf"
    extraction_cache: dict | None = None   # {"lookups", "hits"} of the run-wide rollout cache

    @property
    def trace(self) -> list:
        return [it[0] for it in self.iterations]

    def to_json_dict(self) -> dict:
        hexf = lambda x: float(x).hex()  # noqa: E731
        return {"original_cost": hexf(self.original_cost), "optimized_cost": hexf(self.optimized_cost),
                "speedup_pct": hexf(self.speedup_pct), "final_extractor": self.final_extractor,
                "iterations": [[r, n, c, hexf(x)] for r, n, c, x in self.iterations],
                "rule_histogram": {str(k): v for k, v in sorted(self.rule_histogram.items())},
                "final_program": self.final_program,
                **({"extraction_cache": self.extraction_cache} if self.extraction_cache is not None else {})}


def speedup_pct(orig: float, opt: float) -> float:
    """(orig - opt) / orig * 100."""
    return (orig - opt) / orig * 100.0 if orig else 0.0


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


def rollout_rewards(reward, prev, live, cost) -> None:
    """One rollout step's Eq. 3 update, in place (shared by every engine): a finite extraction
    adds max(prev - cost, 0) when the anchor is finite and becomes the anchor; a failed one adds
    nothing and keeps the anchor."""
    good = live & np.isfinite(cost)
    add = good & np.isfinite(prev)
    reward[add] += np.maximum(prev[add] - cost[add], 0.0)
    prev[good] = cost[good]


class ExtractionCache:
    """Run-wide rollout extraction cache keyed by the e-graph fingerprint. Leaves
    are consulted in leaf order within a step, so a fingerprint first seen in this step is a hit for
    a later leaf of the same step -- the same rule in every engine."""

    def __init__(self):
        self.table, self.lookups, self.hits = {}, 0, 0

    def resolve(self, fps, live, extracted):
        """Per live leaf: the cached cost of its fingerprint, else its own extraction (then cached)."""
        cost = np.full(len(fps), np.inf)
        for l in range(len(fps)):
            if not live[l]:
                continue
            self.lookups += 1
            fp = int(fps[l])
            if fp in self.table:
                self.hits += 1
                cost[l] = self.table[fp]
            else:
                cost[l] = self.table[fp] = float(extracted[l])
        return cost


GROWTH_CAP = 1 << 22   # largest per-leaf growth bound an apply is pre-sized for (e-nodes)


class DeviceEngine:
    """Batched e-graph operations of the search on the device: one LeafPipeline for the whole
    search, and every search state (tree node e-graph, rollout survivor) a slot of a device
    SnapshotStore (EGraph.snapshot, egraph.py:300-312) -- batches are filled from slots and saved
    back to slots device to device; host copies only for ``final`` and ``export_states``."""

    def __init__(self, rules, symtab, language, cost_config, ctx=None, method: str = "ocf", headroom: int = 4096):
        self.ctx = ctx or native.Context(0)
        self.rules, self.symtab, self.language, self.cfg = rules, symtab, language, cost_config
        self.method, self.headroom = method, headroom
        self.regrows = self.presized = 0
        self._pipe = self._drv = None
        self.store = None
        self.cache = None
        self._fp_symbols = -1

    def configure(self, cfg):
        self.method = cfg.main_extractor
        self.cache = ExtractionCache() if cfg.extraction_cache else None

    def _fingerprints(self, b):
        """k_fingerprint of every leaf of the rebuilt batch (egraph.py:247-296, bit-exact)."""
        from .fingerprint import symtab_key_tables

        if self._fp_symbols != len(self.symtab):
            self.ctx.fingerprint_setup(*symtab_key_tables(self.symtab))
            self._fp_symbols = len(self.symtab)
        b.fingerprint()
        fp, st = b.download_fingerprint()
        if np.any(st != 0):
            raise RuntimeError("k_fingerprint failed on a leaf")
        return fp

    # -- batch plumbing ---------------------------------------------------------------
    def _ensure_pipe(self):
        """One pipeline (compiled patterns, rule target programs, symbol tables on the device) for
        the whole search; re-uploaded only when host interning added symbols."""
        self.symtab.finalize()
        if self._pipe is None:
            self.store = native.SnapshotStore(self.ctx)
            self._pipe = LeafPipeline(self.ctx, self.symtab.arrays(), self.rules,
                                      lambda nm: self.symtab.name_id(nm, create=False), self.symtab.code,
                                      method=self.method, pool_entries_per_node=32)
            self._drv = ApplyDriver(self._pipe, self.symtab, self.language, self.cfg)
        elif self._drv.uploaded_symbols != len(self.symtab):
            self._drv.upload()
        return self._pipe, self._drv

    def _open(self, states, headroom=None, kids=None):
        """A batch of ``states`` (slots of this engine's store; host LeafStates are put into slots
        first) with ``headroom`` spare e-nodes per leaf (an int or one per leaf; ``kids`` spare child
        slots, default 2x)."""
        pipe, drv = self._ensure_pipe()
        slots = self.import_states(states)
        head = self.headroom if headroom is None else headroom
        layout, b = pipe.load_slots(self.store, slots, head, kids)
        return [layout, pipe, b, drv, int(np.max(head)) if np.size(head) else self.headroom]

    def import_states(self, states):
        """Host LeafStates as slots of this engine's store (slots of this store pass through)."""
        self._ensure_pipe()
        sid = self.store.id
        return [s if isinstance(s, native.Slot) and s.store == sid else self.store.put(s) for s in states]

    def export_states(self, states):
        """Slots as host LeafStates (for the multi-rank exchange, parallel.ShardedEngine)."""
        return [self.store.download(s) if isinstance(s, native.Slot) else s for s in states]

    def _extract(self, b, method=None):
        out = native.extract_with_retry(b, method or self.method, factor=32, bitsets=2.0, light=True)
        cost = out["root_cost"].copy()
        cost[out["status"] != 0] = np.inf
        return cost, out

    def _clean_states(self, packed, b):
        """Every leaf's last rebuild as a new device slot (a snapshot, egraph.py:300-312; D2D)."""
        return self.store.save(b, range(packed["n_leaves"]))

    def _applicable(self, pipe, b):
        """[L, R] is_rule_applicable (rewrite.py:579-589): one EXISTS-mode e-match of all sources."""
        return pipe.exists()

    def _apply(self, h, rules):
        """esat_apply of rules[l] on every leaf of the rebuilt batch ``h``. A leaf that runs out of
        arena headroom (ESAT_A_CAPACITY) leaves the rebuilt state intact on the device (k_apply
        reads the rebuild's outputs and writes the batch input), so the whole batch is re-packed
        from those rebuilt states with 4x the headroom and the same rules are re-applied: the
        result is the one an unbounded arena gives."""
        rules = np.asarray(rules, np.uint32)
        sized = False
        while True:
            packed, pipe, b, drv, head = h
            mask = pipe.rule_masks(rules)   # each leaf matches only the sources of its own rule
            pipe.ematch(mask)
            if not sized:
                # a leaf whose matches could outgrow its spans (a multi-pattern explosion: tens of
                # thousands of matches) is re-opened once with spans for the bound, so the apply
                # runs once instead of failing at capacity on a ladder of growing arenas
                sized = True
                need_n, need_k = pipe.growth_bound(rules)
                nb, kb, ub = (np.diff(packed[k].astype(np.int64)) for k in ("node_base", "kid_base", "id_base"))
                spare_n = nb - packed["n_cnt"].astype(np.int64)
                spare_k = kb - packed["k_cnt"].astype(np.int64)
                spare_u = ub - packed["u_cnt"].astype(np.int64)
                grow = (need_n > spare_n) | (need_k > spare_k) | (need_n > spare_u)
                if np.any(grow) and int(need_n.max()) <= GROWTH_CAP:
                    clean = self._clean_states(packed, b)
                    b.close()
                    mark = len(self.store) - len(clean)
                    nodes = np.where(grow, np.maximum(need_n, head), head)
                    kids = np.where(grow, np.maximum(need_k, 2 * nodes), 2 * nodes)
                    h[:] = self._open(clean, nodes, kids)
                    self.store.truncate(mark)
                    self.presized += 1
                    h[1].rebuild()
                    continue
            res = drv.apply(rules, leaf_mask=mask)
            st = res["status"]
            if np.any(st == native.A_PROGRAM):
                raise RuntimeError("k_apply: rule target program beyond device limits (ESAT_A_PROGRAM)")
            if np.any((st != native.A_OK) & (st != native.A_CAPACITY)):
                raise RuntimeError(f"k_apply: unexpected statuses {np.unique(st)}")
            if not np.any(st == native.A_CAPACITY):
                return res
            mark = len(self.store)
            clean = self._clean_states(packed, b)   # the rebuild k_apply read is left intact
            b.close()
            self.regrows += 1
            h[:] = self._open(clean, head * 4)
            self.store.truncate(mark)               # the batch holds them now
            h[1].rebuild()

    # -- engine contract ----------------------------------------------------------------
    def initial(self, egraph):
        from .arena import export_state

        return export_state(egraph, self.symtab, self.cfg)

    def evaluate(self, states):
        """Rebuild + extract + applicability of raw states."""
        h = self._open(states)
        packed, pipe, b = h[0], h[1], h[2]
        pipe.rebuild()
        cost, _ = self._extract(b)
        n, c = b.rebuilt_sizes()
        clean = self._clean_states(packed, b)
        app = self._applicable(pipe, b)
        b.close()
        return clean, cost, n, c, app

    def expand(self, states, rules):
        """Apply rules[l] to states[l]: (child clean states, changed, costs, sizes, classes, applicable)."""
        h = self._open(states)
        h[1].rebuild()
        res = self._apply(h, rules)
        changed = res["report"][:, 1] > 0
        packed, pipe, b = h[0], h[1], h[2]
        pipe.rebuild()
        cost, _ = self._extract(b)
        n, c = b.rebuilt_sizes()
        clean = self._clean_states(packed, b)
        app = self._applicable(pipe, b)
        b.close()
        return clean, changed, cost, n, c, app

    def simulate(self, states, costs0, allowed, steps: int, node_limit: int, seeds):
        """Random rollouts: per step every live leaf applies a uniformly drawn
        allowed rule, rebuilds and extracts (rollout_rewards); a leaf stops at the node limit. The
        device batch holds the live leaves only: when leaves stop, the batch is re-packed from the
        survivors' rebuilt states (a stopped leaf -- typically one a multi-pattern rule exploded --
        is never matched, rebuilt or extracted again)."""
        L = len(states)
        rngs = [random.Random(sd) for sd in seeds]
        reward = np.zeros(L)
        prev = np.asarray(costs0, np.float64).copy()
        live = np.array([bool(a) for a in allowed], bool)
        idx = np.nonzero(live)[0]            # batch position -> leaf
        if idx.size == 0:
            return reward
        h = self._open([states[l] for l in idx])
        h[1].rebuild()
        for _ in range(steps):
            rules = np.full(L, NONE, np.uint32)
            for l in range(L):
                if live[l] and allowed[l]:
                    rules[l] = rngs[l].choice(allowed[l])
                else:
                    live[l] = False
            if not live.any():
                break
            if not live[idx].all():          # compact: drop the leaves that stopped
                keep = np.nonzero(live[idx])[0]
                mark = len(self.store)
                clean = self.store.save(h[2], keep)
                h[2].close()
                idx = idx[keep]
                h = self._open(clean)
                self.store.truncate(mark)
                h[1].rebuild()
            self._apply(h, rules[idx])
            h[1].rebuild()
            cb, _ = self._extract(h[2])
            cost = np.full(L, np.inf)
            cost[idx] = cb
            if self.cache is not None:
                fps = np.zeros(L, np.uint64)
                fps[idx] = self._fingerprints(h[2])
                cost = self.cache.resolve(fps, live, cost)
            rollout_rewards(reward, prev, live, cost)
            n, _ = h[2].rebuilt_sizes()
            live[idx] &= n < node_limit
        h[2].close()
        return reward

    def final(self, state, method: str):
        """Final extraction of one state with ``method`` and the program it selects, as
        save_graph text (extraction_to_graph, tensor_ir.py:316-352). Exact extraction runs the
        host branch-and-bound seeded by the device OCF result (exact.py)."""
        from .arena import to_egraph
        from .extraction import ExtractionResult
        from .tensor_ir import GraphFormatError, extraction_to_graph, graph_json

        h = self._open([state], headroom=1)
        packed, pipe, b = h[0], h[1], h[2]
        pipe.rebuild()
        out = native.extract_with_retry(b, "ocf" if method == "exact" else method, factor=32, bitsets=2.0)
        cost = out["root_cost"].copy()
        cost[out["status"] != 0] = np.inf
        mark = len(self.store)
        clean = self.store.download(self._clean_states(packed, b)[0])
        self.store.truncate(mark)
        eg = to_egraph(clean, self.symtab, self.language)
        if not np.isfinite(cost[0]):
            b.close()
            return float("inf"), None
        chosen = _chosen_of(b, out, self.symtab)
        b.close()
        res = ExtractionResult(float(cost[0]), chosen, method)
        if method == "exact":
            from .cost_model import egraph_costs
            from .exact import extract_exact

            res = extract_exact(eg, egraph_costs(eg, self.cfg), seed=res)
        if type(self.language).__name__ != "TensorLanguage":
            return res.total_cost, None
        try:
            return res.total_cost, graph_json(extraction_to_graph(eg, res))
        except GraphFormatError:
            return res.total_cost, None


def _chosen_of(b, out, symtab) -> dict:
    """{class id: ENode} of leaf 0's reachable chosen nodes (extraction.py:106-115)."""
    from .egraph import ENode

    v = b.download_view()
    C = int(v["C"][0])
    cls_id = v["cls_id"][:C]
    nko = v["nd_koff"]
    chosen = {}
    for k in np.nonzero(out["reachable"][:C])[0]:
        j = int(out["choice"][k])
        kids = tuple(int(cls_id[p]) for p in v["nd_kpos"][nko[j]:nko[j + 1]])
        chosen[int(cls_id[k])] = ENode(symtab.symbols[int(v["nd_sym"][j])], kids)
    return chosen


def run_search(root: SearchNode, engine, n_rules: int, cfg: MctsConfig, rng: random.Random):
    """N select/expand/simulate/update iterations (Alg. 1 body), batched."""
    done = 0
    while done < cfg.budget:
        picks = []
        while len(picks) < min(cfg.batch, cfg.budget - done) and not root.exhausted:
            node = root
            while True:   # selection
                free = [r for r in range(n_rules)
                        if r not in node.b and r not in node.children and r not in node.pending]
                kids = [ch for _, ch in sorted(node.children.items()) if not ch.s and not ch.exhausted and ch.n > 0]
                stop = rng.random() < cfg.stop_prob
                if free and (stop or not kids):
                    break                      # expand here (progressive widening)
                if not kids:
                    if not node.pending:
                        node.exhausted = True  # nothing left to expand below (not 'saturated': the
                    node = None                # node still changed its parent's e-graph)
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
        kids, changed, cost, n, _, app = engine.expand([p.state for p, _ in picks], [r for _, r in picks])
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
            seeds = [rng.getrandbits(64) for _ in sims]   # one rollout stream per simulated leaf
            r = engine.simulate([kids[j] for j in sims], anchors,
                                [a if ln < cfg.node_limit else [] for a, ln in zip(allowed, live_n)],
                                cfg.max_sim_steps, cfg.node_limit, seeds)
            rewards[sims] = r
        for j, (node, rule) in enumerate(picks):   # updates in selection order
            update(node.children[rule], float(rewards[j]))
            done += 1
    return best_child(root)


def optimize_mcts(egraph, rules, cfg: MctsConfig, cost_config, symtab=None, engine=None) -> RunReport:
    """Alg. 1: search, apply the best rule to the root, repeat until saturation or
    the node limit (checked before each search and after each application); final extraction with
    ``cfg.final_extractor``. The RNG is one stream seeded by ``cfg.seed``."""
    from .symtab import SymbolTable

    t0 = time.monotonic()
    if engine is None:
        symtab = SymbolTable() if symtab is None else symtab
        engine = DeviceEngine(rules, symtab, egraph.language, cost_config, method=cfg.main_extractor,
                              headroom=cfg.headroom)
    rng = random.Random(cfg.seed)
    if hasattr(engine, "configure"):
        engine.configure(cfg)
    (state,), cost, n, c, app = engine.evaluate([engine.initial(egraph)])
    first = state
    iterations = []
    while int(n[0]) < cfg.node_limit:
        root = SearchNode(state, float(cost[0]), int(n[0]))
        root.b = {r for r in range(len(rules)) if not app[0, r]}
        best = run_search(root, engine, len(rules), cfg, rng)
        if best is None:
            break
        (state,), changed, cost, n, c, app = engine.expand([state], [best])
        iterations.append((int(best), int(n[0]), int(c[0]), float(cost[0])))
        if not changed[0]:
            break
    orig, _ = engine.final(first, cfg.final_extractor)
    opt, program = engine.final(state, cfg.final_extractor)
    cache = getattr(engine, "cache", None) or getattr(getattr(engine, "engine", None), "cache", None)
    stats = {"lookups": cache.lookups, "hits": cache.hits} if cache is not None else None
    return RunReport(orig, opt, speedup_pct(orig, opt), time.monotonic() - t0, iterations,
                     dict(Counter(it[0] for it in iterations)), program, cfg.final_extractor, stats)
