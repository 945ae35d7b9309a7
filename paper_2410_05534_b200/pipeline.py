"""The batched MCTS-leaf pipeline on one B200: rebuild -> all-rule e-match -> join -> extract.

One MCTS simulation step hands every leaf e-graph of a batch through
the reference's hot path:

    EGraph.rebuild()                      egraph.py:203      (the end of apply_rule, rewrite.py:569)
    joint_match(rule.sources) for every rule                  rewrite.py:405  (applicability / next step)
    extract_ocf_greedy / extract_default_greedy               extraction.py:229 / 157

``LeafPipeline`` compiles the rule set against a symbol table, keeps one device batch
resident and runs the four launches (k_rebuild, k_ematch, k_join, k_extract) per step.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import native
from .patterns import compile_pattern


@dataclass
class CompiledRule:
    rule: object
    pattern_ids: list      # positions in the e-match call
    var_names: list        # combined, sorted
    pvar_names: list
    var_maps: list         # per source: output slot of each source var
    pvar_maps: list

    @property
    def multi(self) -> bool:
        return len(self.pattern_ids) > 1


def compile_rules(rules, name_id, code):
    programs, out = [], []
    for r in rules:
        comps = [compile_pattern(p, name_id, code) for p in r.sources]
        vn = sorted({v for c in comps for v in c.var_names})
        qn = sorted({q for c in comps for q in c.pvar_names})
        ids = []
        for c in comps:
            ids.append(len(programs))
            programs.append(c.program)
        cr = CompiledRule(r, ids, vn, qn, [[vn.index(v) for v in c.var_names] for c in comps],
                          [[qn.index(q) for q in c.pvar_names] for c in comps])
        cr._programs = [c.program for c in comps]
        out.append(cr)
    return programs, out


class LeafPipeline:
    def __init__(self, ctx: native.Context, symtab_arrays: dict, rules, name_id, code,
                 method: str = "ocf", pool_entries_per_node: float = 8.0, pool_bitsets_per_node: float = 2.0):
        self.ctx = ctx
        self.method = method
        self.pool = pool_entries_per_node
        self.pool_bitsets = pool_bitsets_per_node
        ctx.upload_symtab(symtab_arrays)
        self.programs, self.rules = compile_rules(rules, name_id, code)
        ctx.upload_patterns(self.programs)
        self.pattern_ids = list(range(len(self.programs)))
        self.joins = [r for r in self.rules if r.multi]
        self.batch = None

    def recompile(self, name_id, code):
        """Recompile and re-upload the source patterns (after the symbol table changed)."""
        rules = [r.rule for r in self.rules]
        self.programs, self.rules = compile_rules(rules, name_id, code)
        self.ctx.upload_patterns(self.programs)
        self.joins = [r for r in self.rules if r.multi]

    def load(self, packed: dict):
        if self.batch is not None:
            self.batch.close()
        self.batch = native.DeviceBatch(self.ctx, packed)
        self.batch.set_pool(self.pool, self.pool_bitsets)
        self.batch.upload(packed)
        return self.batch

    def load_slots(self, store, slots, nodes, kids=None):
        """A batch of device snapshot slots with ``nodes`` spare e-nodes per leaf (D2D, no host
        arena): native.SnapshotStore.layout + esat_batch_load_slots."""
        if self.batch is not None:
            self.batch.close()
        layout = store.layout(slots, nodes, kids)
        self.batch = native.DeviceBatch(self.ctx, layout)
        self.batch.set_pool(self.pool, self.pool_bitsets)
        store.load(self.batch, slots)
        return layout, self.batch

    def grow_pool(self, ext: dict) -> bool:
        """After an extraction that overflowed (ESAT_X_CAPACITY), grow the pool(s) named by the
        overflow mask in err_class. Returns False when nothing overflowed."""
        over = ext["status"] == native.X_CAPACITY
        if not np.any(over):
            return False
        mask = int(np.bitwise_or.reduce(ext["err_class"][over]))
        if mask & 1 or not mask & 3:
            self.pool_bitsets *= 2
        if mask & 2 or not mask & 3:
            self.pool *= 2
        self.batch.set_pool(self.pool, self.pool_bitsets)
        return True

    # the four stages -------------------------------------------------------------
    def rebuild(self):
        self.batch.rebuild()

    def match(self, leaf_mask=None):
        """k_ematch: every source pattern of every rule (LIST mode); ``leaf_mask[l]`` (bit p =
        pattern p) restricts leaf l to the patterns it needs."""
        self.batch.ematch(self.pattern_ids, leaf_mask=leaf_mask)

    def rule_masks(self, leaf_rule) -> np.ndarray:
        """Per-leaf pattern masks for applying rule ``leaf_rule[l]`` (0xFFFFFFFF: none): the bits of
        that rule's source patterns, one 32-pattern chunk per row ([ceil(P/32), L], esat_ematch_masked)."""
        nch = max(1, (len(self.pattern_ids) + 31) // 32)
        bits = np.zeros((len(self.rules) + 1, nch), np.uint32)   # last row: no rule
        for i, r in enumerate(self.rules):
            for p in r.pattern_ids:
                bits[i, p // 32] |= np.uint32(1 << (p % 32))
        sel = np.array([len(self.rules) if int(r) == 0xFFFFFFFF else int(r) for r in leaf_rule], np.int64)
        return np.ascontiguousarray(bits[sel].T)

    def exists(self) -> np.ndarray:
        """is_rule_applicable of every rule on every leaf (rewrite.py:579-589): one EXISTS-mode
        k_ematch over all source patterns; a rule applies iff each of its sources matches. [L, R]"""
        self.batch.ematch(self.pattern_ids, mode=native.MATCH_EXISTS)
        cnt = self.batch.download_counts(len(self.pattern_ids))
        return np.stack([np.all(cnt[r.pattern_ids] > 0, axis=0) for r in self.rules], axis=1)

    def join(self):
        """k_join: multi-pattern rules over the source match lists."""
        if self.joins:
            self.batch.join([(r.pattern_ids, r.var_maps, r.pvar_maps, len(r.var_names), len(r.pvar_names))
                             for r in self.joins])

    def ematch(self, leaf_mask=None):
        self.match(leaf_mask)
        self.join()

    def extract(self):
        self.batch.extract(self.method)

    def extract_async(self):
        self.batch.extract_async(self.method)

    def step(self):
        """rebuild, then OCF extraction on the side stream concurrently with e-match + join."""
        self.rebuild()
        self.ctx.fork()
        self.ematch()
        self.extract_async()
        self.ctx.wait_async()

    LAUNCHES_PER_STEP = 4  # k_rebuild, k_ematch, k_join, k_extract

    def apply_programs(self, name_id, code) -> tuple:
        """Target programs of every rule for esat_apply, wired to this pipeline's match lists
        (single-source rules: the e-match list of their pattern; multi-pattern: their join)."""
        from .apply import compile_rule_targets, pack_rules

        progs = []
        for r in self.rules:
            if r.multi:
                progs.append(compile_rule_targets(r.rule, name_id, code, None, 1, self.joins.index(r)))
            else:
                progs.append(compile_rule_targets(r.rule, name_id, code, None, 0, r.pattern_ids[0]))
        return pack_rules(progs)

    def leaf_rule_counts(self, leaf_rule) -> np.ndarray:
        """Matches of leaf l's own rule ``leaf_rule[l]`` in the last e-match + join (0 for none): [L]."""
        P = self.batch.download_counts(len(self.pattern_ids))
        J = self.batch.download_counts(len(self.joins), from_join=True) if self.joins else None
        out = np.zeros(len(leaf_rule), np.int64)
        for l, r in enumerate(leaf_rule):
            if int(r) == 0xFFFFFFFF:
                continue
            cr = self.rules[int(r)]
            out[l] = J[self.joins.index(cr), l] if cr.multi else P[cr.pattern_ids[0], l]
        return out

    def growth_bound(self, leaf_rule) -> tuple:
        """Upper bounds of the e-nodes and child slots applying ``leaf_rule[l]`` can add to leaf l:
        its matches x the operator nodes (and their children) of the rule's targets -- an
        instantiation adds at most one e-node per target operator (rewrite.py:517-523). [L] x 2"""
        def apps(p):
            if not hasattr(p, "children"):
                return 0, 0
            n, k = 1, len(p.children)
            for ch in p.children:
                a, b = apps(ch)
                n, k = n + a, k + b
            return n, k

        per = [tuple(map(sum, zip(*[apps(t) for t in r.rule.targets]))) if r.rule.targets else (0, 0)
               for r in self.rules]
        cnt = self.leaf_rule_counts(leaf_rule)
        nodes = np.array([0 if int(r) == 0xFFFFFFFF else per[int(r)][0] for r in leaf_rule], np.int64) * cnt
        kids = np.array([0 if int(r) == 0xFFFFFFFF else per[int(r)][1] for r in leaf_rule], np.int64) * cnt
        return nodes, kids

    def match_counts(self) -> np.ndarray:
        """Unique matches per rule per leaf of the last step: [rules, leaves]."""
        rows = []
        for j, r in enumerate(self.rules):
            if r.multi:
                _, _, cnt = self.batch.download_matches(self.joins.index(r), from_join=True)
            else:
                _, _, cnt = self.batch.download_matches(r.pattern_ids[0])
            rows.append(cnt)
        return np.stack(rows) if rows else np.zeros((0, self.batch.n_leaves), np.uint32)
