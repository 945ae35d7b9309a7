"""Device execution of the hot path for host e-graph objects (the drop-in layer).

Each function takes an e-graph with the reference's structure -- ours
(`paper_2410_05534_b200.egraph.EGraph`) or the reference's own `esat.egraph.EGraph`, the
layer only touches `hashcons`, `_uf`, `classes`, `root`, `dirty`, `language`, `_version` --
exports it to the SoA arena (arena.py), runs the CUDA kernel through the C-ABI and writes
the result back in the reference's representation:

    rebuild(eg)                 egraph.py:203-238   -> k_rebuild
    joint_match(eg, patterns)   rewrite.py:405-433  -> k_ematch (+ k_join)
    any_match(eg, pattern)      rewrite.py:579-589  -> k_ematch EXISTS
    extract(eg, costs, method)  extraction.py:121-242 -> k_extract

A rebuilt e-graph's device view is cached per object and version, so matching and
extraction right after a rebuild reuse the resident arena.
"""

from __future__ import annotations

import os
from collections import defaultdict

import numpy as np

from . import native
from .arena import NONE, Batch, export_state
from .patterns import compile_pattern
from .symtab import SymbolTable


class Session:
    """Process-wide device context + symbol table (one per GPU per process)."""

    def __init__(self, device: int | None = None):
        self.ctx = native.Context(int(os.environ.get("ESAT_DEVICE", "0")) if device is None else device)
        self.symtab = SymbolTable()
        self._uploaded = -1

    def sync_symtab(self):
        self.symtab.finalize()
        if self._uploaded != self.symtab._version:
            self.ctx.upload_symtab(self.symtab.arrays())
            self._uploaded = self.symtab._version


_SESSION: Session | None = None


def session() -> Session:
    global _SESSION
    if _SESSION is None:
        _SESSION = Session()
    return _SESSION


class _Resident:
    __slots__ = ("version", "batch", "view", "packed")

    def __init__(self, version, batch, view, packed):
        self.version, self.batch, self.view, self.packed = version, batch, view, packed


def _node_class(eg):
    for node in eg.hashcons:
        return type(node), type(node.symbol)
    from .egraph import ENode, Symbol

    return ENode, Symbol


def _upload(eg, costs=None):
    s = session()
    leaf = export_state(eg, s.symtab, costs=costs)
    if costs is not None:
        missing = [n for n in eg.hashcons if eg.canonicalize(n) not in costs]
        if missing:
            raise KeyError(missing[0])
    s.sync_symtab()
    packed = Batch([leaf]).pack()
    b = native.DeviceBatch(s.ctx, packed)
    b.upload(packed)
    b.rebuild()
    return b, packed


def rebuild(eg) -> int:
    """EGraph.rebuild on the device; the host structure is replaced by the device result."""
    b, packed = _upload(eg)
    return _write_back(eg, b, packed)


def _write_back(eg, b, packed, version_bump: int = 0) -> int:
    """Replace the host structure by batch b's rebuilt leaf 0 (hashcons in the reference's
    order, union-find, classes in ascending id); returns the rebuild's merge count."""
    out = b.download_rebuild()
    view = b.download_view()
    merges = int(out["merges"][0])
    n = int(out["n"][0])
    st = session().symtab
    ENodeT, _ = _node_class(eg)
    sym = out["hc_sym"][:n]
    koff = out["hc_koff"][: n + 1]
    kids = out["hc_kids"]
    cid = out["hc_cid"][:n]
    nodes = [ENodeT(st.symbols[int(sym[i])], tuple(int(k) for k in kids[koff[i]:koff[i + 1]])) for i in range(n)]
    eg.hashcons = {nodes[i]: int(cid[i]) for i in range(n)}
    U = int(b.download_state()["U"][0]) if "u_cnt" in packed else len(out["uf_parent"])
    eg._uf.parent = [int(x) for x in out["uf_parent"][:U]]
    eg._uf.rank = [int(x) for x in out["uf_rank"][:U]]
    groups = defaultdict(set)
    parents = defaultdict(set)
    for node, c in eg.hashcons.items():
        groups[c].add(node)
        for ch in set(node.children):
            parents[ch].add((node, c))   # keys are canonical after the final pass
    EClassT = type(next(iter(eg.classes.values()))) if eg.classes else None
    if EClassT is None:
        from .egraph import EClass as EClassT  # noqa: N806
    order = [int(c) for c in view["cls_id"][: int(view["C"][0])]]
    eg.classes = {c: EClassT(c, groups[c], parents.get(c, set())) for c in order}
    eg.dirty.clear()
    eg._version += merges + version_bump
    eg._esat_resident = _Resident(eg._version, b, view, packed)
    return merges


def _resident(eg, costs=None):
    if eg.dirty:
        return None
    r = getattr(eg, "_esat_resident", None)
    # the resident view is reused only for cost-free calls (matching); every extraction re-exports
    # the node costs from the dict it is given -- a dict's identity says nothing about its content
    # (ids are recycled, dicts are edited in place), and the costs are one f64 per e-node
    if r is not None and r.version == eg._version and costs is None:
        session().sync_symtab()
        return r
    b, packed = _upload(eg, costs)
    r = _Resident(eg._version, b, b.download_view(), packed)
    eg._esat_resident = r
    return r


def joint_match(eg, patterns, language=None):
    """Ordered, deduplicated substitutions of `patterns` (rewrite.py:405-433) on the device.
    Returns (records[M, W], var names, pvar names, n_roots) with class ids / attribute values."""
    r = _resident(eg)
    s = session()
    st = s.symtab
    comps = [compile_pattern(p, lambda n: st.name_id(n, create=False), st.code) for p in patterns]
    s.ctx.upload_patterns([c.program for c in comps])
    r.batch.ematch(list(range(len(comps))))
    vn = sorted({v for c in comps for v in c.var_names})
    qn = sorted({q for c in comps for q in c.pvar_names})
    if len(comps) == 1:
        words, off, cnt = r.batch.download_matches(0)
    else:
        r.batch.join([(list(range(len(comps))), [[vn.index(v) for v in c.var_names] for c in comps],
                       [[qn.index(q) for q in c.pvar_names] for c in comps], len(vn), len(qn))])
        words, off, cnt = r.batch.download_matches(0, from_join=True)
    W = len(comps) + len(vn) + len(qn)
    recs = words[: int(cnt[0]) * W].reshape(-1, W) if cnt[0] else np.zeros((0, W), np.uint32)
    return recs, vn, qn, len(comps)


def any_match(eg, pattern) -> bool:
    r = _resident(eg)
    s = session()
    st = s.symtab
    c = compile_pattern(pattern, lambda n: st.name_id(n, create=False), st.code)
    s.ctx.upload_patterns([c.program])
    r.batch.ematch([0], mode=native.MATCH_EXISTS)
    _, _, cnt = r.batch.download_matches(0)
    return bool(cnt[0])


def extract(eg, costs: dict, method: str):
    """Greedy extraction on the device. Returns (status, err_class, root_cost, chosen {cid: ENode})."""
    r = _resident(eg, costs)
    out = native.extract_with_retry(r.batch, method)
    st = int(out["status"][0])
    if st != native.X_OK:
        return st, int(out["err_class"][0]), None, None
    v = r.view
    C = int(v["C"][0])
    cls_id = v["cls_id"][:C]
    nko = v["nd_koff"]
    ENodeT, _ = _node_class(eg)
    symt = session().symtab
    chosen = {}
    for k in np.nonzero(out["reachable"][:C])[0]:
        j = int(out["choice"][k])
        kids = tuple(int(cls_id[p]) for p in v["nd_kpos"][nko[j]:nko[j + 1]])
        chosen[int(cls_id[k])] = ENodeT(symt.symbols[int(v["nd_sym"][j])], kids)
    return st, NONE, float(out["root_cost"][0]), chosen


def apply_rule(eg, rule, node_limit: int = 0, language=None):
    """apply_rule (rewrite.py:526-570) on the device: k_ematch/k_join for the rule's sources,
    k_apply for the instantiations and unions, k_rebuild; the rebuilt result is written back into
    the host e-graph. New operator symbols are interned on the host (apply.ApplyDriver)."""
    from .apply import ApplyDriver
    from .cost_model import CostModelConfig
    from .egraph import StructuralError
    from .pipeline import LeafPipeline
    from .rewrite import ApplyReport
    from .tensor_ir import TermLanguage

    lang = language or eg.language or TermLanguage()
    if node_limit:
        n = eg.size()[0]
        if n >= node_limit:
            raise StructuralError(f"node limit {node_limit} not above current node count {n}")
    if eg.dirty:
        raise StructuralError("ematch requires a rebuilt e-graph")
    s = session()
    leaf = export_state(eg, s.symtab)
    s.sync_symtab()
    head = max(256, 2 * leaf.n)
    while True:
        packed = Batch([leaf]).pack_with_headroom(nodes=head, kids=2 * head, ids=head)
        pipe = LeafPipeline(s.ctx, s.symtab.arrays(), [rule], lambda nm: s.symtab.name_id(nm, create=False),
                            s.symtab.code)
        b = pipe.load(packed)
        b.set_counts(packed["n_cnt"], packed["u_cnt"])
        pipe.rebuild()
        drv = ApplyDriver(pipe, s.symtab, lang, CostModelConfig(mode="term"), symbol_cls=_node_class(eg)[1])
        pipe.ematch()
        res = drv.apply(np.zeros(1, np.uint32))
        st = int(res["status"][0])
        if st != native.A_CAPACITY:
            break
        head *= 4
    s._uploaded = -1   # the driver re-uploaded the (possibly grown) table
    s.sync_symtab()
    if st != native.A_OK:
        raise RuntimeError(f"device apply failed with status {st}")
    found, changed, cyc, shp, unions, adds = (int(x) for x in res["report"][0][:6])
    rep = ApplyReport(rule_id=rule.id)
    rep.matches_found, rep.cycles_filtered, rep.shape_filtered = found, cyc, shp
    before = eg._version
    pipe.rebuild()
    _write_back(eg, b, packed, version_bump=adds + unions)
    rep.changed = eg._version != before
    rep.nodes_after, rep.classes_after = eg.size()
    rep.hit_node_limit = bool(node_limit) and rep.nodes_after >= node_limit
    return rep
