"""SoA e-graph arena: the layout shared by the host, the CPU oracle and the device.

One *leaf* is one e-graph state in the form the reference's rebuild consumes
(egraph.py:203-226): the insertion-ordered hashcons list ``(node, class id)``
plus the union-find arrays. Order is semantic (rebuild scans hashcons in
insertion order and the survivor of a congruent pair is the first entry,
SURVEY Appendix A.2), so it is kept verbatim.

Per leaf (all little-endian, dense):
    hc_sym   u32[n]     interned symbol of hashcons entry i (symtab.py)
    hc_koff  u32[n+1]   CSR offsets into hc_kids (arity = hc_koff[i+1]-hc_koff[i])
    hc_kids  u32[K]     child class ids as stored in the key (may be stale)
    hc_cid   u32[n]     class id value of the entry
    hc_cost  f64[n]     operator cost of the node (cost_model.py), carried by rebuild
    uf_parent u32[U]    union-find parents, U = ids ever created (egraph.py:87-91)
    uf_rank   u8[U]     union-by-rank ranks (egraph.py:103-115)
    root      u32       raw root id (0xFFFFFFFF = none)

A *batch* concatenates leaves; per-leaf base offsets index every array.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

NONE = 0xFFFFFFFF


@dataclass
class LeafState:
    hc_sym: np.ndarray
    hc_koff: np.ndarray
    hc_kids: np.ndarray
    hc_cid: np.ndarray
    hc_cost: np.ndarray
    uf_parent: np.ndarray
    uf_rank: np.ndarray
    root: int = NONE

    @property
    def n(self) -> int:
        return int(self.hc_sym.shape[0])

    @property
    def n_ids(self) -> int:
        return int(self.uf_parent.shape[0])

    @property
    def n_kids(self) -> int:
        return int(self.hc_kids.shape[0])

    def to_json(self) -> dict:
        return {
            "hc_sym": self.hc_sym.tolist(),
            "hc_koff": self.hc_koff.tolist(),
            "hc_kids": self.hc_kids.tolist(),
            "hc_cid": self.hc_cid.tolist(),
            "hc_cost": [float(x).hex() for x in self.hc_cost],
            "uf_parent": self.uf_parent.tolist(),
            "uf_rank": self.uf_rank.tolist(),
            "root": int(self.root),
        }

    @classmethod
    def from_json(cls, d: dict) -> "LeafState":
        return cls(
            np.array(d["hc_sym"], np.uint32),
            np.array(d["hc_koff"], np.uint32),
            np.array(d["hc_kids"], np.uint32),
            np.array(d["hc_cid"], np.uint32),
            np.array([float.fromhex(x) for x in d["hc_cost"]], np.float64),
            np.array(d["uf_parent"], np.uint32),
            np.array(d["uf_rank"], np.uint8),
            int(d["root"]),
        )


def _class_shape(egraph, cid):
    cls = egraph.classes.get(egraph.find(cid))
    if cls is None:
        return None
    for node in cls.nodes:
        payload = node.symbol.payload
        return payload[1] if isinstance(payload, tuple) and len(payload) == 2 else None
    return None


def export_state(egraph, symtab, cost_config=None, costs: dict | None = None) -> LeafState:
    """Snapshot an e-graph (reference ``EGraph`` or ours, duck-typed) as a leaf.

    Node costs come from ``costs`` (canonical ENode -> float) when given, else
    from ``cost_config`` through cost_model.node_cost on the child class shapes.
    """
    from .cost_model import node_cost

    language = egraph.language
    items = list(egraph.hashcons.items())
    n = len(items)
    sym = np.empty(n, np.uint32)
    koff = np.zeros(n + 1, np.uint32)
    cid = np.empty(n, np.uint32)
    cost = np.zeros(n, np.float64)
    kids: list[int] = []
    shape_cache: dict = {}
    for i, (node, c) in enumerate(items):
        sym[i] = symtab.intern(node.symbol, language)
        kids.extend(node.children)
        koff[i + 1] = len(kids)
        cid[i] = c
        if costs is not None:
            cost[i] = costs.get(egraph.canonicalize(node), 0.0)
        elif cost_config is not None:
            shapes = []
            for ch in node.children:
                r = egraph.find(ch)
                if r not in shape_cache:
                    shape_cache[r] = _class_shape(egraph, r)
                shapes.append(shape_cache[r])
            cost[i] = node_cost(cost_config, node.symbol, tuple(shapes))
    uf = egraph._uf
    return LeafState(
        sym,
        koff,
        np.array(kids, np.uint32),
        cid,
        cost,
        np.array(uf.parent, np.uint32),
        np.array(uf.rank, np.uint8),
        NONE if egraph.root is None else int(egraph.root),
    )


@dataclass
class Batch:
    """Concatenated leaves with per-leaf bases (the C-ABI upload format)."""

    leaves: list = field(default_factory=list)

    def pack(self) -> dict:
        L = len(self.leaves)
        nb = np.zeros(L + 1, np.uint64)
        kb = np.zeros(L + 1, np.uint64)
        ub = np.zeros(L + 1, np.uint64)
        for i, lf in enumerate(self.leaves):
            nb[i + 1] = nb[i] + lf.n
            kb[i + 1] = kb[i] + lf.n_kids
            ub[i + 1] = ub[i] + lf.n_ids
        cat = lambda name, dt: (np.concatenate([getattr(lf, name) for lf in self.leaves]).astype(dt, copy=False)
                                if L else np.zeros(0, dt))
        # per-leaf CSR offsets are leaf-relative; store n+1 entries per leaf
        koff = np.concatenate([lf.hc_koff for lf in self.leaves]).astype(np.uint32) if L else np.zeros(0, np.uint32)
        return {
            "n_leaves": L,
            "node_base": nb,
            "kid_base": kb,
            "id_base": ub,
            "hc_sym": cat("hc_sym", np.uint32),
            "hc_koff": koff,
            "hc_kids": cat("hc_kids", np.uint32),
            "hc_cid": cat("hc_cid", np.uint32),
            "hc_cost": cat("hc_cost", np.float64),
            "uf_parent": cat("uf_parent", np.uint32),
            "uf_rank": cat("uf_rank", np.uint8),
            "root": np.array([lf.root for lf in self.leaves], np.uint32),
        }

    def pack_with_headroom(self, nodes: int, kids: int | None = None, ids: int | None = None) -> dict:
        """Pack with spare capacity per leaf for the device apply loop (esat_apply): leaf l's
        spans are n+nodes entries, K+kids child slots, U+ids union-find ids. Unused slots are
        zero; the live sizes travel as ``n_cnt`` / ``u_cnt`` (esat_batch_set_counts)."""
        kids = 2 * nodes if kids is None else kids
        ids = nodes if ids is None else ids
        L = len(self.leaves)
        nb = np.zeros(L + 1, np.uint64)
        kb = np.zeros(L + 1, np.uint64)
        ub = np.zeros(L + 1, np.uint64)
        for i, lf in enumerate(self.leaves):
            nb[i + 1] = nb[i] + lf.n + nodes
            kb[i + 1] = kb[i] + lf.n_kids + kids
            ub[i + 1] = ub[i] + lf.n_ids + ids
        N, K, U = int(nb[-1]), int(kb[-1]), int(ub[-1])
        out = {"n_leaves": L, "node_base": nb, "kid_base": kb, "id_base": ub,
               "hc_sym": np.zeros(N, np.uint32), "hc_koff": np.zeros(N + L, np.uint32),
               "hc_kids": np.zeros(K, np.uint32), "hc_cid": np.zeros(N, np.uint32),
               "hc_cost": np.zeros(N, np.float64), "uf_parent": np.zeros(U, np.uint32),
               "uf_rank": np.zeros(U, np.uint8), "root": np.array([lf.root for lf in self.leaves], np.uint32),
               "n_cnt": np.array([lf.n for lf in self.leaves], np.uint32),
               "u_cnt": np.array([lf.n_ids for lf in self.leaves], np.uint32)}
        for i, lf in enumerate(self.leaves):
            n0, k0, u0 = int(nb[i]), int(kb[i]), int(ub[i])
            out["hc_sym"][n0:n0 + lf.n] = lf.hc_sym
            out["hc_koff"][n0 + i:n0 + i + lf.n + 1] = lf.hc_koff
            out["hc_kids"][k0:k0 + lf.n_kids] = lf.hc_kids
            out["hc_cid"][n0:n0 + lf.n] = lf.hc_cid
            out["hc_cost"][n0:n0 + lf.n] = lf.hc_cost
            out["uf_parent"][u0:u0 + lf.n_ids] = lf.uf_parent
            out["uf_rank"][u0:u0 + lf.n_ids] = lf.uf_rank
        return out


def unpack_state(packed: dict, state: dict, l: int) -> LeafState:
    """Leaf l of a downloaded device arena with live counts (DeviceBatch.download_state)."""
    n0, k0, u0 = (int(packed[k][l]) for k in ("node_base", "kid_base", "id_base"))
    n, U = int(state["n"][l]), int(state["U"][l])
    koff = state["hc_koff"][n0 + l:n0 + l + n + 1].copy()
    K = int(koff[-1])
    return LeafState(state["hc_sym"][n0:n0 + n].copy(), koff, state["hc_kids"][k0:k0 + K].copy(),
                     state["hc_cid"][n0:n0 + n].copy(), state["hc_cost"][n0:n0 + n].copy(),
                     state["uf_parent"][u0:u0 + U].copy(), state["uf_rank"][u0:u0 + U].copy(),
                     int(packed["root"][l]))


def to_egraph(state: LeafState, symtab, language=None):
    """Host ``EGraph`` (ours) of a rebuilt leaf: the hashcons in the leaf's order, union-find
    arrays and classes regrouped from the hashcons (egraph.py:228-238) -- the inverse of
    export_state for clean states."""
    from collections import defaultdict

    from .egraph import EClass, EGraph, ENode

    eg = EGraph(language)
    ko = state.hc_koff
    nodes = [ENode(symtab.symbols[int(state.hc_sym[i])], tuple(int(k) for k in state.hc_kids[ko[i]:ko[i + 1]]))
             for i in range(state.n)]
    eg.hashcons = {nodes[i]: int(state.hc_cid[i]) for i in range(state.n)}
    eg._uf.parent = [int(x) for x in state.uf_parent]
    eg._uf.rank = [int(x) for x in state.uf_rank]
    groups, parents = defaultdict(set), defaultdict(set)
    for node, c in eg.hashcons.items():
        c = eg.find(c)
        groups[c].add(node)
        for ch in set(node.children):
            parents[eg.find(ch)].add((node, c))
    eg.classes = {c: EClass(c, groups[c], parents.get(c, set())) for c in sorted(groups)}
    eg.root = None if state.root == NONE else int(state.root)
    return eg
