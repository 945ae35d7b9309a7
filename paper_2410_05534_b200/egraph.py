"""Host-side e-graph with the reference's API; `rebuild()` runs on the B200.

Mirrors `esat.egraph` (egraph.py:19-353) closely enough to be a drop-in for the hot path:
`Symbol`, `ENode`, `node_sort_key`, `EClass`, `UnionFind`, `EGraph.add/union/find/
canonicalize/rebuild/size/snapshot/dump`. Construction (`add`, `union`) is host work
with the reference's exact semantics (ids are dense and never reused; union by rank,
ties to the lower id; the insertion-ordered hashcons is semantic). `rebuild()` -- the
congruence closure of egraph.py:203-238 -- is executed by `k_rebuild` through the C-ABI
(`device.rebuild`); there is no host fallback.
"""

from __future__ import annotations

import hashlib
from collections import defaultdict
from dataclasses import dataclass, field
from typing import Any, Optional


class StructuralError(ValueError):
    """Malformed e-graph operation (unknown id, arity mismatch, unsupported payload...)."""


def _valid_payload(p: Any) -> bool:
    if p is None or isinstance(p, (int, str)):
        return True
    return isinstance(p, tuple) and all(_valid_payload(x) for x in p)


@dataclass(frozen=True)
class Symbol:
    name: str
    arity: int
    payload: Any = None

    def __post_init__(self) -> None:
        if self.arity < 0:
            raise StructuralError("negative arity")
        if not _valid_payload(self.payload):  # floats would break bit-exact hashing
            raise StructuralError(f"unsupported symbol payload: {self.payload!r}")

    def key(self) -> tuple:
        return (self.name, self.arity, repr(self.payload))


@dataclass(frozen=True)
class ENode:
    symbol: Symbol
    children: tuple = ()

    def __post_init__(self) -> None:
        if len(self.children) != self.symbol.arity:
            raise StructuralError(f"arity mismatch for {self.symbol.name}: expected {self.symbol.arity}, "
                                  f"got {len(self.children)}")

    def key(self) -> tuple:
        return (self.symbol.name, repr(self.symbol.payload), self.children)


def node_sort_key(node: ENode) -> tuple:
    return node.key()


@dataclass
class EClass:
    id: int
    nodes: set = field(default_factory=set)
    parents: set = field(default_factory=set)


class UnionFind:
    """Dense-id disjoint sets; union by rank with rank ties resolved to the lower id."""

    def __init__(self) -> None:
        self.parent: list = []
        self.rank: list = []

    def make(self) -> int:
        self.parent.append(len(self.parent))
        self.rank.append(0)
        return len(self.parent) - 1

    def find(self, x: int) -> int:
        if not 0 <= x < len(self.parent):
            raise StructuralError(f"unknown e-class id {x}")
        p = self.parent
        r = x
        while p[r] != r:
            r = p[r]
        while p[x] != r:
            p[x], x = r, p[x]
        return r

    def union(self, a: int, b: int) -> tuple:
        ra, rb = self.find(a), self.find(b)
        if ra == rb:
            return ra, ra
        if self.rank[ra] < self.rank[rb] or (self.rank[ra] == self.rank[rb] and rb < ra):
            ra, rb = rb, ra
        if self.rank[ra] == self.rank[rb]:
            self.rank[ra] += 1
        self.parent[rb] = ra
        return ra, rb

    def copy(self) -> "UnionFind":
        u = UnionFind()
        u.parent, u.rank = list(self.parent), list(self.rank)
        return u


class EGraph:
    """Single-writer e-graph; snapshots are independent copies (egraph.py:132-312)."""

    def __init__(self, language: Any = None) -> None:
        self._uf = UnionFind()
        self.classes: dict = {}
        self.hashcons: dict = {}
        self.root: Optional[int] = None
        self.dirty: list = []
        self.language = language
        self._version = 0
        self._fp_cache = None

    # queries ---------------------------------------------------------------
    def find(self, cid: int) -> int:
        return self._uf.find(cid)

    def canonicalize(self, node: ENode) -> ENode:
        return ENode(node.symbol, tuple(self._uf.find(c) for c in node.children))

    def canonical_root(self) -> int:
        if self.root is None:
            raise StructuralError("e-graph has no root")
        return self._uf.find(self.root)

    def canonical_class_ids(self) -> list:
        return sorted(self.classes)

    def enodes(self):
        for cid in self.canonical_class_ids():
            for node in sorted(self.classes[cid].nodes, key=node_sort_key):
                yield cid, node

    @property
    def version(self) -> int:
        return self._version

    def is_clean(self) -> bool:
        return not self.dirty

    def size(self) -> tuple:
        return sum(len(c.nodes) for c in self.classes.values()), len(self.classes)

    # construction ------------------------------------------------------------
    def add(self, node: ENode) -> int:
        canon = self.canonicalize(node)
        hit = self.hashcons.get(canon)
        if hit is not None:
            return self._uf.find(hit)
        cid = self._uf.make()
        self.classes[cid] = EClass(cid, {canon})
        self.hashcons[canon] = cid
        for ch in set(canon.children):
            self.classes[self._uf.find(ch)].parents.add((canon, cid))
        self._version += 1
        return cid

    def union(self, a: int, b: int) -> int:
        ra, rb = self._uf.find(a), self._uf.find(b)
        if ra == rb:
            return ra
        win, lose = self._uf.union(ra, rb)
        gone = self.classes.pop(lose)
        keep = self.classes[win]
        keep.nodes |= gone.nodes
        keep.parents |= gone.parents
        self.dirty.append(win)
        self._version += 1
        return win

    def rebuild(self) -> int:
        """Congruence closure on the B200 (k_rebuild); returns the merge count."""
        from . import device

        return device.rebuild(self)

    # copies / rendering --------------------------------------------------------
    def snapshot(self) -> "EGraph":
        g = EGraph(self.language)
        g._uf = self._uf.copy()
        g.classes = {cid: EClass(cid, set(c.nodes), set(c.parents)) for cid, c in self.classes.items()}
        g.hashcons = dict(self.hashcons)
        g.root, g.dirty, g._version, g._fp_cache = self.root, list(self.dirty), self._version, self._fp_cache
        return g

    def dump(self) -> str:
        out = []
        root = self.canonical_root() if self.root is not None else None
        for cid in self.canonical_class_ids():
            parts = []
            for n in sorted(self.classes[cid].nodes, key=node_sort_key):
                s = n.symbol.name
                if n.children:
                    s += "(" + ",".join(f"ec{self._uf.find(c)}" for c in n.children) + ")"
                if n.symbol.payload is not None:
                    s += f"#{n.symbol.payload!r}"
                parts.append(s)
            out.append(f"ec{cid}: " + " | ".join(parts) + (" <root>" if root == cid else ""))
        return "\n".join(out)

    def to_dot(self) -> str:
        """GraphViz text of the e-graph (egraph.py:331-353): one dashed cluster per canonical class
        (label ``ec<id>``), a circle per e-node labelled with its operator, and an edge from every
        e-node to the first node of each child class (``lhead`` = the child's cluster)."""
        cids = self.canonical_class_ids()
        members = {c: sorted(self.classes[c].nodes, key=node_sort_key) for c in cids}
        name = {}
        for c in cids:
            for n in members[c]:
                name[(c, n)] = f"n{len(name)}"
        lines = ["digraph egraph {", "  compound=true;", "  node [shape=circle];"]
        for c in cids:
            lines += [f"  subgraph cluster_{c} {{", f'    label="ec{c}"; style=dashed;']
            lines += [f'    {name[(c, n)]} [label="{n.symbol.name}"];' for n in members[c]]
            lines.append("  }")
        for c in cids:
            for n in members[c]:
                for ch in n.children:
                    t = self._uf.find(ch)
                    if members.get(t):
                        lines.append(f"  {name[(c, n)]} -> {name[(t, members[t][0])]} [lhead=cluster_{t}];")
        lines.append("}")
        return "\n".join(lines)

    def fingerprint(self) -> int:
        """Weisfeiler-Lehman class-label hash (egraph.py:247-296), host side (cache key only)."""
        if self.dirty:
            raise StructuralError("fingerprint requires a rebuilt e-graph")
        if self._fp_cache is not None and self._fp_cache[0] == self._version:
            return self._fp_cache[1]

        def h(*parts):
            d = hashlib.blake2b(digest_size=8)
            for p in parts:
                d.update(repr(p).encode())
                d.update(b"\x1f")
            return int.from_bytes(d.digest(), "big")

        lab = {c: h(sorted(n.symbol.key() for n in k.nodes)) for c, k in self.classes.items()}
        prev = None
        for _ in range(max(1, len(self.classes))):
            new = {c: h(sorted((n.symbol.key(), tuple(lab[self._uf.find(x)] for x in n.children)) for n in k.nodes))
                   for c, k in self.classes.items()}
            groups = defaultdict(list)
            for c, v in new.items():
                groups[v].append(c)
            part = {c: min(m) for m in groups.values() for c in m}
            lab = new
            if part == prev:
                break
            prev = part
        body = sorted(sorted((n.symbol.key(), tuple(lab[self._uf.find(x)] for x in n.children)) for n in k.nodes)
                      for k in self.classes.values())
        fp = h(body, lab[self.canonical_root()] if self.root is not None else None)
        self._fp_cache = (self._version, fp)
        return fp
