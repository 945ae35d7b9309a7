"""Host symbol table: interned operator symbols -> dense ids for the device arena.

Device kernels never see Python symbols. Every e-node symbol is interned to a
``u32`` id carrying four device-side facts:

* ``name_id``  -- interned operator name; pattern heads match on it together with
                  the arity (rewrite.py:383)
* ``arity``
* ``rank``     -- position of ``(name, repr(payload))`` in sorted order, so that the
                  per-class node order ``node_sort_key = (name, repr(payload),
                  children)`` (egraph.py:65-70) becomes ``(rank, children)``; string
                  order of ``repr`` is kept (shapes sort lexicographically, not
                  numerically)
* ``params``   -- ``language.node_params(symbol)`` (rewrite.py:356) as
                  order-preserving integer codes (ints numerically, then strings),
                  so sorted substitutions (rewrite.py:396-397) sort identically

Ranks and codes depend on the whole interned set, so they are recomputed
(``finalize``) whenever new symbols were interned since the last upload.
"""

from __future__ import annotations

import numpy as np

NO_MATCH_CODE = 0x3FFFFFFF  # literal pattern value absent from every symbol


def _value_key(v):
    if isinstance(v, bool) or not isinstance(v, (int, str)):
        raise TypeError(f"unsupported attribute value {v!r}")
    return (0, v, "") if isinstance(v, int) else (1, 0, v)


class SymbolTable:
    def __init__(self) -> None:
        self.symbols: list = []
        self.params: list[tuple] = []
        self._index: dict = {}
        self.names: list[str] = []
        self._name_index: dict[str, int] = {}
        self._version = 0
        self._final_version = -1
        self.rank = np.zeros(0, np.uint32)
        self._codes: dict = {}
        self.values: list = []

    def __len__(self) -> int:
        return len(self.symbols)

    def name_id(self, name: str, create: bool = True) -> int:
        nid = self._name_index.get(name)
        if nid is None:
            if not create:
                return -1
            nid = len(self.names)
            self.names.append(name)
            self._name_index[name] = nid
        return nid

    def intern(self, symbol, language=None) -> int:
        key = (symbol.name, symbol.arity, repr(symbol.payload))
        sid = self._index.get(key)
        if sid is not None:
            return sid
        sid = len(self.symbols)
        self._index[key] = sid
        self.symbols.append(symbol)
        params = tuple(language.node_params(symbol)) if language is not None else ()
        self.params.append(params)
        self.name_id(symbol.name)
        self._version += 1
        return sid

    def lookup(self, symbol) -> int:
        return self._index.get((symbol.name, symbol.arity, repr(symbol.payload)), -1)

    @property
    def stale(self) -> bool:
        return self._final_version != self._version

    def finalize(self) -> None:
        if not self.stale:
            return
        order = sorted({(s.name, repr(s.payload)) for s in self.symbols})
        pos = {k: i for i, k in enumerate(order)}
        self.rank = np.array([pos[(s.name, repr(s.payload))] for s in self.symbols], np.uint32)
        vals = sorted({v for ps in self.params for v in ps}, key=_value_key)
        self.values = vals
        self._codes = {(type(v), v): i for i, v in enumerate(vals)}
        self._final_version = self._version

    def code(self, value) -> int:
        self.finalize()
        return self._codes.get((type(value), value), NO_MATCH_CODE)

    def decode(self, code: int):
        return self.values[code]

    def arrays(self) -> dict:
        """Device upload arrays (name_id, arity, rank, param CSR)."""
        self.finalize()
        n = len(self.symbols)
        name = np.array([self._name_index[s.name] for s in self.symbols], np.uint32)
        arity = np.array([s.arity for s in self.symbols], np.uint32)
        poff = np.zeros(n + 1, np.uint32)
        flat = []
        for i, ps in enumerate(self.params):
            flat.extend(self._codes[(type(v), v)] for v in ps)
            poff[i + 1] = len(flat)
        return {
            "name": name,
            "arity": arity,
            "rank": self.rank.copy(),
            "poff": poff,
            "params": np.array(flat, np.int32),
        }
