"""Host side of the device WL fingerprint (k_fingerprint; reference egraph.py:247-296).

The reference hashes ``repr`` of sorted tuples that contain ``symbol.key()`` =
``(name, arity, repr(payload))`` (egraph.py:47-48) and integer labels. The device needs, per
symbol, the exact UTF-8 bytes of ``repr(symbol.key())`` and the key's rank in Python's tuple
order (to sort node descriptions the way ``sorted`` does); labels it prints itself.
"""

from __future__ import annotations

import numpy as np


def key_tables(keys: list) -> tuple:
    """keys[i] = (name, arity, repr(payload)) of symbol i -> (krank u32[n], key_off u32[n+1], bytes)."""
    order = sorted(range(len(keys)), key=lambda i: keys[i])
    krank = np.zeros(len(keys), np.uint32)
    for r, i in enumerate(order):
        krank[i] = r
    blobs = [repr(tuple(k)).encode() for k in keys]
    off = np.zeros(len(keys) + 1, np.uint32)
    for i, bl in enumerate(blobs):
        off[i + 1] = off[i] + len(bl)
    return krank, off, b"".join(blobs)


def symtab_key_tables(symtab) -> tuple:
    return key_tables([(s.name, s.arity, repr(s.payload)) for s in symtab.symbols])
