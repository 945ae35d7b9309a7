"""TENSAT-style sequential saturation on the device (SPEC.md:699-709 optimize_sequential).

Per iteration the multi-pattern rules are applied in ascending order (first ``k_multi``
iterations only), then the single-pattern rules in ascending order, with a
rebuild between rules; the loop stops when an iteration changes nothing or the node count reaches
``node_limit``. Every application is the device apply loop (k_ematch/k_join -> k_apply ->
k_rebuild) on a one-leaf batch whose arena headroom is grown when it runs out. Used for the
e-graph explosion stress of BASELINE config 4 (Inception-v3 at a large node limit).
"""

from __future__ import annotations

import numpy as np

from . import native
from .apply import ApplyDriver
from .arena import Batch, LeafState, export_state
from .pipeline import LeafPipeline
from .symtab import SymbolTable


def _clean_leaf(b, packed) -> LeafState:
    reb = b.download_rebuild()
    U = int(b.download_state()["U"][0])
    n = int(reb["n"][0])
    koff = reb["hc_koff"][: n + 1].copy()
    return LeafState(reb["hc_sym"][:n].copy(), koff, reb["hc_kids"][: int(koff[-1])].copy(), reb["hc_cid"][:n].copy(),
                     reb["hc_cost"][:n].copy(), reb["uf_parent"][:U].copy(), reb["uf_rank"][:U].copy(),
                     int(packed["root"][0]))


def saturate_sequential(egraph, rules, cost_config, node_limit: int, k_multi: int = 1, max_iters: int = 100,
                        ctx=None, symtab=None, log=None):
    """Returns (final rebuilt LeafState, symtab, per-application trace [(rule index, matches, added, n)])."""
    symtab = SymbolTable() if symtab is None else symtab
    ctx = ctx if ctx is not None else native.Context(0)
    leaf = export_state(egraph, symtab, cost_config)
    symtab.finalize()
    head = max(4096, 4 * leaf.n)
    trace = []

    def open_batch(state, headroom):
        packed = Batch([state]).pack_with_headroom(nodes=headroom, kids=2 * headroom, ids=headroom)
        pipe = LeafPipeline(ctx, symtab.arrays(), rules, lambda nm: symtab.name_id(nm, create=False), symtab.code)
        b = pipe.load(packed)
        b.set_counts(packed["n_cnt"], packed["u_cnt"])
        drv = ApplyDriver(pipe, symtab, egraph.language, cost_config)
        return packed, pipe, b, drv

    packed, pipe, b, drv = open_batch(leaf, head)
    pipe.rebuild()
    state = _clean_leaf(b, packed)
    order = ([i for i, r in enumerate(pipe.rules) if r.multi], [i for i, r in enumerate(pipe.rules) if not r.multi])
    n = state.n
    for it in range(max_iters):
        changed = False
        for ri in (order[0] if it < k_multi else []) + order[1]:
            while True:
                pipe.ematch()
                res = drv.apply(np.array([ri], np.uint32))
                if res["status"][0] != native.A_CAPACITY:
                    break
                head *= 4   # headroom exhausted: re-pack the pre-apply state with more, retry
                b.close()
                packed, pipe, b, drv = open_batch(state, head)
                pipe.rebuild()
            if res["status"][0] != native.A_OK:
                raise RuntimeError(f"device apply failed with status {int(res['status'][0])}")
            pipe.rebuild()
            state = _clean_leaf(b, packed)
            rep = res["report"][0]
            n = state.n
            trace.append((ri, int(rep[0]), int(rep[5]), n))
            changed |= bool(rep[1])
            if log:
                log(f"iter {it} rule {ri}: {int(rep[0])} matches, +{int(rep[5])} nodes, n={n}")
            if n >= node_limit:
                break
            if state.n + 4 * max(int(rep[5]), 1) > int(packed["node_base"][1]):   # keep headroom ahead
                head = max(head * 2, 8 * state.n)
                b.close()
                packed, pipe, b, drv = open_batch(state, head)
                pipe.rebuild()
        if n >= node_limit or not changed:
            break
    b.close()
    return state, symtab, trace
