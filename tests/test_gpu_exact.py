"""The exact (branch-and-bound) final extractor, exact.extract_exact, against the
reference's own extract_exact (extraction.py:252-349) on the reference's random golden e-graphs:
same total cost bits and the same chosen e-node per reachable class (or the same error). Our side
is seeded by the device's OCF extraction (k_extract), the reference's by its own OCF.

Needs the reference importable (baseline/_ref, installed by the build; the source tree here)."""

import ast

import numpy as np
import pytest

from golden_io import group_batch, load_group

pytestmark = pytest.mark.gpu

N_CASES = 300


def _clean_states(packed, out):
    from paper_2410_05534_b200.arena import LeafState

    states = []
    for l in range(packed["n_leaves"]):
        n0, k0, u0 = (int(packed[k][l]) for k in ("node_base", "kid_base", "id_base"))
        U = int(packed["id_base"][l + 1]) - u0
        n = int(out["n"][l])
        koff = out["hc_koff"][n0 + l:n0 + l + n + 1].copy()
        states.append(LeafState(out["hc_sym"][n0:n0 + n].copy(), koff, out["hc_kids"][k0:k0 + int(koff[-1])].copy(),
                                out["hc_cid"][n0:n0 + n].copy(), out["hc_cost"][n0:n0 + n].copy(),
                                out["uf_parent"][u0:u0 + U].copy(), out["uf_rank"][u0:u0 + U].copy(),
                                int(packed["root"][l])))
    return states


def test_exact_matches_reference_on_random_egraphs():
    from oracle.mcts_ref import import_reference, reference_available

    if not reference_available():
        pytest.skip("reference not importable (baseline/_ref missing)")
    E, R, X, T = import_reference()
    from oracle.ref_pipeline import to_ref_egraph
    from paper_2410_05534_b200 import native
    from paper_2410_05534_b200.arena import to_egraph
    from paper_2410_05534_b200.egraph import Symbol
    from paper_2410_05534_b200.exact import extract_exact
    from paper_2410_05534_b200.extraction import ExtractionError

    g = load_group("random")
    cases = g["cases"][:N_CASES]
    st, packed, _ = group_batch("random", cases)
    ctx = native.Context(0)
    ctx.upload_symtab(st.arrays)
    b = native.DeviceBatch(ctx, packed)
    b.upload()
    b.rebuild()
    clean = _clean_states(packed, b.download_rebuild())
    b.close()

    class Syms:
        symbols = [Symbol(n, a, ast.literal_eval(p)) for n, a, p in g["symtab"]["symbols"]]

    bad, checked = [], 0
    for case, s in zip(cases, clean):
        eg = to_egraph(s, Syms)
        costs = {}
        ko = s.hc_koff
        for i, node in enumerate(eg.hashcons):
            costs[node] = float(s.hc_cost[i])
        ref = to_ref_egraph(s, g["symtab"]["symbols"], E, T)
        ref.rebuild()
        rcosts = {}
        for i, node in enumerate(ref.hashcons):
            rcosts[node] = float(s.hc_cost[i])
        try:
            r = X.extract_exact(ref, rcosts)
            want = (float(r.total_cost).hex(),
                    {c: (n.symbol.name, tuple(n.children)) for c, n in sorted(r.chosen.items())})
        except X.ExtractionError as exc:
            want = (type(exc).__name__, str(exc))
        try:
            o = extract_exact(eg, costs)
            got = (float(o.total_cost).hex(),
                   {c: (n.symbol.name, tuple(n.children)) for c, n in sorted(o.chosen.items())})
        except ExtractionError as exc:
            got = (type(exc).__name__, str(exc))
        checked += 1
        if got != want:
            bad.append((case["name"], got, want))
        assert len(ko) == s.n + 1
    assert checked == len(cases) and not bad, bad[:3]
    assert np.all([c["state"] for c in cases])
