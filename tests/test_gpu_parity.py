"""Device parity: the sm_100a kernels vs the reference's golden vectors and the CPU oracle.

Bit-exact on integers (hashcons order, union-find roots and ranks, class CSR, match
sets, chosen e-nodes) and on the f64 extraction costs (float.hex equality, which is
stricter than north_star's 1e-5 relative bar).
"""

import numpy as np
import pytest

from golden_io import (GROUPS, check_rebuild, compile_rule, decode_extract, decode_matches, group_batch, load_group,
                       rules_of)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2410_05534_b200 import native

    c = native.Context(0)
    yield c
    c.close()


def _device_rebuild(ctx, name):
    from paper_2410_05534_b200 import native

    st, packed, cases = group_batch(name)
    ctx.upload_symtab(st.arrays)
    b = native.DeviceBatch(ctx, packed)
    b.upload()
    b.rebuild()
    out = b.download_rebuild()
    out.update(b.download_view())
    return st, packed, cases, b, out


@pytest.mark.parametrize("group", GROUPS)
def test_rebuild_matches_reference(ctx, group):
    st, packed, cases, b, out = _device_rebuild(ctx, group)
    bad = check_rebuild(packed, out, cases)
    assert not bad, bad[:3]


@pytest.mark.parametrize("group", GROUPS)
@pytest.mark.parametrize("method", ["default", "ocf"])
def test_extract_matches_reference(ctx, group, method):
    from paper_2410_05534_b200 import native

    st, packed, cases, b, view = _device_rebuild(ctx, group)
    ext = native.extract_with_retry(b, method)
    bad = []
    for l, c in enumerate(cases):
        got = decode_extract(packed, view, ext, l)
        if got != c["extract"][method]:
            bad.append((c["name"], got.get("cost", got.get("msg")), c["extract"][method].get("cost")))
    assert not bad, bad[:3]


@pytest.mark.parametrize("group", [g for g in GROUPS if g != "random"])
def test_ematch_matches_reference(ctx, group):
    st, packed, cases, b, view = _device_rebuild(ctx, group)
    g = load_group(group)
    rules = rules_of(g)
    progs, singles, multis = [], [], []
    for r in rules:
        comps, vn, qn, vm, qm = compile_rule(r, st)
        ids = []
        for cp in comps:
            ids.append(len(progs))
            progs.append(cp.program)
        (singles if r.kind == "single" else multis).append((r, ids, vn, qn, vm, qm))
    ctx.upload_patterns(progs)
    b.ematch(list(range(len(progs))))
    if multis:
        b.join([(ids, vm, qm, len(vn), len(qn)) for r, ids, vn, qn, vm, qm in multis])
    bad = []
    for r, ids, vn, qn, vm, qm in singles:
        words, off, cnt = b.download_matches(ids[0])
        W = 1 + len(vn) + len(qn)
        for l, c in enumerate(cases):
            got = decode_matches(words, off, cnt, W, l, 1, vn, qn, st)
            if got != c["ematch"][r.id]["matches"]:
                bad.append((c["name"], r.id, len(got), len(c["ematch"][r.id]["matches"])))
    for j, (r, ids, vn, qn, vm, qm) in enumerate(multis):
        words, off, cnt = b.download_matches(j, from_join=True)
        W = len(ids) + len(vn) + len(qn)
        for l, c in enumerate(cases):
            rec = c["ematch"][r.id]
            if "matches" not in rec:
                continue
            got = decode_matches(words, off, cnt, W, l, len(ids), vn, qn, st)
            if got != rec["matches"]:
                bad.append((c["name"], r.id, len(got), len(rec["matches"])))
    assert not bad, bad[:5]


def test_device_matches_oracle_on_replicated_batch(ctx):
    """Larger batch (all analog states x4) against the C oracle, all stages."""
    from oracle import oracle as O
    from paper_2410_05534_b200 import native
    from paper_2410_05534_b200.arena import Batch, LeafState

    leaves, st = [], None
    for name in ("analog_nasrnn", "analog_inception_v3"):
        g = load_group(name)
        st = g["symtab"]
        leaves += [LeafState.from_json(c["state"]) for c in g["cases"]]
        break
    packed = Batch(leaves * 4).pack()
    from golden_io import FrozenSymtab

    fs = FrozenSymtab(st)
    ctx.upload_symtab(fs.arrays)
    b = native.DeviceBatch(ctx, packed)
    b.upload()
    b.rebuild()
    dev = b.download_rebuild()
    dev.update(b.download_view())
    ref = O.rebuild(packed, fs.arrays["rank"])
    for k in ("n", "merges", "C", "root_pos"):
        assert np.array_equal(dev[k], ref[k]), k
    for method in ("default", "ocf"):
        e_dev = native.extract_with_retry(b, method)
        e_ref = O.extract(packed, ref, method)
        assert np.array_equal(e_dev["status"], e_ref["status"])
        assert np.array_equal(e_dev["root_cost"].view(np.uint64), e_ref["root_cost"].view(np.uint64))
        for l in range(packed["n_leaves"]):
            n0, C = int(packed["node_base"][l]), int(ref["C"][l])
            assert np.array_equal(e_dev["choice"][n0:n0 + C], e_ref["choice"][n0:n0 + C]), (method, l)


@pytest.mark.parametrize("group", [g for g in GROUPS if g != "random"])
def test_exists_mode_matches_reference_source_counts(ctx, group):
    """is_rule_applicable (rewrite.py:579-589) is one EXISTS-mode e-match of every source pattern:
    per (state, source) the device's existence bit must equal ``len(ematch(state, source)) > 0`` of
    the reference (the goldens' source_counts), and the LIST mode's counts must equal the counts."""
    from paper_2410_05534_b200 import native

    st, packed, cases, b, view = _device_rebuild(ctx, group)
    rules = rules_of(load_group(group))
    progs, where = [], []
    for r in rules:
        comps, *_ = compile_rule(r, st)
        for s, cp in enumerate(comps):
            where.append((r.id, s))
            progs.append(cp.program)
    ctx.upload_patterns(progs)
    b.ematch(list(range(len(progs))), mode=native.MATCH_EXISTS)
    exists = [b.download_matches(p)[2].copy() for p in range(len(progs))]
    b.ematch(list(range(len(progs))))
    counts = [b.download_matches(p)[2].copy() for p in range(len(progs))]
    bad = []
    for p, (rid, s) in enumerate(where):
        for l, c in enumerate(cases):
            want = c["ematch"][rid]["source_counts"][s]
            if bool(exists[p][l]) != (want > 0) or int(counts[p][l]) != want:
                bad.append((c["name"], rid, s, int(exists[p][l]), int(counts[p][l]), want))
    assert not bad, bad[:5]
    applicable = {rid: np.ones(len(cases), bool) for rid, _ in where}
    for p, (rid, s) in enumerate(where):
        applicable[rid] &= exists[p] > 0
    for rid, app in applicable.items():
        want = np.array([all(n > 0 for n in c["ematch"][rid]["source_counts"]) for c in cases])
        assert np.array_equal(app, want), rid
