"""Device apply loop (k_apply) against the reference's own rollouts.

Every golden rollout records the dirty state the reference's apply_rule left behind
(rewrite.py:526-570, captured right before its rebuild) together with the ApplyReport. For two
consecutive steps of one rollout, the device must turn step k's state -- rebuilt on the device --
into step k+1's state by applying step k+1's rule: identical hashcons (order, symbols, children,
classes, f64 costs), identical union-find roots and ranks, identical report counters."""

import re

import numpy as np
import pytest

from golden_io import FrozenSymtab, load_group, rules_of

pytestmark = pytest.mark.gpu

GROUPS = {"toy": (0, 0, 0.0), "zoo": (1, 1, 0.0), "analog_bert": (1, 2, 1e-9), "analog_nasrnn": (1, 2, 1e-9),
          "analog_resnext50": (1, 2, 1e-9), "analog_inception_v3": (1, 2, 1e-9), "analog_nasnet_a": (1, 2, 1e-9)}


def frozen_symbol_arrays(fs: FrozenSymtab) -> dict:
    from paper_2410_05534_b200.apply import symbol_arrays

    d = fs.d
    poff, flat = d["poff"], d["params"]
    codes = [flat[poff[i]:poff[i + 1]] for i in range(len(d["name"]))]
    payloads = [s[2] for s in d["symbols"]]
    return symbol_arrays(d["name"], d["arity"], payloads, codes, fs.values)


def consecutive_pairs(cases):
    idx = {c["name"]: i for i, c in enumerate(cases)}
    pairs = []
    for i, c in enumerate(cases):
        m = re.fullmatch(r"(.*)/step(\d+)", c["name"])
        if not m or int(m.group(2)) == 0:
            continue
        prev = f"{m.group(1)}/step{int(m.group(2)) - 1}"
        if prev in idx:
            pairs.append((idx[prev], i))
    return pairs


def find_all(parent):
    parent = parent.astype(np.int64)
    root = parent.copy()
    while True:
        nxt = parent[root]
        if np.array_equal(nxt, root):
            return root
        root = nxt


@pytest.mark.parametrize("group", list(GROUPS))
def test_apply_matches_reference_rollouts(group):
    from paper_2410_05534_b200 import native
    from paper_2410_05534_b200.arena import Batch, LeafState, unpack_state
    from paper_2410_05534_b200.pipeline import LeafPipeline

    lang, cost_mode, coeff = GROUPS[group]
    g = load_group(group)
    fs = FrozenSymtab(g["symtab"])
    cases = g["cases"]
    pairs = consecutive_pairs(cases)
    assert len(pairs) >= 5
    rules = rules_of(g)
    rule_pos = {r.id: i for i, r in enumerate(rules)}
    pre = [LeafState.from_json(cases[a]["state"]) for a, _ in pairs]
    packed = Batch(pre).pack_with_headroom(nodes=2048)
    ctx = native.Context(0)
    pipe = LeafPipeline(ctx, fs.arrays, rules, fs.name_id, fs.code)
    b = pipe.load(packed)
    b.set_counts(packed["n_cnt"], packed["u_cnt"])
    pipe.rebuild()
    pipe.ematch()
    off, words = pipe.apply_programs(fs.name_id, fs.code)
    ctx.apply_setup(lang, cost_mode, coeff, frozen_symbol_arrays(fs), off, words)
    leaf_rule = np.array([rule_pos[cases[post]["rule"]] for _, post in pairs], np.uint32)
    b.apply(leaf_rule)
    res = b.download_apply()
    st = b.download_state()
    bad = []
    for l, (_, post) in enumerate(pairs):
        exp = cases[post]
        rep = exp["apply"]
        if res["status"][l] != 0:
            bad.append((exp["name"], "status", int(res["status"][l])))
            continue
        got_rep = [int(x) for x in res["report"][l][:4]]
        want_rep = [rep["matches_found"], int(rep["changed"]), rep["cycles_filtered"], rep["shape_filtered"]]
        if got_rep != want_rep:
            bad.append((exp["name"], "report", got_rep, want_rep))
        got = unpack_state(packed, st, l)
        want = LeafState.from_json(exp["state"])
        for k in ("hc_sym", "hc_koff", "hc_kids", "hc_cid", "uf_rank"):
            if not np.array_equal(getattr(got, k), getattr(want, k)):
                bad.append((exp["name"], k, getattr(got, k).shape, getattr(want, k).shape))
        if not np.array_equal(got.hc_cost.view(np.uint64), want.hc_cost.view(np.uint64)):
            bad.append((exp["name"], "hc_cost"))
        if got.uf_parent.shape != want.uf_parent.shape or not np.array_equal(find_all(got.uf_parent),
                                                                              find_all(want.uf_parent)):
            bad.append((exp["name"], "uf roots"))
        if got.root != want.root:
            bad.append((exp["name"], "root"))
    b.close()
    ctx.close()
    assert not bad, (len(bad), len(pairs), bad[:6])


@pytest.mark.parametrize("group", ["toy", "analog_resnext50", "analog_inception_v3", "zoo"])
def test_apply_interns_missing_symbols(group):
    """Start from a live symbol table holding only the symbols of the pre-apply states: every new
    operator symbol the rules instantiate comes back as ESAT_A_NEED_SYMBOL, is interned on the
    host (ApplyDriver) and the apply is retried on the unchanged rebuilt view. The result must be
    the reference's post-apply state, compared through symbol identities."""
    import ast

    from paper_2410_05534_b200 import native
    from paper_2410_05534_b200.apply import ApplyDriver
    from paper_2410_05534_b200.arena import Batch, LeafState, unpack_state
    from paper_2410_05534_b200.cost_model import CostModelConfig
    from paper_2410_05534_b200.egraph import Symbol
    from paper_2410_05534_b200.pipeline import LeafPipeline
    from paper_2410_05534_b200.symtab import SymbolTable
    from paper_2410_05534_b200.tensor_ir import TensorLanguage, TermLanguage

    lang, cost_mode, coeff = GROUPS[group]
    g = load_group(group)
    fs = FrozenSymtab(g["symtab"])
    cases = g["cases"]
    # first steps only: the table then lacks the symbols the first application creates
    pairs = [(a, p) for a, p in consecutive_pairs(cases) if cases[a]["name"].endswith("/step0")]
    rules = rules_of(g)
    rule_pos = {r.id: i for i, r in enumerate(rules)}
    gsyms = [Symbol(n, a, ast.literal_eval(p)) for n, a, p in fs.d["symbols"]]
    gkey = [(s.name, s.arity, repr(s.payload)) for s in gsyms]
    language = TensorLanguage() if lang else TermLanguage()
    cfg = CostModelConfig(mode={0: "term", 1: "unit", 2: "analytic"}[cost_mode])
    pre = [LeafState.from_json(cases[a]["state"]) for a, _ in pairs]
    used = sorted({int(s) for lf in pre for s in lf.hc_sym})
    st = SymbolTable()
    remap = np.full(len(gsyms), 0xFFFFFFFF, np.uint32)
    for s in used:
        remap[s] = st.intern(gsyms[s], language)
    for lf in pre:
        lf.hc_sym = remap[lf.hc_sym]
    packed = Batch(pre).pack_with_headroom(nodes=2048)
    ctx = native.Context(0)
    st.finalize()
    pipe = LeafPipeline(ctx, st.arrays(), rules, lambda n: st.name_id(n, create=False), st.code)
    b = pipe.load(packed)
    b.set_counts(packed["n_cnt"], packed["u_cnt"])
    pipe.rebuild()
    drv = ApplyDriver(pipe, st, language, cfg)
    pipe.ematch()
    res = drv.apply(np.array([rule_pos[cases[post]["rule"]] for _, post in pairs], np.uint32))
    fresh = {int(s) for _, p in pairs for s in cases[p]["state"]["hc_sym"]} - set(used)
    assert drv.interned == len(fresh), (drv.interned, len(fresh))
    state = b.download_state()
    bad = []
    for l, (_, post) in enumerate(pairs):
        exp = cases[post]
        if res["status"][l] != 0:
            bad.append((exp["name"], "status", int(res["status"][l])))
            continue
        rep = exp["apply"]
        if [int(x) for x in res["report"][l][:4]] != [rep["matches_found"], int(rep["changed"]), rep["cycles_filtered"],
                                                  rep["shape_filtered"]]:
            bad.append((exp["name"], "report"))
        got = unpack_state(packed, state, l)
        want = LeafState.from_json(exp["state"])
        keys_got = [(s.name, s.arity, repr(s.payload)) for s in (st.symbols[i] for i in got.hc_sym)]
        if keys_got != [gkey[i] for i in want.hc_sym]:
            bad.append((exp["name"], "symbols"))
        for k in ("hc_koff", "hc_kids", "hc_cid", "uf_rank"):
            if not np.array_equal(getattr(got, k), getattr(want, k)):
                bad.append((exp["name"], k))
        if not np.array_equal(got.hc_cost.view(np.uint64), want.hc_cost.view(np.uint64)):
            bad.append((exp["name"], "hc_cost"))
    b.close()
    ctx.close()
    assert not bad, (len(bad), len(pairs), bad[:6])


@pytest.mark.parametrize("group", ["toy", "zoo", "analog_nasrnn", "analog_inception_v3"])
def test_device_resident_rollouts(group):
    """Whole reference rollouts replayed on the device without leaving it: one leaf per rollout,
    each step = rebuild -> e-match + join -> apply (the leaf's recorded rule), the arena's headroom
    absorbing the growth. After every step each leaf must hold the reference's dirty state."""
    from paper_2410_05534_b200 import native
    from paper_2410_05534_b200.arena import Batch, LeafState, unpack_state
    from paper_2410_05534_b200.pipeline import LeafPipeline

    lang, cost_mode, coeff = GROUPS[group]
    g = load_group(group)
    fs = FrozenSymtab(g["symtab"])
    cases = g["cases"]
    seqs = {}
    for i, c in enumerate(cases):
        m = re.fullmatch(r"(.*)/step(\d+)", c["name"])
        if m:
            seqs.setdefault(m.group(1), {})[int(m.group(2))] = i
    seqs = [s for s in seqs.values() if 0 in s and len(s) > 1]
    rules = rules_of(g)
    rule_pos = {r.id: i for i, r in enumerate(rules)}
    packed = Batch([LeafState.from_json(cases[s[0]]["state"]) for s in seqs]).pack_with_headroom(nodes=6144)
    ctx = native.Context(0)
    pipe = LeafPipeline(ctx, fs.arrays, rules, fs.name_id, fs.code)
    b = pipe.load(packed)
    b.set_counts(packed["n_cnt"], packed["u_cnt"])
    off, words = pipe.apply_programs(fs.name_id, fs.code)
    ctx.apply_setup(lang, cost_mode, coeff, frozen_symbol_arrays(fs), off, words)
    bad, checked = [], 0
    for k in range(1, max(max(s) for s in seqs) + 1):
        pipe.rebuild()
        pipe.ematch()
        lr = np.array([rule_pos[cases[s[k]]["rule"]] if k in s else 0xFFFFFFFF for s in seqs], np.uint32)
        b.apply(lr)
        res = b.download_apply()
        st = b.download_state()
        for l, s in enumerate(seqs):
            if k not in s:
                continue
            checked += 1
            want = LeafState.from_json(cases[s[k]]["state"])
            got = unpack_state(packed, st, l)
            same = (res["status"][l] == 0 and all(np.array_equal(getattr(got, f), getattr(want, f))
                                                  for f in ("hc_sym", "hc_koff", "hc_kids", "hc_cid", "uf_rank"))
                    and np.array_equal(got.hc_cost.view(np.uint64), want.hc_cost.view(np.uint64))
                    and np.array_equal(find_all(got.uf_parent), find_all(want.uf_parent)))
            if not same:
                bad.append(cases[s[k]]["name"])
    b.close()
    ctx.close()
    assert checked >= 5 and not bad, (checked, bad[:5])
