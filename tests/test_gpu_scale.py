"""Large-leaf parity: e-graphs far beyond the MCTS analogs (tens of thousands of e-nodes per
leaf, mixed with small leaves in one batch) against the CPU oracle, every stage.

These sizes take the device paths the bench leaves never reach: rebuild leaves larger than
one CTA's shared-memory tables, e-match leaves whose class index does not fit the TMA
staging window, bitset histories of hundreds of words, pool regrowth on ESAT_X_CAPACITY,
and cyclic / infeasible OCF selections in big graphs. Bit-exact on everything
(integers, chosen e-nodes, f64 cost bits)."""

import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

RULES = """
(f0 (f1 ?x) ?y) => ?x
(g ?x ?y ?x) => ?x
(f2 ?x ?x) => ?x
(f3 (f0 ?x ?y) (f0 ?y ?x)) => ?x
(g ?x ?y ?z) |&| (f3 ?x ?w) => ?y |&| ?w
"""


def _random_leaf(rng, symtab, lang, n_adds, union_frac, window, cost_of, block=0):
    from paper_2410_05534_b200.arena import export_state
    from paper_2410_05534_b200.egraph import EGraph, ENode, Symbol

    eg = EGraph(lang)
    ids = [eg.add(ENode(Symbol(f"v{i}", 0))) for i in range(8)]
    for _ in range(n_adds):
        ar = rng.choice((1, 2, 2, 3))
        name = f"f{rng.randrange(4)}" if ar < 3 else "g"
        if block:  # independent blocks over shared atoms: bounded constituent histories
            start = 8 + ((len(ids) - 8) // block) * block
            pool = ids[max(start, len(ids) - window):] or ids[:8]
        else:
            pool = ids[-window:] if rng.random() < 0.9 else ids
        ids.append(eg.add(ENode(Symbol(name, ar), tuple(rng.choice(pool) for _ in range(ar)))))
    eg.root = ids[-1]
    for _ in range(int(union_frac * len(ids))):
        a = rng.randrange(len(ids))
        b = min(len(ids) - 1, max(0, a + rng.randint(-window, window)))
        eg.union(ids[a], ids[b])
    for _ in range(int(union_frac * len(ids))):  # congruence bait: f(a,b), f(a,c), b==c
        a, bb, c = (ids[min(len(ids) - 1, rng.randrange(len(ids)))] for _ in range(3))
        nm = f"f{rng.randrange(4)}"
        eg.add(ENode(Symbol(nm, 2), (a, bb)))
        eg.add(ENode(Symbol(nm, 2), (a, c)))
        eg.union(bb, c)
    for _ in range(int(0.01 * len(ids))):  # stale-key adds after unions
        ids.append(eg.add(ENode(Symbol(f"f{rng.randrange(4)}", 2), (rng.choice(ids), rng.choice(ids)))))
    st = export_state(eg, symtab, costs={})
    for i, s in enumerate(st.hc_sym):
        nm = symtab.symbols[s].name
        st.hc_cost[i] = cost_of.setdefault(nm, rng.choice((0.5, 1.0, 2.0, 3.0, 0.1, 0.7, 0.0)))
    return st


@pytest.fixture(scope="module")
def big_batch():
    from paper_2410_05534_b200.arena import Batch
    from paper_2410_05534_b200.symtab import SymbolTable
    from paper_2410_05534_b200.tensor_ir import TermLanguage

    rng = random.Random(2410)
    symtab, lang, cost_of = SymbolTable(), TermLanguage(), {}
    leaves = []
    for n_adds, uf, win, blk in ((40000, 0.01, 50, 400), (12000, 0.02, 60, 0), (3000, 0.03, 30, 0),
                                 (20000, 0.005, 2000, 1000)):
        leaves.append(_random_leaf(rng, symtab, lang, n_adds, uf, win, cost_of, blk))
    for _ in range(61):
        leaves.append(_random_leaf(rng, symtab, lang, rng.randint(5, 300), 0.05, 20, cost_of))
    leaves.insert(2, _random_leaf(rng, symtab, lang, 5000, 0.05, 5000, cost_of))
    packed = Batch(leaves).pack()
    return symtab, packed


@pytest.fixture(scope="module")
def dev(big_batch):
    from paper_2410_05534_b200 import native

    symtab, packed = big_batch
    ctx = native.Context(0)
    ctx.upload_symtab(symtab.arrays())
    b = native.DeviceBatch(ctx, packed)
    b.upload()
    b.rebuild()
    view = b.download_rebuild()
    view.update(b.download_view())
    yield ctx, b, view
    b.close()
    ctx.close()


def test_large_rebuild(big_batch, dev):
    from oracle import oracle as O

    symtab, packed = big_batch
    _, _, view = dev
    ref = O.rebuild(packed, symtab.arrays()["rank"], threads=8)
    assert int(np.max(ref["C"])) > 10000 and int(np.sum(ref["merges"])) > 100
    for k in ("n", "merges", "C", "root_pos", "uf_parent", "uf_rank"):
        assert np.array_equal(view[k], ref[k]), k
    nb, kb = packed["node_base"], packed["kid_base"]
    for l in range(packed["n_leaves"]):
        n0, n, k0 = int(nb[l]), int(ref["n"][l]), int(kb[l])
        C = int(ref["C"][l])
        for k in ("hc_sym", "hc_cid", "nd_sym", "nd_hc"):
            assert np.array_equal(view[k][n0:n0 + n], ref[k][n0:n0 + n]), (k, l)
        assert np.array_equal(view["cls_id"][n0:n0 + C], ref["cls_id"][n0:n0 + C]), l
        for k in ("hc_koff", "nd_koff"):
            assert np.array_equal(view[k][n0 + l:n0 + l + n + 1], ref[k][n0 + l:n0 + l + n + 1]), (k, l)
        assert np.array_equal(view["cls_off"][n0 + l:n0 + l + C + 1], ref["cls_off"][n0 + l:n0 + l + C + 1]), l
        K = int(ref["hc_koff"][n0 + l + n])
        assert np.array_equal(view["hc_kids"][k0:k0 + K], ref["hc_kids"][k0:k0 + K]), l
        assert np.array_equal(view["nd_kpos"][k0:k0 + K], ref["nd_kpos"][k0:k0 + K]), l
        assert np.array_equal(view["nd_cost"][n0:n0 + n].view(np.uint64), ref["nd_cost"][n0:n0 + n].view(np.uint64))


@pytest.mark.parametrize("method", ["default", "ocf"])
def test_large_extract(big_batch, dev, method):
    from oracle import oracle as O
    from paper_2410_05534_b200 import native

    symtab, packed = big_batch
    _, b, view = dev
    ext = native.extract_with_retry(b, method, factor=4, bitsets=2)
    ref = O.extract(packed, view, method, threads=16)
    assert np.array_equal(ext["status"], ref["status"])
    assert np.array_equal(ext["err_class"][ext["status"] != 0], ref["err_class"][ref["status"] != 0])
    assert np.array_equal(ext["root_cost"].view(np.uint64), ref["root_cost"].view(np.uint64))
    assert np.array_equal(ext["passes"], ref["passes"])
    for l in range(packed["n_leaves"]):
        if ref["status"][l] != 0:
            continue
        n0, C = int(packed["node_base"][l]), int(view["C"][l])
        assert np.array_equal(ext["reachable"][n0:n0 + C], ref["reachable"][n0:n0 + C]), (method, l)
        r = ref["reachable"][n0:n0 + C].astype(bool)
        assert np.array_equal(ext["choice"][n0:n0 + C][r], ref["choice"][n0:n0 + C][r]), (method, l)


def test_large_ematch_and_join(big_batch, dev):
    from oracle import oracle as O
    from paper_2410_05534_b200.patterns import compile_pattern, parse_rules

    symtab, packed = big_batch
    ctx, b, view = dev
    sa = symtab.arrays()
    rules = parse_rules(RULES)
    progs, singles, multis = [], [], []
    for r in rules:
        comps = [compile_pattern(p, symtab.name_id, symtab.code) for p in r.sources]
        ids = list(range(len(progs), len(progs) + len(comps)))
        progs += [c.program for c in comps]
        if len(comps) == 1:
            singles.append((ids[0], comps[0]))
        else:
            vn = sorted({v for c in comps for v in c.var_names})
            qn = sorted({q for c in comps for q in c.pvar_names})
            vm = [[vn.index(v) for v in c.var_names] for c in comps]
            qm = [[qn.index(q) for q in c.pvar_names] for c in comps]
            multis.append((ids, comps, vm, qm, len(vn), len(qn)))
    ctx.upload_patterns(progs)
    b.ematch(list(range(len(progs))))
    b.join([(ids, vm, qm, nv, nq) for ids, comps, vm, qm, nv, nq in multis])
    total = 0
    for pid, comp in singles:
        words, off, cnt = b.download_matches(pid)
        rw, roff, rcnt, W = O.ematch(packed, view, sa, comp.program, threads=16)
        assert np.array_equal(cnt, rcnt), pid
        assert np.array_equal(off, roff), pid
        assert np.array_equal(words[: int(off[-1])], rw), pid
        total += int(cnt.sum())
    for j, (ids, comps, vm, qm, nv, nq) in enumerate(multis):
        words, off, cnt = b.download_matches(j, from_join=True)
        rw, roff, rcnt, W = O.joint(packed, view, sa, [c.program for c in comps], vm, qm, nv, nq, threads=16)
        assert np.array_equal(cnt, rcnt), j
        assert np.array_equal(words[: int(off[-1])], rw), j
        total += int(cnt.sum())
    assert total > 1000
