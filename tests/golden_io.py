"""Loading the reference-generated golden vectors and decoding batch outputs for comparison."""

from __future__ import annotations

import gzip
import json
from functools import lru_cache
from pathlib import Path

import numpy as np

from paper_2410_05534_b200.arena import Batch, LeafState
from paper_2410_05534_b200.patterns import compile_pattern, parse_rules
from paper_2410_05534_b200.symtab import NO_MATCH_CODE

GOLDEN = Path(__file__).resolve().parent / "golden"
RULES = Path(__file__).resolve().parent.parent / "paper_2410_05534_b200" / "rules"
GROUPS = ["toy", "zoo", "analog_bert", "analog_nasrnn", "analog_resnext50", "analog_inception_v3",
          "analog_nasnet_a", "random"]
NONE = 0xFFFFFFFF


@lru_cache(maxsize=None)
def load_group(name: str) -> dict:
    with gzip.open(GOLDEN / f"{name}.json.gz") as fh:
        return json.load(fh)


class FrozenSymtab:
    """The golden file's symbol table (ids, ranks, codes exactly as generated)."""

    def __init__(self, d: dict):
        self.d = d
        self.names = d["names"]
        self.values = d["values"]
        self._nid = {n: i for i, n in enumerate(self.names)}
        self._code = {(type(v), v): i for i, v in enumerate(self.values)}
        self.arrays = {
            "name": np.array(d["name"], np.uint32), "arity": np.array(d["arity"], np.uint32),
            "rank": np.array(d["rank"], np.uint32), "poff": np.array(d["poff"], np.uint32),
            "params": np.array(d["params"], np.int32),   # flat attribute codes (symtab.arrays())
        }

    def name_id(self, name: str) -> int:
        return self._nid.get(name, -1)

    def code(self, value) -> int:
        return self._code.get((type(value), value), NO_MATCH_CODE)


def group_batch(name: str, cases=None):
    g = load_group(name)
    cs = g["cases"] if cases is None else cases
    leaves = [LeafState.from_json(c["state"]) for c in cs]
    return FrozenSymtab(g["symtab"]), Batch(leaves).pack(), cs


def rules_of(group: dict):
    if not group["rules"]:
        return []
    return parse_rules((RULES / group["rules"]).read_text())


def finds(parent: np.ndarray) -> np.ndarray:
    r = parent.astype(np.int64).copy()
    while True:
        nr = r[r]
        if np.array_equal(nr, r):
            return r
        r = nr


def leaf_slice(packed, l):
    nb, kb, ub = packed["node_base"], packed["kid_base"], packed["id_base"]
    return int(nb[l]), int(nb[l + 1]), int(kb[l]), int(kb[l + 1]), int(ub[l]), int(ub[l + 1])


def check_rebuild(packed, out, cases):
    """Compare one batch's rebuild outputs with the reference's (egraph.py:203-238)."""
    bad = []
    for l, c in enumerate(cases):
        g = c["rebuild"]
        n0, n1, k0, k1, u0, u1 = leaf_slice(packed, l)
        n = int(out["n"][l])
        errs = []
        if int(out["merges"][l]) != g["merges"]:
            errs.append(f"merges {out['merges'][l]} != {g['merges']}")
        koff = out["hc_koff"][n0 + l: n0 + l + n + 1]
        hc = [[int(out["hc_sym"][n0 + i]), out["hc_kids"][k0 + koff[i]: k0 + koff[i + 1]].tolist(),
               int(out["hc_cid"][n0 + i])] for i in range(n)]
        if hc != g["hashcons"]:
            errs.append("hashcons differs")
        f = finds(out["uf_parent"][u0:u1].astype(np.int64))
        if f.tolist() != g["find"]:
            errs.append("find differs")
        if out["uf_rank"][u0:u1].tolist() != g["rank"]:
            errs.append("rank differs")
        C = int(out["C"][l])
        cid = out["cls_id"][n0:n0 + C]
        coff = out["cls_off"][n0 + l: n0 + l + C + 1]
        nko = out["nd_koff"][n0 + l: n0 + l + n + 1]
        classes = []
        for k in range(C):
            nodes = []
            for j in range(coff[k], coff[k + 1]):
                kp = out["nd_kpos"][k0 + nko[j]: k0 + nko[j + 1]]
                nodes.append([int(out["nd_sym"][n0 + j]), [int(cid[p]) for p in kp]])
            classes.append([int(cid[k]), nodes])
        if classes != g["classes"]:
            errs.append("classes differ")
        rp = int(out["root_pos"][l])
        root = None if rp == NONE else int(cid[rp])
        if root != g["root"]:
            errs.append(f"root {root} != {g['root']}")
        if errs:
            bad.append((c["name"], errs))
    return bad


def decode_matches(words, off, cnt, W, l, n_roots, vnames, qnames, symtab):
    recs = words[int(off[l]): int(off[l]) + int(cnt[l]) * W].reshape(-1, W) if cnt[l] else np.zeros((0, W), np.uint32)
    out = []
    nv = len(vnames)
    for r in recs.tolist():
        out.append([r[:n_roots], [[v, r[n_roots + i]] for i, v in enumerate(vnames)],
                    [[q, symtab.values[r[n_roots + nv + i]]] for i, q in enumerate(qnames)]])
    return out


def compile_rule(rule, symtab):
    """Per-source programs + the joint-match output maps (sorted combined names)."""
    comps = [compile_pattern(p, symtab.name_id, symtab.code) for p in rule.sources]
    vnames = sorted({v for c in comps for v in c.var_names})
    qnames = sorted({q for c in comps for q in c.pvar_names})
    vmaps = [[vnames.index(v) for v in c.var_names] for c in comps]
    qmaps = [[qnames.index(q) for q in c.pvar_names] for c in comps]
    return comps, vnames, qnames, vmaps, qmaps


EXC = {0: None, 1: ("ExtractionError", "greedy extraction failed to converge"),
       2: ("InfeasibleExtraction", "root e-class has no finite-cost program"),
       3: ("ExtractionError", "cyclic selection through e-class {}"),
       4: ("ExtractionError", "child e-class {} required but not chosen"),
       5: ("ExtractionError", "root e-class not chosen")}


def decode_extract(packed, view, ext, l):
    n0, n1, k0, k1, *_ = leaf_slice(packed, l)
    st = int(ext["status"][l])
    if st != 0:
        typ, msg = EXC[st]
        return {"error": typ, "msg": msg.format(int(ext["err_class"][l]))}
    C = int(view["C"][l])
    cid = view["cls_id"][n0:n0 + C]
    nko = view["nd_koff"][n0 + l: n1 + l + 1]
    chosen = []
    for k in range(C):
        if ext["reachable"][n0 + k]:
            j = int(ext["choice"][n0 + k])
            kp = view["nd_kpos"][k0 + nko[j]: k0 + nko[j + 1]]
            chosen.append([int(cid[k]), int(view["nd_sym"][n0 + j]), [int(cid[p]) for p in kp]])
    return {"cost": float(ext["root_cost"][l]).hex(), "chosen": chosen}
