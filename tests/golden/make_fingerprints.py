"""Golden WL fingerprints by running the REFERENCE (egraph.py:247-296) on every golden state.

    python tests/golden/make_fingerprints.py

For each case of every golden group the dirty state is loaded into a reference ``EGraph``
(hashcons in insertion order, union-find arrays, root), rebuilt with the reference's own
``rebuild`` and fingerprinted with ``EGraph.fingerprint``. Output:
tests/golden/fingerprints.json.gz = {group: {case name: fingerprint (hex)}}.
"""

from __future__ import annotations

import ast
import gzip
import json
import multiprocessing as mp
import sys
from pathlib import Path

REF = "/root/reference/pkg/src"
HERE = Path(__file__).resolve().parent
sys.path.insert(0, REF)
sys.path.insert(0, str(HERE.parent.parent))

GROUPS = ["toy", "zoo", "analog_bert", "analog_nasrnn", "analog_resnext50", "analog_inception_v3",
          "analog_nasnet_a", "random"]


def load(name):
    with gzip.open(HERE / f"{name}.json.gz") as fh:
        return json.load(fh)


def fingerprint_case(args):
    symbols, state = args
    from esat import egraph as E

    syms = [E.Symbol(n, a, ast.literal_eval(p)) for n, a, p in symbols]
    eg = E.EGraph(None)
    eg._uf.parent = list(state["uf_parent"])
    eg._uf.rank = list(state["uf_rank"])
    koff, kids = state["hc_koff"], state["hc_kids"]
    hc = {}
    for i, (s, c) in enumerate(zip(state["hc_sym"], state["hc_cid"])):
        hc[E.ENode(syms[s], tuple(kids[koff[i]:koff[i + 1]]))] = c
    eg.hashcons = hc
    eg.root = None if state["root"] == 0xFFFFFFFF else state["root"]
    eg.dirty = [0]
    eg.rebuild()
    return f"{eg.fingerprint():016x}"


def main():
    out = {}
    with mp.Pool(mp.cpu_count()) as pool:
        for g in GROUPS:
            d = load(g)
            syms = d["symtab"]["symbols"]
            fps = pool.map(fingerprint_case, [(syms, c["state"]) for c in d["cases"]], chunksize=4)
            out[g] = {c["name"]: fp for c, fp in zip(d["cases"], fps)}
            print(g, len(fps), flush=True)
    raw = json.dumps(out, sort_keys=True, separators=(",", ":")).encode()
    with gzip.GzipFile(HERE / "fingerprints.json.gz", "wb", mtime=0) as fh:
        fh.write(raw)


if __name__ == "__main__":
    main()
