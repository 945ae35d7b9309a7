"""ctypes binding of the CPU oracle (oracle/esat_oracle.c) -- TEST INFRASTRUCTURE ONLY.

Importable only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg. The product package never imports this module.

All entry points take the packed batch of paper_2410_05534_b200/arena.py
(``Batch.pack()``) and return numpy arrays laid out exactly like the device
library's outputs, so parity tests compare arrays element for element.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "libesat_oracle.so"
NONE = 0xFFFFFFFF

_lib = None


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        _lib = C.CDLL(str(LIB_PATH))
        _lib.oracle_max_threads.restype = C.c_int
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def rebuild(packed: dict, sym_rank: np.ndarray, threads: int = 0) -> dict:
    """egraph.py:203-238 over every leaf. Returns new hashcons + union-find + clean view."""
    L = packed["n_leaves"]
    nb, kb, ub = packed["node_base"], packed["kid_base"], packed["id_base"]
    N, K = int(nb[-1]), int(kb[-1])
    parent = packed["uf_parent"].copy()
    rank = packed["uf_rank"].copy()
    out = {
        "n": np.zeros(L, np.uint32), "merges": np.zeros(L, np.uint32),
        "hc_sym": np.zeros(N, np.uint32), "hc_koff": np.zeros(N + L, np.uint32),
        "hc_kids": np.zeros(K, np.uint32), "hc_cid": np.zeros(N, np.uint32),
        "hc_cost": np.zeros(N, np.float64),
        "C": np.zeros(L, np.uint32), "root_pos": np.zeros(L, np.uint32),
        "cls_id": np.zeros(N, np.uint32), "cls_off": np.zeros(N + L, np.uint32),
        "nd_sym": np.zeros(N, np.uint32), "nd_koff": np.zeros(N + L, np.uint32),
        "nd_kpos": np.zeros(K, np.uint32), "nd_cost": np.zeros(N, np.float64),
        "nd_hc": np.zeros(N, np.uint32),
    }
    sr = np.ascontiguousarray(sym_rank, np.uint32)
    lib().oracle_rebuild_batch(
        C.c_uint32(L), _p(nb), _p(kb), _p(ub), _p(sr),
        _p(packed["hc_sym"]), _p(packed["hc_koff"]), _p(packed["hc_kids"]), _p(packed["hc_cid"]),
        _p(packed["hc_cost"]), _p(parent), _p(rank), _p(packed["root"]),
        _p(out["n"]), _p(out["merges"]), _p(out["hc_sym"]), _p(out["hc_koff"]), _p(out["hc_kids"]),
        _p(out["hc_cid"]), _p(out["hc_cost"]),
        _p(out["C"]), _p(out["root_pos"]), _p(out["cls_id"]), _p(out["cls_off"]), _p(out["nd_sym"]),
        _p(out["nd_koff"]), _p(out["nd_kpos"]), _p(out["nd_cost"]), _p(out["nd_hc"]), C.c_int(threads))
    out["uf_parent"], out["uf_rank"] = parent, rank
    return out


def _view_args(packed, view):
    return (C.c_uint32(packed["n_leaves"]), _p(packed["node_base"]), _p(packed["kid_base"]), _p(view["C"]),
            _p(view["cls_id"]), _p(view["cls_off"]), _p(view["nd_sym"]), _p(view["nd_koff"]), _p(view["nd_kpos"]))


def _sym_args(symarr):
    return (_p(np.ascontiguousarray(symarr["name"], np.uint32)), _p(np.ascontiguousarray(symarr["arity"], np.uint32)),
            _p(np.ascontiguousarray(symarr["poff"], np.uint32)), _p(np.ascontiguousarray(symarr["params"], np.int32)))


def ematch(packed: dict, view: dict, symarr: dict, program: np.ndarray, threads: int = 0):
    """Single-pattern e-match (rewrite.py:400). Returns (words, word offsets[L+1], counts[L], W)."""
    L = packed["n_leaves"]
    prog = np.ascontiguousarray(program, np.int32)
    W = 1 + int(prog[1]) + int(prog[2])
    off = np.zeros(L + 1, np.uint64)
    cnt = np.zeros(L, np.uint32)
    syms = [np.ascontiguousarray(symarr[k], np.uint32 if k != "params" else np.int32)
            for k in ("name", "arity", "poff", "params")]
    cap = 1 << 16
    while True:
        words = np.zeros(cap, np.uint32)
        rc = lib().oracle_ematch_batch(*_view_args(packed, view), *[_p(a) for a in syms], _p(prog),
                                       C.c_uint64(cap), _p(words), _p(off), _p(cnt), C.c_int(threads))
        if rc == 0:
            return words[: int(off[-1])], off, cnt, W
        cap = int(off[-1]) + 1


def joint(packed: dict, view: dict, symarr: dict, programs: list, var_maps: list, pvar_maps: list,
          n_vars: int, n_pvars: int, threads: int = 0):
    """Multi-pattern joint match (rewrite.py:405). Record = [S roots][vars][pvars]."""
    L = packed["n_leaves"]
    S = len(programs)
    progs = np.concatenate([np.asarray(p, np.int32) for p in programs]).astype(np.int32)
    poff = np.cumsum([0] + [len(p) for p in programs[:-1]]).astype(np.uint32)
    vmap = np.array([x for m in var_maps for x in m] or [0], np.uint32)
    vmo = np.cumsum([0] + [len(m) for m in var_maps[:-1]]).astype(np.uint32)
    pmap = np.array([x for m in pvar_maps for x in m] or [0], np.uint32)
    pmo = np.cumsum([0] + [len(m) for m in pvar_maps[:-1]]).astype(np.uint32)
    W = S + n_vars + n_pvars
    off = np.zeros(L + 1, np.uint64)
    cnt = np.zeros(L, np.uint32)
    syms = [np.ascontiguousarray(symarr[k], np.uint32 if k != "params" else np.int32)
            for k in ("name", "arity", "poff", "params")]
    cap = 1 << 16
    while True:
        words = np.zeros(cap, np.uint32)
        rc = lib().oracle_joint_batch(*_view_args(packed, view), *[_p(a) for a in syms], C.c_uint32(S),
                                      _p(progs), _p(poff), _p(vmap), _p(vmo), _p(pmap), _p(pmo),
                                      C.c_uint32(n_vars), C.c_uint32(n_pvars),
                                      C.c_uint64(cap), _p(words), _p(off), _p(cnt), C.c_int(threads))
        if rc == 0:
            return words[: int(off[-1])], off, cnt, W
        cap = int(off[-1]) + 1


def extract(packed: dict, view: dict, method: str, threads: int = 0) -> dict:
    """extraction.py:157 (method='default') / :229 (method='ocf') over every leaf."""
    L = packed["n_leaves"]
    N = int(packed["node_base"][-1])
    out = {"status": np.zeros(L, np.uint32), "err_class": np.zeros(L, np.uint32),
           "root_cost": np.zeros(L, np.float64), "class_cost": np.zeros(N, np.float64),
           "choice": np.zeros(N, np.uint32), "reachable": np.zeros(N, np.uint8),
           "passes": np.zeros(L, np.uint32)}
    lib().oracle_extract_batch(
        C.c_uint32(L), _p(packed["node_base"]), _p(packed["kid_base"]), _p(view["C"]), _p(view["root_pos"]),
        _p(view["cls_id"]), _p(view["cls_off"]), _p(view["nd_koff"]), _p(view["nd_kpos"]), _p(view["nd_cost"]),
        C.c_int(1 if method == "ocf" else 0),
        _p(out["status"]), _p(out["err_class"]), _p(out["root_cost"]), _p(out["class_cost"]),
        _p(out["choice"]), _p(out["reachable"]), _p(out["passes"]), C.c_int(threads))
    return out


if os.environ.get("ESAT_ORACLE_FORBID"):  # product-path guard used by tests
    raise ImportError("oracle import forbidden in this process")


def pipeline(packed: dict, symarr: dict, compiled_rules, method: str = "ocf", threads: int = 0) -> dict:
    """The CPU restatement of one MCTS leaf step over a batch: rebuild, every rule's
    (joint) match, greedy extraction -- the same stages as paper_2410_05534_b200.pipeline."""
    view = rebuild(packed, symarr["rank"], threads)
    matches = 0
    for r in compiled_rules:
        if r.multi:
            _, _, cnt, _ = joint(packed, view, symarr, [r._programs[i] for i in range(len(r.pattern_ids))],
                                 r.var_maps, r.pvar_maps, len(r.var_names), len(r.pvar_names), threads)
        else:
            _, _, cnt, _ = ematch(packed, view, symarr, r._programs[0], threads)
        matches += int(cnt.sum())
    ext = extract(packed, view, method, threads)
    return {"view": view, "extract": ext, "matches": matches}
