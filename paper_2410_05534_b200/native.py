"""ctypes binding of libesat_b200.so (include/esat_b200.h) -- the only compute path.

There is no CPU fallback: if the library or a CUDA device is missing, every entry
point raises ``NativeUnavailable``. ``DeviceBatch`` owns one device-resident batch
of leaf e-graphs and exposes the C-ABI stages with numpy host buffers.
"""

from __future__ import annotations

import ctypes as C
import os
import weakref
from pathlib import Path
from typing import NamedTuple

import numpy as np

LIB_DIR = Path(__file__).resolve().parent / "_lib"
LIB_PATH = LIB_DIR / ("libesat_b200_debug.so" if os.environ.get("ESAT_DEBUG_LIB") else "libesat_b200.so")
if os.environ.get("ESAT_LIB"):   # measurement A/B: an in-tree variant build (csrc/Makefile `variant`)
    LIB_PATH = LIB_DIR / os.environ["ESAT_LIB"]
NONE = 0xFFFFFFFF

OK, E_ARG, E_CUDA, E_CAPACITY, E_STATE = 0, 1, 2, 3, 4
X_OK, X_NOT_CONVERGED, X_INFEASIBLE, X_CYCLIC, X_CHILD_NOT_CHOSEN, X_ROOT_NOT_CHOSEN, X_NO_ROOT, X_CAPACITY = range(8)
METHODS = {"default": 0, "default_greedy": 0, "ocf": 1, "ocf_greedy": 1}
MATCH_LIST, MATCH_EXISTS = 0, 1


class NativeUnavailable(RuntimeError):
    """The sm_100a library (or a B200) is not available; there is deliberately no fallback."""


class NativeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"esat_b200 error {code}: {msg}")
        self.code = code


_lib = None


def build() -> Path:
    import subprocess

    subprocess.run(["make", "-s", "-C", str(Path(__file__).resolve().parent / "csrc")], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise NativeUnavailable(f"{LIB_PATH} not built (run __graft_entry__.build())")
        L = C.CDLL(str(LIB_PATH))
        vp = C.c_void_p
        L.esat_last_error.restype = C.c_char_p
        L.esat_last_error.argtypes = [vp]
        L.esat_last_kernel_ms.restype = C.c_float
        L.esat_last_kernel_ms.argtypes = [vp]
        L.esat_last_async_ms.restype = C.c_float
        L.esat_last_async_ms.argtypes = [vp]
        for name in ("esat_ctx_create", "esat_ctx_destroy", "esat_ctx_sync", "esat_symtab_upload",
                     "esat_patterns_upload", "esat_batch_create", "esat_batch_destroy", "esat_batch_upload",
                     "esat_rebuild", "esat_ematch", "esat_join", "esat_extract", "esat_batch_set_pool",
                     "esat_download_rebuild", "esat_download_view", "esat_download_matches",
                     "esat_download_extract", "esat_result_device_ptrs", "esat_ctx_set_stream",
                     "esat_copy_results", "esat_extract_async", "esat_wait_async", "esat_fork",
                     "esat_batch_set_pool2", "esat_apply_setup", "esat_batch_set_counts", "esat_apply",
                     "esat_download_apply", "esat_download_state", "esat_fingerprint_setup", "esat_fingerprint",
                     "esat_download_fingerprint", "esat_ematch_masked", "esat_download_counts",
                     "esat_store_create", "esat_store_destroy", "esat_store_truncate", "esat_store_save",
                     "esat_store_put", "esat_store_info", "esat_store_download", "esat_batch_load_slots",
                     "esat_extract_shape", "esat_set_extract_lanes"):
            getattr(L, name).restype = C.c_int
        u32 = C.c_uint32
        L.esat_store_size.restype = u32
        L.esat_store_size.argtypes = [vp]
        L.esat_store_truncate.argtypes = [vp, u32]
        L.esat_store_save.argtypes = [vp, vp, u32, vp, vp]
        L.esat_store_put.argtypes = [vp, u32, u32, u32, u32, vp, vp, vp, vp, vp, vp, vp, vp]
        L.esat_store_info.argtypes = [vp, u32, vp, vp, vp, vp, vp]
        L.esat_store_download.argtypes = [vp, u32, vp, vp, vp, vp, vp, vp, vp]
        L.esat_batch_load_slots.argtypes = [vp, vp, vp]
        L.esat_apply_setup.argtypes = [vp, C.c_int, C.c_int, C.c_double, C.c_uint32, vp, vp, C.c_uint32, vp,
                                       C.c_uint32, vp, C.c_uint32, vp, vp]
        L.esat_batch_set_pool.argtypes = [vp, C.c_double]
        L.esat_batch_set_pool2.argtypes = [vp, C.c_double, C.c_double]
        L.esat_extract_shape.argtypes = [vp, vp, vp]
        L.esat_set_extract_lanes.argtypes = [vp, u32]
        _lib = L
    return _lib


EXPORTED = ("esat_ctx_create", "esat_ctx_destroy", "esat_last_error", "esat_ctx_sync", "esat_symtab_upload",
            "esat_patterns_upload", "esat_batch_create", "esat_batch_destroy", "esat_batch_upload",
            "esat_rebuild", "esat_ematch", "esat_join", "esat_batch_set_pool", "esat_extract",
            "esat_download_rebuild", "esat_download_view", "esat_download_matches", "esat_download_extract",
            "esat_result_device_ptrs", "esat_last_kernel_ms", "esat_ctx_set_stream", "esat_copy_results",
            "esat_extract_async", "esat_wait_async", "esat_last_async_ms", "esat_fork",
            "esat_batch_set_pool2", "esat_apply_setup", "esat_batch_set_counts", "esat_apply",
            "esat_download_apply", "esat_download_state", "esat_fingerprint_setup", "esat_fingerprint",
            "esat_download_fingerprint", "esat_ematch_masked", "esat_download_counts",
            "esat_store_create", "esat_store_destroy", "esat_store_size", "esat_store_truncate", "esat_store_save",
            "esat_store_put", "esat_store_info", "esat_store_download", "esat_batch_load_slots",
            "esat_extract_shape", "esat_set_extract_lanes")

# k_extract lane groups: leaves whose Gauss-Seidel levels average at most this many classes run two
# to a warp (16 lanes each); wider levels keep a warp per leaf (bench.py `extract_shape`)
LANES16_MAX_WIDTH = 6.0
TUNE_MIN_LEAVES = 1024

A_OK, A_NODE_LIMIT, A_NEED_SYMBOL, A_CAPACITY, A_PROGRAM = range(5)


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _u32(a):
    return np.ascontiguousarray(a, np.uint32)


class Context:
    """One CUDA context/stream per GPU per process (esat_ctx)."""

    def __init__(self, device: int = 0):
        self.L = lib()
        self.h = C.c_void_p()
        rc = self.L.esat_ctx_create(C.c_int(device), C.byref(self.h))
        if rc != OK:
            raise NativeUnavailable(f"esat_ctx_create(device={device}) failed with code {rc}: no usable B200")
        self.device = device
        self.symtab_version = None
        self._children = weakref.WeakSet()   # batches / stores: released before the context
        self.extract_lanes = None            # k_extract lanes per leaf: None until tuned (then 32 / 16)
        self.extract_width = None            # mean level width it was tuned on

    def check(self, rc: int):
        if rc != OK:
            raise NativeError(rc, self.L.esat_last_error(self.h).decode())

    def close(self):
        if self.h:
            for ch in list(self._children):
                ch.close()
            self.L.esat_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:   # interpreter teardown: module globals may already be gone
            pass

    def sync(self):
        self.check(self.L.esat_ctx_sync(self.h))

    def set_extract_lanes(self, lanes: int):
        """k_extract lanes per leaf for later extractions (32, 16 or 8; results are identical)."""
        self.check(self.L.esat_set_extract_lanes(self.h, C.c_uint32(lanes)))
        self.extract_lanes = lanes

    def reset_extract_lanes(self):
        """Forget the tuned width (a new workload): one leaf per warp until the next tuning."""
        self.check(self.L.esat_set_extract_lanes(self.h, C.c_uint32(32)))
        self.extract_lanes = None
        self.extract_width = None

    def tune_extract_lanes(self, batch) -> int | None:
        """Once per context, after an extraction of a batch of >= TUNE_MIN_LEAVES leaves: two leaves
        share a warp when the mean Gauss-Seidel level width is at most LANES16_MAX_WIDTH classes."""
        if self.extract_lanes is not None or batch.n_leaves < TUNE_MIN_LEAVES:
            return self.extract_lanes
        classes, levels = batch.extract_shape()
        self.extract_width = classes / max(levels, 1)
        self.set_extract_lanes(16 if self.extract_width <= LANES16_MAX_WIDTH else 32)
        return self.extract_lanes

    def set_stream(self, cuda_stream_handle: int):
        """Issue all work on a caller-owned stream (torch.cuda.current_stream().cuda_stream)."""
        self.check(self.L.esat_ctx_set_stream(self.h, C.c_void_p(cuda_stream_handle)))

    def last_ms(self) -> float:
        return float(self.L.esat_last_kernel_ms(self.h))

    def last_async_ms(self) -> float:
        return float(self.L.esat_last_async_ms(self.h))

    def fork(self):
        self.check(self.L.esat_fork(self.h))

    def wait_async(self):
        self.check(self.L.esat_wait_async(self.h))

    def upload_symtab(self, arrays: dict):
        n = len(arrays["name"])
        keep = [_u32(arrays["name"]), _u32(arrays["arity"]), _u32(arrays["rank"]), _u32(arrays["poff"]),
                np.ascontiguousarray(arrays["params"], np.int32)]
        self.check(self.L.esat_symtab_upload(self.h, C.c_uint32(n), *[_p(a) for a in keep]))

    def apply_setup(self, lang: int, cost_mode: int, coeff: float, sym: dict, rule_off, rule_words):
        """Symbol identities + rule target programs for esat_apply (apply.py)."""
        keep = [np.ascontiguousarray(sym["ndim"], np.uint8), _u32(sym["dims"]), _u32(sym["table"]),
                np.ascontiguousarray(sym["vint"], np.int32), _u32(rule_off),
                np.ascontiguousarray(rule_words, np.int32)]
        self._apply_keep = keep
        self.check(self.L.esat_apply_setup(self.h, lang, cost_mode, C.c_double(coeff), C.c_uint32(len(keep[0])),
                                           _p(keep[0]), _p(keep[1]), C.c_uint32(len(keep[2])), _p(keep[2]),
                                           C.c_uint32(len(keep[3])), _p(keep[3]), C.c_uint32(len(keep[4]) - 1),
                                           _p(keep[4]), _p(keep[5])))

    def fingerprint_setup(self, krank, key_off, key_bytes):
        keep = [_u32(krank), _u32(key_off), np.frombuffer(bytes(key_bytes), np.uint8).copy()]
        self._fp_keep = keep
        self.check(self.L.esat_fingerprint_setup(self.h, C.c_uint32(len(keep[0])), *[_p(a) for a in keep]))

    def upload_patterns(self, programs: list):
        words = np.concatenate([np.asarray(p, np.int32) for p in programs]) if programs else np.zeros(1, np.int32)
        off = np.cumsum([0] + [len(p) for p in programs]).astype(np.uint32)
        self.check(self.L.esat_patterns_upload(self.h, C.c_uint32(len(programs)), _p(off),
                                               C.c_uint32(len(words)), _p(words)))


class DeviceBatch:
    """A device-resident batch of leaf e-graphs (esat_batch)."""

    def __init__(self, ctx: Context, packed: dict):
        self.ctx = ctx
        self.L = ctx.L
        self.packed = packed
        self.n_leaves = packed["n_leaves"]
        self.nb = np.ascontiguousarray(packed["node_base"], np.uint64)
        self.kb = np.ascontiguousarray(packed["kid_base"], np.uint64)
        self.ub = np.ascontiguousarray(packed["id_base"], np.uint64)
        self.h = C.c_void_p()
        ctx.check(self.L.esat_batch_create(ctx.h, C.c_uint32(self.n_leaves), _p(self.nb), _p(self.kb), _p(self.ub),
                                           C.byref(self.h)))
        ctx._children.add(self)

    def close(self):
        if self.h:
            self.L.esat_batch_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:   # interpreter teardown: module globals may already be gone
            pass

    @property
    def N(self):
        return int(self.nb[-1])

    @property
    def K(self):
        return int(self.kb[-1])

    @property
    def U(self):
        return int(self.ub[-1])

    def upload(self, packed: dict | None = None):
        p = packed or self.packed
        self._keep = [p["hc_sym"], p["hc_koff"], p["hc_kids"], p["hc_cid"], p["hc_cost"], p["uf_parent"],
                      p["uf_rank"], p["root"]]
        self.ctx.check(self.L.esat_batch_upload(self.h, *[_p(a) for a in self._keep]))

    def rebuild(self):
        self.ctx.check(self.L.esat_rebuild(self.h))

    def set_counts(self, n_cnt, u_cnt):
        self._cnt_keep = (_u32(n_cnt), _u32(u_cnt))
        self.ctx.check(self.L.esat_batch_set_counts(self.h, *[_p(a) for a in self._cnt_keep]))

    def apply(self, leaf_rule, node_limit: int = 0):
        lr = _u32(leaf_rule)
        self.ctx.check(self.L.esat_apply(self.h, _p(lr), C.c_uint32(node_limit)))

    def fingerprint(self):
        self.ctx.check(self.L.esat_fingerprint(self.h))

    def download_fingerprint(self):
        fp, st = np.zeros(self.n_leaves, np.uint64), np.zeros(self.n_leaves, np.uint32)
        self.ctx.check(self.L.esat_download_fingerprint(self.h, _p(fp), _p(st)))
        return fp, st

    def download_apply(self) -> dict:
        L = self.n_leaves
        st, rep, miss = np.zeros(L, np.uint32), np.zeros((L, 8), np.uint32), np.zeros((L, 16), np.uint32)
        self.ctx.check(self.L.esat_download_apply(self.h, _p(st), _p(rep), _p(miss)))
        return {"status": st, "report": rep, "missing": miss}

    def download_state(self) -> dict:
        """The batch's input arena (dirty state after an apply) and live counts."""
        L, N, K, U = self.n_leaves, self.N, self.K, self.U
        o = {"n": np.zeros(L, np.uint32), "U": np.zeros(L, np.uint32), "hc_sym": np.zeros(N, np.uint32),
             "hc_koff": np.zeros(N + L, np.uint32), "hc_kids": np.zeros(max(K, 1), np.uint32),
             "hc_cid": np.zeros(N, np.uint32), "hc_cost": np.zeros(N, np.float64),
             "uf_parent": np.zeros(U, np.uint32), "uf_rank": np.zeros(U, np.uint8)}
        self.ctx.check(self.L.esat_download_state(self.h, *[_p(o[k]) for k in (
            "n", "U", "hc_sym", "hc_koff", "hc_kids", "hc_cid", "hc_cost", "uf_parent", "uf_rank")]))
        return o

    def live_counts(self):
        """(n_cnt, u_cnt): live hashcons entries and union-find ids of the batch input per leaf."""
        n, u = np.zeros(self.n_leaves, np.uint32), np.zeros(self.n_leaves, np.uint32)
        self.ctx.check(self.L.esat_download_state(self.h, _p(n), _p(u), None, None, None, None, None, None, None))
        return n, u

    def rebuilt_sizes(self):
        """(n, C): e-nodes and e-classes of every leaf's last rebuild (EGraph.size())."""
        n, c = np.zeros(self.n_leaves, np.uint32), np.zeros(self.n_leaves, np.uint32)
        self.ctx.check(self.L.esat_download_rebuild(self.h, _p(n), None, None, None, None, None, None, None, None))
        self.ctx.check(self.L.esat_download_view(self.h, _p(c), None, None, None, None, None, None, None, None))
        return n, c

    def set_pool(self, entries_per_node: float, bitsets_per_node: float | None = None):
        if bitsets_per_node is None:
            self.ctx.check(self.L.esat_batch_set_pool(self.h, C.c_double(entries_per_node)))
        else:
            self.ctx.check(self.L.esat_batch_set_pool2(self.h, C.c_double(entries_per_node),
                                                       C.c_double(bitsets_per_node)))

    def extract(self, method: str):
        self.ctx.check(self.L.esat_extract(self.h, C.c_int(METHODS[method])))

    def extract_async(self, method: str):
        """Extraction on the side stream, overlapping e-matching (join with ctx.wait_async())."""
        self.ctx.check(self.L.esat_extract_async(self.h, C.c_int(METHODS[method])))

    def ematch(self, pattern_ids, mode: int = MATCH_LIST, leaf_mask=None):
        """k_ematch of the call patterns over every leaf; ``leaf_mask`` restricts a leaf to the
        patterns it needs (esat_ematch_masked): shape [L] (bit p = call-pattern p, <= 32 patterns)
        or [ceil(P/32), L] (bit p of row c = call-pattern 32c+p)."""
        ids = _u32(pattern_ids)
        if leaf_mask is None:
            self.ctx.check(self.L.esat_ematch(self.h, C.c_uint32(len(ids)), _p(ids), C.c_int(mode)))
        else:
            m = _u32(leaf_mask).reshape(-1)
            if m.size != ((len(ids) + 31) // 32) * self.n_leaves:
                raise ValueError(f"leaf_mask needs ceil(P/32) x {self.n_leaves} words, got {m.size}")
            self.ctx.check(self.L.esat_ematch_masked(self.h, C.c_uint32(len(ids)), _p(ids), C.c_int(mode), _p(m)))

    def download_counts(self, n: int, from_join: bool = False) -> np.ndarray:
        """[n, L] counts of the last e-match (or join) call's patterns (rules) in one copy."""
        out = np.zeros((n, self.n_leaves), np.uint32)
        self.ctx.check(self.L.esat_download_counts(self.h, C.c_int(int(from_join)), _p(out)))
        return out

    def join(self, specs: list):
        """specs: per rule (source pattern ids, var maps per source, pvar maps per source, NV, NQ)."""
        src_off, src, map_off, vmap, qmap, nv, nq = [0], [], [0], [], [], [], []
        for ids, vmaps, qmaps, NV, NQ in specs:
            src.extend(ids)
            src_off.append(len(src))
            # per source: var map then pvar map, offsets per source
            for vm, qm in zip(vmaps, qmaps):
                vmap.extend(vm)
                qmap.extend(qm)
            nv.append(NV)
            nq.append(NQ)
        # map offsets are per source (var_map and pvar_map each indexed by their own offsets)
        vo, qo = [0], [0]
        for ids, vmaps, qmaps, *_ in specs:
            for vm, qm in zip(vmaps, qmaps):
                vo.append(vo[-1] + len(vm))
                qo.append(qo[-1] + len(qm))
        arrs = [_u32(src_off), _u32(src), _u32(np.stack([vo, qo], 1).reshape(-1)), _u32(vmap or [0]),
                _u32(qmap or [0]), _u32(nv), _u32(nq)]
        self._keep_join = arrs
        self.ctx.check(self.L.esat_join(self.h, C.c_uint32(len(specs)), *[_p(a) for a in arrs]))

    def copy_results(self, root_cost_ptr: int, status_ptr: int):
        """D2D copy of per-leaf root costs / statuses into caller device buffers (torch tensors)."""
        self.ctx.check(self.L.esat_copy_results(self.h, C.c_void_p(root_cost_ptr), C.c_void_p(status_ptr)))

    # ---- downloads ---------------------------------------------------------------
    def download_rebuild(self) -> dict:
        L, N, K, U = self.n_leaves, self.N, self.K, self.U
        o = {"n": np.zeros(L, np.uint32), "merges": np.zeros(L, np.uint32), "hc_sym": np.zeros(N, np.uint32),
             "hc_koff": np.zeros(N + L, np.uint32), "hc_kids": np.zeros(K, np.uint32),
             "hc_cid": np.zeros(N, np.uint32), "hc_cost": np.zeros(N, np.float64),
             "uf_parent": np.zeros(U, np.uint32), "uf_rank": np.zeros(U, np.uint8)}
        self.ctx.check(self.L.esat_download_rebuild(self.h, *[_p(o[k]) for k in (
            "n", "merges", "hc_sym", "hc_koff", "hc_kids", "hc_cid", "hc_cost", "uf_parent", "uf_rank")]))
        return o

    def download_view(self) -> dict:
        L, N, K = self.n_leaves, self.N, self.K
        o = {"C": np.zeros(L, np.uint32), "root_pos": np.zeros(L, np.uint32), "cls_id": np.zeros(N, np.uint32),
             "cls_off": np.zeros(N + L, np.uint32), "nd_sym": np.zeros(N, np.uint32),
             "nd_koff": np.zeros(N + L, np.uint32), "nd_kpos": np.zeros(K, np.uint32),
             "nd_cost": np.zeros(N, np.float64), "nd_hc": np.zeros(N, np.uint32)}
        self.ctx.check(self.L.esat_download_view(self.h, *[_p(o[k]) for k in (
            "C", "root_pos", "cls_id", "cls_off", "nd_sym", "nd_koff", "nd_kpos", "nd_cost", "nd_hc")]))
        return o

    def download_extract(self) -> dict:
        L, N = self.n_leaves, self.N
        o = {"status": np.zeros(L, np.uint32), "err_class": np.zeros(L, np.uint32),
             "root_cost": np.zeros(L, np.float64), "class_cost": np.zeros(N, np.float64),
             "choice": np.zeros(N, np.uint32), "reachable": np.zeros(N, np.uint8), "passes": np.zeros(L, np.uint32)}
        self.ctx.check(self.L.esat_download_extract(self.h, *[_p(o[k]) for k in (
            "status", "err_class", "root_cost", "class_cost", "choice", "reachable", "passes")]))
        self.ctx.tune_extract_lanes(self)
        return o

    def extract_shape(self) -> tuple:
        """(total e-classes, total Gauss-Seidel levels) of the last extraction over the batch."""
        c, lv = C.c_uint64(), C.c_uint64()
        self.ctx.check(self.L.esat_extract_shape(self.h, C.byref(c), C.byref(lv)))
        return int(c.value), int(lv.value)

    def download_extract_light(self) -> dict:
        """Per-leaf status, error class / overflow mask and root cost only."""
        L = self.n_leaves
        o = {"status": np.zeros(L, np.uint32), "err_class": np.zeros(L, np.uint32), "root_cost": np.zeros(L)}
        self.ctx.check(self.L.esat_download_extract(self.h, _p(o["status"]), _p(o["err_class"]), _p(o["root_cost"]),
                                                    None, None, None, None))
        self.ctx.tune_extract_lanes(self)
        return o

    def download_extract_small(self, root_cost: np.ndarray, status: np.ndarray):
        """D2H of the per-leaf root costs (f64) and statuses (u32) only -- the MCTS reward inputs."""
        self.ctx.check(self.L.esat_download_extract(self.h, _p(status), None, _p(root_cost), None, None, None,
                                                    None))
        return root_cost, status

    def download_matches(self, index: int, from_join: bool = False):
        L = self.n_leaves
        cnt = np.zeros(L, np.uint32)
        off = np.zeros(L + 1, np.uint64)
        self.ctx.check(self.L.esat_download_matches(self.h, C.c_int(int(from_join)), C.c_uint32(index), _p(cnt),
                                                    _p(off), None, C.c_uint64(0)))
        words = np.zeros(max(int(off[-1]), 1), np.uint32)
        self.ctx.check(self.L.esat_download_matches(self.h, C.c_int(int(from_join)), C.c_uint32(index), _p(cnt),
                                                    _p(off), _p(words), C.c_uint64(len(words))))
        return words, off, cnt


def extract_with_retry(batch: DeviceBatch, method: str, factor: float = 8.0, max_factor: float = 1 << 16,
                       bitsets: float = 4.0, light: bool = False) -> dict:
    """Run extraction, growing the OCF history pools on ESAT_X_CAPACITY (host regrow path).
    err_class of an overflowed leaf is the overflow mask: 1 grows the bitset pool x2, 2 grows the
    contribution pool x4. ``light``: download the per-leaf status / error / root cost only."""
    batch.set_pool(factor, bitsets)
    while True:
        batch.extract(method)
        out = batch.download_extract_light() if light else batch.download_extract()
        over = out["status"] == X_CAPACITY
        if method.startswith("ocf") and np.any(over) and factor < max_factor and bitsets < max_factor:
            mask = int(np.bitwise_or.reduce(out["err_class"][over]))
            if mask & 1 or not mask & 3:
                bitsets *= 2
            if mask & 2 or not mask & 3:
                factor *= 4
            batch.set_pool(factor, bitsets)
            continue
        return out


class Slot(NamedTuple):
    """A leaf e-graph state held in a device SnapshotStore (hashcons entries n, child slots K,
    union-find ids U, raw root) -- the device counterpart of arena.LeafState."""
    store: int
    index: int
    n: int
    K: int
    U: int
    root: int

    @property
    def n_ids(self) -> int:
        return self.U


class SnapshotStore:
    """EGraph.snapshot (egraph.py:300-312) on the device (esat_store): an append-only slot arena of
    leaf states. ``save`` copies the last rebuild of batch leaves into new slots, ``load`` fills a
    batch's input arena from slots -- both device to device."""

    def __init__(self, ctx: Context):
        self.ctx = ctx
        self.L = ctx.L
        self.h = C.c_void_p()
        ctx.check(self.L.esat_store_create(ctx.h, C.byref(self.h)))
        ctx._children.add(self)
        self.id = id(self)

    def close(self):
        if self.h:
            self.L.esat_store_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __len__(self):
        return int(self.L.esat_store_size(self.h))

    def truncate(self, count: int):
        self.ctx.check(self.L.esat_store_truncate(self.h, count))

    def _slots(self, idx) -> list:
        idx = _u32(idx)
        n, K, U, root = (np.zeros(len(idx), np.uint32) for _ in range(4))
        self.ctx.check(self.L.esat_store_info(self.h, len(idx), _p(idx), _p(n), _p(K), _p(U), _p(root)))
        return [Slot(self.id, int(i), int(a), int(b), int(c), int(r)) for i, a, b, c, r in zip(idx, n, K, U, root)]

    def save(self, batch: "DeviceBatch", leaves) -> list:
        leaves = _u32(leaves)
        out = np.zeros(len(leaves), np.uint32)
        self.ctx.check(self.L.esat_store_save(self.h, batch.h, len(leaves), _p(leaves), _p(out)))
        return self._slots(out)

    def put(self, st) -> Slot:
        """A host LeafState into a new slot."""
        arrs = [_u32(st.hc_sym), _u32(st.hc_koff), _u32(st.hc_kids), _u32(st.hc_cid),
                np.ascontiguousarray(st.hc_cost, np.float64), _u32(st.uf_parent), np.ascontiguousarray(st.uf_rank, np.uint8)]
        out = C.c_uint32()
        self.ctx.check(self.L.esat_store_put(self.h, st.n, st.n_kids, st.n_ids, st.root & 0xFFFFFFFF,
                                             *[_p(a) for a in arrs], C.byref(out)))
        return self._slots([out.value])[0]

    def download(self, slot: Slot):
        """The slot as a host LeafState."""
        from .arena import LeafState

        o = [np.zeros(slot.n, np.uint32), np.zeros(slot.n + 1, np.uint32), np.zeros(slot.K, np.uint32),
             np.zeros(slot.n, np.uint32), np.zeros(slot.n, np.float64), np.zeros(slot.U, np.uint32),
             np.zeros(slot.U, np.uint8)]
        self.ctx.check(self.L.esat_store_download(self.h, slot.index, *[_p(a) for a in o]))
        return LeafState(*o, slot.root)

    def layout(self, slots, nodes, kids=None) -> dict:
        """Arena bases for a batch of ``slots`` with ``nodes`` spare e-nodes per leaf (an int or one
        per leaf), ``kids`` spare child slots (default 2x nodes) and 1x nodes spare ids, as
        arena.Batch.pack_with_headroom lays them out."""
        L = len(slots)
        nodes = np.broadcast_to(np.asarray(nodes, np.int64), (L,))
        kids = 2 * nodes if kids is None else np.broadcast_to(np.asarray(kids, np.int64), (L,))
        nb, kb, ub = (np.zeros(L + 1, np.uint64) for _ in range(3))
        nb[1:] = np.cumsum([s.n + int(x) for s, x in zip(slots, nodes)])
        kb[1:] = np.cumsum([s.K + int(x) for s, x in zip(slots, kids)])
        ub[1:] = np.cumsum([s.U + int(x) for s, x in zip(slots, nodes)])
        return {"n_leaves": L, "node_base": nb, "kid_base": kb, "id_base": ub,
                "root": np.array([s.root for s in slots], np.uint32),
                "n_cnt": np.array([s.n for s in slots], np.uint32), "u_cnt": np.array([s.U for s in slots], np.uint32),
                "k_cnt": np.array([s.K for s in slots], np.uint32)}

    def load(self, batch: "DeviceBatch", slots):
        if any(s.store != self.id for s in slots):
            raise ValueError("slot of another store")
        idx = _u32([s.index for s in slots])
        batch._slot_keep = idx
        self.ctx.check(self.L.esat_batch_load_slots(batch.h, self.h, _p(idx)))


def available() -> bool:
    try:
        lib()
        Context(int(os.environ.get("ESAT_DEVICE", "0"))).close()
        return True
    except (NativeUnavailable, OSError):
        return False
