"""Host side of the device apply loop (reference rewrite.py:460-573).

Compiles rule targets into flat instruction programs for ``k_apply`` and builds the symbol
lookup the device needs to reproduce ``Language.make_symbol`` (rewrite.py:296-298 for terms,
tensor_ir.py:253-265 for tensors) without Python objects:

* ``symbol_key_words`` -- the identity of a symbol as u32 words
  ``[name_id, arity, n_params, param codes..., ndim, dims...]`` (``ndim`` 255 = no shape).
  Two symbols are equal (egraph.py:34-48 dataclass equality on name, arity, payload) iff
  their key words are equal: params are order-preserving codes of the payload attributes and
  the shape is the payload's second half (tensor symbols) -- term symbols' payload is a
  function of the name.
* ``key_hash`` -- the hash the device recomputes (32-bit FNV-1a over the key words).
* a per-code integer table so shape inference can read attribute values (stride, axis, ...).

Target program (int32 words), per rule::

    [from_join, list_index, W, S, NV, NQ, NT, toff_0 .. toff_{NT-1}]   toff relative to rule start
    target: [n_instr, n_instr x INSTR words]

instruction (INSTR = 20 words)::

    0 kind (0 var, 1 app)        1 var: record word of the binding | app: operator name id (-1 unknown)
    2 op enum (tensor ops)       3 arity      4 n_params (-1: params None)
    5..8 child instruction indices (post-order, children before parents)
    9 + 3p .. 11 + 3p  param p: tag (0 literal with a code, 1 pvar, 2 literal absent from the
                        symbol table), code or record word, int value (INT_NONE for strings)
    18 name is an integer literal (term symbols carry int(name) as payload)
"""

from __future__ import annotations

import ast
import re

import numpy as np

from .patterns import _is_pvar, _is_var, pattern_pvars, pattern_vars
from .symtab import NO_MATCH_CODE

INSTR = 20
OPS = ["?", "input", "weight", "ewadd", "ewmul", "matmul", "conv2d", "relu", "tanh", "sigmoid", "concat",
       "split", "maxpool", "transpose", "noop"]
OP_ID = {n: i for i, n in enumerate(OPS)}
INT_NONE = -(2 ** 31)
NO_SHAPE = 255
LANG_TERM, LANG_TENSOR = 0, 1
COST_TERM, COST_UNIT, COST_ANALYTIC = 0, 1, 2


def key_hash(words) -> int:
    """Word-wise FNV-1a over the key words (k_apply's sym_lookup computes the same)."""
    h = 2166136261
    for w in words:
        h = ((h ^ (int(w) & 0xFFFFFFFF)) * 16777619) & 0xFFFFFFFF
    return h


def payload_shape(payload):
    """Shape half of a tensor payload ``(params, shape)``; None for term payloads."""
    if isinstance(payload, tuple) and len(payload) == 2 and isinstance(payload[1], tuple):
        return payload[1]
    return None


def symbol_key_words(name_id: int, arity: int, codes, shape) -> list:
    w = [int(name_id) & 0xFFFFFFFF, int(arity), len(codes), *[int(c) & 0xFFFFFFFF for c in codes]]
    if shape is None:
        w.append(NO_SHAPE)
    else:
        w.append(len(shape))
        w.extend(int(d) for d in shape)
    return w


def symbol_arrays(names, arities, payloads, param_codes, values) -> dict:
    """Device arrays for symbol lookup + shapes.

    ``payloads[i]`` is the symbol payload (a Python object, or its repr string as stored in
    golden files); ``param_codes[i]`` the codes of ``language.node_params(symbol)``."""
    n = len(names)
    ndim = np.full(n, NO_SHAPE, np.uint8)
    dims = np.zeros((n, 4), np.uint32)
    keys = []
    for i in range(n):
        p = payloads[i]
        if isinstance(p, str):
            p = ast.literal_eval(p)
        shp = payload_shape(p)
        if shp is not None:
            ndim[i] = len(shp)
            dims[i, :len(shp)] = shp
        keys.append(symbol_key_words(names[i], arities[i], param_codes[i], shp))
    size = 1
    while size < 2 * max(n, 1):
        size <<= 1
    table = np.full(size, 0xFFFFFFFF, np.uint32)
    for i, k in enumerate(keys):
        s = key_hash(k) & (size - 1)
        while table[s] != 0xFFFFFFFF:
            s = (s + 1) & (size - 1)
        table[s] = i
    vint = np.array([v if isinstance(v, int) and not isinstance(v, bool) and -2 ** 31 < v < 2 ** 31 else INT_NONE
                     for v in values] or [INT_NONE], np.int32)
    return {"ndim": ndim, "dims": dims.reshape(-1), "table": table, "vint": vint}


def symtab_symbol_arrays(symtab) -> dict:
    """symbol_arrays for a live symtab.SymbolTable."""
    symtab.finalize()
    names = [symtab._name_index[s.name] for s in symtab.symbols]
    arities = [s.arity for s in symtab.symbols]
    payloads = [s.payload for s in symtab.symbols]
    codes = [[symtab._codes[(type(v), v)] for v in ps] for ps in symtab.params]
    return symbol_arrays(names, arities, payloads, codes, symtab.values)


def compile_rule_targets(rule, name_id, code, value_of_code, from_join: int, list_index: int) -> np.ndarray:
    """Lower ``rule.targets`` (rewrite.py:526-570) for k_apply.

    The match record of the rule is ``[S roots][vars sorted by name][pvar codes sorted by name]``
    (the joint_match key order, rewrite.py:396-397), so a Var is a record word and a PVar a code
    word."""
    S = len(rule.sources)
    vnames = sorted(set().union(*map(pattern_vars, rule.sources)))
    qnames = sorted(set().union(*map(pattern_pvars, rule.sources)))
    vslot = {v: S + i for i, v in enumerate(vnames)}
    qslot = {q: S + len(vnames) + i for i, q in enumerate(qnames)}
    progs = []
    for t in rule.targets:
        instrs = []

        def emit(p):
            if _is_var(p):
                rec = [0, vslot[p.name]] + [0] * (INSTR - 2)
                instrs.append(rec)
                return len(instrs) - 1
            kids = [emit(c) for c in p.children]
            if len(kids) > 4:
                raise ValueError("target operator arity > 4 is not supported by k_apply")
            rec = [0] * INSTR
            rec[0] = 1
            rec[1] = name_id(p.name)
            rec[2] = OP_ID.get(p.name, 0)
            rec[3] = len(kids)
            rec[4] = -1 if p.params is None else len(p.params)
            if p.params is not None and len(p.params) > 3:
                raise ValueError("more than 3 attributes per target operator")
            for j, k in enumerate(kids):
                rec[5 + j] = k
            for j, s in enumerate(p.params or ()):
                if _is_pvar(s):
                    rec[9 + 3 * j: 12 + 3 * j] = [1, qslot[s.name], 0]
                else:
                    c = code(s)
                    iv = s if isinstance(s, int) and not isinstance(s, bool) else INT_NONE
                    rec[9 + 3 * j: 12 + 3 * j] = [2 if c == NO_MATCH_CODE else 0, c if c != NO_MATCH_CODE else 0,
                                                  iv]
            rec[18] = 1 if re.fullmatch(r"-?\d+", p.name) else 0
            instrs.append(rec)
            return len(instrs) - 1

        emit(t)
        progs.append([len(instrs)] + [w for r in instrs for w in r])
    W = S + len(vnames) + len(qnames)
    head = [from_join, list_index, W, S, len(vnames), len(qnames), len(progs)]
    off = len(head) + len(progs)
    toffs = []
    for p in progs:
        toffs.append(off)
        off += len(p)
    words = head + toffs + [w for p in progs for w in p]
    return np.array(words, np.int64).astype(np.int32)


def pack_rules(programs: list) -> tuple:
    """Concatenate per-rule programs: (offsets u32[R+1], words i32)."""
    off = np.zeros(len(programs) + 1, np.uint32)
    for i, p in enumerate(programs):
        off[i + 1] = off[i] + len(p)
    words = np.concatenate(programs).astype(np.int32) if programs else np.zeros(1, np.int32)
    return off, words


class ApplyDriver:
    """Runs esat_apply over a LeafPipeline's batch with a live symbol table.

    A leaf whose instantiation needs an operator symbol the table has never seen stops with
    ESAT_A_NEED_SYMBOL and a descriptor of it; the driver interns those symbols here (exactly the
    Symbol TensorLanguage/TermLanguage.make_symbol would have built), re-uploads the table, the
    pattern and target programs (attribute codes are order-preserving, so they move), re-matches
    on the unchanged rebuilt view and re-applies -- the rebuilt state is still intact on the device."""

    def __init__(self, pipe, symtab, language, cost_config=None, symbol_cls=None):
        from .cost_model import CostModelConfig
        from .egraph import Symbol

        self.pipe, self.symtab, self.language = pipe, symtab, language
        self.symbol_cls = symbol_cls or Symbol   # the caller's Symbol class (ours or the reference's)
        cfg = cost_config or CostModelConfig()
        # tensor symbols carry (attributes, shape) payloads (tensor_ir.py:243-265); duck-typed so the
        # reference's own language objects work too
        self.lang = LANG_TENSOR if type(language).__name__ == "TensorLanguage" else LANG_TERM
        self.cost_mode = {"term": COST_TERM, "unit": COST_UNIT, "analytic": COST_ANALYTIC}[cfg.mode]
        self.coeff = float(cfg.coefficient)
        self.interned = 0
        self.upload()

    def _name_id(self, name):
        return self.symtab.name_id(name, create=False)

    def upload(self):
        st = self.symtab
        st.finalize()
        self.uploaded_symbols = len(st)
        self.pipe.ctx.upload_symtab(st.arrays())
        self.pipe.recompile(self._name_id, st.code)
        off, words = self.pipe.apply_programs(self._name_id, st.code)
        self.pipe.ctx.apply_setup(self.lang, self.cost_mode, self.coeff, symtab_symbol_arrays(st), off, words)

    def _target_node(self, rule_idx: int, t: int, i: int):
        order = []

        def walk(p):
            if not _is_var(p):
                for c in p.children:
                    walk(c)
            order.append(p)

        walk(self.pipe.rules[rule_idx].rule.targets[t])
        return order[i]

    def _intern(self, desc):
        Symbol = self.symbol_cls  # noqa: N806
        p = self._target_node(int(desc[14]), int(desc[15]) >> 8, int(desc[15]) & 0xFF)
        arity = int(desc[1])
        if self.lang == LANG_TERM:
            payload = int(p.name) if re.fullmatch(r"-?\d+", p.name) else None
        else:
            params = []
            for j, s in enumerate(p.params or ()):
                params.append(self.symtab.values[int(desc[3 + j])] if _is_pvar(s) else s)
            nd = int(desc[9])
            shape = None if nd == NO_SHAPE else tuple(int(x) for x in desc[10:10 + nd])
            payload = (tuple(params), shape)
        before = len(self.symtab)
        self.symtab.intern(Symbol(p.name, arity, payload), self.language)
        self.interned += len(self.symtab) - before

    def apply(self, leaf_rule, node_limit: int = 0, max_rounds: int = 256, leaf_mask=None) -> dict:
        """esat_apply of leaf_rule[l] on every leaf over the match lists of the last e-match (made
        with ``leaf_mask`` when given: the same mask is used to re-match after interning)."""
        from . import native

        b = self.pipe.batch
        for _ in range(max_rounds):
            b.apply(leaf_rule, node_limit)
            res = b.download_apply()
            need = np.nonzero(res["status"] == native.A_NEED_SYMBOL)[0]
            if need.size == 0:
                return res
            before = len(self.symtab)
            for l in need:
                self._intern(res["missing"][l])
            if len(self.symtab) == before:
                raise RuntimeError("device asked for symbols that are already interned")
            self.upload()
            self.pipe.ematch(leaf_mask)   # codes moved: re-derive the match records on the same view
        raise RuntimeError("symbol interning did not converge")
