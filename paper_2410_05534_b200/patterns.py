"""Pattern AST, rule DSL parser and the device match-program compiler.

The DSL is the reference's (rewrite.py:1-14, 140-266): s-expressions, ``?var``,
``op[slot,...]`` attribute lists with literal or ``?pvar`` slots, ``|&|``
between the sources/targets of a multi-pattern rule, ``#`` comments. The AST
types mirror rewrite.py:43-65 (``Var``/``PVar``/``App``) and ``Rule``
(rewrite.py:101-129); errors mirror ``RuleSyntaxError``/``UnboundVariableError``
(rewrite.py:25-33) including line/column reporting.

``compile_pattern`` lowers one pattern to the flat int32 program the CPU oracle
and the CUDA matcher both execute (include/esat_b200.h, "pattern program").
"""

from __future__ import annotations

import re
from dataclasses import dataclass
from typing import Optional, Union

import numpy as np


class RuleSyntaxError(ValueError):
    def __init__(self, message: str, line: int = 1, col: int = 1) -> None:
        super().__init__(f"{message} (line {line}, col {col})")
        self.line = line
        self.col = col


class UnboundVariableError(ValueError):
    pass


@dataclass(frozen=True)
class Var:
    name: str


@dataclass(frozen=True)
class PVar:
    name: str


ParamSlot = Union[int, str, PVar]


@dataclass(frozen=True)
class App:
    name: str
    params: Optional[tuple]
    children: tuple


Pattern = Union[Var, App]


def _is_var(p) -> bool:
    return type(p).__name__ == "Var"


def _is_pvar(p) -> bool:
    return type(p).__name__ == "PVar"


def pattern_vars(pat) -> set:
    if _is_var(pat):
        return {pat.name}
    acc: set = set()
    for c in pat.children:
        acc |= pattern_vars(c)
    return acc


def pattern_pvars(pat) -> set:
    if _is_var(pat):
        return set()
    acc = {s.name for s in (pat.params or ()) if _is_pvar(s)}
    for c in pat.children:
        acc |= pattern_pvars(c)
    return acc


def print_pattern(pat) -> str:
    if _is_var(pat):
        return "?" + pat.name
    head = pat.name
    if pat.params is not None:
        head += "[" + ",".join("?" + s.name if _is_pvar(s) else str(s) for s in pat.params) + "]"
    if not pat.children:
        return head
    return "(" + " ".join([head] + [print_pattern(c) for c in pat.children]) + ")"


@dataclass
class Rule:
    id: int
    name: str
    sources: list
    targets: list

    @property
    def kind(self) -> str:
        return "single" if len(self.sources) < 2 else "multi"

    def __post_init__(self) -> None:
        if not self.sources:
            raise UnboundVariableError("rule has no source pattern")
        if len(self.sources) != len(self.targets):
            raise RuleSyntaxError("source/target pattern counts differ")
        vs = set().union(*map(pattern_vars, self.sources))
        ps = set().union(*map(pattern_pvars, self.sources))
        for t in self.targets:
            free = pattern_vars(t) - vs
            if free:
                raise UnboundVariableError(f"target variables not bound by any source: {sorted(free)}")
            free_p = pattern_pvars(t) - ps
            if free_p:
                raise UnboundVariableError(
                    f"target attribute variables not bound by any source: {sorted(free_p)}")


def print_rule(rule: Rule) -> str:
    return (" |&| ".join(map(print_pattern, rule.sources)) + " => "
            + " |&| ".join(map(print_pattern, rule.targets)))


_INT = re.compile(r"-?\d+")
_ATOM = re.compile(r"[^\s()]+")


def _lex(text: str, line: int):
    i, n = 0, len(text)
    while i < n:
        ch = text[i]
        if ch == " " or ch == "\t":
            i += 1
        elif ch == "(" or ch == ")":
            yield ch, line, i + 1
            i += 1
        else:
            m = _ATOM.match(text, i)
            yield m.group(0), line, i + 1
            i = m.end()


def _atom(tok: str, line: int, col: int):
    if tok[0] == "?":
        if len(tok) == 1:
            raise RuleSyntaxError("empty variable name", line, col)
        return tok[1:], None, True
    name, params = tok, None
    if "[" in tok:
        if tok[-1] != "]":
            raise RuleSyntaxError(f"malformed attribute list in {tok!r}", line, col)
        name, body = tok[:-1].split("[", 1)
        slots = []
        for raw in body.split(","):
            s = raw.strip()
            if not s:
                raise RuleSyntaxError(f"empty attribute slot in {tok!r}", line, col)
            slots.append(PVar(s[1:]) if s[0] == "?" else int(s) if _INT.fullmatch(s) else s)
        params = tuple(slots)
    if not name:
        raise RuleSyntaxError(f"missing operator name in {tok!r}", line, col)
    return name, params, False


def parse_pattern(text: str, line: int = 1):
    toks = list(_lex(text, line))
    at = [0]

    def expr():
        if at[0] >= len(toks):
            raise RuleSyntaxError("unexpected end of pattern", line, len(text) + 1)
        tok, ln, col = toks[at[0]]
        at[0] += 1
        if tok == ")":
            raise RuleSyntaxError("unexpected ')'", ln, col)
        if tok != "(":
            name, params, is_var = _atom(tok, ln, col)
            return Var(name) if is_var else App(name, params, ())
        if at[0] >= len(toks):
            raise RuleSyntaxError("unterminated '('", ln, col)
        head, hl, hc = toks[at[0]]
        at[0] += 1
        if head in ("(", ")"):
            raise RuleSyntaxError("expected operator after '('", hl, hc)
        name, params, is_var = _atom(head, hl, hc)
        if is_var:
            raise RuleSyntaxError("variable cannot head an application", hl, hc)
        kids = []
        while True:
            if at[0] >= len(toks):
                raise RuleSyntaxError("unterminated '('", ln, col)
            if toks[at[0]][0] == ")":
                at[0] += 1
                return App(name, params, tuple(kids))
            kids.append(expr())

    out = expr()
    if at[0] != len(toks):
        tok, ln, col = toks[at[0]]
        raise RuleSyntaxError(f"trailing input {tok!r}", ln, col)
    return out


def parse_rule(text: str, rule_id: int = 0, line: int = 1) -> Rule:
    body = text.split("#", 1)[0].strip()
    if "=>" not in body:
        raise RuleSyntaxError("missing '=>'", line, 1)
    lhs, rhs = body.split("=>", 1)
    rule = Rule(rule_id, "",
                [parse_pattern(p.strip(), line) for p in lhs.split("|&|")],
                [parse_pattern(p.strip(), line) for p in rhs.split("|&|")])
    rule.name = print_rule(rule)
    return rule


def parse_rules(text: str) -> list:
    out = []
    for ln, raw in enumerate(text.splitlines(), start=1):
        body = raw.split("#", 1)[0].strip()
        if body:
            out.append(parse_rule(body, rule_id=len(out), line=ln))
    return out


def load_rules(path_or_name: str) -> list:
    """Rules from a path or a bundled set name (``taso_analog``, ``toy_math``)."""
    from pathlib import Path

    p = Path(path_or_name)
    if p.exists():
        return parse_rules(p.read_text())
    bundled = Path(__file__).parent / "rules" / f"{path_or_name}.rules"
    if bundled.is_file():
        return parse_rules(bundled.read_text())
    raise FileNotFoundError(f"no rule file or bundled rule set named {path_or_name!r}")


# -- device match programs ----------------------------------------------------

PN_VAR, PN_APP = 0, 1
REC = 6  # words per pattern-node record


@dataclass
class CompiledPattern:
    program: np.ndarray          # int32 words (format in include/esat_b200.h)
    var_names: list              # sorted; var index i <-> var_names[i]
    pvar_names: list             # sorted; pvar index q <-> pvar_names[q]


def compile_pattern(pat, name_id, code) -> CompiledPattern:
    """Lower a pattern tree to the pre-order int32 program.

    ``name_id(name)`` -> interned operator name id (or -1 if never interned);
    ``code(value)`` -> order-preserving attribute code (symtab.NO_MATCH_CODE if absent).
    Var/pvar indices follow sorted names, so a match's binding arrays are already
    in the order ``_subst_key`` sorts them (rewrite.py:396-397).
    """
    vnames = sorted(pattern_vars(pat))
    qnames = sorted(pattern_pvars(pat))
    vidx = {v: i for i, v in enumerate(vnames)}
    qidx = {q: i for i, q in enumerate(qnames)}
    index: dict = {}   # pre-order position -> positions of its children
    order: list = []

    def walk2(p):
        order.append(p)
        my = len(order) - 1
        kids = []
        if not _is_var(p):
            for c in p.children:
                kids.append(walk2(c))
        index[my] = kids
        return my

    walk2(pat)
    P = len(order)
    recs = np.zeros((P, REC), np.int32)
    slots: list = []
    childw: list = []
    for i, p in enumerate(order):
        if _is_var(p):
            recs[i] = (PN_VAR, vidx[p.name], 0, -1, 0, 0)
            continue
        nslots = -1 if p.params is None else len(p.params)
        sbase = len(slots)
        for s in p.params or ():
            slots.append(-(qidx[s.name] + 1) if _is_pvar(s) else code(s))
        cbase = len(childw)
        childw.extend(index[i])
        recs[i] = (PN_APP, name_id(p.name), len(p.children), nslots, sbase, cbase)
    head = np.array([P, len(vnames), len(qnames)], np.int32)
    base = 3 + REC * P
    recs[:, 4] += base
    recs[:, 5] += base + len(slots)
    for i, p in enumerate(order):
        if _is_var(p):
            recs[i, 4] = 0
            recs[i, 5] = 0
    prog = np.concatenate([head, recs.reshape(-1), np.array(slots, np.int32),
                           np.array(childw, np.int32)]).astype(np.int32)
    return CompiledPattern(prog, vnames, qnames)
