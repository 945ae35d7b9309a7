"""Rewrite engine with the reference's API (rewrite.py); matching runs on the B200.

`ematch`, `joint_match` and `is_rule_applicable` execute `k_ematch`/`k_join` through
`device.py` and return the reference's ordered, deduplicated `Substitution` list
(rewrite.py:396-433). `apply_rule` runs the reference's sequential instantiate / cycle-filter /
shape-filter / union loop (rewrite.py:526-573) on the device (`k_apply`, with host interning of
new operator symbols) and ends with the device rebuild; `would_create_cycle` stays here as the
host statement of the cycle test `k_apply` answers.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import device
from .egraph import EGraph, StructuralError
from .patterns import (App, PVar, Rule, RuleSyntaxError, UnboundVariableError, Var, load_rules,  # noqa: F401
                       parse_pattern, parse_rule, parse_rules, pattern_pvars, pattern_vars, print_pattern,
                       print_rule)
from .tensor_ir import InstantiationError, Language, TermLanguage  # noqa: F401

_TERM = TermLanguage()


def _lang(egraph, language):
    return language or egraph.language or _TERM


@dataclass(frozen=True)
class Substitution:
    vars: tuple
    params: tuple
    roots: tuple = ()

    def var(self, name: str) -> int:
        return dict(self.vars)[name]

    def param(self, name: str):
        return dict(self.params)[name]


def joint_match(egraph: EGraph, patterns: list, language=None) -> list:
    """All substitutions of `patterns` (threaded bindings), sorted by (roots, vars, params)."""
    if egraph.dirty:
        raise StructuralError("ematch requires a rebuilt e-graph")
    recs, vn, qn, S = device.joint_match(egraph, list(patterns), language)
    values = device.session().symtab.values
    nv = len(vn)
    out = []
    for r in recs.tolist():
        out.append(Substitution(tuple(zip(vn, r[S:S + nv])),
                                tuple((q, values[c]) for q, c in zip(qn, r[S + nv:])), tuple(r[:S])))
    return out


def ematch(egraph: EGraph, pattern, language=None) -> list:
    return joint_match(egraph, [pattern], language)


def is_rule_applicable(egraph: EGraph, rule: Rule, language=None) -> bool:
    """False guarantees apply_rule reports changed=False (rewrite.py:579-589): EXISTS-mode
    e-match of every source independently."""
    if egraph.dirty:
        raise StructuralError("ematch requires a rebuilt e-graph")
    return all(device.any_match(egraph, s) for s in rule.sources)


@dataclass
class ApplyReport:
    rule_id: int
    matches_found: int = 0
    changed: bool = False
    nodes_after: int = 0
    classes_after: int = 0
    hit_node_limit: bool = False
    cycles_filtered: int = 0
    shape_filtered: int = 0


def would_create_cycle(egraph: EGraph, children, matched_root: int) -> bool:
    """True iff matched_root is reachable from any candidate child (rewrite.py:488-505)."""
    goal = egraph.find(matched_root)
    todo = [egraph.find(c) for c in children]
    seen = set()
    while todo:
        c = todo.pop()
        if c == goal:
            return True
        if c in seen:
            continue
        seen.add(c)
        for node in egraph.classes[c].nodes:
            todo.extend(egraph.find(x) for x in node.children)
    return False


def apply_rule(egraph: EGraph, rule: Rule, node_limit: int = 0, language=None) -> ApplyReport:
    """Apply every match of `rule`, union targets with matched classes, rebuild (rewrite.py:526-573).

    Runs on the device (device.apply_rule: k_ematch/k_join -> k_apply -> k_rebuild); the
    helpers above (_refs, would_create_cycle, _shape, _instantiate) are the host restatement of
    the same steps, kept as the reference's public helpers."""
    from . import device

    return device.apply_rule(egraph, rule, node_limit, _lang(egraph, language))


def is_saturated(egraph: EGraph, rules: list, node_limit: int = 0, language=None) -> bool:
    for r in rules:
        if apply_rule(egraph.snapshot(), r, 0, language).changed:
            return False
    return True
