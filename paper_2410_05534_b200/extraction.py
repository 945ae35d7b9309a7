"""Greedy extractors with the reference's API (extraction.py), executed by `k_extract`.

`extract_default_greedy` / `extract_ocf_greedy` take a rebuilt e-graph and a
`costs: dict[ENode, float]` exactly like extraction.py:157/229 and return the same
`ExtractionResult` (root cost, chosen e-node per reachable class) or raise the same
exceptions with the same messages (`ExtractionError`, `InfeasibleExtraction`).
"""

from __future__ import annotations

from dataclasses import dataclass

from . import device, native


class ExtractionError(ValueError):
    pass


class InfeasibleExtraction(ExtractionError):
    pass


class CapacityError(ExtractionError):
    pass


@dataclass
class ExtractionResult:
    total_cost: float
    chosen: dict
    method: str

    def to_json_dict(self) -> dict:
        return {"method": self.method, "total_cost": self.total_cost,
                "chosen": {str(c): {"op": n.symbol.name, "payload": repr(n.symbol.payload),
                                    "children": list(n.children)} for c, n in sorted(self.chosen.items())}}


def validate_extraction(egraph, result: ExtractionResult) -> None:
    """Root coverage, child coverage, acyclicity (extraction.py:67-87), host-side check."""
    root = egraph.canonical_root()
    if root not in result.chosen:
        raise ExtractionError("root e-class not chosen")
    state: dict = {}
    stack = [(root, 0)]
    state[root] = 1
    while stack:
        c, i = stack.pop()
        kids = result.chosen[c].children
        if i == len(kids):
            state[c] = 2
            continue
        stack.append((c, i + 1))
        k = egraph.find(kids[i])
        if state.get(k) == 2:
            continue
        if state.get(k) == 1:
            raise ExtractionError(f"cyclic selection through e-class {k}")
        if k not in result.chosen:
            raise ExtractionError(f"child e-class {k} required but not chosen")
        state[k] = 1
        stack.append((k, 0))


def selection_dag_cost(egraph, chosen: dict, costs: dict) -> float:
    """True cost of a selection: every chosen node charged once (extraction.py:90-103)."""
    total, seen, stack = 0.0, set(), [egraph.canonical_root()]
    while stack:
        c = egraph.find(stack.pop())
        if c in seen:
            continue
        seen.add(c)
        total += costs[chosen[c]]
        stack.extend(chosen[c].children)
    return total


_ERR = {
    native.X_NOT_CONVERGED: (ExtractionError, "greedy extraction failed to converge"),
    native.X_INFEASIBLE: (InfeasibleExtraction, "root e-class has no finite-cost program"),
    native.X_CYCLIC: (ExtractionError, "cyclic selection through e-class {}"),
    native.X_CHILD_NOT_CHOSEN: (ExtractionError, "child e-class {} required but not chosen"),
    native.X_ROOT_NOT_CHOSEN: (ExtractionError, "root e-class not chosen"),
    native.X_CAPACITY: (CapacityError, "constituent-history pool exhausted"),
}


def _run(egraph, costs, method: str, name: str) -> ExtractionResult:
    if egraph.dirty:
        raise ExtractionError("extraction requires a rebuilt e-graph")
    if egraph.root is None:
        from .egraph import StructuralError

        raise StructuralError("e-graph has no root")
    st, err, cost, chosen = device.extract(egraph, costs, method)
    if st != native.X_OK:
        exc, msg = _ERR[st]
        raise exc(msg.format(err))
    return ExtractionResult(cost, chosen, name)


def extract_default_greedy(egraph, costs: dict) -> ExtractionResult:
    return _run(egraph, costs, "default", "default_greedy")


def extract_ocf_greedy(egraph, costs: dict) -> ExtractionResult:
    return _run(egraph, costs, "ocf", "ocf_greedy")
