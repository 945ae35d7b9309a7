"""Analytic operator cost model (restated from SPEC.md:378-437; absent from the reference code).

The reference extraction consumes ``costs: dict[ENode, float]`` (extraction.py:43)
but ships no producer; SPEC's cost-model module defines it:

* analytic mode: ``coefficient x FLOP-estimate``, FLOPs per
  SPEC.md:422 -- matmul ``2MKN``; conv2d ``2*N*C*KH*KW*OH*OW*O``; element-wise,
  activation, concat, split, transpose = output element count. maxpool is not
  listed by SPEC; it is charged ``output elements * kernel^2`` (window reads).
  ``input``/``weight``/``noop`` cost 0.
* unit mode: 1.0 per operator, 0.0 for input/weight/noop.
* ``term`` mode (toy TermLanguage graphs): AST size, 1.0 per node (SPEC AC-1).
* noise is fixed at 0 (SPEC.md:423 allows frozen Gaussian noise; 0 keeps the
  model a pure function, so CPU oracle and device consume identical f64 tables).

Costs are f64 and depend only on (symbol, child-class shapes), so the host
computes one value per e-node at creation and the device carries it through
rebuild.
"""

from __future__ import annotations

from dataclasses import dataclass
from math import prod

LEAF_OPS = ("input", "weight", "noop")


@dataclass(frozen=True)
class CostModelConfig:
    mode: str = "analytic"          # analytic | unit | term
    coefficient: float = 1e-9       # cost per FLOP (SPEC.md example: 1e-9)
    noise_stddev: float = 0.0       # only 0 is supported (deterministic parity)

    def __post_init__(self):
        if self.mode not in ("analytic", "unit", "term"):
            raise ValueError(f"unknown cost mode {self.mode!r}")
        if self.noise_stddev != 0.0:
            raise ValueError("noise_stddev must be 0 (bit-exact parity contract)")


def flop_estimate(op: str, params: tuple, out_shape, in_shapes) -> float:
    if op in LEAF_OPS:
        return 0.0
    if op == "matmul":
        (m, k), (_, n) = in_shapes
        return 2.0 * m * k * n
    if op == "conv2d":
        x, w = in_shapes
        o, c, kh, kw = w
        n, _, oh, ow = out_shape
        return 2.0 * n * c * kh * kw * oh * ow * o
    if op == "maxpool":
        k = int(params[0])
        return float(prod(out_shape) * k * k)
    return float(prod(out_shape))


def operator_cost(config: CostModelConfig, op: str, params: tuple, out_shape, in_shapes) -> float:
    if config.mode == "term":
        return 1.0
    if config.mode == "unit":
        return 0.0 if op in LEAF_OPS else 1.0
    return config.coefficient * flop_estimate(op, params, out_shape, in_shapes)


def node_cost(config: CostModelConfig, symbol, child_shapes) -> float:
    """Cost of one e-node given its symbol and its children's class shapes."""
    if config.mode == "term":
        return 1.0
    payload = symbol.payload
    params, shape = payload if isinstance(payload, tuple) and len(payload) == 2 else ((), None)
    return operator_cost(config, symbol.name, params, shape, child_shapes)


def egraph_costs(egraph, config: CostModelConfig) -> dict:
    """``costs`` dict for every canonical e-node of a rebuilt e-graph (extraction.py:43)."""
    out = {}
    shape_of = {}
    term = config.mode == "term"
    for cid, cls in egraph.classes.items():
        for node in cls.nodes:
            shape_of[cid] = None if term else node.symbol.payload[1]
            break
    for cid, cls in egraph.classes.items():
        for node in cls.nodes:
            shapes = tuple(shape_of[egraph.find(c)] for c in node.children)
            out[node] = node_cost(config, node.symbol, shapes)
    return out
