"""Frozen desk-scale analogs of the five BASELINE.json model graphs.

The reference ships only ``resblock_stack``/``mlp``/``attention_block``/
``inception_cell``/``toy_expr`` (tensor_ir.py:406-481) and deliberately scopes the
13 full-scale architectures out. The BASELINE configs name BERT,
NasRNN, ResNeXt-50, Inception-v3 and NasNet-A, so this module defines analogs of
their characteristic structure inside the 14-operator IR (tensor_ir.py:32-47):

* ``bert``        -- attention + FFN layers with residual adds (sharing => default
                     greedy over-counts, OCF exact; PAPER.md:289-292 pattern)
* ``nasrnn``      -- an 8-gate recurrent cell unrolled over time; every gate
                     multiplies the same x_t / h_{t-1} (fuel for the #128 analog rule)
* ``resnext50``   -- bottleneck blocks whose grouped 3x3 conv is emulated by nested
                     split / concat of conv2d (the IR has no grouped conv)
* ``inception_v3``-- modules of parallel conv / maxpool branches joined by concat
* ``nasnet_a``    -- cells combining the two previous cell outputs through nested,
                     shared branches (the Fig. 8 overlap that makes OCF overestimate)

Every generator takes a builder object with the reference ``GraphBuilder``
interface (``input``/``weight``/``op``/``build``, tensor_ir.py:212-238) so that the
golden-vector script can drive the *reference* builder with the very same code.
The functions are frozen: tests/golden/ was generated from them.
"""

from __future__ import annotations

from typing import Callable


def bert(b, layers: int = 2, seq: int = 64, d: int = 256):
    x = b.input("x", (seq, d))
    for i in range(layers):
        wq = b.weight(f"l{i}_wq", (d, d))
        wk = b.weight(f"l{i}_wk", (d, d))
        wv = b.weight(f"l{i}_wv", (d, d))
        wo = b.weight(f"l{i}_wo", (d, d))
        q = b.op("matmul", x, wq)
        k = b.op("matmul", x, wk)
        v = b.op("matmul", x, wv)
        scores = b.op("sigmoid", b.op("matmul", q, b.op("transpose", k)))
        ctx = b.op("matmul", scores, v)
        att = b.op("ewadd", x, b.op("matmul", ctx, wo))
        w1 = b.weight(f"l{i}_w1", (d, 4 * d))
        w2 = b.weight(f"l{i}_w2", (4 * d, d))
        ffn = b.op("matmul", b.op("relu", b.op("matmul", att, w1)), w2)
        x = b.op("ewadd", att, ffn)
    return b.build(x)


def nasrnn(b, steps: int = 4, hidden: int = 512, batch: int = 1):
    gates = 8
    w = [b.weight(f"w{g}", (hidden, hidden)) for g in range(gates)]
    u = [b.weight(f"u{g}", (hidden, hidden)) for g in range(gates)]
    h = b.input("h0", (batch, hidden))
    acts = ("sigmoid", "tanh", "relu", "sigmoid", "tanh", "relu", "sigmoid", "tanh")
    for t in range(steps):
        x = b.input(f"x{t}", (batch, hidden))
        g = [
            b.op(acts[i], b.op("ewadd", b.op("matmul", x, w[i]), b.op("matmul", h, u[i])))
            for i in range(gates)
        ]
        l1 = [b.op("ewmul", g[0], g[1]), b.op("ewadd", g[2], g[3]),
              b.op("ewmul", g[4], g[5]), b.op("ewadd", g[6], g[7])]
        l2 = [b.op("tanh", b.op("ewmul", l1[0], l1[1])),
              b.op("sigmoid", b.op("ewadd", l1[2], l1[3]))]
        h = b.op("ewmul", l2[0], l2[1])
    return b.build(h)


def _grouped_conv(b, x, cin: int, cout: int, depth: int, tag: str, hw: int = 3):
    """Grouped 3x3 conv as a binary tree of channel splits, one conv per leaf group."""
    if depth == 0:
        w = b.weight(f"{tag}_w", (cout, cin, hw, hw))
        return b.op("conv2d", x, w, stride=1, padding=hw // 2, activation="none")
    lo = _grouped_conv(b, b.op("split", x, axis=1, index=0), cin // 2, cout // 2, depth - 1, tag + "0", hw)
    hi = _grouped_conv(b, b.op("split", x, axis=1, index=1), cin // 2, cout // 2, depth - 1, tag + "1", hw)
    return b.op("concat", lo, hi, axis=1)


def resnext50(b, blocks: int = 4, channels: int = 64, width: int = 32, spatial: int = 14,
              cardinality_depth: int = 2):
    x = b.input("x", (1, channels, spatial, spatial))
    stem = b.weight("stem_w", (channels, channels, 3, 3))
    x = b.op("relu", b.op("conv2d", x, stem, stride=1, padding=1, activation="none"))
    for i in range(blocks):
        w_in = b.weight(f"b{i}_in", (width, channels, 1, 1))
        w_out = b.weight(f"b{i}_out", (channels, width, 1, 1))
        h = b.op("relu", b.op("conv2d", x, w_in, stride=1, padding=0, activation="none"))
        h = b.op("relu", _grouped_conv(b, h, width, width, cardinality_depth, f"b{i}_g"))
        h = b.op("conv2d", h, w_out, stride=1, padding=0, activation="none")
        x = b.op("relu", b.op("ewadd", x, h))
    return b.build(x)


def inception_v3(b, modules: int = 3, channels: int = 32, spatial: int = 17):
    x = b.input("x", (1, channels, spatial, spatial))
    for m in range(modules):
        br = channels // 4
        w1 = b.weight(f"m{m}_1x1", (br, channels, 1, 1))
        b1 = b.op("conv2d", x, w1, stride=1, padding=0, activation="none")
        w2a = b.weight(f"m{m}_3a", (br, channels, 1, 1))
        w2b = b.weight(f"m{m}_3b", (br, br, 3, 3))
        b2 = b.op("conv2d", b.op("relu", b.op("conv2d", x, w2a, stride=1, padding=0, activation="none")),
                  w2b, stride=1, padding=1, activation="none")
        w3a = b.weight(f"m{m}_5a", (br, channels, 1, 1))
        w3b = b.weight(f"m{m}_5b", (br, br, 3, 3))
        w3c = b.weight(f"m{m}_5c", (br, br, 3, 3))
        b3 = b.op("relu", b.op("conv2d", x, w3a, stride=1, padding=0, activation="none"))
        b3 = b.op("relu", b.op("conv2d", b3, w3b, stride=1, padding=1, activation="none"))
        b3 = b.op("conv2d", b3, w3c, stride=1, padding=1, activation="none")
        w4 = b.weight(f"m{m}_pool", (br, channels, 3, 3))
        b4 = b.op("conv2d", b.op("maxpool", x, kernel=3, stride=1), w4, stride=1, padding=2,
                  activation="none")
        cat = b.op("concat", b.op("concat", b1, b2, axis=1), b.op("concat", b3, b4, axis=1), axis=1)
        x = b.op("relu", cat)
    return b.build(x)


def nasnet_a(b, cells: int = 3, channels: int = 16, spatial: int = 16):
    shape = (1, channels, spatial, spatial)
    prev2 = b.input("x0", shape)
    prev = b.input("x1", shape)

    def sep(inp, tag, k):
        w = b.weight(tag, (channels, channels, k, k))
        return b.op("conv2d", b.op("relu", inp), w, stride=1, padding=k // 2, activation="none")

    for c in range(cells):
        # five NASNet-A blocks; h0 = prev, h1 = prev2 are each consumed several times
        s0 = b.op("ewadd", sep(prev, f"c{c}_s0a", 3), sep(prev2, f"c{c}_s0b", 5))
        s1 = b.op("ewadd", sep(prev2, f"c{c}_s1a", 3), sep(prev2, f"c{c}_s1b", 5))
        s2 = b.op("ewadd", sep(prev, f"c{c}_s2a", 3), prev2)
        s3 = b.op("ewadd", sep(s0, f"c{c}_s3a", 3), s1)          # nested reuse of s0/s1
        s4 = b.op("ewadd", sep(s0, f"c{c}_s4a", 5), s2)
        cat = b.op("concat", b.op("concat", s1, s3, axis=1), b.op("concat", s2, s4, axis=1), axis=1)
        w_red = b.weight(f"c{c}_reduce", (channels, 4 * channels, 1, 1))
        out = b.op("conv2d", cat, w_red, stride=1, padding=0, activation="none")
        prev2, prev = prev, out
    return b.build(prev)


ANALOGS: dict[str, Callable] = {
    "bert": bert,
    "nasrnn": nasrnn,
    "resnext50": resnext50,
    "inception_v3": inception_v3,
    "nasnet_a": nasnet_a,
}


def build_analog(name: str, builder_factory, **kwargs):
    """Build analog `name` with a fresh builder from `builder_factory()`."""
    return ANALOGS[name](builder_factory(), **kwargs)
