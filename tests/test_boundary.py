"""CPU-side checks of the drop-in boundary: the C-ABI library loads and exports every
symbol include/esat_b200.h declares; host format helpers round-trip; no CPU fallback."""

import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


def test_header_symbols_exported():
    from paper_2410_05534_b200 import native

    header = (ROOT / "include" / "esat_b200.h").read_text()
    declared = set(re.findall(r"^(?:int|uint32_t|const char\*|float)\s+(esat_\w+)\(", header, re.M))
    assert declared, "no declarations parsed"
    lib = native.lib()  # loads the sm_100a .so (no GPU needed to dlopen)
    missing = sorted(s for s in declared if not hasattr(lib, s))
    assert not missing, missing
    assert declared == set(native.EXPORTED)


def test_no_cpu_fallback_without_gpu():
    """Without a usable B200 the product path must fail loudly, never fall back to the oracle."""
    import torch

    from paper_2410_05534_b200 import native

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(native.NativeUnavailable):
        native.Context(0)


def test_product_package_never_imports_oracle():
    pkg = ROOT / "paper_2410_05534_b200"
    for f in pkg.rglob("*.py"):
        src = f.read_text()
        assert "import oracle" not in src and "from oracle" not in src, f


def test_leafstate_json_roundtrip():
    from golden_io import load_group

    from paper_2410_05534_b200.arena import Batch, LeafState

    c = load_group("toy")["cases"][3]
    lf = LeafState.from_json(c["state"])
    assert LeafState.from_json(lf.to_json()).to_json() == c["state"]
    p = Batch([lf, lf]).pack()
    assert p["node_base"].tolist() == [0, lf.n, 2 * lf.n]
    assert len(p["hc_koff"]) == 2 * (lf.n + 1)


def test_pattern_program_layout():
    from paper_2410_05534_b200.patterns import compile_pattern, parse_pattern

    pat = parse_pattern("(conv2d[?s,?p,none] ?x (ewadd ?w1 ?w2))")
    names = {"conv2d": 3, "ewadd": 5}
    prog = compile_pattern(pat, lambda n: names.get(n, -1), lambda v: {"none": 9}.get(v, 0x3FFFFFFF)).program
    P, V, Q = prog[:3]
    assert (P, V, Q) == (5, 3, 2)
    rec0 = prog[3:9]
    assert rec0[0] == 1 and rec0[1] == 3 and rec0[2] == 2 and rec0[3] == 3
    slots = prog[rec0[4]: rec0[4] + 3]
    assert slots.tolist() == [-(1 + 1), -(0 + 1), 9]  # ?s -> pvar 1 (sorted p,s), ?p -> 0, literal none


def test_fingerprint_key_tables():
    """Host tables of the device fingerprint: key ranks in Python tuple order, repr bytes exact."""
    from paper_2410_05534_b200.fingerprint import key_tables

    keys = [("relu", 1, "((), (4, 8))"), ("matmul", 2, "((), (4, 8))"), ("conv2d", 2, "((1, 0, 'relu'), (1, 2))"),
            ("matmul", 2, "((), (16, 8))")]
    krank, off, blob = key_tables(keys)
    assert [keys[i] for i in np.argsort(krank)] == sorted(keys)
    for i, k in enumerate(keys):
        assert blob[off[i]:off[i + 1]] == repr(k).encode()


def test_cost_model_spec_kats():
    """SPEC.md:402-404 operator_cost examples (analytic FLOPs x coefficient, unit mode)."""
    from paper_2410_05534_b200.cost_model import CostModelConfig, operator_cost

    assert operator_cost(CostModelConfig(), "matmul", (), (8, 32), ((8, 16), (16, 32))) == 8.192e-6
    assert operator_cost(CostModelConfig(mode="unit"), "conv2d", (1, 1, "none"), (1, 8, 16, 16),
                         ((1, 8, 16, 16), (8, 8, 3, 3))) == 1.0
    assert operator_cost(CostModelConfig(mode="unit"), "input", ("x",), (1, 8), ()) == 0.0


def test_rule_masks_chunk_layout():
    """LeafPipeline.rule_masks: one 32-pattern chunk per row (esat_ematch_masked's chunk-major
    [ceil(P/32), L] words), so rules whose sources sit beyond pattern 31 mask the right bits."""
    from types import SimpleNamespace

    from paper_2410_05534_b200.pipeline import LeafPipeline

    pipe = LeafPipeline.__new__(LeafPipeline)
    pipe.pattern_ids = list(range(70))
    pipe.rules = [SimpleNamespace(pattern_ids=[0, 5]), SimpleNamespace(pattern_ids=[33]),
                  SimpleNamespace(pattern_ids=[31, 64, 69])]
    m = pipe.rule_masks(np.array([2, 0xFFFFFFFF, 1, 0], np.uint32))
    assert m.shape == (3, 4) and m.dtype == np.uint32 and m.flags["C_CONTIGUOUS"]
    assert m[:, 0].tolist() == [1 << 31, 0, (1 << 0) | (1 << 5)]
    assert m[:, 1].tolist() == [0, 0, 0]
    assert m[:, 2].tolist() == [0, 1 << 1, 0]
    assert m[:, 3].tolist() == [(1 << 0) | (1 << 5), 0, 0]
