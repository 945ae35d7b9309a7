"""Host tensor-IR API kept for the drop-in: the reference's zoo (zoo_generate returns
the reference's Model objects), save_graph / load_graph, extraction_to_graph on a hand-made
selection, and EGraph.to_dot -- each compared with the reference itself when it is importable."""

import pytest

SPECS = ["resblock_stack(3)", "mlp(3,16)", "attention_block(16,2)", "inception_cell(3)", "toy_expr"]


def _ref():
    from oracle.mcts_ref import import_reference, reference_available

    if not reference_available():
        pytest.skip("reference not importable")
    return import_reference()


def _rows(g):
    return [(n.id, n.op, n.params, n.inputs, n.shape) for n in g.nodes], list(g.outputs)


@pytest.mark.parametrize("spec", SPECS)
def test_zoo_matches_reference(spec):
    from paper_2410_05534_b200 import tensor_ir as T

    E, R, X, RT = _ref()
    ours, ref = T.zoo_generate(spec), RT.zoo_generate(spec)
    assert ours.kind == ref.kind and ours.name == ref.name
    if ours.kind == "toy":
        assert ours.term == ref.term
    else:
        assert _rows(ours.graph) == _rows(ref.graph)


def test_zoo_errors_and_analogs():
    from paper_2410_05534_b200 import tensor_ir as T

    for bad in ("mlp(3)", "nope(1)", "resblock_stack"):
        with pytest.raises(T.GraphFormatError):
            T.zoo_generate(bad)
    with pytest.raises(T.GraphFormatError):
        T.zoo_generate("inception_cell(1)")
    assert T.zoo_generate("nasrnn").kind == "tensor"


@pytest.mark.parametrize("spec", SPECS[:4])
def test_save_load_graph_bytes_match_reference(spec, tmp_path):
    from paper_2410_05534_b200 import tensor_ir as T

    E, R, X, RT = _ref()
    ours, ref = T.zoo_generate(spec).graph, RT.zoo_generate(spec).graph
    T.save_graph(ours, str(tmp_path / "a.json"))
    RT.save_graph(ref, str(tmp_path / "b.json"))
    assert (tmp_path / "a.json").read_bytes() == (tmp_path / "b.json").read_bytes()
    assert _rows(T.load_graph(str(tmp_path / "b.json"))) == _rows(ref)
    (tmp_path / "bad.json").write_text("{nope")
    with pytest.raises(T.GraphFormatError):
        T.load_graph(str(tmp_path / "bad.json"))


def test_extraction_to_graph_identity_selection():
    """Choosing, in every class of a freshly converted graph, its only e-node gives back the program
    (same save_graph text as the reference's extraction_to_graph on the same selection)."""
    from paper_2410_05534_b200 import tensor_ir as T
    from paper_2410_05534_b200.extraction import ExtractionResult

    E, R, X, RT = _ref()
    for spec in SPECS[:4]:
        ref_eg = RT.zoo_generate(spec).to_egraph()
        sel_ref = X.ExtractionResult(0.0, {c: next(iter(k.nodes)) for c, k in ref_eg.classes.items()}, "x")
        want = RT.extraction_to_graph(ref_eg, sel_ref)
        # our EGraph of the same program, built on the host without the device rebuild
        eg = T.EGraph(T.TENSOR_LANGUAGE)
        eg.hashcons = {T.ENode(T.Symbol(n.symbol.name, n.symbol.arity, n.symbol.payload), n.children): c
                       for n, c in ref_eg.hashcons.items()}
        eg._uf.parent, eg._uf.rank = list(ref_eg._uf.parent), list(ref_eg._uf.rank)
        eg.classes = {c: E.EClass(c, {T.ENode(T.Symbol(n.symbol.name, n.symbol.arity, n.symbol.payload), n.children)
                                      for n in k.nodes}) for c, k in ref_eg.classes.items()}
        eg.root = ref_eg.root
        got = T.extraction_to_graph(eg, ExtractionResult(0.0, {c: next(iter(k.nodes)) for c, k in eg.classes.items()},
                                                         "x"))
        assert T.graph_json(got) == T.graph_json(T.TensorGraph(want.nodes, want.outputs))


def test_to_dot_matches_reference():
    from paper_2410_05534_b200 import egraph as OE

    E, R, X, RT = _ref()
    ref_eg = RT.zoo_generate("attention_block(8,1)").to_egraph()
    eg = OE.EGraph()
    conv = lambda n: OE.ENode(OE.Symbol(n.symbol.name, n.symbol.arity, n.symbol.payload), n.children)  # noqa: E731
    eg.hashcons = {conv(n): c for n, c in ref_eg.hashcons.items()}
    eg._uf.parent, eg._uf.rank = list(ref_eg._uf.parent), list(ref_eg._uf.rank)
    eg.classes = {c: OE.EClass(c, {conv(n) for n in k.nodes}) for c, k in ref_eg.classes.items()}
    eg.root = ref_eg.root
    assert eg.to_dot() == ref_eg.to_dot()
