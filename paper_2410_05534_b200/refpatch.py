"""The reference-side binding a maintainer adds to the reference package: it
swaps the hot path of ``esat`` -- ``EGraph.rebuild`` (egraph.py:203), ``joint_match`` / ``ematch``
(rewrite.py:400-433), ``extract_default_greedy`` / ``extract_ocf_greedy`` (extraction.py:157/229)
and, optionally, ``apply_rule`` (rewrite.py:526) -- for this package's device implementations,
which operate directly on the reference's own ``EGraph`` objects (device.py) and return the
reference's own result types and exceptions.

    from esat import egraph, extraction, rewrite
    from paper_2410_05534_b200 import refpatch
    refpatch.install(egraph, rewrite, extraction)
"""

from __future__ import annotations


def install(E, R, X, apply_rule: bool = False) -> dict:
    """Monkey-patch the reference modules ``E`` (esat.egraph), ``R`` (esat.rewrite) and ``X``
    (esat.extraction); returns the originals so ``uninstall`` can restore them."""
    from . import device
    from . import extraction as ours

    orig = {"rebuild": E.EGraph.rebuild, "joint_match": R.joint_match, "ematch": R.ematch,
            "ocf": X.extract_ocf_greedy, "default": X.extract_default_greedy, "apply_rule": R.apply_rule}

    def rebuild(self):
        return device.rebuild(self)

    def joint_match(egraph, patterns, language=None):
        if egraph.dirty:
            raise E.StructuralError("ematch requires a rebuilt e-graph")
        recs, vn, qn, S = device.joint_match(egraph, list(patterns), language)
        vals = device.session().symtab.values
        return [R.Substitution(tuple(zip(vn, r[S:S + len(vn)])), tuple((q, vals[c]) for q, c in zip(qn, r[S + len(vn):])),
                               tuple(r[:S])) for r in recs.tolist()]

    def extractor(fn, name):
        def run(egraph, costs):
            try:
                r = fn(egraph, costs)
            except ours.InfeasibleExtraction as exc:
                raise X.InfeasibleExtraction(str(exc)) from None
            except ours.ExtractionError as exc:
                raise X.ExtractionError(str(exc)) from None
            return X.ExtractionResult(r.total_cost, r.chosen, name)
        return run

    E.EGraph.rebuild = rebuild
    R.joint_match = joint_match
    R.ematch = lambda egraph, pattern, language=None: joint_match(egraph, [pattern], language)
    X.extract_ocf_greedy = extractor(ours.extract_ocf_greedy, "ocf_greedy")
    X.extract_default_greedy = extractor(ours.extract_default_greedy, "default_greedy")
    if apply_rule:
        def apply(egraph, rule, node_limit=0, language=None):
            rep = device.apply_rule(egraph, rule, node_limit, language)
            out = R.ApplyReport(rule_id=rule.id)
            for k in ("matches_found", "changed", "nodes_after", "classes_after", "hit_node_limit", "cycles_filtered",
                      "shape_filtered"):
                setattr(out, k, getattr(rep, k))
            return out
        R.apply_rule = apply
    return orig


def uninstall(E, R, X, orig: dict) -> None:
    E.EGraph.rebuild = orig["rebuild"]
    R.joint_match, R.ematch, R.apply_rule = orig["joint_match"], orig["ematch"], orig["apply_rule"]
    X.extract_ocf_greedy, X.extract_default_greedy = orig["ocf"], orig["default"]
