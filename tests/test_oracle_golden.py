"""The CPU oracle (oracle/esat_oracle.c) pinned against the reference's golden vectors.

tests/golden/*.json.gz were produced by running the reference implementation
(tests/golden/make_golden.py). Every stage must agree exactly: rebuild (hashcons order,
union-find roots/ranks, classes, merge counts), e-match / joint_match (ordered match
lists), default and OCF greedy extraction (float.hex-equal costs, chosen nodes, errors).
"""

import pytest

from golden_io import (GROUPS, check_rebuild, compile_rule, decode_extract, decode_matches, group_batch, load_group,
                       rules_of)
from oracle import oracle as O


@pytest.fixture(scope="module", params=GROUPS)
def group(request):
    st, packed, cases = group_batch(request.param)
    view = O.rebuild(packed, st.arrays["rank"], threads=4)
    return request.param, st, packed, cases, view


def test_rebuild(group):
    name, st, packed, cases, view = group
    assert not check_rebuild(packed, view, cases)


@pytest.mark.parametrize("method", ["default", "ocf"])
def test_extract(group, method):
    name, st, packed, cases, view = group
    ext = O.extract(packed, view, method, threads=4)
    bad = [c["name"] for l, c in enumerate(cases) if decode_extract(packed, view, ext, l) != c["extract"][method]]
    assert not bad, bad[:5]


def test_ematch_and_joint(group):
    name, st, packed, cases, view = group
    rules = rules_of(load_group(name))
    if not rules:
        pytest.skip("no rule set for this group")
    bad, compared = [], 0
    for rule in rules:
        comps, vn, qn, vm, qm = compile_rule(rule, st)
        if rule.kind == "single":
            words, off, cnt, W = O.ematch(packed, view, st.arrays, comps[0].program, threads=4)
        else:
            words, off, cnt, W = O.joint(packed, view, st.arrays, [c.program for c in comps], vm, qm, len(vn),
                                         len(qn), threads=4)
        for l, c in enumerate(cases):
            rec = c["ematch"][rule.id]
            assert [int(x) for x in rec["source_counts"]] is not None
            if "matches" not in rec:
                continue
            compared += 1
            got = decode_matches(words, off, cnt, W, l, len(rule.sources), vn, qn, st)
            if got != rec["matches"]:
                bad.append((c["name"], rule.id))
    assert compared > 0
    assert not bad, bad[:5]


def test_is_rule_applicable_counts(group):
    """is_rule_applicable (rewrite.py:579-589) = every source has >= 1 independent match."""
    name, st, packed, cases, view = group
    rules = rules_of(load_group(name))
    if not rules:
        pytest.skip("no rule set for this group")
    for rule in rules:
        comps, vn, qn, vm, qm = compile_rule(rule, st)
        per_src = [O.ematch(packed, view, st.arrays, cp.program, threads=4)[2] for cp in comps]
        for l, c in enumerate(cases):
            expect = c["ematch"][rule.id]["source_counts"]
            assert [int(p[l]) for p in per_src] == expect, (c["name"], rule.id)
