"""The five BASELINE configs' leaf sets (reference-generated MCTS rollout leaves,
tests/golden/bench_<model>.npz): the device pipeline must reproduce the reference's OCF and
default-greedy root costs bit-exactly on every leaf, and the CPU oracle's per-rule match counts,
merge counts, every match record
(in order) and chosen e-nodes."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

MODELS = ["bert", "nasrnn", "resnext50", "inception_v3", "nasnet_a"]


@pytest.mark.parametrize("model", MODELS)
def test_config_leaves_bit_exact(model):
    import bench
    from oracle import oracle as O
    from paper_2410_05534_b200 import native
    from paper_2410_05534_b200.arena import Batch
    from paper_2410_05534_b200.pipeline import LeafPipeline

    leaves, symarr, name_id, code, ref_ocf, meta = bench.load_leaves(model)
    import json

    ref_default = np.load(bench.ROOT / "tests" / "golden" / f"bench_{model}.npz")["ref_default"]
    ctx = native.Context(0)
    pipe = LeafPipeline(ctx, symarr, bench.rules(), name_id, code)
    packed = Batch(leaves).pack()
    b = pipe.load(packed)
    pipe.rebuild()
    pipe.ematch()
    counts = pipe.match_counts()
    view = b.download_rebuild()
    view.update(b.download_view())
    for method, ref in (("ocf", ref_ocf), ("default", ref_default)):
        ext = native.extract_with_retry(b, method, factor=32)
        assert np.all(ext["status"] == 0), method
        bad = np.nonzero(ext["root_cost"].view(np.uint64) != np.asarray(ref).view(np.uint64))[0]
        assert bad.size == 0, (model, method, bad[:5])
        oe = O.extract(packed, O.rebuild(packed, symarr["rank"]), method, threads=8)
        for l in range(packed["n_leaves"]):
            n0, C = int(packed["node_base"][l]), int(view["C"][l])
            assert np.array_equal(ext["choice"][n0:n0 + C], oe["choice"][n0:n0 + C]), (model, method, l)
    ov = O.rebuild(packed, symarr["rank"], threads=8)
    assert np.array_equal(view["merges"], ov["merges"]) and np.array_equal(view["C"], ov["C"])
    for j, r in enumerate(pipe.rules):
        # every match record, in the reference's order (not just the counts): the device lists
        # and the oracle's share the [leaf][match][W words] layout
        if r.multi:
            ow, ooff, cnt, W = O.joint(packed, ov, symarr, r._programs, r.var_maps, r.pvar_maps, len(r.var_names),
                                       len(r.pvar_names), threads=8)
            dw, doff, dcnt = b.download_matches(pipe.joins.index(r), from_join=True)
        else:
            ow, ooff, cnt, W = O.ematch(packed, ov, symarr, r._programs[0], threads=8)
            dw, doff, dcnt = b.download_matches(r.pattern_ids[0])
        assert np.array_equal(counts[j], cnt), (model, r.rule.id)
        assert np.array_equal(dcnt, cnt), (model, r.rule.id)
        for l in range(packed["n_leaves"]):
            n = int(cnt[l]) * W
            got = dw[int(doff[l]):int(doff[l]) + n]
            want = ow[int(ooff[l]):int(ooff[l]) + n]
            assert np.array_equal(got, want), (model, r.rule.id, l)
    b.close()
    ctx.close()
    del json
