"""k_extract lane groups: one leaf per warp, two (16 lanes) or four (8 lanes) leaves
per warp must give the same extraction -- every status, root and class cost bit, chosen e-node,
reachable flag and pass count -- equal to the reference's root costs; and the per-context tuning
picks 16 lanes only for narrow-level leaf sets."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

KEYS = ("status", "err_class", "root_cost", "class_cost", "choice", "reachable", "passes")


@pytest.mark.parametrize("model", ["resnext50", "bert"])
def test_extraction_identical_at_every_lane_width(model):
    import bench
    from paper_2410_05534_b200 import native
    from paper_2410_05534_b200.arena import Batch
    from paper_2410_05534_b200.pipeline import LeafPipeline

    leaves, symarr, name_id, code, ref_ocf, meta = bench.load_leaves(model)
    ctx = native.Context(0)
    pipe = LeafPipeline(ctx, symarr, bench.rules(), name_id, code)
    b = pipe.load(Batch(leaves).pack())
    pipe.rebuild()
    outs = {}
    for lanes in (32, 16, 8):
        for method in ("ocf", "default"):
            ctx.set_extract_lanes(lanes)   # pinned: tuning only runs while extract_lanes is None
            outs[lanes, method] = native.extract_with_retry(b, method, factor=32)
    for method in ("ocf", "default"):
        for lanes in (16, 8):
            for k in KEYS:
                a, e = outs[lanes, method][k], outs[32, method][k]
                assert np.array_equal(a.view(np.uint64) if a.dtype == np.float64 else a,
                                      e.view(np.uint64) if e.dtype == np.float64 else e), (model, method, lanes, k)
    got = outs[16, "ocf"]["root_cost"].view(np.uint64)
    assert np.array_equal(got, np.asarray(ref_ocf).view(np.uint64)), model
    b.close()
    ctx.close()


def test_lane_tuning_follows_level_width():
    import bench
    from paper_2410_05534_b200 import native
    from paper_2410_05534_b200.arena import Batch
    from paper_2410_05534_b200.pipeline import LeafPipeline

    picked = {}
    for model in ("resnext50", "nasrnn"):
        leaves, symarr, name_id, code, ref_ocf, meta = bench.load_leaves(model)
        reps = -(-native.TUNE_MIN_LEAVES // len(leaves))   # tuning needs >= TUNE_MIN_LEAVES leaves
        ctx = native.Context(0)
        pipe = LeafPipeline(ctx, symarr, bench.rules(), name_id, code)
        b = pipe.load(Batch(leaves * reps).pack())
        pipe.rebuild()
        assert ctx.extract_lanes is None
        native.extract_with_retry(b, "ocf", factor=32)
        classes, levels = b.extract_shape()
        assert classes == int(b.download_view()["C"].sum()) and levels > 0
        picked[model] = (ctx.extract_lanes, ctx.extract_width)
        b.close()
        ctx.close()
    assert picked["resnext50"][0] == 16 and picked["resnext50"][1] <= native.LANES16_MAX_WIDTH, picked
    assert picked["nasrnn"][0] == 32 and picked["nasrnn"][1] > native.LANES16_MAX_WIDTH, picked
