"""BASELINE config 4 (Inception-v3 at a large e-node limit, the e-graph explosion stress) at full
size: the 80,257-e-node state grown on the device by TENSAT-style saturation
(tests/golden/make_c4_state.py) through every device stage, against the CPU oracle.

Rebuild arrays, match lists of every single-pattern rule, both extractions (costs bit-exact,
chosen e-nodes) are compared element for element; the conv-merge join (132,828,819 records, the
explosion) is compared by count and by a size-independent property of its records (every record
joins two conv matches that agree on the shared variables and attributes)."""

import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c4():
    from golden_io import GOLDEN
    from paper_2410_05534_b200.arena import Batch, LeafState
    from paper_2410_05534_b200.symtab import NO_MATCH_CODE

    z = np.load(GOLDEN / "c4_inception_state.npz")
    meta = json.loads(str(z["meta"]))
    lf = LeafState(z["hc_sym"], z["hc_koff"], z["hc_kids"], z["hc_cid"], z["hc_cost"], z["uf_parent"], z["uf_rank"],
                   int(z["root"]))
    symarr = {"name": z["sym_name"], "arity": z["sym_arity"], "rank": z["sym_rank"], "poff": z["sym_poff"],
              "params": z["sym_params"]}
    names = {n: i for i, n in enumerate(meta["names"])}
    codes = {(type(v), v): i for i, v in enumerate(meta["values"])}
    return Batch([lf]).pack(), symarr, (lambda n: names.get(n, -1)), (lambda v: codes.get((type(v), v), NO_MATCH_CODE))


def test_c4_full_size_vs_oracle(c4):
    from oracle import oracle as O
    from paper_2410_05534_b200 import native
    from paper_2410_05534_b200.pipeline import LeafPipeline
    from paper_2410_05534_b200.patterns import load_rules

    packed, symarr, name_id, code = c4
    ctx = native.Context(0)
    pipe = LeafPipeline(ctx, symarr, load_rules("taso_analog"), name_id, code)
    b = pipe.load(packed)
    pipe.rebuild()
    dev = b.download_rebuild()
    dev.update(b.download_view())
    ref = O.rebuild(packed, symarr["rank"])
    assert int(ref["n"][0]) == 80257
    C = int(ref["C"][0])
    for k in ("n", "merges", "C", "root_pos", "hc_sym", "hc_koff", "hc_kids", "hc_cid", "nd_sym", "nd_koff", "nd_kpos",
              "nd_hc"):
        assert np.array_equal(dev[k], ref[k]), k
    assert np.array_equal(dev["cls_id"][:C], ref["cls_id"][:C]) and np.array_equal(dev["cls_off"][:C + 1],
                                                                                  ref["cls_off"][:C + 1])
    for method in ("default", "ocf"):
        e = native.extract_with_retry(b, method, factor=32)
        r = O.extract(packed, ref, method)
        assert np.array_equal(e["status"], r["status"]) and e["status"][0] == 0
        assert e["root_cost"].view(np.uint64)[0] == r["root_cost"].view(np.uint64)[0], method
        reach = r["reachable"].astype(bool)
        assert np.array_equal(e["choice"][reach], r["choice"][reach]), method
    pipe.ematch()
    counts = pipe.match_counts()
    for j, rr in enumerate(pipe.rules):
        if rr.multi:
            continue
        w, off, cnt = b.download_matches(rr.pattern_ids[0])
        rw, roff, rcnt, _ = O.ematch(packed, ref, symarr, rr._programs[0])
        assert np.array_equal(cnt, rcnt) and np.array_equal(w[: int(off[-1])], rw), rr.rule.id
    # the explosion: conv-merge join count = pairs of conv matches agreeing on x and (s, p, c)
    conv = next(rr for rr in pipe.rules if rr.multi and rr.rule.id == 21)
    w, off, cnt = b.download_matches(conv.pattern_ids[0])
    W = 1 + 2 + 3   # [root][w1, x][c, p, s]
    rec = w[: int(off[-1])].reshape(-1, W)
    _, sizes = np.unique(rec[:, 2:], axis=0, return_counts=True)
    assert int(counts[pipe.rules.index(conv), 0]) == int((sizes.astype(np.int64) ** 2).sum()) == 132828819
    # element for element: the device's 132.8M joined records (4.25 GB) hash to the CPU oracle's
    # (tests/golden/make_c4_join_hash.py; the oracle is pinned to the reference's joint_match)
    import hashlib
    import json
    from pathlib import Path

    want = json.loads((Path(__file__).resolve().parent / "golden" / "c4_join_sha256.json").read_text())
    jw, joff, jcnt = b.download_matches(pipe.joins.index(conv), from_join=True)
    assert int(jcnt[0]) == want["records"]
    got = hashlib.sha256(np.ascontiguousarray(jw[: int(joff[-1])], np.uint32).tobytes()).hexdigest()
    assert got == want["sha256_u32_le"]
    b.close()
    ctx.close()
