"""Probe: k_apply on a batch of reference rollout leaves (tests/golden/bench_<model>.npz), each leaf
applying one of its matching rules (seeded), timed with CUDA events; prints the SHA-256 of the
resulting dirty states + reports, so two runs (e.g. with and without ESAT_APPLY_NO_POT) can be
compared for bit-identical results.

    python tools/apply_diff.py [model] [leaves] [max_matches]
"""
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402

import torch  # noqa: E402

from paper_2410_05534_b200 import native  # noqa: E402
from paper_2410_05534_b200.apply import COST_ANALYTIC, LANG_TENSOR, symbol_arrays  # noqa: E402
from paper_2410_05534_b200.arena import Batch  # noqa: E402
from paper_2410_05534_b200.pipeline import LeafPipeline  # noqa: E402

model = sys.argv[1] if len(sys.argv) > 1 else "nasrnn"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
cap = int(sys.argv[3]) if len(sys.argv) > 3 else 600
leaves, symarr, name_id, code, _, meta = bench.load_leaves(model)
ctx = native.Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
packed = Batch([leaves[i % len(leaves)] for i in range(B)]).pack_with_headroom(nodes=max(2048, 8 * cap))
pipe = LeafPipeline(ctx, symarr, bench.rules(), name_id, code)
b = pipe.load(packed)
b.set_counts(packed["n_cnt"], packed["u_cnt"])
pipe.rebuild()
pipe.ematch()
counts = pipe.match_counts()
rng = np.random.default_rng(0)
leaf_rule = np.full(B, 0xFFFFFFFF, np.uint32)
for l in range(B):
    live = np.nonzero((counts[:, l] > 0) & (counts[:, l] <= cap))[0]
    if live.size:
        leaf_rule[l] = int(rng.choice(live))
poff, flat = symarr["poff"], symarr["params"]
codes = [flat[poff[i]:poff[i + 1]] for i in range(len(symarr["name"]))]
sa = symbol_arrays(symarr["name"], symarr["arity"], [s[2] for s in meta["symbols"]], codes, meta["values"])
off, words = pipe.apply_programs(name_id, code)
ctx.apply_setup(LANG_TENSOR, COST_ANALYTIC, 1e-9, sa, off, words)
b.apply(leaf_rule)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    b.apply(leaf_rule)
e1.record()
torch.cuda.synchronize()
res = b.download_apply()
st = b.download_state()
h = hashlib.sha256()
for k in ("n", "U", "hc_sym", "hc_koff", "hc_kids", "hc_cid", "hc_cost", "uf_parent", "uf_rank"):
    h.update(np.ascontiguousarray(st[k]).tobytes())
h.update(res["status"].tobytes())
h.update(res["report"].tobytes())
print(json.dumps({"model": model, "leaves": B, "max_matches": cap, "ms": e0.elapsed_time(e1) / 5,
                  "sha256": h.hexdigest(), "status": np.bincount(res["status"]).tolist(),
                  "matches": int(res["report"][:, 0].sum()), "cycles": int(res["report"][:, 2].sum()),
                  "unions": int(res["report"][:, 4].sum()), "added": int(res["report"][:, 5].sum())}))
