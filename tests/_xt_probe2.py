import sys, os, time; sys.path.insert(0, '.')
import numpy as np, bench
from paper_2410_05534_b200 import native
from paper_2410_05534_b200.pipeline import LeafPipeline
leaves, symarr, name_id, code, ref, meta = bench.load_leaves("nasrnn")
ctx = native.Context(0)
pipe = LeafPipeline(ctx, symarr, bench.rules(), name_id, code, pool_entries_per_node=128)
for B in (256, 1024, 2048, 4096, 8192):
    packed, idx = bench.make_batch(leaves, B, 0)
    b = pipe.load(packed)
    pipe.rebuild()
    res = []
    for m in ("ocf", "default"):
        for _ in range(2): b.extract(m)
        ctx.sync()
        ts = []
        for _ in range(3):
            b.extract(m); ts.append(ctx.last_ms())
        res.append(round(min(ts), 3))
    e = b.download_extract()
    print(B, "ocf/default ms", res, "us/leaf", round(1000*res[0]/B, 3), np.bincount(e["status"]))
