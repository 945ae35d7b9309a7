import sys, os, time; sys.path.insert(0, '.')
import numpy as np, bench
from paper_2410_05534_b200 import native
from paper_2410_05534_b200.pipeline import LeafPipeline
leaves, symarr, name_id, code, ref, meta = bench.load_leaves("nasrnn")
ctx = native.Context(0)
pipe = LeafPipeline(ctx, symarr, bench.rules(), name_id, code, pool_entries_per_node=128)
packed, idx = bench.make_batch(leaves, 4096, 0)
b = pipe.load(packed)
pipe.rebuild()
for m in ("ocf", "default"):
    for _ in range(3): pipe.batch.extract(m)
    ctx.sync()
    ts = []
    for _ in range(5):
        pipe.batch.extract(m); ts.append(ctx.last_ms())
    e = b.download_extract()
    ok = (m != "ocf") or np.array_equal(e["root_cost"].view(np.uint64), ref[idx].view(np.uint64))
    print(os.environ.get("ESAT_EXTRACT_THREADS"), m, "ms", min(ts), "parity", ok, "status", np.bincount(e["status"]))
