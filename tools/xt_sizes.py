"""Probe: extraction time vs leaf size (homogeneous batches of one leaf)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import bench
from paper_2410_05534_b200 import native
from paper_2410_05534_b200.arena import Batch
from paper_2410_05534_b200.pipeline import LeafPipeline

leaves, symarr, name_id, code, ref, meta = bench.load_leaves(sys.argv[1] if len(sys.argv) > 1 else "nasrnn")
sizes = np.array([lf.n for lf in leaves])
order = np.argsort(sizes)
ctx = native.Context(0)
for tag, idx in (("min", order[0]), ("p25", order[64]), ("median", order[128]), ("p75", order[192]), ("max", order[-1]), ("mixed", None)):
    B = 4096
    sel = [leaves[i % 256] for i in range(B)] if idx is None else [leaves[idx]] * B
    pipe = LeafPipeline(ctx, symarr, bench.rules(), name_id, code, pool_entries_per_node=64)
    b = pipe.load(Batch(sel).pack())
    pipe.rebuild()
    native.extract_with_retry(b, "ocf", factor=64)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        pipe.extract()
        torch.cuda.synchronize()
        ts.append(ctx.last_ms())
    ext = b.download_extract()
    print(tag, "n", sel[0].n if idx is not None else "-", "passes", np.bincount(ext["passes"]), "ms", round(min(ts), 3), flush=True)
    b.close()
