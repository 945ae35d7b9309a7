"""Probe: per-phase clock64 breakdown of k_extract (ESAT_DEBUG build) on the NasRNN bench batch.

    ESAT_DEBUG_LIB=1 PYTHONPATH=. python tools/xt_phases.py [model]
"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import bench
from paper_2410_05534_b200 import native
from paper_2410_05534_b200.arena import Batch
from paper_2410_05534_b200.pipeline import LeafPipeline

model = sys.argv[1] if len(sys.argv) > 1 else "nasrnn"
leaves, symarr, name_id, code, ref, meta = bench.load_leaves(model)
B = 4096
sel = [leaves[i % len(leaves)] for i in range(B)]
ctx = native.Context(0)
pipe = LeafPipeline(ctx, symarr, bench.rules(), name_id, code, pool_entries_per_node=64)
b = pipe.load(Batch(sel).pack())
pipe.rebuild()
native.extract_with_retry(b, "ocf", factor=64)
torch.cuda.synchronize()
print("passes", np.bincount(b.download_extract()["passes"]), flush=True)
