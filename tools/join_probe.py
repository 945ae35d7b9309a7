"""Probe: one rebuild + e-match + join of the 4096-leaf bench batch (for ncu captures of k_ematch/k_join).

    PYTHONPATH=. python tools/join_probe.py [model]
"""
import sys
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
pipe = LeafPipeline(ctx, symarr, bench.rules(), name_id, code)
b = pipe.load(Batch(sel).pack())
pipe.rebuild()
for _ in range(2):
    pipe.match()
    pipe.join()
torch.cuda.synchronize()
print("ok", flush=True)
