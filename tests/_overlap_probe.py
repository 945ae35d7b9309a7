"""Probe: one resident batch per step vs two batches on two streams (inter-step overlap)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import bench
from paper_2410_05534_b200 import native
from paper_2410_05534_b200.pipeline import LeafPipeline

leaves, symarr, name_id, code, ref, meta = bench.load_leaves("nasrnn")
packed, _ = bench.make_batch(leaves, 4096, 0)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
pipes = []
for s in (s1, s2):
    ctx = native.Context(0)
    ctx.set_stream(s.cuda_stream)
    p = LeafPipeline(ctx, symarr, bench.rules(), name_id, code, method="ocf", pool_entries_per_node=32)
    p.load(packed)
    for _ in range(4):
        p.step()
    pipes.append(p)
torch.cuda.synchronize()
K = 40
for mode in ("single", "double"):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for i in range(K):
        p = pipes[0] if mode == "single" else pipes[i % 2]
        p.step()
    # join both streams into the default stream before the end event
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    e1.record()
    torch.cuda.synchronize()
    print(mode, "ms/step", e0.elapsed_time(e1) / K, flush=True)
