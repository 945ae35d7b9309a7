"""Probe: the config-4 state through the device pipeline (timings, counts vs oracle for cheap parts)."""
import sys, time, json
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2410_05534_b200 import native
from paper_2410_05534_b200.arena import Batch, LeafState
from paper_2410_05534_b200.pipeline import LeafPipeline
from paper_2410_05534_b200.patterns import load_rules
from paper_2410_05534_b200.symtab import NO_MATCH_CODE

z = np.load("tests/golden/c4_inception_state.npz"); meta = json.loads(str(z["meta"]))
lf = LeafState(z["hc_sym"], z["hc_koff"], z["hc_kids"], z["hc_cid"], z["hc_cost"], z["uf_parent"], z["uf_rank"], int(z["root"]))
symarr = {"name": z["sym_name"], "arity": z["sym_arity"], "rank": z["sym_rank"], "poff": z["sym_poff"], "params": z["sym_params"]}
names = {n: i for i, n in enumerate(meta["names"])}; codes = {(type(v), v): i for i, v in enumerate(meta["values"])}
ctx = native.Context(0)
pipe = LeafPipeline(ctx, symarr, load_rules("taso_analog"), lambda n: names.get(n, -1), lambda v: codes.get((type(v), v), NO_MATCH_CODE))
b = pipe.load(Batch([lf]).pack())
for stage in ("rebuild", "match", "join", "extract"):
    t = time.time()
    getattr(pipe, stage)()
    ctx.sync()
    if stage in ("match", "join"):
        b.download_matches(0)   # settle lazily verified launches
        ctx.sync()
    print(stage, "wall", round(time.time() - t, 3), "kernel_ms", round(ctx.last_ms(), 3), flush=True)
native.extract_with_retry(b, "ocf", factor=32)
for stage in ("rebuild", "match", "join", "extract"):   # second round: sized buffers
    getattr(pipe, stage)(); ctx.sync()
    print("again", stage, "kernel_ms", round(ctx.last_ms(), 3), flush=True)
counts = pipe.match_counts()
print("match counts per rule", counts[:, 0].tolist())
ext = b.download_extract()
print("ocf", ext["status"], ext["root_cost"], ext["passes"])
