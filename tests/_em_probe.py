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
ctx.sync()
sets = {"all": list(range(24)), "none_matmul": [i for i in range(24) if i not in (20, 21)], "matmul_srcs": [20, 21],
        "first": [0], "p4": [4], "relu": [12]}
for name, ids in sets.items():
    for _ in range(2): b.ematch(ids)
    ts = []
    for _ in range(3):
        b.ematch(ids); ts.append(ctx.last_ms())
    print(name, len(ids), "ms", round(min(ts), 3))
for r in pipe.rules:
    print(r.rule.id, r.pattern_ids, r.rule.name[:60])
