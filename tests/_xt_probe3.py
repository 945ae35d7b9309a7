import sys, os; sys.path.insert(0, '.')
import numpy as np, bench
from paper_2410_05534_b200 import native
from paper_2410_05534_b200.pipeline import LeafPipeline
leaves, symarr, name_id, code, ref, meta = bench.load_leaves("nasrnn")
ctx = native.Context(0)
pipe = LeafPipeline(ctx, symarr, bench.rules(), name_id, code, pool_entries_per_node=32)
B = int(os.environ.get("B", "4096"))
packed, idx = bench.make_batch(leaves, B, 0)
b = pipe.load(packed)
pipe.rebuild()
for _ in range(3): b.extract("ocf")
ctx.sync()
print("ms", ctx.last_ms())
