"""Probe: TENSAT-style sequential saturation of an analog on the device up to a large node limit."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2410_05534_b200 import analogs, native
from paper_2410_05534_b200 import tensor_ir as T
from paper_2410_05534_b200.apply import ApplyDriver
from paper_2410_05534_b200.arena import Batch, export_state
from paper_2410_05534_b200.cost_model import CostModelConfig
from paper_2410_05534_b200.patterns import load_rules
from paper_2410_05534_b200.pipeline import LeafPipeline
from paper_2410_05534_b200.symtab import SymbolTable

model, limit = sys.argv[1], int(sys.argv[2])
KMULTI = int(sys.argv[3]) if len(sys.argv) > 3 else 1
rules = load_rules("taso_analog")
eg = T.graph_to_egraph(analogs.build_analog(model, T.GraphBuilder))
st = SymbolTable(); cfg = CostModelConfig()
leaf = export_state(eg, st, cfg)
st.finalize()
ctx = native.Context(0)
packed = Batch([leaf]).pack_with_headroom(nodes=limit * 2, kids=limit * 4, ids=limit * 2)
pipe = LeafPipeline(ctx, st.arrays(), rules, lambda n: st.name_id(n, create=False), st.code)
b = pipe.load(packed); b.set_counts(packed["n_cnt"], packed["u_cnt"])
drv = ApplyDriver(pipe, st, eg.language, cfg)
order = [i for i, r in enumerate(pipe.rules) if r.multi] + [i for i, r in enumerate(pipe.rules) if not r.multi]
t0 = time.time()
n = leaf.n
for it in range(50):
    changed_any = False
    for ri in order:
        if pipe.rules[ri].multi and it >= KMULTI:
            continue
        pipe.rebuild(); pipe.ematch()
        t = time.time()
        res = drv.apply(np.array([ri], np.uint32))
        ctx.sync(); ta = time.time() - t
        if res["status"][0] != 0:
            print("status", res["status"][0]); break
        pipe.rebuild()
        n = int(b.download_rebuild()["n"][0])
        rep = res["report"][0]
        changed_any |= bool(rep[1])
        print(f"it {it} rule {ri} matches {rep[0]} added {rep[5]} n {n} apply {ta:.3f}s total {time.time()-t0:.1f}s", flush=True)
        if n >= limit:
            break
    if n >= limit or not changed_any:
        break
print("final n", n, "time", time.time() - t0)
