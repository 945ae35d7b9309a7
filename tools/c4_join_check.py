"""One-off: config-4 conv-merge join records (132.8M) device vs CPU oracle, element for element."""
import json, sys, time
sys.path.insert(0, ".")
import numpy as np
from oracle import oracle as O
from paper_2410_05534_b200 import native
from paper_2410_05534_b200.arena import Batch, LeafState
from paper_2410_05534_b200.pipeline import LeafPipeline
from paper_2410_05534_b200.patterns import load_rules
from paper_2410_05534_b200.symtab import NO_MATCH_CODE

z = np.load("tests/golden/c4_inception_state.npz"); meta = json.loads(str(z["meta"]))
lf = LeafState(z["hc_sym"], z["hc_koff"], z["hc_kids"], z["hc_cid"], z["hc_cost"], z["uf_parent"], z["uf_rank"], int(z["root"]))
symarr = {"name": z["sym_name"], "arity": z["sym_arity"], "rank": z["sym_rank"], "poff": z["sym_poff"], "params": z["sym_params"]}
names = {n: i for i, n in enumerate(meta["names"])}; codes = {(type(v), v): i for i, v in enumerate(meta["values"])}
packed = Batch([lf]).pack()
ctx = native.Context(0)
pipe = LeafPipeline(ctx, symarr, load_rules("taso_analog"), lambda n: names.get(n, -1), lambda v: codes.get((type(v), v), NO_MATCH_CODE))
b = pipe.load(packed)
pipe.rebuild(); pipe.ematch()
conv = next(r for r in pipe.rules if r.multi and r.rule.id == 21)
j = pipe.joins.index(conv)
w, off, cnt = b.download_matches(j, from_join=True)
print("device", int(cnt[0]), flush=True)
v = O.rebuild(packed, symarr["rank"])
t = time.time()
rw, roff, rcnt, W = O.joint(packed, v, symarr, conv._programs, conv.var_maps, conv.pvar_maps, len(conv.var_names), len(conv.pvar_names))
print("oracle", int(rcnt[0]), round(time.time() - t, 1), "s", flush=True)
n = int(off[-1])
print("equal:", n == len(rw) and bool(np.array_equal(w[:n], rw)), flush=True)
