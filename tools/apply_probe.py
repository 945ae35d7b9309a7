"""Probe: statistics of the device apply parity run (not collected by pytest)."""
import sys
import numpy as np
sys.path.insert(0, "tests")
import test_gpu_apply as T
from golden_io import FrozenSymtab, load_group, rules_of
from paper_2410_05534_b200 import native
from paper_2410_05534_b200.arena import Batch, LeafState
from paper_2410_05534_b200.pipeline import LeafPipeline

for group, (lang, cm, co) in T.GROUPS.items():
    g = load_group(group); fs = FrozenSymtab(g["symtab"]); cases = g["cases"]
    pairs = T.consecutive_pairs(cases)
    rules = rules_of(g); pos = {r.id: i for i, r in enumerate(rules)}
    pre = [LeafState.from_json(cases[a]["state"]) for a, _ in pairs]
    packed = Batch(pre).pack_with_headroom(nodes=2048)
    ctx = native.Context(0)
    pipe = LeafPipeline(ctx, fs.arrays, rules, fs.name_id, fs.code)
    b = pipe.load(packed); b.set_counts(packed["n_cnt"], packed["u_cnt"])
    pipe.rebuild(); pipe.ematch()
    off, words = pipe.apply_programs(fs.name_id, fs.code)
    ctx.apply_setup(lang, cm, co, T.frozen_symbol_arrays(fs), off, words)
    b.apply(np.array([pos[cases[p]["rule"]] for _, p in pairs], np.uint32))
    r = b.download_apply(); st = b.download_state()
    rb = b.download_rebuild()
    added = int(st["n"].sum() - rb["n"].sum())
    rep = r["report"]
    print(group, "pairs", len(pairs), "status", np.bincount(r["status"]), "matches", int(rep[:, 0].sum()),
          "changed", int(rep[:, 1].sum()), "cycles", int(rep[:, 2].sum()), "shape", int(rep[:, 3].sum()),
          "new nodes", added, flush=True)
