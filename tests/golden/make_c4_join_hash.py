"""SHA-256 of the CPU oracle's config-4 conv-merge join (the #138-analog multi-pattern rule on the
80,257-node Inception-v3 state, 132.8M records, 4.25 GB), for tests/test_gpu_c4.py's element-wise
check of the device join. The oracle (oracle/esat_oracle.c) is pinned to the reference's own joint
match outputs (tests/test_oracle_golden.py); this run takes about a minute and 9 GB of host memory.

    python tests/golden/make_c4_join_hash.py   ->   tests/golden/c4_join_sha256.json
"""
import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

from oracle import oracle as O  # noqa: E402
from paper_2410_05534_b200.arena import Batch, LeafState  # noqa: E402
from paper_2410_05534_b200.patterns import load_rules  # noqa: E402
from paper_2410_05534_b200.pipeline import compile_rules  # noqa: E402
from paper_2410_05534_b200.symtab import NO_MATCH_CODE  # noqa: E402


def main():
    z = np.load(HERE / "c4_inception_state.npz")
    meta = json.loads(str(z["meta"]))
    lf = LeafState(z["hc_sym"], z["hc_koff"], z["hc_kids"], z["hc_cid"], z["hc_cost"], z["uf_parent"], z["uf_rank"],
                   int(z["root"]))
    symarr = {"name": z["sym_name"], "arity": z["sym_arity"], "rank": z["sym_rank"], "poff": z["sym_poff"],
              "params": z["sym_params"]}
    names = {n: i for i, n in enumerate(meta["names"])}
    codes = {(type(v), v): i for i, v in enumerate(meta["values"])}
    _, rules_c = compile_rules(load_rules("taso_analog"), lambda n: names.get(n, -1),
                               lambda v: codes.get((type(v), v), NO_MATCH_CODE))
    conv = next(r for r in rules_c if r.multi and r.rule.id == 21)
    packed = Batch([lf]).pack()
    view = O.rebuild(packed, symarr["rank"])
    t = time.time()
    words, _, cnt, W = O.joint(packed, view, symarr, conv._programs, conv.var_maps, conv.pvar_maps,
                               len(conv.var_names), len(conv.pvar_names))
    h = hashlib.sha256(np.ascontiguousarray(words, np.uint32).tobytes()).hexdigest()
    out = {"rule": 21, "records": int(cnt[0]), "words_per_record": int(W), "sha256_u32_le": h,
           "oracle_seconds": round(time.time() - t, 1),
           "generator": "tests/golden/make_c4_join_hash.py (oracle/esat_oracle.c joint match)"}
    (HERE / "c4_join_sha256.json").write_text(json.dumps(out, indent=1) + "\n")
    print(out)


if __name__ == "__main__":
    main()
