"""Generate the config-4 explosion-stress state ON THE DEVICE (needs a B200):

    python tests/golden/make_c4_state.py [out.npz]

Inception-v3 analog + TASO-analog rules, TENSAT-style sequential saturation with the multi-pattern
rules applied every iteration (saturate.saturate_sequential, k_multi unbounded) until the node
count passes 50,000: the conv-merge rule's third application explodes the e-graph (~80k e-nodes).
Every application is the device apply loop, which tests/test_gpu_apply.py pins bit-exactly to the
reference's rollouts. The saved state is the input of tests/test_gpu_c4.py (device vs CPU oracle at
full size) and of the config-4 measurement.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))


def main():
    from paper_2410_05534_b200 import analogs
    from paper_2410_05534_b200 import tensor_ir as T
    from paper_2410_05534_b200.cost_model import CostModelConfig
    from paper_2410_05534_b200.patterns import load_rules
    from paper_2410_05534_b200.saturate import saturate_sequential

    out = Path(sys.argv[1]) if len(sys.argv) > 1 else HERE / "c4_inception_state.npz"
    eg = T.graph_to_egraph(analogs.build_analog("inception_v3", T.GraphBuilder))
    state, st, trace = saturate_sequential(eg, load_rules("taso_analog"), CostModelConfig(), node_limit=50000,
                                           k_multi=1000, log=lambda m: print(m, flush=True))
    arr = st.arrays()
    np.savez_compressed(out, hc_sym=state.hc_sym, hc_koff=state.hc_koff, hc_kids=state.hc_kids, hc_cid=state.hc_cid,
                        hc_cost=state.hc_cost, uf_parent=state.uf_parent, uf_rank=state.uf_rank,
                        root=np.array(state.root, np.uint32), sym_name=arr["name"], sym_arity=arr["arity"],
                        sym_rank=arr["rank"], sym_poff=arr["poff"], sym_params=arr["params"],
                        meta=np.array(json.dumps({"names": st.names, "values": st.values,
                                                  "symbols": [[s.name, s.arity, repr(s.payload)] for s in st.symbols],
                                                  "trace": trace})))
    print(f"wrote {out}: {state.n} e-nodes, {len(trace)} applications")


if __name__ == "__main__":
    main()
