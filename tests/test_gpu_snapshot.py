"""Device snapshot store (EGraph.snapshot, egraph.py:300-312): leaf states saved
from a batch's rebuild and loaded into a new batch device to device must equal the host path
(download -> LeafState -> pack_with_headroom -> upload) entry for entry, and a batch filled from
slots must rebuild, e-match and extract exactly like the host-packed one."""

import numpy as np
import pytest

from golden_io import FrozenSymtab, group_batch, load_group, rules_of

pytestmark = pytest.mark.gpu

FIELDS = ("hc_sym", "hc_koff", "hc_kids", "hc_cid", "hc_cost", "uf_parent", "uf_rank")


def _host_clean(packed, b):
    from paper_2410_05534_b200.arena import LeafState

    reb = b.download_rebuild()
    U = b.live_counts()[1]
    out = []
    for l in range(packed["n_leaves"]):
        n0, k0, u0 = (int(packed[k][l]) for k in ("node_base", "kid_base", "id_base"))
        n = int(reb["n"][l])
        koff = reb["hc_koff"][n0 + l:n0 + l + n + 1].copy()
        out.append(LeafState(reb["hc_sym"][n0:n0 + n].copy(), koff, reb["hc_kids"][k0:k0 + int(koff[-1])].copy(),
                             reb["hc_cid"][n0:n0 + n].copy(), reb["hc_cost"][n0:n0 + n].copy(),
                             reb["uf_parent"][u0:u0 + int(U[l])].copy(), reb["uf_rank"][u0:u0 + int(U[l])].copy(),
                             int(packed["root"][l])))
    return out


def _same(a, b):
    return a.root == b.root and all(np.array_equal(getattr(a, f), getattr(b, f)) for f in FIELDS)


@pytest.mark.parametrize("group", ["toy", "analog_nasrnn", "analog_resnext50"])
def test_store_roundtrip_matches_host_path(group):
    from paper_2410_05534_b200 import native
    from paper_2410_05534_b200.arena import Batch, LeafState
    from paper_2410_05534_b200.pipeline import LeafPipeline

    g = load_group(group)
    st = FrozenSymtab(g["symtab"])
    states = [LeafState.from_json(c["state"]) for c in g["cases"]][:64]
    ctx = native.Context(0)
    try:
        pipe = LeafPipeline(ctx, st.arrays, rules_of(g), st.name_id, st.code)
        store = native.SnapshotStore(ctx)
        packed = Batch(states).pack_with_headroom(nodes=64)
        b = pipe.load(packed)
        b.set_counts(packed["n_cnt"], packed["u_cnt"])
        pipe.rebuild()
        host = _host_clean(packed, b)
        slots = store.save(b, range(len(states)))
        assert [s.index for s in slots] == list(range(len(states))) and len(store) == len(states)
        for s, h in zip(slots, host):   # D2D save == host download, entry for entry
            assert (s.n, s.K, s.U) == (h.n, h.n_kids, h.n_ids)
            assert _same(store.download(s), h)
        # put (host -> slot) / download round trip
        extra = store.put(host[0])
        assert extra.index == len(states) and _same(store.download(extra), host[0])
        store.truncate(len(states))
        assert len(store) == len(states)

        # a batch loaded from slots (D2D) vs the same states packed on the host: identical arena,
        # rebuild, matches and extraction
        layout, bs = pipe.load_slots(store, slots, 128)
        want = Batch(host).pack_with_headroom(nodes=128)
        got = bs.download_state()
        for f in FIELDS:
            assert np.array_equal(got[f][:len(want[f])], want[f]), f
        assert np.array_equal(got["n"], want["n_cnt"]) and np.array_equal(got["U"], want["u_cnt"])
        pipe.rebuild()
        r_slot, x_slot = _host_clean(layout, bs), native.extract_with_retry(bs, "ocf")
        pipe.ematch()
        c_slot = bs.download_counts(len(pipe.pattern_ids))
        bh = pipe.load(want)
        bh.set_counts(want["n_cnt"], want["u_cnt"])
        pipe.rebuild()
        r_host, x_host = _host_clean(want, bh), native.extract_with_retry(bh, "ocf")
        pipe.ematch()
        c_host = bh.download_counts(len(pipe.pattern_ids))
        assert all(_same(a, b) for a, b in zip(r_slot, r_host))   # live spans (headroom is scratch)
        for k in ("status", "root_cost", "passes"):
            assert np.array_equal(x_slot[k], x_host[k]), k
        assert np.array_equal(c_slot, c_host)
        store.close()
    finally:
        ctx.close()


def test_store_rejects_oversized_slot_and_foreign_store():
    from paper_2410_05534_b200 import native
    from paper_2410_05534_b200.arena import LeafState

    g = load_group("toy")
    st = FrozenSymtab(g["symtab"])
    s0 = LeafState.from_json(g["cases"][0]["state"])
    ctx = native.Context(0)
    try:
        a, b = native.SnapshotStore(ctx), native.SnapshotStore(ctx)
        sa = a.put(s0)
        from paper_2410_05534_b200.pipeline import LeafPipeline

        pipe = LeafPipeline(ctx, st.arrays, rules_of(g), st.name_id, st.code)
        with pytest.raises(ValueError):
            pipe.load_slots(b, [sa], 4)
        layout = a.layout([sa], 0)
        layout["node_base"][1] -= 1   # span one entry short of the slot
        bt = native.DeviceBatch(ctx, layout)
        with pytest.raises(native.NativeError):
            a.load(bt, [sa])
        bt.close()
        a.close(); b.close()
    finally:
        ctx.close()
