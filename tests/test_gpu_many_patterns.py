"""e-match calls with more than 32 patterns (one k_ematch launch per 32-pattern chunk):
every call-pattern's match records, EXISTS answers, per-leaf masks and joins over sources in later
chunks must equal those of the same patterns matched in one <= 32-pattern call, which
test_gpu_parity pins to the reference."""

import numpy as np
import pytest

from golden_io import compile_rule, group_batch, load_group, rules_of

pytestmark = pytest.mark.gpu

REPS = 3   # 24 analog source patterns x 3 = 72 call-patterns: three chunks, the last one partial


@pytest.fixture(scope="module")
def setup():
    from paper_2410_05534_b200 import native

    ctx = native.Context(0)
    group = "analog_nasrnn"
    st, packed, cases = group_batch(group)
    ctx.upload_symtab(st.arrays)
    progs, multis = [], []
    for r in rules_of(load_group(group)):
        comps, vn, qn, vm, qm = compile_rule(r, st)
        ids = []
        for cp in comps:
            ids.append(len(progs))
            progs.append(cp.program)
        if r.kind != "single":
            multis.append((ids, vm, qm, len(vn), len(qn)))
    ctx.upload_patterns(progs)
    b = native.DeviceBatch(ctx, packed)
    b.upload()
    b.rebuild()
    P = len(progs)
    b.ematch(list(range(P)))
    base = [tuple(x.copy() for x in b.download_matches(p)) for p in range(P)]
    b.join(multis)
    base_join = [tuple(x.copy() for x in b.download_matches(j, from_join=True)) for j in range(len(multis))]
    yield ctx, b, P, base, multis, base_join
    b.close()
    ctx.close()


def _same(got, want, L):
    """Counts and every leaf's records (download_matches: per-leaf word ranges [off[l], off[l+1]))."""
    if not np.array_equal(got[2], want[2]):
        return False
    return all(np.array_equal(got[0][int(got[1][l]):int(got[1][l + 1])], want[0][int(want[1][l]):int(want[1][l + 1])])
               for l in range(L))


def test_list_mode_beyond_32_patterns(setup):
    ctx, b, P, base, multis, base_join = setup
    ids = list(range(P)) * REPS
    assert len(ids) > 64
    b.ematch(ids)
    for i, p in enumerate(ids):
        assert _same(b.download_matches(i), base[p], b.n_leaves), (i, p)


def test_exists_and_masks_beyond_32_patterns(setup):
    from paper_2410_05534_b200 import native

    ctx, b, P, base, multis, base_join = setup
    ids = list(range(P)) * REPS
    L = b.n_leaves
    b.ematch(ids, mode=native.MATCH_EXISTS)
    cnt = b.download_counts(len(ids))
    for i, p in enumerate(ids):
        assert np.array_equal(cnt[i] > 0, base[p][2] > 0), (i, p)
    nch = (len(ids) + 31) // 32
    rng = np.random.default_rng(7)
    mask = rng.integers(0, 1 << 32, size=(nch, L), dtype=np.uint64).astype(np.uint32)
    b.ematch(ids, leaf_mask=mask)
    cnt = b.download_counts(len(ids))
    for i, p in enumerate(ids):
        on = ((mask[i // 32] >> np.uint32(i % 32)) & 1).astype(bool)
        assert np.array_equal(cnt[i], np.where(on, base[p][2], 0)), (i, p)
    with pytest.raises(ValueError):
        b.ematch(ids, leaf_mask=mask[0])


def test_join_over_sources_in_later_chunks(setup):
    ctx, b, P, base, multis, base_join = setup
    if not multis:
        pytest.skip("no multi-pattern rule in the group")
    ids = list(range(P)) * REPS
    b.ematch(ids)
    shift = P * (REPS - 1)   # the same sources, as call-patterns of the last chunk
    b.join([([s + shift for s in src], vm, qm, nv, nq) for src, vm, qm, nv, nq in multis])
    for j in range(len(multis)):
        assert _same(b.download_matches(j, from_join=True), base_join[j], b.n_leaves), j
