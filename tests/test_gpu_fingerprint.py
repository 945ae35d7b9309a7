"""Device WL fingerprint (k_fingerprint) vs EGraph.fingerprint run by the reference
on every golden state (tests/golden/make_fingerprints.py): all 64 bits equal."""

import gzip
import json

import numpy as np
import pytest

from golden_io import GOLDEN, GROUPS, group_batch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("group", GROUPS)
def test_fingerprint_matches_reference(group):
    from paper_2410_05534_b200 import native
    from paper_2410_05534_b200.fingerprint import key_tables

    with gzip.open(GOLDEN / "fingerprints.json.gz") as fh:
        want = json.load(fh)[group]
    st, packed, cases = group_batch(group)
    ctx = native.Context(0)
    ctx.upload_symtab(st.arrays)
    ctx.fingerprint_setup(*key_tables([(n, a, p) for n, a, p in st.d["symbols"]]))
    b = native.DeviceBatch(ctx, packed)
    b.upload()
    b.rebuild()
    b.fingerprint()
    fp, status = b.download_fingerprint()
    bad = [(c["name"], f"{int(fp[l]):016x}", want[c["name"]]) for l, c in enumerate(cases)
           if status[l] != 0 or f"{int(fp[l]):016x}" != want[c["name"]]]
    b.close()
    ctx.close()
    assert not bad, (len(bad), len(cases), bad[:4])
