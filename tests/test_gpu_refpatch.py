"""INTEGRATION.md §1 executed: paper_2410_05534_b200.refpatch.install on the reference's OWN modules
(baseline/_ref) -- device rebuild, e-matching, greedy extraction and (second variant) apply_rule --
must leave a seeded rollout on the reference's own EGraph objects bit-identical: same rules drawn,
ApplyReports, dump() of every state, extraction costs / chosen nodes, applicability vectors."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
RUN = Path(__file__).resolve().parent / "_refpatch_run.py"


def _run(mode):
    p = subprocess.run([sys.executable, str(RUN), mode], capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    return json.loads(p.stdout.strip().splitlines()[-1])


def test_refpatch_leaves_reference_rollouts_identical():
    from oracle.mcts_ref import reference_available

    if not reference_available():
        pytest.skip("reference not importable (baseline/_ref missing)")
    stock = _run("stock")
    assert all(len(r) > 0 for runs in stock.values() for r in runs)
    assert _run("device") == stock
    assert _run("device_apply") == stock
