"""Parity of the sm_100a solver with the REFERENCE ITSELF: tests/golden/ref_*.npz are outputs
of the unmodified reference sources (oracle/_ref, tests/golden/make_ref_golden.py).  Every
rmpc_solution field is gated (tests/parity.py: tau_ff, F*[0], V_MPC, base_residual <= 1e-4
relative with unit floors; prim_res / dual_res <= 1e-3), statuses and DivergenceError
iterations must be identical.  No CPU checker runs on the GPU side of this test."""
import glob
import os

import numpy as np
import pytest

import paper_2510_12717_b200 as R
from parity import check, compare, fixture_settings, summary

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
FILES = sorted(glob.glob(os.path.join(HERE, "golden", "ref_*.npz")))


@pytest.mark.parametrize("path", FILES, ids=[os.path.basename(f) for f in FILES])
def test_device_matches_reference_outputs(path):
    g = np.load(path)
    m = R.default_model()
    s = fixture_settings(g)
    n = g["states"].shape[0]
    prev = None
    if "prev_z" in g.files:
        psol = np.zeros(n, dtype=R.SOLUTION_DTYPE)
        psol["status"] = g["prev_ok"]
        prev = (psol, g["prev_z"].astype(np.float32))
    sol, z = R.BatchRunner(n, m, s).solve(g["states"], g["cmds"], g["gaits"], prev=prev, want_z=True)
    c = compare(sol, g, z, g["z"])
    print(os.path.basename(path), summary(c))
    check(c, os.path.basename(path))
    assert c["fail_iter_equal"]
    assert c["z"].max() <= 1e-3 if c["n_ok"] else True
