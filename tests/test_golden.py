"""Golden fixtures (tests/golden/, made by tests/golden/make_golden.py from the FP64 oracle):
the oracle reproduces them bit for bit (a guard on the restatement), and on a B200 the device
solve of the same inputs meets the parity tolerances against them (no oracle call needed on
the GPU side of this test)."""
import glob
import os

import numpy as np
import pytest

import paper_2510_12717_b200 as R
from parity import TOL

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FILES = sorted(glob.glob(os.path.join(HERE, "oracle_*.npz")))


def _case(path):
    name = os.path.basename(path)[len("oracle_"):-len(".npz")]
    kind, T, n, seed = name.split("_")
    return kind, int(T[1:]), int(n[1:]), int(seed[1:])


def test_fixtures_present():
    assert len(FILES) >= 4


@pytest.mark.parametrize("path", FILES, ids=[os.path.basename(f) for f in FILES])
def test_oracle_reproduces_golden(oracle, path):
    g = np.load(path)
    kind, T, n, seed = _case(path)
    m, s = R.default_model(), R.default_settings(T)
    sol, z, _, _ = oracle.solve_batch(m, s, g["states"], g["cmds"], g["gaits"], workers=1)
    for k in ("tau_ff", "f0", "q_set", "qd_set", "v_mpc", "status"):
        assert sol[k].tobytes() == g[k].tobytes(), k
    assert z.tobytes() == g["z"].tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("path", FILES, ids=[os.path.basename(f) for f in FILES])
def test_device_matches_golden(path):
    g = np.load(path)
    kind, T, n, seed = _case(path)
    m, s = R.default_model(), R.default_settings(T)
    sol, z = R.BatchRunner(n, m, s).solve(g["states"], g["cmds"], g["gaits"], want_z=True)
    assert (sol["status"] == g["status"]).all()
    floor_t = np.maximum(np.abs(g["tau_ff"]), 1.0)
    floor_f = np.maximum(np.abs(g["f0"]), 1.0)
    assert (np.abs(sol["tau_ff"] - g["tau_ff"]) / floor_t).max() <= TOL
    assert (np.abs(sol["f0"] - g["f0"]) / floor_f).max() <= TOL
    assert np.abs(z - g["z"]).max() <= 1e-3
