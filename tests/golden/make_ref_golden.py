"""Regenerates tests/golden/ref_*.npz: outputs of the REFERENCE ITSELF -- the unmodified
/root/reference/proj/src/*.cpp compiled into oracle/_ref/librmpc_ref.so (oracle/Makefile.ref,
against the Eigen-subset shim oracle/eigen_shim; Eigen's AMDOrdering replaced by the oracle's
minimum-degree ordering, which changes only rounding).

Each fixture holds the inputs, the settings horizon and every MpcSolution field the C ABI
returns (tau_ff, q_set, qd_set, F*[0], base_residual, v_mpc, prim_res, dual_res,
delta_inf_norm, status, fail_iter) plus z*.  tests/test_ref_pin.py checks the restated oracle
against them (<= 1e-10) and tests/test_gpu_ref_parity.py the CUDA path (north-star
tolerance).  Run here, where /root/reference exists:

    python tests/golden/make_ref_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import paper_2510_12717_b200 as R  # noqa: E402
from oracle import ref as F  # noqa: E402

FIELDS = ("tau_ff", "q_set", "qd_set", "f0", "base_residual", "v_mpc", "prim_res", "dual_res",
          "delta_inf_norm", "status", "fail_iter")

# (name, kind, horizon, agents, seed): SURVEY.md §8(d) C1 (standing, and walking at phase 0),
# C2-style random batches at N = 5 / 10 / 20, varied gaits (flight / walk / double stance /
# standing), the reference's velocity KAT input (test_mpc.cpp:261-274, default horizon 12).
CASES = [
    ("c1_standing_T10", "standing", 10, 1, 0),
    ("random_T5", "random", 5, 16, 11),
    ("random_T10", "random", 10, 32, 12),
    ("random_T20", "random", 20, 8, 13),
    ("mixed_T10", "mixed", 10, 32, 14),
    ("mixed_T12", "mixed", 12, 16, 15),
]


def save(name, m, s, st, cm, ga, prev_z=None, prev_ok=None, extra=None):
    sol, z, _, _, _ = F.solve_batch(m, s, st, cm, ga, prev_z=prev_z, prev_ok=prev_ok, workers=1)
    arrays = dict(states=st, cmds=cm, gaits=ga, horizon=np.int32(s.horizon),
                  warm_start=np.int32(s.warm_start), mu=np.float64(s.mu), sigma=np.float64(s.sigma),
                  w_f=np.array(s.w_f[:8]), z=z, **{k: sol[k] for k in FIELDS})
    if prev_z is not None:
        arrays.update(prev_z=prev_z, prev_ok=np.asarray(prev_ok, np.int32))
    if extra:
        arrays.update(extra)
    np.savez_compressed(os.path.join(HERE, f"ref_{name}.npz"), **arrays)
    print("wrote", name, "status", np.bincount(sol["status"], minlength=4))
    return sol, z


def main():
    m = R.default_model()
    nominal = F.nominal_pose(m)
    for name, kind, T, n, seed in CASES:
        s = R.default_settings(T)
        st, cm, ga = R.synthetic_batch(n, kind, seed=seed, model=m, settings=s, nominal=nominal)
        save(name, m, s, st, cm, ga)

    # C1 walking at phase 0 and the velocity KAT (cmd vx = 0.5, default gait, horizon 12)
    for name, T, vx in (("c1_walking_T10", 10, 0.0), ("kat_velocity_T12", 12, 0.5)):
        s = R.default_settings(T)
        st = np.zeros((1, 18))
        st[0, :9] = nominal
        cm = np.array([[1.0, vx, 0.0]])
        ga = np.array([[0.0, 0.8, 0.5, 0.5, 0.5, 0.0, 0.0]])
        save(name, m, s, st, cm, ga)

    # failure isolation: NaN state and NaN command next to healthy agents (mpc.cpp:70-72,
    # qp.cpp:159-161)
    s = R.default_settings(10)
    st, cm, ga = R.synthetic_batch(4, "random", seed=16, model=m, settings=s, nominal=nominal)
    st = st.copy()
    cm = cm.copy()
    st[1, 4] = np.nan
    cm[2, 1] = np.nan
    save("failures_T10", m, s, st, cm, ga)

    # SingularityError (ldl.cpp:159-164): mu = 0 leaves the stance F_z of the last node touched
    # only by explicit-zero friction entries; with sigma = 0 and w_f = 0 its KKT column is zero,
    # so the factorization meets an exact zero pivot (the device: a singular 2x2 pivot block)
    s = R.default_settings(10)
    s.mu, s.sigma = 0.0, 0.0
    for k in range(8):
        s.w_f[k] = 0.0
    st, cm, ga = R.synthetic_batch(4, "mixed", seed=18, model=m, settings=s, nominal=nominal)
    save("singular_T10", m, s, st, cm, ga)

    # warm start: tick 2 from tick 1's z* (mpc.cpp:258-265), one agent with a failed prev
    s = R.default_settings(10)
    s.warm_start = 1
    st, cm, ga = R.synthetic_batch(8, "random", seed=17, model=m, settings=s, nominal=nominal)
    sol1, z1 = save("warm_tick1_T10", m, s, st, cm, ga)
    ok = sol1["status"].copy()
    ok[3] = 2
    save("warm_tick2_T10", m, s, st, cm, ga, prev_z=z1, prev_ok=ok)


if __name__ == "__main__":
    main()
