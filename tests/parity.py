"""Parity metrics between the CUDA solver (FP32 records) and the FP64 CPU checkers (the
restated oracle, oracle/, or the reference built from its own sources, oracle/_ref).

North star (BASELINE.json): relative error <= 1e-4 in FP32 of torques, forces and the QP
objective.  Every metric is a per-agent relative error with an explicit absolute floor (a
quantity near zero has no meaningful relative error); the floors are physical scales:
  * tau_ff, F*[0], base_residual: max_k |gpu - ref| / max(max_k |ref|, 1)   (1 N m, 1 N);
    base_residual is gated at RES_TOL (see GATES)
  * V_MPC ("v"):  |gpu - ref| / max(|ref|, 1)  -- the plain relative error of the objective
    with a 1-unit floor (V is O(1..30) on the walking batches; standing gives V = 0 exactly)
  * V_MPC ("v_terms", reported only): |gpu - ref| / (|1/2 x^T P x| + |q^T x|), the error
    against the size of the two terms V is the difference of (oracle records only)
  * prim_res, dual_res (unscaled ||Ax - z||_inf, ||Px + q + A^T y||_inf after the fixed 25
    iterations, qp.cpp:192-200): |gpu - ref| / max(|ref|, RES_FLOOR).  25 ADMM iterations
    stop far from convergence (prim_res 1..20), and both are max-norms over hundreds of rows
    computed from FP32 iterates, so their bar is RES_TOL (stated, looser than 1e-4).
  * delta_inf_norm (||dz||_inf): relative, floor 1e-3.
"""
from __future__ import annotations

import numpy as np

TOL = 1e-4          # tau_ff, F*[0], V_MPC
RES_TOL = 1e-3      # prim_res, dual_res, base_residual
RES_FLOOR = 1e-2
V_FLOOR = 1.0


def rel_vec(gpu, ref, floor):
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    if gpu.ndim == 1:
        gpu, ref = gpu[:, None], ref[:, None]
    return np.max(np.abs(gpu - ref), axis=-1) / np.maximum(np.max(np.abs(ref), axis=-1), floor)


def v_err(gpu_sol, ref_sol):
    """Term-scaled objective error (oracle records carry v_quad / v_lin)."""
    scale = np.abs(ref_sol["v_quad"]) + np.abs(ref_sol["v_lin"])
    return np.abs(gpu_sol["v_mpc"].astype(np.float64) - ref_sol["v_mpc"]) / np.maximum(scale, 1e-12)


def compare(gpu_sol, ref_sol, gpu_z=None, ref_z=None):
    """Per-agent error arrays (only agents OK on both sides) and status agreement."""
    ok = (gpu_sol["status"] == 0) & (ref_sol["status"] == 0)
    out = dict(
        status_equal=bool(np.all(gpu_sol["status"] == ref_sol["status"])),
        fail_iter_equal=bool(np.all(gpu_sol["fail_iter"] == ref_sol["fail_iter"])),
        n_ok=int(ok.sum()),
        tau=rel_vec(gpu_sol["tau_ff"], ref_sol["tau_ff"], 1.0)[ok],
        f0=rel_vec(gpu_sol["f0"], ref_sol["f0"], 1.0)[ok],
        v=rel_vec(gpu_sol["v_mpc"], ref_sol["v_mpc"], V_FLOOR)[ok],
        base=rel_vec(gpu_sol["base_residual"], ref_sol["base_residual"], 1.0)[ok],
        prim=rel_vec(gpu_sol["prim_res"], ref_sol["prim_res"], RES_FLOOR)[ok],
        dual=rel_vec(gpu_sol["dual_res"], ref_sol["dual_res"], RES_FLOOR)[ok],
        q_set=np.max(np.abs(gpu_sol["q_set"] - ref_sol["q_set"]), axis=-1)[ok],
        qd_set=np.max(np.abs(gpu_sol["qd_set"] - ref_sol["qd_set"]), axis=-1)[ok],
        delta=rel_vec(gpu_sol["delta_inf_norm"], ref_sol["delta_inf_norm"], 1e-3)[ok],
    )
    names = ref_sol.dtype.names if hasattr(ref_sol, "dtype") else tuple(ref_sol.keys())
    if "v_quad" in names and np.all(np.isfinite(ref_sol["v_quad"][ok])):
        out["v_terms"] = v_err(gpu_sol, ref_sol)[ok]
    if gpu_z is not None and ref_z is not None:
        out["z"] = np.max(np.abs(gpu_z.astype(np.float64) - ref_z), axis=(1, 2))[ok]
    return out


# base_residual (rows 0..2 of M qdd + h - J^T F at node 0, robot.cpp:211-233) is a residual of
# the unconverged 25-iteration plan (10..25 N), computed from qdd = (qd*_1 - qd*_0) / dt: FP32
# plan differences amplified by 1/dt = 20, so it is gated with the residuals.
GATES = (("tau", TOL), ("f0", TOL), ("v", TOL), ("base", RES_TOL), ("prim", RES_TOL), ("dual", RES_TOL))


def fixture_settings(g):
    """MpcSettings of a tests/golden/ref_*.npz fixture."""
    from paper_2510_12717_b200.abi import default_settings
    s = default_settings(int(g["horizon"]))
    s.warm_start = int(g["warm_start"])
    if "mu" in g.files:
        s.mu, s.sigma = float(g["mu"]), float(g["sigma"])
        for k in range(8):
            s.w_f[k] = float(g["w_f"][k])
    return s


def check(c, what=""):
    """Assert every gated metric of compare() meets its tolerance."""
    assert c["status_equal"], f"{what}: statuses differ"
    for k, tol in GATES:
        mx = float(c[k].max()) if c[k].size else 0.0
        assert mx <= tol, f"{what}: {k} max rel err {mx:.3e} > {tol:g}"


def summary(c) -> str:
    def mx(a):
        return float(a.max()) if a.size else 0.0
    keys = ("tau", "f0", "v", "base", "prim", "dual", "q_set", "delta") + tuple(k for k in ("v_terms", "z") if k in c)
    return f"ok={c['n_ok']} " + " ".join(f"{k}={mx(c[k]):.2e}" for k in keys)
