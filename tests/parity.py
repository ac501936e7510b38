"""Parity metrics between the CUDA solver (FP32 records) and the FP64 CPU oracle.

Tolerances (north star, BASELINE.json): relative error <= 1e-4 in FP32 for
  * tau_ff and F*[0]: max |gpu - ref| / max(max|ref|, floor), floors 1 N m and 1 N (a near-zero
    torque vector has no meaningful relative error);
  * V_MPC: |gpu - ref| / (|1/2 x^T P x| + |q^T x|): the objective is a difference of two terms
    that can cancel to 1e-5 of their size (tools/precision_study.py), so its error is measured
    against the size of the terms it is computed from.
"""
from __future__ import annotations

import numpy as np

TOL = 1e-4


def rel_vec(gpu, ref, floor):
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return np.max(np.abs(gpu - ref), axis=-1) / np.maximum(np.max(np.abs(ref), axis=-1), floor)


def v_err(gpu_sol, ref_sol):
    scale = np.abs(ref_sol["v_quad"]) + np.abs(ref_sol["v_lin"])
    return np.abs(gpu_sol["v_mpc"].astype(np.float64) - ref_sol["v_mpc"]) / np.maximum(scale, 1e-12)


def compare(gpu_sol, ref_sol, gpu_z=None, ref_z=None):
    """Per-agent error arrays (only agents OK on both sides) and status agreement."""
    ok = (gpu_sol["status"] == 0) & (ref_sol["status"] == 0)
    out = dict(
        status_equal=bool(np.all(gpu_sol["status"] == ref_sol["status"])),
        n_ok=int(ok.sum()),
        tau=rel_vec(gpu_sol["tau_ff"], ref_sol["tau_ff"], 1.0)[ok],
        f0=rel_vec(gpu_sol["f0"], ref_sol["f0"], 1.0)[ok],
        v=v_err(gpu_sol, ref_sol)[ok],
        q_set=np.max(np.abs(gpu_sol["q_set"] - ref_sol["q_set"]), axis=-1)[ok],
        delta=rel_vec(gpu_sol["delta_inf_norm"][:, None], ref_sol["delta_inf_norm"][:, None], 1e-3)[ok],
    )
    if gpu_z is not None and ref_z is not None:
        out["z"] = np.max(np.abs(gpu_z.astype(np.float64) - ref_z), axis=(1, 2))[ok]
    return out


def summary(c) -> str:
    def mx(a):
        return float(a.max()) if a.size else 0.0
    return (f"ok={c['n_ok']} tau={mx(c['tau']):.2e} f0={mx(c['f0']):.2e} v={mx(c['v']):.2e} "
            f"q_set={mx(c['q_set']):.2e} delta={mx(c['delta']):.2e}" +
            (f" z={mx(c['z']):.2e}" if "z" in c else ""))
