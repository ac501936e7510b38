"""Design probe (not product, not a test): FP32 accuracy of candidate GPU formulations of the
25-iteration ADMM solve against the FP64 CPU oracle (reference algorithm: KKT + sparse LDL^T).

Formulations (identical iterates in exact arithmetic, qp.cpp:156-190):
  kkt   : the reference's quasi-definite KKT solve, in FP32 (oracle precision=32)
  dense : reduced SPD system (P^ + sigma I + rho A^T A) x~ = sigma x - q^ + A^T (rho z - y),
          z~ = A^ x~, solved densely in FP32 (LU)
  block : the same reduced system by block-tridiagonal elimination over horizon nodes with
          explicit Schur-complement inverses S_i^-1 (the planned warp-per-agent kernel)

Usage: python tools/precision_study.py [n_agents] [horizon]
"""
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import oracle as O  # noqa: E402
from paper_2510_12717_b200.abi import default_model, default_settings, gait_row  # noqa: E402

NV = 26


def ruiz(P_diag, A, passes, dtype):
    n, m = A.shape[1], A.shape[0]
    P = P_diag.astype(dtype).copy()
    Ah = A.astype(dtype).copy()
    e = np.ones(n, dtype)
    d = np.ones(m, dtype)
    for _ in range(passes):
        absA = np.abs(Ah)
        cn = np.maximum(np.abs(P), absA.max(axis=0) if m else 0)
        rn = absA.max(axis=1)
        de = np.where(cn > 0, 1 / np.sqrt(cn), 1).astype(dtype)
        dd = np.where(rn > 0, 1 / np.sqrt(rn), 1).astype(dtype)
        P = P * de * de
        Ah = Ah * dd[:, None] * de[None, :]
        e *= de
        d *= dd
    return e, d


def admm_reduced(qp, iters, dtype, mode, T, sigma=1e-6, rho=0.1, alpha=1.6):
    A, Pd, q, lo, hi = qp["A"], qp["P_diag"], qp["q"], qp["lo"], qp["hi"]
    e, d = ruiz(Pd, A, 10, dtype)
    A_s = (A.astype(dtype) * d[:, None]) * e[None, :]
    P_s = Pd.astype(dtype) * e * e
    q_s = q.astype(dtype) * e
    lo_s = np.where(lo <= -1e29, -np.inf, lo).astype(dtype) * d
    hi_s = np.where(hi >= 1e29, np.inf, hi).astype(dtype) * d
    n, m = A.shape[1], A.shape[0]
    H = (np.diag(P_s + dtype(sigma)) + dtype(rho) * (A_s.T @ A_s)).astype(dtype)
    if mode == "dense":
        solve = lambda r: np.linalg.solve(H, r).astype(dtype)  # noqa: E731
    else:
        # block tridiagonal: S_0 = H_00, S_{i+1} = H_{i+1,i+1} - C_i S_i^-1 C_i^T
        Sinv, C = [], []
        S = H[:NV, :NV].copy()
        for i in range(T):
            Si = np.linalg.inv(S).astype(dtype)
            Sinv.append(Si)
            if i + 1 < T:
                Ci = H[(i + 1) * NV:(i + 2) * NV, i * NV:(i + 1) * NV]
                C.append(Ci)
                S = (H[(i + 1) * NV:(i + 2) * NV, (i + 1) * NV:(i + 2) * NV] - Ci @ Si @ Ci.T).astype(dtype)

        def solve(r):
            u = [None] * T
            s = [None] * T
            u[0] = r[:NV].copy()
            for i in range(T):
                s[i] = Sinv[i] @ u[i]
                if i + 1 < T:
                    u[i + 1] = r[(i + 1) * NV:(i + 2) * NV] - C[i] @ s[i]
            x = [None] * T
            x[T - 1] = s[T - 1]
            for i in range(T - 2, -1, -1):
                x[i] = s[i] - Sinv[i] @ (C[i].T @ x[i + 1])
            return np.concatenate(x).astype(dtype)
    x = np.zeros(n, dtype)
    y = np.zeros(m, dtype)
    z = np.zeros(m, dtype)
    a, r_, s_ = dtype(alpha), dtype(rho), dtype(sigma)
    for _ in range(iters):
        rhs = s_ * x - q_s + A_s.T @ (r_ * z - y)
        xt = solve(rhs)
        zt = A_s @ xt
        x = a * xt + (1 - a) * x
        w = a * zt + (1 - a) * z
        z = np.minimum(np.maximum(w + y / r_, lo_s), hi_s)
        y = y + r_ * (w - z)
    return (x.astype(np.float64) * e), (y * d).astype(np.float64), (z / d).astype(np.float64)


def outputs_from_x(model, settings, state, gait, x):
    """z* = guess + x and inverse dynamics at node 0 (mpc.cpp:305-330), in FP64."""
    T = settings.horizon
    nom = O.nominal_pose(model)
    stance, _ = O.horizon_schedule(gait, np.array(settings.dt_schedule[:T]))
    W = model.total_mass() * model.gravity
    g = np.zeros((T, NV))
    for i in range(T):
        g[i, :9] = nom
        g[i, 0] = state[0]
        na = stance[i].sum()
        for c in range(4):
            g[i, 18 + 2 * c + 1] = W / na if (stance[i, c] and na > 0) else 0.0
    z = g + x.reshape(T, NV)
    qdd = (z[1, 9:18] - z[0, 9:18]) / settings.dt_schedule[0]
    tau, base = O.inverse_dynamics(model, z[0, :9], z[0, 9:18], qdd, z[0, 18:])
    return tau, z[0, 18:], z


def rel(a, b):
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    model, settings = default_model(), default_settings(T)
    nom = O.nominal_pose(model)
    rng = np.random.default_rng(1)
    states = np.tile(np.concatenate([nom, np.zeros(9)]), (n, 1))
    states[:, 9] = rng.uniform(-0.5, 0.5, n)
    states[:, 11] = rng.uniform(-0.5, 0.5, n)
    cmds = np.tile([1.0, 0.0, 0.0], (n, 1))
    cmds[:, 1] = rng.uniform(-0.6, 0.6, n)
    gaits = np.tile(gait_row(settings), (n, 1))
    gaits[:, 0] = rng.uniform(0, 1, n)
    ref64, z64, _, _ = O.solve_batch(model, settings, states, cmds, gaits)
    ref32, _, _, _ = O.solve_batch(model, settings, states, cmds, gaits, precision=32)
    res = {k: [] for k in ("kkt32", "dense32", "block32", "block64")}
    for i in range(n):
        r = ref64[i]
        res["kkt32"].append((rel(ref32[i]["tau_ff"], r["tau_ff"]), rel(ref32[i]["f0"], r["f0"]),
                             abs(ref32[i]["v_mpc"] - r["v_mpc"]) / abs(r["v_mpc"])))
        qp = O.build_qp(model, settings, states[i], cmds[i], gaits[i])
        for key, dt, mode in (("dense32", np.float32, "dense"), ("block32", np.float32, "block"),
                              ("block64", np.float64, "block")):
            x, y, z = admm_reduced(qp, settings.n_qp, dt, mode, T)
            tau, f0, _ = outputs_from_x(model, settings, states[i], gaits[i], x)
            v = 0.5 * np.sum(qp["P_diag"] * x * x) + qp["q"] @ x
            res[key].append((rel(tau, r["tau_ff"]), rel(f0, r["f0"]), abs(v - r["v_mpc"]) / abs(r["v_mpc"])))
    print(f"N={T} agents={n}: max / median relative error (tau_ff, F0, V_MPC)")
    for k, v in res.items():
        a = np.array(v)
        print(f"  {k:8s} max {a.max(0)}  median {np.median(a, 0)}")


if __name__ == "__main__":
    main()
