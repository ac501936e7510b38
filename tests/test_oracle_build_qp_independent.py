"""Independent numpy restatement of build_qp (mpc.cpp:64-238) from the oracle's kinematics,
checked entry by entry against the oracle's QP.  CPU only."""
import numpy as np
import pytest

from paper_2510_12717_b200.abi import default_settings, gait_row, standing_gait_row


def numpy_build_qp(O, model, s, state, cmd, gait):
    T = s.horizon
    dt = np.array(s.dt_schedule[:T])
    nom = O.nominal_pose(model)
    stance, swt = O.horizon_schedule(gait, dt)
    W = model.total_mass() * model.gravity
    gq = np.tile(nom, (T, 1))
    gq[:, 0] = state[0]
    gqd = np.zeros((T, 9))
    gF = np.zeros((T, 8))
    for i in range(T):
        na = stance[i].sum()
        for c in range(4):
            gF[i, 2 * c + 1] = W / na if stance[i, c] and na else 0.0
    ref = O.desired_trajectory(model, s, cmd, gait)
    n = 26 * T
    wq, wqd, wf = np.array(s.w_q[:]), np.array(s.w_qd[:]), np.array(s.w_f[:])
    P = np.concatenate([np.concatenate([wq, wqd, wf]) * dt[i] for i in range(T)])
    z = np.concatenate([np.concatenate([gq[i], gqd[i], gF[i]]) for i in range(T)])
    zdes = np.concatenate([np.concatenate([ref["q_des"][i], ref["qd_des"][i], ref["F_des"][i]]) for i in range(T)])
    q = P * (z - zdes)
    rows, lo, hi = [], [], []

    def row(entries, l, h):
        a = np.zeros(n)
        for j, v in entries:
            a[j] += v
        rows.append(a)
        lo.append(l)
        hi.append(h)

    vq = lambda i, k: 26 * i + k  # noqa: E731
    vqd = lambda i, k: 26 * i + 9 + k  # noqa: E731
    vf = lambda i, k: 26 * i + 18 + k  # noqa: E731
    for k in range(9):
        row([(vq(0, k), 1.0)], state[k] - gq[0, k], state[k] - gq[0, k])
    for k in range(9):
        row([(vqd(0, k), 1.0)], state[9 + k] - gqd[0, k], state[9 + k] - gqd[0, k])
    for i in range(T - 1):
        for k in range(9):
            r = -(gq[i + 1, k] - gq[i, k] - dt[i] * gqd[i + 1, k])
            row([(vq(i + 1, k), 1.0), (vq(i, k), -1.0), (vqd(i + 1, k), -dt[i])], r, r)
    kin = [O.kinematics(model, gq[i], gqd[i]) for i in range(T)]
    for i in range(T - 1):
        M = O.mass_matrix(model, gq[i])
        h = O.bias_forces(model, gq[i], gqd[i])
        J = kin[i]["c_jac"]
        for b in range(3):
            resid = M[b] @ (gqd[i + 1] - gqd[i]) / dt[i] + h[b] - sum(J[c][:, b] @ gF[i, 2 * c:2 * c + 2] for c in range(4))
            ent = [(vqd(i + 1, k), M[b, k] / dt[i]) for k in range(9)] + [(vqd(i, k), -M[b, k] / dt[i]) for k in range(9)]
            ent += [(vf(i, 2 * c + a), -J[c][a, b]) for c in range(4) for a in range(2)]
            row(ent, -resid, -resid)
    mu = s.mu
    for i in range(T):
        for c in range(4):
            fx, fz = gF[i, 2 * c], gF[i, 2 * c + 1]
            J = kin[i]["c_jac"][c]
            if stance[i, c]:
                row([(vf(i, 2 * c), 1.0), (vf(i, 2 * c + 1), -mu)], -1e30, -(fx - mu * fz))
                row([(vf(i, 2 * c), -1.0), (vf(i, 2 * c + 1), -mu)], -1e30, -(-fx - mu * fz))
                if i == 0:
                    continue
                for ax in range(2):
                    r = -J[ax] @ gqd[i]
                    row([(vqd(i, k), J[ax, k]) for k in range(9)], r, r)
            else:
                row([(vf(i, 2 * c), 1.0)], -fx, -fx)
                row([(vf(i, 2 * c + 1), 1.0)], -fz, -fz)
                if i == 0:
                    continue
                r = ref["swing_height"][i, c] - kin[i]["c_pos"][c, 1]
                row([(vq(i, k), J[1, k]) for k in range(9)], r, r)
    for i in range(1, T):
        for k in range(6):
            row([(vq(i, 3 + k), 1.0)], model.joint_lo[k] - gq[i, 3 + k], model.joint_hi[k] - gq[i, 3 + k])
        for k in range(6):
            row([(vqd(i, 3 + k), 1.0)], -model.qd_limit[k] - gqd[i, 3 + k], model.qd_limit[k] - gqd[i, 3 + k])
    return dict(A=np.array(rows), lo=np.array(lo), hi=np.array(hi), P_diag=P, q=q)


@pytest.mark.parametrize("T,phase,standing,vx", [(3, 0.0, True, 0.0), (10, 0.3, False, 0.5),
                                                 (12, 0.0, False, 0.5), (5, 0.77, False, -0.4)])
def test_build_qp_matches_independent_restatement(oracle, model, T, phase, standing, vx):
    s = default_settings(T)
    state = np.concatenate([oracle.nominal_pose(model), np.zeros(9)])
    state[9], state[11] = 0.2, -0.1
    cmd = np.array([model.nominal_height(), vx, 0.0])
    gait = standing_gait_row() if standing else gait_row(s, phase)
    a = oracle.build_qp(model, s, state, cmd, gait)
    b = numpy_build_qp(oracle, model, s, state, cmd, gait)
    for k in ("A", "lo", "hi", "P_diag", "q"):
        np.testing.assert_allclose(a[k], b[k], rtol=1e-12, atol=1e-12, err_msg=k)
