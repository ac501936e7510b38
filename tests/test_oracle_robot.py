"""Oracle robot model pinned to /root/reference/proj/tests/test_robot.cpp.  CPU only."""
import numpy as np
import pytest


def random_q(r):
    q = np.empty(9)
    q[0] = r.uniform(-1, 1)
    q[1] = r.uniform(0.6, 1.2)
    q[2] = r.uniform(-0.5, 0.5)
    q[3:] = r.uniform(-0.8, 0.8, 6)
    q[4] = r.uniform(0.2, 1.5)
    q[7] = r.uniform(0.2, 1.5)
    return q


def kinetic(O, m, q, qd):
    k = O.kinematics(m, q, qd)
    mass = [m.torso_mass, m.thigh_mass, m.shank_mass, m.foot_mass, m.thigh_mass, m.shank_mass, m.foot_mass]
    inert = [m.torso_inertia, m.thigh_inertia, m.shank_inertia, m.foot_inertia, m.thigh_inertia,
             m.shank_inertia, m.foot_inertia]
    chains = [[2], [2, 3], [2, 3, 4], [2, 3, 4, 5], [2, 6], [2, 6, 7], [2, 6, 7, 8]]
    ke = 0.0
    for l in range(7):
        ke += 0.5 * mass[l] * np.sum(k["com_vel"][l] ** 2) + 0.5 * inert[l] * qd[chains[l]].sum() ** 2
    return ke


def potential(O, m, q):
    k = O.kinematics(m, q, np.zeros(9))
    mass = [m.torso_mass, m.thigh_mass, m.shank_mass, m.foot_mass, m.thigh_mass, m.shank_mass, m.foot_mass]
    return sum(mass[l] * m.gravity * k["com_pos"][l, 1] for l in range(7))


def test_mass_matrix_spd(oracle, model):
    """test_robot.cpp:57-67 (1000 random q)."""
    r = np.random.default_rng(1)
    for _ in range(1000):
        M = oracle.mass_matrix(model, random_q(r))
        assert np.max(np.abs(M - M.T)) <= 1e-12
        np.linalg.cholesky(M)


def test_mass_matrix_xx_is_total_mass(oracle, model):
    """test_robot.cpp:69-76."""
    r = np.random.default_rng(2)
    for _ in range(10):
        assert oracle.mass_matrix(model, random_q(r))[0, 0] == pytest.approx(model.total_mass(), rel=1e-12)


def test_mass_matrix_momentum_fd(oracle, model):
    """test_robot.cpp:78-99: KE = 1/2 qd^T M qd and p = dKE/dqd by central differences."""
    r = np.random.default_rng(3)
    for _ in range(10):
        q, qd = random_q(r), r.normal(size=9)
        M = oracle.mass_matrix(model, q)
        assert kinetic(oracle, model, q, qd) == pytest.approx(0.5 * qd @ M @ qd, rel=1e-10)
        h = 1e-6
        for i in range(9):
            e = np.zeros(9)
            e[i] = h
            fd = (kinetic(oracle, model, q, qd + e) - kinetic(oracle, model, q, qd - e)) / (2 * h)
            assert (M @ qd)[i] == pytest.approx(fd, rel=1e-6, abs=1e-9)


def test_bias_at_rest_is_potential_gradient(oracle, model):
    """test_robot.cpp:101-117."""
    r = np.random.default_rng(4)
    for _ in range(10):
        q = random_q(r)
        h = oracle.bias_forces(model, q, np.zeros(9))
        for i in range(9):
            e = np.zeros(9)
            e[i] = 1e-6
            fd = (potential(oracle, model, q + e) - potential(oracle, model, q - e)) / 2e-6
            assert h[i] == pytest.approx(fd, rel=1e-5, abs=1e-7)


def test_bias_z_is_weight(oracle, model):
    """test_robot.cpp:119-125."""
    h = oracle.bias_forces(model, random_q(np.random.default_rng(5)), np.zeros(9))
    assert h[1] == pytest.approx(model.total_mass() * model.gravity, rel=1e-12)
    assert abs(h[0]) <= 1e-12


def test_contacts_touch_ground_at_nominal(oracle, model):
    """test_robot.cpp:154-165."""
    q = oracle.nominal_pose(model)
    k = oracle.kinematics(model, q, np.zeros(9))
    assert np.all(np.abs(k["c_pos"][:, 1]) <= 1e-12) and np.all(k["c_vel"] == 0)
    assert k["c_pos"][2, 0] > k["c_pos"][0, 0]


def test_contact_jacobian_fd(oracle, model):
    """test_robot.cpp:167-191: v = J qd and J = d pos / dq."""
    r = np.random.default_rng(7)
    for _ in range(5):
        q, qd = random_q(r), r.normal(size=9)
        k = oracle.kinematics(model, q, qd)
        for c in range(4):
            assert np.linalg.norm(k["c_vel"][c] - k["c_jac"][c] @ qd) < 1e-10
            for i in range(9):
                e = np.zeros(9)
                e[i] = 1e-6
                fd = (oracle.kinematics(model, q + e, qd)["c_pos"][c] -
                      oracle.kinematics(model, q - e, qd)["c_pos"][c]) / 2e-6
                assert np.all(np.abs(k["c_jac"][c][:, i] - fd) < 1e-5)


def test_static_stance_equilibrium(oracle, model):
    """test_robot.cpp:205-214: weight/4 per contact balances the base at the nominal pose."""
    q = oracle.nominal_pose(model)
    F = np.zeros(8)
    F[1::2] = model.total_mass() * model.gravity / 4
    _, base = oracle.inverse_dynamics(model, q, np.zeros(9), np.zeros(9), F)
    assert np.max(np.abs(base)) < 1e-6


def test_inverse_dynamics_gravity_compensation(oracle, model):
    """test_robot.cpp:216-224."""
    q = random_q(np.random.default_rng(9))
    tau, _ = oracle.inverse_dynamics(model, q, np.zeros(9), np.zeros(9), np.zeros(8))
    assert np.max(np.abs(tau - oracle.bias_forces(model, q, np.zeros(9))[3:])) < 1e-12


def test_inverse_dynamics_dense_recomputation(oracle, model):
    """test_robot.cpp:234-252: tau = (M qdd + h - J^T F)[3:]."""
    r = np.random.default_rng(10)
    for _ in range(10):
        q, qd, qdd = random_q(r), r.normal(size=9), 3 * r.normal(size=9)
        F = 30 * r.normal(size=8)
        tau, base = oracle.inverse_dynamics(model, q, qd, qdd, F)
        gen = oracle.mass_matrix(model, q) @ qdd + oracle.bias_forces(model, q, qd)
        k = oracle.kinematics(model, q, qd)
        for c in range(4):
            gen -= k["c_jac"][c].T @ F[2 * c:2 * c + 2]
        assert np.max(np.abs(tau - gen[3:])) < 1e-9 and np.max(np.abs(base - gen[:3])) < 1e-9


def test_inverse_dynamics_linear(oracle, model):
    """test_robot.cpp:254-274."""
    r = np.random.default_rng(11)
    q, qd = random_q(r), r.normal(size=9)
    a1, a2, f1, f2 = r.normal(size=9), r.normal(size=9), r.normal(size=8), r.normal(size=8)
    t0, _ = oracle.inverse_dynamics(model, q, qd, np.zeros(9), np.zeros(8))
    ta, _ = oracle.inverse_dynamics(model, q, qd, a1, f1)
    tb, _ = oracle.inverse_dynamics(model, q, qd, a2, f2)
    tab, _ = oracle.inverse_dynamics(model, q, qd, a1 + a2, f1 + f2)
    assert np.max(np.abs((tab - t0) - (ta - t0) - (tb - t0))) < 1e-10


def test_pd_torque_examples(oracle, model):
    """test_robot.cpp:276-301."""
    q = oracle.nominal_pose(model)
    qj, ff = q[3:], np.full(6, 3.0)
    assert np.all(oracle.pd_torque(model, qj, np.zeros(6), q, np.zeros(9), ff) == ff)
    tau = oracle.pd_torque(model, qj + 1.0, np.ones(6), q, np.zeros(9), np.zeros(6))
    np.testing.assert_allclose(tau, np.minimum(31.0, np.array(model.tau_limit)))
    big = oracle.pd_torque(model, qj + 10.0, np.zeros(6), q, np.zeros(9), np.zeros(6))
    assert np.all(big == np.array(model.tau_limit))


def test_nominal_pose_limits_and_height(oracle, model):
    """test_robot.cpp:303-311."""
    q = oracle.nominal_pose(model)
    assert q[1] == pytest.approx(model.nominal_height())
    assert np.all(q[3:] >= np.array(model.joint_lo)) and np.all(q[3:] <= np.array(model.joint_hi))
