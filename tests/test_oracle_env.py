"""The CPU restatement of the closed-loop step (oracle/rmpc_oracle_env.hpp) against the
reference's definitions: Terrain (env.cpp:8-27) from the reference Rng streams, the dynamics
physics_step integrates (momentum balance of M qdd = tau - h + J^T F, env.cpp:38-68),
advance_phase (gait.cpp:31-35), blend / mpc_torque (policy.cpp:133-157, robot.cpp:235-241)
and observe (policy.cpp:104-122).  The reference ships no env test (tests/CMakeLists.txt
names test_env.cpp, absent), so these pin the restatement by construction.  CPU only."""
import numpy as np
import pytest

from paper_2510_12717_b200.abi import SOLUTION_DTYPE, default_model
from paper_2510_12717_b200.synthetic import Xoshiro


def heights_numpy(amplitude=0.04, cell=0.3, extent=80.0, seed=0):
    n = int(extent / cell) + 2
    x = Xoshiro(seed, [0x7e22])
    return np.array([x.uniform(-amplitude, amplitude)[0] for _ in range(n)])


def height_numpy(h, x, cell=0.3, extent=80.0):
    fx = (x + 0.5 * extent) / cell
    if fx <= 0.0:
        return h[0]
    if fx >= len(h) - 1:
        return h[-1]
    i = int(fx)
    t = fx - i
    s = t * t * (3.0 - 2.0 * t)
    return h[i] * (1.0 - s) + h[i + 1] * s


def test_terrain_flat_and_heightfield(oracle):
    c = oracle.env_config_default()
    assert all(oracle.terrain_height_at(c, x) == 0.0 for x in (-100.0, 0.0, 3.7))
    c.terrain_kind = 1
    h = heights_numpy()
    for x in (-60.0, -40.0, -39.99, -1.234, 0.0, 0.15, 7.77, 39.8, 45.0):
        assert oracle.terrain_height_at(c, x) == height_numpy(h, x)
    assert np.abs(h).max() <= 0.04 and len(h) == 268


def _state(q, qd=None):
    s = np.zeros((1, 18))
    s[0, :9] = q
    if qd is not None:
        s[0, 9:] = qd
    return s


def _com_velocity(oracle, m, q, qd):
    k = oracle.kinematics(m, q, qd)
    ml = np.array([m.torso_mass, m.thigh_mass, m.shank_mass, m.foot_mass, m.thigh_mass,
                   m.shank_mass, m.foot_mass])
    return (ml[:, None] * k["com_vel"]).sum(0) / ml.sum()


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_free_flight_momentum_balance(oracle, seed):
    """Airborne, one substep: rows 0/1 of M qdd + h = S^T tau are the total linear momentum
    balance sum_l m_l (J_l qdd + Jdot_l qd) = (0, -M g), so with J at the pre-step q the CoM
    velocity moves by -dt sum_l m_l Jdot_l qd / M + (0, -g dt) for any joint torque."""
    rng = np.random.default_rng(seed)
    m = default_model()
    c = oracle.env_config_default()
    c.substeps = 1
    q = oracle.nominal_pose(m) + rng.uniform(-0.2, 0.2, 9)
    q[1] += 3.0  # far above the ground: no contact force
    qd = rng.uniform(-1, 1, 9)
    tau = rng.uniform(-20, 20, (1, 6))
    gait = np.array([[0.3, 0.8, 0.5, 0.5, 0.5, 0.0, 0.0]])
    st, ga, status = oracle.physics_step_batch(m, c, _state(q, qd), gait, tau)
    assert status[0] == 0
    qd1 = st[0, 9:]
    dv = _com_velocity(oracle, m, q, qd1) - _com_velocity(oracle, m, q, qd)
    ml = np.array([m.torso_mass, m.thigh_mass, m.shank_mass, m.foot_mass, m.thigh_mass,
                   m.shank_mass, m.foot_mass])
    jdq = (ml[:, None] * oracle.kinematics(m, q, qd)["com_jdq"]).sum(0) / ml.sum()
    expect = -c.control_dt * jdq + [0.0, -m.gravity * c.control_dt]
    np.testing.assert_allclose(dv, expect, rtol=0, atol=1e-12)
    np.testing.assert_allclose(st[0, :9], q + c.control_dt * qd1, rtol=0, atol=1e-15)
    assert ga[0, 0] == pytest.approx(0.3 + 0.01 / 0.8)


def test_phase_wraps(oracle):
    m, c = default_model(), oracle.env_config_default()
    q = oracle.nominal_pose(m)
    q[1] += 2.0
    _, ga, _ = oracle.physics_step_batch(m, c, _state(q), np.array([[0.995, 0.8, 0.5, 0.5, 0.5, 0, 0]]),
                                         np.zeros((1, 6)))
    assert ga[0, 0] == pytest.approx((0.995 + 0.0125) % 1.0)


def test_penetration_pushes_up_and_friction_opposes_slip(oracle):
    m, c = default_model(), oracle.env_config_default()
    c.substeps = 1
    q = oracle.nominal_pose(m)
    q[1] -= 0.01  # every contact 1 cm into the ground
    qd = np.zeros(9)
    qd[0] = 0.3  # sliding forward
    st, _, _ = oracle.physics_step_batch(m, c, _state(q, qd), np.zeros((1, 7)) + [0, .8, .5, .5, .5, 0, 0],
                                         np.zeros((1, 6)))
    dv = _com_velocity(oracle, m, q, st[0, 9:]) - _com_velocity(oracle, m, q, qd)
    assert dv[1] > -m.gravity * c.control_dt  # the springs carry more than the weight
    assert dv[0] < -0.01                       # Coulomb-tanh friction decelerates the slide
    # mass scale and friction enter through rmpc_body
    st2, _, _ = oracle.physics_step_batch(m, c, _state(q, qd), np.zeros((1, 7)) + [0, .8, .5, .5, .5, 0, 0],
                                          np.zeros((1, 6)), bodies=[[0.0, 1.0]])
    dv2 = _com_velocity(oracle, m, q, st2[0, 9:]) - _com_velocity(oracle, m, q, qd)
    assert dv2[0] == pytest.approx(0.0, abs=1e-9)  # mu = 0: no horizontal force at all


def _solutions(n, rng, status=None):
    s = np.zeros(n, SOLUTION_DTYPE)
    s["tau_ff"] = rng.uniform(-20, 20, (n, 6))
    s["q_set"] = rng.uniform(-1, 1, (n, 6))
    s["qd_set"] = rng.uniform(-1, 1, (n, 6))
    s["v_mpc"] = rng.uniform(-5, 5, n)
    s["status"] = 0 if status is None else status
    return s


def test_blend_strategies(oracle):
    rng = np.random.default_rng(3)
    m, c = default_model(), oracle.env_config_default()
    n = 6
    q = np.tile(oracle.nominal_pose(m), (n, 1)) + rng.uniform(-0.1, 0.1, (n, 9))
    q[:, 1] += 2.0
    st = np.concatenate([q, rng.uniform(-1, 1, (n, 9))], 1)
    ga = np.tile([0.1, 0.8, 0.5, 0.5, 0.5, 0, 0], (n, 1))
    sols = _solutions(n, rng, status=[0, 0, 0, 0, 0, 2])
    act = rng.uniform(-0.3, 0.3, (n, 6))
    kp, kd, lim = np.array(m.kp), np.array(m.kd), np.array(m.tau_limit)

    def mpc(i):
        return np.clip(kp * (sols["q_set"][i] - st[i, 3:9]) + kd * (sols["qd_set"][i] - st[i, 12:18])
                       + sols["tau_ff"][i], -lim, lim)
    for strategy in (0, 1, 2):
        _, _, tau0, _ = oracle.control_step_batch(m, c, sols, st, ga, act, strategy, 0.0)
        for i in range(5):  # lambda = 0: every strategy is the plain MPC torque
            np.testing.assert_allclose(tau0[i], mpc(i), rtol=0, atol=1e-5)
        assert not tau0[5].any()  # failed solution: zero torque (ppo.cpp:345-349)
    _, _, tau2, _ = oracle.control_step_batch(m, c, sols, st, ga, act, 2, 0.5)
    for i in range(5):
        np.testing.assert_allclose(tau2[i], np.clip(mpc(i) + 0.5 * act[i], -lim, lim), atol=1e-5)
    _, _, tau1, _ = oracle.control_step_batch(m, c, sols, st, ga, act, 1, 0.5)
    qhat = oracle.nominal_pose(m)[3:]
    for i in range(5):
        res = kp * (act[i] + qhat - st[i, 3:9]) - kd * st[i, 12:18]
        np.testing.assert_allclose(tau1[i], np.clip(mpc(i) + 0.5 * res, -lim, lim), atol=1e-5)


def test_observe_layout(oracle):
    rng = np.random.default_rng(4)
    n = 3
    st = rng.uniform(-1, 1, (n, 18))
    ga = np.tile([0.3, 0.8, 0.5, 0.5, 0.5, 0.0, 0.0], (n, 1))
    sols = _solutions(n, rng, status=[0, 0, 3])
    o = oracle.observe_batch(st, ga, sols)
    assert o.shape == (n, 23)
    np.testing.assert_array_equal(o[:, 0], st[:, 1])
    np.testing.assert_allclose(o[:, 1], np.sin(st[:, 2]))
    np.testing.assert_array_equal(o[:, 3:9], st[:, 3:9])
    np.testing.assert_array_equal(o[:, 9:12], st[:, 9:12])
    np.testing.assert_array_equal(o[:, 12:18], st[:, 12:18])
    np.testing.assert_allclose(o[:, 18], np.sin(2 * np.pi * 0.8))  # right foot phase 0.3 + 0.5
    np.testing.assert_allclose(o[:, 20], np.sin(2 * np.pi * 0.3))
    np.testing.assert_allclose(o[:2, 22], 1e-2 * sols["v_mpc"][:2].astype(np.float64))
    assert o[2, 22] == 10.0


def test_policy_init_and_forward(oracle):
    """init_policy (policy.cpp:57-83): num_params, zero-initialised last policy layer (the
    residual action is exactly zero at the start), log_std = log 0.5; mlp_forward restated
    against a numpy evaluation of the same flattened (column-major) weights."""
    p = oracle.init_policy()
    sizes = [23, 64, 64, 64]
    n_pi = sum(a * b + b for a, b in zip(sizes, sizes[1:] + [6]))
    n_v = sum(a * b + b for a, b in zip(sizes, sizes[1:] + [1]))
    assert p.size == n_pi + n_v + 6
    np.testing.assert_array_equal(p[-6:], np.log(0.5))
    obs = np.random.default_rng(0).uniform(-1, 1, (5, 23))
    mean, value = oracle.policy_forward(p, obs)
    assert not mean.any() and value.any()
    q = oracle.init_policy(zero_final=False)
    mean, value = oracle.policy_forward(q, obs)

    def mlp(w, x, outs):
        off = 0
        for l, (i, o) in enumerate(zip(sizes, sizes[1:] + [outs])):
            W = w[off:off + i * o].reshape(i, o).T  # column-major (out x in)
            b = w[off + i * o:off + i * o + o]
            off += i * o + o
            x = W @ x + b
            if l < 3:
                x = np.where(x > 0, x, np.expm1(x))
        return x, off
    for k in range(5):
        m_np, off = mlp(q, obs[k], 6)
        v_np, _ = mlp(q[off:], obs[k], 1)
        np.testing.assert_allclose(mean[k], m_np, rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(value[k], v_np[0], rtol=1e-12, atol=1e-14)
