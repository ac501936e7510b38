"""Parity of the device closed-loop step (include/rmpc_b200_env.h, csrc/rmpc_env.cu) with the
FP64 CPU oracle (oracle/rmpc_oracle_env.hpp) on identical inputs: physics_step on a heightfield
with randomized bodies, the fused mpc_torque + blend + physics control step fed with the
device solver's own solutions (failed ones included), observe, and a closed loop of solve ->
control step chained on the device.  Both sides are FP64; the device differs only by FMA
contraction and libm ulps, so one step agrees to 1e-9 (relative, 1e-9 floor).  Needs a B200."""
import numpy as np
import pytest
import torch

import paper_2510_12717_b200 as R
from paper_2510_12717_b200.abi import SOLUTION_DTYPE, default_model, default_settings
from paper_2510_12717_b200.env import Env, default_env_config

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def rel_err(a, b, floor=1e-9):
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), floor))) if a.size else 0.0


def near_ground_batch(oracle, n, seed):
    """Nominal stance +- noise, feet around the ground, random velocities / phases / bodies."""
    rng = np.random.default_rng(seed)
    m = default_model()
    q = np.tile(oracle.nominal_pose(m), (n, 1)) + rng.uniform(-0.05, 0.05, (n, 9))
    q[:, 0] = rng.uniform(-30, 30, n)           # across the heightfield
    q[:, 1] += rng.uniform(-0.03, 0.02, n)      # some feet in the ground, some above
    qd = rng.uniform(-0.5, 0.5, (n, 9))
    st = np.concatenate([q, qd], 1)
    ga = np.tile([0.0, 0.8, 0.5, 0.5, 0.5, 0.0, 0.0], (n, 1))
    ga[:, 0] = rng.uniform(0, 1, n)
    bodies = np.stack([rng.uniform(0.5, 1.0, n), rng.uniform(0.9, 1.1, n)], 1)
    tau = rng.uniform(-30, 30, (n, 6))
    return m, st, ga, bodies, tau


def dev(a, dtype=torch.float64):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV, dtype)


@pytest.mark.parametrize("terrain,steps", [(0, 1), (1, 1), (1, 20)])
def test_physics_step_parity(oracle, terrain, steps):
    n = 2048
    m, st, ga, bodies, tau = near_ground_batch(oracle, n, seed=terrain + 10 * steps)
    if steps > 1:
        # A chain in flight (base 0.5 m up, 0.2 s): the default penalty contact is explicit and
        # stiff for the light feet (damping c_n dt / m_eff >> 2 on the toe/heel rocking mode),
        # so states in contact go chaotic within a few steps on the reference model as restated
        # (oracle and device alike) and only single steps are comparable there.
        rng = np.random.default_rng(77)
        st[:, 1] += 0.5
        st[:, 9:] *= 0.5
        tau = rng.uniform(-5, 5, (n, 6))
    cfg = default_env_config(terrain_kind=terrain)
    env = Env(m, cfg)
    for x in (-30.0, -0.7, 0.0, 12.3):
        assert env.height_at(x) == oracle.terrain_height_at(cfg, x)
    ds, dg, db, dt = dev(st), dev(ga), dev(bodies), dev(tau)
    dstat = torch.zeros(n, dtype=torch.int32, device=DEV)
    rs, rg = st, ga
    for _ in range(steps):
        env.physics_step(ds, dg, dt, bodies=db, sim_status=dstat)
        rs, rg, rstat = oracle.physics_step_batch(m, cfg, rs, rg, tau, bodies)
    torch.cuda.synchronize()
    gs, gg = ds.cpu().numpy(), dg.cpu().numpy()
    assert (dstat.cpu().numpy() == rstat).all() and (rstat == 0).all()
    tol = 1e-9 if steps == 1 else 1e-6
    assert rel_err(gs, rs) <= tol, rel_err(gs, rs)
    np.testing.assert_allclose(gg, rg, rtol=0, atol=1e-15)
    assert (np.abs(rs[:, 9:] - st[:, 9:]).max()) > 0.1  # the step did something
    if steps > 1:
        assert np.abs(rs).max() < 1e3  # the flight chain stays physical


def test_control_step_with_device_solutions(oracle):
    """solve -> tau = blend(mpc_torque) (zero when failed) -> physics, all three strategies."""
    n, T = 1024, 10
    m, s = default_model(), default_settings(T)
    st, cm, ga = R.synthetic_batch(n, "mixed", seed=5, model=m, settings=s)
    st[3, 0] = np.nan  # one failed agent (RMPC_STATUS_NONFINITE_INPUT)
    sol, _ = R.BatchRunner(n, m, s).solve(st, cm, ga)
    assert sol["status"][3] != 0 and (np.delete(sol["status"], 3) == 0).all()
    st[3, 0] = 0.0
    cfg = default_env_config(terrain_kind=1)
    env = Env(m, cfg)
    rng = np.random.default_rng(6)
    act = rng.uniform(-0.2, 0.2, (n, 6))
    bodies = np.stack([rng.uniform(0.5, 1.0, n), rng.uniform(0.9, 1.1, n)], 1)
    for strategy, lam in ((0, 0.3), (1, 0.5), (2, 2.0)):
        ds, dg = dev(st), dev(ga)
        dsol = torch.from_numpy(sol.view(np.uint8).copy()).to(DEV)
        dtau = torch.zeros((n, 6), dtype=torch.float64, device=DEV)
        dstat = torch.zeros(n, dtype=torch.int32, device=DEV)
        env.control_step(dsol, ds, dg, action=dev(act), strategy=strategy, lam=lam, bodies=dev(bodies),
                         tau_out=dtau, sim_status=dstat)
        torch.cuda.synchronize()
        rs, rg, rtau, rstat = oracle.control_step_batch(m, cfg, sol, st, ga, act, strategy, lam, bodies)
        gtau = dtau.cpu().numpy()
        assert not gtau[3].any() and not rtau[3].any()
        np.testing.assert_allclose(gtau, rtau, rtol=1e-12, atol=1e-12)
        assert rel_err(ds.cpu().numpy(), rs) <= 1e-9
        assert (dstat.cpu().numpy() == rstat).all()


def test_observe_parity(oracle):
    n = 512
    m, st, ga, _, _ = near_ground_batch(oracle, n, seed=7)
    sol = np.zeros(n, SOLUTION_DTYPE)
    sol["v_mpc"] = np.random.default_rng(8).uniform(-3, 3, n)
    sol["status"][::7] = 2
    obs = torch.zeros((n, 23), dtype=torch.float64, device=DEV)
    Env(m).observe(dev(st), dev(ga), torch.from_numpy(sol.view(np.uint8).copy()).to(DEV), obs)
    torch.cuda.synchronize()
    ref = oracle.observe_batch(st, ga, sol)
    np.testing.assert_allclose(obs.cpu().numpy(), ref, rtol=1e-14, atol=1e-15)


def test_closed_loop_on_device(oracle):
    """20 ticks of solve -> control step chained on the device (the C5 loop, no host round
    trip).  The restated reference simulator is not stable under this controller (its explicit
    penalty contact rocks the light feet), so this checks the loop's contracts, not walking:
    sim status 1 exactly for non-finite states, and the solver's per-agent failure status for
    them on the next tick (RMPC_STATUS_NONFINITE_INPUT) instead of an aborted batch."""
    n, T = 512, 10
    m, s = default_model(), default_settings(T)
    st, cm, ga = R.synthetic_batch(n, "random", seed=9, model=m, settings=s)
    br = R.BatchRunner(n, m, s)
    env = Env(m, default_env_config())
    ds, dc, dg = dev(st), dev(cm), dev(ga)
    dsol = torch.zeros(n * SOLUTION_DTYPE.itemsize, dtype=torch.uint8, device=DEV)
    dstat = torch.zeros(n, dtype=torch.int32, device=DEV)
    for _ in range(20):
        br.solve_device(ds, dc, dg, dsol)
        env.control_step(dsol, ds, dg, sim_status=dstat)
    br.solve_device(ds, dc, dg, dsol)
    torch.cuda.synchronize()
    sol = dsol.cpu().numpy().view(SOLUTION_DTYPE)
    fin = np.isfinite(ds.cpu().numpy()).all(1)
    sim = dstat.cpu().numpy()
    assert set(np.unique(sim)) <= {0, 1}
    assert ((sim == 1) == ~fin).all()
    assert (sol["status"][~fin] == R.STATUS_NONFINITE_INPUT).all()
    assert fin.mean() > 0.5


@pytest.mark.parametrize("obs_dim,act,hidden,n", [(23, 6, 64, 4096), (23, 6, 24, 777), (64, 32, 64, 1000)])
def test_policy_forward_parity(oracle, obs_dim, act, hidden, n):
    """Default shapes run the FP64 tensor-core kernel (rmpc_ppo.cu forward_kernel_mma); obs 64 /
    act 32 exceeds its layout and runs the CUDA-core warp-per-agent kernel."""
    from paper_2510_12717_b200.env import Policy
    params = oracle.init_policy(obs_dim, act, hidden, seed=3, zero_final=False)
    obs = np.random.default_rng(10).uniform(-2, 2, (n, obs_dim))
    pol = Policy(params, obs_dim, act, hidden)
    mean = torch.zeros((n, act), dtype=torch.float64, device=DEV)
    value = torch.zeros(n, dtype=torch.float64, device=DEV)
    pol.forward(dev(obs), mean, value)
    torch.cuda.synchronize()
    rm, rv = oracle.policy_forward(params, obs, act, hidden)
    np.testing.assert_allclose(mean.cpu().numpy(), rm, rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(value.cpu().numpy(), rv, rtol=1e-12, atol=1e-13)
    np.testing.assert_array_equal(pol.log_std, np.log(0.5))
    only_value = torch.zeros(n, dtype=torch.float64, device=DEV)
    pol.forward(dev(obs), None, only_value)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(only_value.cpu().numpy(), value.cpu().numpy())
