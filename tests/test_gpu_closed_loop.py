"""§8(f) row 1 closed loop (SPEC.md acceptance #4: standing, zero command, 5 s survival) on the
device -- the batched solve, mpc_torque and physics_step kernels, tick after tick -- against
the REFERENCE's own closed loop (oracle/_ref: rti_step -> mpc_torque -> Env::step, the
run_episode loop of analysis.cpp:75-149, randomisation pinned, termination by the reference's
check_termination on the device states).

What the reference itself does (tests/test_ref_pin.py::test_reference_closed_loop):
  * at its default physics (4 substeps of 2.5 ms, k_n = 5e4, c_n = 500) the explicit penalty
    contact is unstable for the 0.5 kg feet (c_n dt / m_eff >> 2): ankle rates of hundreds of
    rad/s after one tick, self-collision within 0.02 s -- the device loop does the same;
  * with 16 substeps the contact is stable; the default controller (n_qp = 25) then tips over
    after ~3 s, n_qp = 100 with warm start stands for the 5 s -- the device loop reproduces the
    survival and follows the reference's trajectory.
"""
import numpy as np
import pytest

import paper_2510_12717_b200 as R
from paper_2510_12717_b200.abi import SOLUTION_DTYPE

pytestmark = pytest.mark.gpu


def _ref():
    from oracle import ref as F
    try:
        F.lib()
    except Exception as e:  # noqa: BLE001
        pytest.skip(f"oracle/_ref unavailable ({e})")
    return F


def device_closed_loop(F, m, s, cfg, phase_switch, ticks):
    """1 agent from the nominal pose at zero command: (ticks survived, reason, trace)."""
    import torch
    from paper_2510_12717_b200.env import Env
    dev = torch.device("cuda:0")
    nom = F.nominal_pose(m)
    st = np.zeros((1, 18))
    st[0, :9] = nom
    cm = np.array([[m.nominal_height(), 0.0, 0.0]])
    ga = np.array([[0.0, s.gait_period, phase_switch, *s.phase_offsets[:4]]])
    br = R.BatchRunner(1, m, s)
    env = Env(m, cfg)
    d_st, d_cm, d_ga = (torch.from_numpy(x).to(dev) for x in (st, cm, ga))
    out = torch.zeros(SOLUTION_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    z = torch.zeros(s.horizon * 26, dtype=torch.float32, device=dev)
    p_out, p_z = torch.zeros_like(out), torch.zeros_like(z)
    trace = np.full((ticks, 18), np.nan)
    for t in range(ticks):
        warm = s.warm_start and t > 0
        br.solve_device(d_st, d_cm, d_ga, out, z_out=z, prev=p_out if warm else None, prev_z=p_z if warm else None)
        env.control_step(out, d_st, d_ga, strategy="joint-torque", lam=0.0)  # = mpc_torque
        p_out.copy_(out)
        p_z.copy_(z)
        sol = out.cpu().numpy().view(SOLUTION_DTYPE)
        x = d_st.cpu().numpy()[0]
        if sol["status"][0] != 0:
            return t, "controller_failed", trace
        why = F.check_termination(m, cfg, x)
        if why != "survived":
            return t, why, trace
        trace[t] = x
    br.close()
    env.close()
    return ticks, "survived", trace


@pytest.mark.parametrize("substeps,n_qp,warm,ticks", [(4, 25, 0, 20), (16, 100, 1, 500), (16, 25, 0, 500)])
def test_standing_closed_loop_matches_reference(substeps, n_qp, warm, ticks):
    F = _ref()
    from oracle import oracle as O
    m = R.default_model()
    s = R.default_settings(10)
    s.n_qp, s.warm_start = n_qp, warm
    cfg = O.env_config_default()
    cfg.substeps = substeps
    ra, rwhy, rtr = F.closed_loop(m, s, cfg, phase_switch=1.0, ticks=ticks)
    da, dwhy, dtr = device_closed_loop(F, m, s, cfg, 1.0, ticks)
    k = min(ra, da, 100)
    err = np.abs(dtr[:k] - rtr[:k]).max(axis=1) if k else np.zeros(1)
    print(f"substeps={substeps} n_qp={n_qp} warm={warm}: reference {ra} ticks ({rwhy}), device {da} ticks "
          f"({dwhy}); max |state diff| over the first {k} ticks {err.max():.2e}, at tick {k - 1}: {err[-1]:.2e}")
    if ra == ticks:  # the reference stands for the whole run: so must the device
        assert da == ticks
    else:  # the same failure, within 5% of the reference's survival time
        assert dwhy == rwhy or (dwhy in ("self_collision", "orientation") and rwhy in ("self_collision", "orientation"))
        assert abs(da - ra) <= max(2, 0.05 * ra)
    if substeps >= 16:  # a stable contact: the device follows the reference's trajectory
        assert err[: min(k, 50)].max() <= 1e-3
