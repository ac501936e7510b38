"""ctypes / numpy mirrors of the C ABI in include/rmpc_b200.h (declarations only, no compute).

The layouts here must match the header byte for byte; tests/test_abi.py checks the sizes
against the library's own sizeof exports.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

NQ, NJ, NC, NF, NV = 9, 6, 4, 8, 26
MAX_HORIZON = 32
NUM_STAGES = 7

RMPC_OK = 0
RMPC_ERR_STRUCTURAL = 1
RMPC_ERR_INVALID_ARG = 2
RMPC_ERR_CUDA = 3
RMPC_ERR_NO_KERNEL = 4

STATUS_OK = 0
STATUS_NONFINITE_INPUT = 1
STATUS_DIVERGED = 2
STATUS_SINGULAR = 3

STAGE_NAMES = ("init_guess", "param", "kkt_build", "ruiz", "factorize", "admm_iters", "rnea")

_d = C.c_double
_i = C.c_int32


class Model(C.Structure):
    """rmpc_model == rmpc::ModelParams (robot.hpp:24-50)."""

    _fields_ = [
        ("torso_mass", _d), ("torso_len", _d), ("torso_inertia", _d),
        ("thigh_mass", _d), ("thigh_len", _d), ("thigh_inertia", _d),
        ("shank_mass", _d), ("shank_len", _d), ("shank_inertia", _d),
        ("foot_mass", _d), ("foot_half_len", _d), ("foot_inertia", _d),
        ("ankle_drop", _d),
        ("joint_lo", _d * NJ), ("joint_hi", _d * NJ),
        ("qd_limit", _d * NJ), ("tau_limit", _d * NJ),
        ("kp", _d * NJ), ("kd", _d * NJ),
        ("mu", _d), ("gravity", _d),
        ("nominal_stagger", _d), ("nominal_drop", _d),
    ]

    def total_mass(self) -> float:
        return self.torso_mass + 2.0 * (self.thigh_mass + self.shank_mass + self.foot_mass)

    def nominal_height(self) -> float:
        return self.ankle_drop + self.nominal_drop + 0.5 * self.torso_len


class Settings(C.Structure):
    """rmpc_settings == rmpc::MpcSettings (mpc.hpp:16-57) + AdmmSettings::ruiz_iters."""

    _fields_ = [
        ("horizon", _i),
        ("dt_schedule", _d * MAX_HORIZON),
        ("w_q", _d * NQ), ("w_qd", _d * NQ), ("w_f", _d * NF),
        ("gait_period", _d), ("phase_switch", _d), ("phase_offsets", _d * NC),
        ("z_swing", _d), ("v_to", _d), ("v_td", _d),
        ("n_qp", _i),
        ("mu", _d), ("sigma", _d), ("rho", _d), ("over_relax", _d),
        ("warm_start", _i),
        ("ruiz_iters", _i),
    ]


class Timing(C.Structure):
    """rmpc_timing == rmpc::TimingReport (batch.hpp:12-18), device-timed."""

    _fields_ = [
        ("batch_size", _i), ("devices", _i),
        ("total_ms", _d), ("h2d_ms", _d), ("kernel_ms", _d), ("d2h_ms", _d),
        ("stage_ms", _d * NUM_STAGES), ("stage_mean_ms", _d * NUM_STAGES), ("stage_std_ms", _d * NUM_STAGES),
    ]


# Batches are numpy arrays whose rows are the C structs:
#   states (n, 18) f64 = rmpc_state {q[9], qd[9]}
#   cmds   (n, 3)  f64 = rmpc_command {height, vx, wpitch}
#   gaits  (n, 7)  f64 = rmpc_gait {phase, period, phase_switch, offsets[4]}
SOLUTION_DTYPE = np.dtype([
    ("tau_ff", np.float32, (NJ,)),
    ("q_set", np.float32, (NJ,)),
    ("qd_set", np.float32, (NJ,)),
    ("f0", np.float32, (NF,)),
    ("base_residual", np.float32, (3,)),
    ("v_mpc", np.float32),
    ("prim_res", np.float32),
    ("dual_res", np.float32),
    ("delta_inf_norm", np.float32),
    ("status", np.int32),
    ("fail_iter", np.int32),
])
assert SOLUTION_DTYPE.itemsize == 140

STATE_W, CMD_W, GAIT_W = 2 * NQ, 3, 3 + NC


def default_model() -> Model:
    m = Model()
    m.torso_mass, m.torso_len = 10.0, 0.4
    m.torso_inertia = 10.0 * 0.4 * 0.4 / 12.0
    m.thigh_mass, m.thigh_len = 2.5, 0.4
    m.thigh_inertia = 2.5 * 0.4 * 0.4 / 12.0
    m.shank_mass, m.shank_len = 1.5, 0.4
    m.shank_inertia = 1.5 * 0.4 * 0.4 / 12.0
    m.foot_mass, m.foot_half_len = 0.5, 0.09
    m.foot_inertia = 0.5 * 0.18 * 0.18 / 12.0
    m.ankle_drop = 0.05
    m.joint_lo[:] = (-1.5, 0.05, -1.2, -1.5, 0.05, -1.2)
    m.joint_hi[:] = (1.5, 2.4, 1.2, 1.5, 2.4, 1.2)
    m.qd_limit[:] = (20.0,) * NJ
    m.tau_limit[:] = (60.0, 60.0, 30.0, 60.0, 60.0, 30.0)
    m.kp[:] = (30.0,) * NJ
    m.kd[:] = (1.0,) * NJ
    m.mu, m.gravity = 0.8, 9.81
    m.nominal_stagger, m.nominal_drop = 0.15, 0.75
    return m


def default_settings(horizon: int = 12, dt: float = 0.05) -> Settings:
    s = Settings()
    s.horizon = horizon
    for i in range(MAX_HORIZON):
        s.dt_schedule[i] = dt if i < horizon else 0.0
    s.w_q[:] = (0.0, 500.0, 300.0, 5.0, 5.0, 5.0, 5.0, 5.0, 5.0)
    s.w_qd[:] = (100.0, 100.0, 50.0, 0.1, 0.1, 0.1, 0.1, 0.1, 0.1)
    s.w_f[:] = (1e-3,) * NF
    s.gait_period, s.phase_switch = 0.8, 0.5
    s.phase_offsets[:] = (0.5, 0.5, 0.0, 0.0)
    s.z_swing, s.v_to, s.v_td = 0.075, 0.2, -0.3
    s.n_qp = 25
    s.mu, s.sigma, s.rho, s.over_relax = 0.6, 1e-6, 0.1, 1.6
    s.warm_start = 0
    s.ruiz_iters = 10
    return s


def gait_row(settings: Settings, phase: float = 0.0) -> np.ndarray:
    """GaitState from MpcSettings::make_gait (mpc.hpp:44-50) at `phase`."""
    return np.array([phase, settings.gait_period, settings.phase_switch,
                     *settings.phase_offsets], dtype=np.float64)


def standing_gait_row(period: float = 0.8) -> np.ndarray:
    """GaitState::standing (gait.cpp:24-29): switch = 1, every contact in stance."""
    return np.array([0.0, period, 1.0, 0.5, 0.5, 0.0, 0.0], dtype=np.float64)


def ptr(a: np.ndarray | None, ctype=C.c_double):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.POINTER(ctype))
