"""TEST INFRASTRUCTURE ONLY — ctypes wrapper of the CPU oracle (oracle/_build/librmpc_oracle.so).

The oracle is a plain-C++ restatement of the reference's hot path (see rmpc_oracle.hpp).
Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and --impl reference arm)
may load it, and only as the checker / CPU baseline.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2510_12717_b200.abi import (NV, Model, Settings, default_model,  # noqa: F401
                                       default_settings, ptr)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_build", "librmpc_oracle.so")

ORACLE_SOLUTION_DTYPE = np.dtype([
    ("tau_ff", np.float64, (6,)), ("q_set", np.float64, (6,)), ("qd_set", np.float64, (6,)),
    ("f0", np.float64, (8,)), ("base_residual", np.float64, (3,)),
    ("v_mpc", np.float64), ("prim_res", np.float64), ("dual_res", np.float64),
    ("delta_inf_norm", np.float64), ("v_quad", np.float64), ("v_lin", np.float64),
    ("status", np.int32), ("fail_iter", np.int32), ("n_vars", np.int32), ("n_cons", np.int32),
    ("ldl_nnz", np.int32), ("pad", np.int32),
])

_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.oracle_solve_batch.restype = C.c_int32
        L.oracle_flops.restype = C.c_int32
        L.oracle_build_qp.restype = C.c_int32
        L.oracle_bezier.restype = C.c_double
        L.oracle_bezier.argtypes = [C.c_double] * 4 + [C.POINTER(C.c_double)]
        L.oracle_admm_dense.restype = C.c_int32
        L.oracle_admm_dense.argtypes = [C.c_int32, C.c_int32] + [C.POINTER(C.c_double)] * 5 + [
            C.c_double, C.c_double, C.c_double, C.c_int32, C.c_int32, C.c_double] + [
            C.POINTER(C.c_double)] * 6 + [C.POINTER(C.c_int32)]
        L.oracle_sizeof_solution.restype = C.c_int32
        assert L.oracle_sizeof_solution() == ORACLE_SOLUTION_DTYPE.itemsize
        _lib = L
    return _lib


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None:
        a = a.reshape(shape)
    return a


def solve_batch(model: Model, settings: Settings, states, cmds, gaits, *, prev_z=None,
                prev_ok=None, workers: int = 1, precision: int = 64, want_z: bool = True,
                timed: bool = False):
    """BatchRunner::solve on the CPU oracle.  Returns (solutions, z_star[n,T,26] or None,
    stage_ms[7] or None, wall_ms)."""
    states = _f64(states)
    n = states.shape[0]
    cmds, gaits = _f64(cmds, (n, 3)), _f64(gaits, (n, 7))
    T = settings.horizon
    out = np.zeros(n, dtype=ORACLE_SOLUTION_DTYPE)
    z = np.zeros((n, T, NV)) if want_z else None
    stage = np.zeros(7) if timed else None
    wall = C.c_double(0.0)
    pz = _f64(prev_z) if prev_z is not None else None
    pok = np.ascontiguousarray(prev_ok, dtype=np.int32) if prev_ok is not None else None
    rc = lib().oracle_solve_batch(C.byref(model), C.byref(settings), C.c_int32(n), ptr(states),
                                  ptr(cmds), ptr(gaits), ptr(pz), ptr(pok, C.c_int32),
                                  C.c_int32(workers), C.c_int32(precision),
                                  out.ctypes.data_as(C.c_void_p), ptr(z), ptr(stage),
                                  C.byref(wall))
    if rc != 0:
        raise ValueError(f"oracle_solve_batch: structural error (code {rc})")
    return out, z, stage, wall.value


def flops(model: Model, settings: Settings, state, cmd, gait):
    """Exact per-stage FLOP counts of one rti_step (reference algorithm, FP64)."""
    by = np.zeros(7)
    ops = np.zeros(6)
    st = _f64(state, (18,))
    lib().oracle_flops(C.byref(model), C.byref(settings), ptr(st), ptr(_f64(cmd, (3,))),
                       ptr(_f64(gait, (7,))), ptr(by), ptr(ops))
    return by, dict(zip(("add", "mul", "div", "sqrt", "trig", "cmp"), ops))


def rng_uniform(seed: int, stream: int, n: int) -> np.ndarray:
    """n uniform() draws of rmpc::Rng(seed, stream) (rng.hpp), C++ restatement."""
    out = np.zeros(n)
    lib().oracle_rng_uniform(C.c_uint64(seed), C.c_uint64(stream), C.c_int32(n), ptr(out))
    return out


def nominal_pose(model: Model) -> np.ndarray:
    q = np.zeros(9)
    lib().oracle_nominal_pose(C.byref(model), ptr(q))
    return q


def kinematics(model: Model, q, qd):
    q, qd = _f64(q, (9,)), _f64(qd, (9,))
    out = dict(com_pos=np.zeros((7, 2)), com_vel=np.zeros((7, 2)), com_jac=np.zeros((7, 2, 9)),
               com_jdq=np.zeros((7, 2)), c_pos=np.zeros((4, 2)), c_vel=np.zeros((4, 2)),
               c_jac=np.zeros((4, 2, 9)))
    lib().oracle_kinematics(C.byref(model), ptr(q), ptr(qd), *(ptr(out[k]) for k in (
        "com_pos", "com_vel", "com_jac", "com_jdq", "c_pos", "c_vel", "c_jac")))
    return out


def mass_matrix(model: Model, q) -> np.ndarray:
    M = np.zeros((9, 9))
    lib().oracle_mass_matrix(C.byref(model), ptr(_f64(q, (9,))), ptr(M))
    return M


def bias_forces(model: Model, q, qd) -> np.ndarray:
    h = np.zeros(9)
    lib().oracle_bias_forces(C.byref(model), ptr(_f64(q, (9,))), ptr(_f64(qd, (9,))), ptr(h))
    return h


def inverse_dynamics(model: Model, q, qd, qdd, F):
    tau, base = np.zeros(6), np.zeros(3)
    lib().oracle_inverse_dynamics(C.byref(model), ptr(_f64(q, (9,))), ptr(_f64(qd, (9,))),
                                  ptr(_f64(qdd, (9,))), ptr(_f64(F, (8,))), ptr(tau), ptr(base))
    return tau, base


def pd_torque(model: Model, q_des, qd_des, q, qd, tau_ff) -> np.ndarray:
    out = np.zeros(6)
    lib().oracle_pd_torque(C.byref(model), ptr(_f64(q_des, (6,))), ptr(_f64(qd_des, (6,))),
                           ptr(_f64(q, (9,))), ptr(_f64(qd, (9,))), ptr(_f64(tau_ff, (6,))),
                           ptr(out))
    return out


def bezier(t: float, z_swing: float, v_to: float, v_td: float):
    v = C.c_double(0.0)
    h = lib().oracle_bezier(t, z_swing, v_to, v_td, C.byref(v))
    return h, v.value


def horizon_schedule(gait, dt):
    dt = _f64(dt)
    T = dt.shape[0]
    st = np.zeros((T, 4), dtype=np.int32)
    sw = np.zeros((T, 4))
    lib().oracle_horizon_schedule(ptr(_f64(gait, (7,))), ptr(dt), C.c_int32(T),
                                  ptr(st, C.c_int32), ptr(sw))
    return st.astype(bool), sw


def desired_trajectory(model: Model, settings: Settings, cmd, gait):
    T = settings.horizon
    qd_, qdd_, F, sh = np.zeros((T, 9)), np.zeros((T, 9)), np.zeros((T, 8)), np.zeros((T, 4))
    lib().oracle_desired_trajectory(C.byref(model), C.byref(settings), ptr(_f64(cmd, (3,))),
                                    ptr(_f64(gait, (7,))), ptr(qd_), ptr(qdd_), ptr(F), ptr(sh))
    return dict(q_des=qd_, qd_des=qdd_, F_des=F, swing_height=sh)


def build_qp(model: Model, settings: Settings, state, cmd, gait, guess_z=None):
    """Dense view of build_qp's problem: dict(A, P_diag, q, lo, hi, nnz) or None on failure."""
    n, m, nnz = C.c_int32(), C.c_int32(), C.c_int32()
    args = (C.byref(model), C.byref(settings), ptr(_f64(state, (18,))), ptr(_f64(cmd, (3,))),
            ptr(_f64(gait, (7,))), ptr(_f64(guess_z)) if guess_z is not None else None)
    rc = lib().oracle_build_qp(*args, C.byref(n), C.byref(m), C.byref(nnz), None, None, None,
                               None, None)
    if rc != 0:
        return None
    A = np.zeros((m.value, n.value))
    P, q = np.zeros(n.value), np.zeros(n.value)
    lo, hi = np.zeros(m.value), np.zeros(m.value)
    lib().oracle_build_qp(*args, C.byref(n), C.byref(m), C.byref(nnz), ptr(A), ptr(P), ptr(q),
                          ptr(lo), ptr(hi))
    return dict(A=A, P_diag=P, q=q, lo=lo, hi=hi, nnz=nnz.value)


def csc_from_triplets(rows, cols, vals, nrows, ncols):
    rows = np.ascontiguousarray(rows, dtype=np.int32)
    cols = np.ascontiguousarray(cols, dtype=np.int32)
    vals = _f64(vals)
    nt = rows.shape[0]
    colptr = np.zeros(ncols + 1, dtype=np.int32)
    rowidx = np.zeros(max(nt, 1), dtype=np.int32)
    v = np.zeros(max(nt, 1))
    nnz = C.c_int32()
    rc = lib().oracle_csc_from_triplets(C.c_int32(nt), ptr(rows, C.c_int32), ptr(cols, C.c_int32),
                                        ptr(vals), C.c_int32(nrows), C.c_int32(ncols),
                                        ptr(colptr, C.c_int32), ptr(rowidx, C.c_int32), ptr(v),
                                        C.byref(nnz))
    if rc != 0:
        raise ValueError("csc_from_triplets: entry outside matrix")
    k = nnz.value
    return colptr, rowidx[:k], v[:k]


def ruiz(K, passes=10):
    K = _f64(K).copy()
    n = K.shape[0]
    s = np.zeros(n)
    rc = lib().oracle_ruiz_dense(C.c_int32(n), ptr(K), C.c_int32(passes), ptr(s))
    if rc != 0:
        raise ValueError("ruiz_equilibrate: structural error")
    return np.triu(K) + np.triu(K, 1).T, s


def ldl(K, use_ordering=True):
    K = _f64(K)
    n = K.shape[0]
    perm = np.zeros(n, dtype=np.int32)
    D, L = np.zeros(n), np.zeros((n, n))
    lnnz = C.c_int32()
    err = C.create_string_buffer(256)
    rc = lib().oracle_ldl_dense(C.c_int32(n), ptr(K), C.c_int32(int(use_ordering)),
                                ptr(perm, C.c_int32), ptr(D), ptr(L), C.byref(lnnz), err, 256)
    if rc != 0:
        raise ArithmeticError(err.value.decode()) if rc == 3 else ValueError(err.value.decode())
    return perm, D, L, lnnz.value


def ldl_solve(K, b, use_ordering=True):
    K, b = _f64(K), _f64(b)
    x = np.zeros_like(b)
    rc = lib().oracle_ldl_solve_dense(C.c_int32(K.shape[0]), ptr(K), C.c_int32(int(use_ordering)),
                                      ptr(b), ptr(x))
    if rc != 0:
        raise ValueError("ldl solve failed")
    return x


class DivergenceError(ArithmeticError):
    def __init__(self, iteration):
        super().__init__(f"admm: non-finite iterate at iteration {iteration}")
        self.iteration = iteration


def admm(P, q, A, lo, hi, *, sigma=1e-6, rho=0.1, alpha=1.6, iters=25, ruiz_iters=10,
         eps_exit=0.0, x0=None, y0=None):
    P, q, A, lo, hi = _f64(P), _f64(q), _f64(A), _f64(lo), _f64(hi)
    n, m = P.shape[0], A.shape[0]
    A = A.reshape(m, n)
    x, y, z, info = np.zeros(n), np.zeros(m), np.zeros(m), np.zeros(4)
    fi = C.c_int32()
    rc = lib().oracle_admm_dense(n, m, ptr(P), ptr(q), ptr(A), ptr(lo), ptr(hi), sigma, rho, alpha,
                                 iters, ruiz_iters, eps_exit, ptr(_f64(x0)) if x0 is not None else None,
                                 ptr(_f64(y0)) if y0 is not None else None, ptr(x), ptr(y), ptr(z),
                                 ptr(info), C.byref(fi))
    if rc == 2:
        raise DivergenceError(fi.value)
    if rc != 0:
        raise ValueError("admm: structural error")
    return dict(x=x, y=y, z=z, prim=info[0], dual=info[1], obj=info[2], iters=int(info[3]))


# ---------------------------------------------------------------- closed-loop step (env.cpp)
def _env_lib():
    L = lib()
    if not getattr(L, "_env_bound", False):
        L.oracle_terrain_height_at.restype = C.c_double
        L.oracle_terrain_height_at.argtypes = [C.c_void_p, C.c_double]
        L.oracle_control_step_batch.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                                C.c_int32, C.c_double] + [C.c_void_p] * 5
        L.oracle_observe_batch.argtypes = [C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double,
                                           C.c_double, C.c_void_p]
        L._env_bound = True
    return L


def env_config_default():
    from paper_2510_12717_b200.env import EnvConfig
    c = EnvConfig()
    _env_lib().oracle_env_config_default(C.byref(c))
    return c


def terrain_height_at(cfg, x: float) -> float:
    return _env_lib().oracle_terrain_height_at(C.byref(cfg), float(x))


def physics_step_batch(model: Model, cfg, states, gaits, tau, bodies=None):
    """physics_step + advance_phase for every agent: returns (states, gaits, status)."""
    st, ga = _f64(states).copy().reshape(-1, 18), _f64(gaits).copy().reshape(-1, 7)
    n = st.shape[0]
    tau = _f64(tau, (n, 6))
    bo = None if bodies is None else _f64(bodies, (n, 2))
    status = np.zeros(n, np.int32)
    _env_lib().oracle_physics_step_batch(C.byref(model), C.byref(cfg), C.c_int32(n), ptr(st), ptr(ga),
                                         ptr(bo), ptr(tau), status.ctypes.data_as(C.POINTER(C.c_int32)))
    return st, ga, status


def control_step_batch(model: Model, cfg, solutions, states, gaits, action=None, strategy=0, lam=0.0,
                       bodies=None):
    """Trainer::train's control (zero torque on failure, else blend(mpc_torque)) + physics:
    returns (states, gaits, tau, status).  `solutions` is the device's SOLUTION_DTYPE array."""
    st, ga = _f64(states).copy().reshape(-1, 18), _f64(gaits).copy().reshape(-1, 7)
    n = st.shape[0]
    sols = np.ascontiguousarray(solutions)
    act = None if action is None else _f64(action, (n, 6))
    bo = None if bodies is None else _f64(bodies, (n, 2))
    tau = np.zeros((n, 6))
    status = np.zeros(n, np.int32)
    _env_lib().oracle_control_step_batch(C.byref(model), C.byref(cfg), n, sols.ctypes.data,
                                         None if act is None else act.ctypes.data, int(strategy), float(lam),
                                         st.ctypes.data, ga.ctypes.data,
                                         None if bo is None else bo.ctypes.data, tau.ctypes.data,
                                         status.ctypes.data)
    return st, ga, tau, status


def observe_batch(states, gaits, solutions, scale=1e-2, sentinel=10.0):
    st, ga = _f64(states).reshape(-1, 18), _f64(gaits).reshape(-1, 7)
    n = st.shape[0]
    sols = np.ascontiguousarray(solutions)
    obs = np.zeros((n, 23))
    _env_lib().oracle_observe_batch(n, st.ctypes.data, ga.ctypes.data, sols.ctypes.data, scale, sentinel,
                                    obs.ctypes.data)
    return obs


def init_policy(obs=23, act=6, hidden=64, seed=0, zero_final=True) -> np.ndarray:
    """init_policy (policy.cpp:57-83) in flatten_into order: pi, value, log_std."""
    L = lib()
    L.oracle_init_policy.restype = C.c_int32
    n = L.oracle_init_policy(obs, act, hidden, C.c_uint64(seed), int(zero_final), None, 0)
    out = np.zeros(n)
    L.oracle_init_policy(obs, act, hidden, C.c_uint64(seed), int(zero_final), ptr(out), n)
    return out


def policy_forward(params, obs, act=6, hidden=64):
    o = _f64(obs)
    o = o.reshape(-1, o.shape[-1])
    n, od = o.shape
    mean, value = np.zeros((n, act)), np.zeros(n)
    lib().oracle_policy_forward_batch(ptr(_f64(params)), od, act, hidden, n, ptr(o), ptr(mean), ptr(value))
    return mean, value


def active_set_batch(model: Model, settings: Settings, states, cmds, gaits, workers=0):
    """Final-iterate active set on the device's (node + 1, slot) grid: codes (n, T+1, 40) int8
    (0 inactive, 1 at lo, 2 at hi, 3 equality / no row) and the scaled-space margin."""
    st, cm, ga = _f64(states).reshape(-1, 18), _f64(cmds).reshape(-1, 3), _f64(gaits).reshape(-1, 7)
    n, T = st.shape[0], settings.horizon
    act = np.zeros((n, T + 1, 40), np.int8)
    margin = np.zeros((n, T + 1, 40))
    rc = lib().oracle_active_set_batch(C.byref(model), C.byref(settings), C.c_int32(n), ptr(st), ptr(cm),
                                       ptr(ga), C.c_int32(workers), act.ctypes.data_as(C.c_void_p), ptr(margin))
    if rc != 0:
        raise ValueError(f"oracle_active_set_batch: {rc}")
    return act, margin


# ---------------------------------------------------------------- PPO batch (ppo.cpp:28-276)
class PpoConfig(C.Structure):
    _fields_ = [("gamma", C.c_double), ("lam_gae", C.c_double), ("clip_eps", C.c_double), ("epochs", C.c_int32),
                ("minibatches", C.c_int32), ("lr", C.c_double), ("entropy_coef", C.c_double),
                ("value_coef", C.c_double), ("max_grad_norm", C.c_double)]


def ppo_config(**overrides) -> PpoConfig:
    c = PpoConfig()
    lib().oracle_ppo_config_default(C.byref(c))
    for k, v in overrides.items():
        setattr(c, k, v)
    return c


def ppo_loss(params, obs, actions, old_logp, adv, ret, cfg=None, act=6, hidden=64, grads=True):
    """ppo_loss: ((total, surrogate, value_loss, entropy), flatten_grads vector or None)."""
    p = _f64(params)
    o, a = _f64(obs), _f64(actions)
    n, od = o.shape
    cfg = cfg or ppo_config()
    info = (C.c_double * 4)()
    g = np.zeros(p.size) if grads else None
    lib().oracle_ppo_loss(ptr(p), od, act, hidden, n, ptr(o), ptr(a), ptr(_f64(old_logp)), ptr(_f64(adv)),
                          ptr(_f64(ret)), C.byref(cfg), ptr(g) if g is not None else None, p.size, info)
    return tuple(info), g


def gae(rewards, values, dones, bootstrap, gamma=0.99, lam=0.95):
    r, v, d, b = _f64(rewards), _f64(values), _f64(dones), _f64(bootstrap)
    T, E = r.shape
    adv, ret = np.zeros((T, E)), np.zeros((T, E))
    lib().oracle_gae(T, E, ptr(r), ptr(v), ptr(d), ptr(b), C.c_double(gamma), C.c_double(lam), ptr(adv), ptr(ret))
    return adv, ret


class AdamState:
    def __init__(self, n_params):
        self.m, self.v, self.t = np.zeros(n_params), np.zeros(n_params), C.c_int32(0)


def rng_words(seed, stream):
    """Rng(seed, stream)'s xoshiro256++ state (rng.hpp:15-25)."""
    mask = (1 << 64) - 1

    def splitmix(x):
        x = (x + 0x9E3779B97F4A7C15) & mask
        x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & mask
        x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & mask
        return x ^ (x >> 31)

    x = seed ^ splitmix((stream + 0x9E3779B97F4A7C15) & mask)
    out = (C.c_uint64 * 4)()
    for k in range(4):
        x = (x + 0x9E3779B97F4A7C15) & mask
        out[k] = splitmix(x)
    return out


def ppo_update(params, adam: AdamState, obs, actions, logp, values, rewards, dones, bootstrap, cfg=None, rng=None,
               act=6, hidden=64):
    """ppo_update in place on params (float64 array) / adam / rng; returns (loss, surrogate,
    value_loss, entropy)."""
    assert params.dtype == np.float64 and params.flags["C_CONTIGUOUS"]
    o, a = _f64(obs), _f64(actions)
    T, E = _f64(rewards).shape
    cfg = cfg or ppo_config()
    rng = rng if rng is not None else rng_words(0, 0x0272)
    st = (C.c_double * 4)()
    lib().oracle_ppo_update(ptr(params), o.shape[-1], act, hidden, T, E, ptr(o), ptr(a), ptr(_f64(logp)),
                            ptr(_f64(values)), ptr(_f64(rewards)), ptr(_f64(dones)), ptr(_f64(bootstrap)),
                            C.byref(cfg), ptr(adam.m), ptr(adam.v), C.byref(adam.t), params.size, rng, st)
    return tuple(st)
