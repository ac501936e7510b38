"""TEST INFRASTRUCTURE ONLY — ctypes wrapper of oracle/_ref/librmpc_ref.so: the UNMODIFIED
reference sources (/root/reference/proj/src/{gait,robot,mpc,csc,ruiz,qp,ldl,batch,env,policy,
ppo}.cpp) compiled against the Eigen-subset shim (oracle/eigen_shim, Makefile.ref) behind
oracle/ref_capi.cpp.

It pins the restated oracle (oracle.py) and the CUDA path to numbers the reference code itself
produces.  Only tests/ (golden-fixture generation runs here, where /root/reference exists),
__graft_entry__.build() and bench.py's `--impl reference` / cpu_baseline legs load it.  The
library travels to the GPU box prebuilt (oracle/_ref is git-ignored, not gpurun-ignored); the
box has no /root/reference, so nothing here rebuilds it there.

Deviation from the reference build: Eigen's AMDOrdering is replaced by the oracle's
approximate-minimum-degree ordering (eigen_shim/Eigen/OrderingMethods); the permutation only
changes rounding.  Everything else is the reference's own code.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2510_12717_b200.abi import NV, Model, Settings, ptr  # noqa: F401

from .oracle import ORACLE_SOLUTION_DTYPE

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "librmpc_ref.so")
REF_SRC = os.environ.get("RMPC_REFERENCE", "/root/reference/proj")

_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH) or os.path.isdir(os.path.join(REF_SRC, "src"))


def build() -> str:
    """Compile the reference sources (needs /root/reference; the GPU box uses the prebuilt .so)."""
    subprocess.run(["make", "-s", "-j8", "-C", _HERE, "-f", "Makefile.ref", f"REF={REF_SRC}"], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.ref_solve_batch.restype = C.c_int32
        L.ref_build_qp.restype = C.c_int32
        L.ref_sizeof_solution.restype = C.c_int32
        L.ref_terrain_height_at.restype = C.c_double
        L.ref_terrain_height_at.argtypes = [C.c_void_p, C.c_double]
        L.ref_init_policy.restype = C.c_int32
        assert L.ref_sizeof_solution() == ORACLE_SOLUTION_DTYPE.itemsize
        _lib = L
    return _lib


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None:
        a = a.reshape(shape)
    return a


def solve_batch(model: Model, settings: Settings, states, cmds, gaits, *, prev_z=None,
                prev_ok=None, workers: int = 1, want_z: bool = True):
    """rmpc::BatchRunner(n, model, settings, workers).solve(...).  Returns (solutions with
    ORACLE_SOLUTION_DTYPE (v_quad / v_lin are NaN: the reference does not expose them),
    z_star [n,T,26] or None, stage mean ms [7], stage std ms [7], wall ms)."""
    states = _f64(states)
    n = states.shape[0]
    cmds, gaits = _f64(cmds, (n, 3)), _f64(gaits, (n, 7))
    T = settings.horizon
    out = np.zeros(n, dtype=ORACLE_SOLUTION_DTYPE)
    z = np.zeros((n, T, NV)) if want_z else None
    mean, std = np.zeros(7), np.zeros(7)
    wall = C.c_double(0.0)
    pz = _f64(prev_z) if prev_z is not None else None
    pok = np.ascontiguousarray(prev_ok, dtype=np.int32) if prev_ok is not None else None
    rc = lib().ref_solve_batch(C.byref(model), C.byref(settings), C.c_int32(n), ptr(states), ptr(cmds),
                               ptr(gaits), ptr(pz), ptr(pok, C.c_int32), C.c_int32(workers),
                               out.ctypes.data_as(C.c_void_p), ptr(z), ptr(mean), ptr(std), C.byref(wall))
    if rc != 0:
        raise ValueError(f"ref_solve_batch: structural error (code {rc})")
    return out, z, mean, std, wall.value


def nominal_pose(model: Model) -> np.ndarray:
    q = np.zeros(9)
    lib().ref_nominal_pose(C.byref(model), ptr(q))
    return q


def build_qp(model: Model, settings: Settings, state, cmd, gait):
    """Dense view of the reference's build_qp at rti_step's cold guess: dict(A, P_diag, q, lo,
    hi, nnz) or None when build_qp throws."""
    n, m, nnz = C.c_int32(), C.c_int32(), C.c_int32()
    args = (C.byref(model), C.byref(settings), ptr(_f64(state, (18,))), ptr(_f64(cmd, (3,))),
            ptr(_f64(gait, (7,))))
    if lib().ref_build_qp(*args, C.byref(n), C.byref(m), C.byref(nnz), None, None, None, None, None) != 0:
        return None
    A = np.zeros((m.value, n.value))
    P, q = np.zeros(n.value), np.zeros(n.value)
    lo, hi = np.zeros(m.value), np.zeros(m.value)
    lib().ref_build_qp(*args, C.byref(n), C.byref(m), C.byref(nnz), ptr(A), ptr(P), ptr(q), ptr(lo), ptr(hi))
    return dict(A=A, P_diag=P, q=q, lo=lo, hi=hi, nnz=nnz.value)


def mass_matrix(model: Model, q) -> np.ndarray:
    M = np.zeros((9, 9))
    lib().ref_mass_matrix(C.byref(model), ptr(_f64(q, (9,))), ptr(M))
    return M


def bias_forces(model: Model, q, qd) -> np.ndarray:
    h = np.zeros(9)
    lib().ref_bias_forces(C.byref(model), ptr(_f64(q, (9,))), ptr(_f64(qd, (9,))), ptr(h))
    return h


def inverse_dynamics(model: Model, q, qd, qdd, F):
    tau, base = np.zeros(6), np.zeros(3)
    lib().ref_inverse_dynamics(C.byref(model), ptr(_f64(q, (9,))), ptr(_f64(qd, (9,))), ptr(_f64(qdd, (9,))),
                               ptr(_f64(F, (8,))), ptr(tau), ptr(base))
    return tau, base


# ---------------------------------------------------------------- env / policy / ppo
def terrain_height_at(cfg, x: float) -> float:
    return lib().ref_terrain_height_at(C.byref(cfg), float(x))


def physics_step_batch(model: Model, cfg, states, gaits, tau, bodies=None):
    st, ga = _f64(states).copy().reshape(-1, 18), _f64(gaits).copy().reshape(-1, 7)
    n = st.shape[0]
    tau = _f64(tau, (n, 6))
    bo = None if bodies is None else _f64(bodies, (n, 2))
    status = np.zeros(n, np.int32)
    lib().ref_physics_step_batch(C.byref(model), C.byref(cfg), C.c_int32(n), ptr(st), ptr(ga), ptr(bo), ptr(tau),
                                 status.ctypes.data_as(C.c_void_p))
    return st, ga, status


def control_step_batch(model: Model, cfg, solutions, states, gaits, action=None, strategy=0, lam=0.0,
                       bodies=None):
    st, ga = _f64(states).copy().reshape(-1, 18), _f64(gaits).copy().reshape(-1, 7)
    n = st.shape[0]
    sols = np.ascontiguousarray(solutions)
    act = None if action is None else _f64(action, (n, 6))
    bo = None if bodies is None else _f64(bodies, (n, 2))
    tau = np.zeros((n, 6))
    status = np.zeros(n, np.int32)
    lib().ref_control_step_batch(C.byref(model), C.byref(cfg), C.c_int32(n), C.c_void_p(sols.ctypes.data),
                                 ptr(act), C.c_int32(int(strategy)), C.c_double(lam), ptr(st), ptr(ga), ptr(bo),
                                 ptr(tau), status.ctypes.data_as(C.c_void_p))
    return st, ga, tau, status


def observe_batch(states, gaits, solutions, scale=1e-2, sentinel=10.0):
    st, ga = _f64(states).reshape(-1, 18), _f64(gaits).reshape(-1, 7)
    n = st.shape[0]
    sols = np.ascontiguousarray(solutions)
    obs = np.zeros((n, 23))
    lib().ref_observe_batch(C.c_int32(n), ptr(st), ptr(ga), C.c_void_p(sols.ctypes.data), C.c_double(scale),
                            C.c_double(sentinel), ptr(obs))
    return obs


def init_policy(obs=23, act=6, hidden=64, seed=0) -> np.ndarray:
    n = lib().ref_init_policy(obs, act, hidden, C.c_uint64(seed), None, 0)
    out = np.zeros(n)
    lib().ref_init_policy(obs, act, hidden, C.c_uint64(seed), ptr(out), n)
    return out


def policy_forward(params, obs, act=6, hidden=64):
    o = _f64(obs)
    o = o.reshape(-1, o.shape[-1])
    n, od = o.shape
    mean, value = np.zeros((n, act)), np.zeros(n)
    lib().ref_policy_forward_batch(ptr(_f64(params)), od, act, hidden, n, ptr(o), ptr(mean), ptr(value))
    return mean, value


def ppo_loss(params, obs, actions, old_logp, adv, ret, cfg, act=6, hidden=64, grads=True):
    p = _f64(params)
    o, a = _f64(obs), _f64(actions)
    n, od = o.shape
    info = (C.c_double * 4)()
    g = np.zeros(p.size) if grads else None
    lib().ref_ppo_loss(ptr(p), od, act, hidden, n, ptr(o), ptr(a), ptr(_f64(old_logp)), ptr(_f64(adv)),
                       ptr(_f64(ret)), C.byref(cfg), ptr(g), info)
    return tuple(info), g


def gae(rewards, values, dones, bootstrap, gamma=0.99, lam=0.95):
    r, v, d, b = _f64(rewards), _f64(values), _f64(dones), _f64(bootstrap)
    T, E = r.shape
    adv, ret = np.zeros((T, E)), np.zeros((T, E))
    lib().ref_gae(T, E, ptr(r), ptr(v), ptr(d), ptr(b), C.c_double(gamma), C.c_double(lam), ptr(adv), ptr(ret))
    return adv, ret


def ppo_update_seq(params, obs, actions, logp, values, rewards, dones, bootstrap, cfg, seed=0, stream=0x0272,
                   n_updates=1, act=6, hidden=64):
    """n_updates consecutive ppo_update calls with one Adam and one Rng(seed, stream) carried:
    returns (params after, [stats per call])."""
    p = _f64(params).copy()
    o, a = _f64(obs), _f64(actions)
    T, E = _f64(rewards).shape
    st = (C.c_double * (4 * n_updates))()
    lib().ref_ppo_update_seq(ptr(p), o.shape[-1], act, hidden, T, E, ptr(o), ptr(a), ptr(_f64(logp)),
                             ptr(_f64(values)), ptr(_f64(rewards)), ptr(_f64(dones)), ptr(_f64(bootstrap)),
                             C.byref(cfg), C.c_uint64(seed), C.c_uint64(stream), C.c_int32(n_updates), st)
    return p, [tuple(st[4 * k:4 * k + 4]) for k in range(n_updates)]


REASONS = ("survived", "non_finite", "height", "orientation", "velocity", "self_collision",
           "controller_failed")


def closed_loop(model: Model, settings: Settings, cfg, phase_switch=1.0, ticks=500):
    """The reference's own closed loop (rti_step -> mpc_torque -> Env::step) from the nominal
    standing pose at zero command: (ticks survived, reason, trace (ticks, 18) of the states)."""
    trace = np.full((ticks, 18), np.nan)
    reason = C.c_int32(0)
    lib().ref_closed_loop.restype = C.c_int32
    alive = lib().ref_closed_loop(C.byref(model), C.byref(settings), C.byref(cfg), C.c_double(phase_switch),
                                  C.c_int32(ticks), ptr(trace), C.byref(reason))
    return alive, REASONS[reason.value], trace


def check_termination(model: Model, cfg, state) -> str:
    """The reference's check_termination on one state (n/a reasons: 'survived' = not terminated)."""
    lib().ref_check_termination.restype = C.c_int32
    return REASONS[lib().ref_check_termination(C.byref(model), C.byref(cfg), ptr(_f64(state, (18,))))]
