"""Closed-loop step after the solve over include/rmpc_b200_env.h:
physics_step (env.cpp:38-68), the fused mpc_torque + blend + physics control step
(mpc.cpp:340-344, policy.cpp:133-157, ppo.cpp:340-349) and observe (policy.cpp:104-122), all
device-resident on CUDA tensors.  Layouts: states (n, 18) f64 = rmpc_state, gaits (n, 7) f64 =
rmpc_gait, bodies (n, 2) f64 = rmpc_body {mu, mass_scale}, tau / action (n, 6) f64,
solutions SOLUTION_DTYPE bytes, observations (n, 23) f64."""
from __future__ import annotations

import ctypes as C

from .abi import Model, default_model
from .runtime import RmpcError, library

OBS_DIM = 23
BLEND = {"joint-joint": 0, "joint-torque": 1, "torque-torque": 2}
SIM_OK, SIM_BLOWUP = 0, 1

_VP, _I, _D = C.c_void_p, C.c_int32, C.c_double


class EnvConfig(C.Structure):
    """EnvConfig physics + TerrainConfig (env.hpp:16-63)."""
    _fields_ = [("control_dt", _D), ("substeps", _I), ("terrain_kind", _I), ("k_n", _D),
                ("c_n", _D), ("v_slip", _D), ("amplitude", _D), ("cell", _D), ("extent", _D),
                ("terrain_seed", C.c_uint64)]


def _bind(L):
    if getattr(L, "_env_bound", False):
        return L
    L.rmpc_env_config_default.argtypes = [_VP]
    L.rmpc_env_config_default.restype = None
    L.rmpc_env_create.argtypes = [_VP, _VP, _I, C.POINTER(_VP)]
    L.rmpc_env_create.restype = _I
    L.rmpc_env_destroy.argtypes = [_VP]
    L.rmpc_env_destroy.restype = None
    L.rmpc_env_height_at.argtypes = [_VP, _D, C.POINTER(_D)]
    L.rmpc_env_height_at.restype = _I
    L.rmpc_physics_step_device.argtypes = [_VP, _I, _VP, _VP, _VP, _VP, _VP, _VP]
    L.rmpc_physics_step_device.restype = _I
    L.rmpc_control_step_device.argtypes = [_VP, _I, _VP, _VP, _I, _D, _VP, _VP, _VP, _VP, _VP, _VP]
    L.rmpc_control_step_device.restype = _I
    L.rmpc_observe_device.argtypes = [_I, _VP, _VP, _VP, _D, _D, _VP, _VP]
    L.rmpc_observe_device.restype = _I
    L.rmpc_plan_feedback_device.argtypes = [_I, _I, _VP, _VP, _VP, _VP, _D, _VP]
    L.rmpc_plan_feedback_device.restype = _I
    L.rmpc_policy_create.argtypes = [_I, _I, _I, _VP, _I, _I, C.POINTER(_VP)]
    L.rmpc_policy_create.restype = _I
    L.rmpc_policy_destroy.argtypes = [_VP]
    L.rmpc_policy_destroy.restype = None
    L.rmpc_policy_forward_device.argtypes = [_VP, _I, _VP, _VP, _VP, _VP]
    L.rmpc_policy_forward_device.restype = _I
    L.rmpc_env_sizeof.argtypes = [_I]
    L.rmpc_env_sizeof.restype = _I
    L.rmpc_policy_num_params.argtypes = [_VP]
    L.rmpc_policy_num_params.restype = _I
    L.rmpc_policy_get_params.argtypes = [_VP, _VP, _I]
    L.rmpc_policy_get_params.restype = _I
    L.rmpc_policy_set_params.argtypes = [_VP, _VP, _I]
    L.rmpc_policy_set_params.restype = _I
    L._env_bound = True
    return L


def default_env_config(**overrides) -> EnvConfig:
    c = EnvConfig()
    _bind(library()).rmpc_env_config_default(C.byref(c))
    for k, v in overrides.items():
        setattr(c, k, v)
    return c


def _p(t):
    if t is None:
        return None
    return t if isinstance(t, int) else t.data_ptr()


def _s(stream):
    if stream is None:
        return None
    s = stream if isinstance(stream, int) else stream.cuda_stream
    return 1 if s == 0 else s  # cudaStreamLegacy


class Env:
    """The reference's per-env simulator step, batched on one GPU (device `device`)."""

    def __init__(self, model: Model | None = None, config: EnvConfig | None = None, device: int = 0):
        self._lib = _bind(library())
        self.model = model if model is not None else default_model()
        self.config = config if config is not None else default_env_config()
        h = _VP()
        rc = self._lib.rmpc_env_create(C.byref(self.model), C.byref(self.config), device, C.byref(h))
        if rc != 0:
            raise RmpcError(rc, "rmpc_env_create failed")
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            self._lib.rmpc_env_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def height_at(self, x: float) -> float:
        v = _D()
        self._lib.rmpc_env_height_at(self._h, float(x), C.byref(v))
        return v.value

    def physics_step(self, states, gaits, tau, bodies=None, sim_status=None, stream=None):
        n = states.shape[0]
        rc = self._lib.rmpc_physics_step_device(self._h, n, _p(states), _p(gaits), _p(bodies), _p(tau),
                                                _p(sim_status), _s(stream))
        if rc != 0:
            raise RmpcError(rc, "rmpc_physics_step_device failed")

    def control_step(self, solutions, states, gaits, action=None, strategy: str | int = "joint-joint",
                     lam: float = 0.0, bodies=None, tau_out=None, sim_status=None, stream=None):
        n = states.shape[0]
        st = BLEND[strategy] if isinstance(strategy, str) else int(strategy)
        rc = self._lib.rmpc_control_step_device(self._h, n, _p(solutions), _p(action), st, float(lam),
                                                _p(states), _p(gaits), _p(bodies), _p(tau_out),
                                                _p(sim_status), _s(stream))
        if rc != 0:
            raise RmpcError(rc, "rmpc_control_step_device failed")

    def observe(self, states, gaits, solutions, obs, v_mpc_scale: float = 1e-2,
                v_mpc_sentinel: float = 10.0, stream=None):
        n = states.shape[0]
        rc = self._lib.rmpc_observe_device(n, _p(states), _p(gaits), _p(solutions), v_mpc_scale,
                                           v_mpc_sentinel, _p(obs), _s(stream))
        if rc != 0:
            raise RmpcError(rc, "rmpc_observe_device failed")


def plan_feedback(z, solutions, states, gaits, horizon: int, dt: float = 0.01, stream=None):
    """C5 open-loop replanning: state <- (q*[1], qd*[1]) of the last plan, phase += dt/period."""
    L = _bind(library())
    rc = L.rmpc_plan_feedback_device(states.shape[0], horizon, _p(z), _p(solutions), _p(states), _p(gaits),
                                     float(dt), _s(stream))
    if rc != 0:
        raise RmpcError(rc, "rmpc_plan_feedback_device failed")


class Policy:
    """Residual policy (policy_forward, policy.cpp:85-102) on the device, FP64.  `params` is the
    flat PolicyParams vector in MlpParams::flatten_into order (pi, value, log_std)."""

    def __init__(self, params, obs_dim: int = OBS_DIM, act_dim: int = 6, hidden: int = 64, device: int = 0):
        import numpy as np
        self._lib = _bind(library())
        p = np.ascontiguousarray(params, dtype=np.float64)
        self.obs_dim, self.act_dim, self.hidden = obs_dim, act_dim, hidden
        h = _VP()
        rc = self._lib.rmpc_policy_create(obs_dim, act_dim, hidden, p.ctypes.data, p.size, device, C.byref(h))
        if rc != 0:
            raise RmpcError(rc, "rmpc_policy_create failed (parameter count or dims)")
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            self._lib.rmpc_policy_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def num_params(self) -> int:
        return int(self._lib.rmpc_policy_num_params(self._h))

    def get_params(self):
        """flatten_policy (ppo.cpp:144-153): a host copy of the device parameters."""
        import numpy as np
        out = np.zeros(self.num_params)
        rc = self._lib.rmpc_policy_get_params(self._h, out.ctypes.data, out.size)
        if rc != 0:
            raise RmpcError(rc, "rmpc_policy_get_params failed")
        return out

    def set_params(self, params):
        """unflatten_policy (ppo.cpp:155-162) from a host vector."""
        import numpy as np
        p = np.ascontiguousarray(params, dtype=np.float64)
        rc = self._lib.rmpc_policy_set_params(self._h, p.ctypes.data, p.size)
        if rc != 0:
            raise RmpcError(rc, "rmpc_policy_set_params failed (parameter count)")

    @property
    def log_std(self):
        return self.get_params()[-self.act_dim:]

    def forward(self, obs, mean=None, value=None, stream=None):
        rc = self._lib.rmpc_policy_forward_device(self._h, obs.shape[0], _p(obs), _p(mean), _p(value), _s(stream))
        if rc != 0:
            raise RmpcError(rc, "rmpc_policy_forward_device failed")
