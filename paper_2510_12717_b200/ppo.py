"""PPO batch on the device over include/rmpc_b200_env.h, FP64 like the
reference (/root/reference/proj/src/ppo.cpp):

  ppo_loss    ppo_loss (ppo.cpp:79-135): loss terms and the gradient of every parameter
  gae         gae_advantages (ppo.cpp:28-45)
  Adam        AdamOptimizer (ppo.cpp:179-193), moments on the policy's device
  ppo_update  ppo_update (ppo.cpp:195-276) on a device-resident rollout

Tensors are CUDA float64; rollouts are (steps, envs[, dim]) row-major like RolloutBuffer.
"""
from __future__ import annotations

import ctypes as C

from .env import Policy, _bind as _bind_env, _p, _s
from .runtime import RmpcError, library

_VP, _I, _D = C.c_void_p, C.c_int32, C.c_double


class PpoConfig(C.Structure):
    """PpoConfig (ppo.hpp:14-24), the update part."""
    _fields_ = [("gamma", _D), ("lam_gae", _D), ("clip_eps", _D), ("epochs", _I), ("minibatches", _I),
                ("lr", _D), ("entropy_coef", _D), ("value_coef", _D), ("max_grad_norm", _D)]


class LossInfo(C.Structure):
    """PpoLossInfo (ppo.hpp:70-75)."""
    _fields_ = [("total", _D), ("surrogate", _D), ("value_loss", _D), ("entropy", _D)]


class UpdateStats(C.Structure):
    """PpoUpdateStats (ppo.hpp:103-108)."""
    _fields_ = [("loss", _D), ("surrogate", _D), ("value_loss", _D), ("entropy", _D)]


def _bind(L):
    _bind_env(L)
    if getattr(L, "_ppo_bound", False):
        return L
    L.rmpc_ppo_config_default.argtypes = [_VP]
    L.rmpc_ppo_config_default.restype = None
    L.rmpc_ppo_loss_device.argtypes = [_VP, _I, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP]
    L.rmpc_ppo_loss_device.restype = _I
    L.rmpc_gae_device.argtypes = [_I, _I, _VP, _VP, _VP, _VP, _D, _D, _VP, _VP, _VP]
    L.rmpc_gae_device.restype = _I
    L.rmpc_adam_create.argtypes = [_VP, _D, C.POINTER(_VP)]
    L.rmpc_adam_create.restype = _I
    L.rmpc_adam_destroy.argtypes = [_VP]
    L.rmpc_adam_destroy.restype = None
    L.rmpc_rng_seed.argtypes = [C.c_uint64, C.c_uint64, _VP]
    L.rmpc_rng_seed.restype = None
    L.rmpc_ppo_update_device.argtypes = [_VP, _VP, _I, _I, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP]
    L.rmpc_ppo_update_device.restype = _I
    L._ppo_bound = True
    return L


def default_ppo_config(**overrides) -> PpoConfig:
    c = PpoConfig()
    _bind(library()).rmpc_ppo_config_default(C.byref(c))
    for k, v in overrides.items():
        setattr(c, k, v)
    return c


def rng_state(seed: int, stream: int):
    """Rng(seed, stream) (rng.hpp:15-25) as four xoshiro256++ words (advanced by ppo_update)."""
    st = (C.c_uint64 * 4)()
    _bind(library()).rmpc_rng_seed(seed, stream, st)
    return st


def ppo_loss(policy: Policy, obs, actions, old_logp, advantages, returns, cfg: PpoConfig | None = None,
             grads=None, stream=None):
    """ppo_loss over a batch of n samples; returns (LossInfo, grads) where grads is the
    flatten_grads vector (a new CUDA tensor unless one is passed; None skips the gradient when
    grads is False)."""
    import torch
    L = _bind(library())
    cfg = cfg or default_ppo_config()
    n = obs.shape[0]
    if grads is None:
        grads = torch.zeros(policy.num_params, dtype=torch.float64, device=obs.device)
    info = torch.zeros(4, dtype=torch.float64, device=obs.device)
    rc = L.rmpc_ppo_loss_device(policy._h, n, _p(obs), _p(actions), _p(old_logp), _p(advantages), _p(returns),
                                C.byref(cfg), None if grads is False else _p(grads), _p(info), _s(stream))
    if rc != 0:
        raise RmpcError(rc, "rmpc_ppo_loss_device failed")
    v = info.cpu().tolist()
    return LossInfo(*v), (None if grads is False else grads)


def gae(rewards, values, dones, bootstrap, gamma: float = 0.99, lam: float = 0.95, stream=None):
    """gae_advantages: (advantages, returns), raw, (steps, envs)."""
    import torch
    T, E = rewards.shape
    adv = torch.empty_like(rewards)
    ret = torch.empty_like(rewards)
    rc = _bind(library()).rmpc_gae_device(T, E, _p(rewards), _p(values), _p(dones), _p(bootstrap), gamma, lam,
                                          _p(adv), _p(ret), _s(stream))
    if rc != 0:
        raise RmpcError(rc, "rmpc_gae_device failed")
    return adv, ret


class Adam:
    """AdamOptimizer(num_params, lr) bound to a policy (betas 0.9 / 0.999, eps 1e-8)."""

    def __init__(self, policy: Policy, lr: float = 3e-4):
        self._lib = _bind(library())
        self.policy = policy
        h = _VP()
        rc = self._lib.rmpc_adam_create(policy._h, lr, C.byref(h))
        if rc != 0:
            raise RmpcError(rc, "rmpc_adam_create failed")
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            self._lib.rmpc_adam_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def ppo_update(policy: Policy, adam: Adam, obs, actions, logp, values, rewards, dones, bootstrap,
               cfg: PpoConfig | None = None, rng=None, stream=None) -> UpdateStats:
    """ppo_update on a device-resident rollout (obs (T, E, obs_dim), actions (T, E, act_dim),
    logp / values / rewards / dones (T, E), bootstrap (E,)); policy parameters are updated in
    place and `rng` (rng_state) advances like the reference's update_rng."""
    L = _bind(library())
    cfg = cfg or default_ppo_config()
    rng = rng if rng is not None else rng_state(0, 0x0272)
    T, E = rewards.shape
    st = UpdateStats()
    rc = L.rmpc_ppo_update_device(policy._h, adam._h, T, E, _p(obs), _p(actions), _p(logp), _p(values), _p(rewards),
                                  _p(dones), _p(bootstrap), C.byref(cfg), rng, C.byref(st), _s(stream))
    if rc != 0:
        raise RmpcError(rc, "rmpc_ppo_update_device failed")
    return st
