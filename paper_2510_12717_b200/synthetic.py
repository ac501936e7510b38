"""Synthetic agent batches from bit-exact xoshiro256++ streams.

rng.hpp (/root/reference/proj/include/rmpc/rng.hpp:15-75) restated with numpy uint64
arithmetic, vectorised over agents: agent i draws from Rng(seed, stream=i).
"""
from __future__ import annotations

import numpy as np

from .abi import Model, Settings, default_model, default_settings

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_G = np.uint64(0x9E3779B97F4A7C15)


def _splitmix(x):
    x = x + _G
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def _rotl(x, k):
    return (x << np.uint64(k)) | (x >> np.uint64(64 - k))


class Xoshiro:
    """Vectorised rmpc::Rng: one independent stream per element of `streams`."""

    def __init__(self, seed: int, streams):
        streams = np.asarray(streams, dtype=np.uint64)
        with np.errstate(over="ignore"):
            x = np.uint64(seed) ^ _splitmix(streams + _G)
            s = []
            for _ in range(4):
                x = x + _G
                s.append(_splitmix(x))
        self.s = s

    def next_u64(self):
        s0, s1, s2, s3 = self.s
        with np.errstate(over="ignore"):
            result = _rotl(s0 + s3, 23) + s0
            t = s1 << np.uint64(17)
            s2 = s2 ^ s0
            s3 = s3 ^ s1
            s1 = s1 ^ s2
            s0 = s0 ^ s3
            s2 = s2 ^ t
            s3 = _rotl(s3, 45)
        self.s = [s0, s1, s2, s3]
        return result

    def uniform(self, lo=0.0, hi=1.0):
        u = (self.next_u64() >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
        return lo + (hi - lo) * u

    def uniform_int(self, n: int):
        return (self.next_u64() % np.uint64(n)).astype(np.int64)


PHASE_SWITCHES = (0.4, 0.5, 0.65, 1.0)  # flight, walk, double stance, standing (analysis.cpp:305-307)


def synthetic_batch(n: int, kind: str = "random", seed: int = 0, model: Model | None = None,
                    settings: Settings | None = None, nominal=None):
    """(states (n,18), cmds (n,3), gaits (n,7)) float64.

    kind="standing": nominal pose at rest, standing gait, zero command (C1, test_mpc.cpp:235).
    kind="random":   nominal pose, qd[0], qd[2] ~ U(-0.5, 0.5), walking gait with phase ~ U(0,1),
                     cmd.vx ~ U(-0.6, 0.6), cmd.height = nominal height (C2-C4, batch.cpp:95-104,
                     env.hpp:63-72); draws per agent in that order from Rng(seed, i).
    kind="mixed":    as "random" plus phase_switch drawn from PHASE_SWITCHES (C5).
    """
    model = model or default_model()
    settings = settings or default_settings()
    if nominal is None:
        from .runtime import nominal_pose
        nominal = nominal_pose(model)
    states = np.zeros((n, 18))
    states[:, :9] = nominal
    cmds = np.zeros((n, 3))
    cmds[:, 0] = model.nominal_height()
    gaits = np.zeros((n, 7))
    gaits[:, 1] = settings.gait_period
    gaits[:, 2] = settings.phase_switch
    gaits[:, 3:] = np.array(settings.phase_offsets[:])
    if kind == "standing":
        gaits[:, 2] = 1.0
        gaits[:, 3:] = (0.5, 0.5, 0.0, 0.0)
        return states, cmds, gaits
    rng = Xoshiro(seed, np.arange(n))
    states[:, 9] = rng.uniform(-0.5, 0.5)
    states[:, 11] = rng.uniform(-0.5, 0.5)
    gaits[:, 0] = rng.uniform()
    cmds[:, 1] = rng.uniform(-0.6, 0.6)
    if kind == "mixed":
        gaits[:, 2] = np.asarray(PHASE_SWITCHES)[rng.uniform_int(len(PHASE_SWITCHES))]
    elif kind != "random":
        raise ValueError(f"unknown synthetic batch kind {kind!r}")
    return states, cmds, gaits
