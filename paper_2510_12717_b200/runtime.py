"""ctypes binding of lib/librmpc_b200.so and the BatchRunner mirror.

BatchRunner keeps the reference's method names and argument order
(/root/reference/proj/include/rmpc/batch.hpp:24-46):
    BatchRunner(n_envs, model, settings, workers=0)   # workers -> number of GPUs
    solve(states, cmds, gaits, prev=None, order=None) -> solutions
    size(), workers(), last_timing()
Batches are numpy arrays whose rows are the C structs (abi.py); solutions come back as a
numpy structured array with SOLUTION_DTYPE (rmpc_solution).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .abi import (NV, RMPC_ERR_STRUCTURAL, SOLUTION_DTYPE, STAGE_NAMES, Model, Settings, Timing,
                  default_model, default_settings)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RMPC_B200_LIB") or os.path.join(_HERE, "lib", "librmpc_b200.so")
_lib = None

_VP = C.c_void_p
_I = C.c_int32

EXPORTS = ("rmpc_model_default", "rmpc_settings_default", "rmpc_create", "rmpc_destroy",
           "rmpc_solve", "rmpc_solve_device", "rmpc_solve_device_active_set", "rmpc_size", "rmpc_workers", "rmpc_horizon",
           "rmpc_last_timing", "rmpc_last_error", "rmpc_status_message", "rmpc_stage_name",
           "rmpc_nominal_pose", "rmpc_mpc_torque", "rmpc_set_stage_profiling", "rmpc_build_info",
           "rmpc_smem_bytes", "rmpc_agents_per_cta", "rmpc_sizeof", "rmpc_fma_peak",
           "rmpc_solve_device_sharded", "rmpc_shard_info", "rmpc_set_schedule_sharing",
           "rmpc_solve_soa", "rmpc_solve_soa_device", "rmpc_kernel_launches", "rmpc_shard_range")

SOA_FIELDS = 28  # RMPC_SOA_FIELDS: q 0..8, qd 9..17, height, vx, wpitch, phase, period, phase_switch, offsets 24..27


class RmpcError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(f"rmpc error {code}: {message}")
        self.code = code


def load_library(path: str | None = None, build_if_missing: bool = True):
    """Load (and if needed build) the sm_100a library; raises if it cannot be loaded."""
    path = path or LIB_PATH
    if not os.path.exists(path):
        if not build_if_missing:
            raise OSError(f"{path} missing: run paper_2510_12717_b200/build.py")
        from .build import build
        build()
    L = C.CDLL(path)
    L.rmpc_create.argtypes = [_VP, _VP, _I, C.POINTER(_I), _I, C.POINTER(_VP)]
    L.rmpc_create.restype = _I
    L.rmpc_destroy.argtypes = [_VP]
    L.rmpc_destroy.restype = None
    L.rmpc_solve.argtypes = [_VP] * 8
    L.rmpc_solve.restype = _I
    L.rmpc_solve_device.argtypes = [_VP] * 9
    L.rmpc_solve_device.restype = _I
    L.rmpc_solve_soa.argtypes = [_VP, _VP, C.c_int64, _VP, _VP, _VP, _VP]
    L.rmpc_solve_soa.restype = _I
    L.rmpc_solve_soa_device.argtypes = [_VP, _VP, C.c_int64, _VP, _VP, _VP, _VP, _VP]
    L.rmpc_solve_soa_device.restype = _I
    L.rmpc_solve_device_active_set.argtypes = [_VP] * 7
    L.rmpc_solve_device_active_set.restype = _I
    L.rmpc_solve_device_sharded.argtypes = [_VP] * 9
    L.rmpc_solve_device_sharded.restype = _I
    L.rmpc_shard_info.argtypes = [_VP, _I, C.POINTER(_I), C.POINTER(_I), C.POINTER(_I)]
    L.rmpc_shard_info.restype = _I
    L.rmpc_shard_range.argtypes = [_I, _I, _I, C.POINTER(_I), C.POINTER(_I)]
    L.rmpc_shard_range.restype = _I
    for f in ("rmpc_size", "rmpc_workers", "rmpc_horizon"):
        getattr(L, f).argtypes = [_VP]
        getattr(L, f).restype = _I
    L.rmpc_last_timing.argtypes = [_VP, _VP]
    L.rmpc_last_timing.restype = _I
    L.rmpc_last_error.argtypes = [_VP]
    L.rmpc_last_error.restype = C.c_char_p
    L.rmpc_status_message.argtypes = [_I]
    L.rmpc_status_message.restype = C.c_char_p
    L.rmpc_stage_name.argtypes = [_I]
    L.rmpc_stage_name.restype = C.c_char_p
    L.rmpc_nominal_pose.argtypes = [_VP, _VP]
    L.rmpc_mpc_torque.argtypes = [_VP, _VP, _VP, _VP]
    L.rmpc_mpc_torque.restype = _I
    L.rmpc_set_stage_profiling.argtypes = [_VP, _I]
    L.rmpc_set_stage_profiling.restype = _I
    L.rmpc_set_schedule_sharing.argtypes = [_VP, _I]
    L.rmpc_set_schedule_sharing.restype = _I
    L.rmpc_build_info.restype = C.c_char_p
    L.rmpc_smem_bytes.argtypes = [_I]
    L.rmpc_smem_bytes.restype = _I
    L.rmpc_sizeof.argtypes = [_I]
    L.rmpc_sizeof.restype = _I
    L.rmpc_kernel_launches.argtypes = []
    L.rmpc_kernel_launches.restype = C.c_int64
    L.rmpc_fma_peak.argtypes = [_I, _VP]
    L.rmpc_fma_peak.restype = _I
    return L


def kernel_launches() -> int:
    """Solve-path kernels launched by this process so far (rmpc_kernel_launches)."""
    return int(library().rmpc_kernel_launches())


def fma_peak_tflops(device: int = 0) -> float:
    """Measured FP32 FMA peak of `device` (TFLOP/s), the roofline denominator."""
    v = C.c_double(0.0)
    rc = library().rmpc_fma_peak(device, C.byref(v))
    if rc != 0:
        raise RmpcError(rc, "rmpc_fma_peak failed")
    return v.value


def library():
    global _lib
    if _lib is None:
        _lib = load_library()
    return _lib


def _arr(a, cols, dtype=np.float64):
    a = np.ascontiguousarray(a, dtype=dtype)
    if a.ndim == 1:
        a = a.reshape(1, -1)
    if a.shape[1] != cols:
        raise ValueError(f"expected rows of {cols} values, got shape {a.shape}")
    return a


def to_soa(states, cmds, gaits, ld: int | None = None) -> np.ndarray:
    """The FP32 structure-of-arrays block of rmpc_solve_soa: row r = component r of every agent
    (RMPC_SOA_* order: the 18 state values, the 3 command values, the 7 gait values)."""
    states, cmds, gaits = _arr(states, 18), _arr(cmds, 3), _arr(gaits, 7)
    n = states.shape[0]
    out = np.zeros((SOA_FIELDS, ld or n), dtype=np.float32)
    out[:, :n] = np.hstack([states, cmds, gaits]).T
    return out


def from_soa(soa, n: int):
    """FP64 records (states, cmds, gaits) holding the block's values widened exactly to FP64:
    rmpc_solve on them equals rmpc_solve_soa on the block."""
    a = np.asarray(soa, dtype=np.float32)[:, :n].T.astype(np.float64)
    return np.ascontiguousarray(a[:, :18]), np.ascontiguousarray(a[:, 18:21]), np.ascontiguousarray(a[:, 21:28])


def nominal_pose(model: Model | None = None) -> np.ndarray:
    q = np.zeros(9)
    library().rmpc_nominal_pose(C.byref(model or default_model()), q.ctypes.data)
    return q


class BatchRunner:
    """rmpc::BatchRunner on B200: n_envs independent RTI-MPC instances per solve."""

    def __init__(self, n_envs: int, model: Model | None = None, settings: Settings | None = None,
                 workers: int = 0, devices=None):
        self._lib = library()
        self.model = model if model is not None else default_model()
        self.settings = settings if settings is not None else default_settings()
        if devices is None:
            devices = list(range(workers)) if workers > 0 else [0]
        devs = (_I * len(devices))(*devices)
        h = _VP()
        rc = self._lib.rmpc_create(C.byref(self.model), C.byref(self.settings), int(n_envs), devs,
                                   len(devices), C.byref(h))
        if rc != 0:
            raise RmpcError(rc, self._lib.rmpc_last_error(None).decode())
        self._h = h
        self._n = int(n_envs)
        self.horizon = int(self.settings.horizon)

    def close(self):
        if getattr(self, "_h", None):
            self._lib.rmpc_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def size(self) -> int:
        return self._lib.rmpc_size(self._h)

    def workers(self) -> int:
        return self._lib.rmpc_workers(self._h)

    def _err(self, rc):
        raise RmpcError(rc, self._lib.rmpc_last_error(self._h).decode())

    def solve(self, states, cmds, gaits, prev=None, order=None, *, want_z: bool = False,
              out: np.ndarray | None = None, z_out: np.ndarray | None = None):
        """BatchRunner::solve.  states (n,18), cmds (n,3), gaits (n,7) float64; prev =
        (solutions, z_star) of the previous tick (read only when settings.warm_start; z_star
        (n, T, 26) float32 -- without it no agent is warm-started, the reference's fallback for
        a prev without a valid plan, mpc.cpp:258).  `order` is accepted for API parity: results
        never depend on processing order.  Returns (solutions, z_star or None)."""
        del order
        states, cmds, gaits = _arr(states, 18), _arr(cmds, 3), _arr(gaits, 7)
        n, T = self._n, self.horizon
        if states.shape[0] != n or cmds.shape[0] != n or gaits.shape[0] != n:
            raise RmpcError(RMPC_ERR_STRUCTURAL, "BatchRunner::solve: input lengths != n_envs")
        if out is None:
            out = np.zeros(n, dtype=SOLUTION_DTYPE)
        elif out.dtype != SOLUTION_DTYPE or out.shape != (n,) or not out.flags["C_CONTIGUOUS"]:
            raise ValueError(f"out must be a contiguous SOLUTION_DTYPE array of length {n}")
        if want_z and z_out is None:
            z_out = np.zeros((n, T, NV), dtype=np.float32)
        if z_out is not None and (z_out.dtype != np.float32 or z_out.shape != (n, T, NV)
                                  or not z_out.flags["C_CONTIGUOUS"]):
            raise ValueError(f"z_out must be a contiguous float32 array of shape ({n}, {T}, {NV})")
        pv = pz = None
        if prev is not None:
            psol, pzs = prev
            if len(psol) != n:
                raise RmpcError(RMPC_ERR_STRUCTURAL, "BatchRunner::solve: prev length != n_envs")
            if pzs is not None:
                pz = np.asarray(pzs)
                if pz.dtype != np.float32 or pz.shape != (n, T, NV):
                    raise ValueError(f"prev z_star must be float32 of shape ({n}, {T}, {NV})")
                pz = np.ascontiguousarray(pz)
                pv = np.ascontiguousarray(psol, dtype=SOLUTION_DTYPE)
        rc = self._lib.rmpc_solve(self._h, states.ctypes.data, cmds.ctypes.data, gaits.ctypes.data,
                                  pv.ctypes.data if pv is not None else None,
                                  pz.ctypes.data if pz is not None else None, out.ctypes.data,
                                  z_out.ctypes.data if z_out is not None else None)
        if rc != 0:
            self._err(rc)
        return out, z_out

    def solve_soa(self, soa, prev=None, *, want_z: bool = False, out: np.ndarray | None = None,
                  z_out: np.ndarray | None = None):
        """rmpc_solve_soa: the inputs as one float32 (28, ld >= n) block (to_soa).  Same results
        as solve() on from_soa(soa); prev as in solve().  Returns (solutions, z_star or None)."""
        soa = np.asarray(soa)
        n, T = self._n, self.horizon
        if soa.dtype != np.float32 or soa.ndim != 2 or soa.shape[0] != SOA_FIELDS or soa.shape[1] < n \
                or not soa.flags["C_CONTIGUOUS"]:
            raise ValueError(f"soa must be a contiguous float32 array of shape ({SOA_FIELDS}, >= {n})")
        if out is None:
            out = np.zeros(n, dtype=SOLUTION_DTYPE)
        elif out.dtype != SOLUTION_DTYPE or out.shape != (n,) or not out.flags["C_CONTIGUOUS"]:
            raise ValueError(f"out must be a contiguous SOLUTION_DTYPE array of length {n}")
        if want_z and z_out is None:
            z_out = np.zeros((n, T, NV), dtype=np.float32)
        if z_out is not None and (z_out.dtype != np.float32 or z_out.shape != (n, T, NV)
                                  or not z_out.flags["C_CONTIGUOUS"]):
            raise ValueError(f"z_out must be a contiguous float32 array of shape ({n}, {T}, {NV})")
        pv = pz = None
        if prev is not None and prev[1] is not None:
            pz = np.asarray(prev[1])
            if pz.dtype != np.float32 or pz.shape != (n, T, NV):
                raise ValueError(f"prev z_star must be float32 of shape ({n}, {T}, {NV})")
            pz = np.ascontiguousarray(pz)
            pv = np.ascontiguousarray(prev[0], dtype=SOLUTION_DTYPE)
            if pv.shape != (n,):
                raise RmpcError(RMPC_ERR_STRUCTURAL, "BatchRunner::solve: prev length != n_envs")
        rc = self._lib.rmpc_solve_soa(self._h, soa.ctypes.data, soa.shape[1],
                                      pv.ctypes.data if pv is not None else None,
                                      pz.ctypes.data if pz is not None else None, out.ctypes.data,
                                      z_out.ctypes.data if z_out is not None else None)
        if rc != 0:
            self._err(rc)
        return out, z_out

    def solve_soa_device(self, soa, out, z_out=None, prev=None, prev_z=None, stream=None):
        """rmpc_solve_soa_device: `soa` a contiguous float32 CUDA tensor (28, ld >= n); other
        arguments as solve_device."""
        def p(t):
            if t is None:
                return None
            return t if isinstance(t, int) else t.data_ptr()
        n, T = self._n, self.horizon
        if not isinstance(soa, int):
            if soa.dim() != 2 or soa.shape[0] != SOA_FIELDS or soa.shape[1] < n or str(soa.dtype) != "torch.float32":
                raise ValueError(f"soa must be a float32 CUDA tensor of shape ({SOA_FIELDS}, >= {n})")
            self._check_device("soa", soa, SOA_FIELDS * n * 4)
            ld = soa.shape[1]
        else:
            ld = n
        for name, t, nb in (("out", out, n * SOLUTION_DTYPE.itemsize), ("z_out", z_out, n * T * NV * 4),
                            ("prev", prev, n * SOLUTION_DTYPE.itemsize), ("prev_z", prev_z, n * T * NV * 4)):
            self._check_device(name, t, nb)
        s = self._stream(stream, (soa, out))
        rc = self._lib.rmpc_solve_soa_device(self._h, p(soa), ld, p(prev), p(prev_z), p(out), p(z_out), s)
        if rc != 0:
            self._err(rc)

    @staticmethod
    def _stream(stream, tensors):
        """cudaStream_t for a launch: an explicit torch.cuda.Stream / int, else torch's current
        stream of the tensors' device (so the launch is ordered after the torch ops that
        produced them), else 0 = the legacy default stream."""
        if stream is not None:
            return stream if isinstance(stream, int) else stream.cuda_stream
        for t in tensors:
            if t is not None and not isinstance(t, int) and hasattr(t, "device"):
                import torch
                return torch.cuda.current_stream(t.device).cuda_stream
        return 0

    def _check_device(self, name, t, nbytes):
        if t is None or isinstance(t, int):
            return
        if not t.is_cuda or not t.is_contiguous():
            raise ValueError(f"{name} must be a contiguous CUDA tensor")
        if t.numel() * t.element_size() < nbytes:
            raise ValueError(f"{name} holds {t.numel() * t.element_size()} bytes, needs {nbytes}")

    def solve_device(self, states, cmds, gaits, out, z_out=None, prev=None, prev_z=None,
                     stream=None):
        """Device-resident solve: arguments are CUDA tensors (or raw device pointers) on this
        runner's device; enqueued on `stream` (default: torch's current stream), no sync."""
        def p(t):
            if t is None:
                return None
            return t if isinstance(t, int) else t.data_ptr()
        n, T = self._n, self.horizon
        for name, t, nb in (("states", states, n * 144), ("cmds", cmds, n * 24), ("gaits", gaits, n * 56),
                            ("out", out, n * SOLUTION_DTYPE.itemsize), ("z_out", z_out, n * T * NV * 4),
                            ("prev", prev, n * SOLUTION_DTYPE.itemsize), ("prev_z", prev_z, n * T * NV * 4)):
            self._check_device(name, t, nb)
        s = self._stream(stream, (states, out))
        rc = self._lib.rmpc_solve_device(self._h, p(states), p(cmds), p(gaits), p(prev), p(prev_z),
                                         p(out), p(z_out), s)
        if rc != 0:
            self._err(rc)

    def shard_info(self, g: int):
        """(device, begin, count) of shard g (rmpc_shard_info)."""
        d, b, c = _I(), _I(), _I()
        rc = self._lib.rmpc_shard_info(self._h, g, C.byref(d), C.byref(b), C.byref(c))
        if rc != 0:
            self._err(rc)
        return d.value, b.value, c.value

    def solve_device_sharded(self, states, cmds, gaits, out, z_out=None, streams=None):
        """Multi-device handle: per shard g lists of CUDA tensors on shard g's device holding its
        `count` agents (rmpc_solve_device_sharded); streams[g] default: torch's current stream."""
        G = self.workers()
        P = C.c_void_p * G

        def arr(ts):
            return None if ts is None else P(*[None if t is None else t.data_ptr() for t in ts])
        ss = P(*[self._stream(None if streams is None else streams[g], (states[g],)) for g in range(G)])
        rc = self._lib.rmpc_solve_device_sharded(self._h, arr(states), arr(cmds), arr(gaits), None, None,
                                                 arr(out), arr(z_out), ss)
        if rc != 0:
            self._err(rc)

    def solve_device_active_set(self, states, cmds, gaits, out, active, stream=None):
        """rmpc_solve_device plus the final iterate's active set: `active` is a uint8 CUDA
        tensor of n x (T+1) x 40 codes (0 inactive, 1 at lo, 2 at hi, 3 equality / no row)."""
        def p(t):
            return t if isinstance(t, int) else t.data_ptr()
        s = self._stream(stream, (states, out))
        rc = self._lib.rmpc_solve_device_active_set(self._h, p(states), p(cmds), p(gaits), p(out), p(active), s)
        if rc != 0:
            self._err(rc)

    def set_stage_profiling(self, enabled: bool = True):
        self._lib.rmpc_set_stage_profiling(self._h, int(enabled))

    def set_schedule_sharing(self, level=True):
        """Cold-start schedule sharing (rmpc_set_schedule_sharing): each distinct contact
        schedule is factorized once.  True / 2 (default): lane-per-agent squads where the
        horizon fits them (T <= 10) and the batch exceeds two waves of the per-agent kernel,
        else the per-agent kernel; 3: squads always; 1: warp-pair CTAs per schedule,
        bit-identical to the per-agent solve; False / 0: per-agent factorization."""
        level = 2 if level is True else int(level)
        self._lib.rmpc_set_schedule_sharing(self._h, level)

    def last_timing(self) -> dict:
        t = Timing()
        self._lib.rmpc_last_timing(self._h, C.byref(t))
        return dict(batch_size=t.batch_size, devices=t.devices, total_ms=t.total_ms,
                    h2d_ms=t.h2d_ms, kernel_ms=t.kernel_ms, d2h_ms=t.d2h_ms,
                    stage_ms=dict(zip(STAGE_NAMES, list(t.stage_ms))),
                    stage_mean_ms=dict(zip(STAGE_NAMES, list(t.stage_mean_ms))),
                    stage_std_ms=dict(zip(STAGE_NAMES, list(t.stage_std_ms))))

    def mpc_torque(self, solution, state) -> np.ndarray:
        """mpc_torque (mpc.cpp:340-344): PD + feed-forward, clamped; raises on a failed solve."""
        sol = np.ascontiguousarray(np.asarray(solution, dtype=SOLUTION_DTYPE).reshape(1))
        st = _arr(state, 18)
        tau = np.zeros(6)
        rc = self._lib.rmpc_mpc_torque(C.byref(self.model), sol.ctypes.data, st.ctypes.data,
                                       tau.ctypes.data)
        if rc != 0:
            raise RmpcError(rc, "mpc_torque: solution status is failed")
        return tau
