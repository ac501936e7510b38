"""Trajectory log: the reference's binary LogRecord stream
(/root/reference/proj/include/rmpc/trajlog.hpp:20-45, proj/src/trajlog.cpp:13-98) -- magic
"RMPCLG01", uint32 version 1, uint32 record size, then packed LogRecord structs -- written
from the batched closed loop's arrays, plus the reader and the CSV export with the reference's
column names.  Host-side IO (numpy); the records are assembled from device results.
"""
from __future__ import annotations

import numpy as np

MAGIC = b"RMPCLG01"
VERSION = 1
REWARD_TERMS = ("lin_vel", "ang_vel", "action_rate1", "action_rate2", "torques", "orientation",
                "height", "joint_reg", "self_collision", "termination")

LOG_RECORD_DTYPE = np.dtype([
    ("time", np.float64), ("q", np.float64, (9,)), ("qd", np.float64, (9,)),
    ("tau_mpc", np.float64, (6,)), ("tau_res", np.float64, (6,)), ("f_contact", np.float64, (8,)),
    ("phase", np.float64), ("v_mpc", np.float64), ("reward_total", np.float64),
    ("reward_terms", np.float64, (10,)), ("flags", np.uint32), ("pad", np.uint32),
])
assert LOG_RECORD_DTYPE.itemsize == 424  # sizeof(rmpc::LogRecord)


def records_from_tick(time: float, states, gaits, solutions, tau_mpc=None, tau_res=None,
                      reward_total=None, reward_terms=None, flags=None) -> np.ndarray:
    """One LogRecord per env of a tick: state (n, 18), gait (n, 7), device solutions
    (SOLUTION_DTYPE; v_mpc and F*[0] as the logged contact forces)."""
    st = np.asarray(states, np.float64).reshape(-1, 18)
    n = st.shape[0]
    r = np.zeros(n, LOG_RECORD_DTYPE)
    r["time"] = time
    r["q"], r["qd"] = st[:, :9], st[:, 9:]
    r["phase"] = np.asarray(gaits, np.float64).reshape(-1, 7)[:, 0]
    r["v_mpc"] = solutions["v_mpc"]
    r["f_contact"] = solutions["f0"]
    if tau_mpc is not None:
        r["tau_mpc"] = tau_mpc
    if tau_res is not None:
        r["tau_res"] = tau_res
    if reward_total is not None:
        r["reward_total"] = reward_total
    if reward_terms is not None:
        r["reward_terms"] = reward_terms
    if flags is not None:
        r["flags"] = flags
    return r


class TrajLogWriter:
    """TrajLogWriter (trajlog.cpp:13-37): header at open, append(records), close()."""

    def __init__(self, path: str):
        self._f = open(path, "wb")
        self._f.write(MAGIC)
        self._f.write(np.array([VERSION, LOG_RECORD_DTYPE.itemsize], np.uint32).tobytes())

    def append(self, records: np.ndarray):
        if self._f is None:
            raise ValueError("TrajLogWriter: writer is closed")
        self._f.write(np.ascontiguousarray(records, LOG_RECORD_DTYPE).tobytes())

    def close(self):
        if self._f is not None:
            self._f.close()
            self._f = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def read_traj_log(path: str) -> np.ndarray:
    """read_traj_log (trajlog.cpp:39-55): validates magic, version and record size."""
    with open(path, "rb") as f:
        if f.read(8) != MAGIC:
            raise ValueError(f"read_traj_log: bad magic in {path}")
        version, size = np.frombuffer(f.read(8), np.uint32)
        if version != VERSION or size != LOG_RECORD_DTYPE.itemsize:
            raise ValueError("read_traj_log: unsupported version or record size")
        return np.frombuffer(f.read(), LOG_RECORD_DTYPE).copy()


def export_traj_csv(csv_path: str, records: np.ndarray):
    """export_traj_csv (trajlog.cpp:57-95): the reference's header and %.12g values."""
    cols = (["time"] + [f"q{i}" for i in range(9)] + [f"qd{i}" for i in range(9)] +
            [f"tau_mpc{i}" for i in range(6)] + [f"tau_res{i}" for i in range(6)] +
            [f"f{i}" for i in range(8)] + ["phase", "v_mpc", "reward_total"] +
            [f"r_{t}" for t in REWARD_TERMS] + ["flags"])
    with open(csv_path, "w") as f:
        f.write(",".join(cols) + "\n")
        for r in records:
            vals = ([r["time"]] + list(r["q"]) + list(r["qd"]) + list(r["tau_mpc"]) + list(r["tau_res"]) +
                    list(r["f_contact"]) + [r["phase"], r["v_mpc"], r["reward_total"]] + list(r["reward_terms"]))
            f.write(",".join(f"{float(v):.12g}" for v in vals) + f",{int(r['flags'])}\n")
