"""The trajectory log keeps the reference's binary format (trajlog.hpp:20-45: 424-byte packed
LogRecord after an 8-byte magic and two uint32) and CSV columns (trajlog.cpp:57-95).  CPU only."""
import numpy as np
import pytest

from paper_2510_12717_b200.abi import SOLUTION_DTYPE
from paper_2510_12717_b200.trajlog import (LOG_RECORD_DTYPE, TrajLogWriter, export_traj_csv, read_traj_log,
                                           records_from_tick)


def test_round_trip_and_header(tmp_path):
    rng = np.random.default_rng(0)
    sol = np.zeros(5, SOLUTION_DTYPE)
    sol["v_mpc"] = rng.uniform(-1, 1, 5)
    sol["f0"] = rng.uniform(0, 100, (5, 8))
    st, ga = rng.uniform(-1, 1, (5, 18)), np.tile([0.25, 0.8, 0.5, 0.5, 0.5, 0, 0], (5, 1))
    recs = records_from_tick(0.01, st, ga, sol, tau_mpc=rng.uniform(-5, 5, (5, 6)), flags=np.arange(5))
    p = tmp_path / "log.bin"
    with TrajLogWriter(str(p)) as w:
        w.append(recs)
        w.append(recs[:2])
    raw = p.read_bytes()
    assert raw[:8] == b"RMPCLG01" and np.frombuffer(raw[8:16], np.uint32).tolist() == [1, 424]
    assert len(raw) == 16 + 7 * 424
    back = read_traj_log(str(p))
    assert back.tobytes() == np.concatenate([recs, recs[:2]]).tobytes()
    np.testing.assert_array_equal(back["q"][:5], st[:, :9])
    np.testing.assert_array_equal(back["phase"][:5], 0.25)
    np.testing.assert_array_equal(back["f_contact"][:5], sol["f0"].astype(np.float64))
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"XXXXXXXX" + raw[8:])
    with pytest.raises(ValueError):
        read_traj_log(str(bad))


def test_csv_columns(tmp_path):
    recs = np.zeros(2, LOG_RECORD_DTYPE)
    recs["time"] = [0.0, 0.01]
    p = tmp_path / "log.csv"
    export_traj_csv(str(p), recs)
    lines = p.read_text().splitlines()
    head = lines[0].split(",")
    assert head[0] == "time" and head[1] == "q0" and head[-1] == "flags" and "r_self_collision" in head
    assert len(head) == 1 + 9 + 9 + 6 + 6 + 8 + 3 + 10 + 1
    assert lines[2].startswith("0.01,")
