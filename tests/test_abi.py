"""The C-ABI library loads without a GPU, exports every symbol include/rmpc_b200.h declares,
and its host-side logic (defaults, nominal pose, PD torque, error paths) matches the oracle.
No kernel launches here.  CPU only."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2510_12717_b200 as R
from paper_2510_12717_b200 import abi, runtime

INCLUDE = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include")
HEADERS = [os.path.join(INCLUDE, h) for h in ("rmpc_b200.h", "rmpc_b200_env.h")]


def declared_functions():
    names = set()
    for h in HEADERS:
        src = re.sub(r"/\*.*?\*/", "", open(h).read(), flags=re.S)
        names |= set(re.findall(r"\b(rmpc_[a-z_0-9]+)\s*\(", src))
    return sorted(names)


def test_library_exports_every_declared_symbol():
    L = R.library()
    names = declared_functions()
    assert len(names) >= 27
    for n in names:
        assert hasattr(L, n), n


def test_struct_sizes_match_header():
    L = R.library()
    sizes = [C.sizeof(abi.Model), C.sizeof(abi.Settings), 18 * 8, 3 * 8, 7 * 8,
             abi.SOLUTION_DTYPE.itemsize, C.sizeof(abi.Timing)]
    assert [L.rmpc_sizeof(i) for i in range(7)] == sizes
    assert L.rmpc_sizeof(99) == -1
    from paper_2510_12717_b200.env import EnvConfig, _bind
    _bind(L)
    from paper_2510_12717_b200.ppo import LossInfo, PpoConfig, UpdateStats
    assert [L.rmpc_env_sizeof(i) for i in range(5)] == [C.sizeof(EnvConfig), 16, C.sizeof(PpoConfig),
                                                        C.sizeof(LossInfo), C.sizeof(UpdateStats)]
    assert L.rmpc_env_sizeof(5) == -1


def test_ppo_config_defaults_match_oracle(oracle):
    from paper_2510_12717_b200.ppo import default_ppo_config, rng_state
    c = default_ppo_config()
    assert bytes(c) == bytes(oracle.ppo_config())
    assert (c.gamma, c.lam_gae, c.clip_eps, c.epochs, c.minibatches, c.lr, c.value_coef, c.max_grad_norm) == \
        (0.99, 0.95, 0.2, 4, 4, 3e-4, 0.5, 1.0)
    assert list(rng_state(7, 0x0272)) == list(oracle.rng_words(7, 0x0272))


def test_env_config_defaults_and_terrain_match_oracle(oracle):
    from paper_2510_12717_b200.env import default_env_config
    c = default_env_config()
    assert bytes(c) == bytes(oracle.env_config_default())
    assert (c.control_dt, c.substeps, c.k_n, c.c_n, c.v_slip) == (0.01, 4, 5e4, 500.0, 0.05)


def test_defaults_match_library_defaults():
    L = R.library()
    m, s = abi.Model(), abi.Settings()
    L.rmpc_model_default(C.byref(m))
    L.rmpc_settings_default(C.byref(s), 10)
    assert bytes(m) == bytes(abi.default_model())
    assert bytes(s) == bytes(abi.default_settings(10, 0.05))


def test_nominal_pose_matches_oracle_bitwise(oracle):
    m = abi.default_model()
    assert runtime.nominal_pose(m).tobytes() == oracle.nominal_pose(m).tobytes()


def test_stage_names_and_status_messages():
    L = R.library()
    assert [L.rmpc_stage_name(i).decode() for i in range(7)] == list(abi.STAGE_NAMES)
    assert L.rmpc_stage_name(7) == b"unknown"
    assert b"non-finite" in L.rmpc_status_message(abi.STATUS_NONFINITE_INPUT)
    assert b"sm_100a" in L.rmpc_build_info()


def test_cta_shape_six_agents_per_sm_at_n10():
    """T=10: 6 warp pairs per CTA (TMEM: 3 warps x 160 columns per lane quarter), their shared
    memory within 227 KB; longer horizons keep the node blocks that exceed a warp's TMEM share
    in shared memory; every horizon up to 32 gets at least two agents per CTA."""
    L = R.library()
    L.rmpc_agents_per_cta.argtypes = [C.c_int32]
    assert L.rmpc_agents_per_cta(10) == 6
    assert 6 * L.rmpc_smem_bytes(10) <= 227 * 1024 - 128
    # T = 12: 5 agents (one node block per warp in shared memory); T = 20: 3 (two per warp)
    assert L.rmpc_agents_per_cta(12) == 5 and L.rmpc_agents_per_cta(20) == 3
    assert L.rmpc_agents_per_cta(32) == 2
    for T in range(2, 33):
        A = L.rmpc_agents_per_cta(T)
        assert 1 <= A <= 8 and A * L.rmpc_smem_bytes(T) <= 227 * 1024 - 128
        assert (A == 8) == (T <= 8)  # the dense variant: all node blocks in TMEM at 16 warps
    assert L.rmpc_agents_per_cta(0) == -1 and L.rmpc_agents_per_cta(33) == -1


def test_mpc_torque_matches_oracle_pd(oracle):
    """mpc_torque -> pd_torque (mpc.cpp:340-344, robot.cpp:235-241) on the host."""
    m = abi.default_model()
    br_lib = R.library()
    q = oracle.nominal_pose(m)
    state = np.concatenate([q + 0.01, np.full(9, 0.2)])
    sol = np.zeros(1, dtype=abi.SOLUTION_DTYPE)
    sol["q_set"] = q[3:] + 0.05
    sol["qd_set"] = 0.3
    sol["tau_ff"] = np.array([5.0, -70.0, 2.0, 1.0, 0.0, -40.0])
    tau = np.zeros(6)
    rc = br_lib.rmpc_mpc_torque(C.byref(m), sol.ctypes.data, state.ctypes.data, tau.ctypes.data)
    assert rc == 0
    expect = oracle.pd_torque(m, sol["q_set"][0].astype(np.float64), sol["qd_set"][0].astype(np.float64),
                              state[:9], state[9:], sol["tau_ff"][0].astype(np.float64))
    np.testing.assert_allclose(tau, expect, rtol=0, atol=1e-12)
    sol["status"] = abi.STATUS_DIVERGED
    assert br_lib.rmpc_mpc_torque(C.byref(m), sol.ctypes.data, state.ctypes.data,
                                  tau.ctypes.data) == abi.RMPC_ERR_STRUCTURAL


def test_create_rejects_structural_errors():
    """BatchRunner/MpcController ctor errors (batch.cpp:19, mpc.cpp:243-245) come back as codes."""
    m = abi.default_model()
    for n, T in ((0, 10), (4, 1), (4, 33)):
        s = abi.default_settings(max(T, 1))
        s.horizon = T
        with pytest.raises(R.RmpcError) as e:
            R.BatchRunner(n, m, s)
        assert e.value.code == abi.RMPC_ERR_STRUCTURAL


@pytest.mark.skipif(__import__("conftest").HAS_GPU, reason="CPU-only behaviour")
def test_create_fails_loudly_without_gpu():
    with pytest.raises(R.RmpcError) as e:
        R.BatchRunner(4, abi.default_model(), abi.default_settings(10))
    assert e.value.code == abi.RMPC_ERR_CUDA and "no CUDA device" in str(e.value)


def test_synthetic_rng_matches_cpp_restatement(oracle):
    """The Python xoshiro256++ streams equal the C++ restatement of rng.hpp bit for bit."""
    from paper_2510_12717_b200.synthetic import Xoshiro
    for stream in (0, 1, 7, 4095, 123456):
        x = Xoshiro(0, [stream])
        py = np.array([x.uniform()[0] for _ in range(6)])
        assert py.tobytes() == oracle.rng_uniform(0, stream, 6).tobytes()
    x = Xoshiro(5, np.arange(100))
    a = x.uniform()
    assert a.tobytes() == np.array([oracle.rng_uniform(5, i, 1)[0] for i in range(100)]).tobytes()


def test_synthetic_batch_ranges():
    m, s = abi.default_model(), abi.default_settings(10)
    st, cm, ga = R.synthetic_batch(1000, "random", seed=0, model=m, settings=s)
    assert st.shape == (1000, 18) and cm.shape == (1000, 3) and ga.shape == (1000, 7)
    assert np.all(np.abs(st[:, [9, 11]]) <= 0.5) and np.all(np.abs(cm[:, 1]) <= 0.6)
    assert np.all((ga[:, 0] >= 0) & (ga[:, 0] < 1)) and np.all(ga[:, 2] == 0.5)
    _, _, gm = R.synthetic_batch(1000, "mixed", seed=0, model=m, settings=s)
    assert set(np.unique(gm[:, 2])) == {0.4, 0.5, 0.65, 1.0}
    st1, cm1, ga1 = R.synthetic_batch(3, "standing", model=m, settings=s)
    assert np.all(ga1[:, 2] == 1.0) and np.all(st1[:, 9:] == 0)


def test_soa_layout_matches_header():
    """RMPC_SOA_* rows (include/rmpc_b200.h) = the to_soa layout: the 18 state values, the 3
    command values, the 7 gait values, each row one component of every agent."""
    import re
    hdr = open(os.path.join(INCLUDE, "rmpc_b200.h")).read()
    d = {k: int(v) for k, v in re.findall(r"#define RMPC_SOA_(\w+) (\d+)", hdr)}
    assert d == {"Q": 0, "QD": 9, "HEIGHT": 18, "VX": 19, "WPITCH": 20, "PHASE": 21, "PERIOD": 22,
                 "PHASE_SWITCH": 23, "OFFSETS": 24, "FIELDS": 28}
    assert R.SOA_FIELDS == d["FIELDS"]
    st, cm, ga = R.synthetic_batch(7, "mixed", seed=1)
    soa = R.to_soa(st, cm, ga, ld=9)
    assert soa.shape == (28, 9) and soa.dtype == np.float32 and not soa[:, 7:].any()
    np.testing.assert_array_equal(soa[d["Q"] + 1, :7], st[:, 1].astype(np.float32))
    np.testing.assert_array_equal(soa[d["QD"] + 4, :7], st[:, 9 + 4].astype(np.float32))
    np.testing.assert_array_equal(soa[d["VX"], :7], cm[:, 1].astype(np.float32))
    np.testing.assert_array_equal(soa[d["OFFSETS"] + 3, :7], ga[:, 6].astype(np.float32))
    s2, c2, g2 = R.from_soa(soa, 7)
    np.testing.assert_array_equal(s2, st.astype(np.float32).astype(np.float64))
    np.testing.assert_array_equal(g2, ga.astype(np.float32).astype(np.float64))
    assert s2.flags["C_CONTIGUOUS"] and c2.shape == (7, 3)
