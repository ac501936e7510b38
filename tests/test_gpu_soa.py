"""The structure-of-arrays boundary (rmpc_solve_soa / rmpc_solve_soa_device, the north star's SoA
layout): FP32 component rows in, the same records out as rmpc_solve on the FP64 records that
hold the widened values -- bit for bit, on every solve path.  Needs a B200."""
import numpy as np
import pytest
import torch

import paper_2510_12717_b200 as R
from paper_2510_12717_b200.abi import SOLUTION_DTYPE, STATUS_NONFINITE_INPUT, default_model, default_settings

pytestmark = pytest.mark.gpu


def batch(n, kind, T, seed=2):
    m, s = default_model(), default_settings(T)
    st, cm, ga = R.synthetic_batch(n, kind, seed=seed, model=m, settings=s)
    return m, s, R.to_soa(st, cm, ga, ld=n + 5)


@pytest.mark.parametrize("T,kind,n,share", [(10, "random", 4096, 2), (10, "mixed", 1000, 3), (10, "mixed", 300, 1),
                                            (10, "random", 300, 0), (5, "random", 2000, 3), (20, "mixed", 256, 3),
                                            (10, "random", 700, 2)])
def test_soa_equals_aos_records(T, kind, n, share):
    m, s, soa = batch(n, kind, T)
    br = R.BatchRunner(n, m, s)
    br.set_schedule_sharing(share)
    a, za = br.solve_soa(soa, want_z=True)
    b, zb = br.solve(*R.from_soa(soa, n), want_z=True)
    assert (a["status"] == 0).all()
    assert a.tobytes() == b.tobytes() and za.tobytes() == zb.tobytes()
    t = br.last_timing()
    assert t["batch_size"] == n and t["kernel_ms"] > 0


def test_soa_warm_start_chunked_and_pinned():
    """Warm start runs the chunked per-agent path (the records are unpacked ahead of chunk 0);
    a pinned SoA block is copied without staging.  12 000 agents: three chunks on one B200."""
    n, T = 12000, 10
    m, s, soa = batch(n, "random", T, seed=7)
    cold = R.BatchRunner(n, m, s)
    prev = cold.solve_soa(soa, want_z=True)
    s.warm_start = 1
    br = R.BatchRunner(n, m, s)
    pinned = torch.from_numpy(soa).pin_memory().numpy()
    a, za = br.solve_soa(pinned, prev=prev, want_z=True)
    b, zb = br.solve(*R.from_soa(soa, n), prev=prev, want_z=True)
    assert a.tobytes() == b.tobytes() and za.tobytes() == zb.tobytes()


def test_soa_two_shards_on_one_device():
    n = 3001
    m, s, soa = batch(n, "mixed", 10, seed=3)
    one = R.BatchRunner(n, m, s).solve_soa(soa, want_z=True)
    two = R.BatchRunner(n, m, s, devices=[0, 0]).solve_soa(soa, want_z=True)
    assert one[0].tobytes() == two[0].tobytes() and one[1].tobytes() == two[1].tobytes()


def test_soa_device_path_matches_host_path():
    n, T = 2048, 10
    m, s, soa = batch(n, "random", T, seed=5)
    soa[3, 17] = np.nan  # a non-finite input fails alone, as in the AoS path
    br = R.BatchRunner(n, m, s)
    host, zh = br.solve_soa(soa, want_z=True)
    assert host["status"][17] == STATUS_NONFINITE_INPUT and (np.delete(host["status"], 17) == 0).all()
    dev = torch.device("cuda:0")
    d_soa = torch.from_numpy(soa).to(dev)
    out = torch.zeros(n * SOLUTION_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    z = torch.zeros(n * T * 26, dtype=torch.float32, device=dev)
    br.solve_soa_device(d_soa, out, z_out=z)
    torch.cuda.synchronize()
    assert out.cpu().numpy().tobytes() == host.tobytes()
    assert z.cpu().numpy().tobytes() == zh.tobytes()


def test_soa_argument_errors():
    n = 16
    m, s, soa = batch(n, "random", 10)
    br = R.BatchRunner(n, m, s)
    with pytest.raises(ValueError):
        br.solve_soa(soa[:, :n - 1].copy())
    with pytest.raises(ValueError):
        br.solve_soa(soa.astype(np.float64))
    L = R.library()
    out = np.zeros(n, dtype=SOLUTION_DTYPE)
    assert L.rmpc_solve_soa(br._h, soa.ctypes.data, n - 1, None, None, out.ctypes.data, None) == 1
    assert b"ld < n_envs" in L.rmpc_last_error(br._h)
    assert L.rmpc_solve_soa(br._h, None, n, None, None, out.ctypes.data, None) == 1
