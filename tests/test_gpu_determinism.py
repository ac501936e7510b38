"""Race evidence without compute-sanitizer (closed on this GPU pool): the squad
solve's bytes do not depend on which squad slot of a CTA serves a squad, nor on whether the
CTA's other slot is busy (RMPC_SQUAD_SOLO=1 / 2 run one squad per CTA in slot 0 / slot 1), nor on
the output path (device buffers, mapped host buffers, split launch with copy-out).  Needs a B200."""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2510_12717_b200 as R

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, %r)
import paper_2510_12717_b200 as R
m, s = R.default_model(), R.default_settings(%d)
st, cm, ga = R.synthetic_batch(%d, "mixed", seed=9, model=m, settings=s)
sol, z = R.BatchRunner(len(st), m, s).solve(st, cm, ga, want_z=True)
sys.stdout.buffer.write(sol.tobytes() + z.tobytes())
"""


def run(T, n, solo):
    env = dict(os.environ)
    env.pop("RMPC_SQUAD_SOLO", None)
    if solo:
        env["RMPC_SQUAD_SOLO"] = str(solo)
    r = subprocess.run([sys.executable, "-c", SCRIPT % (ROOT, T, n)], env=env, capture_output=True, timeout=600)
    assert r.returncode == 0, r.stderr.decode()[-2000:]
    return r.stdout


@pytest.mark.parametrize("T,n", [(10, 5000), (3, 1500), (7, 700)])
def test_squad_slot_independence(T, n):
    base = run(T, n, 0)
    assert len(base) > 0
    assert run(T, n, 1) == base
    assert run(T, n, 2) == base


def test_output_paths_agree():
    """Host solve (split launch: first wave copied out beside the second, which writes the mapped
    buffers) == device solve, at C3 where the squads span two waves."""
    import torch
    from paper_2510_12717_b200.abi import SOLUTION_DTYPE
    n, T = 16384, 10
    m, s = R.default_model(), R.default_settings(T)
    st, cm, ga = R.synthetic_batch(n, "random", seed=21, model=m, settings=s)
    br = R.BatchRunner(n, m, s)
    host, zh = br.solve(st, cm, ga, want_z=True)
    rec_only, _ = br.solve(st, cm, ga)
    dev = torch.device("cuda:0")
    d = [torch.from_numpy(x).to(dev) for x in (st, cm, ga)]
    out = torch.zeros(n * SOLUTION_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    z = torch.zeros(n * T * 26, dtype=torch.float32, device=dev)
    br.solve_device(*d, out, z_out=z)
    torch.cuda.synchronize()
    assert (host["status"] == 0).all()
    assert out.cpu().numpy().tobytes() == host.tobytes() == rec_only.tobytes()
    assert z.cpu().numpy().tobytes() == zh.tobytes()
    pinned = torch.zeros((n, T, 26), dtype=torch.float32).pin_memory().numpy()
    po = torch.zeros(n * SOLUTION_DTYPE.itemsize, dtype=torch.uint8).pin_memory().numpy().view(SOLUTION_DTYPE)
    br.solve(st, cm, ga, out=po, z_out=pinned)
    assert po.tobytes() == host.tobytes() and pinned.tobytes() == zh.tobytes()
    assert np.isfinite(zh).all()


def test_many_shards_on_one_device():
    """A handle over eight shards of one GPU (eight persistent host workers, eight streams and
    schedule workspaces) gives the one-shard bytes at C3: the split changes nothing."""
    n, T = 16384, 10
    m, s = R.default_model(), R.default_settings(T)
    st, cm, ga = R.synthetic_batch(n, "mixed", seed=4, model=m, settings=s)
    one = R.BatchRunner(n, m, s).solve(st, cm, ga, want_z=True)
    br = R.BatchRunner(n, m, s, devices=[0] * 8)
    assert br.workers() == 8
    ranges = [br.shard_info(g)[1:] for g in range(8)]
    from paper_2510_12717_b200.sharding import shard_range
    assert [(b, b + c) for b, c in ranges] == [shard_range(g, 8, n) for g in range(8)]
    for _ in range(2):
        eight = br.solve(st, cm, ga, want_z=True)
        assert eight[0].tobytes() == one[0].tobytes() and eight[1].tobytes() == one[1].tobytes()


def test_store_build_independent_of_representative_state():
    """The squad pass builds each schedule's store from the nominal state (the cold-start QP
    matrices, Ruiz scales and factor depend on the schedule alone; rmpc_kernel.cu synth_rep), so
    the host path can start it before the states and commands have arrived.  The results equal,
    byte for byte, a store built from each schedule's first agent (RMPC_SYNTH_REP=0)."""
    env = dict(os.environ)
    script = SCRIPT % (ROOT, 10, 5000)
    a = subprocess.run([sys.executable, "-c", script], env={**env, "RMPC_SYNTH_REP": "1"}, capture_output=True,
                       timeout=600)
    b = subprocess.run([sys.executable, "-c", script], env={**env, "RMPC_SYNTH_REP": "0"}, capture_output=True,
                       timeout=600)
    assert a.returncode == 0 and b.returncode == 0, (a.stderr.decode()[-1500:], b.stderr.decode()[-1500:])
    assert len(a.stdout) > 0 and a.stdout == b.stdout


@pytest.mark.parametrize("T", [11, 16, 20])
def test_long_squads_repeatable_and_path_independent(T):
    """Long squads (T = 11..20: four warps per squad, the recurrences handed between warps
    through producer / consumer barriers): repeated solves and the host / device paths give the
    same bytes, and the result is within the parity gates of the per-agent factorization."""
    import torch
    from paper_2510_12717_b200.abi import SOLUTION_DTYPE
    from parity import check, compare
    n = 3000
    m, s = R.default_model(), R.default_settings(T)
    st, cm, ga = R.synthetic_batch(n, "mixed", seed=T, model=m, settings=s)
    br = R.BatchRunner(n, m, s)
    a = br.solve(st, cm, ga, want_z=True)
    b = br.solve(st, cm, ga, want_z=True)
    assert a[0].tobytes() == b[0].tobytes() and a[1].tobytes() == b[1].tobytes()
    dev = torch.device("cuda:0")
    d = [torch.from_numpy(x).to(dev) for x in (st, cm, ga)]
    out = torch.zeros(n * SOLUTION_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    z = torch.zeros(n * T * 26, dtype=torch.float32, device=dev)
    br.solve_device(*d, out, z_out=z)
    torch.cuda.synchronize()
    assert out.cpu().numpy().tobytes() == a[0].tobytes() and z.cpu().numpy().tobytes() == a[1].tobytes()
    br.set_schedule_sharing(0)
    p = br.solve(st, cm, ga, want_z=True)
    c = compare(a[0], p[0], a[1], p[1])
    check(c, f"long squads vs per-agent T={T}")
