"""N > 1 path on CPU: world_size-2 gloo ranks each take their contiguous agent shard from the
product library's own planner (rmpc_shard_range, loaded without a GPU) and solve it (the CPU
oracle stands in for the device here) with no collective on the data path; the gathered shards
equal a single-process solve bit for bit, and the timing reduction is max-over-ranks.  The
device side of the same split runs in the GPU suite (test_many_shards_on_one_device)."""
import ctypes as C
import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_12717_b200.sharding import max_over_ranks, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_total, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2510_12717_b200 as R
    from oracle import oracle as O
    m, s = R.default_model(), R.default_settings(10)
    st, cm, ga = R.synthetic_batch(n_total, "mixed", seed=0, model=m, settings=s, nominal=O.nominal_pose(m))
    lo, hi = shard_range(rank, world, n_total)  # the library's planner, as bench.py's ranks use it
    b, c = C.c_int32(), C.c_int32()
    assert R.library().rmpc_shard_range(n_total, world, rank, C.byref(b), C.byref(c)) == 0
    assert (b.value, b.value + c.value) == (lo, hi)
    sol, z, _, wall = O.solve_batch(m, s, st[lo:hi], cm[lo:hi], ga[lo:hi], workers=1)
    t = max_over_ranks([wall, float(rank)], dist=dist)
    np.save(os.path.join(out_dir, f"sol{rank}.npy"), sol)
    np.save(os.path.join(out_dir, f"z{rank}.npy"), z)
    np.save(os.path.join(out_dir, f"t{rank}.npy"), np.array(t + [wall]))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_ranges_partition():
    import paper_2510_12717_b200 as R
    L = R.library()
    b = C.c_int32()
    assert L.rmpc_shard_range(10, 0, 0, C.byref(b), None) != 0 and L.rmpc_shard_range(10, 2, 2, None, None) != 0
    for n in (0, 1, 7, 4096, 16384, 65536):
        for w in (1, 2, 3, 4, 8):
            rs = [shard_range(r, w, n) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))
            assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1
            assert rs == [(r * n // w, (r + 1) * n // w) for r in range(w)]


def test_two_rank_gloo_shards_equal_single_process(tmp_path):
    n, world = 24, 2
    mp.spawn(_worker, args=(world, _free_port(), n, str(tmp_path)), nprocs=world, join=True)
    import paper_2510_12717_b200 as R
    from oracle import oracle as O
    m, s = R.default_model(), R.default_settings(10)
    st, cm, ga = R.synthetic_batch(n, "mixed", seed=0, model=m, settings=s, nominal=O.nominal_pose(m))
    ref, zr, _, _ = O.solve_batch(m, s, st, cm, ga, workers=1)
    sol = np.concatenate([np.load(tmp_path / f"sol{r}.npy") for r in range(world)])
    z = np.concatenate([np.load(tmp_path / f"z{r}.npy") for r in range(world)])
    assert sol.tobytes() == ref.tobytes() and z.tobytes() == zr.tobytes()
    t0, t1 = np.load(tmp_path / "t0.npy"), np.load(tmp_path / "t1.npy")
    assert t0[0] == t1[0] == max(t0[2], t1[2])  # max over ranks of the wall times
    assert t0[1] == t1[1] == 1.0
