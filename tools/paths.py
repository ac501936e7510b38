"""Device time per tick of every solve path at C3 (16 384 agents, N = 10) and beside it:
per-agent factorization (sharing off), shared-schedule warp-pair CTAs (level 1), squads (level 2,
the default), and the warm-started per-agent path.  python tools/paths.py  (on a B200)"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_12717_b200 as R  # noqa: E402
from time_solve import time_solve  # noqa: E402
from paper_2510_12717_b200.abi import SOLUTION_DTYPE  # noqa: E402


def warm(n, T, reps=10):
    m, s = R.default_model(), R.default_settings(T)
    st, cm, ga = R.synthetic_batch(n, "random", seed=0, model=m, settings=s)
    prev = R.BatchRunner(n, m, s).solve(st, cm, ga, want_z=True)
    s.warm_start = 1
    br = R.BatchRunner(n, m, s)
    dev = torch.device("cuda:0")
    d = [torch.from_numpy(x).to(dev) for x in (st, cm, ga)]
    pv = torch.from_numpy(prev[0].view(dtype="uint8")).to(dev)
    pz = torch.from_numpy(prev[1]).to(dev)
    out = torch.zeros(n * SOLUTION_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    z = torch.zeros(n * T * 26, dtype=torch.float32, device=dev)
    for _ in range(3):
        br.solve_device(*d, out, z_out=z, prev=pv, prev_z=pz)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        br.solve_device(*d, out, z_out=z, prev=pv, prev_z=pz)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


rows = []
for n, T, kind in ((16384, 10, "random"), (16384, 10, "mixed"), (65536, 10, "random"), (8192, 5, "random")):
    for share in (0, 1, 2):
        ms = time_solve(n, T, kind=kind, share=share)
        rows.append({"agents": n, "horizon": T, "kind": kind, "path": ["per-agent", "shared warp pairs", "squads"][share],
                     "ms_per_tick": ms, "solves_per_s": n / ms * 1e3})
        print(json.dumps(rows[-1]), flush=True)
ms = warm(16384, 10)
rows.append({"agents": 16384, "horizon": 10, "kind": "random", "path": "warm start (per-agent)", "ms_per_tick": ms,
             "solves_per_s": 16384 / ms * 1e3})
print(json.dumps(rows[-1]), flush=True)
