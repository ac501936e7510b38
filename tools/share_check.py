"""Schedule-shared factorization: bit-identity against the per-agent factorization and timing.
python tools/share_check.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_12717_b200 as R  # noqa: E402
from paper_2510_12717_b200.abi import SOLUTION_DTYPE  # noqa: E402

m = R.default_model()
for T, kind, n in ((10, "random", 4096), (10, "mixed", 4096), (5, "random", 2048), (20, "mixed", 1024),
                   (3, "mixed", 512), (12, "random", 1000), (32, "mixed", 64)):
    s = R.default_settings(T)
    st, cm, ga = R.synthetic_batch(n, kind, seed=T, model=m, settings=s)
    st = st.copy()
    st[5, 3] = np.nan
    br = R.BatchRunner(n, m, s)
    a, za = br.solve(st, cm, ga, want_z=True)
    br.set_schedule_sharing(False)
    b, zb = br.solve(st, cm, ga, want_z=True)
    print(T, kind, n, "shared == per-agent:", a.tobytes() == b.tobytes() and za.tobytes() == zb.tobytes(),
          "status", np.bincount(a["status"], minlength=4), flush=True)
    br.close()

dev = torch.device("cuda:0")
for T, n in ((10, 16384), (10, 4096), (5, 8192), (20, 8192), (12, 8192)):
    s = R.default_settings(T)
    st, cm, ga = R.synthetic_batch(n, "random", seed=0, model=m, settings=s)
    br = R.BatchRunner(n, m, s)
    d = [torch.from_numpy(x).to(dev) for x in (st, cm, ga)]
    out = torch.zeros(n * SOLUTION_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    z = torch.zeros(n * T * 26, dtype=torch.float32, device=dev)
    for share in (True, False):
        br.set_schedule_sharing(share)
        for _ in range(3):
            br.solve_device(*d, out, z_out=z)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            br.solve_device(*d, out, z_out=z)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        br.set_stage_profiling(True)
        br.solve(st, cm, ga)
        tm = br.last_timing()
        br.set_stage_profiling(False)
        print(f"T={T} n={n} share={share}: {ms:.3f} ms/tick -> {n / ms / 1e3:.2f} M solves/s | stages",
              {k: round(v, 3) for k, v in tm["stage_ms"].items()}, flush=True)
    br.close()
