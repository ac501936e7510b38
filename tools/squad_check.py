"""Squad (lane-per-agent, schedule-shared) solve vs the per-agent and warp-pair shared solves and
the FP64 oracle: parity metrics and timing.  python tools/squad_check.py [--quick]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2510_12717_b200 as R  # noqa: E402
from paper_2510_12717_b200.abi import SOLUTION_DTYPE  # noqa: E402
from parity import compare, summary  # noqa: E402
from oracle import oracle as O  # noqa: E402

quick = "--quick" in sys.argv
m = R.default_model()
cases = [(10, "random", 1024), (10, "mixed", 1024), (2, "mixed", 256), (3, "random", 256), (5, "random", 512),
         (7, "mixed", 300), (10, "standing", 64)]
for T, kind, n in cases[:3] if quick else cases:
    s = R.default_settings(T)
    st, cm, ga = R.synthetic_batch(n, kind, seed=T, model=m, settings=s)
    st = st.copy()
    if n > 8:
        st[5, 3] = np.nan
    br = R.BatchRunner(n, m, s)
    res = {}
    for lvl in (3, 1, 0):
        br.set_schedule_sharing(lvl)
        res[lvl] = br.solve(st, cm, ga, want_z=True)
    ref, zr, _, _ = O.solve_batch(m, s, st, cm, ga, workers=16)
    a, za = res[3]
    print(f"T={T} {kind} n={n} status counts {np.bincount(a['status'], minlength=4)}", flush=True)
    print("  squad vs per-agent:", summary(compare(a, res[0][0], za, res[0][1])), flush=True)
    print("  squad vs oracle:   ", summary(compare(a, ref, za, zr)), flush=True)
    print("  per-agent vs oracle:", summary(compare(res[0][0], ref, res[0][1], zr)), flush=True)
    print("  pair == per-agent bytes:", res[1][0].tobytes() == res[0][0].tobytes(), flush=True)
    br.close()

dev = torch.device("cuda:0")
for T, n in ((10, 16384),) if quick else ((10, 16384), (10, 4096), (5, 8192), (3, 8192), (10, 65536)):
    s = R.default_settings(T)
    st, cm, ga = R.synthetic_batch(n, "random", seed=0, model=m, settings=s)
    br = R.BatchRunner(n, m, s)
    d = [torch.from_numpy(x).to(dev) for x in (st, cm, ga)]
    out = torch.zeros(n * SOLUTION_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    z = torch.zeros(n * T * 26, dtype=torch.float32, device=dev)
    for lvl in (3, 1):
        br.set_schedule_sharing(lvl)
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
        print(f"T={T} n={n} level={lvl}: {ms:.3f} ms/tick -> {n / ms / 1e3:.2f} M solves/s | stages",
              {k: round(v, 3) for k, v in tm["stage_ms"].items()}, "| per-agent means (us)",
              {k: round(v * 1e3, 1) for k, v in tm["stage_mean_ms"].items() if v > 0}, flush=True)
    br.close()
