"""BASELINE.json's configs C1-C4 on one B200 beside the reference on the host cores: device time
per tick (CUDA events, records + z*), end to end through rmpc_solve with pinned host buffers,
the FP32 roofline fraction on FLOP_alg, and the reference's own BatchRunner::solve (oracle/_ref,
all host threads, a bounded sample of the same workload).  Writes JSON to stdout.

python tools/configs.py > profiles/r02_configs.json   (on a B200)
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2510_12717_b200 as R  # noqa: E402
from paper_2510_12717_b200.abi import SOLUTION_DTYPE  # noqa: E402
from paper_2510_12717_b200.runtime import fma_peak_tflops  # noqa: E402


def flop_alg(kind, T):
    d = json.load(open(os.path.join(ROOT, "profiles", "flops_per_solve.json")))["configs"]
    return d.get(f"{kind}_T{T}", d.get(f"random_T{T}", {})).get("mean")


def gpu(n, T, kind, reps=20):
    m, s = R.default_model(), R.default_settings(T)
    st, cm, ga = R.synthetic_batch(n, kind, seed=0, model=m, settings=s)
    br = R.BatchRunner(n, m, s)
    dev = torch.device("cuda:0")
    d = [torch.from_numpy(x).to(dev) for x in (st, cm, ga)]
    out = torch.zeros(n * SOLUTION_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    z = torch.zeros(n * T * 26, dtype=torch.float32, device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    for _ in range(3):
        br.solve_device(*d, out, z_out=z)
    ms = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        br.solve_device(*d, out, z_out=z)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
    h = [pin(x) for x in (st, cm, ga)]
    ho = torch.zeros(n * SOLUTION_DTYPE.itemsize, dtype=torch.uint8).pin_memory().numpy().view(SOLUTION_DTYPE)
    hz = torch.zeros((n, T, 26), dtype=torch.float32).pin_memory().numpy()
    for _ in range(3):
        br.solve(*h, out=ho, z_out=hz)
    t0 = time.perf_counter()
    for _ in range(reps):
        br.solve(*h, out=ho, z_out=hz)
    e2e = (time.perf_counter() - t0) * 1e3 / reps
    br.close()
    return float(np.median(ms)), e2e, int((ho["status"] == 0).sum())


def cpu_ref(n, T, kind, budget_s=8.0):
    from oracle import ref as F
    m, s = R.default_model(), R.default_settings(T)
    st, cm, ga = R.synthetic_batch(n, kind, seed=0, model=m, settings=s, nominal=F.nominal_pose(m))
    cores = os.cpu_count() or 1
    F.solve_batch(m, s, st[:64], cm[:64], ga[:64], workers=cores, want_z=False)
    done, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < budget_s or done == 0:
        F.solve_batch(m, s, st, cm, ga, workers=cores, want_z=False)
        done += n
        if n >= 4096:
            break
    return done / (time.perf_counter() - t0), cores


def main():
    peak = fma_peak_tflops(0)
    rows = []
    for name, n, T, kind in (("C1", 1, 10, "standing"), ("C2", 4096, 10, "random"), ("C3", 16384, 10, "random"),
                             ("C4", 8192, 5, "random"), ("C4", 8192, 10, "random"), ("C4", 8192, 20, "random")):
        ms, e2e, ok = gpu(n, T, kind)
        fl = flop_alg(kind, T)
        cpu, cores = cpu_ref(n, T, kind)
        rows.append({"config": name, "agents": n, "horizon": T, "kind": kind, "status_ok": ok,
                     "gpu_ms_per_tick_p50": ms, "gpu_solves_per_s": n / ms * 1e3,
                     "e2e_ms_per_tick": e2e, "e2e_solves_per_s": n / e2e * 1e3,
                     "roofline_frac_flop_alg": fl * n / (ms * 1e-3) / 1e12 / peak if fl else None,
                     "reference_cpu_solves_per_s": cpu, "reference_cpu_threads": cores,
                     "e2e_speedup_vs_reference": (n / e2e * 1e3) / cpu})
        print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
    print(json.dumps({"fp32_peak_tflops_measured": peak, "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
