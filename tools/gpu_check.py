"""Quick GPU parity + timing probe (development tool; the real gates are tests/ and bench.py).

python tools/gpu_check.py [n_parity] [n_timing]
"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2510_12717_b200 as R  # noqa: E402
from oracle import oracle as O  # noqa: E402


def rel(a, b):
    return np.max(np.abs(a - b), axis=-1) / np.maximum(np.max(np.abs(b), axis=-1), 1e-30)


def parity(kind, T, n, warm=False):
    m, s = R.default_model(), R.default_settings(T)
    st, cm, ga = R.synthetic_batch(n, kind, seed=1, model=m, settings=s)
    br = R.BatchRunner(n, m, s)
    sol, z = br.solve(st, cm, ga, want_z=True)
    ref, zr, _, _ = O.solve_batch(m, s, st, cm, ga, workers=8)
    ok = (sol["status"] == 0) & (ref["status"] == 0)
    et = rel(sol["tau_ff"].astype(np.float64), ref["tau_ff"])[ok]
    ef = rel(sol["f0"].astype(np.float64), ref["f0"])[ok]
    ev = (np.abs(sol["v_mpc"] - ref["v_mpc"]) / np.maximum(np.abs(ref["v_mpc"]), 1e-30))[ok]
    ez = np.max(np.abs(z - zr), axis=(1, 2))[ok]
    print(f"{kind:8s} T={T:2d} n={n:5d} status gpu {np.bincount(sol['status'], minlength=4)} "
          f"ref {np.bincount(ref['status'], minlength=4)} | max rel tau {et.max():.2e} F0 {ef.max():.2e} "
          f"V {ev.max():.2e} | max|dz*| {ez.max():.2e} | prim {np.max(np.abs(sol['prim_res'] - ref['prim_res'])):.2e}")
    if warm:
        s2 = R.default_settings(T)
        s2.warm_start = 1
        br2 = R.BatchRunner(n, m, s2)
        sol2, z2 = br2.solve(st, cm, ga, prev=(sol, z), want_z=True)
        okp = np.where(sol["status"] == 0, 0, 1).astype(np.int32)
        ref2, _, _, _ = O.solve_batch(m, s2, st, cm, ga, prev_z=z.astype(np.float64), prev_ok=okp,
                                      workers=8)
        ok = (sol2["status"] == 0) & (ref2["status"] == 0)
        et = rel(sol2["tau_ff"].astype(np.float64), ref2["tau_ff"])[ok]
        ev = (np.abs(sol2["v_mpc"] - ref2["v_mpc"]) / np.maximum(np.abs(ref2["v_mpc"]), 1e-30))[ok]
        print(f"   warm-start tick: max rel tau {et.max():.2e} V {ev.max():.2e} status {np.bincount(sol2['status'], minlength=4)}")


def timing(T, n, reps=20):
    import torch
    m, s = R.default_model(), R.default_settings(T)
    st, cm, ga = R.synthetic_batch(n, "random", seed=0, model=m, settings=s)
    br = R.BatchRunner(n, m, s)
    dev = torch.device("cuda:0")
    dst = torch.from_numpy(st).to(dev)
    dcm = torch.from_numpy(cm).to(dev)
    dga = torch.from_numpy(ga).to(dev)
    dout = torch.zeros(n * R.SOLUTION_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    for _ in range(3):
        br.solve_device(dst, dcm, dga, dout, stream=stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        br.solve_device(dst, dcm, dga, dout, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    sol, _ = br.solve(st, cm, ga)
    t = br.last_timing()
    br.set_stage_profiling(True)
    br.solve(st, cm, ga)
    tp = br.last_timing()
    print(f"T={T} n={n}: device {ms:.3f} ms/tick -> {n / ms * 1e3 / 1e6:.3f} M solves/s | host-API "
          f"total {t['total_ms']:.3f} (h2d {t['h2d_ms']:.3f} kern {t['kernel_ms']:.3f} d2h {t['d2h_ms']:.3f}) "
          f"| status {np.bincount(sol['status'], minlength=4)}")
    print("   stage split:", {k: round(v, 3) for k, v in tp["stage_ms"].items()})


if __name__ == "__main__":
    n_par = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    n_tim = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
    parity("standing", 10, 1)
    parity("random", 10, n_par, warm=True)
    parity("mixed", 10, n_par)
    parity("random", 5, n_par // 2)
    parity("random", 20, n_par // 4)
    for T in (10, 5, 20):
        timing(T, n_tim if T == 10 else 8192)
