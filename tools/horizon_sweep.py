"""C4 horizon sweep (BASELINE.json configs[3]): 8 192 agents at N = 5 / 10 / 12 / 20, device
time per tick with CUDA events (L2 flushed between ticks), solves/s, agents per CTA, and the
FP32 roofline fraction on the per-horizon FLOP_alg of profiles/flops_per_solve.json.

python tools/horizon_sweep.py [agents] > profiles/rNN_horizon_sweep.json   (on a B200)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_12717_b200 as R  # noqa: E402
from paper_2510_12717_b200.abi import SOLUTION_DTYPE  # noqa: E402
from paper_2510_12717_b200.runtime import fma_peak_tflops  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def flop_alg(T):
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "flops_per_solve.json")))["configs"]
        return d[f"random_T{T}"]["mean"]
    except Exception:
        return None


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    dev = torch.device("cuda:0")
    peak = fma_peak_tflops(0)
    L = R.library()
    import ctypes
    L.rmpc_agents_per_cta.argtypes = [ctypes.c_int32]
    rows = []
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    for T in (5, 10, 12, 20):
        m, s = R.default_model(), R.default_settings(T)
        st, cm, ga = R.synthetic_batch(n, "random", seed=0, model=m, settings=s)
        br = R.BatchRunner(n, m, s)
        d_st, d_cm, d_ga = (torch.from_numpy(a).to(dev) for a in (st, cm, ga))
        out = torch.zeros(n * SOLUTION_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        z = torch.zeros(n * T * 26, dtype=torch.float32, device=dev)
        for _ in range(3):
            br.solve_device(d_st, d_cm, d_ga, out, z_out=z, stream=torch.cuda.current_stream())
        ms = []
        for _ in range(20):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            br.solve_device(d_st, d_cm, d_ga, out, z_out=z, stream=torch.cuda.current_stream())
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        t = float(np.median(ms))
        fl = flop_alg(T)
        ach = fl * n / (t * 1e-3) / 1e12 if fl else None
        ok = int((out.cpu().numpy().view(SOLUTION_DTYPE)["status"] == 0).sum())
        rows.append({"horizon": T, "agents": n,
                     "path": "squads (32 agents per warp pair, 2 per SM)" if T <= 10 else
                             ("long squads (32 agents on four warps, 1 per SM)" if T <= 20 else
                              "shared-schedule CTAs (warp pair per agent)"),
                     "ms_per_tick_p50": t, "solves_per_s": n / (t * 1e-3), "status_ok": ok,
                     "flop_alg_per_solve": fl, "achieved_tflops": ach,
                     "roofline_frac": (ach / peak) if ach else None})
        br.close()
    print(json.dumps({"config": "C4: horizon sweep at %d agents, 1 B200, random synthetic batch, "
                                "L2 flushed between ticks, records + z* written" % n, "fp32_peak_tflops_measured": peak,
                      "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
