"""Device time per tick of the batched solve for a list of horizons (CUDA events, 10 ticks after
3 warm-up).  python tools/time_solve.py [agents] [T ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_12717_b200 as R  # noqa: E402
from paper_2510_12717_b200.abi import SOLUTION_DTYPE  # noqa: E402


def time_solve(n, T, kind="random", share=True, reps=10):
    m, s = R.default_model(), R.default_settings(T)
    st, cm, ga = R.synthetic_batch(n, kind, seed=0, model=m, settings=s)
    br = R.BatchRunner(n, m, s)
    br.set_schedule_sharing(share)
    dev = torch.device("cuda:0")
    d = [torch.from_numpy(x).to(dev) for x in (st, cm, ga)]
    out = torch.zeros(n * SOLUTION_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    z = torch.zeros(n * T * 26, dtype=torch.float32, device=dev)
    for _ in range(3):
        br.solve_device(*d, out, z_out=z)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        br.solve_device(*d, out, z_out=z)
    e1.record()
    torch.cuda.synchronize()
    br.close()
    return e0.elapsed_time(e1) / reps


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    Ts = [int(a) for a in sys.argv[2:]] or [5, 10, 20]
    tag = os.environ.get("RMPC_SHARED_AGENTS", "default")
    for T in Ts:
        ms = time_solve(n, T)
        print(f"shared_agents={tag} T={T} n={n}: {ms:.3f} ms/tick  {n / ms / 1e3:.2f} M solves/s", flush=True)
