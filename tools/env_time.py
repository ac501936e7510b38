"""Device time of the closed-loop kernels for n agents: physics_step (env.cpp:38-68), the fused
control step (mpc_torque + blend + physics), observe.   python tools/env_time.py [n]  (B200)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_12717_b200 as R  # noqa: E402
from paper_2510_12717_b200.abi import SOLUTION_DTYPE  # noqa: E402
from paper_2510_12717_b200.env import Env, default_env_config  # noqa: E402


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
m, s = R.default_model(), R.default_settings(10)
st, cm, ga = R.synthetic_batch(n, "mixed", seed=0, model=m, settings=s)
env = Env(m, default_env_config(terrain_kind=1))
d_st, d_cm, d_ga = (torch.from_numpy(a).cuda() for a in (st, cm, ga))
tau = torch.zeros((n, 6), dtype=torch.float64, device="cuda")
br = R.BatchRunner(n, m, s)
sol = torch.zeros(n * SOLUTION_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
br.solve_device(d_st, d_cm, d_ga, sol)
obs = torch.zeros((n, 23), dtype=torch.float64, device="cuda")
st0, ga0 = d_st.clone(), d_ga.clone()


def phys():
    d_st.copy_(st0)
    d_ga.copy_(ga0)
    env.physics_step(d_st, d_ga, tau)


def ctrl():
    d_st.copy_(st0)
    d_ga.copy_(ga0)
    env.control_step(sol, d_st, d_ga)


print(f"n={n}: physics_step {timed(phys):.4f} ms, control_step {timed(ctrl):.4f} ms, "
      f"observe {timed(lambda: env.observe(d_st, d_ga, sol, obs)):.4f} ms (state copies included in the first two)")
