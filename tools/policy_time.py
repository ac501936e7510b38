"""Device time of rmpc_policy_forward_device (policy_forward, policy.cpp:85-102) for n agents.
python tools/policy_time.py [n]   (on a B200)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_12717_b200.env import Policy  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
obs, act, hidden = 23, 6, 64
rng = np.random.default_rng(0)
n_par = sum(i * o + o for out in (act, 1) for i, o in zip((obs, hidden, hidden, hidden), (hidden, hidden, hidden, out)))
pol = Policy(np.concatenate([rng.uniform(-0.2, 0.2, n_par), np.full(act, np.log(0.5))]), obs, act, hidden)
o = torch.randn(n, obs, dtype=torch.float64, device="cuda")
mean = torch.empty(n, act, dtype=torch.float64, device="cuda")
val = torch.empty(n, dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream()
for _ in range(3):
    pol.forward(o, mean, val, stream=s)
ts = []
for _ in range(20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    pol.forward(o, mean, val, stream=s)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = float(np.median(ts))
fl = 2 * n_par * n
print(f"policy forward n={n}: {ms:.4f} ms, {fl / (ms * 1e-3) / 1e12:.2f} TFLOP/s FP64")
