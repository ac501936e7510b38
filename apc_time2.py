import sys, os
sys.path.insert(0, ".")
import torch, numpy as np
import paper_2510_12717_b200 as R
from paper_2510_12717_b200.abi import SOLUTION_DTYPE
res = {}
for T in (2, 3, 4, 5, 6, 7, 8):
    n = 16384
    m, s = R.default_model(), R.default_settings(T)
    st, cm, ga = R.synthetic_batch(n, "random", seed=0, model=m, settings=s)
    br = R.BatchRunner(n, m, s)
    d = [torch.from_numpy(a).cuda() for a in (st, cm, ga)]
    out = torch.zeros(n * SOLUTION_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
    cs = torch.cuda.current_stream()
    for _ in range(3): br.solve_device(*d, out, stream=cs)
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); br.solve_device(*d, out, stream=cs); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    res[T] = round(float(np.median(ts)), 3)
print(os.environ.get("RMPC_B200_LIB", "").split("/")[-1], res)
