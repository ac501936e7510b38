"""A/B timing of solver builds on one box (run on a B200 via gpurun): median device time per
solve_device call (CUDA events) for a list of (horizon, agents) cases.  Select the library
with RMPC_B200_LIB, e.g.

    for L in lib_A.so lib_B.so; do RMPC_B200_LIB=$PWD/$L python tools/time_lib.py 10:16384 5:8192; done

Two builds timed back to back in one call differ reproducibly at the ~0.1% level; box-to-box
spread is ~1-2%.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_12717_b200 as R  # noqa: E402
from paper_2510_12717_b200.abi import SOLUTION_DTYPE  # noqa: E402


def main():
    cases = [tuple(int(v) for v in a.split(":")) for a in sys.argv[1:]] or [(10, 16384), (10, 4096), (5, 8192)]
    res = {}
    for T, n in cases:
        m, s = R.default_model(), R.default_settings(T)
        st, cm, ga = R.synthetic_batch(n, "random", seed=0, model=m, settings=s)
        br = R.BatchRunner(n, m, s)
        d = [torch.from_numpy(a).cuda() for a in (st, cm, ga)]
        out = torch.zeros(n * SOLUTION_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
        cs = torch.cuda.current_stream()
        for _ in range(3):
            br.solve_device(*d, out, stream=cs)
        ts = []
        for _ in range(15):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            br.solve_device(*d, out, stream=cs)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        res[f"T{T}/n{n}"] = round(float(np.median(ts)), 4)
    print(os.path.basename(os.environ.get("RMPC_B200_LIB", "in-tree")), res)


if __name__ == "__main__":
    main()
