"""compute-sanitizer target: one small solve (2 CTAs = 12 agents, N=10) plus the env kernels.

compute-sanitizer --tool racecheck python tools/racecheck.py
"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2510_12717_b200 as R  # noqa: E402


def main():
    m, s = R.default_model(), R.default_settings(10)
    st, cm, ga = R.synthetic_batch(12, "mixed", seed=3, model=m, settings=s)
    sol, z = R.BatchRunner(12, m, s).solve(st, cm, ga, want_z=True)
    print("ok", int((sol["status"] == 0).sum()), float(np.abs(z).max()))


if __name__ == "__main__":
    main()
