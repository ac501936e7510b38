"""Regenerates the golden fixtures of tests/test_golden.py from the FP64 oracle (oracle/).

The reference cannot be built here (no Eigen), so these fixtures pin the *restatement*: any
change to the oracle that moves a result shows up as a golden diff that has to be explained
(the oracle itself is pinned to the reference's known-answer tests).

python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import paper_2510_12717_b200 as R  # noqa: E402
from oracle import oracle as O  # noqa: E402

CASES = [("standing", 10, 1, 0), ("mixed", 10, 16, 3), ("random", 5, 8, 7), ("random", 20, 4, 9)]


def case_arrays(kind, T, n, seed):
    m, s = R.default_model(), R.default_settings(T)
    st, cm, ga = R.synthetic_batch(n, kind, seed=seed, model=m, settings=s, nominal=O.nominal_pose(m))
    sol, z, _, _ = O.solve_batch(m, s, st, cm, ga, workers=1)
    return dict(states=st, cmds=cm, gaits=ga, tau_ff=sol["tau_ff"], f0=sol["f0"], q_set=sol["q_set"],
                qd_set=sol["qd_set"], v_mpc=sol["v_mpc"], status=sol["status"], z=z)


def main():
    for kind, T, n, seed in CASES:
        a = case_arrays(kind, T, n, seed)
        np.savez_compressed(os.path.join(HERE, f"oracle_{kind}_T{T}_n{n}_s{seed}.npz"), **a)
        print("wrote", kind, T, n, seed)


if __name__ == "__main__":
    main()
