"""Algorithmic FLOPs per agent-solve of the reference algorithm, counted
exactly by the Counted<double> instantiation of the CPU oracle over a sample of each bench
workload.  Writes profiles/flops_per_solve.json (read by bench.py for roofline.achieved).

python tools/count_flops.py [sample]
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_12717_b200 as R  # noqa: E402
from oracle import oracle as O  # noqa: E402

STAGES = ("init_guess", "param", "kkt_build", "ruiz", "factorize", "admm_iters", "rnea")


def count(kind, T, sample):
    m, s = R.default_model(), R.default_settings(T)
    st, cm, ga = R.synthetic_batch(sample, kind, seed=0, model=m, settings=s,
                                   nominal=O.nominal_pose(m))
    tot = np.zeros(7)
    per = []
    for i in range(sample):
        by, _ = O.flops(m, s, st[i], cm[i], ga[i])
        tot += by
        per.append(by.sum())
    return dict(mean=float(np.mean(per)), min=float(np.min(per)), max=float(np.max(per)),
                by_stage=dict(zip(STAGES, (tot / sample).tolist())), sample=sample)


def main():
    sample = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    out = {"note": "FP64 reference algorithm (KKT + sparse LDL^T with min-degree ordering, 25 ADMM "
                   "iterations), add/mul/div/sqrt/trig counted once each, per agent-solve",
           "configs": {}}
    for kind, T in (("random", 10), ("random", 5), ("random", 20), ("random", 12),
                    ("mixed", 10), ("standing", 10)):
        out["configs"][f"{kind}_T{T}"] = count(kind, T, sample if kind != "standing" else 1)
        print(kind, T, out["configs"][f"{kind}_T{T}"]["mean"])
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                        "flops_per_solve.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
