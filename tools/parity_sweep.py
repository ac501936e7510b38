"""Broad parity sweep (run on a B200): every horizon 2..32, three input kinds, 1 024 agents each,
device solver vs the FP64 oracle on the box's host cores; max relative errors of tau_ff, F*[0]
and V (tests/parity.py metrics) and status agreement per case.

python tools/parity_sweep.py > profiles/rNN_parity_sweep.json
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402

import paper_2510_12717_b200 as R  # noqa: E402
from oracle import oracle as O  # noqa: E402
from parity import TOL, compare  # noqa: E402


def main():
    rows = []
    kinds = ("random", "mixed", "standing")
    for T in range(2, 33):
        for kind in kinds:
            n = 1024
            m, s = R.default_model(), R.default_settings(T)
            st, cm, ga = R.synthetic_batch(n, kind, seed=T * 7 + len(kind), model=m, settings=s,
                                           nominal=O.nominal_pose(m))
            sol, _ = R.BatchRunner(n, m, s).solve(st, cm, ga)
            ref, _, _, _ = O.solve_batch(m, s, st, cm, ga, workers=os.cpu_count() or 1)
            c = compare(sol, ref)
            rows.append({"horizon": T, "kind": kind, "agents": n, "status_equal": c["status_equal"],
                         "ok": c["n_ok"], "tau_max": float(c["tau"].max()), "f0_max": float(c["f0"].max()),
                         "v_max": float(c["v"].max()),
                         "pass": bool(c["status_equal"] and max(c["tau"].max(), c["f0"].max(), c["v"].max()) <= TOL)})
            print(rows[-1], file=sys.stderr, flush=True)
    print(json.dumps({"tolerance": TOL, "cases": len(rows), "passed": sum(r["pass"] for r in rows),
                      "worst": {k: max(r[k] for r in rows) for k in ("tau_max", "f0_max", "v_max")},
                      "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
