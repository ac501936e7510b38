"""Parity measurement of the CUDA path against (a) the reference built from its own sources
(tests/golden/ref_*.npz, produced by oracle/_ref) and (b) the restated FP64 oracle at the
real C4 sizes (8 192 agents x N = 5 / 10 / 20) -- every rmpc_solution field, max and p99 of
the per-agent relative error (tests/parity.py metrics).  Writes JSON to argv[1].

python tools/ref_parity.py gpurun_out/ref_parity.json
"""
import glob
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2510_12717_b200 as R  # noqa: E402
from parity import compare, fixture_settings  # noqa: E402


def stats(c):
    out = {"n_ok": c["n_ok"], "status_equal": c["status_equal"], "fail_iter_equal": c["fail_iter_equal"]}
    for k, v in c.items():
        if isinstance(v, np.ndarray) and v.size:
            out[k] = {"max": float(v.max()), "p99": float(np.percentile(v, 99)), "p50": float(np.median(v))}
    return out


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else "ref_parity.json"
    res = {"ref_fixtures": {}, "oracle_c4": {}}
    m = R.default_model()
    for f in sorted(glob.glob(os.path.join(ROOT, "tests", "golden", "ref_*.npz"))):
        g = np.load(f)
        s = fixture_settings(g)
        n = g["states"].shape[0]
        br = R.BatchRunner(n, m, s)
        prev = None
        if "prev_z" in g.files:
            psol = np.zeros(n, dtype=R.SOLUTION_DTYPE)
            psol["status"] = g["prev_ok"]
            prev = (psol, g["prev_z"].astype(np.float32))
        sol, z = br.solve(g["states"], g["cmds"], g["gaits"], prev=prev, want_z=True)
        c = compare(sol, g, z, g["z"])
        name = os.path.basename(f)[4:-4]
        res["ref_fixtures"][name] = stats(c)
        print(name, {k: (round(v["max"], 8) if isinstance(v, dict) else v) for k, v in stats(c).items()}, flush=True)
        br.close()
    from oracle import oracle as O
    workers = os.cpu_count() or 1
    for T in (5, 10, 20):
        for kind in ("random", "mixed"):
            s = R.default_settings(T)
            n = 8192
            st, cm, ga = R.synthetic_batch(n, kind, seed=40 + T, model=m, settings=s)
            br = R.BatchRunner(n, m, s)
            sol, z = br.solve(st, cm, ga, want_z=True)
            ref, zr, _, _ = O.solve_batch(m, s, st, cm, ga, workers=workers)
            c = compare(sol, ref, z, zr)
            key = f"{kind}_T{T}_n{n}"
            res["oracle_c4"][key] = stats(c)
            print(key, {k: (round(v["max"], 8) if isinstance(v, dict) else v) for k, v in stats(c).items()}, flush=True)
            br.close()
    with open(out_path, "w") as fh:
        json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
