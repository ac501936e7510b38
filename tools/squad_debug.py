"""Debug: squad vs per-agent solve at n_qp = 0, 1, 2, 25 (z*, records)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_12717_b200 as R  # noqa: E402

m = R.default_model()
for T in (10, 3):
    for nq in (1, 2, 3, 25):
        s = R.default_settings(T)
        s.n_qp = nq
        n = 64
        st, cm, ga = R.synthetic_batch(n, "random", seed=T, model=m, settings=s)
        br = R.BatchRunner(n, m, s)
        br.set_schedule_sharing(2)
        a, za = br.solve(st, cm, ga, want_z=True)
        br.set_schedule_sharing(0)
        b, zb = br.solve(st, cm, ga, want_z=True)
        dz = np.abs(za - zb)
        worst = np.unravel_index(np.argmax(dz), dz.shape)
        print(f"T={T} n_qp={nq}: status {np.bincount(a['status'], minlength=4)} vs {np.bincount(b['status'], minlength=4)}"
              f" | max|dz*| {dz.max():.3e} at {worst} (node, var) ; per node max: {np.round(dz.max(axis=(0, 2)), 6)}")
        for f in ("v_mpc", "prim_res", "dual_res", "delta_inf_norm"):
            print(f"   {f}: squad {a[f][:3]} per-agent {b[f][:3]}")
        if nq <= 3:
            print("   per var max |dz| node-avg:", np.round(dz.max(axis=(0, 1)), 5))
        br.close()
