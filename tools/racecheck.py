"""compute-sanitizer target: small solves at N = 2, 3, 10 and 20 -- shared-schedule and per-agent
(sharing off, and warm start) paths -- on 1-2 CTAs each.

compute-sanitizer --tool racecheck python tools/racecheck.py [T ...]
"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2510_12717_b200 as R  # noqa: E402


def main():
    Ts = [int(a) for a in sys.argv[1:]] or [2, 3, 10, 20]
    m = R.default_model()
    for T in Ts:
        s = R.default_settings(T)
        n = 12
        st, cm, ga = R.synthetic_batch(n, "mixed", seed=3, model=m, settings=s)
        br = R.BatchRunner(n, m, s)
        sol, z = br.solve(st, cm, ga, want_z=True)
        br.set_schedule_sharing(False)
        sol2, z2 = br.solve(st, cm, ga, want_z=True)
        br.close()
        s.warm_start = 1
        bw = R.BatchRunner(n, m, s)
        sol3, _ = bw.solve(st, cm, ga, prev=(sol, z), want_z=True)
        bw.close()
        print("T", T, "ok", int((sol["status"] == 0).sum()), int((sol3["status"] == 0).sum()),
              "shared == per-agent", sol.tobytes() == sol2.tobytes() and z.tobytes() == z2.tobytes(),
              float(np.abs(z).max()), flush=True)
    # full squads: 70 agents of the random batch share few schedules (lanes 0..31 of a squad busy)
    s = R.default_settings(10)
    st, cm, ga = R.synthetic_batch(70, "random", seed=5, model=m, settings=s)
    br = R.BatchRunner(70, m, s)
    sol, z = br.solve(st, cm, ga, want_z=True)
    br.close()
    print("T 10 random squads ok", int((sol["status"] == 0).sum()), flush=True)


if __name__ == "__main__":
    main()
