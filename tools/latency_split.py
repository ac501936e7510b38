"""Latency of one agent alone on an SM, by stage (per-agent kernel, sharing off, stage profiling):
what the schedule store's factorization (one warp pair per schedule) costs before the squads run.

python tools/latency_split.py [T]
"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2510_12717_b200 as R  # noqa: E402


def main():
    T = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    m, s = R.default_model(), R.default_settings(T)
    for n in (1, 6, 148):
        st, cm, ga = R.synthetic_batch(n, "random", seed=1, model=m, settings=s)
        br = R.BatchRunner(n, m, s)
        br.set_schedule_sharing(0)
        for _ in range(3):
            br.solve(st, cm, ga)
        ks = []
        for _ in range(5):
            br.solve(st, cm, ga)
            ks.append(br.last_timing()["kernel_ms"])
        br.set_stage_profiling(True)
        br.solve(st, cm, ga)
        t = br.last_timing()
        print(f"T={T} n={n}: kernel {np.median(ks) * 1e3:.1f} us; per-agent stage means (us): " +
              ", ".join(f"{k} {v * 1e3:.1f}" for k, v in t["stage_mean_ms"].items()), flush=True)
        br.close()


if __name__ == "__main__":
    main()
