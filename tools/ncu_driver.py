"""Minimal driver for ncu captures: warm-up launches then timed device-resident solves.

python tools/ncu_driver.py [n_agents] [horizon] [launches] [sharing level: 0 per-agent .. 3 squads, default 2]
"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2510_12717_b200 as R  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    launches = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    level = int(sys.argv[4]) if len(sys.argv) > 4 else 2
    m, s = R.default_model(), R.default_settings(T)
    st, cm, ga = R.synthetic_batch(n, "random", seed=0, model=m, settings=s)
    br = R.BatchRunner(n, m, s)
    br.set_schedule_sharing(level)
    dev = torch.device("cuda:0")
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        dst, dcm, dga = (torch.from_numpy(a).to(dev) for a in (st, cm, ga))
        dout = torch.zeros(n * R.SOLUTION_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        for _ in range(launches):
            br.solve_device(dst, dcm, dga, dout, stream=stream)
    torch.cuda.synchronize()
    print("ok", n, T, launches)


if __name__ == "__main__":
    main()
