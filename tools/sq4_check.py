import sys, os, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_2510_12717_b200 as R
from paper_2510_12717_b200.abi import SOLUTION_DTYPE
from parity import compare, summary
from oracle import oracle as O
m = R.default_model()
for T, kind, n in ((11, 'random', 300), (12, 'random', 999), (15, 'mixed', 500), (20, 'mixed', 1024), (20, 'random', 700)):
    s = R.default_settings(T)
    st, cm, ga = R.synthetic_batch(n, kind, seed=T, model=m, settings=s)
    st = st.copy(); st[5, 3] = np.nan
    br = R.BatchRunner(n, m, s)
    res = {}
    for lvl in (3, 0):
        br.set_schedule_sharing(lvl)
        res[lvl] = br.solve(st, cm, ga, want_z=True)
    ref, zr, _, _ = O.solve_batch(m, s, st, cm, ga, workers=16)
    a, za = res[3]
    print(f"T={T} {kind} n={n} status {np.bincount(a['status'], minlength=4)}", flush=True)
    print("  long squads vs oracle:", summary(compare(a, ref, za, zr)), flush=True)
    print("  per-agent vs oracle:  ", summary(compare(res[0][0], ref, res[0][1], zr)), flush=True)
    br.close()
dev = torch.device('cuda:0')
for T, n in ((12, 8192), (20, 8192), (16, 8192)):
    s = R.default_settings(T)
    st, cm, ga = R.synthetic_batch(n, 'random', seed=0, model=m, settings=s)
    br = R.BatchRunner(n, m, s)
    d = [torch.from_numpy(x).to(dev) for x in (st, cm, ga)]
    out = torch.zeros(n * SOLUTION_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    z = torch.zeros(n * T * 26, dtype=torch.float32, device=dev)
    for lvl in (3, 1):
        br.set_schedule_sharing(lvl)
        for _ in range(3): br.solve_device(*d, out, z_out=z)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): br.solve_device(*d, out, z_out=z)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        ok = int((out.cpu().numpy().view(SOLUTION_DTYPE)['status'] == 0).sum())
        br.set_stage_profiling(True); br.solve(st, cm, ga); tm = br.last_timing(); br.set_stage_profiling(False)
        print(f"T={T} n={n} level={lvl}: {ms:.3f} ms ok={ok} per-agent us", {k: round(v*1e3,1) for k, v in tm['stage_mean_ms'].items() if v > 0}, flush=True)
    br.close()
