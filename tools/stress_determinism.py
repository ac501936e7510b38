"""Determinism stress (the race-safety evidence without compute-sanitizer): 1 000
device-resident ticks per configuration, every 50th compared byte for byte with the first tick, then
200 host-path ticks (split launch, copy-out) compared with the device bytes.  C3, C4 N = 5 / 20 and an
over-capacity batch (the device-dispatched per-agent list), each with one non-finite agent.

python tools/stress_determinism.py   (on a B200)
"""
import sys, time; sys.path.insert(0, '/root/repo')
import numpy as np, torch, paper_2510_12717_b200 as R
from paper_2510_12717_b200.abi import SOLUTION_DTYPE
dev = torch.device('cuda:0')
m = R.default_model()
for T, n, kind in ((10, 16384, 'random'), (5, 8192, 'mixed'), (20, 8192, 'random'), (10, 3000, 'overcap')):
    s = R.default_settings(T)
    st, cm, ga = R.synthetic_batch(n, 'random' if kind == 'overcap' else kind, seed=T, model=m, settings=s)
    if kind == 'overcap':
        rng = np.random.default_rng(8); ga = ga.copy(); ga[:, 1] = rng.uniform(0.35, 0.9, n); ga[:, 2] = rng.uniform(0.45, 0.7, n)
    st = st.copy(); st[7, 2] = np.nan
    br = R.BatchRunner(n, m, s)
    d = [torch.from_numpy(x).to(dev) for x in (st, cm, ga)]
    out = torch.zeros(n * SOLUTION_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    z = torch.zeros(n * T * 26, dtype=torch.float32, device=dev)
    br.solve_device(*d, out, z_out=z); torch.cuda.synchronize()
    ref_o, ref_z = out.clone(), z.clone()
    bad = 0; t0 = time.time()
    for k in range(1000):
        out.zero_(); z.zero_()
        br.solve_device(*d, out, z_out=z)
        if k % 50 == 49:
            torch.cuda.synchronize()
            if not (torch.equal(out, ref_o) and torch.equal(z, ref_z)): bad += 1
    torch.cuda.synchronize()
    ok = torch.equal(out, ref_o) and torch.equal(z, ref_z)
    # host path repeated, bytes equal to the device path's
    h = [torch.from_numpy(x).pin_memory().numpy() for x in (st, cm, ga)]
    ho = torch.zeros(n * SOLUTION_DTYPE.itemsize, dtype=torch.uint8).pin_memory().numpy().view(SOLUTION_DTYPE)
    hz = torch.zeros((n, T, 26), dtype=torch.float32).pin_memory().numpy()
    hbad = 0
    for k in range(200):
        br.solve(*h, out=ho, z_out=hz)
        if k % 20 == 19 and not (ho.tobytes() == ref_o.cpu().numpy().tobytes() and hz.tobytes() == ref_z.cpu().numpy().tobytes()): hbad += 1
    print(f"T={T} n={n} {kind}: 1000 device ticks, mismatching checks {bad}, final equal {ok}; 200 host ticks mismatching checks {hbad}; {time.time()-t0:.1f}s", flush=True)
    br.close()
