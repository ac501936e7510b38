import sys, torch
sys.path.insert(0, ".")
import paper_2510_12717_b200 as R
for T, n in ((5, 8192 * 2), (10, 16384)):
    m, s = R.default_model(), R.default_settings(T)
    st, cm, ga = R.synthetic_batch(n, "random", seed=0, model=m, settings=s)
    br = R.BatchRunner(n, m, s)
    dev = torch.device("cuda:0")
    dst, dcm, dga = (torch.from_numpy(a).to(dev) for a in (st, cm, ga))
    dout = torch.zeros(n * R.SOLUTION_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    for _ in range(3): br.solve_device(dst, dcm, dga, dout, stream=stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); 
    for _ in range(10): br.solve_device(dst, dcm, dga, dout, stream=stream)
    e1.record(); torch.cuda.synchronize()
    print(sys.argv[1], "T", T, "n", n, "ms", e0.elapsed_time(e1) / 10)
