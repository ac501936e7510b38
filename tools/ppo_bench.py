"""PPO batch measurement: one ppo_update (ppo.cpp:195-276) at the
reference Trainer's shape -- n_steps 24 x E envs, 4 epochs x 4 minibatches, hidden 64, obs 23,
act 6 -- on a device-resident synthetic rollout, plus one ppo_loss call (loss + reduce kernels)
on one minibatch with its FP64 roofline (algorithmic FLOPs / kernel time vs the measured FP64 FMA
peak), and the FP64 CPU oracle on a bounded sample of the same loss.

python tools/ppo_bench.py [envs] > profiles/rNN_ppo_bench.json   (on a B200)
"""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_12717_b200.env import Policy  # noqa: E402
from paper_2510_12717_b200.ppo import Adam, default_ppo_config, ppo_loss, ppo_update, rng_state  # noqa: E402
from paper_2510_12717_b200.runtime import library  # noqa: E402

LOG_SQRT_2PI = 0.91893853320467274178032973640562


def flop_per_sample(obs, act, hidden):
    """Multiply-adds x 2 of one sample's forward (both trunks), backward W^T delta (layers 1-3)
    and gradient outer products: the algorithmic count, exp/expm1 and the loss head excluded."""
    rc = []
    for out in (act, 1):
        rc.append([obs * hidden, hidden * hidden, hidden * hidden, hidden * out])
    fwd = sum(sum(t) for t in rc)
    bwd = sum(sum(t[1:]) for t in rc)
    return 2 * (fwd + bwd + fwd)


def measure(E=4096, cpu_seconds=5.0):
    T, obs, act, hidden = 24, 23, 6, 64
    N = T * E
    rng = np.random.default_rng(0)
    # synthetic weights, flatten_policy layout: two 4-layer trunks then log_std
    n_par = sum(i * o + o for out in (act, 1) for i, o in zip((obs, hidden, hidden, hidden), (hidden, hidden, hidden, out)))
    params = np.concatenate([rng.uniform(-0.2, 0.2, n_par), np.full(act, np.log(0.5))])
    o = rng.normal(size=(T, E, obs))
    a = 0.5 * rng.normal(size=(T, E, act))
    logp = (-0.5 * (a / 0.5) ** 2 - np.log(0.5) - LOG_SQRT_2PI).sum(-1) + 0.2 * rng.normal(size=(T, E))
    roll = [o, a, logp, rng.normal(size=(T, E)), rng.normal(size=(T, E)), (rng.random((T, E)) < 0.02) * 1.0,
            rng.normal(size=E)]
    d = [torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda() for x in roll]
    pol = Policy(params, obs, act, hidden)
    adam = Adam(pol, 3e-4)
    cfg = default_ppo_config()
    st = rng_state(0, 0x0272)
    for _ in range(2):
        ppo_update(pol, adam, *d, cfg, st)
    torch.cuda.synchronize()
    ups = []
    for _ in range(5):
        t0 = time.perf_counter()
        ppo_update(pol, adam, *d, cfg, st)  # synchronous (stats come back to the host)
        ups.append(time.perf_counter() - t0)
    t_up = float(np.median(ups))
    # the loss kernel alone on one minibatch (device time, CUDA events)
    mb = N // cfg.minibatches
    flat = [x.reshape(N, -1) if x.dim() == 3 else x.reshape(N) for x in d[:3]]
    adv, ret = torch.randn(N, dtype=torch.float64, device="cuda"), torch.randn(N, dtype=torch.float64, device="cuda")
    batch = [flat[0][:mb], flat[1][:mb], flat[2][:mb], adv[:mb], ret[:mb]]
    grads = torch.zeros(pol.num_params, dtype=torch.float64, device="cuda")
    for _ in range(3):
        ppo_loss(pol, *batch, cfg, grads)
    ms = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ppo_loss(pol, *batch, cfg, grads)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    t_loss = float(np.median(ms)) * 1e-3
    L = library()
    L.rmpc_fma_peak_f64.argtypes = [C.c_int32, C.c_void_p]
    peak = C.c_double()
    L.rmpc_fma_peak_f64(0, C.byref(peak))
    fl = flop_per_sample(obs, act, hidden)
    # CPU baseline: the FP64 oracle's ppo_loss + gradient on a bounded sample (the reference's
    # ppo_loss is serial); the oracle is only the baseline here, never the measured path
    from oracle import oracle as O
    ns = 2048
    cb = [roll[0].reshape(N, obs)[:ns], roll[1].reshape(N, act)[:ns], roll[2].reshape(N)[:ns],
          rng.normal(size=ns), rng.normal(size=ns)]
    O.ppo_loss(params, *cb, O.ppo_config(), act, hidden)
    t0 = time.perf_counter()
    reps = 0
    while time.perf_counter() - t0 < cpu_seconds:
        O.ppo_loss(params, *cb, O.ppo_config(), act, hidden)
        reps += 1
    cpu_sps = reps * ns / (time.perf_counter() - t0)
    samples_per_update = N * cfg.epochs
    return {
        "workload": f"ppo_update: {T} steps x {E} envs = {N} samples, {cfg.epochs} epochs x {cfg.minibatches} "
                    f"minibatches, MLP {obs}-{hidden}-{hidden}-{hidden}-{act} (+ value), FP64, synthetic rollout",
        "ppo_update_ms": t_up * 1e3,
        "samples_per_s": samples_per_update / t_up,
        "note_update": "host wall time of the synchronous rmpc_ppo_update_device call: GAE, normalisation, per epoch "
                       "a host Fisher-Yates (overlapping the device) + H2D, 16 x (loss + reduce + clip/Adam) launches",
        "ppo_loss": {
            "launches": "loss_kernel + reduce_kernel", "minibatch": mb, "ms": t_loss * 1e3, "samples_per_s": mb / t_loss,
            "flop_alg_per_sample": fl,
            "roofline": {"bound": "fp64", "achieved": fl * mb / t_loss / 1e12, "peak": peak.value,
                         "unit": "TFLOP/s", "frac": fl * mb / t_loss / 1e12 / peak.value,
                         "peak_source": "measured FP64 FMA loop on this GPU (rmpc_fma_peak_f64)"},
        },
        "cpu_baseline": {"samples_per_s": cpu_sps, "cores": 1, "kind": "port",
                         "sample": f"oracle ppo_loss + gradient on {ns} samples, repeated for {cpu_seconds:g} s "
                                   "(the reference's ppo_loss loop is single-threaded)"},
    }


def main():
    print(json.dumps(measure(int(sys.argv[1]) if len(sys.argv) > 1 else 4096)))


if __name__ == "__main__":
    main()
