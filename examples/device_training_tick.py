"""A device-resident Residual-MPC training iteration from the public APIs (what
Trainer::train, /root/reference/proj/src/ppo.cpp:299-394, does per iteration), as a usage
example: every tick solve the MPC batch, observe, run the residual policy, blend and step the
simulator; after n_steps ticks run one PPO update on the collected rollout.  Rewards and
resets stay with the caller (out of scope here): a placeholder reward is used, and agents
whose simulation blew up (sim_status, the reference's SimBlowupError) are reset to their
initial state with done = 1.  The first iteration is a warm-up (workspaces, caches).

python examples/device_training_tick.py [envs] [steps]     (on a B200)
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_12717_b200 as R  # noqa: E402
from paper_2510_12717_b200.abi import SOLUTION_DTYPE  # noqa: E402
from paper_2510_12717_b200.env import Env, Policy, default_env_config  # noqa: E402
from paper_2510_12717_b200.ppo import Adam, default_ppo_config, ppo_update, rng_state  # noqa: E402

LOG_SQRT_2PI = 0.91893853320467274178032973640562


def main():
    E = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 24
    dev = torch.device("cuda:0")
    m, s = R.default_model(), R.default_settings(10)
    st, cm, ga = R.synthetic_batch(E, "mixed", seed=0, model=m, settings=s)
    states, cmds, gaits = (torch.from_numpy(a).to(dev) for a in (st, cm, ga))
    runner = R.BatchRunner(E, m, s)
    env = Env(m, default_env_config())
    obs_dim, act_dim, hidden = 23, 6, 64
    rng = np.random.default_rng(0)
    n_par = sum(i * o + o for out in (act_dim, 1)
                for i, o in zip((obs_dim, hidden, hidden, hidden), (hidden, hidden, hidden, out)))
    policy = Policy(np.concatenate([rng.uniform(-0.1, 0.1, n_par), np.full(act_dim, np.log(0.5))]))
    adam, update_rng = Adam(policy, 3e-4), rng_state(0, 0x0272)
    f64 = dict(dtype=torch.float64, device=dev)
    buf = dict(obs=torch.zeros((T, E, obs_dim), **f64), act=torch.zeros((T, E, act_dim), **f64),
               logp=torch.zeros((T, E), **f64), val=torch.zeros((T, E), **f64),
               rew=torch.zeros((T, E), **f64), done=torch.zeros((T, E), **f64))
    sol = torch.zeros(E * SOLUTION_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    mean = torch.zeros((E, act_dim), **f64)
    value = torch.zeros(E, **f64)
    sd = torch.exp(torch.from_numpy(policy.log_std).to(dev))
    sim = torch.zeros(E, dtype=torch.int32, device=dev)
    st0, ga0 = states.clone(), gaits.clone()
    for it in range(2):  # iteration 0 warms up
        stats, t_roll, t_upd = iteration(E, T, runner, env, policy, adam, update_rng, states, cmds, gaits, st0, ga0,
                                         sol, mean, value, sd, sim, buf, f64, obs_dim)
    print(f"{E} envs x {T} ticks: rollout {1e3 * t_roll:.1f} ms ({1e3 * t_roll / T:.2f} ms/tick), "
          f"ppo_update {1e3 * t_upd:.1f} ms, loss {stats.loss:.4g}, value loss {stats.value_loss:.4g}")


def iteration(E, T, runner, env, policy, adam, update_rng, states, cmds, gaits, st0, ga0, sol, mean, value, sd,
              sim, buf, f64, obs_dim):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for t in range(T):
        runner.solve_device(states, cmds, gaits, sol)                       # MPC batch (Alg. 1)
        env.observe(states, gaits, sol, buf["obs"][t])                       # policy input
        policy.forward(buf["obs"][t], mean, value)                           # residual policy
        a = mean + sd * torch.randn_like(mean)                               # Gaussian action
        buf["act"][t] = a
        buf["logp"][t] = (-0.5 * ((a - mean) / sd) ** 2 - torch.log(sd) - LOG_SQRT_2PI).sum(1)
        buf["val"][t] = value
        env.control_step(sol, states, gaits, action=a, strategy="joint-torque", lam=0.1, sim_status=sim)
        blown = sim != 0
        buf["done"][t] = blown.to(torch.float64)
        buf["rew"][t] = torch.where(blown, torch.zeros_like(value), -states[:, 10].abs().clamp(max=10.0))
        states[blown] = st0[blown]                                           # reset (placeholder)
        gaits[blown] = ga0[blown]
    bootstrap_obs = torch.zeros((E, obs_dim), **f64)
    env.observe(states, gaits, sol, bootstrap_obs)
    policy.forward(bootstrap_obs, None, value)                               # bootstrap value
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    stats = ppo_update(policy, adam, buf["obs"], buf["act"], buf["logp"], buf["val"], buf["rew"], buf["done"],
                       value, default_ppo_config(), update_rng)
    t2 = time.perf_counter()
    return stats, t1 - t0, t2 - t1


if __name__ == "__main__":
    main()
