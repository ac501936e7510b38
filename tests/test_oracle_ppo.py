"""The CPU restatement of the PPO batch (oracle/rmpc_oracle_ppo.hpp) pinned by construction:
the reference ships no PPO test (tests/CMakeLists.txt has none), so ppo_loss's gradient
(ppo.cpp:79-135) is checked against central finite differences of its own total loss, the
loss terms against an independent numpy restatement of policy_forward / gaussian_log_prob
(policy.cpp:15-31, 85-102, 168-176), gae_advantages (ppo.cpp:28-45) against a numpy loop, and
ppo_update (ppo.cpp:195-276) against the closed form of one Adam step (t = 1) and the Rng
draws its shuffles consume.  CPU only."""
import numpy as np
import pytest

from paper_2510_12717_b200.synthetic import Xoshiro

LOG_SQRT_2PI = 0.91893853320467274178032973640562


def trunk_np(p, off, sizes, x):
    h = x
    for l in range(4):
        rows, cols = sizes[l + 1], sizes[l]
        W = p[off:off + rows * cols].reshape(cols, rows).T  # column-major (Eigen)
        off += rows * cols
        b = p[off:off + rows]
        off += rows
        z = h @ W.T + b
        h = np.where(z > 0, z, np.expm1(z)) if l < 3 else z
    return h, off


def batch(seed, n, obs=23, act=6, hidden=16, spread=0.4):
    from oracle import oracle as O
    rng = np.random.default_rng(seed)
    params = O.init_policy(obs, act, hidden, seed=seed, zero_final=False)
    o = rng.normal(size=(n, obs))
    mean, _ = O.policy_forward(params, o, act, hidden)
    a = mean + 0.5 * rng.normal(size=(n, act))
    sd = np.exp(params[-act:])
    logp = (-0.5 * ((a - mean) / sd) ** 2 - params[-act:] - LOG_SQRT_2PI).sum(1)
    old = logp + spread * rng.normal(size=n)  # ratios spread across both clip edges
    adv = rng.normal(size=n)
    ret = rng.normal(size=n)
    return params, o, a, old, adv, ret


def test_loss_terms_match_numpy(oracle):
    obs, act, hidden = 23, 6, 16
    params, o, a, old, adv, ret = batch(1, 33, obs, act, hidden)
    cfg = oracle.ppo_config(entropy_coef=0.01)
    (total, sur, vl, ent), _ = oracle.ppo_loss(params, o, a, old, adv, ret, cfg, act, hidden, grads=False)
    mean, off = trunk_np(params, 0, [obs, hidden, hidden, hidden, act], o)
    value, off = trunk_np(params, off, [obs, hidden, hidden, hidden, 1], o)
    ls = params[off:]
    logp = (-0.5 * ((a - mean) / np.exp(ls)) ** 2 - ls - LOG_SQRT_2PI).sum(1)
    ratio = np.exp(logp - old)
    surr = np.minimum(ratio * adv, np.clip(ratio, 0.8, 1.2) * adv)
    np.testing.assert_allclose(sur, -surr.mean(), rtol=1e-12)
    np.testing.assert_allclose(vl, 0.5 * ((value[:, 0] - ret) ** 2).mean(), rtol=1e-12)
    np.testing.assert_allclose(ent, (ls + LOG_SQRT_2PI + 0.5).sum(), rtol=1e-14)
    np.testing.assert_allclose(total, sur + 0.5 * vl - 0.01 * ent, rtol=1e-14)


@pytest.mark.parametrize("entropy_coef", [0.0, 0.01])
def test_gradient_matches_finite_differences(oracle, entropy_coef):
    obs, act, hidden = 23, 6, 16
    params, o, a, old, adv, ret = batch(2, 24, obs, act, hidden)
    cfg = oracle.ppo_config(entropy_coef=entropy_coef)
    _, g = oracle.ppo_loss(params, o, a, old, adv, ret, cfg, act, hidden)
    rng = np.random.default_rng(3)
    idx = np.concatenate([rng.choice(params.size - act, 150, replace=False), params.size - act + np.arange(act)])
    for k in idx:
        h = 1e-6 * max(1.0, abs(params[k]))
        pp, pm = params.copy(), params.copy()
        pp[k] += h
        pm[k] -= h
        fp = oracle.ppo_loss(pp, o, a, old, adv, ret, cfg, act, hidden, grads=False)[0][0]
        fm = oracle.ppo_loss(pm, o, a, old, adv, ret, cfg, act, hidden, grads=False)[0][0]
        fd = (fp - fm) / (2 * h)
        assert abs(fd - g[k]) <= 1e-6 * max(1e-3, abs(g[k])) + 1e-9, (k, fd, g[k])


def test_gae_matches_numpy(oracle):
    rng = np.random.default_rng(4)
    T, E = 9, 5
    r, v = rng.normal(size=(T, E)), rng.normal(size=(T, E))
    d = (rng.random((T, E)) < 0.2).astype(float)
    b = rng.normal(size=E)
    adv, ret = oracle.gae(r, v, d, b, 0.99, 0.95)
    ea, er = np.zeros((T, E)), np.zeros((T, E))
    for e in range(E):
        run = 0.0
        for t in reversed(range(T)):
            nd = 1.0 - d[t, e]
            nv = b[e] if t == T - 1 else v[t + 1, e]
            run = r[t, e] + 0.99 * nv * nd - v[t, e] + 0.99 * 0.95 * nd * run
            ea[t, e], er[t, e] = run, run + v[t, e]
    np.testing.assert_array_equal(adv, ea)
    np.testing.assert_array_equal(ret, er)


def rollout(seed, T, E, obs=23, act=6, hidden=16):
    from oracle import oracle as O
    rng = np.random.default_rng(seed)
    params = O.init_policy(obs, act, hidden, seed=seed, zero_final=False)
    o = rng.normal(size=(T, E, obs))
    mean, value = O.policy_forward(params, o.reshape(-1, obs), act, hidden)
    a = mean + 0.5 * rng.normal(size=mean.shape)
    sd = np.exp(params[-act:])
    logp = (-0.5 * ((a - mean) / sd) ** 2 - params[-act:] - LOG_SQRT_2PI).sum(1)
    return dict(params=params, obs=o, actions=a.reshape(T, E, act), logp=logp.reshape(T, E),
                values=value.reshape(T, E), rewards=rng.normal(size=(T, E)),
                dones=(rng.random((T, E)) < 0.1).astype(float), bootstrap=rng.normal(size=E))


def test_update_single_step_closed_form(oracle):
    """epochs = minibatches = 1: one Adam step at t = 1 moves every parameter by
    -lr g / (|g| + eps), g = the clipped full-batch gradient on normalised advantages."""
    obs, act, hidden, T, E = 23, 6, 16, 4, 8
    R = rollout(5, T, E, obs, act, hidden)
    cfg = oracle.ppo_config(epochs=1, minibatches=1, lr=1e-3, max_grad_norm=0.5)
    adv, ret = oracle.gae(R["rewards"], R["values"], R["dones"], R["bootstrap"])
    adv = adv.ravel()
    m = adv.sum() / adv.size
    var = ((adv - m) ** 2).sum() / adv.size
    adv_n = (adv - m) / np.sqrt(var + 1e-8)
    _, g = oracle.ppo_loss(R["params"], R["obs"].reshape(-1, obs), R["actions"].reshape(-1, act), R["logp"].ravel(),
                           adv_n, ret.ravel(), cfg, act, hidden)
    nrm = np.sqrt((g ** 2).sum())
    if nrm > cfg.max_grad_norm:
        g = g * (cfg.max_grad_norm / nrm)
    p = R["params"].copy()
    adam = oracle.AdamState(p.size)
    rng = oracle.rng_words(0, 0x0272)
    st = oracle.ppo_update(p, adam, R["obs"], R["actions"], R["logp"], R["values"], R["rewards"], R["dones"],
                           R["bootstrap"], cfg, rng, act, hidden)
    # the shuffle only reorders the sum: the step agrees to rounding
    np.testing.assert_allclose(p - R["params"], -1e-3 * g / (np.abs(g) + 1e-8), rtol=1e-6, atol=1e-12)
    assert adam.t.value == 1
    # the Rng advanced by exactly N - 1 uniform_int draws (Fisher-Yates, ppo.cpp:230)
    x = Xoshiro(0, [0x0272])
    for _ in range(T * E - 1):
        x.next_u64()
    assert [int(w[0]) for w in x.s] == list(rng)
    assert np.isfinite(st).all()


def test_update_stats_average_over_minibatches(oracle):
    obs, act, hidden, T, E = 23, 6, 16, 3, 10
    R = rollout(6, T, E, obs, act, hidden)
    cfg = oracle.ppo_config(epochs=2, minibatches=4)  # 30 samples: minibatches of 8, 8, 8, 6
    p = R["params"].copy()
    adam = oracle.AdamState(p.size)
    loss, sur, vl, ent = oracle.ppo_update(p, adam, R["obs"], R["actions"], R["logp"], R["values"], R["rewards"],
                                           R["dones"], R["bootstrap"], cfg, None, act, hidden)
    assert adam.t.value == 8
    np.testing.assert_allclose(loss, sur + 0.5 * vl, rtol=1e-12, atol=1e-15)  # entropy_coef 0
    # entropy of the last minibatch's parameters: log_std moved by at most 7 lr-sized steps
    np.testing.assert_allclose(ent, R["params"][-act:].sum() + act * (LOG_SQRT_2PI + 0.5), atol=7 * act * 3e-4)
