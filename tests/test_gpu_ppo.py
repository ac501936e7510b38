"""PPO batch on the device (rmpc_ppo_*, paper_2510_12717_b200/csrc/rmpc_ppo.cu) against the FP64
oracle (oracle/rmpc_oracle_ppo.hpp, itself pinned by tests/test_oracle_ppo.py): ppo_loss terms
and every gradient entry, gae_advantages, and whole ppo_update calls (GAE, normalisation,
shuffled minibatches, clip, Adam) carried across two updates.  Both sides are FP64; they differ
only in summation order, so the tolerance is relative 1e-9 of the quantity's scale."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

LOG_SQRT_2PI = 0.91893853320467274178032973640562


def make_batch(O, seed, n, obs=23, act=6, hidden=64, spread=0.4):
    rng = np.random.default_rng(seed)
    params = O.init_policy(obs, act, hidden, seed=seed, zero_final=False)
    o = rng.normal(size=(n, obs))
    mean, _ = O.policy_forward(params, o, act, hidden)
    a = mean + 0.5 * rng.normal(size=(n, act))
    sd = np.exp(params[-act:])
    logp = (-0.5 * ((a - mean) / sd) ** 2 - params[-act:] - LOG_SQRT_2PI).sum(1)
    return params, o, a, logp + spread * rng.normal(size=n), rng.normal(size=n), rng.normal(size=n)


def cuda(*arrays):
    import torch
    return [torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda() for x in arrays]


def close(dev, ref, rel=1e-9):
    dev, ref = np.asarray(dev), np.asarray(ref)
    scale = max(np.abs(ref).max(), 1e-300)
    assert np.abs(dev - ref).max() <= rel * scale, (np.abs(dev - ref).max(), scale)


@pytest.mark.parametrize("n", [1, 7, 16, 17, 300, 5000])
@pytest.mark.parametrize("hidden", [64, 24])
def test_loss_and_gradient_parity(oracle, n, hidden):
    from paper_2510_12717_b200.env import Policy
    from paper_2510_12717_b200.ppo import default_ppo_config, ppo_loss
    obs, act = 23, 6
    params, o, a, old, adv, ret = make_batch(oracle, n + hidden, n, obs, act, hidden)
    cfg_o = oracle.ppo_config(entropy_coef=0.01)
    info_o, g_o = oracle.ppo_loss(params, o, a, old, adv, ret, cfg_o, act, hidden)
    pol = Policy(params, obs, act, hidden)
    info, g = ppo_loss(pol, *cuda(o, a, old, adv, ret), default_ppo_config(entropy_coef=0.01))
    for k, name in enumerate(("total", "surrogate", "value_loss", "entropy")):
        np.testing.assert_allclose(getattr(info, name), info_o[k], rtol=1e-9, atol=1e-13, err_msg=name)
    g = g.cpu().numpy()
    tp = (obs * hidden + hidden) + 2 * (hidden * hidden + hidden) + hidden * act + act
    close(g[:tp], g_o[:tp])  # pi trunk
    close(g[tp:-act], g_o[tp:-act])  # value trunk
    close(g[-act:], g_o[-act:])  # log_std


@pytest.mark.parametrize("obs,act,hidden", [(17, 3, 20), (31, 7, 40)])
def test_loss_parity_padded_shapes(oracle, obs, act, hidden):
    """Shapes that are not multiples of the 8 x 8 tensor-core blocks (zero-padded operands)."""
    from paper_2510_12717_b200.env import Policy
    from paper_2510_12717_b200.ppo import default_ppo_config, ppo_loss
    n = 333
    params, o, a, old, adv, ret = make_batch(oracle, 6, n, obs, act, hidden)
    info_o, g_o = oracle.ppo_loss(params, o, a, old, adv, ret, oracle.ppo_config(), act, hidden)
    pol = Policy(params, obs, act, hidden)
    info, g = ppo_loss(pol, *cuda(o, a, old, adv, ret), default_ppo_config())
    np.testing.assert_allclose(info.total, info_o[0], rtol=1e-9)
    close(g.cpu().numpy(), g_o)


def test_loss_parity_cuda_core_fallback(oracle):
    """obs 64 / act 32 / hidden 64 exceeds the tensor-core layout's shared memory: the CUDA-core
    kernel runs and must agree just the same."""
    from paper_2510_12717_b200.env import Policy
    from paper_2510_12717_b200.ppo import default_ppo_config, ppo_loss
    obs, act, hidden, n = 64, 32, 64, 300
    params, o, a, old, adv, ret = make_batch(oracle, 5, n, obs, act, hidden)
    info_o, g_o = oracle.ppo_loss(params, o, a, old, adv, ret, oracle.ppo_config(), act, hidden)
    pol = Policy(params, obs, act, hidden)
    info, g = ppo_loss(pol, *cuda(o, a, old, adv, ret), default_ppo_config())
    np.testing.assert_allclose(info.total, info_o[0], rtol=1e-9)
    close(g.cpu().numpy(), g_o)


def test_loss_deterministic_and_default_dims(oracle):
    import torch
    from paper_2510_12717_b200.env import Policy
    from paper_2510_12717_b200.ppo import ppo_loss
    params, o, a, old, adv, ret = make_batch(oracle, 9, 4096)
    pol = Policy(params)
    d = cuda(o, a, old, adv, ret)
    i1, g1 = ppo_loss(pol, *d)
    i2, g2 = ppo_loss(pol, *d)
    assert torch.equal(g1, g2) and i1.total == i2.total
    assert pol.num_params == params.size
    np.testing.assert_array_equal(pol.get_params(), params)


def test_gae_parity(oracle):
    from paper_2510_12717_b200.ppo import gae
    rng = np.random.default_rng(11)
    T, E = 24, 1000
    r, v, b = rng.normal(size=(T, E)), rng.normal(size=(T, E)), rng.normal(size=E)
    d = (rng.random((T, E)) < 0.05).astype(float)
    adv_o, ret_o = oracle.gae(r, v, d, b, 0.99, 0.95)
    adv, ret = gae(*cuda(r, v, d, b), 0.99, 0.95)
    np.testing.assert_allclose(adv.cpu().numpy(), adv_o, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(ret.cpu().numpy(), ret_o, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("T,E,epochs,mb,hidden", [(4, 16, 1, 1, 64), (8, 64, 2, 3, 64), (5, 37, 2, 4, 32)])
def test_update_parity_over_two_updates(oracle, T, E, epochs, mb, hidden):
    from paper_2510_12717_b200.env import Policy
    from paper_2510_12717_b200.ppo import Adam, default_ppo_config, ppo_update, rng_state
    obs, act = 23, 6
    rng = np.random.default_rng(T * E)
    params = oracle.init_policy(obs, act, hidden, seed=E, zero_final=False)
    pol = Policy(params, obs, act, hidden)
    adam = Adam(pol, lr=3e-4)
    adam_o = oracle.AdamState(params.size)
    p_o = params.copy()
    rng_d, rng_o = rng_state(7, 0x0272), oracle.rng_words(7, 0x0272)
    cfg = default_ppo_config(epochs=epochs, minibatches=mb)
    cfg_o = oracle.ppo_config(epochs=epochs, minibatches=mb)
    for _ in range(2):
        o = rng.normal(size=(T, E, obs))
        mean, value = oracle.policy_forward(p_o, o.reshape(-1, obs), act, hidden)
        a = mean + 0.5 * rng.normal(size=mean.shape)
        sd = np.exp(p_o[-act:])
        logp = (-0.5 * ((a - mean) / sd) ** 2 - p_o[-act:] - LOG_SQRT_2PI).sum(1) + 0.2 * rng.normal(size=T * E)
        roll = [o, a.reshape(T, E, act), logp.reshape(T, E), value.reshape(T, E), rng.normal(size=(T, E)),
                (rng.random((T, E)) < 0.1).astype(float), rng.normal(size=E)]
        st = ppo_update(pol, adam, *cuda(*roll), cfg, rng_d)
        st_o = oracle.ppo_update(p_o, adam_o, *roll, cfg_o, rng_o, act, hidden)
        assert list(rng_d) == list(rng_o)
        np.testing.assert_allclose([st.loss, st.surrogate, st.value_loss, st.entropy], st_o, rtol=1e-8, atol=1e-12)
        p = pol.get_params()
        # Adam normalises each step to ~lr, so compare the accumulated step against its own scale
        close(p - params, p_o - params, rel=1e-7)


def test_empty_batch_is_structural_error():
    import torch
    from paper_2510_12717_b200.env import Policy
    from paper_2510_12717_b200.ppo import ppo_loss
    from paper_2510_12717_b200.runtime import RmpcError
    from oracle import oracle as O
    pol = Policy(O.init_policy())
    z = torch.zeros((0, 23), dtype=torch.float64, device="cuda")
    e = torch.zeros(0, dtype=torch.float64, device="cuda")
    with pytest.raises(RmpcError):
        ppo_loss(pol, z, torch.zeros((0, 6), dtype=torch.float64, device="cuda"), e, e, e)
