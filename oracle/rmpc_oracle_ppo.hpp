// rmpc_oracle_ppo.hpp — TEST INFRASTRUCTURE ONLY: FP64 CPU restatement of the PPO batch
// (the "PPO batch" half), the parity oracle for the rmpc_ppo_* entry
// points of include/rmpc_b200_env.h.  Only tests/ and bench.py's CPU legs may call it.
//
//   mlp_forward (with cache)   /root/reference/proj/src/policy.cpp:15-31
//   gaussian_log_prob          policy.cpp:168-176
//   mlp_backward               ppo.cpp:63-77
//   ppo_loss                   ppo.cpp:79-135
//   gae_advantages             ppo.cpp:28-45
//   AdamOptimizer::step        ppo.cpp:179-193 (defaults ppo.hpp:93-94)
//   ppo_update                 ppo.cpp:195-276 (Fisher-Yates with Rng::uniform_int, rng.hpp:43)
//
// Parameters are the flat vector of flatten_policy (ppo.cpp:144-153): per trunk and layer W
// (out x in, column-major) then b; pi, then value, then log_std.
#pragma once

#include <algorithm>
#include <cmath>
#include <vector>

#include "../include/rmpc_b200_env.h"
#include "rmpc_oracle_rng.hpp"

namespace oracle {

constexpr double kLogSqrt2PiPpo = 0.91893853320467274178032973640562;

struct TrunkShape {
  int sizes[5];
  int w[4], b[4], total;
};

inline TrunkShape trunk_shape(int obs, int hidden, int out_dim, int base) {
  TrunkShape t{{obs, hidden, hidden, hidden, out_dim}, {}, {}, 0};
  int off = base;
  for (int l = 0; l < 4; ++l) {
    t.w[l] = off;
    off += t.sizes[l] * t.sizes[l + 1];
    t.b[l] = off;
    off += t.sizes[l + 1];
  }
  t.total = off - base;
  return t;
}

struct TrunkCache {
  std::vector<double> post[4];  // inputs of layers 0..3 (post[0] = the observation)
  std::vector<double> pre[4];   // pre-activations z of layers 0..3
};

// mlp_forward with the cache (policy.cpp:15-31); returns the trunk output.
inline std::vector<double> trunk_forward(const double* p, const TrunkShape& t, const double* in,
                                         TrunkCache& c) {
  std::vector<double> h(in, in + t.sizes[0]);
  for (int l = 0; l < 4; ++l) {
    const int rows = t.sizes[l + 1], cols = t.sizes[l];
    c.post[l] = h;
    std::vector<double> z(rows);
    for (int i = 0; i < rows; ++i) {
      double acc = 0.0;
      for (int k = 0; k < cols; ++k) acc += p[t.w[l] + k * rows + i] * h[k];
      z[i] = acc + p[t.b[l] + i];
    }
    c.pre[l] = z;
    if (l < 3)
      for (double& v : z) v = v > 0.0 ? v : std::expm1(v);
    h = z;
  }
  return h;
}

// mlp_backward (ppo.cpp:63-77): grads += d(loss)/d(params) of one trunk for output gradient g.
inline void trunk_backward(const double* p, const TrunkShape& t, const TrunkCache& c,
                           std::vector<double> delta, double* g) {
  for (int l = 3; l >= 0; --l) {
    const int rows = t.sizes[l + 1], cols = t.sizes[l];
    for (int k = 0; k < cols; ++k)
      for (int i = 0; i < rows; ++i) g[t.w[l] + k * rows + i] += delta[i] * c.post[l][k];
    for (int i = 0; i < rows; ++i) g[t.b[l] + i] += delta[i];
    if (l > 0) {
      std::vector<double> back(cols, 0.0);
      for (int k = 0; k < cols; ++k) {
        double acc = 0.0;
        for (int i = 0; i < rows; ++i) acc += p[t.w[l] + k * rows + i] * delta[i];
        back[k] = acc;
      }
      for (int k = 0; k < cols; ++k) {
        const double z = c.pre[l - 1][k];
        back[k] *= z > 0.0 ? 1.0 : std::exp(z);  // elu_grad, ppo.cpp:12
      }
      delta = back;
    }
  }
}

inline void ppo_config_default(rmpc_ppo_config* c) {  // PpoConfig, ppo.hpp:14-24
  c->gamma = 0.99;
  c->lam_gae = 0.95;
  c->clip_eps = 0.2;
  c->epochs = 4;
  c->minibatches = 4;
  c->lr = 3e-4;
  c->entropy_coef = 0.0;
  c->value_coef = 0.5;
  c->max_grad_norm = 1.0;
}

// ppo_loss (ppo.cpp:79-135) on n samples; grads (num_params, zeroed by the caller) may be null.
inline rmpc_ppo_loss_info ppo_loss(const double* params, int obs_dim, int act, int hidden, int n,
                                   const double* obs, const double* actions, const double* old_logp,
                                   const double* adv, const double* ret, const rmpc_ppo_config& cfg,
                                   double* grads) {
  const TrunkShape tp = trunk_shape(obs_dim, hidden, act, 0);
  const TrunkShape tv = trunk_shape(obs_dim, hidden, 1, tp.total);
  const double* log_std = params + tp.total + tv.total;
  const double inv_n = 1.0 / n;
  rmpc_ppo_loss_info info{0.0, 0.0, 0.0, 0.0};
  TrunkCache cp, cv;
  std::vector<double> grad_mean(act);
  for (int s = 0; s < n; ++s) {
    const double* o = obs + (size_t)s * obs_dim;
    const double* a = actions + (size_t)s * act;
    const std::vector<double> mean = trunk_forward(params, tp, o, cp);
    const double value = trunk_forward(params, tv, o, cv)[0];
    double logp = 0.0;  // gaussian_log_prob, policy.cpp:168-176
    for (int j = 0; j < act; ++j) {
      const double sd = std::exp(log_std[j]);
      const double z = (a[j] - mean[j]) / sd;
      logp += -0.5 * z * z - log_std[j] - kLogSqrt2PiPpo;
    }
    const double ratio = std::exp(logp - old_logp[s]);
    const double surr1 = ratio * adv[s];
    const double clipped = std::min(std::max(ratio, 1.0 - cfg.clip_eps), 1.0 + cfg.clip_eps) * adv[s];
    info.surrogate += -std::min(surr1, clipped) * inv_n;
    const double verr = value - ret[s];
    info.value_loss += 0.5 * verr * verr * inv_n;
    if (grads) {
      const double g_r = surr1 <= clipped ? -adv[s] * inv_n : 0.0;
      if (g_r != 0.0) {
        const double g_logp = g_r * ratio;
        for (int j = 0; j < act; ++j) {
          const double sd = std::exp(log_std[j]);
          const double z = (a[j] - mean[j]) / sd;
          grad_mean[j] = g_logp * z / sd;
          grads[tp.total + tv.total + j] += g_logp * (z * z - 1.0);
        }
        trunk_backward(params, tp, cp, grad_mean, grads);
      }
      trunk_backward(params, tv, cv, {cfg.value_coef * verr * inv_n}, grads);
    }
  }
  for (int j = 0; j < act; ++j) info.entropy += log_std[j] + kLogSqrt2PiPpo + 0.5;
  if (grads && cfg.entropy_coef != 0.0)
    for (int j = 0; j < act; ++j) grads[tp.total + tv.total + j] -= cfg.entropy_coef;
  info.total = info.surrogate + cfg.value_coef * info.value_loss - cfg.entropy_coef * info.entropy;
  return info;
}

// gae_advantages (ppo.cpp:28-45); arrays steps x envs row-major.
inline void gae(int T, int E, const double* rewards, const double* values, const double* dones,
                const double* bootstrap, double gamma, double lam, double* adv, double* ret) {
  for (int e = 0; e < E; ++e) {
    double running = 0.0;
    for (int t = T - 1; t >= 0; --t) {
      const double not_done = 1.0 - dones[t * E + e];
      const double next_value = t == T - 1 ? bootstrap[e] : values[(t + 1) * E + e];
      const double delta = rewards[t * E + e] + gamma * next_value * not_done - values[t * E + e];
      running = delta + gamma * lam * not_done * running;
      adv[t * E + e] = running;
      ret[t * E + e] = running + values[t * E + e];
    }
  }
}

struct Adam {  // AdamOptimizer (ppo.cpp:179-193)
  double lr, beta1 = 0.9, beta2 = 0.999, eps = 1e-8;
  int t = 0;
  std::vector<double> m, v;
  Adam(int dim, double lr_) : lr(lr_), m(dim, 0.0), v(dim, 0.0) {}
  void step(double* params, const double* g) {
    ++t;
    const double bc1 = 1.0 - std::pow(beta1, t), bc2 = 1.0 - std::pow(beta2, t);
    for (size_t i = 0; i < m.size(); ++i) {
      m[i] = beta1 * m[i] + (1.0 - beta1) * g[i];
      v[i] = beta2 * v[i] + (1.0 - beta2) * (g[i] * g[i]);
      params[i] -= lr * (m[i] / bc1) / (std::sqrt(v[i] / bc2) + eps);
    }
  }
};

// ppo_update (ppo.cpp:195-276) over a rollout of T steps x E envs (obs T x E x obs_dim,
// actions T x E x act, the rest T x E; bootstrap E).  params are updated in place.
inline rmpc_ppo_update_stats ppo_update(double* params, int obs_dim, int act, int hidden, int T, int E,
                                        const double* obs, const double* actions, const double* logp,
                                        const double* values, const double* rewards, const double* dones,
                                        const double* bootstrap, const rmpc_ppo_config& cfg, Adam& adam,
                                        Rng& rng) {
  const int N = T * E;
  const int np = static_cast<int>(adam.m.size());
  std::vector<double> adv(N), ret(N);
  gae(T, E, rewards, values, dones, bootstrap, cfg.gamma, cfg.lam_gae, adv.data(), ret.data());
  double mean = 0.0;
  for (double a : adv) mean += a;
  mean /= N;
  double var = 0.0;
  for (double a : adv) var += (a - mean) * (a - mean);
  var /= N;
  const double inv_std = 1.0 / std::sqrt(var + 1e-8);
  for (double& a : adv) a = (a - mean) * inv_std;
  std::vector<int> order(N);
  for (int i = 0; i < N; ++i) order[i] = i;
  rmpc_ppo_update_stats st{0.0, 0.0, 0.0, 0.0};
  int count = 0;
  const int mbc = std::max(1, cfg.minibatches);
  std::vector<double> so, sa, sl, sv, sr, g(np);
  for (int ep = 0; ep < cfg.epochs; ++ep) {
    for (int i = N - 1; i > 0; --i) std::swap(order[i], order[rng.uniform_int(i + 1)]);
    const int mb = (N + mbc - 1) / mbc;
    for (int b = 0; b < mbc; ++b) {
      const int lo = b * mb, hi = std::min(N, lo + mb);
      if (lo >= hi) continue;
      const int n = hi - lo;
      so.resize((size_t)n * obs_dim);
      sa.resize((size_t)n * act);
      sl.resize(n);
      sv.resize(n);
      sr.resize(n);
      for (int s = 0; s < n; ++s) {
        const int src = order[lo + s];
        std::copy(obs + (size_t)src * obs_dim, obs + (size_t)(src + 1) * obs_dim, so.begin() + (size_t)s * obs_dim);
        std::copy(actions + (size_t)src * act, actions + (size_t)(src + 1) * act, sa.begin() + (size_t)s * act);
        sl[s] = logp[src];
        sv[s] = adv[src];
        sr[s] = ret[src];
      }
      std::fill(g.begin(), g.end(), 0.0);
      const rmpc_ppo_loss_info info = ppo_loss(params, obs_dim, act, hidden, n, so.data(), sa.data(), sl.data(),
                                               sv.data(), sr.data(), cfg, g.data());
      double norm = 0.0;
      for (double x : g) norm += x * x;
      norm = std::sqrt(norm);
      if (cfg.max_grad_norm > 0.0 && norm > cfg.max_grad_norm)
        for (double& x : g) x *= cfg.max_grad_norm / norm;
      adam.step(params, g.data());
      st.loss += info.total;
      st.surrogate += info.surrogate;
      st.value_loss += info.value_loss;
      st.entropy = info.entropy;
      ++count;
    }
  }
  if (count > 0) {
    st.loss /= count;
    st.surrogate /= count;
    st.value_loss /= count;
  }
  return st;
}

}  // namespace oracle
