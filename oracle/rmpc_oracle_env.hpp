// rmpc_oracle_env.hpp — TEST INFRASTRUCTURE ONLY: FP64 CPU restatement of the simulator step
// and the control epilogue around the solve, the parity oracle for
// include/rmpc_b200_env.h.  Only tests/ and bench.py's CPU legs may call it.
//
//   Terrain::Terrain / height_at      /root/reference/proj/src/env.cpp:8-27
//   physics_step                      env.cpp:38-68 (compute_kinematics, mass_matrix,
//                                     bias_forces: robot.cpp:29-195; Eigen LLT solve)
//   randomize_model                   env.cpp:196-208
//   advance_phase, contact_phase      gait.cpp:14,31-35
//   mpc_torque, blend, observe        mpc.cpp:340-344, policy.cpp:104-157
//   init_policy, mlp_forward,         policy.cpp:15-31, 40-102 (flatten_into order)
//   policy_forward
#pragma once

#include <cmath>
#include <vector>

#include "../include/rmpc_b200_env.h"
#include "rmpc_oracle.hpp"
#include "rmpc_oracle_rng.hpp"

namespace oracle {

inline void env_config_default(rmpc_env_config* c) {  // env.hpp:16-23, 52-63
  c->control_dt = 0.01;
  c->substeps = 4;
  c->terrain_kind = 0;
  c->k_n = 5e4;
  c->c_n = 500.0;
  c->v_slip = 0.05;
  c->amplitude = 0.04;
  c->cell = 0.3;
  c->extent = 80.0;
  c->terrain_seed = 0;
}

struct Terrain {  // env.cpp:8-27
  rmpc_env_config cfg;
  std::vector<double> heights;
  explicit Terrain(const rmpc_env_config& c) : cfg(c) {
    if (c.terrain_kind == 1) {
      const int n = static_cast<int>(c.extent / c.cell) + 2;
      heights.resize(n);
      Rng rng(c.terrain_seed, 0x7e22);
      for (double& h : heights) h = rng.uniform(-c.amplitude, c.amplitude);
    }
  }
  double height_at(double x) const {
    if (heights.empty()) return 0.0;
    const double fx = (x + 0.5 * cfg.extent) / cfg.cell;
    const int n = static_cast<int>(heights.size());
    if (fx <= 0.0) return heights.front();
    if (fx >= n - 1) return heights.back();
    const int i = static_cast<int>(fx);
    const double t = fx - i;
    const double s = t * t * (3.0 - 2.0 * t);
    return heights[i] * (1.0 - s) + heights[i + 1] * s;
  }
};

inline rmpc_model randomized(const rmpc_model& base, const rmpc_body* b) {  // env.cpp:196-208
  rmpc_model m = base;
  if (!b) return m;
  m.mu = b->mu;
  const double s = b->mass_scale;
  m.torso_mass *= s; m.thigh_mass *= s; m.shank_mass *= s; m.foot_mass *= s;
  m.torso_inertia *= s; m.thigh_inertia *= s; m.shank_inertia *= s; m.foot_inertia *= s;
  return m;
}

// Cholesky M = L L^T (column by column) and the two triangular solves, in place on b.
inline bool llt_solve(double M[kNq][kNq], double b[kNq]) {
  double L[kNq][kNq] = {};
  for (int j = 0; j < kNq; ++j) {
    double d = M[j][j];
    for (int k = 0; k < j; ++k) d -= L[j][k] * L[j][k];
    if (!(d > 0.0)) return false;
    L[j][j] = std::sqrt(d);
    for (int i = j + 1; i < kNq; ++i) {
      double s = M[i][j];
      for (int k = 0; k < j; ++k) s -= L[i][k] * L[j][k];
      L[i][j] = s / L[j][j];
    }
  }
  for (int i = 0; i < kNq; ++i) {
    double s = b[i];
    for (int k = 0; k < i; ++k) s -= L[i][k] * b[k];
    b[i] = s / L[i][i];
  }
  for (int i = kNq - 1; i >= 0; --i) {
    double s = b[i];
    for (int k = i + 1; k < kNq; ++k) s -= L[k][i] * b[k];
    b[i] = s / L[i][i];
  }
  return true;
}

// physics_step (env.cpp:38-68) + advance_phase (gait.cpp:31-35).  Returns RMPC_SIM_*.
inline int physics_step(const rmpc_model& m, const rmpc_env_config& cfg, const Terrain& ter,
                        rmpc_state& s, rmpc_gait& g, const double tau[kNj]) {
  const double dt = cfg.control_dt / cfg.substeps;
  double* q = s.q;
  double* qd = s.qd;
  bool ok = true;
  for (int sub = 0; sub < cfg.substeps; ++sub) {
    const Kin<double> k = kinematics<double>(m, q, qd);
    double M[kNq][kNq], h[kNq], gen[kNq];
    mass_matrix(m, k, M);
    bias_forces(m, k, h);
    for (int i = 0; i < kNq; ++i) gen[i] = -h[i];
    for (int j = 0; j < kNj; ++j) gen[3 + j] += tau[j];
    for (int c = 0; c < kNc; ++c) {
      const double ground = ter.height_at(k.c[c].px);
      const double pen = ground - k.c[c].pz;
      if (pen <= 0.0) continue;
      const double fz = std::max(0.0, cfg.k_n * pen - cfg.c_n * k.c[c].vz);
      const double fx = -m.mu * fz * std::tanh(k.c[c].vx / cfg.v_slip);
      for (int i = 0; i < kNq; ++i) gen[i] += k.c_jac[c][0][i] * fx + k.c_jac[c][1][i] * fz;
    }
    if (!llt_solve(M, gen)) ok = false;
    for (int i = 0; i < kNq; ++i) qd[i] += dt * gen[i];
    for (int i = 0; i < kNq; ++i) q[i] += dt * qd[i];
  }
  for (int i = 0; i < kNq; ++i) ok = ok && std::isfinite(q[i]) && std::isfinite(qd[i]);
  g.phase = wrap01(g.phase + cfg.control_dt / g.period);
  return ok ? RMPC_SIM_OK : RMPC_SIM_BLOWUP;
}

// blend (policy.cpp:133-157) of the MPC torque with the policy action.
inline void blend(const rmpc_model& m, const double* tau_mpc, const double* tau_ff,
                  const double* q_set, const double* qd_set, const double* action,
                  const rmpc_state& st, int strategy, double lambda, double out[kNj]) {
  if (strategy == RMPC_BLEND_JOINT_JOINT) {
    double q_cmd[kNj];
    for (int j = 0; j < kNj; ++j) q_cmd[j] = q_set[j] + lambda * action[j];
    pd_torque(m, q_cmd, qd_set, st.q, st.qd, tau_ff, out);
    return;
  }
  double qhat[kNq];
  nominal_pose(m, qhat);
  for (int j = 0; j < kNj; ++j) {
    double t;
    if (strategy == RMPC_BLEND_JOINT_TORQUE) {
      const double res = m.kp[j] * (action[j] + qhat[3 + j] - st.q[3 + j]) - m.kd[j] * st.qd[3 + j];
      t = tau_mpc[j] + lambda * res;
    } else {
      t = tau_mpc[j] + lambda * action[j];
    }
    out[j] = std::min(std::max(t, -m.tau_limit[j]), m.tau_limit[j]);
  }
}

// Trainer::train's per-env control (ppo.cpp:340-349): zero torque for a failed solution,
// else blend(mpc_torque(...)); then Env::step's physics.
inline int control_step(const rmpc_model& m, const rmpc_env_config& cfg, const Terrain& ter,
                        const rmpc_solution& sol, const double* action, int strategy,
                        double lambda, rmpc_state& st, rmpc_gait& g, double tau[kNj]) {
  for (int j = 0; j < kNj; ++j) tau[j] = 0.0;
  if (sol.status == 0) {
    double tff[kNj], qs[kNj], qds[kNj], tm[kNj], zero[kNj] = {};
    for (int j = 0; j < kNj; ++j) {
      tff[j] = sol.tau_ff[j];
      qs[j] = sol.q_set[j];
      qds[j] = sol.qd_set[j];
    }
    pd_torque(m, qs, qds, st.q, st.qd, tff, tm);
    blend(m, tm, tff, qs, qds, action ? action : zero, st, strategy, lambda, tau);
  }
  return physics_step(m, cfg, ter, st, g, tau);
}

// observe (policy.cpp:104-122).
inline void observe(const rmpc_state& st, const rmpc_gait& g, const rmpc_solution& sol,
                    double v_mpc_scale, double sentinel, double o[RMPC_OBS_DIM]) {
  constexpr double kTwoPi = 6.283185307179586476925286766559;
  o[0] = st.q[1];
  o[1] = std::sin(st.q[2]);
  o[2] = std::cos(st.q[2]);
  for (int j = 0; j < kNj; ++j) o[3 + j] = st.q[3 + j];
  o[9] = st.qd[0];
  o[10] = st.qd[1];
  o[11] = st.qd[2];
  for (int j = 0; j < kNj; ++j) o[12 + j] = st.qd[3 + j];
  const double pr = wrap01(g.phase + g.offsets[0]), pl = wrap01(g.phase + g.offsets[2]);
  o[18] = std::sin(kTwoPi * pr);
  o[19] = std::cos(kTwoPi * pr);
  o[20] = std::sin(kTwoPi * pl);
  o[21] = std::cos(kTwoPi * pl);
  o[22] = sol.status == 0 ? v_mpc_scale * (double)sol.v_mpc : sentinel;
}

// init_policy (policy.cpp:57-83) flattened as MlpParams::flatten_into (policy.cpp:40-47): per
// layer W (out x in) column-major, then b; pi, then value, then log_std.  zero_final = the
// reference's zero-initialised last policy layer (tests pass false to exercise it).
inline std::vector<double> init_policy_flat(int obs, int act, int hidden, uint64_t seed, bool zero_final) {
  Rng rng(seed, 0xB0117);
  std::vector<double> out;
  auto build = [&](int out_dim, bool zero_last) {
    const int sizes[5] = {obs, hidden, hidden, hidden, out_dim};
    for (int l = 0; l < 4; ++l) {
      const int rows = sizes[l + 1], cols = sizes[l];
      const double limit = std::sqrt(6.0 / (rows + cols));
      std::vector<double> W(static_cast<size_t>(rows) * cols);
      for (int i = 0; i < rows; ++i)
        for (int j = 0; j < cols; ++j) W[static_cast<size_t>(j) * rows + i] = rng.uniform(-limit, limit);
      if (zero_last && l == 3) std::fill(W.begin(), W.end(), 0.0);
      out.insert(out.end(), W.begin(), W.end());
      out.insert(out.end(), rows, 0.0);
    }
  };
  build(act, zero_final);
  build(1, false);
  out.insert(out.end(), act, std::log(0.5));
  return out;
}

// mlp_forward (policy.cpp:15-31) on a flattened trunk starting at p; returns the end offset.
inline size_t mlp_forward_flat(const double* p, int obs, int hidden, int out_dim, const double* in,
                               double* out) {
  const int sizes[5] = {obs, hidden, hidden, hidden, out_dim};
  std::vector<double> h(in, in + obs), z;
  size_t off = 0;
  for (int l = 0; l < 4; ++l) {
    const int rows = sizes[l + 1], cols = sizes[l];
    const double* W = p + off;
    const double* b = W + static_cast<size_t>(rows) * cols;
    z.assign(rows, 0.0);
    for (int i = 0; i < rows; ++i) {
      double acc = 0.0;
      for (int j = 0; j < cols; ++j) acc += W[static_cast<size_t>(j) * rows + i] * h[j];
      z[i] = acc + b[i];
    }
    off += static_cast<size_t>(rows) * cols + rows;
    if (l < 3)
      for (double& v : z) v = v > 0.0 ? v : std::expm1(v);
    h = z;
  }
  for (int i = 0; i < out_dim; ++i) out[i] = h[i];
  return off;
}

// policy_forward (policy.cpp:85-102) without the cache.
inline void policy_forward_flat(const double* params, int obs, int act, int hidden, const double* o,
                                double* mean, double* value) {
  const size_t off = mlp_forward_flat(params, obs, hidden, act, o, mean);
  mlp_forward_flat(params + off, obs, hidden, 1, o, value);
}

}  // namespace oracle
