// ref_capi.cpp — TEST INFRASTRUCTURE ONLY.
// extern "C" surface over the UNMODIFIED reference sources (/root/reference/proj/src/*.cpp,
// compiled against the Eigen-subset shim in eigen_shim/, see Makefile.ref).  It converts the
// repo's plain-C ABI records (include/rmpc_b200.h, rmpc_b200_env.h) to the reference's types,
// calls the reference's own functions and converts back.  tests/ use it to pin the restated
// oracle (oracle_capi.cpp) and the CUDA path to numbers the reference code produces; bench.py's
// `--impl reference` arm times ref_solve_batch (the reference's BatchRunner) on the host cores.
// Nothing here is linked into the product library.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../include/rmpc_b200.h"
#include "../include/rmpc_b200_env.h"
#include "oracle_abi.h"
#include "rmpc/batch.hpp"
#include "rmpc/env.hpp"
#include "rmpc/gait.hpp"
#include "rmpc/mpc.hpp"
#include "rmpc/policy.hpp"
#include "rmpc/ppo.hpp"
#include "rmpc/robot.hpp"

namespace {

using namespace rmpc;

ModelParams to_model(const rmpc_model& m) {
  ModelParams p;
  p.torso_mass = m.torso_mass; p.torso_len = m.torso_len; p.torso_inertia = m.torso_inertia;
  p.thigh_mass = m.thigh_mass; p.thigh_len = m.thigh_len; p.thigh_inertia = m.thigh_inertia;
  p.shank_mass = m.shank_mass; p.shank_len = m.shank_len; p.shank_inertia = m.shank_inertia;
  p.foot_mass = m.foot_mass; p.foot_half_len = m.foot_half_len; p.foot_inertia = m.foot_inertia;
  p.ankle_drop = m.ankle_drop;
  for (int j = 0; j < kNumJoints; ++j) {
    p.joint_lo[j] = m.joint_lo[j]; p.joint_hi[j] = m.joint_hi[j];
    p.qd_limit[j] = m.qd_limit[j]; p.tau_limit[j] = m.tau_limit[j];
    p.kp[j] = m.kp[j]; p.kd[j] = m.kd[j];
  }
  p.mu = m.mu;
  p.gravity = m.gravity;
  p.nominal_stagger = m.nominal_stagger;
  p.nominal_drop = m.nominal_drop;
  return p;
}

MpcSettings to_settings(const rmpc_settings& s) {
  MpcSettings o;
  o.horizon = s.horizon;
  o.dt_schedule.assign(s.dt_schedule, s.dt_schedule + s.horizon);
  for (int k = 0; k < kNq; ++k) { o.w_q[k] = s.w_q[k]; o.w_qd[k] = s.w_qd[k]; }
  for (int k = 0; k < kContactDim; ++k) o.w_f[k] = s.w_f[k];
  o.gait_period = s.gait_period;
  o.phase_switch = s.phase_switch;
  for (int c = 0; c < kNumContacts; ++c) o.phase_offsets[c] = s.phase_offsets[c];
  o.z_swing = s.z_swing; o.v_to = s.v_to; o.v_td = s.v_td;
  o.n_qp = s.n_qp; o.mu = s.mu; o.sigma = s.sigma; o.rho = s.rho; o.over_relax = s.over_relax;
  o.warm_start = s.warm_start != 0;
  return o;
}

RobotState to_state(const rmpc_state& s) {
  RobotState r;
  for (int k = 0; k < kNq; ++k) { r.q[k] = s.q[k]; r.qd[k] = s.qd[k]; }
  return r;
}
void from_state(const RobotState& r, rmpc_state& s) {
  for (int k = 0; k < kNq; ++k) { s.q[k] = r.q[k]; s.qd[k] = r.qd[k]; }
}
GaitState to_gait(const rmpc_gait& g) {
  GaitState o;
  o.phase = g.phase; o.period = g.period; o.phase_switch = g.phase_switch;
  for (int c = 0; c < kNumContacts; ++c) o.offsets[c] = g.offsets[c];
  return o;
}
void from_gait(const GaitState& o, rmpc_gait& g) {
  g.phase = o.phase; g.period = o.period; g.phase_switch = o.phase_switch;
  for (int c = 0; c < kNumContacts; ++c) g.offsets[c] = o.offsets[c];
}
MpcCommand to_cmd(const rmpc_command& c) {
  MpcCommand o;
  o.height = c.height; o.vx = c.vx; o.wpitch = c.wpitch;
  return o;
}
EnvConfig to_env(const rmpc_env_config& c) {
  EnvConfig e;
  e.control_dt = c.control_dt;
  e.substeps = c.substeps;
  e.k_n = c.k_n; e.c_n = c.c_n; e.v_slip = c.v_slip;
  e.terrain.kind = c.terrain_kind == 1 ? TerrainConfig::Kind::kHeightfield : TerrainConfig::Kind::kFlat;
  e.terrain.amplitude = c.amplitude; e.terrain.cell = c.cell; e.terrain.extent = c.extent;
  e.terrain.seed = c.terrain_seed;
  return e;
}
// randomize_model's draw (env.cpp:188-201) applied from a recorded {mu, mass_scale}
ModelParams with_body(const ModelParams& base, const rmpc_body* b) {
  ModelParams m = base;
  if (!b) return m;
  m.mu = b->mu;
  const double s = b->mass_scale;
  m.torso_mass *= s; m.thigh_mass *= s; m.shank_mass *= s; m.foot_mass *= s;
  m.torso_inertia *= s; m.thigh_inertia *= s; m.shank_inertia *= s; m.foot_inertia *= s;
  return m;
}

// MpcSolution::message -> the repo's per-agent status codes (rmpc_b200.h)
void status_of(const MpcSolution& s, int32_t& status, int32_t& fail_iter) {
  fail_iter = -1;
  if (s.status == MpcStatus::kOk) { status = RMPC_STATUS_OK; return; }
  const std::string& m = s.message;
  if (m.find("non-finite linearization point") != std::string::npos) {
    status = RMPC_STATUS_NONFINITE_INPUT;
  } else if (m.find("zero pivot") != std::string::npos) {
    status = RMPC_STATUS_SINGULAR;
  } else {
    status = RMPC_STATUS_DIVERGED;
    const size_t k = m.find("at iteration ");
    if (k != std::string::npos) fail_iter = std::atoi(m.c_str() + k + 13);
  }
}

PolicyParams policy_from_flat(const double* flat, int obs, int act, int hidden) {
  PolicyParams p = init_policy(obs, act, hidden, 0);  // shapes; values overwritten
  Vec f(p.num_params());
  std::copy(flat, flat + p.num_params(), f.data());
  unflatten_policy(f, p);
  return p;
}

}  // namespace

extern "C" {

int32_t ref_sizeof_solution(void) { return (int32_t)sizeof(oracle_solution); }

void ref_nominal_pose(const rmpc_model* m, double* q) {
  const Vec9 n = nominal_pose(to_model(*m));
  for (int k = 0; k < kNq; ++k) q[k] = n[k];
}

// rmpc::BatchRunner(n, model, settings, workers).solve(states, cmds, gaits, prev) -- the
// reference's own batch runtime and rti_step (batch.cpp:26-79, mpc.cpp:248-338).  prev_z
// [n][T][26] / prev_ok [n] build the `prev` solutions (read only with warm_start).
// stage_mean_ms / stage_std_ms (7 each, may be NULL) are last_timing()'s per-stage statistics
// over agents; wall_ms its total_ms.  Returns RMPC_ERR_STRUCTURAL on a StructuralError.
int32_t ref_solve_batch(const rmpc_model* model, const rmpc_settings* st, int32_t n,
                        const rmpc_state* states, const rmpc_command* cmds, const rmpc_gait* gaits,
                        const double* prev_z, const int32_t* prev_ok, int32_t workers,
                        oracle_solution* out, double* z_out, double* stage_mean_ms,
                        double* stage_std_ms, double* wall_ms) {
  try {
    const ModelParams mp = to_model(*model);
    const MpcSettings ms = to_settings(*st);
    const int T = st->horizon;
    std::vector<RobotState> S(n);
    std::vector<MpcCommand> Cm(n);
    std::vector<GaitState> G(n);
    for (int i = 0; i < n; ++i) { S[i] = to_state(states[i]); Cm[i] = to_cmd(cmds[i]); G[i] = to_gait(gaits[i]); }
    std::vector<MpcSolution> prev;
    if (prev_z) {
      prev.resize(n);
      for (int i = 0; i < n; ++i) {
        prev[i].status = (prev_ok && prev_ok[i] == RMPC_STATUS_OK) ? MpcStatus::kOk : MpcStatus::kFailed;
        prev[i].z_star.resize(T);
        const double* z = prev_z + (size_t)i * T * 26;
        for (int t = 0; t < T; ++t) {
          for (int k = 0; k < kNq; ++k) {
            prev[i].z_star.q(t, k) = z[t * 26 + k];
            prev[i].z_star.qd(t, k) = z[t * 26 + kNq + k];
          }
          for (int k = 0; k < kContactDim; ++k) prev[i].z_star.F(t, k) = z[t * 26 + 2 * kNq + k];
        }
      }
    }
    BatchRunner runner(n, mp, ms, workers);
    const std::vector<MpcSolution> sol = runner.solve(S, Cm, G, prev_z ? &prev : nullptr);
    for (int i = 0; i < n; ++i) {
      const MpcSolution& s = sol[i];
      oracle_solution& o = out[i];
      std::memset(&o, 0, sizeof(o));
      for (int j = 0; j < kNumJoints; ++j) { o.tau_ff[j] = s.tau_ff[j]; o.q_set[j] = s.q_set[j]; o.qd_set[j] = s.qd_set[j]; }
      const bool have_z = s.z_star.F.rows() == T;
      for (int k = 0; k < kContactDim; ++k) o.f0[k] = have_z ? s.z_star.F(0, k) : 0.0;
      for (int b = 0; b < 3; ++b) o.base_residual[b] = s.base_residual[b];
      o.v_mpc = s.v_mpc; o.prim_res = s.prim_res; o.dual_res = s.dual_res; o.delta_inf_norm = s.delta_inf_norm;
      o.v_quad = o.v_lin = std::nan("");
      status_of(s, o.status, o.fail_iter);
      if (z_out) {
        double* z = z_out + (size_t)i * T * 26;
        for (int t = 0; t < T; ++t) {
          for (int k = 0; k < kNq; ++k) {
            z[t * 26 + k] = have_z ? s.z_star.q(t, k) : 0.0;
            z[t * 26 + kNq + k] = have_z ? s.z_star.qd(t, k) : 0.0;
          }
          for (int k = 0; k < kContactDim; ++k) z[t * 26 + 2 * kNq + k] = have_z ? s.z_star.F(t, k) : 0.0;
        }
      }
    }
    const TimingReport& tr = runner.last_timing();
    for (int k = 0; k < kNumStages; ++k) {
      if (stage_mean_ms) stage_mean_ms[k] = tr.mean_ms[k];
      if (stage_std_ms) stage_std_ms[k] = tr.std_ms[k];
    }
    if (wall_ms) *wall_ms = tr.total_ms;
    return RMPC_OK;
  } catch (const StructuralError&) {
    return RMPC_ERR_STRUCTURAL;
  }
}

// build_qp at the cold guess of rti_step (mpc.cpp:266-276, 64-238): sizes, nnz(A) and, when
// the buffers are non-NULL, dense A (m x n row-major), diag P, q, lo, hi (kInf = 1e30 kept).
int32_t ref_build_qp(const rmpc_model* m, const rmpc_settings* st, const rmpc_state* state,
                     const rmpc_command* cmd, const rmpc_gait* g, int32_t* n_out, int32_t* m_out,
                     int32_t* nnz_out, double* A_dense, double* P_diag, double* q_lin, double* lo,
                     double* hi) {
  const ModelParams mp = to_model(*m);
  const MpcSettings ms = to_settings(*st);
  const RobotState rs = to_state(*state);
  const GaitState gs = to_gait(*g);
  const int T = ms.horizon;
  DecisionTrajectory guess;
  guess.resize(T);
  const auto stance = horizon_contact_flags(gs, ms.dt_schedule);
  const double weight = mp.total_mass() * mp.gravity;
  const Vec9 nominal = nominal_pose(mp);
  for (int i = 0; i < T; ++i) {
    guess.q.row(i) = nominal.transpose();
    guess.q(i, 0) = rs.q[0];
    int na = 0;
    for (bool s : stance[i]) na += s ? 1 : 0;
    for (int c = 0; c < kNumContacts; ++c) guess.F(i, 2 * c + 1) = (stance[i][c] && na > 0) ? weight / na : 0.0;
  }
  try {
    const MpcReference ref = desired_trajectory(rs, to_cmd(*cmd), gs, ms, mp);
    const QpProblem qp = build_qp(rs, guess, ref, ms, mp);
    const int n = qp.num_vars(), mm = qp.num_cons();
    *n_out = n;
    *m_out = mm;
    *nnz_out = qp.A.nnz();
    if (A_dense) {
      std::fill(A_dense, A_dense + (size_t)mm * n, 0.0);
      for (int j = 0; j < n; ++j)
        for (int p = qp.A.col_ptr[j]; p < qp.A.col_ptr[j + 1]; ++p) A_dense[(size_t)qp.A.row_idx[p] * n + j] = qp.A.values[p];
    }
    if (P_diag)
      for (int j = 0; j < n; ++j) {
        P_diag[j] = 0.0;
        for (int p = qp.P.col_ptr[j]; p < qp.P.col_ptr[j + 1]; ++p)
          if (qp.P.row_idx[p] == j) P_diag[j] = qp.P.values[p];
      }
    if (q_lin) for (int j = 0; j < n; ++j) q_lin[j] = qp.q_lin[j];
    if (lo) for (int i = 0; i < mm; ++i) lo[i] = qp.lo[i];
    if (hi) for (int i = 0; i < mm; ++i) hi[i] = qp.hi[i];
    return RMPC_STATUS_OK;
  } catch (const std::exception&) {
    return RMPC_STATUS_NONFINITE_INPUT;
  }
}

void ref_mass_matrix(const rmpc_model* m, const double* q, double* M) {
  Vec9 qq;
  for (int k = 0; k < kNq; ++k) qq[k] = q[k];
  const Mat99 Mm = mass_matrix(to_model(*m), qq);
  for (int i = 0; i < kNq; ++i)
    for (int j = 0; j < kNq; ++j) M[i * kNq + j] = Mm(i, j);
}

void ref_bias_forces(const rmpc_model* m, const double* q, const double* qd, double* h) {
  Vec9 qq, vv;
  for (int k = 0; k < kNq; ++k) { qq[k] = q[k]; vv[k] = qd[k]; }
  const Vec9 hh = bias_forces(to_model(*m), qq, vv);
  for (int k = 0; k < kNq; ++k) h[k] = hh[k];
}

void ref_inverse_dynamics(const rmpc_model* m, const double* q, const double* qd, const double* qdd,
                          const double* F, double* tau, double* base) {
  Vec9 qq, vv, aa;
  Eigen::Matrix<double, kContactDim, 1> f;
  for (int k = 0; k < kNq; ++k) { qq[k] = q[k]; vv[k] = qd[k]; aa[k] = qdd[k]; }
  for (int k = 0; k < kContactDim; ++k) f[k] = F[k];
  const InverseDynamicsResult r = inverse_dynamics_torque(to_model(*m), qq, vv, aa, f);
  for (int j = 0; j < kNumJoints; ++j) tau[j] = r.tau[j];
  for (int b = 0; b < 3; ++b) base[b] = r.base_residual[b];
}

// ---------------------------------------------------------------- env.cpp / policy.cpp / ppo.cpp
double ref_terrain_height_at(const rmpc_env_config* c, double x) { return Terrain(to_env(*c).terrain).height_at(x); }

// physics_step (env.cpp:38-68) per agent with its randomized body; states / gaits in place;
// status 1 on SimBlowupError.
void ref_physics_step_batch(const rmpc_model* base, const rmpc_env_config* cfg, int32_t n, rmpc_state* states,
                            rmpc_gait* gaits, const rmpc_body* bodies, const double* tau, int32_t* status) {
  const EnvConfig ec = to_env(*cfg);
  const Terrain ter(ec.terrain);
  const ModelParams mb = to_model(*base);
  for (int a = 0; a < n; ++a) {
    EnvState es;
    es.robot = to_state(states[a]);
    es.gait = to_gait(gaits[a]);
    Vec6 t;
    for (int j = 0; j < kNumJoints; ++j) t[j] = tau[6 * a + j];
    try {
      const EnvState nx = physics_step(es, t, ec, with_body(mb, bodies ? bodies + a : nullptr), ter);
      from_state(nx.robot, states[a]);
      from_gait(nx.gait, gaits[a]);
      status[a] = 0;
    } catch (const SimBlowupError&) {
      status[a] = 1;
    }
  }
}

// Trainer::train's per-env control (ppo.cpp:340-349): zero torque for a failed solution, else
// blend(mpc_torque(sol, state, env model), ...), then physics_step.  Solutions are the repo's
// FP32 records (the fields blend and mpc_torque read).
void ref_control_step_batch(const rmpc_model* base, const rmpc_env_config* cfg, int32_t n, const rmpc_solution* sols,
                            const double* action, int32_t strategy, double lambda, rmpc_state* states,
                            rmpc_gait* gaits, const rmpc_body* bodies, double* tau_out, int32_t* status) {
  const EnvConfig ec = to_env(*cfg);
  const Terrain ter(ec.terrain);
  const ModelParams mb = to_model(*base);
  for (int a = 0; a < n; ++a) {
    const ModelParams m = with_body(mb, bodies ? bodies + a : nullptr);
    EnvState es;
    es.robot = to_state(states[a]);
    es.gait = to_gait(gaits[a]);
    MpcSolution s;
    s.status = sols[a].status == RMPC_STATUS_OK ? MpcStatus::kOk : MpcStatus::kFailed;
    for (int j = 0; j < kNumJoints; ++j) {
      s.tau_ff[j] = sols[a].tau_ff[j]; s.q_set[j] = sols[a].q_set[j]; s.qd_set[j] = sols[a].qd_set[j];
    }
    Vec6 act = Vec6::Zero();
    if (action)
      for (int j = 0; j < kNumJoints; ++j) act[j] = action[6 * a + j];
    Vec6 tau = Vec6::Zero();
    if (s.status == MpcStatus::kOk) {
      const Vec6 tau_mpc = mpc_torque(s, es.robot, m);
      tau = blend(tau_mpc, s.tau_ff, s.q_set, s.qd_set, act, es.robot, static_cast<BlendStrategy>(strategy), lambda, m);
    }
    for (int j = 0; j < kNumJoints; ++j) tau_out[6 * a + j] = tau[j];
    try {
      const EnvState nx = physics_step(es, tau, ec, m, ter);
      from_state(nx.robot, states[a]);
      from_gait(nx.gait, gaits[a]);
      status[a] = 0;
    } catch (const SimBlowupError&) {
      status[a] = 1;
    }
  }
}

void ref_observe_batch(int32_t n, const rmpc_state* states, const rmpc_gait* gaits, const rmpc_solution* sols,
                       double scale, double sentinel, double* obs) {
  ObsSettings os;
  os.v_mpc_scale = scale;
  os.v_mpc_sentinel = sentinel;
  for (int a = 0; a < n; ++a) {
    EnvState es;
    es.robot = to_state(states[a]);
    es.gait = to_gait(gaits[a]);
    MpcSolution s;
    s.status = sols[a].status == RMPC_STATUS_OK ? MpcStatus::kOk : MpcStatus::kFailed;
    s.v_mpc = sols[a].v_mpc;
    const Vec o = observe(es, s, os);
    for (int k = 0; k < kObsDim; ++k) obs[(size_t)a * kObsDim + k] = o[k];
  }
}

// init_policy (policy.cpp:57-83) flattened in flatten_policy order (ppo.cpp:144-152).
int32_t ref_init_policy(int32_t obs, int32_t act, int32_t hidden, uint64_t seed, double* out, int32_t cap) {
  const PolicyParams p = init_policy(obs, act, hidden, seed);
  const Vec f = flatten_policy(p);
  if (out && cap >= (int32_t)f.size()) std::copy(f.data(), f.data() + f.size(), out);
  return (int32_t)f.size();
}

void ref_policy_forward_batch(const double* params, int32_t obs, int32_t act, int32_t hidden, int32_t n,
                              const double* o, double* mean, double* value) {
  const PolicyParams p = policy_from_flat(params, obs, act, hidden);
  for (int a = 0; a < n; ++a) {
    Vec x(obs);
    for (int k = 0; k < obs; ++k) x[k] = o[(size_t)a * obs + k];
    const PolicyOutput y = policy_forward(p, x);
    for (int j = 0; j < act; ++j) mean[(size_t)a * act + j] = y.mean[j];
    value[a] = y.value;
  }
}

static PpoConfig to_ppo(const rmpc_ppo_config& c) {
  PpoConfig p;
  p.gamma = c.gamma; p.lam_gae = c.lam_gae; p.clip_eps = c.clip_eps;
  p.epochs = c.epochs; p.minibatches = c.minibatches;
  p.lr = c.lr; p.entropy_coef = c.entropy_coef; p.value_coef = c.value_coef; p.max_grad_norm = c.max_grad_norm;
  return p;
}

// ppo_loss (ppo.cpp:79-135): loss terms and (grads != NULL) flatten_grads of the gradient.
void ref_ppo_loss(const double* params, int32_t obs, int32_t act, int32_t hidden, int32_t n, const double* o,
                  const double* a, const double* old_logp, const double* adv, const double* ret,
                  const rmpc_ppo_config* cfg, double* grads, rmpc_ppo_loss_info* info) {
  const PolicyParams p = policy_from_flat(params, obs, act, hidden);
  PpoBatch b;
  b.obs.resize(n, obs);
  b.actions.resize(n, act);
  b.old_logp.resize(n);
  b.advantages.resize(n);
  b.returns.resize(n);
  for (int s = 0; s < n; ++s) {
    for (int k = 0; k < obs; ++k) b.obs(s, k) = o[(size_t)s * obs + k];
    for (int k = 0; k < act; ++k) b.actions(s, k) = a[(size_t)s * act + k];
    b.old_logp[s] = old_logp[s];
    b.advantages[s] = adv[s];
    b.returns[s] = ret[s];
  }
  PolicyGrads g = zero_grads(p);
  const PpoLossInfo li = ppo_loss(p, b, to_ppo(*cfg), grads ? &g : nullptr);
  info->total = li.total; info->surrogate = li.surrogate; info->value_loss = li.value_loss; info->entropy = li.entropy;
  if (grads) {
    const Vec f = flatten_grads(g);
    std::copy(f.data(), f.data() + f.size(), grads);
  }
}

void ref_gae(int32_t T, int32_t E, const double* rew, const double* val, const double* done, const double* boot,
             double gamma, double lam, double* adv, double* ret) {
  RolloutBuffer b;
  b.resize(T, E, 1, 1);
  for (int t = 0; t < T; ++t)
    for (int e = 0; e < E; ++e) {
      b.rewards(t, e) = rew[t * E + e];
      b.values(t, e) = val[t * E + e];
      b.dones(t, e) = done[t * E + e];
    }
  for (int e = 0; e < E; ++e) b.bootstrap_value[e] = boot[e];
  const GaeResult r = gae_advantages(b, gamma, lam);
  for (int t = 0; t < T; ++t)
    for (int e = 0; e < E; ++e) { adv[t * E + e] = r.advantages(t, e); ret[t * E + e] = r.returns(t, e); }
}

// n_updates consecutive ppo_update calls (ppo.cpp:195-276) on one rollout with one
// AdamOptimizer(num_params, cfg.lr) and one Rng(seed, stream) carried across them (the
// reference keeps both private); params updated in place, stats of each call in stats[k].
void ref_ppo_update_seq(double* params, int32_t obs, int32_t act, int32_t hidden, int32_t T, int32_t E,
                        const double* o, const double* a, const double* logp, const double* values,
                        const double* rewards, const double* dones, const double* boot, const rmpc_ppo_config* cfg,
                        uint64_t seed, uint64_t stream, int32_t n_updates, rmpc_ppo_update_stats* stats) {
  PolicyParams p = policy_from_flat(params, obs, act, hidden);
  RolloutBuffer b;
  b.resize(T, E, obs, act);
  for (int t = 0; t < T; ++t)
    for (int e = 0; e < E; ++e) {
      const size_t s = (size_t)t * E + e;
      for (int k = 0; k < obs; ++k) b.obs[t](e, k) = o[s * obs + k];
      for (int k = 0; k < act; ++k) b.actions[t](e, k) = a[s * act + k];
      b.logp(t, e) = logp[s];
      b.values(t, e) = values[s];
      b.rewards(t, e) = rewards[s];
      b.dones(t, e) = dones[s];
    }
  for (int e = 0; e < E; ++e) b.bootstrap_value[e] = boot[e];
  const PpoConfig pc = to_ppo(*cfg);
  AdamOptimizer adam(p.num_params(), pc.lr);
  Rng rng(seed, stream);
  for (int k = 0; k < n_updates; ++k) {
    const PpoUpdateStats s = ppo_update(p, b, pc, adam, rng);
    stats[k].loss = s.loss; stats[k].surrogate = s.surrogate; stats[k].value_loss = s.value_loss;
    stats[k].entropy = s.entropy;
  }
  const Vec f = flatten_policy(p);
  std::copy(f.data(), f.data() + f.size(), params);
}

// check_termination (env.cpp:111-140) on a state with the base model: the reason code of
// ref_closed_loop (0 = none).
int32_t ref_check_termination(const rmpc_model* model, const rmpc_env_config* cfg, const rmpc_state* state) {
  EnvState es;
  es.robot = to_state(*state);
  const TerminationCheck t = check_termination(es, to_env(*cfg), to_model(*model));
  if (!t.terminated) return 0;
  const std::string& w = t.reason;
  return w == "height" ? 2 : w == "orientation" ? 3 : w == "velocity" ? 4 : w == "self_collision" ? 5 : 1;
}

// The reference's own closed loop (run_episode without a policy, analysis.cpp:75-149): every
// control tick rti_step on the env state -> mpc_torque (zero torque for a failed solve) ->
// Env::step (physics_step, termination).  The env is the reference's Env with randomisation
// pinned (friction = model mu, mass scale 1, no initial velocity, zero command) and the gait
// of `settings`.  SPEC.md acceptance #4: standing, zero command, 5 s survival.  Writes
// trace[t] = {q[0..8], qd[0..8]} after tick t (ticks x 18) and returns the ticks survived;
// *reason: 0 survived, 1 non_finite / sim_blowup, 2 height, 3 orientation, 4 velocity,
// 5 self_collision, 6 controller_failed.
int32_t ref_closed_loop(const rmpc_model* model, const rmpc_settings* st, const rmpc_env_config* cfg,
                        double phase_switch, int32_t ticks, double* trace, int32_t* reason) {
  const ModelParams mp = to_model(*model);
  MpcSettings ms = to_settings(*st);
  EnvConfig ec = to_env(*cfg);
  ec.friction_lo = ec.friction_hi = mp.mu;
  ec.mass_scale_lo = ec.mass_scale_hi = 1.0;
  ec.init_vx = 0.0;
  ec.init_pitch_rate = 0.0;
  ec.cmd_vx_lo = ec.cmd_vx_hi = 0.0;
  ec.cmd_height_lo = ec.cmd_height_hi = mp.nominal_height();
  ec.gait_period = ms.gait_period;
  ec.phase_switch = phase_switch;
  ec.phase_offsets = ms.phase_offsets;
  ec.episode_length = 1e9;
  Env env(mp, ec, 0, 0);
  MpcController ctrl(mp, ms);
  MpcSolution prev;
  bool have_prev = false;
  *reason = 0;
  for (int t = 0; t < ticks; ++t) {
    const EnvState s = env.state();
    const MpcSolution sol = ctrl.rti_step(s.robot, s.cmd, s.gait, have_prev ? &prev : nullptr);
    const bool failed = sol.status != MpcStatus::kOk;
    const Vec6 tau = failed ? Vec6::Zero() : mpc_torque(sol, s.robot, env.model());
    const EnvState before = env.state();
    const Env::StepResult res = env.step(tau, Vec6::Zero(), failed);
    const RobotState& r = res.done ? before.robot : env.state().robot;  // reset() replaced it
    for (int k = 0; k < kNq; ++k) {
      trace[(size_t)t * 18 + k] = res.done ? std::nan("") : r.q[k];
      trace[(size_t)t * 18 + 9 + k] = res.done ? std::nan("") : r.qd[k];
    }
    if (res.done) {
      const std::string& w = res.reason;
      *reason = w == "height" ? 2 : w == "orientation" ? 3 : w == "velocity" ? 4 : w == "self_collision" ? 5
              : w == "controller_failed" ? 6 : 1;
      return t;
    }
    prev = sol;
    have_prev = true;
  }
  return ticks;
}

}  // extern "C"
