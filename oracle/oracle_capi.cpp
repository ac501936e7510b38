// oracle_capi.cpp — TEST INFRASTRUCTURE ONLY (see rmpc_oracle.hpp).
// extern "C" surface of the CPU oracle, loaded by tests/ (ctypes) and by bench.py's
// cpu_baseline / --impl reference arm.  Never linked into the product library.
#include <atomic>
#include <chrono>
#include <thread>

#include "rmpc_oracle.hpp"
#include "rmpc_oracle_env.hpp"
#include "rmpc_oracle_ppo.hpp"
#include "rmpc_oracle_rng.hpp"
#include "oracle_flops.hpp"
#include "oracle_abi.h"

using namespace oracle;

extern "C" {


void oracle_model_default(rmpc_model* m) { model_default(m); }
void oracle_settings_default(rmpc_settings* s, int32_t horizon) { settings_default(s, horizon); }
void oracle_nominal_pose(const rmpc_model* m, double* q) { nominal_pose(*m, q); }
int32_t oracle_sizeof_solution(void) { return (int32_t)sizeof(oracle_solution); }

static void fill(const Solution& s, oracle_solution* o) {
  for (int j = 0; j < 6; ++j) { o->tau_ff[j] = s.tau_ff[j]; o->q_set[j] = s.q_set[j]; o->qd_set[j] = s.qd_set[j]; }
  for (int k = 0; k < 8; ++k) o->f0[k] = s.f0[k];
  for (int b = 0; b < 3; ++b) o->base_residual[b] = s.base_res[b];
  o->v_mpc = s.v_mpc; o->prim_res = s.prim_res; o->dual_res = s.dual_res; o->delta_inf_norm = s.delta_inf;
  o->v_quad = s.v_quad; o->v_lin = s.v_lin;
  o->status = s.status; o->fail_iter = s.fail_iter;
  o->n_vars = s.n; o->n_cons = s.m; o->ldl_nnz = s.ldl_nnz; o->pad = 0;
}

// BatchRunner::solve restated (batch.cpp:26-79): an atomic-cursor std::thread pool over whole
// agents; element i is identical whatever the worker count.  precision: 64 (parity oracle)
// or 32 (FP32 probe).  prev_z [n][T][26] and prev_ok [n] are read only when warm_start.
// stage_ms (7, may be NULL) receives the per-stage mean per agent; wall_ms the tick time.
int32_t oracle_solve_batch(const rmpc_model* model, const rmpc_settings* st, int32_t n,
                           const rmpc_state* states, const rmpc_command* cmds, const rmpc_gait* gaits,
                           const double* prev_z, const int32_t* prev_ok, int32_t workers,
                           int32_t precision, oracle_solution* out, double* z_out,
                           double* stage_ms, double* wall_ms) {
  if (n < 1 || st->horizon < 2 || st->horizon > RMPC_MAX_HORIZON) return RMPC_ERR_STRUCTURAL;
  double nominal[kNq];
  nominal_pose(*model, nominal);
  const int T = st->horizon;
  const bool timed = stage_ms != nullptr;
  std::vector<std::array<double, kNumStages>> stage((size_t)n);
  auto solve_one = [&](int i) {
    const double* pz = prev_z ? prev_z + (size_t)i * T * kNv : nullptr;
    const bool ok = prev_ok ? prev_ok[i] == RMPC_STATUS_OK : false;
    Solution s = precision == 32
                     ? rti_step<float>(*model, *st, nominal, states[i], cmds[i], gaits[i], pz, ok, timed)
                     : rti_step<double>(*model, *st, nominal, states[i], cmds[i], gaits[i], pz, ok, timed);
    fill(s, &out[i]);
    if (z_out) {
      double* zo = z_out + (size_t)i * T * kNv;
      for (int k = 0; k < T * kNv; ++k) zo[k] = s.z_star.empty() ? 0.0 : s.z_star[k];
    }
    for (int k = 0; k < kNumStages; ++k) stage[i][k] = s.stage_s[k];
  };
  const auto t0 = std::chrono::steady_clock::now();
  int nw = workers > 0 ? workers : (int)std::thread::hardware_concurrency();
  nw = std::max(1, std::min(nw, (int)n));
  if (nw == 1) {
    for (int i = 0; i < n; ++i) solve_one(i);
  } else {
    std::atomic<int> cursor{0};
    std::vector<std::thread> pool;
    for (int w = 0; w < nw; ++w)
      pool.emplace_back([&]() {
        for (;;) {
          const int i = cursor.fetch_add(1);
          if (i >= n) break;
          solve_one(i);
        }
      });
    for (auto& t : pool) t.join();
  }
  if (wall_ms)
    *wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  if (stage_ms)
    for (int k = 0; k < kNumStages; ++k) {
      double acc = 0.0;
      for (int i = 0; i < n; ++i) acc += stage[i][k];
      stage_ms[k] = acc * 1e3 / n;
    }
  return RMPC_OK;
}

// Exact operation counts of one rti_step (FP64 reference algorithm), per stage:
// by_stage[7] = flops (add+mul+div+sqrt+trig); ops[6] = totals {add, mul, div, sqrt, trig, cmp}.
int32_t oracle_flops(const rmpc_model* model, const rmpc_settings* st, const rmpc_state* state,
                     const rmpc_command* cmd, const rmpc_gait* gait, double* by_stage, double* ops) {
  double nominal[kNq];
  nominal_pose(*model, nominal);
  for (auto& c : g_ops) c = OpCount{};
  const Solution s = rti_step<Cd>(*model, *st, nominal, *state, *cmd, *gait, nullptr, false, false);
  OpCount tot;
  for (int k = 0; k < kNumStages; ++k) {
    if (by_stage) by_stage[k] = (double)g_ops[k].flops();
    tot.add += g_ops[k].add; tot.mul += g_ops[k].mul; tot.div += g_ops[k].div;
    tot.sqrt += g_ops[k].sqrt; tot.trig += g_ops[k].trig; tot.cmp += g_ops[k].cmp;
  }
  if (ops) {
    ops[0] = (double)tot.add; ops[1] = (double)tot.mul; ops[2] = (double)tot.div;
    ops[3] = (double)tot.sqrt; ops[4] = (double)tot.trig; ops[5] = (double)tot.cmp;
  }
  return s.status;
}

void oracle_rng_uniform(uint64_t seed, uint64_t stream, int32_t n, double* out) {
  Rng r(seed, stream);
  for (int i = 0; i < n; ++i) out[i] = r.uniform();
}

// ---------------------------------------------------------------- model-level functions
void oracle_kinematics(const rmpc_model* m, const double* q, const double* qd, double* com_pos,
                       double* com_vel, double* com_jac, double* com_jdq, double* c_pos,
                       double* c_vel, double* c_jac) {
  const Kin<double> k = kinematics<double>(*m, q, qd);
  for (int l = 0; l < 7; ++l) {
    com_pos[2 * l] = k.com[l].px; com_pos[2 * l + 1] = k.com[l].pz;
    com_vel[2 * l] = k.com[l].vx; com_vel[2 * l + 1] = k.com[l].vz;
    com_jdq[2 * l] = k.com_jdq[l][0]; com_jdq[2 * l + 1] = k.com_jdq[l][1];
    for (int r = 0; r < 2; ++r)
      for (int c = 0; c < kNq; ++c) com_jac[(l * 2 + r) * kNq + c] = k.com_jac[l][r][c];
  }
  for (int c = 0; c < kNc; ++c) {
    c_pos[2 * c] = k.c[c].px; c_pos[2 * c + 1] = k.c[c].pz;
    c_vel[2 * c] = k.c[c].vx; c_vel[2 * c + 1] = k.c[c].vz;
    for (int r = 0; r < 2; ++r)
      for (int j = 0; j < kNq; ++j) c_jac[(c * 2 + r) * kNq + j] = k.c_jac[c][r][j];
  }
}

void oracle_mass_matrix(const rmpc_model* m, const double* q, double* M) {
  double zero[kNq] = {0};
  const Kin<double> k = kinematics<double>(*m, q, zero);
  double Mm[kNq][kNq];
  mass_matrix(*m, k, Mm);
  for (int i = 0; i < kNq; ++i)
    for (int j = 0; j < kNq; ++j) M[i * kNq + j] = Mm[i][j];
}

void oracle_bias_forces(const rmpc_model* m, const double* q, const double* qd, double* h) {
  const Kin<double> k = kinematics<double>(*m, q, qd);
  bias_forces(*m, k, h);
}

void oracle_inverse_dynamics(const rmpc_model* m, const double* q, const double* qd,
                             const double* qdd, const double* F, double* tau, double* base) {
  inverse_dynamics<double>(*m, q, qd, qdd, F, tau, base);
}

void oracle_pd_torque(const rmpc_model* m, const double* q_des, const double* qd_des,
                      const double* q, const double* qd, const double* tau_ff, double* out) {
  pd_torque(*m, q_des, qd_des, q, qd, tau_ff, out);
}

double oracle_bezier(double t, double z_swing, double v_to, double v_td, double* vel) {
  return bezier_swing(t, z_swing, v_to, v_td, vel);
}

void oracle_horizon_schedule(const rmpc_gait* g, const double* dt, int32_t T, int32_t* stance,
                             double* swing_t) {
  std::vector<std::array<bool, kNc>> s(T);
  std::vector<std::array<double, kNc>> t(T);
  horizon_schedule(*g, dt, T, s.data(), t.data());
  for (int i = 0; i < T; ++i)
    for (int c = 0; c < kNc; ++c) { stance[i * kNc + c] = s[i][c]; swing_t[i * kNc + c] = t[i][c]; }
}

void oracle_desired_trajectory(const rmpc_model* m, const rmpc_settings* st, const rmpc_command* cmd,
                               const rmpc_gait* g, double* q_des, double* qd_des, double* F_des,
                               double* swing_h) {
  double nominal[kNq];
  nominal_pose(*m, nominal);
  const Reference r = desired_trajectory(*cmd, *g, *st, *m, nominal);
  const int T = st->horizon;
  for (int i = 0; i < T * kNq; ++i) { q_des[i] = r.q_des[i]; qd_des[i] = r.qd_des[i]; }
  for (int i = 0; i < T * kNf; ++i) F_des[i] = r.F_des[i];
  for (int i = 0; i < T; ++i)
    for (int c = 0; c < kNc; ++c) swing_h[i * kNc + c] = r.swing_height[i][c];
}

// build_qp at a guess: guess_z [T][26] (NULL = the cold guess of rti_step).  Returns
// n, m, nnz(A) and, when the buffers are non-NULL, the dense A (m x n, row-major), P diag,
// q, lo, hi.  Status RMPC_STATUS_NONFINITE_INPUT if build_qp throws.
int32_t oracle_build_qp(const rmpc_model* m, const rmpc_settings* st, const rmpc_state* state,
                        const rmpc_command* cmd, const rmpc_gait* g, const double* guess_z,
                        int32_t* n_out, int32_t* m_out, int32_t* nnz_out, double* A_dense,
                        double* P_diag, double* q_lin, double* lo, double* hi) {
  double nominal[kNq];
  nominal_pose(*m, nominal);
  const int T = st->horizon;
  Traj<double> guess;
  guess.resize(T);
  std::vector<std::array<bool, kNc>> stance(T);
  std::vector<std::array<double, kNc>> swt(T);
  horizon_schedule(*g, st->dt_schedule, T, stance.data(), swt.data());
  const double weight = total_mass(*m) * m->gravity;
  for (int i = 0; i < T; ++i) {
    if (guess_z) {
      for (int k = 0; k < kNq; ++k) {
        guess.q[i * kNq + k] = guess_z[i * kNv + k];
        guess.qd[i * kNq + k] = guess_z[i * kNv + kNq + k];
      }
      for (int k = 0; k < kNf; ++k) guess.F[i * kNf + k] = guess_z[i * kNv + 2 * kNq + k];
    } else {
      for (int k = 0; k < kNq; ++k) guess.q[i * kNq + k] = nominal[k];
      guess.q[i * kNq] = state->q[0];
      const int na = n_active(stance[i]);
      for (int c = 0; c < kNc; ++c)
        guess.F[i * kNf + 2 * c + 1] = (stance[i][c] && na > 0) ? weight / na : 0.0;
    }
  }
  try {
    const Reference ref = desired_trajectory(*cmd, *g, *st, *m, nominal);
    const Qp<double> qp = build_qp<double>(*state, guess, ref, *st, *m);
    *n_out = qp.n();
    *m_out = qp.m();
    *nnz_out = qp.A.nnz();
    if (A_dense) {
      std::fill(A_dense, A_dense + (size_t)qp.m() * qp.n(), 0.0);
      for (int j = 0; j < qp.n(); ++j)
        for (int p = qp.A.colptr[j]; p < qp.A.colptr[j + 1]; ++p)
          A_dense[(size_t)qp.A.rowidx[p] * qp.n() + j] = qp.A.val[p];
    }
    if (P_diag)
      for (int j = 0; j < qp.n(); ++j) {
        P_diag[j] = 0.0;
        for (int p = qp.P.colptr[j]; p < qp.P.colptr[j + 1]; ++p)
          if (qp.P.rowidx[p] == j) P_diag[j] = qp.P.val[p];
      }
    if (q_lin) for (int j = 0; j < qp.n(); ++j) q_lin[j] = qp.q[j];
    if (lo) for (int i = 0; i < qp.m(); ++i) lo[i] = qp.lo[i];
    if (hi) for (int i = 0; i < qp.m(); ++i) hi[i] = qp.hi[i];
    return RMPC_STATUS_OK;
  } catch (const std::exception&) {
    return RMPC_STATUS_NONFINITE_INPUT;
  }
}

// ---------------------------------------------------------------- generic QP / linalg
static Csc<double> dense_to_csc(int nr, int nc, const double* a, bool upper) {
  std::vector<Trip<double>> ts;
  for (int j = 0; j < nc; ++j)
    for (int i = 0; i < (upper ? j + 1 : nr); ++i) {
      const double v = a[(size_t)i * nc + j];
      if (v != 0.0 || (upper && i == j)) ts.push_back({i, j, v});
    }
  return csc_from_triplets(ts, nr, nc);
}

int32_t oracle_csc_from_triplets(int32_t nt, const int32_t* rows, const int32_t* cols,
                                 const double* vals, int32_t nr, int32_t nc, int32_t* colptr,
                                 int32_t* rowidx, double* v_out, int32_t* nnz) {
  std::vector<Trip<double>> ts(nt);
  for (int k = 0; k < nt; ++k) ts[k] = {rows[k], cols[k], vals[k]};
  try {
    const Csc<double> a = csc_from_triplets(ts, nr, nc);
    for (int j = 0; j <= nc; ++j) colptr[j] = a.colptr[j];
    for (int p = 0; p < a.nnz(); ++p) { rowidx[p] = a.rowidx[p]; v_out[p] = a.val[p]; }
    *nnz = a.nnz();
    return RMPC_OK;
  } catch (const StructuralError&) {
    return RMPC_ERR_STRUCTURAL;
  }
}

// Ruiz on a dense symmetric matrix given by its upper triangle (structural pattern = non-zero
// upper entries + diagonal).  K is overwritten with the scaled upper triangle.
int32_t oracle_ruiz_dense(int32_t n, double* K, int32_t passes, double* scale) {
  Csc<double> a = dense_to_csc(n, n, K, true);
  try {
    const std::vector<double> s = ruiz_equilibrate(a, passes);
    for (int i = 0; i < n; ++i) scale[i] = s[i];
  } catch (const StructuralError&) {
    return RMPC_ERR_STRUCTURAL;
  }
  for (int j = 0; j < n; ++j)
    for (int p = a.colptr[j]; p < a.colptr[j + 1]; ++p) K[(size_t)a.rowidx[p] * n + j] = a.val[p];
  return RMPC_OK;
}

// LDL^T of a dense symmetric (upper-read) matrix.  perm[n], D[n], L dense (n x n, unit
// lower, in permuted order), lnnz = strictly-lower nnz.  Error text into err.
int32_t oracle_ldl_dense(int32_t n, const double* K, int32_t use_ordering, int32_t* perm,
                         double* D, double* L, int32_t* lnnz, char* err, int32_t errlen) {
  try {
    const Ldl<double> f(dense_to_csc(n, n, K, true), use_ordering != 0);
    for (int k = 0; k < n; ++k) { perm[k] = f.perm[k]; D[k] = f.D[k]; }
    std::fill(L, L + (size_t)n * n, 0.0);
    for (int k = 0; k < n; ++k) {
      L[(size_t)k * n + k] = 1.0;
      for (int p = f.Lp[k]; p < f.Lp[k + 1]; ++p) L[(size_t)f.Li[p] * n + k] = f.Lx[p];
    }
    *lnnz = f.Lp[n];
    return RMPC_OK;
  } catch (const std::exception& e) {
    if (err && errlen > 0) { std::strncpy(err, e.what(), errlen - 1); err[errlen - 1] = 0; }
    return dynamic_cast<const SingularityError*>(&e) ? 3 : RMPC_ERR_STRUCTURAL;
  }
}

int32_t oracle_ldl_solve_dense(int32_t n, const double* K, int32_t use_ordering, const double* b,
                               double* x) {
  try {
    const Ldl<double> f(dense_to_csc(n, n, K, true), use_ordering != 0);
    std::vector<double> v(b, b + n), w;
    f.solve_inplace(v, w);
    for (int i = 0; i < n; ++i) x[i] = v[i];
    return RMPC_OK;
  } catch (const std::exception&) {
    return RMPC_ERR_STRUCTURAL;
  }
}

// admm_solve on a dense QP (P symmetric n x n, A m x n row-major).  info[4] = {prim, dual,
// objective, iters_run}.  Returns 0, or RMPC_STATUS_DIVERGED with *fail_iter.
int32_t oracle_admm_dense(int32_t n, int32_t m, const double* P, const double* q, const double* A,
                          const double* lo, const double* hi, double sigma, double rho,
                          double alpha, int32_t iters, int32_t ruiz_iters, double eps_exit,
                          const double* x0, const double* y0, double* x, double* y, double* z,
                          double* info, int32_t* fail_iter) {
  Qp<double> qp;
  qp.P = dense_to_csc(n, n, P, true);
  qp.A = dense_to_csc(m, n, A, false);
  qp.q.assign(q, q + n);
  qp.lo.assign(lo, lo + m);
  qp.hi.assign(hi, hi + m);
  AdmmSettings st;
  st.sigma = sigma; st.rho = rho; st.alpha = alpha; st.iters = iters;
  st.ruiz_iters = ruiz_iters; st.eps_exit = eps_exit;
  std::vector<double> vx0, vy0;
  if (x0 && y0) { vx0.assign(x0, x0 + n); vy0.assign(y0, y0 + m); }
  try {
    const QpResult<double> r = admm_solve<double>(qp, st, x0 ? &vx0 : nullptr, y0 ? &vy0 : nullptr);
    for (int i = 0; i < n; ++i) x[i] = r.x[i];
    for (int i = 0; i < m; ++i) { y[i] = r.y[i]; z[i] = r.z[i]; }
    info[0] = r.prim; info[1] = r.dual; info[2] = r.obj; info[3] = r.iters_run;
    *fail_iter = -1;
    return RMPC_OK;
  } catch (const DivergenceError& e) {
    *fail_iter = e.iteration;
    return RMPC_STATUS_DIVERGED;
  } catch (const std::exception&) {
    return RMPC_ERR_STRUCTURAL;
  }
}

// ---------------------------------------------------------------- closed-loop step (env.cpp)
void oracle_env_config_default(rmpc_env_config* c) { env_config_default(c); }

double oracle_terrain_height_at(const rmpc_env_config* c, double x) { return Terrain(*c).height_at(x); }

void oracle_physics_step_batch(const rmpc_model* base, const rmpc_env_config* cfg, int32_t n,
                               rmpc_state* states, rmpc_gait* gaits, const rmpc_body* bodies,
                               const double* tau, int32_t* status) {
  const Terrain ter(*cfg);
  for (int a = 0; a < n; ++a) {
    const rmpc_model m = randomized(*base, bodies ? bodies + a : nullptr);
    status[a] = physics_step(m, *cfg, ter, states[a], gaits[a], tau + 6 * a);
  }
}

void oracle_control_step_batch(const rmpc_model* base, const rmpc_env_config* cfg, int32_t n,
                               const rmpc_solution* sols, const double* action, int32_t strategy,
                               double lambda, rmpc_state* states, rmpc_gait* gaits,
                               const rmpc_body* bodies, double* tau_out, int32_t* status) {
  const Terrain ter(*cfg);
  for (int a = 0; a < n; ++a) {
    const rmpc_model m = randomized(*base, bodies ? bodies + a : nullptr);
    status[a] = control_step(m, *cfg, ter, sols[a], action ? action + 6 * a : nullptr, strategy,
                             lambda, states[a], gaits[a], tau_out + 6 * a);
  }
}

void oracle_observe_batch(int32_t n, const rmpc_state* states, const rmpc_gait* gaits,
                          const rmpc_solution* sols, double scale, double sentinel, double* obs) {
  for (int a = 0; a < n; ++a) observe(states[a], gaits[a], sols[a], scale, sentinel, obs + RMPC_OBS_DIM * a);
}

int32_t oracle_init_policy(int32_t obs, int32_t act, int32_t hidden, uint64_t seed, int32_t zero_final,
                           double* out, int32_t cap) {
  const std::vector<double> p = init_policy_flat(obs, act, hidden, seed, zero_final != 0);
  if (out && cap >= (int32_t)p.size()) std::copy(p.begin(), p.end(), out);
  return (int32_t)p.size();
}

void oracle_policy_forward_batch(const double* params, int32_t obs, int32_t act, int32_t hidden, int32_t n,
                                 const double* o, double* mean, double* value) {
  for (int a = 0; a < n; ++a)
    policy_forward_flat(params, obs, act, hidden, o + (size_t)obs * a, mean + (size_t)act * a, value + a);
}

// ppo_loss (ppo.cpp:79-135); grads (num_params) is zeroed here and may be null.
void oracle_ppo_loss(const double* params, int32_t obs, int32_t act, int32_t hidden, int32_t n, const double* o,
                     const double* a, const double* old_logp, const double* adv, const double* ret,
                     const rmpc_ppo_config* cfg, double* grads, int32_t n_params, rmpc_ppo_loss_info* info) {
  if (grads) std::fill(grads, grads + n_params, 0.0);
  *info = ppo_loss(params, obs, act, hidden, n, o, a, old_logp, adv, ret, *cfg, grads);
}

void oracle_gae(int32_t T, int32_t E, const double* rew, const double* val, const double* done, const double* boot,
                double gamma, double lam, double* adv, double* ret) {
  gae(T, E, rew, val, done, boot, gamma, lam, adv, ret);
}

// ppo_update (ppo.cpp:193-276) with the Adam state (m, v, t) and the update Rng words carried
// by the caller across calls.
void oracle_ppo_update(double* params, int32_t obs, int32_t act, int32_t hidden, int32_t T, int32_t E,
                       const double* o, const double* a, const double* logp, const double* values,
                       const double* rewards, const double* dones, const double* boot, const rmpc_ppo_config* cfg,
                       double* adam_m, double* adam_v, int32_t* adam_t, int32_t n_params, uint64_t rng_state[4],
                       rmpc_ppo_update_stats* stats) {
  Adam adam(n_params, cfg->lr);
  std::copy(adam_m, adam_m + n_params, adam.m.begin());
  std::copy(adam_v, adam_v + n_params, adam.v.begin());
  adam.t = *adam_t;
  Rng rng(0, 0);
  for (int k = 0; k < 4; ++k) rng.s[k] = rng_state[k];
  *stats = ppo_update(params, obs, act, hidden, T, E, o, a, logp, values, rewards, dones, boot, *cfg, adam, rng);
  std::copy(adam.m.begin(), adam.m.end(), adam_m);
  std::copy(adam.v.begin(), adam.v.end(), adam_v);
  *adam_t = adam.t;
  for (int k = 0; k < 4; ++k) rng_state[k] = rng.s[k];
}

void oracle_ppo_config_default(rmpc_ppo_config* c) { ppo_config_default(c); }

// Active set of the final ADMM iterate per agent on the device's (node + 1, slot) grid:
// act (n x (T+1) x 40 int8), margin (same shape, FP64, scaled space).  Cold start.
int32_t oracle_active_set_batch(const rmpc_model* model, const rmpc_settings* st, int32_t n,
                                const rmpc_state* states, const rmpc_command* cmds, const rmpc_gait* gaits,
                                int32_t workers, int8_t* act, double* margin) {
  if (n < 1 || st->horizon < 2 || st->horizon > RMPC_MAX_HORIZON) return RMPC_ERR_STRUCTURAL;
  double nominal[kNq];
  nominal_pose(*model, nominal);
  const size_t W = (size_t)(st->horizon + 1) * 40;
  std::atomic<int> cursor{0};
  auto work = [&]() {
    for (;;) {
      const int i = cursor.fetch_add(1);
      if (i >= n) break;
      const Solution s = rti_step<double>(*model, *st, nominal, states[i], cmds[i], gaits[i], nullptr, false, false);
      for (size_t k = 0; k < W; ++k) {
        act[i * W + k] = s.act.empty() ? 3 : s.act[k];
        margin[i * W + k] = s.act_margin.empty() ? 0.0 : s.act_margin[k];
      }
    }
  };
  const int nw = std::max(1, std::min(workers > 0 ? workers : (int)std::thread::hardware_concurrency(), (int)n));
  std::vector<std::thread> pool;
  for (int w = 0; w < nw; ++w) pool.emplace_back(work);
  for (auto& t : pool) t.join();
  return 0;
}

}  // extern "C"
