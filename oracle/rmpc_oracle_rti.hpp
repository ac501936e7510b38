// rmpc_oracle_rti.hpp — TEST INFRASTRUCTURE ONLY (see rmpc_oracle.hpp).
// MpcController::rti_step restated (/root/reference/proj/src/mpc.cpp:248-338).
#pragma once

#include <chrono>

namespace oracle {

template <class T>
Solution rti_step(const rmpc_model& model, const rmpc_settings& st, const double* nominal,
                  const rmpc_state& state, const rmpc_command& cmd, const rmpc_gait& gait,
                  const double* prev_z, bool prev_ok, bool timed) {
  using Clock = std::chrono::steady_clock;
  Solution sol;
  const int NT = st.horizon;
  auto now = [&]() { return timed ? Clock::now() : Clock::time_point(); };
  auto secs = [&](Clock::time_point t0) {
    return timed ? std::chrono::duration<double>(Clock::now() - t0).count() : 0.0;
  };
  try {
    // f_init (mpc.cpp:255-278)
    g_stage = kInit;
    auto t0 = now();
    std::vector<std::array<bool, kNc>> stance(NT);
    {
      std::vector<std::array<double, kNc>> swing_t(NT);
      horizon_schedule(gait, st.dt_schedule, NT, stance.data(), swing_t.data());
    }
    const double weight = total_mass(model) * model.gravity;
    Traj<T> guess;
    guess.resize(NT);
    if (st.warm_start && prev_z != nullptr && prev_ok) {
      for (int i = 0; i < NT; ++i) {
        const int j = std::min(i + 1, NT - 1);
        for (int k = 0; k < kNq; ++k) {
          guess.q[i * kNq + k] = T(prev_z[j * kNv + k]);
          guess.qd[i * kNq + k] = T(prev_z[j * kNv + kNq + k]);
        }
        for (int k = 0; k < kNf; ++k) guess.F[i * kNf + k] = T(prev_z[j * kNv + 2 * kNq + k]);
      }
    } else {
      for (int i = 0; i < NT; ++i) {
        for (int k = 0; k < kNq; ++k) guess.q[i * kNq + k] = T(nominal[k]);
        guess.q[i * kNq + 0] = T(state.q[0]);
        const int na = n_active(stance[i]);
        for (int c = 0; c < kNc; ++c) {
          guess.F[i * kNf + 2 * c] = T(0.0);
          guess.F[i * kNf + 2 * c + 1] = (stance[i][c] && na > 0) ? T(weight / na) : T(0.0);
        }
      }
    }
    sol.stage_s[kInit] = secs(t0);

    // f_param (mpc.cpp:280-282)
    g_stage = kParam;
    t0 = now();
    const Reference ref = desired_trajectory(cmd, gait, st, model, nominal);
    sol.stage_s[kParam] = secs(t0);

    // f_KKT part 1 (mpc.cpp:284-287)
    g_stage = kKkt;
    t0 = now();
    const Qp<T> qp = build_qp<T>(state, guess, ref, st, model);
    sol.stage_s[kKkt] = secs(t0);
    sol.m = qp.m();
    sol.n = qp.n();

    // equilibrate / assemble / factorize / run (mpc.cpp:289-303); the stages are timed as
    // one block here (admm_solve attributes its FLOPs to the right stage via g_stage).
    AdmmSettings as;
    as.sigma = st.sigma;
    as.rho = st.rho;
    as.alpha = st.over_relax;
    as.iters = st.n_qp;
    as.ruiz_iters = st.ruiz_iters;
    const QpResult<T> r = admm_solve<T>(qp, as, nullptr, nullptr, true, timed ? sol.stage_s : nullptr);
    sol.ldl_nnz = r.ldl_nnz;
    sol.act.assign((size_t)(NT + 1) * 40, 3);
    sol.act_margin.assign((size_t)(NT + 1) * 40, 0.0);
    for (int k = 0; k < qp.m(); ++k) {
      sol.act[qp.tag[k]] = r.act[k];
      sol.act_margin[qp.tag[k]] = (double)r.margin[k];
    }

    // full step + inverse dynamics at node 0 (mpc.cpp:305-330)
    g_stage = kRnea;
    t0 = now();
    for (int i = 0; i < sol.n; ++i)
      if (!std::isfinite((double)r.x[i]))
        throw DivergenceError("rti_step: non-finite QP solution", r.iters_run);
    sol.z_star.assign((size_t)NT * kNv, 0.0);
    std::vector<T> zq((size_t)NT * kNq), zqd((size_t)NT * kNq), zf((size_t)NT * kNf);
    for (int i = 0; i < NT; ++i) {
      for (int k = 0; k < kNq; ++k) {
        zq[i * kNq + k] = guess.q[i * kNq + k] + r.x[i * kNv + k];
        zqd[i * kNq + k] = guess.qd[i * kNq + k] + r.x[i * kNv + kNq + k];
        sol.z_star[i * kNv + k] = (double)zq[i * kNq + k];
        sol.z_star[i * kNv + kNq + k] = (double)zqd[i * kNq + k];
      }
      for (int k = 0; k < kNf; ++k) {
        zf[i * kNf + k] = guess.F[i * kNf + k] + r.x[i * kNv + 2 * kNq + k];
        sol.z_star[i * kNv + 2 * kNq + k] = (double)zf[i * kNf + k];
      }
    }
    T dinf = T(0.0);
    for (int i = 0; i < sol.n; ++i) {
      const T a = abs(r.x[i]);
      if (a > dinf) dinf = a;
    }
    sol.delta_inf = (double)dinf;
    sol.v_mpc = (double)r.obj;
    sol.v_quad = (double)r.obj_quad;
    sol.v_lin = (double)r.obj_lin;
    sol.prim_res = (double)r.prim;
    sol.dual_res = (double)r.dual;
    T qdd[kNq];
    const T dt0 = T(st.dt_schedule[0]);
    for (int k = 0; k < kNq; ++k) qdd[k] = (zqd[kNq + k] - zqd[k]) / dt0;
    T tau[kNj], base[3];
    inverse_dynamics<T>(model, &zq[0], &zqd[0], qdd, &zf[0], tau, base);
    for (int j = 0; j < kNj; ++j) {
      sol.tau_ff[j] = (double)tau[j];
      sol.q_set[j] = (double)zq[3 + j];
      sol.qd_set[j] = (double)zqd[3 + j];
    }
    for (int b = 0; b < 3; ++b) sol.base_res[b] = (double)base[b];
    for (int k = 0; k < kNf; ++k) sol.f0[k] = (double)zf[k];
    sol.stage_s[kRnea] = secs(t0);
    sol.status = RMPC_STATUS_OK;
  } catch (const DivergenceError& e) {
    sol.status = RMPC_STATUS_DIVERGED;
    sol.fail_iter = e.iteration;
    sol.message = e.what();
  } catch (const SingularityError& e) {
    sol.status = RMPC_STATUS_SINGULAR;
    sol.message = e.what();
  } catch (const std::exception& e) {
    sol.status = RMPC_STATUS_NONFINITE_INPUT;
    sol.message = e.what();
  }
  return sol;
}

}  // namespace oracle
