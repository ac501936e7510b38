// rmpc_env.cu — the closed-loop step after the batched solve on sm_100a (SURVEY.md §8(f) rows
// 1-2): the simulator's physics_step (/root/reference/proj/src/env.cpp:38-68), the control
// epilogue mpc_torque + blend (mpc.cpp:340-344, policy.cpp:133-157) fused in front of it, and
// observe (policy.cpp:104-122).  One thread per agent, FP64 (the simulator integrates its state
// over whole episodes); device-resident arrays, asynchronous on the caller's stream.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <cstring>
#include <new>
#include <vector>

#include "../../include/rmpc_b200_env.h"
#include "rmpc_device.cuh"
#include "rmpc_kin.cuh"

namespace rmpc_env_dev {

using rmpc_dev::contact_jac;
using rmpc_dev::fk_frames;
using rmpc_dev::Frames;
using rmpc_dev::kchain;
constexpr int NQ = 9, NJ = 6, NC = 4;

struct Geo {  // the field names fk_frames expects
  double torso_len, thigh_len, shank_len, foot_half, ankle_drop;
};

struct EnvParams {
  Geo geo;
  double m_link[7], I_link[7];  // base model (scaled per agent by rmpc_body.mass_scale)
  double mu, gravity;
  double kp[NJ], kd[NJ], tau_limit[NJ];
  double nominal[NQ];
  double control_dt;
  int substeps, n_heights;
  double k_n, c_n, v_slip, extent, cell;
  const double* heights;  // device, n_heights (0: flat)
};

// Terrain::height_at (env.cpp:17-27): smoothstep value noise, clamped at the ends.
__device__ __forceinline__ double height_at(const EnvParams& E, double x) {
  if (E.n_heights == 0) return 0.0;
  const double fx = (x + 0.5 * E.extent) / E.cell;
  const int n = E.n_heights;
  if (fx <= 0.0) return __ldg(E.heights);
  if (fx >= n - 1) return __ldg(E.heights + n - 1);
  const int i = (int)fx;
  const double t = fx - i;
  const double s = t * t * (3.0 - 2.0 * t);
  return __ldg(E.heights + i) * (1.0 - s) + __ldg(E.heights + i + 1) * s;
}

__device__ __forceinline__ double wrap01(double x) {
  const double w = fmod(x, 1.0);
  return w < 0.0 ? w + 1.0 : w;
}

// One control period of physics_step: `substeps` semi-implicit Euler steps of
// M qdd = tau - h + sum_c J_c^T (fx, fz) (LLT), then advance_phase.  Returns RMPC_SIM_*.
__device__ int physics(const EnvParams& E, double mu, double mscale, rmpc_state& s, rmpc_gait& g,
                       const double tau[NJ]) {
  const double dt = E.control_dt / E.substeps;
  bool ok = true;
#pragma unroll 1
  for (int sub = 0; sub < E.substeps; ++sub) {
    Frames F;
    fk_frames(E.geo, s.q, s.qd, F, s.q[0]);  // absolute x, as the terrain lookup needs
    double L[NQ * (NQ + 1) / 2];     // lower triangle of M, row-major, then its Cholesky factor
    double gen[NQ];
#pragma unroll
    for (int k = 0; k < NQ * (NQ + 1) / 2; ++k) L[k] = 0.0;
#pragma unroll
    for (int k = 0; k < NQ; ++k) gen[k] = 0.0;
    // M = sum_l m_l J_l^T J_l + I_l w_l w_l^T, h = sum_l m_l J_l^T (Jdot_l qd + g)
    // (robot.cpp:169-195); gen = -h first
#pragma unroll
    for (int l = 0; l < 7; ++l) {
      double Jx[NQ], Jz[NQ];
      bool inc[NQ];
#pragma unroll
      for (int k = 0; k < NQ; ++k) {
        Jx[k] = Jz[k] = 0.0;
        inc[k] = false;
      }
      Jx[0] = 1.0;
      Jz[1] = 1.0;
      double ax = 0.0, az = 0.0;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int a = kchain(l, c);
        if (a >= 0) {
          Jx[a] = -(F.com[l].pz - F.piv[a].pz);
          Jz[a] = F.com[l].px - F.piv[a].px;
          ax += s.qd[a] * (-(F.com[l].vz - F.piv[a].vz));
          az += s.qd[a] * (F.com[l].vx - F.piv[a].vx);
          inc[a] = true;
        }
      }
      const double m = E.m_link[l] * mscale, I = E.I_link[l] * mscale;
#pragma unroll
      for (int i = 0; i < NQ; ++i) {
#pragma unroll
        for (int j = 0; j <= i; ++j) {
          L[i * (i + 1) / 2 + j] += m * (Jx[i] * Jx[j] + Jz[i] * Jz[j]);
          if (inc[i] && inc[j]) L[i * (i + 1) / 2 + j] += I;
        }
        gen[i] -= m * (Jx[i] * ax + Jz[i] * (az + E.gravity));
      }
    }
#pragma unroll
    for (int j = 0; j < NJ; ++j) gen[3 + j] += tau[j];
    // penalty contacts (env.cpp:49-56)
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const double ground = height_at(E, F.con[c].px);
      const double pen = ground - F.con[c].pz;
      if (pen > 0.0) {
        const double fz = fmax(0.0, E.k_n * pen - E.c_n * F.con[c].vz);
        const double fx = -mu * fz * tanh(F.con[c].vx / E.v_slip);
        double Jx[NQ], Jz[NQ];
        contact_jac(F, c, Jx, Jz);
#pragma unroll
        for (int i = 0; i < NQ; ++i) gen[i] += Jx[i] * fx + Jz[i] * fz;
      }
    }
    // M.llt().solve(gen): Cholesky in place, then L y = gen, L^T qdd = y
#pragma unroll
    for (int j = 0; j < NQ; ++j) {
      double d = L[j * (j + 1) / 2 + j];
#pragma unroll
      for (int k = 0; k < j; ++k) d -= L[j * (j + 1) / 2 + k] * L[j * (j + 1) / 2 + k];
      ok = ok && d > 0.0;
      const double ljj = sqrt(d);
      L[j * (j + 1) / 2 + j] = ljj;
#pragma unroll
      for (int i = j + 1; i < NQ; ++i) {
        double v = L[i * (i + 1) / 2 + j];
#pragma unroll
        for (int k = 0; k < j; ++k) v -= L[i * (i + 1) / 2 + k] * L[j * (j + 1) / 2 + k];
        L[i * (i + 1) / 2 + j] = v / ljj;
      }
    }
#pragma unroll
    for (int i = 0; i < NQ; ++i) {
      double v = gen[i];
#pragma unroll
      for (int k = 0; k < i; ++k) v -= L[i * (i + 1) / 2 + k] * gen[k];
      gen[i] = v / L[i * (i + 1) / 2 + i];
    }
#pragma unroll
    for (int i = NQ - 1; i >= 0; --i) {
      double v = gen[i];
#pragma unroll
      for (int k = i + 1; k < NQ; ++k) v -= L[k * (k + 1) / 2 + i] * gen[k];
      gen[i] = v / L[i * (i + 1) / 2 + i];
    }
#pragma unroll
    for (int i = 0; i < NQ; ++i) s.qd[i] += dt * gen[i];
#pragma unroll
    for (int i = 0; i < NQ; ++i) s.q[i] += dt * s.qd[i];
  }
#pragma unroll
  for (int i = 0; i < NQ; ++i) ok = ok && isfinite(s.q[i]) && isfinite(s.qd[i]);
  g.phase = wrap01(g.phase + E.control_dt / g.period);  // advance_phase (gait.cpp:31-35)
  return ok ? RMPC_SIM_OK : RMPC_SIM_BLOWUP;
}

__device__ __forceinline__ double clampd(double v, double lim) { return fmin(fmax(v, -lim), lim); }

// Trainer::train's control for one env (ppo.cpp:340-349): zero torque for a failed solution,
// else blend(mpc_torque(sol, state), ...) (policy.cpp:133-157, robot.cpp:235-241).
__device__ void control_torque(const EnvParams& E, const rmpc_solution& sol, const double* action,
                               int strategy, double lambda, const rmpc_state& s, double tau[NJ]) {
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    const double qs = sol.q_set[j], qds = sol.qd_set[j], tff = sol.tau_ff[j];
    const double a = action ? action[j] : 0.0;
    const double q = s.q[3 + j], qd = s.qd[3 + j];
    const double tmpc = clampd(E.kp[j] * (qs - q) + E.kd[j] * (qds - qd) + tff, E.tau_limit[j]);
    double t;
    if (strategy == RMPC_BLEND_JOINT_JOINT) {
      t = clampd(E.kp[j] * ((qs + lambda * a) - q) + E.kd[j] * (qds - qd) + tff, E.tau_limit[j]);
    } else if (strategy == RMPC_BLEND_JOINT_TORQUE) {
      const double res = E.kp[j] * (a + E.nominal[3 + j] - q) - E.kd[j] * qd;
      t = clampd(tmpc + lambda * res, E.tau_limit[j]);
    } else {
      t = clampd(tmpc + lambda * a, E.tau_limit[j]);
    }
    tau[j] = sol.status == RMPC_STATUS_OK ? t : 0.0;
  }
}

__global__ void __launch_bounds__(128) physics_kernel(const EnvParams E, int n, rmpc_state* states,
                                                      rmpc_gait* gaits, const rmpc_body* bodies,
                                                      const double* tau, int32_t* status) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= n) return;
  rmpc_state s = states[a];
  rmpc_gait g = gaits[a];
  const double mu = bodies ? bodies[a].mu : E.mu, ms = bodies ? bodies[a].mass_scale : 1.0;
  double t[NJ];
#pragma unroll
  for (int j = 0; j < NJ; ++j) t[j] = tau[NJ * a + j];
  const int st = physics(E, mu, ms, s, g, t);
  states[a] = s;
  gaits[a] = g;
  if (status) status[a] = st;
}

__global__ void __launch_bounds__(128) control_kernel(const EnvParams E, int n, const rmpc_solution* sols,
                                                      const double* action, int strategy, double lambda,
                                                      rmpc_state* states, rmpc_gait* gaits,
                                                      const rmpc_body* bodies, double* tau_out,
                                                      int32_t* status) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= n) return;
  rmpc_state s = states[a];
  rmpc_gait g = gaits[a];
  const rmpc_solution sol = sols[a];
  double t[NJ];
  control_torque(E, sol, action ? action + NJ * a : nullptr, strategy, lambda, s, t);
  if (tau_out)
#pragma unroll
    for (int j = 0; j < NJ; ++j) tau_out[NJ * a + j] = t[j];
  const double mu = bodies ? bodies[a].mu : E.mu, ms = bodies ? bodies[a].mass_scale : 1.0;
  const int st = physics(E, mu, ms, s, g, t);
  states[a] = s;
  gaits[a] = g;
  if (status) status[a] = st;
}

__global__ void __launch_bounds__(128) observe_kernel(int n, const rmpc_state* states, const rmpc_gait* gaits,
                                                      const rmpc_solution* sols, double scale,
                                                      double sentinel, double* obs) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= n) return;
  const rmpc_state& s = states[a];
  const rmpc_gait& g = gaits[a];
  double* o = obs + (size_t)RMPC_OBS_DIM * a;
  constexpr double kTwoPi = 6.283185307179586476925286766559;
  o[0] = s.q[1];
  o[1] = sin(s.q[2]);
  o[2] = cos(s.q[2]);
#pragma unroll
  for (int j = 0; j < NJ; ++j) o[3 + j] = s.q[3 + j];
  o[9] = s.qd[0];
  o[10] = s.qd[1];
  o[11] = s.qd[2];
#pragma unroll
  for (int j = 0; j < NJ; ++j) o[12 + j] = s.qd[3 + j];
  const double pr = wrap01(g.phase + g.offsets[0]), pl = wrap01(g.phase + g.offsets[2]);
  o[18] = sin(kTwoPi * pr);
  o[19] = cos(kTwoPi * pr);
  o[20] = sin(kTwoPi * pl);
  o[21] = cos(kTwoPi * pl);
  o[22] = sols[a].status == RMPC_STATUS_OK ? scale * (double)sols[a].v_mpc : sentinel;
}

__global__ void __launch_bounds__(128) plan_feedback_kernel(int n, int T, const float* z, const rmpc_solution* sols,
                                                            rmpc_state* states, rmpc_gait* gaits, double dt) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= n) return;
  if (sols[a].status == RMPC_STATUS_OK && T > 1) {
    const float* z1 = z + ((size_t)a * T + 1) * 26;
#pragma unroll
    for (int k = 0; k < NQ; ++k) {
      states[a].q[k] = (double)z1[k];
      states[a].qd[k] = (double)z1[NQ + k];
    }
  }
  gaits[a].phase = wrap01(gaits[a].phase + dt / gaits[a].period);
}

// xoshiro256++ stream Rng(seed, stream) (rng.hpp:15-41), for the heightfield draw.
struct HostRng {
  uint64_t s[4];
  static uint64_t splitmix(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
  }
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  HostRng(uint64_t seed, uint64_t stream) {
    uint64_t x = seed ^ splitmix(stream + 0x9e3779b97f4a7c15ULL);
    for (auto& w : s) {
      x += 0x9e3779b97f4a7c15ULL;
      w = splitmix(x);
    }
  }
  uint64_t next() {
    const uint64_t r = rotl(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return r;
  }
  double uniform(double lo, double hi) {
    return lo + (hi - lo) * (static_cast<double>(next() >> 11) * 0x1.0p-53);
  }
};

}  // namespace rmpc_env_dev

struct rmpc_env {
  int device = 0;
  rmpc_env_dev::EnvParams P{};
  std::vector<double> heights;  // host copy (Terrain::heights_)
  double* d_heights = nullptr;
};

extern "C" {

void rmpc_env_config_default(rmpc_env_config* c) {
  if (!c) return;
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

int32_t rmpc_env_create(const rmpc_model* m, const rmpc_env_config* cfg, int32_t device, rmpc_env** out) {
  if (!m || !cfg || !out) return RMPC_ERR_INVALID_ARG;
  *out = nullptr;
  if (cfg->substeps < 1 || !(cfg->control_dt > 0.0) || (cfg->terrain_kind == 1 && !(cfg->cell > 0.0)))
    return RMPC_ERR_STRUCTURAL;
  if (cudaSetDevice(device) != cudaSuccess) return RMPC_ERR_CUDA;
  rmpc_env* e = new (std::nothrow) rmpc_env;
  if (!e) return RMPC_ERR_CUDA;
  e->device = device;
  rmpc_env_dev::EnvParams& P = e->P;
  P.geo = {m->torso_len, m->thigh_len, m->shank_len, m->foot_half_len, m->ankle_drop};
  const double ml[7] = {m->torso_mass, m->thigh_mass, m->shank_mass, m->foot_mass,
                        m->thigh_mass, m->shank_mass, m->foot_mass};
  const double il[7] = {m->torso_inertia, m->thigh_inertia, m->shank_inertia, m->foot_inertia,
                        m->thigh_inertia, m->shank_inertia, m->foot_inertia};
  for (int l = 0; l < 7; ++l) {
    P.m_link[l] = ml[l];
    P.I_link[l] = il[l];
  }
  P.mu = m->mu;
  P.gravity = m->gravity;
  for (int j = 0; j < 6; ++j) {
    P.kp[j] = m->kp[j];
    P.kd[j] = m->kd[j];
    P.tau_limit[j] = m->tau_limit[j];
  }
  rmpc_nominal_pose(m, P.nominal);  // randomize_model scales every mass alike: same pose
  P.control_dt = cfg->control_dt;
  P.substeps = cfg->substeps;
  P.k_n = cfg->k_n;
  P.c_n = cfg->c_n;
  P.v_slip = cfg->v_slip;
  P.extent = cfg->extent;
  P.cell = cfg->cell;
  P.n_heights = 0;
  P.heights = nullptr;
  if (cfg->terrain_kind == 1) {  // Terrain::Terrain (env.cpp:8-15)
    const int n = static_cast<int>(cfg->extent / cfg->cell) + 2;
    e->heights.resize(n);
    rmpc_env_dev::HostRng rng(cfg->terrain_seed, 0x7e22);
    for (double& h : e->heights) h = rng.uniform(-cfg->amplitude, cfg->amplitude);
    if (cudaMalloc(&e->d_heights, n * sizeof(double)) != cudaSuccess ||
        cudaMemcpy(e->d_heights, e->heights.data(), n * sizeof(double), cudaMemcpyHostToDevice) !=
            cudaSuccess) {
      cudaFree(e->d_heights);
      delete e;
      return RMPC_ERR_CUDA;
    }
    P.n_heights = n;
    P.heights = e->d_heights;
  }
  *out = e;
  return RMPC_OK;
}

void rmpc_env_destroy(rmpc_env* e) {
  if (!e) return;
  if (e->d_heights) {
    cudaSetDevice(e->device);
    cudaFree(e->d_heights);
  }
  delete e;
}

int32_t rmpc_env_height_at(const rmpc_env* e, double x, double* h) {
  if (!e || !h) return RMPC_ERR_INVALID_ARG;
  const auto& H = e->heights;
  if (H.empty()) {
    *h = 0.0;
    return RMPC_OK;
  }
  const double fx = (x + 0.5 * e->P.extent) / e->P.cell;
  const int n = static_cast<int>(H.size());
  if (fx <= 0.0) {
    *h = H.front();
  } else if (fx >= n - 1) {
    *h = H.back();
  } else {
    const int i = static_cast<int>(fx);
    const double t = fx - i, s = t * t * (3.0 - 2.0 * t);
    *h = H[i] * (1.0 - s) + H[i + 1] * s;
  }
  return RMPC_OK;
}

static cudaStream_t env_stream(void* s) { return s ? (cudaStream_t)s : cudaStreamLegacy; }

int32_t rmpc_physics_step_device(rmpc_env* e, int32_t n, rmpc_state* states, rmpc_gait* gaits,
                                 const rmpc_body* bodies, const double* tau, int32_t* status, void* stream) {
  if (!e || n < 0 || (n > 0 && (!states || !gaits || !tau))) return RMPC_ERR_INVALID_ARG;
  if (n == 0) return RMPC_OK;
  if (cudaSetDevice(e->device) != cudaSuccess) return RMPC_ERR_CUDA;
  rmpc_env_dev::physics_kernel<<<(n + 127) / 128, 128, 0, env_stream(stream)>>>(e->P, n, states, gaits, bodies,
                                                                               tau, status);
  return cudaGetLastError() == cudaSuccess ? RMPC_OK : RMPC_ERR_CUDA;
}

int32_t rmpc_control_step_device(rmpc_env* e, int32_t n, const rmpc_solution* sols, const double* action,
                                 int32_t strategy, double lambda, rmpc_state* states, rmpc_gait* gaits,
                                 const rmpc_body* bodies, double* tau_out, int32_t* status, void* stream) {
  if (!e || n < 0 || (n > 0 && (!sols || !states || !gaits))) return RMPC_ERR_INVALID_ARG;
  if (strategy < RMPC_BLEND_JOINT_JOINT || strategy > RMPC_BLEND_TORQUE_TORQUE) return RMPC_ERR_STRUCTURAL;
  if (n == 0) return RMPC_OK;
  if (cudaSetDevice(e->device) != cudaSuccess) return RMPC_ERR_CUDA;
  rmpc_env_dev::control_kernel<<<(n + 127) / 128, 128, 0, env_stream(stream)>>>(
      e->P, n, sols, action, strategy, lambda, states, gaits, bodies, tau_out, status);
  return cudaGetLastError() == cudaSuccess ? RMPC_OK : RMPC_ERR_CUDA;
}

int32_t rmpc_observe_device(int32_t n, const rmpc_state* states, const rmpc_gait* gaits,
                            const rmpc_solution* sols, double scale, double sentinel, double* obs,
                            void* stream) {
  if (n < 0 || (n > 0 && (!states || !gaits || !sols || !obs))) return RMPC_ERR_INVALID_ARG;
  if (n == 0) return RMPC_OK;
  rmpc_env_dev::observe_kernel<<<(n + 127) / 128, 128, 0, env_stream(stream)>>>(n, states, gaits, sols, scale,
                                                                               sentinel, obs);
  return cudaGetLastError() == cudaSuccess ? RMPC_OK : RMPC_ERR_CUDA;
}

int32_t rmpc_plan_feedback_device(int32_t n, int32_t horizon, const float* z, const rmpc_solution* sols,
                                  rmpc_state* states, rmpc_gait* gaits, double dt, void* stream) {
  if (n < 0 || horizon < 1 || (n > 0 && (!z || !sols || !states || !gaits))) return RMPC_ERR_INVALID_ARG;
  if (n == 0) return RMPC_OK;
  rmpc_env_dev::plan_feedback_kernel<<<(n + 127) / 128, 128, 0, env_stream(stream)>>>(n, horizon, z, sols, states,
                                                                                     gaits, dt);
  return cudaGetLastError() == cudaSuccess ? RMPC_OK : RMPC_ERR_CUDA;
}

int32_t rmpc_env_sizeof(int32_t which) {
  switch (which) {
    case 0: return (int32_t)sizeof(rmpc_env_config);
    case 1: return (int32_t)sizeof(rmpc_body);
    case 2: return (int32_t)sizeof(rmpc_ppo_config);
    case 3: return (int32_t)sizeof(rmpc_ppo_loss_info);
    case 4: return (int32_t)sizeof(rmpc_ppo_update_stats);
    default: return -1;
  }
}

}  // extern "C"
