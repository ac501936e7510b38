// rmpc_model.cuh — FP64 model pieces on the device: base-dynamics rows, inverse dynamics, gait schedule, guess and targets.
// Part of the fused solve kernel: included once, in order, by rmpc_kernel.cu.
#pragma once

#include "rmpc_device.cuh"
#include "rmpc_kin.cuh"

namespace rmpc_dev {

#ifndef FULL
#define FULL 0xffffffffu
#endif

// ------------------------------------------------------------------------- FP64 kinematics
// Fr, attach, kchain, Frames, fk_frames, contact_jac: rmpc_kin.cuh (shared with rmpc_env.cu).


// Row b (< 3) of M (robot.cpp:169-178) and h (robot.cpp:184-195): one lane per (node, row).
__device__ void base_dynamics_row(const KParams& P, const double* qd, const Frames& F, int b,
                                  double Mr[9], double& hr) {
  hr = 0.0;
#pragma unroll
  for (int k = 0; k < 9; ++k) Mr[k] = 0.0;
#pragma unroll
  for (int l = 0; l < 7; ++l) {
    double Jx[9], Jz[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) Jx[k] = Jz[k] = 0.0;
    Jx[0] = 1.0;
    Jz[1] = 1.0;
    double ax = 0.0, az = 0.0;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int a = kchain(l, s);
      if (a >= 0) {
        Jx[a] = -(F.com[l].pz - F.piv[a].pz);
        Jz[a] = F.com[l].px - F.piv[a].px;
        ax += qd[a] * (-(F.com[l].vz - F.piv[a].vz));
        az += qd[a] * (F.com[l].vx - F.piv[a].vx);
      }
    }
    const double m = P.m_link[l];
    const double jxb = b == 0 ? Jx[0] : (b == 1 ? Jx[1] : Jx[2]);
    const double jzb = b == 0 ? Jz[0] : (b == 1 ? Jz[1] : Jz[2]);
#pragma unroll
    for (int k = 0; k < 9; ++k) Mr[k] += m * (jxb * Jx[k] + jzb * Jz[k]);
    hr += m * (jxb * ax + jzb * (az + P.gravity));
    if (b == 2) {  // rotational part: coordinate 2 is in every chain
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const int a = kchain(l, s);
        if (a >= 0) Mr[a] += P.I_link[l];
      }
    }
  }
}

// gen = M qdd + h - J^T F (robot.cpp:211-233).
__device__ void inverse_dynamics(const KParams& P, const double* q, const double* qd,
                                 const double* qdd, const double* Fc, double gen[9]) {
  Frames F;
  fk_frames(P, q, qd, F);
#pragma unroll
  for (int k = 0; k < 9; ++k) gen[k] = 0.0;
#pragma unroll
  for (int l = 0; l < 7; ++l) {
    double Jx[9], Jz[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) Jx[k] = Jz[k] = 0.0;
    Jx[0] = 1.0;
    Jz[1] = 1.0;
    double ax = 0.0, az = P.gravity, wdot = 0.0;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int a = kchain(l, s);
      if (a >= 0) {
        Jx[a] = -(F.com[l].pz - F.piv[a].pz);
        Jz[a] = F.com[l].px - F.piv[a].px;
        ax += qd[a] * (-(F.com[l].vz - F.piv[a].vz));
        az += qd[a] * (F.com[l].vx - F.piv[a].vx);
        wdot += qdd[a];
      }
    }
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      ax += Jx[k] * qdd[k];
      az += Jz[k] * qdd[k];
    }
    const double m = P.m_link[l];
#pragma unroll
    for (int k = 0; k < 9; ++k) gen[k] += m * (Jx[k] * ax + Jz[k] * az);
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int a = kchain(l, s);
      if (a >= 0) gen[a] += P.I_link[l] * wdot;
    }
  }
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    double Jx[9], Jz[9];
    contact_jac(F, c, Jx, Jz);
#pragma unroll
    for (int k = 0; k < 9; ++k) gen[k] -= Jx[k] * Fc[2 * c] + Jz[k] * Fc[2 * c + 1];
  }
}

__device__ __forceinline__ double wrap01(double x) {
  // fmod(x, 1.0) (gait.cpp's std::fmod) without the division loop: for finite |x| < 2^53 the
  // fraction x - trunc(x) is a multiple of ulp(x) below 1 in magnitude, so the subtraction is
  // exact and equals fmod bit for bit (larger |x|: both give 0)
  const double w = x - trunc(x);
  return w < 0.0 ? w + 1.0 : w;
}

// Quintic Bezier swing height (gait.cpp:65-99).
__device__ __forceinline__ double bezier_height(double t_sw, double zs, double v_to, double v_td) {
  const double t = fmin(1.0, fmax(0.0, t_sw));
  const double p1 = v_to / 5.0, p4 = -v_td / 5.0;
  const double p2 = (32.0 * zs - 5.0 * (p1 + p4)) / 20.0;
  const double s = 1.0 - t;
  return 5.0 * s * s * s * s * t * p1 + 10.0 * s * s * s * t * t * p2 + 10.0 * s * s * t * t * t * p2 +
         5.0 * s * t * t * t * t * p4;
}

// Stance bits (bit c) of node i and swing progress (gait.cpp:37-63): node i uses the
// cumulative dt of nodes < i, summed in the reference's order.
__device__ __forceinline__ uint32_t node_schedule(const KParams& P, const rmpc_gait& g, int i,
                                                  double swing_t[4]) {
  double shift = 0.0;
  for (int j = 0; j < i; ++j) shift += P.dt[j] / g.period;
  uint32_t bits = 0;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const double ph = wrap01(g.phase + shift + g.offsets[c]);
    if (ph < g.phase_switch) bits |= 1u << c;
    swing_t[c] = (ph >= g.phase_switch && g.phase_switch < 1.0)
                     ? (ph - g.phase_switch) / (1.0 - g.phase_switch)
                     : 0.0;
  }
  return bits;
}

// Guess of node i (mpc.cpp:258-277): warm = previous z* shifted by one node, cold = nominal
// pose at the measured base x, zero velocity, weight shared by the stance contacts.
__device__ __forceinline__ void node_guess(const KParams& P, int i, bool warm, const float* pz,
                                           const rmpc_state& st, uint32_t bits, double* q,
                                           double* qd, double* F) {
  if (warm) {
    const int j = min(i + 1, P.NT - 1);
    const float* r = pz + j * NV;
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      q[k] = (double)r[k];
      qd[k] = (double)r[NQ + k];
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) F[k] = (double)r[18 + k];
  } else {
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      q[k] = P.nominal[k];
      qd[k] = 0.0;
    }
    q[0] = st.q[0];
    const int na = __popc(bits);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      F[2 * c] = 0.0;
      F[2 * c + 1] = ((bits >> c) & 1u) && na > 0 ? P.weight / na : 0.0;
    }
  }
}

// Guess component j (< 26) of node i and its tracking target (mpc.cpp:28-62, 266-276).
__device__ __forceinline__ void guess_and_target(const KParams& P, int i, int j, bool warm,
                                                 const float* pz, const rmpc_state& st,
                                                 const rmpc_command& cmd, uint32_t bits,
                                                 double& g, double& des) {
  const int na = __popc(bits);
  if (j < 9) {
    des = j == 0 ? 0.0 : (j == 1 ? cmd.height : (j == 2 ? 0.0 : P.nominal[j]));
    g = j == 0 ? st.q[0] : P.nominal[j];
  } else if (j < 18) {
    des = j == 9 ? cmd.vx : (j == 11 ? cmd.wpitch : 0.0);
    g = 0.0;
  } else {
    const int c = (j - 18) >> 1;
    const bool fz = (j - 18) & 1;
    des = fz && ((bits >> c) & 1u) && na > 0 ? P.weight / na : 0.0;
    g = des;
  }
  if (warm) g = (double)pz[min(i + 1, P.NT - 1) * NV + j];
}

__device__ __forceinline__ float to_f(double v) { return (float)v; }
__device__ __forceinline__ float bound_f(double v) {  // kInf sentinel -> +-inf in FP32
  return v <= -1e29 ? -INFINITY : (v >= 1e29 ? INFINITY : (float)v);
}
__device__ __forceinline__ void set_row(float4* r, double lo, double hi) {
  *r = make_float4(bound_f(lo), bound_f(hi), 0.f, 0.f);
}

}  // namespace rmpc_dev
