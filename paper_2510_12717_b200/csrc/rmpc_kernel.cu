// rmpc_kernel.cu — fused warp-per-agent RTI-MPC solve for sm_100a.
//
// One warp runs MpcController::rti_step (/root/reference/proj/src/mpc.cpp:248-338) for one
// agent: gait schedule and cold/warm guess (f_init, gait.cpp:37-99), FP64 linearization of
// the floating-base dynamics and contacts (robot.cpp:29-195), QP rows (build_qp,
// mpc.cpp:64-238), 10 Ruiz passes (ruiz.cpp:7-36 via qp.cpp:64-95), factorization, exactly
// n_qp ADMM iterations (qp.cpp:156-190), unscaled residuals/objective (qp.cpp:192-200), the
// full step z* = guess + dz and inverse dynamics at node 0 (mpc.cpp:305-330, robot.cpp:211-233).
//
// Linear algebra: instead of the reference's quasi-definite KKT + sparse LDL^T (qp.cpp:11-34,
// ldl.cpp:123-192) each iteration solves the reduced SPD system
//     H x~ = sigma x - q^ + A^T (rho z - y),  H = P^ + sigma I + rho A^T A,  z~ = A^ x~,
// identical in exact arithmetic (nu = rho (A^ x~ - z) + y eliminates the dual block).  H is
// block tridiagonal over horizon nodes; it is eliminated node by node with explicit
// Schur-complement inverses S_i^-1 (26 x 26, shared memory), the off-diagonal blocks
// C_i = rho A_int/dyn^(i+1)^T A_int/dyn^(i) being applied in their rank-12 factored form.
//
// Precision: gait, guess, linearization, constraint right-hand sides, the objective sum and
// inverse dynamics in FP64; Ruiz, H, S^-1 and the ADMM iterations in FP32.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "rmpc_device.cuh"

namespace rmpc_dev {

#define FULL 0xffffffffu

// ------------------------------------------------------------------------- helpers
struct Sm {
  float* sinv;
  float* coef;
  float* vec;
  float4* row;
  float* dsc;
  float* icoef;
  float* tbuf;
  float* bc;
  float* g;
  uint32_t* flags;
  int NT;
  __device__ __forceinline__ float* V(int i, int which) const {
    return vec + (i * V_NUM + which) * V_STRIDE;
  }
  __device__ __forceinline__ float* C(int i) const { return coef + i * C_SIZE; }
  __device__ __forceinline__ float* Sinv(int i) const { return sinv + i * NV * SROW; }
  __device__ __forceinline__ int ridx(int i, int s) const {
    return s < NSLOT ? i * NSLOT + s : NT * NSLOT + (s - NSLOT);
  }
};

__device__ __forceinline__ float wsum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}
__device__ __forceinline__ float wmax(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(FULL, v, o));
  return v;
}
__device__ __forceinline__ double wsumd(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

struct OpSum {  // sum_j A_rj v_j
  __device__ static __forceinline__ float id() { return 0.f; }
  __device__ static __forceinline__ float comb(float a, float c, float v) { return fmaf(c, v, a); }
  __device__ static __forceinline__ float red(float a, float b) { return a + b; }
};
struct OpMax {  // max_j |A_rj| v_j  (v = positive Ruiz scales)
  __device__ static __forceinline__ float id() { return 0.f; }
  __device__ static __forceinline__ float comb(float a, float c, float v) { return fmaxf(a, fabsf(c) * v); }
  __device__ static __forceinline__ float red(float a, float b) { return fmaxf(a, b); }
};

// Non-zero columns of a foot contact Jacobian: base x, base z, pitch, then the leg's three
// joints (right foot coords 6..8 for contacts 0,1; left foot 3..5 for contacts 2,3).
__device__ __forceinline__ int chain_col(int c, int s) { return s < 3 ? s : (c < 2 ? 6 : 3) + s - 3; }

// ------------------------------------------------------------------------- A^ views
// Row view: for the 40 (+18 at node 0) row slots of node i, out_r = Op_j(A_rj, v_j) with v
// the per-node vector `which` of nodes i and i+1.  Lane l returns slot l in o0, slot 32+l
// (l < 8) in o1, init slot l (node 0, l < 18) in o2.
template <class Op>
__device__ __forceinline__ void row_view(const Sm& sm, int i, int lane, int which, float& o0,
                                         float& o1, float& o2) {
  const float* cf = sm.C(i);
  const float* vi = sm.V(i, which);
  const float* vn = (i + 1 < sm.NT) ? sm.V(i + 1, which) : vi;  // coefficients are 0 then
  o0 = Op::id();
  o1 = Op::id();
  o2 = Op::id();
  if (lane < 9) {  // integration rows: a1 q_{i+1,k} + a2 q_{i,k} + a3 qd_{i+1,k}
    const float4 a = *reinterpret_cast<const float4*>(cf + C_INT + 4 * lane);
    o0 = Op::comb(o0, a.x, vn[lane]);
    o0 = Op::comb(o0, a.y, vi[lane]);
    o0 = Op::comb(o0, a.z, vn[NQ + lane]);
  } else if (lane >= 12 && lane < 28) {  // contact force rows t0, t1
    const int c = (lane - 12) >> 2, t = (lane - 12) & 3;
    if (t < 2) {
      o0 = Op::comb(o0, cf[C_FORCE + 4 * c + 2 * t], vi[18 + 2 * c]);
      o0 = Op::comb(o0, cf[C_FORCE + 4 * c + 2 * t + 1], vi[19 + 2 * c]);
    }
  } else if (lane >= 28) {  // joint position boxes 0..3
    const int m = lane - 28;
    o0 = Op::comb(o0, cf[C_BOX + m], vi[3 + m]);
  }
  if (lane < 8) {  // boxes 4..11
    const int m = 4 + lane;
    const int var = m < 6 ? 3 + m : NQ + 3 + (m - 6);
    o1 = Op::comb(o1, cf[C_BOX + m], vi[var]);
  }
  if (i == 0 && lane < NINIT) o2 = Op::comb(o2, sm.icoef[lane], vi[lane]);
  {  // base-dynamics rows: lane = one of the 26 support entries (qd_{i+1}: 9, node-i 9..25)
    float p0 = Op::id(), p1 = Op::id(), p2 = Op::id();
    if (lane < 9) {
      const float v = vn[NQ + lane];
      p0 = Op::comb(p0, cf[C_DYNU + lane], v);
      p1 = Op::comb(p1, cf[C_DYNU + 12 + lane], v);
      p2 = Op::comb(p2, cf[C_DYNU + 24 + lane], v);
    } else if (lane < NV) {
      const float v = vi[lane];
      p0 = Op::comb(p0, cf[C_DYNV + lane], v);
      p1 = Op::comb(p1, cf[C_DYNV + 28 + lane], v);
      p2 = Op::comb(p2, cf[C_DYNV + 56 + lane], v);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      p0 = Op::red(p0, __shfl_xor_sync(FULL, p0, o));
      p1 = Op::red(p1, __shfl_xor_sync(FULL, p1, o));
      p2 = Op::red(p2, __shfl_xor_sync(FULL, p2, o));
    }
    if (lane == 9) o0 = p0;
    else if (lane == 10) o0 = p1;
    else if (lane == 11) o0 = p2;
  }
  {  // contact Jacobian rows (t2: height on q / velocity-x on qd, t3: velocity-z on qd):
     // 8-lane group per contact, one lane per non-zero column
    const int c = lane >> 3, s = lane & 7;
    float pa = Op::id(), pb = Op::id();
    if (s < 6) {
      const int col = chain_col(c, s);
      const float vq = vi[col], vd = vi[NQ + col];
      pa = Op::comb(pa, cf[C_JQ + 9 * c + col], vq);
      pa = Op::comb(pa, cf[C_JV0 + 9 * c + col], vd);
      pb = Op::comb(pb, cf[C_JV1 + 9 * c + col], vd);
    }
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
      pa = Op::red(pa, __shfl_xor_sync(FULL, pa, o));
      pb = Op::red(pb, __shfl_xor_sync(FULL, pb, o));
    }
    const bool mine = lane >= 12 && lane < 28;
    const int src = mine ? ((lane - 12) >> 2) << 3 : 0;
    const float ga = __shfl_sync(FULL, pa, src), gb = __shfl_sync(FULL, pb, src);
    if (mine) {
      const int t = (lane - 12) & 3;
      if (t == 2) o0 = ga;
      else if (t == 3) o0 = gb;
    }
  }
}

// Column view: for var j = lane (< 26) of node i, Op_r(A_rj, t_r) over every row touching
// node i: its own slots (tc[0..40), init slots tc[40..58) at node 0) and the integration /
// dynamics slots of node i-1 (tp[0..12)).
template <class Op>
__device__ __forceinline__ float col_view(const Sm& sm, int i, int lane, const float* tc,
                                          const float* tp) {
  const float* cf = sm.C(i);
  float acc = Op::id();
  if (lane < 9) {  // q_k
    const int k = lane;
    acc = Op::comb(acc, cf[C_INT + 4 * k + 1], tc[k]);
    if (i > 0) acc = Op::comb(acc, sm.C(i - 1)[C_INT + 4 * k], tp[k]);
#pragma unroll
    for (int c = 0; c < NC; ++c) acc = Op::comb(acc, cf[C_JQ + 9 * c + k], tc[14 + 4 * c]);
    if (k >= 3) acc = Op::comb(acc, cf[C_BOX + k - 3], tc[28 + k - 3]);
    if (i == 0) acc = Op::comb(acc, sm.icoef[k], tc[NSLOT + k]);
  } else if (lane < 18) {  // qd_k
    const int k = lane - 9;
    if (i > 0) {
      const float* cp = sm.C(i - 1);
      acc = Op::comb(acc, cp[C_INT + 4 * k + 2], tp[k]);
#pragma unroll
      for (int b = 0; b < 3; ++b) acc = Op::comb(acc, cp[C_DYNU + 12 * b + k], tp[9 + b]);
    }
#pragma unroll
    for (int b = 0; b < 3; ++b) acc = Op::comb(acc, cf[C_DYNV + 28 * b + lane], tc[9 + b]);
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      acc = Op::comb(acc, cf[C_JV0 + 9 * c + k], tc[14 + 4 * c]);
      acc = Op::comb(acc, cf[C_JV1 + 9 * c + k], tc[15 + 4 * c]);
    }
    if (k >= 3) acc = Op::comb(acc, cf[C_BOX + 6 + k - 3], tc[34 + k - 3]);
    if (i == 0) acc = Op::comb(acc, sm.icoef[NQ + k], tc[NSLOT + NQ + k]);
  } else if (lane < NV) {  // F_{2c+a}
    const int c = (lane - 18) >> 1, a = (lane - 18) & 1;
#pragma unroll
    for (int b = 0; b < 3; ++b) acc = Op::comb(acc, cf[C_DYNV + 28 * b + lane], tc[9 + b]);
    acc = Op::comb(acc, cf[C_FORCE + 4 * c + a], tc[12 + 4 * c]);
    acc = Op::comb(acc, cf[C_FORCE + 4 * c + 2 + a], tc[13 + 4 * c]);
  }
  return acc;
}

// Fill tc (node i's slot values) from the row data with f(row{lo,hi,z,y}, d).
template <class F>
__device__ __forceinline__ void fill_t(const Sm& sm, int i, int lane, float* tc, F f) {
  __syncwarp();
  int r = sm.ridx(i, lane);
  tc[lane] = f(sm.row[r], sm.dsc[r]);
  if (lane < 8) {
    r = sm.ridx(i, 32 + lane);
    tc[32 + lane] = f(sm.row[r], sm.dsc[r]);
  }
  if (i == 0 && lane < NINIT) {
    r = sm.ridx(0, NSLOT + lane);
    tc[NSLOT + lane] = f(sm.row[r], sm.dsc[r]);
  }
  __syncwarp();
}

// out_j = sum_l S_i^-1[j][l] u_l for j = lane < 26 (u published through bcbuf).
__device__ __forceinline__ float sinv_mv(const Sm& sm, int i, int lane, float* bcbuf, float u) {
  bcbuf[lane] = lane < NV ? u : 0.f;
  __syncwarp();
  const int j = lane < NV ? lane : NV - 1;
  const float2* rw = reinterpret_cast<const float2*>(sm.Sinv(i) + j * SROW);
  const float4* b4 = reinterpret_cast<const float4*>(bcbuf);
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
  for (int q = 0; q < 6; ++q) {
    const float4 bb = b4[q];
    const float2 r0 = rw[2 * q], r1 = rw[2 * q + 1];
    a0 = fmaf(r0.x, bb.x, a0);
    a1 = fmaf(r0.y, bb.y, a1);
    a2 = fmaf(r1.x, bb.z, a2);
    a3 = fmaf(r1.y, bb.w, a3);
  }
  {
    const float2 bb = reinterpret_cast<const float2*>(bcbuf)[12];
    const float2 r = rw[12];
    a0 = fmaf(r.x, bb.x, a0);
    a1 = fmaf(r.y, bb.y, a1);
  }
  __syncwarp();
  return (a0 + a1) + (a2 + a3);
}

// ------------------------------------------------------------------------- FP64 kinematics
struct Fr {
  double px, pz, vx, vz;
};

// Point attached to `f` at offset (x, z) in the frame rotated by `ang`, spinning at `w`
// (robot.cpp:39-43).
__device__ __forceinline__ Fr attach(const Fr& f, double ang, double w, double x, double z) {
  double s, c;
  sincos(ang, &s, &c);
  const double rx = c * x - s * z, rz = s * x + c * z;
  Fr o;
  o.px = f.px + rx;
  o.pz = f.pz + rz;
  o.vx = f.vx - w * rz;
  o.vz = f.vz + w * rx;
  return o;
}

// Kinematic chains of the 7 links (robot.cpp:18-21): coordinate indices, -1 padded.
__device__ __forceinline__ int kchain(int l, int s) {
  const int t[7][4] = {{2, -1, -1, -1}, {2, 3, -1, -1}, {2, 3, 4, -1}, {2, 3, 4, 5},
                       {2, 6, -1, -1},  {2, 6, 7, -1},  {2, 6, 7, 8}};
  return t[l][s];
}

// Frames of the planar biped at (q, qd) with base x taken as 0: Jacobians, J-dot qd and
// masses depend only on position differences (robot.cpp:98), contact heights only on z.
struct Frames {
  Fr piv[9];  // pivots of angle coordinates 2..8
  Fr com[7];
  Fr con[4];
};

__device__ void fk_frames(const KParams& P, const double* q, const double* qd, Frames& F) {
  Fr base;
  base.px = 0.0;
  base.pz = q[1];
  base.vx = qd[0];
  base.vz = qd[1];
  const double th = q[2];
  const Fr hip = attach(base, th, qd[2], 0.0, -0.5 * P.torso_len);
  F.piv[2] = base;
  F.piv[3] = hip;
  F.piv[6] = hip;
  F.com[0] = base;
#pragma unroll
  for (int leg = 0; leg < 2; ++leg) {  // 0 = left (3..5), 1 = right (6..8)
    const int h = 3 + 3 * leg;
    const double a1 = th + q[h], a2 = a1 + q[h + 1], a3 = a2 + q[h + 2];
    const double w1 = qd[2] + qd[h], w2 = w1 + qd[h + 1], w3 = w2 + qd[h + 2];
    const Fr knee = attach(hip, a1, w1, 0.0, -P.thigh_len);
    const Fr ankle = attach(knee, a2, w2, 0.0, -P.shank_len);
    F.piv[h + 1] = knee;
    F.piv[h + 2] = ankle;
    F.com[1 + 3 * leg] = attach(hip, a1, w1, 0.0, -0.5 * P.thigh_len);
    F.com[2 + 3 * leg] = attach(knee, a2, w2, 0.0, -0.5 * P.shank_len);
    F.com[3 + 3 * leg] = attach(ankle, a3, w3, 0.0, -P.ankle_drop);
    const int c0 = leg == 0 ? 2 : 0;  // contacts (R toe, R heel, L toe, L heel)
    F.con[c0] = attach(ankle, a3, w3, P.foot_half, -P.ankle_drop);
    F.con[c0 + 1] = attach(ankle, a3, w3, -P.foot_half, -P.ankle_drop);
  }
}

// Top three rows of M (robot.cpp:169-178) and of h (robot.cpp:184-195).
__device__ void base_dynamics(const KParams& P, const double* qd, const Frames& F,
                              double Mb[3][9], double hb[3]) {
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    hb[b] = 0.0;
#pragma unroll
    for (int k = 0; k < 9; ++k) Mb[b][k] = 0.0;
  }
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
#pragma unroll
    for (int b = 0; b < 3; ++b) {
#pragma unroll
      for (int k = 0; k < 9; ++k) Mb[b][k] += m * (Jx[b] * Jx[k] + Jz[b] * Jz[k]);
      hb[b] += m * (Jx[b] * ax + Jz[b] * (az + P.gravity));
    }
#pragma unroll
    for (int s = 0; s < 4; ++s) {  // rotational part: coordinate 2 is in every chain
      const int a = kchain(l, s);
      if (a >= 0) Mb[2][a] += P.I_link[l];
    }
  }
}

// Contact Jacobian rows (2 x 9) of contact c (robot.cpp:91-101,137-146).
__device__ __forceinline__ void contact_jac(const Frames& F, int c, double Jx[9], double Jz[9]) {
#pragma unroll
  for (int k = 0; k < 9; ++k) Jx[k] = Jz[k] = 0.0;
  Jx[0] = 1.0;
  Jz[1] = 1.0;
  const int h = c < 2 ? 6 : 3;
  const int chain[4] = {2, h, h + 1, h + 2};
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const int a = chain[s];
    Jx[a] = -(F.con[c].pz - F.piv[a].pz);
    Jz[a] = F.con[c].px - F.piv[a].px;
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
  const double w = fmod(x, 1.0);
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

// Stance bits (bit c) of node i and, for swing contacts, progress (gait.cpp:37-63): node i
// uses the cumulative dt of nodes < i, summed in the reference's order.
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

__device__ __forceinline__ float to_f(double v) { return (float)v; }
__device__ __forceinline__ float bound_f(double v) {  // kInf sentinel -> +-inf in FP32
  return v <= -1e29 ? -INFINITY : (v >= 1e29 ? INFINITY : (float)v);
}

__device__ __forceinline__ void set_row(const Sm& sm, int r, double lo, double hi) {
  sm.row[r] = make_float4(bound_f(lo), bound_f(hi), 0.f, 0.f);
}

// ------------------------------------------------------------------------- stage: setup
// Lane i < NT builds node i of the QP (build_qp, mpc.cpp:64-238) in FP64 and stores the
// unscaled coefficients, bounds, P diagonal and q in shared memory.  Returns false if the
// linearization point is non-finite (StructuralError, mpc.cpp:70-72).
__device__ bool setup_nodes(const KParams& P, const Sm& sm, int lane, const rmpc_state& st,
                            const rmpc_command& cmd, const rmpc_gait& gait, bool warm,
                            const float* pz) {
  const int NT = P.NT;
  bool ok = true;
#pragma unroll 1
  for (int i = lane; i < NT; i += 32) {
    double swt[4], swt_n[4];
    const uint32_t bits = node_schedule(P, gait, i, swt);
    const uint32_t bits_n = i + 1 < NT ? node_schedule(P, gait, i + 1, swt_n) : 0u;
    double gq[9], gqd[9], gF[8], nq[9], nqd[9], nF[8];
    node_guess(P, i, warm, pz, st, bits, gq, gqd, gF);
    if (i + 1 < NT) node_guess(P, i + 1, warm, pz, st, bits_n, nq, nqd, nF);
#pragma unroll
    for (int k = 0; k < 9; ++k) ok = ok && isfinite(gq[k]) && isfinite(gqd[k]);
#pragma unroll
    for (int k = 0; k < 8; ++k) ok = ok && isfinite(gF[k]);
    sm.flags[i] = bits;
    float* cf = sm.C(i);
    const double dt = P.dt[i];

    Frames F;
    fk_frames(P, gq, gqd, F);
    double Jx[4][9], Jz[4][9];
#pragma unroll
    for (int c = 0; c < 4; ++c) contact_jac(F, c, Jx[c], Jz[c]);

    // cost (mpc.cpp:81-103): P = diag(w dt), q = w dt (guess - desired)
    {
      const int na = __popc(bits);
      float* pd = sm.V(i, V_PD);
      float* qh = sm.V(i, V_QH);
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        double qdes = P.nominal[k];
        if (k == 0) qdes = 0.0;
        if (k == 1) qdes = cmd.height;
        if (k == 2) qdes = 0.0;
        const double qddes = k == 0 ? cmd.vx : (k == 2 ? cmd.wpitch : 0.0);
        const double wq = P.wq[k] * dt, wqd = P.wqd[k] * dt;
        pd[k] = to_f(wq);
        pd[NQ + k] = to_f(wqd);
        qh[k] = to_f(wq * (gq[k] - qdes));
        qh[NQ + k] = to_f(wqd * (gqd[k] - qddes));
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const double fdes = ((k & 1) && ((bits >> (k >> 1)) & 1u) && na > 0) ? P.weight / na : 0.0;
        const double wf = P.wf[k] * dt;
        pd[18 + k] = to_f(wf);
        qh[18 + k] = to_f(wf * (gF[k] - fdes));
      }
    }
    if (i + 1 < NT) {
      // integration rows (mpc.cpp:138-148)
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        cf[C_INT + 4 * k + 0] = 1.f;
        cf[C_INT + 4 * k + 1] = -1.f;
        cf[C_INT + 4 * k + 2] = to_f(-dt);
        const double r = -(nq[k] - gq[k] - dt * nqd[k]);
        set_row(sm, sm.ridx(i, k), r, r);
      }
      // base dynamics with qdd eliminated (mpc.cpp:150-175)
      double Mb[3][9], hb[3];
      base_dynamics(P, gqd, F, Mb, hb);
      const double dt_inv = 1.0 / dt;
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        double mq = 0.0;
#pragma unroll
        for (int k = 0; k < 9; ++k) mq += Mb[b][k] * (nqd[k] - gqd[k]);
        double jbf = 0.0;
#pragma unroll
        for (int c = 0; c < 4; ++c) jbf += Jx[c][b] * gF[2 * c] + Jz[c][b] * gF[2 * c + 1];
        const double resid = mq * dt_inv + hb[b] - jbf;
#pragma unroll
        for (int k = 0; k < 9; ++k) {
          const double mv = Mb[b][k] * dt_inv;
          cf[C_DYNU + 12 * b + k] = to_f(mv);
          cf[C_DYNV + 28 * b + NQ + k] = to_f(-mv);
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          cf[C_DYNV + 28 * b + 18 + 2 * c] = to_f(-Jx[c][b]);
          cf[C_DYNV + 28 * b + 19 + 2 * c] = to_f(-Jz[c][b]);
        }
        set_row(sm, sm.ridx(i, 9 + b), -resid, -resid);
      }
    }
    // contact rows (mpc.cpp:181-218)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const double fx = gF[2 * c], fz = gF[2 * c + 1];
      const int s0 = 12 + 4 * c;
      if ((bits >> c) & 1u) {
        cf[C_FORCE + 4 * c + 0] = 1.f;
        cf[C_FORCE + 4 * c + 1] = to_f(-P.mu);
        cf[C_FORCE + 4 * c + 2] = -1.f;
        cf[C_FORCE + 4 * c + 3] = to_f(-P.mu);
        set_row(sm, sm.ridx(i, s0), -1e30, -(fx - P.mu * fz));
        set_row(sm, sm.ridx(i, s0 + 1), -1e30, -(-fx - P.mu * fz));
        if (i > 0) {
          double r0 = 0.0, r1 = 0.0;
#pragma unroll
          for (int k = 0; k < 9; ++k) {
            r0 += Jx[c][k] * gqd[k];
            r1 += Jz[c][k] * gqd[k];
            cf[C_JV0 + 9 * c + k] = to_f(Jx[c][k]);
            cf[C_JV1 + 9 * c + k] = to_f(Jz[c][k]);
          }
          set_row(sm, sm.ridx(i, s0 + 2), -r0, -r0);
          set_row(sm, sm.ridx(i, s0 + 3), -r1, -r1);
        }
      } else {
        cf[C_FORCE + 4 * c + 0] = 1.f;
        cf[C_FORCE + 4 * c + 3] = 1.f;
        set_row(sm, sm.ridx(i, s0), -fx, -fx);
        set_row(sm, sm.ridx(i, s0 + 1), -fz, -fz);
        if (i > 0) {
          const double h = bezier_height(swt[c], P.z_swing, P.v_to, P.v_td);
          const double r = h - F.con[c].pz;
#pragma unroll
          for (int k = 0; k < 9; ++k) cf[C_JQ + 9 * c + k] = to_f(Jz[c][k]);
          set_row(sm, sm.ridx(i, s0 + 2), r, r);
        }
      }
    }
    if (i > 0) {  // joint boxes (mpc.cpp:220-232)
#pragma unroll
      for (int m = 0; m < 6; ++m) {
        cf[C_BOX + m] = 1.f;
        set_row(sm, sm.ridx(i, 28 + m), P.jlo[m] - gq[3 + m], P.jhi[m] - gq[3 + m]);
        cf[C_BOX + 6 + m] = 1.f;
        set_row(sm, sm.ridx(i, 34 + m), -P.qdlim[m] - gqd[3 + m], P.qdlim[m] - gqd[3 + m]);
      }
    } else {  // initial state (mpc.cpp:126-136)
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        sm.icoef[k] = 1.f;
        sm.icoef[NQ + k] = 1.f;
        const double rq = st.q[k] - gq[k], rqd = st.qd[k] - gqd[k];
        set_row(sm, sm.ridx(0, NSLOT + k), rq, rq);
        set_row(sm, sm.ridx(0, NSLOT + NQ + k), rqd, rqd);
      }
    }
  }
  return __all_sync(FULL, ok);
}

// ------------------------------------------------------------------------- stage: Ruiz
// AdmmSolver::equilibrate (qp.cpp:64-95) + ruiz_equilibrate (ruiz.cpp:7-36) on
// [[P, A^T], [A, 0]]: per pass delta = 1/sqrt(inf-norm) of every row/column of the current
// scaled matrix (1 for empty ones), d *= delta (rows), e *= delta (columns).
__device__ void ruiz(const KParams& P, const Sm& sm, int lane) {
  const int NT = P.NT;
#pragma unroll 1
  for (int pass = 0; pass < P.ruiz_iters; ++pass) {
#pragma unroll 1
    for (int i = 0; i < NT; ++i) {
      float o0, o1, o2;
      row_view<OpMax>(sm, i, lane, V_E, o0, o1, o2);
      auto stash = [&](int s, float o) {  // delta of row slot s into row.z (z is 0 here)
        const int r = sm.ridx(i, s);
        const float nrm = sm.dsc[r] * o;
        sm.row[r].z = nrm > 0.f ? 1.f / sqrtf(nrm) : 1.f;
      };
      float* tc = sm.tbuf + (i & 1) * 64;
      const float* tp = sm.tbuf + ((i + 1) & 1) * 64;
      // row deltas must not be visible before every column norm of this pass is formed:
      // column norms use d (dsc), deltas live in row.z until the apply step.
      fill_t(sm, i, lane, tc, [](float4, float d) { return d; });
      const float cv = col_view<OpMax>(sm, i, lane, tc, tp);
      stash(lane, o0);
      if (lane < 8) stash(32 + lane, o1);
      if (i == 0 && lane < NINIT) stash(NSLOT + lane, o2);
      if (lane < NV) {
        const float e = sm.V(i, V_E)[lane];
        const float nrm = e * fmaxf(fabsf(sm.V(i, V_PD)[lane]) * e, cv);
        sm.V(i, V_S)[lane] = nrm > 0.f ? 1.f / sqrtf(nrm) : 1.f;
      }
    }
    __syncwarp();
    const int nrow = NT * NSLOT + NINIT;
    for (int r = lane; r < nrow; r += 32) {
      sm.dsc[r] *= sm.row[r].z;
      sm.row[r].z = 0.f;
    }
    for (int i = 0; i < NT; ++i)
      if (lane < NV) sm.V(i, V_E)[lane] *= sm.V(i, V_S)[lane];
    __syncwarp();
  }
}

// Scale coefficients, bounds and cost in place: A^ = D A E, P^ = E P E, q^ = E q,
// lo^ = D lo, hi^ = D hi (qp.cpp:86-94).
__device__ void apply_scaling(const KParams& P, const Sm& sm, int lane) {
  const int NT = P.NT;
  for (int i = 0; i < NT; ++i) {
    float* cf = sm.C(i);
    const float* ei = sm.V(i, V_E);
    const float* en = i + 1 < NT ? sm.V(i + 1, V_E) : ei;
    auto d = [&](int s) { return sm.dsc[sm.ridx(i, s)]; };
    if (lane < 9) {
      const float dr = d(lane);
      cf[C_INT + 4 * lane + 0] *= dr * en[lane];
      cf[C_INT + 4 * lane + 1] *= dr * ei[lane];
      cf[C_INT + 4 * lane + 2] *= dr * en[NQ + lane];
#pragma unroll
      for (int b = 0; b < 3; ++b) cf[C_DYNU + 12 * b + lane] *= d(9 + b) * en[NQ + lane];
    } else if (lane < NV) {
#pragma unroll
      for (int b = 0; b < 3; ++b) cf[C_DYNV + 28 * b + lane] *= d(9 + b) * ei[lane];
    }
    if (lane < 16) {
      const int c = lane >> 2, t = (lane >> 1) & 1, a = lane & 1;
      cf[C_FORCE + lane] *= d(12 + 4 * c + t) * ei[18 + 2 * c + a];
    }
    for (int idx = lane; idx < 36; idx += 32) {
      const int c = idx / 9, k = idx % 9;
      cf[C_JQ + idx] *= d(14 + 4 * c) * ei[k];
      cf[C_JV0 + idx] *= d(14 + 4 * c) * ei[NQ + k];
      cf[C_JV1 + idx] *= d(15 + 4 * c) * ei[NQ + k];
    }
    if (lane < 12) cf[C_BOX + lane] *= d(28 + lane) * ei[lane < 6 ? 3 + lane : NQ + 3 + (lane - 6)];
    if (i == 0 && lane < NINIT) sm.icoef[lane] *= d(NSLOT + lane) * ei[lane];
    if (lane < NV) {
      const float e = ei[lane];
      sm.V(i, V_PD)[lane] *= e * e;
      sm.V(i, V_QH)[lane] *= e;
    }
  }
  const int nrow = NT * NSLOT + NINIT;
  for (int r = lane; r < nrow; r += 32) {
    float4 rd = sm.row[r];
    const float dr = sm.dsc[r];
    rd.x *= dr;
    rd.y *= dr;
    sm.row[r] = rd;
  }
  __syncwarp();
}

// ------------------------------------------------------------------------- stage: factor
// Block elimination of H: S_0 = H_00, S_{i+1} = H_{i+1,i+1} - C_i S_i^-1 C_i^T, S_i^-1
// stored.  Lane j holds row j of the 26 x 26 blocks in registers.  Returns false on a
// non-positive pivot (SingularityError analogue, ldl.cpp:155-160).
__device__ bool factorize(const KParams& P, const Sm& sm, int lane) {
  const int NT = P.NT;
  const float rho = (float)P.rho, sigma = (float)P.sigma;
  const int j = lane;
  float Yp[18];
#pragma unroll
  for (int l = 0; l < 18; ++l) Yp[l] = 0.f;
  bool good = true;
#pragma unroll 1
  for (int i = 0; i < NT; ++i) {
    const float* cf = sm.C(i);
    const float* cp = i > 0 ? sm.C(i - 1) : cf;
    const uint32_t bits = sm.flags[i];
    float S[NV];
    // (a) diagonal and the single paired off-diagonal entry per row
    {
      float dg = 0.f, pt = 0.f;
      int pidx = -1;
      if (j < NV) dg = sm.V(i, V_PD)[j] + sigma;
      if (j < 9) {
        const float a2 = cf[C_INT + 4 * j + 1];
        dg += rho * a2 * a2;
        if (i > 0) {
          const float a1 = cp[C_INT + 4 * j], a3 = cp[C_INT + 4 * j + 2];
          dg += rho * a1 * a1;
          pt = rho * a1 * a3;
          pidx = NQ + j;
        }
        if (j >= 3) { const float b = cf[C_BOX + j - 3]; dg += rho * b * b; }
        if (i == 0) { const float b = sm.icoef[j]; dg += rho * b * b; }
      } else if (j < 18) {
        const int k = j - 9;
        if (i > 0) {
          const float a1 = cp[C_INT + 4 * k], a3 = cp[C_INT + 4 * k + 2];
          dg += rho * a3 * a3;
          pt = rho * a1 * a3;
          pidx = k;
        }
        if (k >= 3) { const float b = cf[C_BOX + 6 + k - 3]; dg += rho * b * b; }
        if (i == 0) { const float b = sm.icoef[NQ + k]; dg += rho * b * b; }
      } else if (j < NV) {
        const int c = (j - 18) >> 1, a = (j - 18) & 1;
        const float f0 = cf[C_FORCE + 4 * c + a], g0 = cf[C_FORCE + 4 * c + 1 - a];
        const float f1 = cf[C_FORCE + 4 * c + 2 + a], g1 = cf[C_FORCE + 4 * c + 3 - a];
        dg += rho * (f0 * f0 + f1 * f1);
        pt = rho * (f0 * g0 + f1 * g1);
        pidx = 18 + 2 * c + (1 - a);
      }
#pragma unroll
      for (int l = 0; l < NV; ++l) S[l] = (l == j ? dg : 0.f) + (l == pidx ? pt : 0.f);
    }
    // (b) dense rank-1 terms: dynamics rows of intervals i and i-1, contact Jacobian rows
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const float* vb = cf + C_DYNV + 28 * b;
      const float s = j < NV ? rho * vb[j] : 0.f;
      const float4* v4 = reinterpret_cast<const float4*>(vb);
#pragma unroll
      for (int q = 0; q < 7; ++q) {
        const float4 w = v4[q];
        S[4 * q] = fmaf(s, w.x, S[4 * q]);
        S[4 * q + 1] = fmaf(s, w.y, S[4 * q + 1]);
        if (4 * q + 2 < NV) S[4 * q + 2] = fmaf(s, w.z, S[4 * q + 2]);
        if (4 * q + 3 < NV) S[4 * q + 3] = fmaf(s, w.w, S[4 * q + 3]);
      }
    }
    if (i > 0) {
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        const float* ub = cp + C_DYNU + 12 * b;
        const float s = (j >= 9 && j < 18) ? rho * ub[j - 9] : 0.f;
#pragma unroll
        for (int m = 0; m < 9; ++m) S[NQ + m] = fmaf(s, ub[m], S[NQ + m]);
      }
    }
    if (i > 0) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if ((bits >> c) & 1u) {  // stance: velocity rows on qd
          const float* j0 = cf + C_JV0 + 9 * c;
          const float* j1 = cf + C_JV1 + 9 * c;
          const bool mine = j >= 9 && j < 18;
          const float s0 = mine ? rho * j0[j - 9] : 0.f, s1 = mine ? rho * j1[j - 9] : 0.f;
#pragma unroll
          for (int m = 0; m < 9; ++m) S[NQ + m] = fmaf(s0, j0[m], fmaf(s1, j1[m], S[NQ + m]));
        } else {  // swing: height row on q
          const float* jq = cf + C_JQ + 9 * c;
          const float s = j < 9 ? rho * jq[j] : 0.f;
#pragma unroll
          for (int m = 0; m < 9; ++m) S[m] = fmaf(s, jq[m], S[m]);
        }
      }
    }
    // (c) Schur update from the previous node
#pragma unroll
    for (int l = 0; l < 18; ++l) S[l] -= Yp[l];
    // (d) Gauss-Jordan inversion in place (SPD, no pivoting), rows exchanged through smem
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      float* buf = sm.bc + 32 * (k & 1);
      if (j == k) {
        float4* b4 = reinterpret_cast<float4*>(buf);
#pragma unroll
        for (int q = 0; q < 6; ++q) b4[q] = make_float4(S[4 * q], S[4 * q + 1], S[4 * q + 2], S[4 * q + 3]);
        reinterpret_cast<float2*>(buf)[12] = make_float2(S[24], S[25]);
      }
      __syncwarp();
      float R[NV];
      {
        const float4* b4 = reinterpret_cast<const float4*>(buf);
#pragma unroll
        for (int q = 0; q < 6; ++q) {
          const float4 w = b4[q];
          R[4 * q] = w.x; R[4 * q + 1] = w.y; R[4 * q + 2] = w.z; R[4 * q + 3] = w.w;
        }
        const float2 w = reinterpret_cast<const float2*>(buf)[12];
        R[24] = w.x;
        R[25] = w.y;
      }
      const float p = R[k];
      good = good && (p > 0.f);
      const float pinv = 1.f / p;
      const float f = S[k];
      const bool me = (j == k);
      const float keep = me ? 0.f : 1.f;
      const float alpha = me ? pinv : -f * pinv;
#pragma unroll
      for (int l = 0; l < NV; ++l) S[l] = fmaf(alpha, R[l], keep * S[l]);
      S[k] = me ? pinv : -f * pinv;
    }
    // (e) store S_i^-1
    if (j < NV) {
      float2* dst = reinterpret_cast<float2*>(sm.Sinv(i) + j * SROW);
#pragma unroll
      for (int q = 0; q < 13; ++q) dst[q] = make_float2(S[2 * q], S[2 * q + 1]);
    }
    // (f) Schur update for node i+1 in factored form: Y = rho^2 U G U^T,
    //     G = V^T S^-1 V (12 x 12), V/U = node-i / node-(i+1) parts of the 9 integration and
    //     3 dynamics rows of interval i.
    if (i + 1 < NT) {
      float W[3];
#pragma unroll
      for (int b = 0; b < 3; ++b) {  // W_b = S^-1 v_b (lane j: component j)
        const float4* v4 = reinterpret_cast<const float4*>(cf + C_DYNV + 28 * b);
        float acc = 0.f;
#pragma unroll
        for (int q = 0; q < 7; ++q) {
          const float4 w = v4[q];
          acc = fmaf(S[4 * q], w.x, acc);
          acc = fmaf(S[4 * q + 1], w.y, acc);
          if (4 * q + 2 < NV) acc = fmaf(S[4 * q + 2], w.z, acc);
          if (4 * q + 3 < NV) acc = fmaf(S[4 * q + 3], w.w, acc);
        }
        W[b] = j < NV ? acc : 0.f;
      }
      float* G = sm.g + 96;  // 12 x 13 (odd stride)
      if (j < 9) {
        const float a2 = cf[C_INT + 4 * j + 1];
#pragma unroll
        for (int k = 0; k < 9; ++k) G[j * 13 + k] = a2 * S[k] * cf[C_INT + 4 * k + 1];
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          G[j * 13 + 9 + b] = a2 * W[b];
          G[(9 + b) * 13 + j] = a2 * W[b];
        }
      }
      float gdd[3][3];
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        const float vb = j < NV ? cf[C_DYNV + 28 * b + j] : 0.f;
#pragma unroll
        for (int b2 = 0; b2 < 3; ++b2) gdd[b][b2] = wsum(vb * W[b2]);
      }
      if (j == 0) {
#pragma unroll
        for (int b = 0; b < 3; ++b)
#pragma unroll
          for (int b2 = 0; b2 < 3; ++b2) G[(9 + b) * 13 + 9 + b2] = 0.5f * (gdd[b][b2] + gdd[b2][b]);
      }
      __syncwarp();
      float Z[12];
      if (j < 9) {
        const float a1 = cf[C_INT + 4 * j];
#pragma unroll
        for (int s = 0; s < 12; ++s) Z[s] = a1 * G[j * 13 + s];
      } else if (j < 18) {
        const int k = j - 9;
        const float a3 = cf[C_INT + 4 * k + 2];
        const float u0 = cf[C_DYNU + k], u1 = cf[C_DYNU + 12 + k], u2 = cf[C_DYNU + 24 + k];
#pragma unroll
        for (int s = 0; s < 12; ++s)
          Z[s] = a3 * G[k * 13 + s] + u0 * G[9 * 13 + s] + u1 * G[10 * 13 + s] + u2 * G[11 * 13 + s];
      } else {
#pragma unroll
        for (int s = 0; s < 12; ++s) Z[s] = 0.f;
      }
      const float r2 = rho * rho;
#pragma unroll
      for (int m = 0; m < 9; ++m) Yp[m] = r2 * Z[m] * cf[C_INT + 4 * m];
#pragma unroll
      for (int k = 0; k < 9; ++k)
        Yp[NQ + k] = r2 * (Z[k] * cf[C_INT + 4 * k + 2] + Z[9] * cf[C_DYNU + k] +
                           Z[10] * cf[C_DYNU + 12 + k] + Z[11] * cf[C_DYNU + 24 + k]);
      __syncwarp();
    }
  }
  return __all_sync(FULL, good);
}

// ------------------------------------------------------------------------- stage: ADMM
// AdmmSolver::run (qp.cpp:156-190): exactly n_qp iterations from x = y = z = 0.  Returns the
// first iteration with a non-finite iterate, or -1.
__device__ int admm(const KParams& P, const Sm& sm, int lane) {
  const int NT = P.NT;
  const float rho = (float)P.rho, sigma = (float)P.sigma, alpha = (float)P.alpha;
  const float rho_inv = (float)(1.0 / P.rho);
  const float oma = 1.f - alpha;
#pragma unroll 1
  for (int it = 0; it < P.n_qp; ++it) {
    // forward sweep: r_i = sigma x - q^ + A^T(rho z - y); u_i = r_i - C_{i-1} s_{i-1};
    // s_i = S_i^-1 u_i
    float g_int = 0.f, gd0 = 0.f, gd1 = 0.f, gd2 = 0.f;
#pragma unroll 1
    for (int i = 0; i < NT; ++i) {
      float* tc = sm.tbuf + (i & 1) * 64;
      const float* tp = sm.tbuf + ((i + 1) & 1) * 64;
      fill_t(sm, i, lane, tc, [rho](float4 r, float) { return rho * r.z - r.w; });
      const float cv = col_view<OpSum>(sm, i, lane, tc, tp);
      float r = 0.f;
      if (lane < NV) r = sigma * sm.V(i, V_X)[lane] - sm.V(i, V_QH)[lane] + cv;
      if (i > 0) {
        const float* cp = sm.C(i - 1);
        const float gk = __shfl_sync(FULL, g_int, lane >= 9 && lane < 18 ? lane - 9 : 0);
        if (lane < 9) {
          r -= rho * cp[C_INT + 4 * lane] * g_int;
        } else if (lane < 18) {
          const int k = lane - 9;
          r -= rho * (cp[C_INT + 4 * k + 2] * gk + cp[C_DYNU + k] * gd0 +
                      cp[C_DYNU + 12 + k] * gd1 + cp[C_DYNU + 24 + k] * gd2);
        }
      }
      const float s = sinv_mv(sm, i, lane, sm.bc, r);
      if (lane < NV) sm.V(i, V_S)[lane] = s;
      if (i + 1 < NT) {
        const float* cf = sm.C(i);
        g_int = lane < 9 ? cf[C_INT + 4 * lane + 1] * s : 0.f;
        const bool dv = lane >= 9 && lane < NV;
        gd0 = wsum(dv ? cf[C_DYNV + lane] * s : 0.f);
        gd1 = wsum(dv ? cf[C_DYNV + 28 + lane] * s : 0.f);
        gd2 = wsum(dv ? cf[C_DYNV + 56 + lane] * s : 0.f);
      }
    }
    // backward sweep: x~_i = s_i - S_i^-1 C_i^T x~_{i+1}; then the row updates of node i
    // (z~ = A^ x~, relaxation, projection, dual step) and the x relaxation.
    bool bad = false;
#pragma unroll 1
    for (int i = NT - 1; i >= 0; --i) {
      __syncwarp();
      float xt = lane < NV ? sm.V(i, V_S)[lane] : 0.f;
      if (i + 1 < NT) {
        const float* cf = sm.C(i);
        const float* xn = sm.V(i + 1, V_S);
        float dint = 0.f;
        if (lane < 9) dint = cf[C_INT + 4 * lane] * xn[lane] + cf[C_INT + 4 * lane + 2] * xn[NQ + lane];
        const float xq = lane < 9 ? xn[NQ + lane] : 0.f;
        const float e0 = wsum(lane < 9 ? cf[C_DYNU + lane] * xq : 0.f);
        const float e1 = wsum(lane < 9 ? cf[C_DYNU + 12 + lane] * xq : 0.f);
        const float e2 = wsum(lane < 9 ? cf[C_DYNU + 24 + lane] * xq : 0.f);
        float w = 0.f;
        if (lane < 9) {
          w = rho * cf[C_INT + 4 * lane + 1] * dint;
        } else if (lane < NV) {
          w = rho * (cf[C_DYNV + lane] * e0 + cf[C_DYNV + 28 + lane] * e1 + cf[C_DYNV + 56 + lane] * e2);
        }
        xt -= sinv_mv(sm, i, lane, sm.bc, w);
        if (lane < NV) sm.V(i, V_S)[lane] = xt;
        __syncwarp();
      }
      bad = bad || !isfinite(xt);
      float o0, o1, o2;
      row_view<OpSum>(sm, i, lane, V_S, o0, o1, o2);
      auto upd = [&](int s, float zt) {
        const int ri = sm.ridx(i, s);
        float4 rd = sm.row[ri];
        const float w = alpha * zt + oma * rd.z;
        const float zn = fminf(fmaxf(w + rho_inv * rd.w, rd.x), rd.y);
        rd.w = rd.w + rho * (w - zn);
        rd.z = zn;
        sm.row[ri] = rd;
        bad = bad || !isfinite(zt);
      };
      upd(lane, o0);
      if (lane < 8) upd(32 + lane, o1);
      if (i == 0 && lane < NINIT) upd(NSLOT + lane, o2);
      if (lane < NV) {
        float* x = sm.V(i, V_X);
        x[lane] = alpha * xt + oma * x[lane];
      }
    }
    if (__any_sync(FULL, bad)) return it;
  }
  __syncwarp();
  return -1;
}

// ------------------------------------------------------------------------- kernel
__device__ __forceinline__ void prof_mark(const KParams& P, int lane, int stage, long long& t0) {
  if (P.profile) {
    const long long t1 = clock64();
    if (lane == 0) atomicAdd(P.prof + stage, (unsigned long long)(t1 - t0));
    t0 = t1;
  }
}

__global__ void __launch_bounds__(32) rti_kernel(const KParams P) {
  extern __shared__ __align__(16) float smem[];
  const int agent = blockIdx.x;
  if (agent >= P.n_agents) return;
  const int lane = threadIdx.x;
  const int NT = P.NT;
  const Layout L = make_layout(NT);
  Sm sm;
  sm.sinv = smem + L.sinv;
  sm.coef = smem + L.coef;
  sm.vec = smem + L.vec;
  sm.row = reinterpret_cast<float4*>(smem + L.row);
  sm.dsc = smem + L.dsc;
  sm.icoef = smem + L.icoef;
  sm.tbuf = smem + L.tbuf;
  sm.bc = smem + L.bc;
  sm.g = smem + L.g;
  sm.flags = reinterpret_cast<uint32_t*>(smem + L.flags);
  sm.NT = NT;
  long long t0 = P.profile ? clock64() : 0;

  // zero-initialise coefficients, rows, vectors; d = e = 1
  for (int k = lane; k < NT * C_SIZE; k += 32) sm.coef[k] = 0.f;
  const int nrow = NT * NSLOT + NINIT;
  for (int r = lane; r < nrow; r += 32) {
    sm.row[r] = make_float4(0.f, 0.f, 0.f, 0.f);
    sm.dsc[r] = 1.f;
  }
  for (int k = lane; k < NT * V_NUM * V_STRIDE; k += 32) sm.vec[k] = 0.f;
  for (int i = 0; i < NT; ++i)
    if (lane < NV) sm.V(i, V_E)[lane] = 1.f;
  if (lane < 20) sm.icoef[lane] = 0.f;
  for (int k = lane; k < 256; k += 32) sm.g[k] = 0.f;
  if (lane < 32) { sm.tbuf[lane] = 0.f; sm.tbuf[32 + lane] = 0.f; sm.tbuf[64 + lane] = 0.f; sm.tbuf[96 + lane] = 0.f; }
  __syncwarp();

  const rmpc_state st = P.states[agent];
  const rmpc_command cmd = P.cmds[agent];
  const rmpc_gait gait = P.gaits[agent];
  const bool warm = P.warm_start && P.prev != nullptr && P.prev_z != nullptr &&
                    P.prev[agent].status == RMPC_STATUS_OK;
  const float* pz = warm ? P.prev_z + (size_t)agent * NT * NV : nullptr;

  rmpc_solution out;
  {
    float* o = reinterpret_cast<float*>(&out);
    for (int k = 0; k < 33; ++k) o[k] = 0.f;
    out.status = RMPC_STATUS_OK;
    out.fail_iter = -1;
  }
  bool st_ok = true;
#pragma unroll
  for (int k = 0; k < 9; ++k) st_ok = st_ok && isfinite(st.q[k]) && isfinite(st.qd[k]);
  prof_mark(P, lane, 0, t0);

  bool ok = setup_nodes(P, sm, lane, st, cmd, gait, warm, pz) && st_ok;
  __syncwarp();
  prof_mark(P, lane, 2, t0);
  if (!ok) {
    out.status = RMPC_STATUS_NONFINITE_INPUT;
  } else {
    if (P.ruiz_iters > 0) ruiz(P, sm, lane);
    apply_scaling(P, sm, lane);
    prof_mark(P, lane, 3, t0);
    if (!factorize(P, sm, lane)) {
      out.status = RMPC_STATUS_SINGULAR;
    } else {
      prof_mark(P, lane, 4, t0);
      const int bad_it = admm(P, sm, lane);
      prof_mark(P, lane, 5, t0);
      if (bad_it >= 0) {
        out.status = RMPC_STATUS_DIVERGED;
        out.fail_iter = bad_it;
      }
    }
  }

  if (out.status == RMPC_STATUS_OK) {
    // residuals and objective on the unscaled problem (qp.cpp:192-200), z*, ||dz||_inf
    float prim = 0.f, dual = 0.f, dinf = 0.f;
    double obj = 0.0;
#pragma unroll 1
    for (int i = 0; i < NT; ++i) {
      float o0, o1, o2;
      row_view<OpSum>(sm, i, lane, V_X, o0, o1, o2);
      auto pr = [&](int s, float ax) {
        const int r = sm.ridx(i, s);
        prim = fmaxf(prim, fabsf(ax - sm.row[r].z) / sm.dsc[r]);
      };
      pr(lane, o0);
      if (lane < 8) pr(32 + lane, o1);
      if (i == 0 && lane < NINIT) pr(NSLOT + lane, o2);
      float* tc = sm.tbuf + (i & 1) * 64;
      const float* tp = sm.tbuf + ((i + 1) & 1) * 64;
      fill_t(sm, i, lane, tc, [](float4 r, float) { return r.w; });
      const float aty = col_view<OpSum>(sm, i, lane, tc, tp);
      if (lane < NV) {
        const float x = sm.V(i, V_X)[lane], e = sm.V(i, V_E)[lane];
        const float pd = sm.V(i, V_PD)[lane], qh = sm.V(i, V_QH)[lane];
        dual = fmaxf(dual, fabsf(pd * x + qh + aty) / e);
        obj += 0.5 * (double)pd * (double)x * (double)x + (double)qh * (double)x;
        dinf = fmaxf(dinf, fabsf(e * x));
      }
    }
    prim = wmax(prim);
    dual = wmax(dual);
    dinf = wmax(dinf);
    obj = wsumd(obj);
    out.prim_res = prim;
    out.dual_res = dual;
    out.delta_inf_norm = dinf;
    out.v_mpc = (float)obj;

    // z* = guess + dz (mpc.cpp:308-314), double guess + float step
    const bool want_z = P.z_out != nullptr;
#pragma unroll 1
    for (int i = 0; i < NT; ++i) {
      const uint32_t bits = sm.flags[i];
      double g = 0.0;
      if (lane < NV) {
        if (warm) {
          g = (double)pz[min(i + 1, NT - 1) * NV + lane];
        } else if (lane < 9) {
          g = lane == 0 ? st.q[0] : P.nominal[lane];
        } else if (lane >= 18) {
          const int c = (lane - 18) >> 1;
          const int na = __popc(bits);
          g = ((lane - 18) & 1) && ((bits >> c) & 1u) && na > 0 ? P.weight / na : 0.0;
        }
        const double zv = g + (double)sm.V(i, V_E)[lane] * (double)sm.V(i, V_X)[lane];
        if (want_z) P.z_out[((size_t)agent * NT + i) * NV + lane] = (float)zv;
        if (i < 2) reinterpret_cast<double*>(sm.sinv)[i * 32 + lane] = zv;  // S^-1 is dead now
      }
    }
    __syncwarp();
    // inverse dynamics at node 0 (mpc.cpp:320-330), FP64 on lane 0
    if (lane == 0) {
      const double* z0 = reinterpret_cast<const double*>(sm.sinv);
      const double* z1 = z0 + 32;
      double q[9], qd[9], qdd[9], F[8], gen[9];
      const double dt0 = P.dt[0];
      for (int k = 0; k < 9; ++k) {
        q[k] = z0[k];
        qd[k] = z0[NQ + k];
        qdd[k] = (z1[NQ + k] - z0[NQ + k]) / dt0;
      }
      for (int k = 0; k < 8; ++k) F[k] = z0[18 + k];
      inverse_dynamics(P, q, qd, qdd, F, gen);
      for (int b = 0; b < 3; ++b) out.base_residual[b] = (float)gen[b];
      for (int m = 0; m < 6; ++m) {
        out.tau_ff[m] = (float)gen[3 + m];
        out.q_set[m] = (float)q[3 + m];
        out.qd_set[m] = (float)qd[3 + m];
      }
      for (int k = 0; k < 8; ++k) out.f0[k] = (float)F[k];
    }
  } else if (P.z_out != nullptr) {
    for (int k = lane; k < NT * NV; k += 32) P.z_out[(size_t)agent * NT * NV + k] = 0.f;
  }
  prof_mark(P, lane, 6, t0);
  if (lane == 0) P.out[agent] = out;
}

}  // namespace rmpc_dev

int rmpc_kernel_setup(int NT) {
  const int bytes = rmpc_dev::smem_bytes(NT);
  return (int)cudaFuncSetAttribute(rmpc_dev::rti_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

int rmpc_launch_rti(const rmpc_dev::KParams& params, void* stream) {
  if (params.n_agents <= 0) return 0;
  const int bytes = rmpc_dev::smem_bytes(params.NT);
  rmpc_dev::rti_kernel<<<params.n_agents, 32, bytes, (cudaStream_t)stream>>>(params);
  return (int)cudaGetLastError();
}
