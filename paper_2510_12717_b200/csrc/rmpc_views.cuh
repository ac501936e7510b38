// rmpc_views.cuh — column view (A^T v per variable, 17 uniform terms per lane) and row view (A v per constraint slot) of the padded per-node QP.
// Part of the fused solve kernel: included once, in order, by rmpc_kernel.cu.
#pragma once

#include "rmpc_device.cuh"
#include "rmpc_kin.cuh"

namespace rmpc_dev {

#ifndef FULL
#define FULL 0xffffffffu
#endif

// ------------------------------------------------------------------------- column view
// Every variable j of node i is touched by at most 17 constraint rows, from its own block
// and from block i-1 (integration/dynamics rows of interval i-1; the initial-state rows in
// block -1 for node 0).  Lane j keeps the 17 (coefficient offset, row offset) pairs of the
// universal pattern in registers; absent rows point at a zero coefficient, so the same
// instruction stream serves every node.  Terms 2..5 are contact row t2 (JA), which acts on
// q for a swing contact and on qd for a stance contact: a per-node 0/1 multiplier selects.
struct Terms {
  int co[17];
  int to[17];
  int kind;  // 0 q, 1 qd, 2 F, 3 idle
};

__device__ __forceinline__ void build_terms(int lane, Terms& T) {
#pragma unroll
  for (int k = 0; k < 17; ++k) { T.co[k] = C_ZERO; T.to[k] = 0; }
  const int CS = C_SIZE;
  if (lane < 9) {
    const int k = lane;
    T.kind = 0;
    T.co[0] = C_A2 + k;        T.to[0] = k;
    T.co[1] = -CS + C_A1 + k;      T.to[1] = -NSLOT + k;
#pragma unroll
    for (int c = 0; c < 4; ++c) { T.co[2 + c] = C_JAQ + 9 * c + k; T.to[2 + c] = 14 + 4 * c; }
    if (k >= 3) { T.co[6] = C_BOX + k - 3; T.to[6] = 28 + k - 3; }
    T.co[7] = C_INIT + k;               T.to[7] = -NSLOT + INIT0 + k;
  } else if (lane < 18) {
    const int k = lane - 9;
    T.kind = 1;
    T.co[0] = -CS + C_A3 + k;  T.to[0] = -NSLOT + k;
    T.co[1] = -CS + C_DYNU + k;         T.to[1] = -NSLOT + 9;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      T.co[2 + c] = C_JA + 9 * c + k; T.to[2 + c] = 14 + 4 * c;
      T.co[6 + c] = C_JB + 9 * c + k; T.to[6 + c] = 15 + 4 * c;
    }
    T.co[10] = -CS + C_DYNU + 12 + k;   T.to[10] = -NSLOT + 10;
    T.co[11] = -CS + C_DYNU + 24 + k;   T.to[11] = -NSLOT + 11;
#pragma unroll
    for (int b = 0; b < 3; ++b) { T.co[12 + b] = C_DYNV + 20 * b + k; T.to[12 + b] = 9 + b; }
    if (k >= 3) { T.co[15] = C_BOX + 6 + k - 3; T.to[15] = 34 + k - 3; }
    T.co[16] = C_INIT + 9 + k;          T.to[16] = -NSLOT + INIT0 + 9 + k;
  } else if (lane < NV) {
    const int c = (lane - 18) >> 1, a = (lane - 18) & 1, idx = lane - 9;
    T.kind = 2;
    T.co[0] = C_DYNV + idx;             T.to[0] = 9;
    T.co[1] = C_DYNV + 20 + idx;        T.to[1] = 10;
    T.co[6] = C_DYNV + 40 + idx;        T.to[6] = 11;
    T.co[7] = C_FORCE + 4 * c + a;      T.to[7] = 12 + 4 * c;
    T.co[8] = C_FORCE + 4 * c + 2 + a;  T.to[8] = 13 + 4 * c;
  } else {
    T.kind = 3;
  }
}

// Byte offsets of the 17 terms: coefficients relative to C(i), row values relative to R(i)
// (+12 = t, +8 = {z, t}) or to D(i).
struct TermBytes {
  int cb[17];
  int tb[17];
};
enum { TV_T = 0, TV_Y = 1, TV_D = 2 };
template <int MODE>
__device__ __forceinline__ void term_bytes(const Terms& T, TermBytes& B) {
#pragma unroll
  for (int k = 0; k < 17; ++k) {
    B.cb[k] = T.co[k] * 4;
    B.tb[k] = MODE == TV_Y ? T.to[k] * 16 + 8 : T.to[k] * 4;
  }
}

// acc_j = Op_r (A_rj, t_r) over the rows touching var j of node i; t_r is rows[r].t (TV_T),
// y_r = rho z_r - t_r (TV_Y) or the Ruiz row scale d_r (TV_D).
template <class Op, int MODE>
__device__ __forceinline__ float col_view(const Sm& sm, int i, const Terms& T, const TermBytes& B,
                                          float rho = 0.f) {
  const char* cb = reinterpret_cast<const char*>(sm.C(i));
  const char* tb = MODE == TV_D ? reinterpret_cast<const char*>(sm.D(i))
                   : (MODE == TV_T ? reinterpret_cast<const char*>(sm.T(i))
                                   : reinterpret_cast<const char*>(sm.R(i)));
  float acc[4] = {Op::id(), Op::id(), Op::id(), Op::id()};  // four chains: 5 deep instead of 9
#pragma unroll
  for (int k = 0; k < 17; ++k) {
    const float c = *reinterpret_cast<const float*>(cb + B.cb[k]);
    float v;
    if (MODE == TV_Y) {
      const float2 zt = *reinterpret_cast<const float2*>(tb + B.tb[k]);
      v = fmaf(rho, zt.x, -zt.y);
    } else {
      v = *reinterpret_cast<const float*>(tb + B.tb[k]);
    }
    acc[k & 3] = Op::comb(acc[k & 3], c, v);
  }
  return Op::red(Op::red(acc[0], acc[1]), Op::red(acc[2], acc[3]));
}

// ------------------------------------------------------------------------- full row view
// out_r = Op_j(A_rj, v_j) for the 40 slots of node i (lane l: slot l in o0, slot 32+l in
// o1) and the 18 initial-state rows (lane l < 18 in o2; C_INIT is zero unless i == 0).  Used
// by Ruiz and the residuals; the ADMM loop gets the integration/dynamics rows from the
// recurrences instead.  Branch-free: every lane runs the same instructions with clamped
// indices and zero coefficients (C_ZERO) where its slot has no term.
template <class Op>
__device__ __forceinline__ void row_view(const Sm& sm, int i, int lane, int which, float& o0,
                                         float& o1, float& o2) {
  const float* cf = sm.C(i);
  const float* vi = sm.V(i, which);
  const float* vn = (i + 1 < sm.NT) ? sm.V(i + 1, which) : vi;  // coefficients are 0 then
  // own terms: integration (lanes 0..8), force cones (12..27, t < 2), boxes (28..31)
  const bool li = lane < 9, lb = lane >= 28;
  const int cq = (lane - 12) >> 2, tq = (lane - 12) & 3;
  const bool lf = lane >= 12 && lane < 28 && tq < 2;
  const int c1 = li ? C_A1 + lane : (lf ? C_FORCE + 4 * cq + 2 * tq : (lb ? C_BOX + lane - 28 : C_ZERO));
  const int c2 = li ? C_A2 + lane : (lf ? C_FORCE + 4 * cq + 2 * tq + 1 : C_ZERO);
  const int c3 = li ? C_A3 + lane : C_ZERO;
  const float* v1 = li ? vn + lane : vi + (lf ? 18 + 2 * cq : (lb ? lane - 25 : 0));
  const float* v2 = vi + (li ? lane : (lf ? 19 + 2 * cq : 0));
  const float* v3 = vn + (li ? NQ + lane : 0);
  o0 = Op::comb(Op::comb(Op::comb(Op::id(), cf[c1], *v1), cf[c2], *v2), cf[c3], *v3);
  const int m4 = 4 + lane;  // slot 32 + lane: boxes 4..11
  o1 = Op::comb(Op::id(), cf[lane < 8 ? C_BOX + m4 : C_ZERO],
                vi[lane < 8 ? (m4 < 6 ? 3 + m4 : NQ + m4 - 3) : 0]);
  o2 = Op::comb(Op::id(), cf[lane < NINIT ? C_INIT + lane : C_ZERO], vi[lane < NINIT ? lane : 0]);
  // dynamics rows 9..11: lane = support entry (qd_{i+1}: 0..8, node-i vars 9..25)
  const bool du = lane < 9, dv = lane >= 9 && lane < NV;
  const int dc = du ? C_DYNU + lane : (dv ? C_DYNV + lane - 9 : C_ZERO);
  const int ds = du ? 12 : (dv ? 20 : 0);
  const float dval = du ? vn[NQ + lane] : vi[dv ? lane : 0];
  const float p0 = Op::comb(Op::id(), cf[dc], dval), p1 = Op::comb(Op::id(), cf[dc + ds], dval),
              p2 = Op::comb(Op::id(), cf[dc + 2 * ds], dval), p3 = Op::id();
  // contact Jacobian rows t2, t3: 8-lane group per contact
  const int c = lane >> 3, s = lane & 7;
  const int col = chain_col(c, s < 6 ? s : 0);
  const float vd = vi[NQ + col];
  const float pa = Op::comb(Op::comb(Op::id(), cf[s < 6 ? C_JAQ + 9 * c + col : C_ZERO], vi[col]),
                            cf[s < 6 ? C_JA + 9 * c + col : C_ZERO], vd);
  const float pb = Op::comb(Op::id(), cf[s < 6 ? C_JB + 9 * c + col : C_ZERO], vd);
  // Transposed butterflies: 4 dynamics partials -> row (lane >> 3) in 6 shuffles; the
  // (pa, pb) pair -> pa in lanes 8c..8c+3, pb in 8c+4..8c+7 in 3 shuffles.
  const bool h = lane & 16, g = lane & 8, e = lane & 4;
  float k0 = h ? p2 : p0, k1 = h ? p3 : p1;
  k0 = Op::red(k0, __shfl_xor_sync(FULL, h ? p0 : p2, 16));
  k1 = Op::red(k1, __shfl_xor_sync(FULL, h ? p1 : p3, 16));
  float kd = Op::red(g ? k1 : k0, __shfl_xor_sync(FULL, g ? k0 : k1, 8));
  float kc = Op::red(e ? pb : pa, __shfl_xor_sync(FULL, e ? pa : pb, 4));
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) kd = Op::red(kd, __shfl_xor_sync(FULL, kd, o));
#pragma unroll
  for (int o = 2; o > 0; o >>= 1) kc = Op::red(kc, __shfl_xor_sync(FULL, kc, o));
  const bool ld = lane >= 9 && lane < 12, lc = lane >= 12 && lane < 28 && tq >= 2;
  const float rd = __shfl_sync(FULL, kd, ld ? 8 * (lane - 9) : 0);
  const float rc = __shfl_sync(FULL, kc, lc ? 8 * cq + 4 * (tq - 2) : 0);
  o0 = ld ? rd : (lc ? rc : o0);
}

}  // namespace rmpc_dev
