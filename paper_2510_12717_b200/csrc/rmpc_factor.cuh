// rmpc_factor.cuh — stage factorize: two-sided block elimination of H with Schur-complement inverses (2x2-pivot Gauss-Jordan).
// Part of the fused solve kernel: included once, in order, by rmpc_kernel.cu.
#pragma once

#include "rmpc_device.cuh"
#include "rmpc_kin.cuh"

namespace rmpc_dev {

#ifndef FULL
#define FULL 0xffffffffu
#endif

// ------------------------------------------------------------------------- stage: factor
// Two-sided block elimination of the block-tridiagonal H (26 x 26 blocks):
//   top    (warp 0, i = 0..m-1):   S_i = D_i - rho^2 U_{i-1} G_{i-1} U_{i-1}^T,  G = V^T S^-1 V
//   bottom (warp 1, i = T-1..m+1): T_i = D_i - rho^2 V_i G'_i V_i^T,            G' = U^T T^-1 U
//   middle (warp 0, i = m):        M   = D_m - (top update) - (bottom update)
// with U/V the node-(i+1)/node-i parts of the 12 rows of interval i.  Lane j holds row j of a
// block in registers; inverses by Gauss-Jordan (SPD, no pivoting).  Stored per node (29 x 26):
// rows 0..25 the inverse, rows 26..28 W_b = S_i^-1 v_b (top) or W'_b = T_i^-1 u_b (bottom).
// G_dd / G'_dd (3 x 3 dynamics part) go to C(i)[C_G] of the coupling interval.

// D_i = P^_i + sigma I + rho sum (rows touching node i) a a^T, row j of it into S.
__device__ __forceinline__ void assemble_diag(const KParams& P, const Sm& sm, int i, int j, float S[NV]) {
  const float rho = (float)P.rho, sigma = (float)P.sigma;
  const float* cf = sm.C(i);
  const float* cp = sm.C(i - 1);  // block -1 is zero for i == 0
  float dg = 0.f, pt = 0.f;
  int pidx = -1;
  if (j < NV) dg = phat(P, sm, i, j) + sigma;
  if (j < 9) {
    const float a2 = cf[C_A2 + j], a1 = cp[C_A1 + j], a3 = cp[C_A3 + j];
    const float bx = j >= 3 ? cf[C_BOX + j - 3] : 0.f, bi = cf[C_INIT + j];
    dg += rho * (a2 * a2 + a1 * a1 + bx * bx + bi * bi);
    pt = rho * a1 * a3;
    pidx = NQ + j;
  } else if (j < 18) {
    const int k = j - 9;
    const float a1 = cp[C_A1 + k], a3 = cp[C_A3 + k];
    const float bx = k >= 3 ? cf[C_BOX + 6 + k - 3] : 0.f, bi = cf[C_INIT + j];
    dg += rho * (a3 * a3 + bx * bx + bi * bi);
    pt = rho * a1 * a3;
    pidx = k;
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
#pragma unroll
  for (int b = 0; b < 3; ++b) {  // dynamics rows of interval i (qd_i, F_i) and i-1 (qd_i)
    const float* vb = cf + C_DYNV + 20 * b;
    const float s = (j >= 9 && j < NV) ? rho * vb[j - 9] : 0.f;
    const float4* v4 = reinterpret_cast<const float4*>(vb);
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      const float4 w = v4[q];
      if (9 + 4 * q < NV) S[9 + 4 * q] = fmaf(s, w.x, S[9 + 4 * q]);
      if (10 + 4 * q < NV) S[10 + 4 * q] = fmaf(s, w.y, S[10 + 4 * q]);
      if (11 + 4 * q < NV) S[11 + 4 * q] = fmaf(s, w.z, S[11 + 4 * q]);
      if (12 + 4 * q < NV) S[12 + 4 * q] = fmaf(s, w.w, S[12 + 4 * q]);
    }
    const float* ub = cp + C_DYNU + 12 * b;
    const float s2 = (j >= 9 && j < 18) ? rho * ub[j - 9] : 0.f;
#pragma unroll
    for (int m = 0; m < 9; ++m) S[NQ + m] = fmaf(s2, ub[m], S[NQ + m]);
  }
#pragma unroll
  for (int c = 0; c < 4; ++c) {  // contact rows t2/t3: velocity on qd (stance), height on q
    const float *ja = cf + C_JA + 9 * c, *jb = cf + C_JB + 9 * c, *jq = cf + C_JAQ + 9 * c;
    const bool mine = j >= 9 && j < 18;
    const float s0 = mine ? rho * ja[j - 9] : 0.f, s1 = mine ? rho * jb[j - 9] : 0.f;
    const float sq = j < 9 ? rho * jq[j] : 0.f;
#pragma unroll
    for (int m = 0; m < 9; ++m) {
      S[NQ + m] = fmaf(s0, ja[m], fmaf(s1, jb[m], S[NQ + m]));
      S[m] = fmaf(sq, jq[m], S[m]);
    }
  }
}

// In-place Gauss-Jordan inverse of the SPD block held row-wise by the warp (lane j: row j),
// pivot rows exchanged through shared memory.  Returns false on a non-positive pivot.
// 2 x 2 pivot blocks: 13 elimination steps instead of 26 (the step's
// latency -- pivot rows through shared memory, one reciprocal -- is what bounds the
// factorization).  Pivot rows k, k+1 go through `buf` (>= 112 floats, the warp's G scratch,
// double-buffered).  Block GJ on [[a, b], [c, d]] = S[k:k+2, k:k+2] with P = its inverse:
//   rows j != k, k+1:  S_j -= (f P) [R_k; R_k+1],  S_j[k:k+2] = -(f P),   f = S_j[k:k+2]
//   rows k, k+1:       [R_k; R_k+1] <- P [R_k; R_k+1],  S[k:k+2, k:k+2] = P
// written as one FMA pair per element for every lane (the pivot rows hold S_j = R_k / R_k+1).
// A 2 x 2 pivot block of an SPD matrix is PD: a > 0 and det > 0 (both LDL^T pivots positive,
// the reference's SingularityError test, ldl.cpp:155-160).
__device__ __forceinline__ bool gauss_jordan2(int j, float S[NV], float* buf) {
  bool good = true;
#pragma unroll
  for (int p = 0; p < NV / 2; ++p) {
    const int k = 2 * p;
    float* bb = buf + 56 * (p & 1);
    if (j == k || j == k + 1) {
      float4* b4 = reinterpret_cast<float4*>(bb + 28 * (j - k));
#pragma unroll
      for (int q = 0; q < 6; ++q) b4[q] = make_float4(S[4 * q], S[4 * q + 1], S[4 * q + 2], S[4 * q + 3]);
      reinterpret_cast<float2*>(bb + 28 * (j - k))[12] = make_float2(S[24], S[25]);
    }
    __syncwarp();
    float R0[NV], R1[NV];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const float4* b4 = reinterpret_cast<const float4*>(bb + 28 * r);
      float* R = r == 0 ? R0 : R1;
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        const float4 w = b4[q];
        R[4 * q] = w.x; R[4 * q + 1] = w.y; R[4 * q + 2] = w.z; R[4 * q + 3] = w.w;
      }
      const float2 w = reinterpret_cast<const float2*>(bb + 28 * r)[12];
      R[24] = w.x;
      R[25] = w.y;
    }
    const float a = R0[k], b = R0[k + 1], c = R1[k], d = R1[k + 1];
    const float det = fmaf(a, d, -b * c);
    good = good && a > 0.f && det > 0.f;
    const float idet = __frcp_rn(det);
    const float p00 = d * idet, p01 = -b * idet, p10 = -c * idet, p11 = a * idet;
    const float f0 = S[k], f1 = S[k + 1];
    const bool m0 = j == k, m1 = j == k + 1;
    const float al0 = m0 ? 1.f - p00 : (m1 ? -p10 : fmaf(f0, p00, f1 * p10));
    const float al1 = m0 ? -p01 : (m1 ? 1.f - p11 : fmaf(f0, p01, f1 * p11));
#pragma unroll
    for (int l = 0; l < NV; ++l) S[l] = fmaf(-al0, R0[l], fmaf(-al1, R1[l], S[l]));
    S[k] = m0 ? p00 : (m1 ? p10 : -al0);
    S[k + 1] = m0 ? p01 : (m1 ? p11 : -al1);
  }
  return good;
}

__device__ __forceinline__ void store_block(const Sm& sm, int i, int j, const float S[NV], const float W[3],
                                            float* tr) {
#pragma unroll
  for (int b = 0; b < 3; ++b) tr[32 * b + j] = W[b];
  __syncwarp();
  const bool wrow = j >= NV && j < SROWS;
  const float* src = tr + 32 * (wrow ? j - NV : 0);
  float v[TCOLS];
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = wrow ? src[k] : S[k];
#pragma unroll
  for (int b = 0; b < 3; ++b) v[NV + b] = wrow ? 0.f : W[b];
#pragma unroll
  for (int k = SROWS; k < TCOLS; ++k) v[k] = 0.f;
  blk_store(sm, i, j, v);
  __syncwarp();  // tr is reused by the caller
}

// Top Schur step after S_i^-1 (rows in S): W_b = S^-1 v_b, the node block into TMEM, G_dd ->
// C(i)[C_G], and the update Yp (rows j < 18, cols < 18) of node i+1: rho^2 U_i G_i U_i^T.
__device__ __forceinline__ void top_schur(const KParams& P, const Sm& sm, int i, int j, const float S[NV],
                                          float Yp[18]) {
  const float rho = (float)P.rho;
  const float* cf = sm.C(i);
  float* G = sm.scr;  // the top warp's 12 x 13 G block
  float W[3];
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    const float* vb = cf + C_DYNV + 20 * b;
    float acc = 0.f;
#pragma unroll
    for (int l = 9; l < NV; ++l) acc = fmaf(S[l], vb[l - 9], acc);
    W[b] = j < NV ? acc : 0.f;
  }
  store_block(sm, i, j, S, W, G);
  // G_dd[b][b2] = v_b . W_b2 over node vars 9..25, lane 3 b + b2 < 9, from W^T still in G
  const int gb = j < 9 ? j / 3 : 0, gb2 = j < 9 ? j % 3 : 0;
  float gacc0 = 0.f, gacc1 = 0.f;
#pragma unroll
  for (int l = 0; l < 17; l += 2) {
    gacc0 = fmaf(cf[C_DYNV + 20 * gb + l], G[32 * gb2 + 9 + l], gacc0);
    if (l + 1 < 17) gacc1 = fmaf(cf[C_DYNV + 20 * gb + l + 1], G[32 * gb2 + 10 + l], gacc1);
  }
  const float gacc = gacc0 + gacc1;
  const float gv = 0.5f * (gacc + __shfl_sync(FULL, gacc, 3 * gb2 + gb));
  __syncwarp();  // W^T read before G overwrites it
  if (j < 9) {
    const float a2 = cf[C_A2 + j];
#pragma unroll
    for (int k = 0; k < 9; ++k) G[j * 13 + k] = a2 * S[k] * cf[C_A2 + k];
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      G[j * 13 + 9 + b] = a2 * W[b];
      G[(9 + b) * 13 + j] = a2 * W[b];
    }
  }
  if (j < 9) {
    G[(9 + gb) * 13 + 9 + gb2] = gv;
    sm.C(i)[C_G + 3 * gb + gb2] = gv;
  }
  __syncwarp();
  float Z[12];
  if (j < 9) {
    const float a1 = cf[C_A1 + j];
#pragma unroll
    for (int s = 0; s < 12; ++s) Z[s] = a1 * G[j * 13 + s];
  } else if (j < 18) {
    const int k = j - 9;
    const float a3 = cf[C_A3 + k];
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
  for (int m = 0; m < 9; ++m) Yp[m] = r2 * Z[m] * cf[C_A1 + m];
#pragma unroll
  for (int k = 0; k < 9; ++k)
    Yp[NQ + k] = r2 * (Z[k] * cf[C_A3 + k] + Z[9] * cf[C_DYNU + k] + Z[10] * cf[C_DYNU + 12 + k] +
                       Z[11] * cf[C_DYNU + 24 + k]);
  __syncwarp();
}

// Update of node `iv` (the upper node of interval iv) from the bottom half: row j of
// rho^2 V_iv G'_iv V_iv^T, G' (12 x 13) in G.
__device__ __forceinline__ void bottom_update(const KParams& P, const Sm& sm, int iv, int j, const float* G,
                                              float Yb[NV]) {
  const float* cp = sm.C(iv);
  float Z[12];  // Z[j][s] = sum_r V[j][r] G'[r][s]
  if (j < 9) {
    const float a2 = cp[C_A2 + j];
#pragma unroll
    for (int s = 0; s < 12; ++s) Z[s] = a2 * G[j * 13 + s];
  } else if (j < NV) {
    const float v0 = cp[C_DYNV + j - 9], v1 = cp[C_DYNV + 20 + j - 9], v2 = cp[C_DYNV + 40 + j - 9];
#pragma unroll
    for (int s = 0; s < 12; ++s) Z[s] = v0 * G[9 * 13 + s] + v1 * G[10 * 13 + s] + v2 * G[11 * 13 + s];
  } else {
#pragma unroll
    for (int s = 0; s < 12; ++s) Z[s] = 0.f;
  }
  const float r2 = (float)P.rho * (float)P.rho;
#pragma unroll
  for (int l = 0; l < 9; ++l) Yb[l] = r2 * Z[l] * cp[C_A2 + l];
#pragma unroll
  for (int l = 9; l < NV; ++l)
    Yb[l] = r2 * (Z[9] * cp[C_DYNV + l - 9] + Z[10] * cp[C_DYNV + 20 + l - 9] + Z[11] * cp[C_DYNV + 40 + l - 9]);
}

// Bottom Schur step after T_i^-1 (rows in S), interval i-1 couples nodes i-1 and i:
// W'_b = T^-1 u_b, the node block into TMEM, G'_dd -> C(i-1)[C_G], G' = U^T T^-1 U (12 x 12)
// into the bottom warp's scratch (read by the top warp at the middle) and the update Yb of
// node i-1.
__device__ __forceinline__ void bottom_schur(const KParams& P, const Sm& sm, int i, int j, const float S[NV],
                                             float Yb[NV]) {
  const float* cp = sm.C(i - 1);
  float* G = sm.scr + G_SCR;
  float W[3];
#pragma unroll
  for (int b = 0; b < 3; ++b) {  // W'_b[j] = sum_k T^-1[j][9+k] u_b[k]
    const float* ub = cp + C_DYNU + 12 * b;
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < 9; ++k) acc = fmaf(S[NQ + k], ub[k], acc);
    W[b] = j < NV ? acc : 0.f;
  }
  store_block(sm, i, j, S, W, G);
  // G'_dd[b][b2] = u_b . W'_b2 over qd (node vars 9..17), lane 3 b + b2 < 9
  const int gb = j < 9 ? j / 3 : 0, gb2 = j < 9 ? j % 3 : 0;
  float gacc0 = 0.f, gacc1 = 0.f;
#pragma unroll
  for (int l = 0; l < 9; l += 2) {
    gacc0 = fmaf(cp[C_DYNU + 12 * gb + l], G[32 * gb2 + 9 + l], gacc0);
    if (l + 1 < 9) gacc1 = fmaf(cp[C_DYNU + 12 * gb + l + 1], G[32 * gb2 + 10 + l], gacc1);
  }
  const float gacc = gacc0 + gacc1;
  const float gv = 0.5f * (gacc + __shfl_sync(FULL, gacc, 3 * gb2 + gb));
  __syncwarp();  // W'^T read before G overwrites it
  // int-int / int-dyn parts: lane k (row k) and lane 9+k (row 9+k) of T^-1
  float Pk[9];
#pragma unroll
  for (int l = 0; l < 9; ++l) Pk[l] = cp[C_A1 + l] * S[l] + cp[C_A3 + l] * S[NQ + l];
  const float a1 = j < 9 ? cp[C_A1 + j] : 0.f, a3 = j < 9 ? cp[C_A3 + j] : 0.f;
#pragma unroll
  for (int l = 0; l < 9; ++l) {
    const float q = __shfl_down_sync(FULL, Pk[l], 9);
    if (j < 9) G[j * 13 + l] = a1 * Pk[l] + a3 * q;
  }
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    const float w9 = __shfl_down_sync(FULL, W[b], 9);
    if (j < 9) {
      const float g = a1 * W[b] + a3 * w9;
      G[j * 13 + 9 + b] = g;
      G[(9 + b) * 13 + j] = g;
    }
  }
  if (j < 9) {
    G[(9 + gb) * 13 + 9 + gb2] = gv;
    sm.C(i - 1)[C_G + 3 * gb + gb2] = gv;
  }
  __syncwarp();
  bottom_update(P, sm, i - 1, j, G, Yb);
}

// Returns false (pair-uniform) on a non-positive pivot (SingularityError, ldl.cpp:155-160).
// Both warps run the same loop (one Gauss-Jordan / assembly instance in the code): step t
// factorizes node t (warp 0, top) or node T-1-t (warp 1, bottom); warp 0's last step is the
// middle node, whose bottom update it rebuilds from the G' block the bottom warp left in its
// scratch.
__device__ bool factorize(const KParams& P, const Sm& sm, int lane, int warp) {
  const int NT = P.NT;
  const int m = mid_node(NT);
  const int nbot = NT - 1 - m;
  const int steps = (m > nbot ? m : nbot) + 1;
  const int j = lane;
  bool good = true;
  float Y[NV];  // update of the next node to eliminate (top: rows/cols < 18 non-zero)
#pragma unroll
  for (int l = 0; l < NV; ++l) Y[l] = 0.f;
#pragma unroll 1
  for (int t = 0; t < steps; ++t) {
    const bool middle = t == steps - 1;
    if (middle) {
      pair_sync(sm);  // the bottom half's G' of interval m is complete
      if (warp == 1) break;
    }
    const int i = warp == 0 ? (middle ? m : t) : NT - 1 - t;
    const bool active = middle || (warp == 0 ? t < m : t < nbot);
    if (!active) continue;  // the shorter half waits at the middle
    float S[NV];
    assemble_diag(P, sm, i, j, S);
    if (middle && m + 1 < NT) {
      float Yb[NV];
      bottom_update(P, sm, m, j, sm.scr + G_SCR, Yb);
#pragma unroll
      for (int l = 0; l < NV; ++l) S[l] -= Yb[l];
    }
#pragma unroll
    for (int l = 0; l < NV; ++l) S[l] -= Y[l];
    __syncwarp();
    good = gauss_jordan2(j, S, sm.scr + G_SCR * warp) && good;
    if (middle) {
      const float W0[3] = {0.f, 0.f, 0.f};
      store_block(sm, i, j, S, W0, sm.scr);
    } else if (warp == 0) {
      float Yp[18];
      top_schur(P, sm, i, j, S, Yp);
#pragma unroll
      for (int l = 0; l < NV; ++l) Y[l] = l < 18 ? Yp[l] : 0.f;
    } else {
      bottom_schur(P, sm, i, j, S, Y);
    }
  }
  return pair_and(sm, good);
}

}  // namespace rmpc_dev
