// rmpc_admm.cuh — stage ADMM: exactly n_qp iterations (qp.cpp:156-190) as two recurrences meeting at the middle node.
// Part of the fused solve kernel: included once, in order, by rmpc_kernel.cu.
#pragma once

#include "rmpc_device.cuh"
#include "rmpc_kin.cuh"

namespace rmpc_dev {

#ifndef FULL
#define FULL 0xffffffffu
#endif

// ------------------------------------------------------------------------- stage: ADMM
// One constraint-row update (qp.cpp:163-170) on the stored {lo, hi, z, t = rho z - y}; the
// store is predicated on `active` (r must point at a valid row either way).  Returns false
// on a non-finite z~ of an active row.
__device__ __forceinline__ bool row_update(float4* r, float* tr, bool active, float zt, float alpha,
                                           float oma, float rho, float rho_inv) {
  float4 rd = *r;
  const float y = fmaf(rho, rd.z, -rd.w);
  const float w = alpha * zt + oma * rd.z;
  const float zn = fminf(fmaxf(w + rho_inv * y, rd.x), rd.y);
  const float yn = y + rho * (w - zn);
  rd.z = zn;
  rd.w = fmaf(rho, zn, -yn);
  if (active) {
    *r = rd;
    *tr = rd.w;
  }
  return !active || isfinite(zt);
}

// [S_i^-1 ; W_i^T] u for lanes 0..28 (u published through buf, the block row from TMEM).
__device__ __forceinline__ float ext_mv(const Sm& sm, int i, int lane, float* buf, float u) {
  buf[lane] = lane < NV ? u : 0.f;
  float v[TCOLS];
  blk_load(sm, i, lane, v);
  __syncwarp();
  const float4* b4 = reinterpret_cast<const float4*>(buf);
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
  for (int q = 0; q < 6; ++q) {
    const float4 bb = b4[q];
    a0 = fmaf(v[4 * q], bb.x, a0);
    a1 = fmaf(v[4 * q + 1], bb.y, a1);
    a2 = fmaf(v[4 * q + 2], bb.z, a2);
    a3 = fmaf(v[4 * q + 3], bb.w, a3);
  }
  {
    const float2 bb = reinterpret_cast<const float2*>(buf)[12];
    a0 = fmaf(v[24], bb.x, a0);
    a1 = fmaf(v[25], bb.y, a1);
  }
  return lane < SROWS ? (a0 + a1) + (a2 + a3) : 0.f;
}

// The matvec half of ext_mv on an already loaded block row v (u published in buf).
__device__ __forceinline__ float block_row_dot(const float v[TCOLS], const float* buf, int lane) {
  const float4* b4 = reinterpret_cast<const float4*>(buf);
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
  for (int q = 0; q < 6; ++q) {
    const float4 bb = b4[q];
    a0 = fmaf(v[4 * q], bb.x, a0);
    a1 = fmaf(v[4 * q + 1], bb.y, a1);
    a2 = fmaf(v[4 * q + 2], bb.z, a2);
    a3 = fmaf(v[4 * q + 3], bb.w, a3);
  }
  const float2 bb = reinterpret_cast<const float2*>(buf)[12];
  a0 = fmaf(v[24], bb.x, a0);
  a1 = fmaf(v[25], bb.y, a1);
  return lane < SROWS ? (a0 + a1) + (a2 + a3) : 0.f;
}

struct AdmmConst {
  float rho, sigma, alpha, oma, rho_inv;
};

// Rows of node i that act on node-i variables only (contact forces, contact Jacobian rows,
// joint boxes; the initial-state rows at node 0): z~ from x~_i, then the row update.  Lanes
// 8c..8c+5 reduce rows t2/t3 of contact c; lane 8c takes t2, 8c+1 t3, 8c+2..4 boxes 3c..3c+2,
// 8c+6/8c+7 the force rows t0/t1 (8c+5 has no row).  Branch-free: every lane evaluates every
// candidate from clamped addresses and keeps its own.
__device__ __forceinline__ bool node_rows(const Sm& sm, int lane, int i, const float* xs,
                                          const AdmmConst& K) {
  const int c = lane >> 3, s = lane & 7;
  const float* cf = sm.C(i);
  const int col = chain_col(c, s < 6 ? s : 0);
  const float vd = xs[NQ + col];
  const float on = s < 6 ? 1.f : 0.f;
  float pa = on * (cf[C_JAQ + 9 * c + col] * xs[col] + cf[C_JA + 9 * c + col] * vd);
  float pb = on * cf[C_JB + 9 * c + col] * vd;
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) {
    pa += __shfl_xor_sync(FULL, pa, o);
    pb += __shfl_xor_sync(FULL, pb, o);
  }
  const int t = s & 1;  // force row t0 / t1 for s = 6 / 7
  const float zf = cf[C_FORCE + 4 * c + 2 * t] * xs[18 + 2 * c] + cf[C_FORCE + 4 * c + 2 * t + 1] * xs[19 + 2 * c];
  const int mb = 3 * c + (s >= 2 && s <= 4 ? s - 2 : 0);  // box index
  const float zb = cf[C_BOX + mb] * xs[mb < 6 ? 3 + mb : NQ + 3 + (mb - 6)];
  const float zt = s == 0 ? pa : (s == 1 ? pb : (s >= 6 ? zf : zb));
  const int slot = s == 0 ? 14 + 4 * c : (s == 1 ? 15 + 4 * c : (s >= 6 ? 12 + 4 * c + t : 28 + mb));
  bool ok = row_update(sm.R(i) + slot, sm.T(i) + slot, s != 5, zt, K.alpha, K.oma, K.rho, K.rho_inv);
  if (i == 0) {
    const int l = lane < NINIT ? lane : 0;
    ok = row_update(sm.R(-1) + INIT0 + l, sm.T(-1) + INIT0 + l, lane < NINIT, cf[C_INIT + l] * xs[l], K.alpha, K.oma, K.rho,
                    K.rho_inv) && ok;
  }
  return !ok;
}

// AdmmSolver::run (qp.cpp:156-190): exactly n_qp iterations from x = y = z = 0.  Returns the
// first iteration with a non-finite iterate, or -1 (pair-uniform).
//
// Two-sided solve of H x~ = r (factorize): warp 0 owns nodes [0, m) and the middle node m,
// warp 1 owns (m, T); each warp also does the node-local work of its nodes (r_i from the
// column view, the rows acting on node i alone, x_i), so the warps meet only at the middle:
//   top forward     i = 0..m-1:   u_i = r_i - rho U_{i-1} g_{i-1};  [s_i; g_i^dyn] = [S_i^-1; W_i^T] u_i
//   bottom forward  i = T-1..m+1: u_i = r_i - rho V_i g'_{i+1};     [s_i; g_i'^dyn] = [T_i^-1; W_i'^T] u_i
//   middle:         x_m = M^-1 (r_m - rho U_{m-1} g_{m-1} - rho V_m g'_{m+1})
//   top backward    i = m-1..0:   x_i = s_i - rho [S_i^-1(:, q) | W_i] xi_i,  xi = diag(a2,1) U_i^T x_{i+1}
//   bottom backward i = m+1..T-1: x_i = s_i - rho [T_i^-1(:, q), T_i^-1(:, qd) | W'_i] xi'_i,
//                                  xi' = (a1, a3) (x) V_{i-1}^T x_{i-1}
// with g = V^T s, g' = U^T s'.  z~ of the integration/dynamics rows comes out of the
// backward steps; no warp reduction sits on either recurrence.
__device__ int admm(const KParams& P, const Sm& sm, int lane, int warp) {
  const int NT = P.NT;
  const int m = mid_node(NT);
  const AdmmConst K{(float)P.rho, (float)P.sigma, (float)P.alpha, 1.f - (float)P.alpha,
                    (float)(1.0 / P.rho)};
  const float rho = K.rho;
  Terms T;
  build_terms(lane, T);
  TermBytes B;
  term_bytes<TV_T>(T, B);
  float* ubuf = sm.bc + 64 * warp;  // broadcast of u_i (this warp)
  float* xib = ubuf + 32;           // broadcast of xi_i (this warp)
  float* gb = sm.bc + 64 + 32;      // warp 1's xi buffer doubles as the g'_{m+1} hand-over
  // lane roles, all branch-free below: q_k lanes 0..8, qd_k lanes 9..17, F lanes 18..25,
  // W / dynamics lanes 26..28
  const bool is_q = lane < 9, is_qd = lane >= 9 && lane < 18, is_var = lane < NV;
  const bool is_dv = lane >= 9 && lane < NV, is_w = lane >= NV && lane < SROWS;
  const int kq = is_q ? lane : (is_qd ? lane - 9 : 0);    // k of q_k / qd_k
  const int jv = is_dv ? lane - 9 : 0;                     // index into v_b (node vars 9..25)
  const int bw = is_w ? lane - NV : (lane >= 9 && lane < 12 ? lane - 9 : 0);
  const float f_q = is_q ? 1.f : 0.f, f_qd = is_qd ? 1.f : 0.f, f_dv = is_dv ? 1.f : 0.f;
  auto r_of = [&](int i, bool first) {  // (sigma x - q^ + A^T(rho z - y)) restricted to node i
    const float cv = first ? 0.f : col_view<OpSum, TV_T>(sm, i, T, B);
    return is_var ? K.sigma * sm.V(i, V_X)[lane] - sm.V(i, V_QH)[lane] + cv : 0.f;
  };
  auto store_s = [&](int i, float s) {  // s_i, and g^dyn in the spare slots of node i
    float* vs = sm.V(i, V_S);
    if (lane < NV + 2) vs[lane] = s;
    if (lane == NV + 2) sm.V(i, V_X)[NV] = s;
  };
  auto gamma_of = [&](int i) { return bw < 2 ? sm.V(i, V_S)[NV + bw] : sm.V(i, V_X)[NV]; };
  auto finish_node = [&](int i) {  // node i's own rows and the x relaxation, from x~_i
    float* xs = sm.V(i, V_S);
    const bool b = node_rows(sm, lane, i, xs, K);
    if (is_var) {
      float* x = sm.V(i, V_X);
      x[lane] = K.alpha * xs[lane] + K.oma * x[lane];
    }
    return b;
  };
  // - rho U g : top correction of node i from node i-1 (coefficients of interval i-1)
  auto top_corr = [&](const float* cp, float gint, float g0, float g1, float g2) {
    const float gk = __shfl_sync(FULL, gint, kq);
    const float ci = cp[(is_q ? C_A1 : C_A3) + kq];
    return rho * ((f_q + f_qd) * ci * gk +
                  f_qd * (cp[C_DYNU + kq] * g0 + cp[C_DYNU + 12 + kq] * g1 + cp[C_DYNU + 24 + kq] * g2));
  };
  // - rho V g' : bottom correction of node i from node i+1 (coefficients of interval i)
  auto bot_corr = [&](const float* cf, float gint, float g0, float g1, float g2) {
    return rho * (f_q * cf[C_A2 + kq] * gint +
                  f_dv * (cf[C_DYNV + jv] * g0 + cf[C_DYNV + 20 + jv] * g1 + cf[C_DYNV + 40 + jv] * g2));
  };
  int first_bad = 0x7fffffff;  // this lane's first iteration with a non-finite value
#pragma unroll 1
  for (int it = 0; it < P.n_qp; ++it) {
    const bool first = it == 0;  // x = y = z = 0: r = -q^
    bool bad = false;
    // ---------------------------------------------------------------- forward
    float gint = 0.f, g0 = 0.f, g1 = 0.f, g2 = 0.f;  // g of the last eliminated node
    // software-pipelined: r of the next node is gathered while this node's TMEM row loads
    // (the middle's r waits for the barrier: the bottom half's previous backward writes the
    // interval-m rows it reads)
    float rc = warp == 0 ? (m > 0 ? r_of(0, first) : 0.f) : (NT - 1 > m ? r_of(NT - 1, first) : 0.f);
    if (warp == 0) {
#pragma unroll 1
      for (int i = 0; i < m; ++i) {
        const float u = rc - top_corr(sm.C(i - 1), gint, g0, g1, g2);
        ubuf[lane] = lane < NV ? u : 0.f;
        float v[TCOLS];
        blk_load_issue(sm, i, lane, v);
        if (i + 1 < m) rc = r_of(i + 1, first);
        blk_load_wait(sm, i, v);
        __syncwarp();
        const float s = block_row_dot(v, ubuf, lane);
        store_s(i, s);
        gint = f_q * sm.C(i)[C_A2 + kq] * s;
        g0 = __shfl_sync(FULL, s, 26);
        g1 = __shfl_sync(FULL, s, 27);
        g2 = __shfl_sync(FULL, s, 28);
        __syncwarp();
      }
    } else {
#pragma unroll 1
      for (int i = NT - 1; i > m; --i) {
        const float u = rc - bot_corr(sm.C(i), gint, g0, g1, g2);
        ubuf[lane] = lane < NV ? u : 0.f;
        float v[TCOLS];
        blk_load_issue(sm, i, lane, v);
        if (i - 1 > m) rc = r_of(i - 1, first);
        blk_load_wait(sm, i, v);
        __syncwarp();
        const float s = block_row_dot(v, ubuf, lane);
        store_s(i, s);
        const float* cp = sm.C(i - 1);  // g'_int_k = a1_k s[q_k] + a3_k s[qd_k]
        const float sq = __shfl_down_sync(FULL, s, 9);
        gint = f_q * (cp[C_A1 + kq] * s + cp[C_A3 + kq] * sq);
        g0 = __shfl_sync(FULL, s, 26);
        g1 = __shfl_sync(FULL, s, 27);
        g2 = __shfl_sync(FULL, s, 28);
        __syncwarp();
      }
      gb[lane] = lane < 9 ? gint : (lane == 9 ? g0 : (lane == 10 ? g1 : (lane == 11 ? g2 : 0.f)));
    }
    pair_sync(sm);
    // ---------------------------------------------------------------- middle
    if (warp == 0) {
      float u = r_of(m, first) - top_corr(sm.C(m - 1), gint, g0, g1, g2);
      if (m + 1 < NT) u -= bot_corr(sm.C(m), gb[kq], gb[9], gb[10], gb[11]);
      const float x = ext_mv(sm, m, lane, ubuf, u);
      if (is_var) sm.V(m, V_S)[lane] = x;
      bad = bad || !isfinite(x);
    }
    pair_sync(sm);
    // ---------------------------------------------------------------- backward
    if (warp == 0) {
      // software-pipelined: step i's TMEM row and xi are loaded before node i+1's own rows
      // (finish_node, independent of step i) are updated, and consumed after
#pragma unroll 1
      for (int i = m - 1; i >= 0; --i) {
        const float* cf = sm.C(i);
        float* vs = sm.V(i, V_S);
        const float* xn = sm.V(i + 1, V_S);
        // xi_k = a2_k (a1_k x[q_k] + a3_k x[qd_k]) (lanes 0..8), xi_b = u_b . x[qd] (9..11)
        const float dl = cf[C_A1 + kq] * xn[kq] + cf[C_A3 + kq] * xn[NQ + kq];
        const float* ub = cf + C_DYNU + 12 * bw;
        float a0 = ub[0] * xn[NQ], a1 = ub[1] * xn[NQ + 1], a2 = ub[2] * xn[NQ + 2];
        a0 = fmaf(ub[3], xn[NQ + 3], a0);
        a1 = fmaf(ub[4], xn[NQ + 4], a1);
        a2 = fmaf(ub[5], xn[NQ + 5], a2);
        a0 = fmaf(ub[6], xn[NQ + 6], a0);
        a1 = fmaf(ub[7], xn[NQ + 7], a1);
        a2 = fmaf(ub[8], xn[NQ + 8], a2);
        const float xd = a0 + a1 + a2;
        xib[lane] = is_q ? cf[C_A2 + kq] * dl : (lane < 12 ? xd : 0.f);
        __syncwarp();
        // lanes < 26: row j of S^-1 (cols 0..8 = column j) and W_b[j];  26..28: W_b, G_b
        float v[TCOLS];
        blk_load(sm, i, lane, v);
        float xi[12];
#pragma unroll
        for (int k = 0; k < 12; ++k) xi[k] = xib[k];
        float wg[3];
#pragma unroll
        for (int b = 0; b < 3; ++b) wg[b] = lane < NV ? v[NV + b] : cf[C_G + 3 * bw + b];
        const float vsl = vs[lane < NV ? lane : 0], gam = gamma_of(i);
        bad = finish_node(i + 1) || bad;
        float acc0 = 0.f, acc1 = 0.f;
#pragma unroll
        for (int k = 0; k < 9; k += 2) {
          acc0 = fmaf(v[k], xi[k], acc0);
          if (k + 1 < 9) acc1 = fmaf(v[k + 1], xi[k + 1], acc1);
        }
#pragma unroll
        for (int b = 0; b < 3; ++b) acc1 = fmaf(wg[b], xi[9 + b], acc1);
        const float acc = acc0 + acc1;
        const float xt = is_var ? vsl - rho * acc : 0.f;
        if (is_var) vs[lane] = xt;
        bad = bad || !isfinite(xt);
        // z~: integration row k (lane k) = a2 x~_i[q_k] + dl ; dynamics row b (lane 26+b) =
        // v_b.x~_i + u_b.x~_{i+1} = g_b - rho acc + xi_b
        const float xib_b = bw == 0 ? xi[9] : (bw == 1 ? xi[10] : xi[11]);
        const float zt = is_q ? fmaf(cf[C_A2 + kq], xt, dl) : gam - rho * acc + xib_b;
        const int slot = is_q ? kq : 9 + bw;
        bad = !row_update(sm.R(i) + slot, sm.T(i) + slot, is_q || is_w, zt, K.alpha, K.oma, K.rho, K.rho_inv) || bad;
        __syncwarp();
      }
      bad = finish_node(0) || bad;  // nodes m..1 were finished inside the loop
    } else {
#pragma unroll 1
      for (int i = m + 1; i < NT; ++i) {
        const float* cp = sm.C(i - 1);  // interval i-1 couples nodes i-1 and i
        const float* xp = sm.V(i - 1, V_S);
        float* vs = sm.V(i, V_S);
        // xi'_k = a2_k x_{i-1}[q_k] (lanes 0..8, published as a1 xi', a3 xi'); xi'_b = v_b . x_{i-1}
        const float xiv = cp[C_A2 + kq] * xp[kq];
        const float* vb = cp + C_DYNV + 20 * bw;
        float a0 = 0.f, a1 = 0.f, a2 = 0.f;
#pragma unroll
        for (int k = 0; k < 17; k += 3) {
          a0 = fmaf(vb[k], xp[9 + k], a0);
          if (k + 1 < 17) a1 = fmaf(vb[k + 1], xp[10 + k], a1);
          if (k + 2 < 17) a2 = fmaf(vb[k + 2], xp[11 + k], a2);
        }
        const float xd = a0 + a1 + a2;
        if (is_q) {
          xib[lane] = cp[C_A1 + kq] * xiv;
          xib[9 + lane] = cp[C_A3 + kq] * xiv;
        }
        if (lane >= 9 && lane < 12) xib[18 + bw] = xd;
        __syncwarp();
        float v[TCOLS];  // lanes < 26: row j of T^-1 and W'_b[j]; 26..28: W'_b, G'_b
        blk_load(sm, i, lane, v);
        float acc0 = 0.f, acc1 = 0.f;
#pragma unroll
        for (int k = 0; k < 9; ++k) {
          acc0 = fmaf(v[k], xib[k], acc0);
          acc1 = fmaf(v[NQ + k], xib[9 + k], acc1);
        }
#pragma unroll
        for (int b = 0; b < 3; ++b) acc0 = fmaf(lane < NV ? v[NV + b] : cp[C_G + 3 * bw + b], xib[18 + b], acc0);
        const float acc = acc0 + acc1;
        const float xt = is_var ? vs[lane] - rho * acc : 0.f;
        if (is_var) vs[lane] = xt;
        bad = bad || !isfinite(xt);
        const float xq = __shfl_down_sync(FULL, xt, 9);  // lane k: x_i[qd_k]
        // z~: integration row k = xi'_k + a1 x_i[q_k] + a3 x_i[qd_k];
        //     dynamics row b = v_b.x_{i-1} + u_b.x_i = xi'_b + g'_b - rho acc
        const float zt = is_q ? xiv + cp[C_A1 + kq] * xt + cp[C_A3 + kq] * xq
                              : xib[18 + bw] + gamma_of(i) - rho * acc;
        const int slot = is_q ? kq : 9 + bw;
        bad = !row_update(sm.R(i - 1) + slot, sm.T(i - 1) + slot, is_q || is_w, zt, K.alpha, K.oma, K.rho, K.rho_inv) || bad;
        __syncwarp();
        bad = finish_node(i) || bad;
      }
    }
    // no barrier between iterations: the halves exchange data only at the middle (the two
    // barriers above order every cross-half access), so a non-finite iterate is recorded here
    // and the pair agrees on the first one after the loop (qp.cpp:159-161 reports the first).
    if (bad && first_bad > it) first_bad = it;
  }
  const int wfirst = __reduce_min_sync(FULL, first_bad);
  int* fb = reinterpret_cast<int*>(sm.bc);  // the broadcast buffers are free after the loop
  pair_sync(sm);
  if (lane == 0) fb[warp] = wfirst;
  pair_sync(sm);
  const int f = fb[0] < fb[1] ? fb[0] : fb[1];
  return f == 0x7fffffff ? -1 : f;
}

}  // namespace rmpc_dev
