// rmpc_squad4.cuh — long squads: the lane-per-agent schedule-shared ADMM of rmpc_squad.cuh for
// horizons 11..20, where one warp's TMEM lane cannot hold a half of the horizon (five 98-column
// node slabs per thread).  Part of the fused solve kernel: included once, after rmpc_squad.cuh,
// by rmpc_kernel.cu.
//
// A long squad is up to 32 agents of one schedule on four warps, one CTA per squad:
//   warp 0  top-A     nodes 0 .. nA-1             (lane quarter 0, + the initial-state rows)
//   warp 1  bottom-A  nodes i0 .. T-1              (quarter 1)
//   warp 2  top-B     nodes nA .. m (m the middle) (quarter 2)
//   warp 3  bottom-B  nodes m+1 .. i0-1            (quarter 3)
// Each half's recurrences run through its two warps in turn (the node chain is sequential):
// forward top-A -> top-B, bottom-A -> bottom-B, the middle node split over top-B / bottom-B as
// in rmpc_squad.cuh, backward top-B -> top-A, bottom-B -> bottom-A.  The hand-overs are
// producer / consumer pairs of named barriers (bar.arrive by the producer, bar.sync by the
// consumer) over vectors in shared memory.  Interval rows live in the slab of their lower node,
// except interval m (the pair's cross elements, as for squads) and interval i0-1 between the two
// bottom warps (cross elements too: both warps update or read it).
#pragma once

#include "rmpc_squad.cuh"

namespace rmpc_dev {

// Cross-thread elements, named barriers and the layout of a long squad: rmpc_device.cuh.

__device__ __forceinline__ void s4_arrive(int id) { asm volatile("bar.arrive %0, 64;" ::"r"(id) : "memory"); }
__device__ __forceinline__ void s4_sync(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }
__device__ __forceinline__ void s4_all() { asm volatile("bar.sync %0, 128;" ::"r"(S4B_ALL) : "memory"); }

// One warp's part of AdmmSolver::run (qp.cpp:156-190) for the agent of its lane: the steps of
// sq_admm_top / sq_admm_bot (rmpc_squad.cuh) over this warp's nodes.  role: 0 top-A, 1 bottom-A,
// 2 top-B, 3 bottom-B.  Returns the first iteration with a non-finite iterate (or INT_MAX).
__device__ __forceinline__ int sq4_admm(const KParams& P, const Sq& q, const AdmmConst& K, int role) {
  const int NT = q.NT, m = q.m, nA = sq4_na(NT), i0 = sq4_i0(NT);
  const float rho = K.rho;
  const bool top = (role & 1) == 0, inner = role >= 2;
  int first_bad = 0x7fffffff;
  if (role == 3 && P.n_qp > 0) s4_arrive(S4B_TM);  // interval m's rows (zero) for the first middle step
  // (one iteration loop per half, as sq_admm_top / sq_admm_bot: a loop holding both halves' code
  // costs registers)
  if (top) {
#pragma unroll 1
    for (int it = 0; it < P.n_qp; ++it) {
      const bool first = it == 0;
      bool bad = false;
      // ============================================================ top half
      float gint[9], g[3], tp[12], xn[NV];
      const int f0 = inner ? nA : 0, f1 = inner ? m : nA;  // this warp's forward nodes [f0, f1) (+ m for B)
      if (!inner) {
#pragma unroll
        for (int k = 0; k < 9; ++k) gint[k] = 0.f;
        g[0] = g[1] = g[2] = 0.f;
#pragma unroll
        for (int k = 0; k < 12; ++k) tp[k] = 0.f;
      } else {
        s4_sync(S4B_TF);  // top-A's forward sweep is done
#pragma unroll
        for (int k = 0; k < 9; ++k) gint[k] = q.cx(S4X_HTF + k);
#pragma unroll
        for (int k = 0; k < 3; ++k) g[k] = q.cx(S4X_HTF + 9 + k);
#pragma unroll
        for (int k = 0; k < 12; ++k) tp[k] = q.cx(S4X_HTF + 12 + k);
      }
#pragma unroll 1
      for (int i = f0; i < f1; ++i) {
        const int b = i - f0;
        float ti[12];
        tq_ld<12>(q.slab(b) + SQ_TI, ti);  // (waited for inside sq_rhs)
        float u[NV];
        sq_rhs(P, q, i, b, ti, tp, u);
        sq_top_corr(q.C(i - 1), gint, g, rho, u);
        sq_matvec_tm(q.MF(i), u, q.slab(b) + SQ_S, 8);
        tq_wait_st();
        float s9[9], s3[3];
        tq_ld<9>(q.slab(b) + SQ_S, s9);
        tq_ld<3>(q.slab(b) + SQ_S + 26, s3);
        tq_wait_ld();
        tq_fence<9>(s9);
        tq_fence<3>(s3);
        const float* cf = q.C(i);
#pragma unroll
        for (int k = 0; k < 9; ++k) gint[k] = cf[C_A2 + k] * s9[k];
        g[0] = s3[0];
        g[1] = s3[1];
        g[2] = s3[2];
#pragma unroll
        for (int k = 0; k < 12; ++k) tp[k] = ti[k];
      }
      if (!inner) {  // hand the chain to top-B
#pragma unroll
        for (int k = 0; k < 9; ++k) q.cx(S4X_HTF + k) = gint[k];
#pragma unroll
        for (int k = 0; k < 3; ++k) q.cx(S4X_HTF + 9 + k) = g[k];
#pragma unroll
        for (int k = 0; k < 12; ++k) q.cx(S4X_HTF + 12 + k) = tp[k];
        s4_arrive(S4B_TF);
        s4_sync(S4B_TB);  // top-B's backward sweep hands x~_nA back
#pragma unroll
        for (int j = 0; j < NV; ++j) xn[j] = q.cx(S4X_HTB + j);
      } else {  // the middle node, split with bottom-B (rmpc_squad.cuh)
        const int b = m - nA;
        float ti[12], u[NV];
        tq_wait_st();
        s4_sync(S4B_TM);  // interval m's rows are written (bottom-B's first backward step)
#pragma unroll
        for (int k = 0; k < 12; ++k) ti[k] = q.cx(SQX_TM + k);
        sq_rhs(P, q, m, b, ti, tp, u);
        sq_top_corr(q.C(m - 1), gint, g, rho, u);
#pragma unroll
        for (int j = 0; j < NV; ++j) q.cx(S4X_UA + j) = u[j];
        s4_sync(S4B_MID);  // bottom-B's forward sweep is done (g'_{m+1})
        float gb[12];
#pragma unroll
        for (int k = 0; k < 12; ++k) gb[k] = q.cx(SQX_GB + k);
        sq_bot_corr(q.C(m), gb, gb + 9, rho, u);
        bad = sq_matvec_mid(q, q.MF(m), u, 0, 4) || bad;
        s4_sync(S4B_MID);  // x~_m published
#pragma unroll
        for (int j = 0; j < NV; ++j) xn[j] = q.cx(SQX_XM + j);
      }
      // backward: nodes i = (B: m-1 .. nA, A: nA-1 .. 0), each then the own rows of node i+1
      const int b1 = inner ? nA : 0;  // lowest node stepped by this warp
#pragma unroll 1
      for (int i = (inner ? m - 1 : nA - 1); i >= b1 - 1; --i) {
        float xc[NV];
        const bool step = i >= b1;
        if (step) {
          const int b = i - b1;
          const float* cf = q.C(i);
          float s[SROWS], ti[12];
          tq_ld<SROWS>(q.slab(b) + SQ_S, s);
          tq_ld<12>(q.slab(b) + SQ_TI, ti);
          float dl[9], xi[12];
#pragma unroll
          for (int k = 0; k < 9; ++k) {
            dl[k] = cf[C_A1 + k] * xn[k] + cf[C_A3 + k] * xn[NQ + k];
            xi[k] = cf[C_A2 + k] * dl[k];
          }
#pragma unroll
          for (int bb = 0; bb < 3; ++bb) {
            float a0 = 0.f, a1 = 0.f;
#pragma unroll
            for (int k = 0; k < 9; ++k) {
              if (k & 1) a1 = fmaf(cf[C_DYNU + 12 * bb + k], xn[NQ + k], a1);
              else a0 = fmaf(cf[C_DYNU + 12 * bb + k], xn[NQ + k], a0);
            }
            xi[9 + bb] = a0 + a1;
          }
#pragma unroll
          for (int r = 0; r < 12; ++r) q.pv(q.XS(r)) = xi[r];
          const float* M = q.MF(i);
          float acc[NV];
#pragma unroll
          for (int j = 0; j < NV; ++j) acc[j] = 0.f;
          sq_axpy_tm(q, M, 9, 12, acc);
          tq_wait_ld();
          tq_fence<SROWS>(s);
          tq_fence<12>(ti);
#pragma unroll
          for (int j = 0; j < NV; ++j) {
            xc[j] = s[j] - rho * acc[j];
            bad = bad || !isfinite(xc[j]);
          }
#pragma unroll
          for (int k = 0; k < 9; ++k) {
            const float zt = fmaf(cf[C_A2 + k], xc[k], dl[k]);
            sq_rupd_eq(ti[k], q.LO(i, k), first, zt, K);
            bad = bad || !isfinite(zt);
          }
#pragma unroll
          for (int bb = 0; bb < 3; ++bb) {
            float a = 0.f;
#pragma unroll
            for (int k = 0; k < 9; ++k) a = fmaf(M[(26 + bb) * SQ_MROW + k], xi[k], a);
#pragma unroll
            for (int b2 = 0; b2 < 3; ++b2) a = fmaf(cf[C_G + 3 * bb + b2], xi[9 + b2], a);
            const float zt = s[26 + bb] - rho * a + xi[9 + bb];
            sq_rupd_eq(ti[9 + bb], q.LO(i, 9 + bb), first, zt, K);
            bad = bad || !isfinite(zt);
          }
          tq_st<NV>(q.slab(b) + SQ_S, xc);
          tq_st<12>(q.slab(b) + SQ_TI, ti);
        }
        // node i+1's own rows: always this warp's but for top-A's first step (node nA: top-B's)
        if (inner || i + 1 < nA) bad = sq_finish_node(q, i + 1, i + 1 - b1, xn, first, K) || bad;
        tq_wait_st();
        if (step) {
#pragma unroll
          for (int j = 0; j < NV; ++j) xn[j] = xc[j];
        }
      }
      if (inner) {  // hand x~_nA to top-A
#pragma unroll
        for (int j = 0; j < NV; ++j) q.cx(S4X_HTB + j) = xn[j];
        s4_arrive(S4B_TB);
      }
      if (bad && first_bad > it) first_bad = it;
    }
  } else {
#pragma unroll 1
    for (int it = 0; it < P.n_qp; ++it) {
      const bool first = it == 0;
      bool bad = false;
      // ============================================================ bottom half
      float gint[9], g[3], ti[12], xp[NV];
      const int f0 = inner ? i0 - 1 : NT - 1, f1 = inner ? m : i0 - 1;  // forward nodes f0 down to f1+1
      if (!inner) {
#pragma unroll
        for (int k = 0; k < 9; ++k) gint[k] = 0.f;
        g[0] = g[1] = g[2] = 0.f;
        tq_ld<12>(q.slab(NT - 1 - i0) + SQ_TI, ti);  // interval T-1 (zero rows)
        tq_wait_ld();
        tq_fence<12>(ti);
      } else {
        s4_sync(S4B_BF);  // bottom-A's forward sweep is done
#pragma unroll
        for (int k = 0; k < 9; ++k) gint[k] = q.cx(S4X_HBF + k);
#pragma unroll
        for (int k = 0; k < 3; ++k) g[k] = q.cx(S4X_HBF + 9 + k);
#pragma unroll
        for (int k = 0; k < 12; ++k) ti[k] = q.cx(S4X_BT + k);  // interval i0-1
      }
      const int base = inner ? m + 1 : i0;  // this warp's lowest node (slab 0)
#pragma unroll 1
      for (int i = f0; i > f1; --i) {
        const int b = i - base;
        float tp[12];
        if (i - 1 >= base) {
          tq_ld<12>(q.slab(b - 1) + SQ_TI, tp);  // (waited for inside sq_rhs)
        } else {  // the interval below this warp's nodes: BT (bottom-A) or interval m (bottom-B)
#pragma unroll
          for (int k = 0; k < 12; ++k) tp[k] = q.cx((inner ? SQX_TM : S4X_BT) + k);
        }
        float u[NV];
        sq_rhs(P, q, i, b, ti, tp, u);
        sq_bot_corr(q.C(i), gint, g, rho, u);
        sq_matvec_tm(q.MF(i), u, q.slab(b) + SQ_S, 8);
        tq_wait_st();
        float s18[18], s3[3];
        tq_ld<18>(q.slab(b) + SQ_S, s18);
        tq_ld<3>(q.slab(b) + SQ_S + 26, s3);
        tq_wait_ld();
        tq_fence<18>(s18);
        tq_fence<3>(s3);
        const float* cp = q.C(i - 1);
#pragma unroll
        for (int k = 0; k < 9; ++k) gint[k] = cp[C_A1 + k] * s18[k] + cp[C_A3 + k] * s18[NQ + k];
        g[0] = s3[0];
        g[1] = s3[1];
        g[2] = s3[2];
#pragma unroll
        for (int k = 0; k < 12; ++k) ti[k] = tp[k];
      }
      if (!inner) {  // hand the chain to bottom-B
#pragma unroll
        for (int k = 0; k < 9; ++k) q.cx(S4X_HBF + k) = gint[k];
#pragma unroll
        for (int k = 0; k < 3; ++k) q.cx(S4X_HBF + 9 + k) = g[k];
        s4_arrive(S4B_BF);
        s4_sync(S4B_BB);  // bottom-B's backward sweep hands x~_{i0-1} back
#pragma unroll
        for (int j = 0; j < NV; ++j) xp[j] = q.cx(S4X_HBB + j);
      } else {  // the middle node's rows 16..25
#pragma unroll
        for (int k = 0; k < 9; ++k) q.cx(SQX_GB + k) = gint[k];
        q.cx(SQX_GB + 9) = g[0];
        q.cx(SQX_GB + 10) = g[1];
        q.cx(SQX_GB + 11) = g[2];
        s4_sync(S4B_MID);  // (top-B's u_m is published)
        float u[NV];
#pragma unroll
        for (int j = 0; j < NV; ++j) u[j] = q.cx(S4X_UA + j);
        sq_bot_corr(q.C(m), gint, g, rho, u);
        bad = sq_matvec_mid(q, q.MF(m), u, 4, 3) || bad;
        s4_sync(S4B_MID);  // x~_m published
#pragma unroll
        for (int j = 0; j < NV; ++j) xp[j] = q.cx(SQX_XM + j);
      }
      // backward: nodes i = base .. (B: i0-1, A: T-1)
      const int top_node = inner ? i0 - 1 : NT - 1;
#pragma unroll 1
      for (int i = base; i <= top_node; ++i) {
        const int b = i - base;
        const float* cp = q.C(i - 1);
        float s[SROWS], tr[12];
        tq_ld<SROWS>(q.slab(b) + SQ_S, s);
        const bool own_tr = i - 1 >= base;
        if (own_tr) {
          tq_ld<12>(q.slab(b - 1) + SQ_TI, tr);
        } else {
#pragma unroll
          for (int k = 0; k < 12; ++k) tr[k] = q.cx((inner ? SQX_TM : S4X_BT) + k);
        }
        float xiv[9], xib[21];
#pragma unroll
        for (int k = 0; k < 9; ++k) {
          xiv[k] = cp[C_A2 + k] * xp[k];
          xib[k] = cp[C_A1 + k] * xiv[k];
          xib[9 + k] = cp[C_A3 + k] * xiv[k];
        }
#pragma unroll
        for (int bb = 0; bb < 3; ++bb) {
          float a0 = 0.f, a1 = 0.f, a2 = 0.f;
#pragma unroll
          for (int k = 0; k < 17; ++k) {
            const float t = cp[C_DYNV + 20 * bb + k] * xp[9 + k];
            if (k % 3 == 0) a0 += t; else if (k % 3 == 1) a1 += t; else a2 += t;
          }
          xib[18 + bb] = a0 + a1 + a2;
        }
#pragma unroll
        for (int r = 0; r < 21; ++r) q.pv(q.XS(r)) = xib[r];
        const float* M = q.MF(i);
        float acc[NV];
#pragma unroll
        for (int j = 0; j < NV; ++j) acc[j] = 0.f;
        sq_axpy_tm(q, M, 18, 21, acc);
        tq_wait_ld();
        tq_fence<SROWS>(s);
        if (own_tr) tq_fence<12>(tr);
        float xt[NV];
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          xt[j] = s[j] - rho * acc[j];
          bad = bad || !isfinite(xt[j]);
        }
#pragma unroll
        for (int k = 0; k < 9; ++k) {
          const float zt = xiv[k] + cp[C_A1 + k] * xt[k] + cp[C_A3 + k] * xt[NQ + k];
          sq_rupd_eq(tr[k], q.LO(i - 1, k), first, zt, K);
          bad = bad || !isfinite(zt);
        }
#pragma unroll
        for (int bb = 0; bb < 3; ++bb) {
          float a = 0.f;
#pragma unroll
          for (int k = 0; k < 18; ++k) a = fmaf(M[(26 + bb) * SQ_MROW + k], xib[k], a);
#pragma unroll
          for (int b2 = 0; b2 < 3; ++b2) a = fmaf(cp[C_G + 3 * bb + b2], xib[18 + b2], a);
          const float zt = xib[18 + bb] + s[26 + bb] - rho * a;
          sq_rupd_eq(tr[9 + bb], q.LO(i - 1, 9 + bb), first, zt, K);
          bad = bad || !isfinite(zt);
        }
        tq_st<NV>(q.slab(b) + SQ_S, xt);
        if (own_tr) {
          tq_st<12>(q.slab(b - 1) + SQ_TI, tr);
        } else {
#pragma unroll
          for (int k = 0; k < 12; ++k) q.cx((inner ? SQX_TM : S4X_BT) + k) = tr[k];
          if (inner && it + 1 < P.n_qp) s4_arrive(S4B_TM);  // for top-B's next middle step
        }
        bad = sq_finish_node(q, i, b, xt, first, K) || bad;
        tq_wait_st();
#pragma unroll
        for (int j = 0; j < NV; ++j) xp[j] = xt[j];
      }
      if (inner) {  // hand x~_{i0-1} to bottom-A
#pragma unroll
        for (int j = 0; j < NV; ++j) q.cx(S4X_HBB + j) = xp[j];
        s4_arrive(S4B_BB);
      }
      if (bad && first_bad > it) first_bad = it;
    }
  }
  return first_bad;
}

// ------------------------------------------------------------------------- setup / solve / kernel
// this warp's node range in a long squad: [lo, lo + own)
__device__ __forceinline__ void sq4_nodes(int NT, int role, int& lo, int& own) {
  const int m = mid_node(NT), nA = sq4_na(NT), i0 = sq4_i0(NT);
  if (role == 0) { lo = 0; own = nA; }
  else if (role == 2) { lo = nA; own = m + 1 - nA; }
  else if (role == 3) { lo = m + 1; own = i0 - 1 - m; }
  else { lo = i0; own = NT - i0; }
}

// sq_setup (rmpc_squad.cuh) for one warp of a long squad: its slabs, its nodes' agent-dependent
// bounds and q^ parts, the initial-state rows on top-A; the cross-element interval rows start at 0.
__device__ __forceinline__ bool sq4_setup(const KParams& P, const Sq& q, int role, int lo, int own,
                                          const rmpc_state& st, const rmpc_command& cmd, const rmpc_gait& gait,
                                          const double* con_pz) {
  float zero[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) zero[k] = 0.f;
#pragma unroll 1
  for (int b = 0; b < own; ++b) {
    tq_st<32>(q.slab(b), zero);
    tq_st<32>(q.slab(b) + 32, zero);
    tq_st<32>(q.slab(b) + 64, zero);
    tq_st<SQ_SLAB - 96>(q.slab(b) + 96, zero);
  }
  if (role == 0) tq_st<NINIT>(q.tm + SQ_TINIT, zero);
  for (int k = 0; k < q.nb * SQ_NZ; ++k) q.pv(k) = 0.f;
  if (role == 3)
    for (int k = 0; k < 12; ++k) q.cx(SQX_TM + k) = 0.f;
  if (role == 1)
    for (int k = 0; k < 12; ++k) q.cx(S4X_BT + k) = 0.f;
  bool same = true;
#pragma unroll 1
  for (int b = 0; b < own; ++b) {
    const int i = lo + b;
    double swt[4];
    const uint32_t bits = node_schedule(P, gait, i, swt);
    same = same && bits == q.flags[i];
    const float* ei = q.e + i * NV;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int j = a == 0 ? 0 : (a == 1 ? 1 : (a == 2 ? 9 : 11));
      double g, des;
      guess_and_target(P, i, j, false, nullptr, st, cmd, q.flags[i], g, des);
      q.pv(q.QA(b, a)) = to_f(wcost(P, j) * P.dt[i] * (g - des)) * ei[j];
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      float v = 0.f;
      if (i > 0 && !((bits >> c) & 1u)) {
        const double h = bezier_height(swt[c], P.z_swing, P.v_to, P.v_td);
        v = bound_f(h - con_pz[c]) * q.DS(i, 14 + 4 * c);
      }
      q.pv(q.AL(b, c)) = v;
    }
  }
  if (role == 0) {
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      const double gq = k == 0 ? st.q[0] : P.nominal[k];
      const double rq = st.q[k] - gq, rqd = st.qd[k] - 0.0;
      q.pv(q.IL(k)) = bound_f(rq) * q.DS(-1, INIT0 + k);
      q.pv(q.IL(9 + k)) = bound_f(rqd) * q.DS(-1, INIT0 + 9 + k);
    }
  }
  tq_wait_st();
  return same;
}

// sq_finish (rmpc_squad.cuh) for one warp of a long squad: its nodes [lo, lo + own); the values
// at the warp boundaries (x and interval rows of the node below this warp's first) are
// published by their owners first.  role 0 (top-A) combines the partials and writes the record.
__device__ __forceinline__ void sq4_finish(const KParams& P, const Sq& q, int role, int lo, int own, int agent,
                                           bool write, int status, int fail_iter, const rmpc_state& st,
                                           const rmpc_command& cmd, float* fin) {
  const int NT = q.NT, m = q.m, lane = q.lane, nA = sq4_na(NT), i0 = sq4_i0(NT);
  const bool top = role == 0;  // (the writer of the record)
  double* fz = reinterpret_cast<double*>(fin);                  // z* rows of nodes 0, 1 (FP64), [2][26][32]
  float* fc = fin + 2 * 2 * NV * 32;                            // [warp][prim, dual, dinf, obj (FP64)][32]
  float* xp = fin + 2 * 2 * NV * 32 + 4 * 5 * 32 + (threadIdx.x >> 5) * 32 * 27;  // transpose buffer [lane][27]
  const bool ok = status == RMPC_STATUS_OK;
  const float rho = (float)P.rho;
  const bool eqz = P.n_qp > 0;  // equality rows: z = lo after the first update
  {  // the warp boundaries: x of the node below each warp's first, and interval nA-1's rows
    float x[NV], t[12];
    if (role != 1) {
      const int bx = role == 0 ? nA - 1 : (role == 2 ? m - nA : i0 - 1 - (m + 1));
      tq_ld<NV>(q.slab(bx) + SQ_X, x);
      if (role == 0) tq_ld<12>(q.slab(nA - 1) + SQ_TI, t);
      tq_wait_ld();
      tq_fence<NV>(x);
      const int dst = role == 0 ? S4X_HTB : (role == 2 ? SQX_XM : S4X_HBB);
#pragma unroll
      for (int j = 0; j < NV; ++j) q.cx(dst + j) = x[j];
      if (role == 0) {
        tq_fence<12>(t);
#pragma unroll
        for (int k = 0; k < 12; ++k) q.cx(S4X_HTF + k) = t[k];
      }
    }
  }
  s4_all();
  float prim = 0.f, dual = 0.f, dinf = 0.f;
  double obj = 0.0;
  float xprev[NV], tp[12];
  if (role == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) xprev[j] = 0.f;
#pragma unroll
    for (int k = 0; k < 12; ++k) tp[k] = 0.f;
  } else {
    const int sx = role == 2 ? S4X_HTB : (role == 3 ? SQX_XM : S4X_HBB);
    const int st_ = role == 2 ? S4X_HTF : (role == 3 ? SQX_TM : S4X_BT);
#pragma unroll
    for (int j = 0; j < NV; ++j) xprev[j] = q.cx(sx + j);
#pragma unroll
    for (int k = 0; k < 12; ++k) tp[k] = q.cx(st_ + k);
  }
#pragma unroll 1
  for (int b = 0; b < own; ++b) {
    const int i = lo + b;
    const bool node0 = i == 0;
    float x[NV], to[28], ti[12], tin[NINIT];
    tq_ld<NV>(q.slab(b) + SQ_X, x);
    tq_ld<28>(q.slab(b) + SQ_TO, to);
    if (i == m || i == i0 - 1) {  // interval m / i0-1: cross elements
#pragma unroll
      for (int k = 0; k < 12; ++k) ti[k] = q.cx((i == m ? SQX_TM : S4X_BT) + k);
    } else {
      tq_ld<12>(q.slab(b) + SQ_TI, ti);
    }
    if (node0) tq_ld<NINIT>(q.tm + SQ_TINIT, tin);
    tq_wait_ld();
    tq_fence<NV>(x);
    tq_fence<28>(to);
    tq_fence<12>(ti);
    if (node0) tq_fence<NINIT>(tin);
    const float* cf = q.C(i);
    const float* cp = q.C(i - 1);
    const uint32_t bits = q.flags[i];
    // z of node i's own rows (equality rows: lo), y = rho z - t
    float zo[28], yo[28], yi[12], yp[12], yin[NINIT];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      zo[4 * c] = q.pv(q.ZO(b, 2 * c));
      zo[4 * c + 1] = q.pv(q.ZO(b, 2 * c + 1));
      const float lo2 = ((bits >> c) & 1u) || i == 0 ? q.LO(i, 14 + 4 * c) : q.pv(q.AL(b, c));
      zo[4 * c + 2] = eqz ? lo2 : 0.f;
      zo[4 * c + 3] = eqz ? q.LO(i, 15 + 4 * c) : 0.f;
    }
#pragma unroll
    for (int mb = 0; mb < 12; ++mb) zo[16 + mb] = q.pv(q.ZO(b, 8 + mb));
#pragma unroll
    for (int k = 0; k < 28; ++k) yo[k] = fmaf(rho, zo[k], -to[k]);
#pragma unroll
    for (int k = 0; k < 12; ++k) {
      yi[k] = fmaf(rho, eqz ? q.LO(i, k) : 0.f, -ti[k]);
      yp[k] = fmaf(rho, eqz ? q.LO(i - 1, k) : 0.f, -tp[k]);
    }
    if (node0) {
#pragma unroll
      for (int l = 0; l < NINIT; ++l) yin[l] = fmaf(rho, eqz ? q.pv(q.IL(l)) : 0.f, -tin[l]);
    }
    // primal residual, own rows of node i
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      float pa = 0.f, pb = 0.f;
#pragma unroll
      for (int s = 0; s < 6; ++s) {
        const int col = s < 3 ? s : (c < 2 ? 6 : 3) + s - 3;
        pa = fmaf(cf[C_JAQ + 9 * c + col], x[col], pa);
        pa = fmaf(cf[C_JA + 9 * c + col], x[NQ + col], pa);
        pb = fmaf(cf[C_JB + 9 * c + col], x[NQ + col], pb);
      }
      const float f0 = x[18 + 2 * c], f1 = x[19 + 2 * c];
      const float a0 = cf[C_FORCE + 4 * c] * f0 + cf[C_FORCE + 4 * c + 1] * f1;
      const float a1 = cf[C_FORCE + 4 * c + 2] * f0 + cf[C_FORCE + 4 * c + 3] * f1;
      const int s0 = 12 + 4 * c;
      prim = fmaxf(prim, __fdividef(fabsf(a0 - zo[4 * c]), q.DS(i, s0)));
      prim = fmaxf(prim, __fdividef(fabsf(a1 - zo[4 * c + 1]), q.DS(i, s0 + 1)));
      prim = fmaxf(prim, __fdividef(fabsf(pa - zo[4 * c + 2]), q.DS(i, s0 + 2)));
      prim = fmaxf(prim, __fdividef(fabsf(pb - zo[4 * c + 3]), q.DS(i, s0 + 3)));
    }
#pragma unroll
    for (int mb = 0; mb < 12; ++mb) {
      const float ab = cf[C_BOX + mb] * x[mb < 6 ? 3 + mb : 6 + mb];
      prim = fmaxf(prim, __fdividef(fabsf(ab - zo[16 + mb]), q.DS(i, 28 + mb)));
    }
    if (node0) {
#pragma unroll
      for (int l = 0; l < NINIT; ++l) {
        const float zl = eqz ? q.pv(q.IL(l)) : 0.f;
        prim = fmaxf(prim, __fdividef(fabsf(cf[C_INIT + l] * x[l] - zl), q.DS(-1, INIT0 + l)));
      }
    }
    // interval i-1 rows: x_{i-1} (xprev) and x_i
    if (i > 0) {
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        const float a = cp[C_A1 + k] * x[k] + cp[C_A2 + k] * xprev[k] + cp[C_A3 + k] * x[NQ + k];
        prim = fmaxf(prim, __fdividef(fabsf(a - (eqz ? q.LO(i - 1, k) : 0.f)), q.DS(i - 1, k)));
      }
#pragma unroll
      for (int bb = 0; bb < 3; ++bb) {
        float a = 0.f;
#pragma unroll
        for (int k = 0; k < 9; ++k) a = fmaf(cp[C_DYNU + 12 * bb + k], x[NQ + k], a);
#pragma unroll
        for (int jv = 0; jv < 17; ++jv) a = fmaf(cp[C_DYNV + 20 * bb + jv], xprev[9 + jv], a);
        prim = fmaxf(prim, __fdividef(fabsf(a - (eqz ? q.LO(i - 1, 9 + bb) : 0.f)), q.DS(i - 1, 9 + bb)));
      }
    }
    // dual residual |P^ x + q^ + A^T y| / e, objective, z*
    float aty[NV], zr[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) aty[j] = 0.f;
    sq_colview(cf, cp, yi, yp, yo, yin, node0, aty);
    float qh[NV];
    sq_qhat(q, i, b, qh);
    const float* ei = q.e + i * NV;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const float e = ei[j];
      const float ph = (float)(wcost(P, j) * P.dt[i]) * e * e;
      dual = fmaxf(dual, __fdividef(fabsf(ph * x[j] + qh[j] + aty[j]), e));
      double g, des;
      guess_and_target(P, i, j, false, nullptr, st, cmd, bits, g, des);
      const double w = wcost(P, j) * P.dt[i];
      const double dz = (double)e * (double)x[j];
      obj += 0.5 * w * dz * dz + w * (g - des) * dz;
      dinf = fmaxf(dinf, fabsf(e * x[j]));
      const double zv = g + dz;  // z* = guess + dz (mpc.cpp:308-314)
      zr[j] = ok ? (float)zv : 0.f;  // (a failed agent's z* is zero)
      if (i < 2) fz[(i * NV + j) * 32 + lane] = zv;
    }
    if (P.z_out) tq_st<NV>(q.slab(b) + SQ_X, zr);  // (node i's x columns are dead: sq_zstar_out)
    if (P.act_out && write) {  // final active set (scaled space)
      uint8_t* ao = P.act_out + (size_t)agent * (NT + 1) * NSLOT + (size_t)(i + 1) * NSLOT;
      auto code = [](float lo, float hi, float z) -> uint8_t {
        return lo == hi ? 3 : (z == lo ? 1 : (z == hi ? 2 : 0));
      };
      for (int sl = 0; sl < NSLOT; ++sl) {
        uint8_t cd = 3;
        if (sl >= 12 && sl < 28 && ((sl - 12) & 3) < 2) cd = code(q.LO(i, sl), q.HI(i, sl), zo[sl - 12]);
        if (sl >= 28) cd = code(q.LO(i, sl), q.HI(i, sl), zo[sl - 12]);
        ao[sl] = ok ? cd : 3;
      }
      if (node0)
        for (int sl = 0; sl < NSLOT; ++sl) ao[sl - NSLOT] = 3;
    }
#pragma unroll
    for (int j = 0; j < NV; ++j) xprev[j] = x[j];
#pragma unroll
    for (int k = 0; k < 12; ++k) tp[k] = ti[k];
  }
  if (P.z_out) sq_zstar_out(P, q, xp, lo, own, agent, write);
  {
    float* fw = fc + (threadIdx.x >> 5) * 5 * 32;
    fw[lane] = prim;
    fw[32 + lane] = dual;
    fw[64 + lane] = dinf;
    reinterpret_cast<double*>(fw + 96)[lane] = obj;
  }
  s4_all();
  if (!top) return;
  prim = dual = dinf = 0.f;
  obj = 0.0;
#pragma unroll
  for (int w = 0; w < 4; ++w) {  // the same order for every agent
    const float* fw = fc + w * 5 * 32;
    prim = fmaxf(prim, fw[lane]);
    dual = fmaxf(dual, fw[32 + lane]);
    dinf = fmaxf(dinf, fw[64 + lane]);
    obj += reinterpret_cast<const double*>(fw + 96)[lane];
  }
  rmpc_solution out;
  {
    float* o = reinterpret_cast<float*>(&out);
    for (int k = 0; k < 33; ++k) o[k] = 0.f;
  }
  out.status = status;
  out.fail_iter = status == RMPC_STATUS_DIVERGED ? fail_iter : -1;
  if (ok) {
    out.prim_res = prim;
    out.dual_res = dual;
    out.delta_inf_norm = dinf;
    out.v_mpc = (float)obj;
    double qv[9], qd[9], qdd[9], F[8], gen[9];  // inverse dynamics at node 0 (mpc.cpp:320-330)
    const double dt0 = P.dt[0];
    for (int k = 0; k < 9; ++k) {
      qv[k] = fz[k * 32 + lane];
      qd[k] = fz[(NQ + k) * 32 + lane];
      qdd[k] = (fz[(NV + NQ + k) * 32 + lane] - qd[k]) / dt0;
    }
    for (int k = 0; k < 8; ++k) F[k] = fz[(18 + k) * 32 + lane];
    inverse_dynamics(P, qv, qd, qdd, F, gen);
    for (int bb = 0; bb < 3; ++bb) out.base_residual[bb] = (float)gen[bb];
    for (int mm = 0; mm < 6; ++mm) {
      out.tau_ff[mm] = (float)gen[3 + mm];
      out.q_set[mm] = (float)qv[3 + mm];
      out.qd_set[mm] = (float)qd[3 + mm];
    }
    for (int k = 0; k < 8; ++k) out.f0[k] = (float)F[k];
  }
  // the records through shared memory (the transpose buffers; every z* row is out): one
  // contiguous 140-byte record per agent
  constexpr int RW = (int)(sizeof(rmpc_solution) / 4);  // 35 words, odd stride: no bank conflicts
  float* rs = fin + 2 * 2 * NV * 32 + 4 * 5 * 32;
  const float* o = reinterpret_cast<const float*>(&out);
#pragma unroll
  for (int k = 0; k < RW; ++k) rs[lane * RW + k] = o[k];
  __syncwarp();
  const unsigned wm = __ballot_sync(FULL, write);
#pragma unroll 1
  for (int l = 0; l < 32; ++l) {
    const int al = __shfl_sync(FULL, agent, l);
    if ((wm >> l) & 1u) {
      float* dst = reinterpret_cast<float*>(P.out + al);
      dst[lane] = rs[l * RW + lane];
      if (lane < RW - 32) dst[32 + lane] = rs[l * RW + 32 + lane];
    }
  }
}


// One long squad on the CTA's four warps: `cnt` agents order[first ...] of schedule `g`.
__device__ void sq4_solve(const KParams& P, float* reg, uint32_t tm, int g, int first, int cnt, const double* con_pz) {
  const int NT = P.NT, lane = threadIdx.x & 31, role = threadIdx.x >> 5;
  const SqLayout L = sq_layout(NT);
  const Sq4Layout L4 = sq4_layout(NT);
  Sq q;
  q.coef = reg + L.coef;
  q.mf = reg + L.mf;
  q.lo = reg + L.lo;
  q.hi = reg + L.hi;
  q.d = reg + L.d;
  q.e = reg + L.e;
  q.qh = reg + L.qh;
  q.flags = reinterpret_cast<const uint32_t*>(reg + L.flags);
  q.priv = reg + L4.priv + role * L4.priv_warp;
  q.cross = reg + L4.cross;
  q.tm = tm;
  q.lane = lane;
  q.NT = NT;
  q.m = mid_node(NT);
  q.nb = 5;
  q.bar = S4B_MID;
  int lo, own;
  sq4_nodes(NT, role, lo, own);
  long long t0 = P.profile ? clock64() : 0;
  const bool in = lane < cnt;
  const int agent = P.order[first + (in ? lane : 0)];
  const rmpc_state st = P.states[agent];
  const rmpc_command cmd = P.cmds[agent];
  const rmpc_gait gait = P.gaits[agent];
  sq_prof(P, in && role == 0, 0, t0);
  const bool same = sq4_setup(P, q, role, lo, own, st, cmd, gait, con_pz);
  q.cx(S4X_SAME + role) = same ? 1.f : 0.f;
  s4_all();
  const bool mine = in && q.cx(S4X_SAME) != 0.f && q.cx(S4X_SAME + 1) != 0.f && q.cx(S4X_SAME + 2) != 0.f &&
                    q.cx(S4X_SAME + 3) != 0.f;
  if (role == 0 && in && !mine) P.list_out[atomicAdd(P.n_list, 1)] = agent;  // not this schedule: rti_kernel's list
  sq_prof(P, mine && role == 0, 2, t0);
  const int fstat = reinterpret_cast<const int32_t*>(q.flags)[NT];
  int status = RMPC_STATUS_OK, fail_iter = -1;
  if (fstat != 1) {
    status = RMPC_STATUS_SINGULAR;
  } else {
    sq_prof(P, mine && role == 0, 4, t0);
    const AdmmConst K{(float)P.rho, (float)P.sigma, (float)P.alpha, 1.f - (float)P.alpha, (float)(1.0 / P.rho)};
    const int fb = sq4_admm(P, q, K, role);
    q.cx(S4X_BAD + role) = __int_as_float(fb);
  }
  s4_all();  // every warp done: the matrices are dead, their space is the finish scratch
  if (fstat == 1) {
    sq_prof(P, mine && role == 0, 5, t0);
    int f = 0x7fffffff;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const int fw = __float_as_int(q.cx(S4X_BAD + w));
      f = fw < f ? fw : f;
    }
    if (f != 0x7fffffff) {
      status = RMPC_STATUS_DIVERGED;
      fail_iter = f;
    }
  }
  sq4_finish(P, q, role, lo, own, agent, mine, status, fail_iter, st, cmd, reg + L.mf);
  sq_prof(P, mine && role == 0, 6, t0);
}

// CTA = one long squad (four warps, one per TMEM lane quarter, all 512 columns each).  Squad s of
// the launch serves agents [32 k, 32 k + 32) of schedule group g (grp_cta: squad prefix per group).
__global__ void __launch_bounds__(128, 1) rti_squad4_kernel(const KParams P) {
  extern __shared__ __align__(16) float smem[];
  __shared__ uint32_t tmem_base;
  __shared__ int s_g, s_first, s_cnt;
  __shared__ double s_con[4];
  __shared__ uint64_t s_mbar;
  const int w = threadIdx.x >> 5, tid = threadIdx.x;
  const int NT = P.NT;
  if (tid == 0) {
    sq_mbar_init(&s_mbar);
    sq_mbar_fence_init();
    const int ng = min(*P.n_sched, P.store_cap);
    const int sq = (int)blockIdx.x + P.sq_cta_base;
    int g = -1, first = 0, cnt = 0;
    if (ng > 0 && sq < P.grp_cta[ng]) {
      int lo = 0, hi = ng - 1;  // last group whose first squad is <= sq
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (P.grp_cta[mid] <= sq) lo = mid; else hi = mid - 1;
      }
      g = lo;
      const int k = sq - P.grp_cta[g];
      first = P.grp_first[g] + 32 * k;
      cnt = min(32, P.grp_count[g] - 32 * k);
    }
    s_g = g;
    s_first = first;
    s_cnt = cnt;
  }
  __syncthreads();
  if (s_cnt <= 0) return;  // idle CTA
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tmem_base))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  const SqLayout L = sq_layout(NT);
  if (tid == 0)  // the schedule image (sq_pack_kernel) into shared memory
    sq_bulk_image(smem, P.sqpack + (size_t)s_g * L.priv, (uint32_t)L.priv * 4u, &s_mbar);
  if (tid < 4) s_con[tid] = P.con_pz[tid];  // contact heights of the nominal pose (sched_key_kernel)
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = tmem_base;
  sq_mbar_wait(&s_mbar, 0);
  sq4_solve(P, smem, tb + ((uint32_t)(32 * w) << 16), s_g, s_first, s_cnt, s_con);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb) : "memory");
}

}  // namespace rmpc_dev
