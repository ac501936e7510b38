// rmpc_ruiz.cuh — stage Ruiz: AdmmSolver::equilibrate (qp.cpp:64-95, ruiz.cpp:7-36) and the scaling.
// Part of the fused solve kernel: included once, in order, by rmpc_kernel.cu.
#pragma once

#include "rmpc_device.cuh"
#include "rmpc_kin.cuh"

namespace rmpc_dev {

#ifndef FULL
#define FULL 0xffffffffu
#endif

// ------------------------------------------------------------------------- stage: Ruiz
// AdmmSolver::equilibrate (qp.cpp:64-95) + ruiz_equilibrate (ruiz.cpp:7-36) on
// [[P, A^T], [A, 0]]: each pass takes delta = 1/sqrt(inf-norm) of every row/column of the
// current scaled matrix (1 for empty ones), then d *= delta (rows), e *= delta (columns).
// Row deltas are parked in row.z, column deltas in V_S until the pass is applied.
// The pass loop runs on `nw` warps (wi = this warp's index among them): the agent's warp pair
// (nw = 2, its pair barrier), or in the schedule store build the pair plus helper warps of its
// CTA (nw > 2, CTA barrier RUIZ_BAR over `cnt` threads) -- nodes are independent within a
// pass, so the split changes nothing but the latency.
constexpr int RUIZ_BAR = 15;
__device__ __forceinline__ void ruiz_sync(const Sm& sm, int nw, int cnt) {
  if (nw <= 2) pair_sync(sm);
  else asm volatile("bar.sync %0, %1;" ::"r"(RUIZ_BAR), "r"(cnt) : "memory");
}
__device__ void ruiz(const KParams& P, const Sm& sm, int lane, int wi, int nw, int cnt) {
  const int NT = P.NT;
  Terms T;
  build_terms(lane, T);
  TermBytes B;
  term_bytes<TV_D>(T, B);
  // Double-buffered scales: pass p reads (d, e) from one copy and writes d delta, e delta to
  // the other, so one barrier per pass suffices.  The second d lives in the scratch region,
  // the second e in V_S.
  const int nd = (NT + 1) * NSLOT;
  for (int r = lane + 32 * wi; r < nd; r += 32 * nw) sm.scr[r] = sm.dsc[r];
  ruiz_sync(sm, nw, cnt);
  const float wl = lane < NV ? (float)wcost(P, lane) : 0.f;
  auto inv_sqrt1 = [](float nrm) { return nrm > 0.f ? rsqrtf(nrm) : 1.f; };  // MUFU.RSQ
#pragma unroll 1
  for (int pass = 0; pass < P.ruiz_iters; ++pass) {
    const bool odd = pass & 1;
    Sm src = sm;
    src.dsc = odd ? sm.scr : sm.dsc;
    float* dst = odd ? sm.dsc : sm.scr;
    const int es = odd ? V_S : V_E, ed = odd ? V_E : V_S;
    struct Norms {
      float o0, o1, o2, cv;
    };
    auto norms = [&](int i) {  // reads only the source copies
      Norms n;
      row_view<OpMax>(src, i, lane, es, n.o0, n.o1, n.o2);
      n.cv = col_view<OpMax, TV_D>(src, i, T, B);
      return n;
    };
    auto update = [&](int i, const Norms& n) {  // writes only the destination copies
      const float* d = src.D(i);
      float* dn = dst + (i + 1) * NSLOT;
      dn[lane] = d[lane] * inv_sqrt1(d[lane] * n.o0);
      if (lane < 8) dn[32 + lane] = d[32 + lane] * inv_sqrt1(d[32 + lane] * n.o1);
      if (i == 0 && lane < NINIT) {
        const float* d0 = src.D(-1) + INIT0;
        dst[INIT0 + lane] = d0[lane] * inv_sqrt1(d0[lane] * n.o2);
      }
      if (lane < NV) {
        const float e = sm.V(i, es)[lane];
        const float pd = wl * (float)P.dt[i];
        sm.V(i, ed)[lane] = e * inv_sqrt1(e * fmaxf(fabsf(pd) * e, n.cv));
      }
    };
    // nodes are independent within a pass: two per iteration, all loads ahead of the stores
    int i = wi;
#pragma unroll 1
    for (; i + nw < NT; i += 2 * nw) {
      const Norms a = norms(i), b = norms(i + nw);
      update(i, a);
      update(i + nw, b);
    }
    if (i < NT) update(i, norms(i));
    ruiz_sync(sm, nw, cnt);  // every norm of the next pass uses the scales of this one
  }
  if (P.ruiz_iters & 1) {  // the last pass wrote the second copies
    for (int r = lane + 32 * wi; r < nd; r += 32 * nw) sm.dsc[r] = sm.scr[r];
    for (int i = wi; i < NT; i += nw)
      if (lane < NV) sm.V(i, V_E)[lane] = sm.V(i, V_S)[lane];
    ruiz_sync(sm, nw, cnt);
  }
}

// A^ = D A E, q^ = E q, lo^ = D lo, hi^ = D hi in place (qp.cpp:86-94); P^ = E P E is
// recomputed where needed (phat).
__device__ void apply_scaling(const KParams& P, const Sm& sm, int lane, int warp) {
  const int NT = P.NT;
  for (int i = warp; i < NT; i += 2) {
    float* cf = sm.C(i);
    const float* ei = sm.V(i, V_E);
    const float* en = i + 1 < NT ? sm.V(i + 1, V_E) : ei;
    const float* d = sm.D(i);
    if (lane < 9) {
      const float dr = d[lane];
      cf[C_A1 + lane] *= dr * en[lane];
      cf[C_A2 + lane] *= dr * ei[lane];
      cf[C_A3 + lane] *= dr * en[NQ + lane];
#pragma unroll
      for (int b = 0; b < 3; ++b) cf[C_DYNU + 12 * b + lane] *= d[9 + b] * en[NQ + lane];
    } else if (lane < NV) {
#pragma unroll
      for (int b = 0; b < 3; ++b) cf[C_DYNV + 20 * b + lane - 9] *= d[9 + b] * ei[lane];
    }
    if (lane < 16) {
      const int c = lane >> 2, t = (lane >> 1) & 1, a = lane & 1;
      cf[C_FORCE + lane] *= d[12 + 4 * c + t] * ei[18 + 2 * c + a];
    }
    for (int idx = lane; idx < 36; idx += 32) {
      const int c = idx / 9, k = idx % 9;
      cf[C_JA + idx] *= d[14 + 4 * c] * ei[NQ + k];
      cf[C_JAQ + idx] *= d[14 + 4 * c] * ei[k];
      cf[C_JB + idx] *= d[15 + 4 * c] * ei[NQ + k];
    }
    if (lane < 12) cf[C_BOX + lane] *= d[28 + lane] * ei[lane < 6 ? 3 + lane : NQ + 3 + (lane - 6)];
    if (i == 0 && lane < NINIT) cf[C_INIT + lane] *= sm.D(-1)[INIT0 + lane] * ei[lane];
    if (lane < NV) sm.V(i, V_QH)[lane] *= ei[lane];
  }
  for (int r = lane + 32 * warp; r < (NT + 1) * NSLOT; r += 64) {
    float4 rd = sm.row[r];
    const float dr = sm.dsc[r];
    rd.x *= dr;
    rd.y *= dr;
    sm.row[r] = rd;
  }
  pair_sync(sm);
}

}  // namespace rmpc_dev
