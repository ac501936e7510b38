// rmpc_squad.cuh — lane-per-agent ADMM for schedule-shared cold-start solves ("squads").
// Part of the fused solve kernel: included once, in order, by rmpc_kernel.cu.
//
// With the cold guess (mpc.cpp:266-276) every agent of one stance schedule has the same QP
// matrices, Ruiz scales and factor; only the initial-state and swing-height
// bounds and four components of q^ differ.  A squad is up to 32 agents of one schedule on a warp
// pair: lane l of the "top" warp runs the top half of agent l's two-sided recurrence (nodes
// 0..m, AdmmSolver::run, qp.cpp:156-190, in the reduced form of rmpc_admm.cuh), lane l of the
// "bottom" warp the bottom half (nodes m+1..T-1).  Every matrix entry is warp-uniform: the
// factor's node blocks and the coefficient blocks sit once per squad in shared memory and are
// read as LDS.128 broadcasts, each feeding 4 FFMAs of all 32 agents, instead of one warp pair
// per agent walking 26-lane dependency chains.  Per-agent state lives in the thread's own TMEM
// lane (x, s, the rows' t = rho z - y: 96 columns per node) and in shared memory laid out
// [element][lane] (z of the inequality rows, the agent's bounds / q^ parts).  A CTA holds two
// squads (4 warps, one per TMEM lane quarter, all 512 columns).
#pragma once

#include "rmpc_device.cuh"
#include "rmpc_kin.cuh"

namespace rmpc_dev {

#ifndef FULL
#define FULL 0xffffffffu
#endif

// Layout constants and sq_layout: rmpc_device.cuh.

// ------------------------------------------------------------------------- bulk image load
// A squad's schedule image (sq_pack_kernel, contiguous in global and in shared memory) as bulk
// asynchronous copies (`cp.async.bulk`, the TMA engine) completing on an mbarrier: one thread
// issues them, the squad's threads wait on the barrier's phase 0 -- instead of 64 threads each
// walking ~55 dependent L2 round trips of float4 loads.
__device__ __forceinline__ void sq_mbar_init(uint64_t* mbar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(mbar)) : "memory");
}
__device__ __forceinline__ void sq_mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void sq_bulk_image(float* dst, const float* src, uint32_t bytes, uint64_t* mbar) {
  const uint32_t m = (uint32_t)__cvta_generic_to_shared(mbar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(m), "r"(bytes) : "memory");
  constexpr uint32_t CHUNK = 16384;
  for (uint32_t o = 0; o < bytes; o += CHUNK) {
    const uint32_t n = bytes - o < CHUNK ? bytes - o : CHUNK;
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(dst) + o),
                 "l"(reinterpret_cast<const char*>(src) + o), "r"(n), "r"(m)
                 : "memory");
  }
}
__device__ __forceinline__ void sq_mbar_wait(uint64_t* mbar, uint32_t parity) {
  const uint32_t m = (uint32_t)__cvta_generic_to_shared(mbar);
  asm volatile(
      "{\n .reg .pred p;\n SQ_WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra SQ_WAIT_%=;\n}" ::"r"(m),
      "r"(parity)
      : "memory");
}

// Cross-thread elements of an agent (shared by its two threads), [element][lane].
constexpr int SQX_XM = 0;     // x~_m of the middle node (rows 0..15 from the top, 16..25 from the bottom)
constexpr int SQX_TM = 26;    // t of interval m's rows (bottom writes, both read)
constexpr int SQX_GB = 38;    // g'_{m+1}: gint (9), g (3) (bottom -> top)
constexpr int SQX_BAD = 50;   // first non-finite iteration, top / bottom
constexpr int SQX_SAME = 52;  // schedule check, top / bottom
constexpr int SQX_UA = 56;    // the middle node's rhs with the top's coupling (top -> bottom), 26

// ------------------------------------------------------------------------- TMEM (own lane)
__device__ __forceinline__ void tq_ld1(uint32_t a, float* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=f"(v[0]) : "r"(a));
}
__device__ __forceinline__ void tq_ld2(uint32_t a, float* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=f"(v[0]), "=f"(v[1]) : "r"(a));
}
__device__ __forceinline__ void tq_ld4(uint32_t a, float* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3])
               : "r"(a));
}
__device__ __forceinline__ void tq_ld8(uint32_t a, float* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
               : "r"(a));
}
__device__ __forceinline__ void tq_ld16(uint32_t a, float* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]),
        "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15])
      : "r"(a));
}
__device__ __forceinline__ void tq_st1(uint32_t a, const float* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(a), "f"(v[0]) : "memory");
}
__device__ __forceinline__ void tq_st2(uint32_t a, const float* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(a), "f"(v[0]), "f"(v[1]) : "memory");
}
__device__ __forceinline__ void tq_st4(uint32_t a, const float* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(a), "f"(v[0]), "f"(v[1]),
               "f"(v[2]), "f"(v[3])
               : "memory");
}
__device__ __forceinline__ void tq_st8(uint32_t a, const float* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(a), "f"(v[0]),
               "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
               : "memory");
}
__device__ __forceinline__ void tq_st16(uint32_t a, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(a),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
      "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15])
      : "memory");
}
// N consecutive columns of the thread's lane (any column offset; sizes decomposed in powers of 2)
template <int N>
__device__ __forceinline__ void tq_ld(uint32_t a, float* v) {
  if constexpr (N >= 16) {
    tq_ld16(a, v);
    tq_ld<N - 16>(a + 16, v + 16);
  } else if constexpr (N >= 8) {
    tq_ld8(a, v);
    tq_ld<N - 8>(a + 8, v + 8);
  } else if constexpr (N >= 4) {
    tq_ld4(a, v);
    tq_ld<N - 4>(a + 4, v + 4);
  } else if constexpr (N >= 2) {
    tq_ld2(a, v);
    tq_ld<N - 2>(a + 2, v + 2);
  } else if constexpr (N == 1) {
    tq_ld1(a, v);
  }
}
template <int N>
__device__ __forceinline__ void tq_st(uint32_t a, const float* v) {
  if constexpr (N >= 16) {
    tq_st16(a, v);
    tq_st<N - 16>(a + 16, v + 16);
  } else if constexpr (N >= 8) {
    tq_st8(a, v);
    tq_st<N - 8>(a + 8, v + 8);
  } else if constexpr (N >= 4) {
    tq_st4(a, v);
    tq_st<N - 4>(a + 4, v + 4);
  } else if constexpr (N >= 2) {
    tq_st2(a, v);
    tq_st<N - 2>(a + 2, v + 2);
  } else if constexpr (N == 1) {
    tq_st1(a, v);
  }
}
__device__ __forceinline__ void tq_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tq_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// After tq_wait_ld: the registers of v are defined here (the loads' outputs are not usable
// before the wait; this pins every use after it).
template <int N>
__device__ __forceinline__ void tq_fence(float* v) {
#pragma unroll
  for (int k = 0; k < N; ++k) asm volatile("" : "+f"(v[k]));
}

__device__ __forceinline__ void sq_bar(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }
// Producer / consumer halves of a pair barrier: the bottom warp arrives (no wait) once interval m's
// rows are written, the top warp waits for that before reading them at the middle node.
__device__ __forceinline__ void sq_arrive(int id) { asm volatile("bar.arrive %0, 64;" ::"r"(id) : "memory"); }

// ------------------------------------------------------------------------- squad view
struct Sq {
  const float* coef;
  const float* mf;
  const float* lo;
  const float* hi;
  const float* d;
  const float* e;
  const float* qh;
  const uint32_t* flags;
  float* priv;   // this warp's private elements, [element][32]
  float* cross;  // the agents' cross-thread elements, [element][32]
  uint32_t tm;   // this thread's TMEM lane, column 0
  int lane, NT, m, nb, bar;
  __device__ __forceinline__ const float* C(int i) const { return coef + (i + 1) * C_SIZE; }
  __device__ __forceinline__ const float* MF(int i) const { return mf + i * SQ_MF; }
  __device__ __forceinline__ float LO(int i, int s) const { return lo[(i + 1) * NSLOT + s]; }
  __device__ __forceinline__ float HI(int i, int s) const { return hi[(i + 1) * NSLOT + s]; }
  __device__ __forceinline__ float DS(int i, int s) const { return d[(i + 1) * NSLOT + s]; }
  __device__ __forceinline__ float& pv(int k) const { return priv[k * 32 + lane]; }
  __device__ __forceinline__ float& cx(int k) const { return cross[k * 32 + lane]; }
  __device__ __forceinline__ uint32_t slab(int b) const { return tm + (uint32_t)(SQ_SLAB * b); }
  // private element indices
  __device__ __forceinline__ int ZO(int b, int k) const { return b * SQ_NZ + k; }
  __device__ __forceinline__ int AL(int b, int c) const { return nb * SQ_NZ + 4 * b + c; }
  __device__ __forceinline__ int QA(int b, int q) const { return nb * 24 + 4 * b + q; }
  __device__ __forceinline__ int IL(int l) const { return nb * SQ_PRIV + l; }
  __device__ __forceinline__ int XS(int r) const { return nb * SQ_PRIV + NINIT + r; }
};

// foot-contact Jacobian columns (chain_col): does column k belong to contact c's chain?
__host__ __device__ constexpr bool in_chain(int c, int k) { return k < 3 || (c < 2 ? k >= 6 : (k >= 3 && k < 6)); }
// index of q^ component j among the agent-dependent ones {0, 1, 9, 11} (cold guess, guess_and_target)
__host__ __device__ constexpr int qa_index(int j) { return j == 0 ? 0 : (j == 1 ? 1 : (j == 9 ? 2 : (j == 11 ? 3 : -1))); }

// q^ of node i (own slab b): the schedule's, with the agent's four components
__device__ __forceinline__ void sq_qhat(const Sq& q, int i, int b, float qh[NV]) {
  const float* s = q.qh + i * NV;
#pragma unroll
  for (int j = 0; j < NV; ++j) qh[j] = qa_index(j) >= 0 ? q.pv(q.QA(b, qa_index(j))) : s[j];
}

// acc += (A^T v) restricted to node i's variables: cf = C(i), cp = C(i-1); vi = values of node
// i's interval rows (slots 0..11), vp = node i-1's interval rows, vo = node i's own rows (slots
// 12..39), vin = the initial-state rows (node 0 only).  The column-view terms of build_terms.
__device__ __forceinline__ void sq_colview(const float* cf, const float* cp, const float vi[12], const float vp[12],
                                           const float vo[28], const float* vin, bool node0, float acc[NV]) {
#pragma unroll
  for (int k = 0; k < 9; ++k) {  // q_k
    float a = fmaf(cf[C_A2 + k], vi[k], acc[k]);
    float b = cp[C_A1 + k] * vp[k];
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (in_chain(c, k)) b = fmaf(cf[C_JAQ + 9 * c + k], vo[2 + 4 * c], b);
    if (k >= 3) a = fmaf(cf[C_BOX + k - 3], vo[16 + k - 3], a);
    acc[k] = a + b;
  }
#pragma unroll
  for (int k = 0; k < 9; ++k) {  // qd_k
    float a = fmaf(cp[C_A3 + k], vp[k], acc[9 + k]);
    float b = cp[C_DYNU + k] * vp[9];
    a = fmaf(cp[C_DYNU + 12 + k], vp[10], a);
    b = fmaf(cp[C_DYNU + 24 + k], vp[11], b);
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (in_chain(c, k)) {
        a = fmaf(cf[C_JA + 9 * c + k], vo[2 + 4 * c], a);
        b = fmaf(cf[C_JB + 9 * c + k], vo[3 + 4 * c], b);
      }
#pragma unroll
    for (int bb = 0; bb < 3; ++bb) a = fmaf(cf[C_DYNV + 20 * bb + k], vi[9 + bb], a);
    if (k >= 3) b = fmaf(cf[C_BOX + 6 + k - 3], vo[22 + k - 3], b);
    acc[9 + k] = a + b;
  }
#pragma unroll
  for (int f = 0; f < 8; ++f) {  // F_f, contact c = f / 2
    const int c = f >> 1, a1 = f & 1;
    float a = fmaf(cf[C_DYNV + 9 + f], vi[9], acc[18 + f]);
    a = fmaf(cf[C_DYNV + 20 + 9 + f], vi[10], a);
    a = fmaf(cf[C_DYNV + 40 + 9 + f], vi[11], a);
    a = fmaf(cf[C_FORCE + 4 * c + a1], vo[4 * c], a);
    acc[18 + f] = fmaf(cf[C_FORCE + 4 * c + 2 + a1], vo[4 * c + 1], a);
  }
  if (node0) {
#pragma unroll
    for (int l = 0; l < NINIT; ++l) acc[l] = fmaf(cf[C_INIT + l], vin[l], acc[l]);
  }
}

// Rows [0, 4 nch) of the packed node matrix times u, 4 rows per step (8 independent FMA chains),
// each step's 4 results stored to TMEM columns dst + 4 c.  A runtime loop: the matvec is the
// bulk of every node step, and a fully unrolled copy per call site overflows the instruction
// cache at one warp per scheduler.
__device__ __forceinline__ void sq_matvec_tm(const float* M, const float u[NV], uint32_t dst, int nch) {
#pragma unroll 2
  for (int c = 0; c < nch; ++c) {
    const float4* R = reinterpret_cast<const float4*>(M + 4 * SQ_MROW * c);
    float a[4][2];
#pragma unroll
    for (int r = 0; r < 4; ++r) a[r][0] = a[r][1] = 0.f;
#pragma unroll
    for (int qq = 0; qq < SQ_MROW / 4; ++qq) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const float4 w = R[(SQ_MROW / 4) * r + qq];
        a[r][0] = fmaf(w.x, u[4 * qq], a[r][0]);
        a[r][1] = fmaf(w.y, u[4 * qq + 1], a[r][1]);
        if (4 * qq + 2 < NV) {
          a[r][0] = fmaf(w.z, u[4 * qq + 2], a[r][0]);
          a[r][1] = fmaf(w.w, u[4 * qq + 3], a[r][1]);
        }
      }
    }
    float o[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) o[r] = a[r][0] + a[r][1];
    tq_st4(dst + 4 * c, o);
  }
}

// The middle node's x~_m = S_m^-1 u split over the pair: rows [4 c0, 4 (c0 + nch)) of the node
// matrix times u, stored to the pair's cross elements XM (rows < 26); returns whether any is
// non-finite.  Same chunk loop as sq_matvec_tm.
__device__ __forceinline__ bool sq_matvec_mid(const Sq& q, const float* M, const float u[NV], int c0, int nch) {
  bool bad = false;
#pragma unroll 1
  for (int c = c0; c < c0 + nch; ++c) {
    const float4* R = reinterpret_cast<const float4*>(M + 4 * SQ_MROW * c);
    float a[4][2];
#pragma unroll
    for (int r = 0; r < 4; ++r) a[r][0] = a[r][1] = 0.f;
#pragma unroll
    for (int qq = 0; qq < SQ_MROW / 4; ++qq) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const float4 w = R[(SQ_MROW / 4) * r + qq];
        a[r][0] = fmaf(w.x, u[4 * qq], a[r][0]);
        a[r][1] = fmaf(w.y, u[4 * qq + 1], a[r][1]);
        if (4 * qq + 2 < NV) {
          a[r][0] = fmaf(w.z, u[4 * qq + 2], a[r][0]);
          a[r][1] = fmaf(w.w, u[4 * qq + 3], a[r][1]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const float o = a[r][0] + a[r][1];
      if (4 * c + r < NV) {
        q.cx(SQX_XM + 4 * c + r) = o;
        bad = bad || !isfinite(o);
      }
    }
  }
  return bad;
}

// acc[0..25] += sum_r xs[r] M[row(r)][:], row(r) = r < NQR ? r : 26 + r - NQR, for r < NR; the
// coefficients come from the lane's private scratch (shared memory), the rows as broadcasts.
__device__ __forceinline__ void sq_axpy_tm(const Sq& q, const float* M, int nqr, int nr, float acc[NV]) {
#pragma unroll 3
  for (int r = 0; r < nr; ++r) {
    const float c = q.pv(q.XS(r));
    const float4* R = reinterpret_cast<const float4*>(M + SQ_MROW * (r < nqr ? r : 26 + r - nqr));
#pragma unroll
    for (int qq = 0; qq < SQ_MROW / 4; ++qq) {
      const float4 w = R[qq];
      acc[4 * qq] = fmaf(c, w.x, acc[4 * qq]);
      acc[4 * qq + 1] = fmaf(c, w.y, acc[4 * qq + 1]);
      if (4 * qq + 2 < NV) {
        acc[4 * qq + 2] = fmaf(c, w.z, acc[4 * qq + 2]);
        acc[4 * qq + 3] = fmaf(c, w.w, acc[4 * qq + 3]);
      }
    }
  }
}

// One constraint-row update (row_update, qp.cpp:163-170) on (t = rho z - y, z).
__device__ __forceinline__ void sq_rupd(float& t, float& z, float lo, float hi, float zt, const AdmmConst& K) {
  const float y = fmaf(K.rho, z, -t);
  const float w = K.alpha * zt + K.oma * z;
  const float zn = fminf(fmaxf(w + K.rho_inv * y, lo), hi);
  const float yn = y + K.rho * (w - zn);
  z = zn;
  t = fmaf(K.rho, zn, -yn);
}
// An equality row (lo == hi): z is 0 before the first update and lo ever after.
__device__ __forceinline__ void sq_rupd_eq(float& t, float lo, bool first, float zt, const AdmmConst& K) {
  float z = first ? 0.f : lo;
  sq_rupd(t, z, lo, lo, zt, K);
}

// The rows of node i acting on node-i variables only (node_rows): contact rows t0..t3, joint
// boxes, the initial-state rows at node 0; then the x relaxation.  xs = x~_i.  Own slab b.
__device__ __forceinline__ bool sq_finish_node(const Sq& q, int i, int b, const float xs[NV], bool first,
                                               const AdmmConst& K) {
  float to[28], x[NV], tin[NINIT];
  tq_ld<28>(q.slab(b) + SQ_TO, to);
  tq_ld<NV>(q.slab(b) + SQ_X, x);
  const bool node0 = i == 0;
  if (node0) tq_ld<NINIT>(q.tm + SQ_TINIT, tin);
  float z[SQ_NZ];
#pragma unroll
  for (int k = 0; k < SQ_NZ; ++k) z[k] = q.pv(q.ZO(b, k));
  const float* cf = q.C(i);
  const uint32_t bits = q.flags[i];
  tq_wait_ld();
  tq_fence<28>(to);
  tq_fence<NV>(x);
  if (node0) tq_fence<NINIT>(tin);
  bool fin = true;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    float pa = 0.f, pb = 0.f;
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      const int col = s < 3 ? s : (c < 2 ? 6 : 3) + s - 3;
      pa = fmaf(cf[C_JAQ + 9 * c + col], xs[col], pa);
      pa = fmaf(cf[C_JA + 9 * c + col], xs[NQ + col], pa);
      pb = fmaf(cf[C_JB + 9 * c + col], xs[NQ + col], pb);
    }
    const float f0 = xs[18 + 2 * c], f1 = xs[19 + 2 * c];
    const float z0 = cf[C_FORCE + 4 * c] * f0 + cf[C_FORCE + 4 * c + 1] * f1;
    const float z1 = cf[C_FORCE + 4 * c + 2] * f0 + cf[C_FORCE + 4 * c + 3] * f1;
    const int s0 = 12 + 4 * c;
    sq_rupd(to[4 * c], z[2 * c], q.LO(i, s0), q.HI(i, s0), z0, K);
    sq_rupd(to[4 * c + 1], z[2 * c + 1], q.LO(i, s0 + 1), q.HI(i, s0 + 1), z1, K);
    const float lo2 = ((bits >> c) & 1u) || i == 0 ? q.LO(i, s0 + 2) : q.pv(q.AL(b, c));
    sq_rupd_eq(to[4 * c + 2], lo2, first, pa, K);
    sq_rupd_eq(to[4 * c + 3], q.LO(i, s0 + 3), first, pb, K);
    fin = fin && isfinite(z0) && isfinite(z1) && isfinite(pa) && isfinite(pb);
  }
#pragma unroll
  for (int mb = 0; mb < 12; ++mb) {
    const float zb = cf[C_BOX + mb] * xs[mb < 6 ? 3 + mb : 6 + mb];
    sq_rupd(to[16 + mb], z[8 + mb], q.LO(i, 28 + mb), q.HI(i, 28 + mb), zb, K);
    fin = fin && isfinite(zb);
  }
  if (node0) {
#pragma unroll
    for (int l = 0; l < NINIT; ++l) {
      const float zt = cf[C_INIT + l] * xs[l];
      sq_rupd_eq(tin[l], q.pv(q.IL(l)), first, zt, K);
      fin = fin && isfinite(zt);
    }
  }
#pragma unroll
  for (int j = 0; j < NV; ++j) x[j] = K.alpha * xs[j] + K.oma * x[j];
  tq_st<28>(q.slab(b) + SQ_TO, to);
  tq_st<NV>(q.slab(b) + SQ_X, x);
  if (node0) tq_st<NINIT>(q.tm + SQ_TINIT, tin);
#pragma unroll
  for (int k = 0; k < SQ_NZ; ++k) q.pv(q.ZO(b, k)) = z[k];
  return !fin;
}

// rhs r_i = sigma x - q^ + A^T t of node i (own slab b), given the interval-row t of node i
// (ti) and of node i-1 (tp); loads x, the own rows' t and (node 0) the initial rows' t.
// ti / tp may still be in flight from tcgen05.ld: they are pinned after the wait here.
__device__ __forceinline__ void sq_rhs(const KParams& P, const Sq& q, int i, int b, float ti[12], float tp[12],
                                       float r[NV]) {
  float x[NV], to[28], tin[NINIT];
  tq_ld<NV>(q.slab(b) + SQ_X, x);
  tq_ld<28>(q.slab(b) + SQ_TO, to);
  const bool node0 = i == 0;
  if (node0) tq_ld<NINIT>(q.tm + SQ_TINIT, tin);
  float qh[NV];
  sq_qhat(q, i, b, qh);
  tq_wait_ld();
  tq_fence<NV>(x);
  tq_fence<28>(to);
  tq_fence<12>(ti);
  tq_fence<12>(tp);
  if (node0) tq_fence<NINIT>(tin);
  const float sigma = (float)P.sigma;
#pragma unroll
  for (int j = 0; j < NV; ++j) r[j] = sigma * x[j] - qh[j];
  sq_colview(q.C(i), q.C(i - 1), ti, tp, to, tin, node0, r);
}

// ------------------------------------------------------------------------- the two halves
// - rho U_{i-1} g_{i-1} (top_corr): cp = C(i-1)
__device__ __forceinline__ void sq_top_corr(const float* cp, const float gint[9], const float g[3], float rho,
                                            float u[NV]) {
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    u[k] -= rho * (cp[C_A1 + k] * gint[k]);
    u[9 + k] -= rho * (cp[C_A3 + k] * gint[k] +
                       (cp[C_DYNU + k] * g[0] + cp[C_DYNU + 12 + k] * g[1] + cp[C_DYNU + 24 + k] * g[2]));
  }
}
// - rho V_i g'_{i+1} (bot_corr): cf = C(i)
__device__ __forceinline__ void sq_bot_corr(const float* cf, const float gint[9], const float g[3], float rho,
                                            float u[NV]) {
#pragma unroll
  for (int k = 0; k < 9; ++k) u[k] -= rho * (cf[C_A2 + k] * gint[k]);
#pragma unroll
  for (int jv = 0; jv < 17; ++jv)
    u[9 + jv] -= rho * (cf[C_DYNV + jv] * g[0] + cf[C_DYNV + 20 + jv] * g[1] + cf[C_DYNV + 40 + jv] * g[2]);
}

// AdmmSolver::run (qp.cpp:156-190) for the agent of this lane, top half (nodes 0..m): forward
// sweep with the middle node as its last step, backward sweep with node 0's own rows as its
// last step -- admm() (rmpc_admm.cuh) with the agent in the lane and the node-vector index in
// registers, one copy of each step in the code.  Returns the first iteration with a non-finite
// iterate (or INT_MAX).
__device__ __forceinline__ int sq_admm_top(const KParams& P, const Sq& q, const AdmmConst& K) {
  const int NT = q.NT, m = q.m;
  const float rho = K.rho;
  int first_bad = 0x7fffffff;
#pragma unroll 1
  for (int it = 0; it < P.n_qp; ++it) {
    const bool first = it == 0;
    bool bad = false;
    float gint[9], g[3], tp[12], xn[NV];
#pragma unroll
    for (int k = 0; k < 9; ++k) gint[k] = 0.f;
#pragma unroll
    for (int k = 0; k < 12; ++k) tp[k] = 0.f;
    g[0] = g[1] = g[2] = 0.f;
    // ------------------------------------------------ forward i = 0..m-1, then the middle i = m
#pragma unroll 1
    for (int i = 0; i <= m; ++i) {
      const bool mid = i == m;
      float ti[12];
      if (mid) {
        tq_wait_st();
        sq_bar(q.bar + 2);  // interval m's rows are written (the bottom's first backward step)
#pragma unroll
        for (int k = 0; k < 12; ++k) ti[k] = q.cx(SQX_TM + k);
      } else {
        tq_ld<12>(q.slab(i) + SQ_TI, ti);  // (waited for inside sq_rhs)
      }
      float u[NV];
      sq_rhs(P, q, i, i, ti, tp, u);
      sq_top_corr(q.C(i - 1), gint, g, rho, u);
      if (mid) {  // the middle node, split over the pair: both halves finish u_m and each
                  // multiplies half of S_m^-1's rows
#pragma unroll
        for (int j = 0; j < NV; ++j) q.cx(SQX_UA + j) = u[j];
        sq_bar(q.bar);  // the bottom half's forward sweep is done (g'_{m+1})
        float gb[12];
#pragma unroll
        for (int k = 0; k < 12; ++k) gb[k] = q.cx(SQX_GB + k);
        sq_bot_corr(q.C(m), gb, gb + 9, rho, u);
        bad = sq_matvec_mid(q, q.MF(m), u, 0, 4) || bad;  // rows 0..15
        break;
      }
      sq_matvec_tm(q.MF(i), u, q.slab(i) + SQ_S, 8);
      tq_wait_st();
      {
        float s9[9], s3[3];
        tq_ld<9>(q.slab(i) + SQ_S, s9);
        tq_ld<3>(q.slab(i) + SQ_S + 26, s3);
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
    }
    sq_bar(q.bar);  // x~_m published (both halves)
#pragma unroll
    for (int j = 0; j < NV; ++j) xn[j] = q.cx(SQX_XM + j);
    // ------------------------------------------------ backward i = m-1..0, then node 0's rows
#pragma unroll 1
    for (int i = m - 1; i >= -1; --i) {
      float xc[NV];
      if (i >= 0) {
        const float* cf = q.C(i);
        float s[SROWS], ti[12];
        tq_ld<SROWS>(q.slab(i) + SQ_S, s);
        tq_ld<12>(q.slab(i) + SQ_TI, ti);
        // xi_k = a2_k (a1_k x[q_k] + a3_k x[qd_k]) = a2_k dl_k; xi_{9+b} = u_b . x_{i+1}[qd]
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
        // x~_i = s_i - rho (S_i^-1[:, 0..8] xi_int + W_i xi_dyn): by symmetry rows 0..8 and 26..28
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
        // z~: integration row k = a2 x~_i[q_k] + dl_k; dynamics row b = g_b - rho (W_b^T xi_int + G_b xi_dyn) + xi_b
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
        tq_st<NV>(q.slab(i) + SQ_S, xc);
        tq_st<12>(q.slab(i) + SQ_TI, ti);
      }
      bad = sq_finish_node(q, i + 1, i + 1, xn, first, K) || bad;  // node i+1's own rows, x
      tq_wait_st();
      if (i >= 0) {
#pragma unroll
        for (int j = 0; j < NV; ++j) xn[j] = xc[j];
      }
    }
    if (bad && first_bad > it) first_bad = it;
  }
  return first_bad;
}

// Bottom half (nodes m+1..T-1), mirrored recurrences (T_i = D_i - rho^2 V_i G'_i V_i^T).
__device__ __forceinline__ int sq_admm_bot(const KParams& P, const Sq& q, const AdmmConst& K) {
  const int NT = q.NT, m = q.m;
  const float rho = K.rho;
  int first_bad = 0x7fffffff;
  if (P.n_qp > 0) sq_arrive(q.bar + 2);  // interval m's rows (zero) are ready for the first middle step
#pragma unroll 1
  for (int it = 0; it < P.n_qp; ++it) {
    const bool first = it == 0;
    bool bad = false;
    float gint[9], g[3], ti[12];
#pragma unroll
    for (int k = 0; k < 9; ++k) gint[k] = 0.f;
    g[0] = g[1] = g[2] = 0.f;
    // ---------------------------------------------------------------- forward i = T-1..m+1
    tq_ld<12>(q.slab(NT - 1 - (m + 1)) + SQ_TI, ti);
    tq_wait_ld();
    tq_fence<12>(ti);
#pragma unroll 1
    for (int i = NT - 1; i > m; --i) {
      const int b = i - m - 1;
      float tp[12];
      if (i - 1 > m) {
        tq_ld<12>(q.slab(b - 1) + SQ_TI, tp);  // (waited for inside sq_rhs)
      } else {
#pragma unroll
        for (int k = 0; k < 12; ++k) tp[k] = q.cx(SQX_TM + k);
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
      const float* cp = q.C(i - 1);  // g'_int_k = a1_k s[q_k] + a3_k s[qd_k]
#pragma unroll
      for (int k = 0; k < 9; ++k) gint[k] = cp[C_A1 + k] * s18[k] + cp[C_A3 + k] * s18[NQ + k];
      g[0] = s3[0];
      g[1] = s3[1];
      g[2] = s3[2];
#pragma unroll
      for (int k = 0; k < 12; ++k) ti[k] = tp[k];
    }
#pragma unroll
    for (int k = 0; k < 9; ++k) q.cx(SQX_GB + k) = gint[k];
    q.cx(SQX_GB + 9) = g[0];
    q.cx(SQX_GB + 10) = g[1];
    q.cx(SQX_GB + 11) = g[2];
    sq_bar(q.bar);  // (the top half's u_m is published)
    {  // the middle node's rows 16..25: u_m = the top's part - rho V_m g'_{m+1} (same operations as the top)
      float u[NV];
#pragma unroll
      for (int j = 0; j < NV; ++j) u[j] = q.cx(SQX_UA + j);
      sq_bot_corr(q.C(m), gint, g, rho, u);
      bad = sq_matvec_mid(q, q.MF(m), u, 4, 3) || bad;
    }
    sq_bar(q.bar);  // the middle node's x~_m is published
    // ---------------------------------------------------------------- backward i = m+1..T-1
    float xp[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) xp[j] = q.cx(SQX_XM + j);
#pragma unroll 1
    for (int i = m + 1; i < NT; ++i) {
      const int b = i - m - 1;
      const float* cp = q.C(i - 1);  // interval i-1 couples nodes i-1 and i
      float s[SROWS], tr[12];
      tq_ld<SROWS>(q.slab(b) + SQ_S, s);
      if (i - 1 > m) {
        tq_ld<12>(q.slab(b - 1) + SQ_TI, tr);
      } else {
#pragma unroll
        for (int k = 0; k < 12; ++k) tr[k] = q.cx(SQX_TM + k);
      }
      // xi'_k = a2_k x_{i-1}[q_k]; xi'_b = v_b . x_{i-1}[9..25]
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
      if (i - 1 > m) tq_fence<12>(tr);
      float xt[NV];
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        xt[j] = s[j] - rho * acc[j];
        bad = bad || !isfinite(xt[j]);
      }
      // z~: integration row k = xi'_k + a1 x_i[q_k] + a3 x_i[qd_k]; dynamics row b = xi'_b + g'_b - rho acc_b
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
      if (i - 1 > m) {
        tq_st<12>(q.slab(b - 1) + SQ_TI, tr);
      } else {
#pragma unroll
        for (int k = 0; k < 12; ++k) q.cx(SQX_TM + k) = tr[k];
        if (it + 1 < P.n_qp) sq_arrive(q.bar + 2);  // for the top half's next middle step
      }
      bad = sq_finish_node(q, i, b, xt, first, K) || bad;
      tq_wait_st();
#pragma unroll
      for (int j = 0; j < NV; ++j) xp[j] = xt[j];
    }
    if (bad && first_bad > it) first_bad = it;
  }
  return first_bad;
}

// ------------------------------------------------------------------------- setup / finish
// The agent's own data (solve_agent_shared): zero state; q^ components 0, 1, 9, 11 (the only
// ones the cold guess makes agent-dependent, guess_and_target); the swing-height bounds of its
// swing contacts (mpc.cpp:210-216); the initial-state bounds (top, mpc.cpp:126-136), all in
// FP64 by the operations of setup_nodes / setup_dynamics / apply_scaling.  Returns whether the
// agent's stance flags equal the squad's (a 64-bit schedule-hash collision otherwise).
__device__ __forceinline__ bool sq_setup(const KParams& P, const Sq& q, bool top, int own, const rmpc_state& st,
                         const rmpc_command& cmd, const rmpc_gait& gait, const double* con_pz) {
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
  if (top) tq_st<NINIT>(q.tm + SQ_TINIT, zero);
  for (int k = 0; k < q.nb * SQ_NZ; ++k) q.pv(k) = 0.f;
  if (!top)  // interval m's rows start at t = 0 (read by both halves before the first update)
    for (int k = 0; k < 12; ++k) q.cx(SQX_TM + k) = 0.f;
  bool same = true;
#pragma unroll 1
  for (int b = 0; b < own; ++b) {
    const int i = top ? b : q.m + 1 + b;
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
  if (top) {
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

// z* out: this warp's nodes [i0, i0 + own) of an agent are one contiguous run of own x 26 floats.
// The finish leaves each node's z* row in the node's dead x columns of the thread's TMEM lane; six
// agents at a time go through the warp's transpose buffer `xp` (6 x 130 <= 32 x 27 floats) and out
// as float2 words on consecutive lanes -- whole 128-byte lines instead of one 104-byte row per
// store (mapped host memory over PCIe: 47 vs 38 GB/s, tools/micro/mapped_write.cu).
__device__ __forceinline__ void sq_zstar_out(const KParams& P, const Sq& q, float* xp, int i0, int own, int agent,
                                             bool write) {
  constexpr int RUN = 5 * NV;  // xp floats per agent (own <= 5)
  const int lane = q.lane, nw = own * NV / 2;
  tq_wait_st();
  const unsigned wm = __ballot_sync(FULL, write);
#pragma unroll 1
  for (int l0 = 0; l0 < 32; l0 += 6) {
    if (((wm >> l0) & 0x3Fu) == 0u) continue;
#pragma unroll 1
    for (int b = 0; b < own; ++b) {
      float v[NV];
      tq_ld<NV>(q.slab(b) + SQ_X, v);
      tq_wait_ld();
      tq_fence<NV>(v);
      if (lane >= l0 && lane < l0 + 6) {
#pragma unroll
        for (int j = 0; j < NV; ++j) xp[(lane - l0) * RUN + b * NV + j] = v[j];
      }
    }
    __syncwarp();
#pragma unroll 1
    for (int k = 0; k < 6 && l0 + k < 32; ++k) {
      const int al = __shfl_sync(FULL, agent, l0 + k);
      if ((wm >> (l0 + k)) & 1u) {
        float2* dst = reinterpret_cast<float2*>(P.z_out + ((size_t)al * q.NT + i0) * NV);
        const float2* src = reinterpret_cast<const float2*>(xp + k * RUN);
        for (int w = lane; w < nw; w += 32) dst[w] = src[w];
      }
    }
    __syncwarp();
  }
}

// Residuals and objective on the unscaled problem (qp.cpp:192-200), z* = guess + dz and the
// inverse dynamics at node 0 (mpc.cpp:305-330), the active set (optional) and the record
// (finish_agent), lane-parallel.  fin: the squad's finish scratch (the matrices are dead).
// Every lane runs it (the pair barriers); `write` lanes store.
__device__ __forceinline__ void sq_finish(const KParams& P, const Sq& q, bool top, int own, int agent, bool write, int status,
                          int fail_iter, const rmpc_state& st, const rmpc_command& cmd, float* fin) {
  const int NT = q.NT, m = q.m, lane = q.lane;
  float* fx = fin;                                      // x_m, [26][32]
  double* fz = reinterpret_cast<double*>(fin + 26 * 32);  // z* rows of nodes 0, 1 (FP64), [2][26][32]
  float* fc = fin + 26 * 32 + 2 * 2 * NV * 32;          // bottom's prim, dual, dinf, obj (FP64)
  float* xp = fin + SQ_FIN_XP + (top ? 0 : 32 * 27);     // this warp's transpose buffer [lane][27]
  const bool ok = status == RMPC_STATUS_OK;
  const float rho = (float)P.rho;
  const bool eqz = P.n_qp > 0;  // equality rows: z = lo after the first update
  if (top) {
    float x[NV];
    tq_ld<NV>(q.slab(m) + SQ_X, x);
    tq_wait_ld();
    tq_fence<NV>(x);
#pragma unroll
    for (int j = 0; j < NV; ++j) fx[j * 32 + lane] = x[j];
  }
  sq_bar(q.bar);
  float prim = 0.f, dual = 0.f, dinf = 0.f;
  double obj = 0.0;
  float xprev[NV], tp[12];
  if (top) {
#pragma unroll
    for (int j = 0; j < NV; ++j) xprev[j] = 0.f;
#pragma unroll
    for (int k = 0; k < 12; ++k) tp[k] = 0.f;
  } else {
#pragma unroll
    for (int j = 0; j < NV; ++j) xprev[j] = fx[j * 32 + lane];
#pragma unroll
    for (int k = 0; k < 12; ++k) tp[k] = q.cx(SQX_TM + k);
  }
#pragma unroll 1
  for (int b = 0; b < own; ++b) {
    const int i = top ? b : m + 1 + b;
    const bool node0 = i == 0;
    float x[NV], to[28], ti[12], tin[NINIT];
    tq_ld<NV>(q.slab(b) + SQ_X, x);
    tq_ld<28>(q.slab(b) + SQ_TO, to);
    if (top && i == m) {
#pragma unroll
      for (int k = 0; k < 12; ++k) ti[k] = q.cx(SQX_TM + k);
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
  if (P.z_out) sq_zstar_out(P, q, xp, top ? 0 : m + 1, own, agent, write);
  if (!top) {
    fc[lane] = prim;
    fc[32 + lane] = dual;
    fc[64 + lane] = dinf;
    reinterpret_cast<double*>(fc + 96)[lane] = obj;
  }
  sq_bar(q.bar);
  if (!top) return;
  prim = fmaxf(prim, fc[lane]);
  dual = fmaxf(dual, fc[32 + lane]);
  dinf = fmaxf(dinf, fc[64 + lane]);
  obj += reinterpret_cast<const double*>(fc + 96)[lane];
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
  // the records through shared memory (both transpose buffers; the bottom's z* rows are out):
  // one contiguous 140-byte record per agent
  constexpr int RW = (int)(sizeof(rmpc_solution) / 4);  // 35 words, odd stride: no bank conflicts
  float* rs = fin + SQ_FIN_XP;
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

__device__ __forceinline__ void sq_prof(const KParams& P, bool on, int stage, long long& t0) {
  if (P.profile) {
    const long long t1 = clock64();
    if (on) {
      const unsigned long long d = (unsigned long long)(t1 - t0);
      atomicAdd(P.prof + stage, d);
      atomicAdd(P.prof + RMPC_NUM_STAGES + stage, d * d);
    }
    t0 = t1;
  }
}

// One squad on warps (2 sq, 2 sq + 1): `cnt` agents order[first ...] of schedule `g`.
__device__ void sq_solve(const KParams& P, float* reg, uint32_t tm, int sqi, int g, int first, int cnt,
                         const double* con_pz) {
  const int NT = P.NT, lane = threadIdx.x & 31;
  const bool top = ((threadIdx.x >> 5) & 1) == 0;
  const SqLayout L = sq_layout(NT);
  Sq q;
  q.coef = reg + L.coef;
  q.mf = reg + L.mf;
  q.lo = reg + L.lo;
  q.hi = reg + L.hi;
  q.d = reg + L.d;
  q.e = reg + L.e;
  q.qh = reg + L.qh;
  q.flags = reinterpret_cast<const uint32_t*>(reg + L.flags);
  q.priv = reg + L.priv + (top ? 0 : L.priv_warp);
  q.cross = reg + L.cross;
  q.tm = tm;
  q.lane = lane;
  q.NT = NT;
  q.m = mid_node(NT);
  q.nb = nodes_per_warp(NT);
  q.bar = 1 + sqi;
  const int own = top ? q.m + 1 : NT - 1 - q.m;
  long long t0 = P.profile ? clock64() : 0;
  const bool in = lane < cnt;
  const int agent = P.order[first + (in ? lane : 0)];
  const rmpc_state st = P.states[agent];
  const rmpc_command cmd = P.cmds[agent];
  const rmpc_gait gait = P.gaits[agent];
  sq_prof(P, in && top, 0, t0);
  const bool same = sq_setup(P, q, top, own, st, cmd, gait, con_pz);
  q.cx(SQX_SAME + (top ? 0 : 1)) = same ? 1.f : 0.f;
  sq_bar(q.bar);
  const bool mine = in && q.cx(SQX_SAME) != 0.f && q.cx(SQX_SAME + 1) != 0.f;
  if (top && in && !mine) P.list_out[atomicAdd(P.n_list, 1)] = agent;  // not this schedule: rti_kernel's list
  sq_prof(P, mine && top, 2, t0);  // (Ruiz and the factorization ran once per schedule)
  const int fstat = reinterpret_cast<const int32_t*>(q.flags)[NT];
  int status = RMPC_STATUS_OK, fail_iter = -1;
  if (fstat != 1) {
    status = RMPC_STATUS_SINGULAR;
  } else {
    sq_prof(P, mine && top, 4, t0);
    const AdmmConst K{(float)P.rho, (float)P.sigma, (float)P.alpha, 1.f - (float)P.alpha, (float)(1.0 / P.rho)};
    const int fb = top ? sq_admm_top(P, q, K) : sq_admm_bot(P, q, K);
    q.cx(SQX_BAD + (top ? 0 : 1)) = __int_as_float(fb);
  }
  sq_bar(q.bar);  // both halves done: the matrices are dead, their space is the finish scratch
  if (fstat == 1) sq_prof(P, mine && top, 5, t0);
  if (fstat == 1) {
    const int f0 = __float_as_int(q.cx(SQX_BAD)), f1 = __float_as_int(q.cx(SQX_BAD + 1));
    const int f = f0 < f1 ? f0 : f1;
    if (f != 0x7fffffff) {
      status = RMPC_STATUS_DIVERGED;
      fail_iter = f;
    }
  }
  sq_finish(P, q, top, own, agent, mine, status, fail_iter, st, cmd, reg + L.mf);
  sq_prof(P, mine && top, 6, t0);
}

// CTA = two squads: warps 0/1 squad 0 (top / bottom half), warps 2/3 squad 1.  Squad s of the
// launch serves agents [32 k, 32 k + 32) of schedule group g (grp_cta: squad prefix per group).
// Each squad copies its schedule's store entry into its shared-memory region: coefficients,
// bounds, scales, q^, flags, and the factor's node blocks packed as 29 x 26 row-major matrices.
__global__ void __launch_bounds__(128, 1) rti_squad_kernel(const KParams P) {
  extern __shared__ __align__(16) float smem[];
  __shared__ uint32_t tmem_base;
  __shared__ int s_g[2], s_first[2], s_cnt[2];
  __shared__ double s_con[4];
  __shared__ uint64_t s_mbar[2];
  const int w = threadIdx.x >> 5, tid = threadIdx.x;
  const int NT = P.NT;
  if (tid == 0) {
    sq_mbar_init(&s_mbar[0]);
    sq_mbar_init(&s_mbar[1]);
    sq_mbar_fence_init();
  }
  if (tid < 2) {
    const int ng = min(*P.n_sched, P.store_cap);
    const int cta = (int)blockIdx.x + P.sq_cta_base;
    const int sq = P.pad2_ ? (tid == P.pad2_ - 1 ? cta : 1 << 30) : 2 * cta + tid;
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
    s_g[tid] = g;
    s_first[tid] = first;
    s_cnt[tid] = cnt;
  }
  __syncthreads();
  if (s_cnt[0] <= 0 && s_cnt[1] <= 0) return;  // whole CTA idle
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tmem_base))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  const SqLayout L = sq_layout(NT);
  const StoreLayout SL = store_layout(NT);
  const int sqi = w >> 1;
  float* reg = smem + sqi * L.total;
  if (s_cnt[sqi] > 0 && (tid & 63) == 0)  // this squad's schedule image (sq_pack_kernel) into its region
    sq_bulk_image(reg, P.sqpack + (size_t)s_g[sqi] * L.priv, (uint32_t)L.priv * 4u, &s_mbar[sqi]);
  if (tid < 4) s_con[tid] = P.con_pz[tid];  // contact heights of the nominal pose (sched_key_kernel)
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = tmem_base;
  if (s_cnt[sqi] > 0) sq_mbar_wait(&s_mbar[sqi], 0);
  if (s_cnt[sqi] > 0)
    sq_solve(P, reg, tb + ((uint32_t)(32 * w) << 16), sqi, s_g[sqi], s_first[sqi], s_cnt[sqi], s_con);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb) : "memory");
}

// The squad image of every stored schedule (the region [0, L.priv) of sq_layout): coefficients,
// the factor's node blocks packed as 28-float rows (inverse symmetrized: the backward sweep reads
// its columns as rows; rows >= 29 zero), bounds, scales, q^, flags.  One CTA per schedule id.
__global__ void sq_pack_kernel(const KParams P) {
  const int g = blockIdx.x;
  if (g >= min(*P.n_sched, P.store_cap)) return;
  const int NT = P.NT;
  const SqLayout L = sq_layout(NT);
  const StoreLayout SL = store_layout(NT);
  const float* entry = P.store + (size_t)g * P.store_stride;
  float* reg = P.sqpack + (size_t)g * L.priv;
  // SQ_PACK_SLICES CTAs per schedule (blockIdx.y): a few independent loads per thread, not a
  // serial loop of dependent L2 round trips
  const int t0 = blockIdx.y * blockDim.x + threadIdx.x, ts = gridDim.y * blockDim.x;
  for (int k = t0; k < (NT + 1) * C_SIZE; k += ts) reg[L.coef + k] = entry[SL.coef + k];
  for (int k = t0; k < (NT + 1) * NSLOT; k += ts) {
    reg[L.lo + k] = entry[SL.rows + 2 * k];
    reg[L.hi + k] = entry[SL.rows + 2 * k + 1];
    reg[L.d + k] = entry[SL.d + k];
  }
  for (int k = t0; k < NT * NV; k += ts) {
    reg[L.e + k] = entry[SL.e + k];
    reg[L.qh + k] = entry[SL.qh + k];
  }
  for (int k = t0; k <= NT; k += ts) reg[L.flags + k] = entry[SL.flags + k];
  for (int k = t0; k < NT * SQ_MF; k += ts) {
    const int i = k / SQ_MF, r = (k % SQ_MF) / SQ_MROW, c = k % SQ_MROW;
    const float* blk = entry + SL.blocks + (size_t)i * 32 * TCOLS;
    float v = 0.f;
    if (r < NV && c < NV) v = 0.5f * (blk[r * TCOLS + c] + blk[c * TCOLS + r]);
    else if (r < SROWS && c < NV) v = blk[r * TCOLS + c];
    reg[L.mf + k] = v;
  }
}

// Position in `order` of squad sq's first agent (squads are laid out group by group, so the
// agents of squads [0, sq) are the prefix order[0, sq_pos(sq))); sq past the last squad: the
// number of grouped agents.
__device__ __forceinline__ int sq_pos(const KParams& P, int sq) {
  const int ng = min(*P.n_sched, P.store_cap);
  if (ng <= 0) return 0;
  if (sq >= P.grp_cta[ng]) return P.grp_first[ng - 1] + P.grp_count[ng - 1];
  int lo = 0, hi = ng - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (P.grp_cta[mid] <= sq) lo = mid; else hi = mid - 1;
  }
  return P.grp_first[lo] + 32 * (sq - P.grp_cta[lo]);
}

// End-to-end output path of a split squad solve (rmpc_launch_shared with host outputs): copy the
// records and z* rows of the agents of squad CTAs [cta_lo, cta_hi) -- and, with `list`, of the
// per-agent list -- from the device buffers P.out / P.z_out to the mapped host buffers, one warp
// per agent, consecutive lanes on consecutive 8-byte words.  Runs beside the squad launch of the
// next CTA range, so the PCIe transfer of one wave overlaps the solve of the next.
__global__ void __launch_bounds__(256) sq_copyout_kernel(const KParams P, int cta_lo, int cta_hi, int list,
                                                         rmpc_solution* h_out, float* h_z, int spc) {
  const int p0 = sq_pos(P, spc * cta_lo), p1 = cta_hi >= (1 << 29) ? sq_pos(P, 1 << 30) : sq_pos(P, spc * cta_hi);
  const int nl = list ? *P.n_list : 0;
  const int lane = threadIdx.x & 31;
  const int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  const int zw = P.NT * NV / 2;  // float2 words of one agent's z*
  for (int k = wg; k < (p1 - p0) + nl; k += nw) {
    const int a = k < p1 - p0 ? P.order[p0 + k] : P.agent_list[k - (p1 - p0)];
    const float* rs = reinterpret_cast<const float*>(P.out + a);
    float* rd = reinterpret_cast<float*>(h_out + a);
    constexpr int RW = (int)(sizeof(rmpc_solution) / 4);
    for (int w = lane; w < RW; w += 32) rd[w] = rs[w];
    if (h_z) {
      const float2* zs = reinterpret_cast<const float2*>(P.z_out + (size_t)a * P.NT * NV);
      float2* zd = reinterpret_cast<float2*>(h_z + (size_t)a * P.NT * NV);
      for (int w = lane; w < zw; w += 32) zd[w] = zs[w];
    }
  }
}

}  // namespace rmpc_dev
