// rmpc_kernel.cu — fused warp-pair-per-agent RTI-MPC solve for sm_100a.
//
// One warp pair runs MpcController::rti_step (/root/reference/proj/src/mpc.cpp:248-338) for one
// agent: gait schedule and cold/warm guess (f_init, gait.cpp:37-99), FP64 linearization of
// the floating-base dynamics and contacts (robot.cpp:29-195), QP rows (build_qp,
// mpc.cpp:64-238), Ruiz passes (ruiz.cpp:7-36 via qp.cpp:64-95), factorization, exactly n_qp
// ADMM iterations (qp.cpp:156-190), unscaled residuals/objective (qp.cpp:192-200), the full
// step z* = guess + dz and inverse dynamics at node 0 (mpc.cpp:305-330, robot.cpp:211-233).
//
// Linear algebra.  Instead of the reference's quasi-definite KKT + sparse LDL^T (qp.cpp:11-34,
// ldl.cpp:123-192) each iteration solves the reduced SPD system
//     H x~ = r,  r = sigma x - q^ + A^T (rho z - y),  H = P^ + sigma I + rho A^T A,  z~ = A^ x~,
// identical in exact arithmetic (nu = rho (A^ x~ - z) + y eliminates the dual block).  H is
// block tridiagonal over horizon nodes; its off-diagonal blocks C_i = rho U_i V_i^T have rank
// 12 (the 9 integration + 3 dynamics rows of interval i).  Block elimination keeps
//     S_0 = H_00,  S_{i+1} = H_{i+1,i+1} - rho^2 U_i (V_i^T S_i^-1 V_i) U_i^T
// with S_i^-1 and W_i = S_i^-1 V_i(dyn) in tensor memory, so each iteration is
//     forward:  u_i = r_i - rho U_{i-1} gamma_{i-1},  s_i = S_i^-1 u_i,  gamma_i = V_i^T s_i
//     backward: x~_i = s_i - rho [S_i^-1 | W_i] xi_i,   xi_i = diag(a2, 1) U_i^T x~_{i+1}
// where gamma comes out of the same 29-row matvec as s (rows 26..28 = W^T) and the backward
// step is a 12-column update: no warp reductions on either recurrence.  The elimination is
// two-sided: warp 0 of the agent's pair runs nodes [0, m) top-down and the middle node m, warp 1
// runs (m, T) bottom-up (mirrored recurrences with T_i = D_i - rho^2 V_i G'_i V_i^T); the pair
// meets at the middle node only.  Six agents (warp pairs) share a CTA / SM.
//
// Precision: gait, guess, linearization, constraint right-hand sides, the objective and the
// inverse dynamics in FP64; Ruiz, H, S^-1 and the ADMM iterations in FP32.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "rmpc_device.cuh"
#include "rmpc_kin.cuh"

namespace rmpc_dev {

#define FULL 0xffffffffu

// ------------------------------------------------------------------------- helpers
struct Sm {
  float* scr;   // scratch (Ruiz d copy, factorization G blocks, FP64 z* rows)
  float* coef;  // block -1 at coef, node i at coef + (i + 1) * C_SIZE
  float* vec;
  float4* row;  // block -1 at row, node i at row + (i + 1) * NSLOT
  float* tt;    // rows[.].t again, one float per slot: conflict-free column-view gathers
  float* dsc;
  float* bc;
  uint32_t* flags;
  int NT;
  int mid;      // middle node: the top warp owns [0, mid], the bottom warp (mid, NT)
  uint32_t tm;  // TMEM address of this warp's first node block (lane quarter | column)
  int tmn;      // node blocks of this warp in TMEM; the rest are in `spill` (shared memory)
  float* spill;
  bool spills;  // compile-time constant per kernel instantiation (folds the TMEM-only path)
  int bar;      // named barrier of the agent's warp pair
  __device__ __forceinline__ float* C(int i) const { return coef + (i + 1) * C_SIZE; }
  __device__ __forceinline__ float4* R(int i) const { return row + (i + 1) * NSLOT; }
  __device__ __forceinline__ float* D(int i) const { return dsc + (i + 1) * NSLOT; }
  __device__ __forceinline__ float* T(int i) const { return tt + (i + 1) * NSLOT; }
  __device__ __forceinline__ float* V(int i, int which) const {
    return vec + (i * V_NUM + which) * V_STRIDE;
  }
  // index of node i among the blocks of the warp that owns it
  __device__ __forceinline__ int blk(int i) const { return i <= mid ? i : i - mid - 1; }
};

// ------------------------------------------------------------------------- sync / TMEM
// The two warps of an agent synchronise on their own named barrier (64 threads); barrier 0
// is the CTA-wide one used only around TMEM allocation.
__device__ __forceinline__ void pair_sync(const Sm& sm) {
  asm volatile("bar.sync %0, 64;" ::"r"(sm.bar) : "memory");
}
__device__ __forceinline__ bool pair_or(const Sm& sm, bool v) {
  int r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\tsetp.ne.s32 p, %1, 0;\n\tbar.red.or.pred q, %2, 64, p;\n\t"
      "selp.s32 %0, 1, 0, q;\n\t}"
      : "=r"(r)
      : "r"((int)v), "r"(sm.bar)
      : "memory");
  return r != 0;
}
__device__ __forceinline__ bool pair_and(const Sm& sm, bool v) {
  int r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\tsetp.ne.s32 p, %1, 0;\n\tbar.red.and.pred q, %2, 64, p;\n\t"
      "selp.s32 %0, 1, 0, q;\n\t}"
      : "=r"(r)
      : "r"((int)v), "r"(sm.bar)
      : "memory");
  return r != 0;
}

#define RMPC_X32(F, v)                                                                        \
  F(v[0]), F(v[1]), F(v[2]), F(v[3]), F(v[4]), F(v[5]), F(v[6]), F(v[7]), F(v[8]), F(v[9]),  \
      F(v[10]), F(v[11]), F(v[12]), F(v[13]), F(v[14]), F(v[15]), F(v[16]), F(v[17]),         \
      F(v[18]), F(v[19]), F(v[20]), F(v[21]), F(v[22]), F(v[23]), F(v[24]), F(v[25]),         \
      F(v[26]), F(v[27]), F(v[28]), F(v[29]), F(v[30]), F(v[31])
#define RMPC_OUT(x) "=f"(x)
#define RMPC_IN(x) "f"(x)
#define RMPC_OPS32                                                                              \
  "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24," \
  "%25,%26,%27,%28,%29,%30,%31}"
#define RMPC_OPS32_1                                                                           \
  "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25," \
  "%26,%27,%28,%29,%30,%31,%32}"

// Lane l of the warp reads / writes its TMEM row (lane quarter of the warp) at columns
// [a, a + 32): one 32x32b.x32 access moves a whole 26-float block row plus its W entries.
// Split form: issue the load, do independent work, then wait (v is tied to the wait so the
// compiler cannot consume it earlier).
__device__ __forceinline__ void tm_load_issue(uint32_t a, float v[TCOLS]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 " RMPC_OPS32 ", [%32];"
               : RMPC_X32(RMPC_OUT, v)
               : "r"(a));
}
#define RMPC_INOUT(x) "+f"(x)
__device__ __forceinline__ void tm_load_wait(float v[TCOLS]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" : RMPC_X32(RMPC_INOUT, v)::"memory");
}
__device__ __forceinline__ void tm_store(uint32_t a, const float v[TCOLS]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], " RMPC_OPS32_1 ";"
               ::"r"(a), RMPC_X32(RMPC_IN, v)
               : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// Node block rows: TMEM for the warp's first `tmn` blocks, else a shared-memory copy whose
// rows (32 floats per lane) have their float4 chunks XOR-swizzled by lane & 7 so eight
// consecutive lanes' LDS.128 hit distinct banks.  The branch is warp-uniform.
__device__ __forceinline__ const float4* spill_row(const Sm& sm, int b, int lane) {
  return reinterpret_cast<const float4*>(sm.spill + (b - sm.tmn) * SPILL_BLK + lane * TCOLS);
}
__device__ __forceinline__ void blk_load_issue(const Sm& sm, int i, int lane, float v[TCOLS]) {
  const int b = sm.blk(i);
  if (!sm.spills || b < sm.tmn) {
    tm_load_issue(sm.tm + (uint32_t)(TCOLS * b), v);
  } else {
    const float4* r = spill_row(sm, b, lane);
#pragma unroll
    for (int c = 0; c < TCOLS / 4; ++c) {
      const float4 w = r[c ^ (lane & 7)];
      v[4 * c] = w.x; v[4 * c + 1] = w.y; v[4 * c + 2] = w.z; v[4 * c + 3] = w.w;
    }
  }
}
__device__ __forceinline__ void blk_load_wait(const Sm& sm, int i, float v[TCOLS]) {
  if (!sm.spills || sm.blk(i) < sm.tmn) tm_load_wait(v);
}
__device__ __forceinline__ void blk_load(const Sm& sm, int i, int lane, float v[TCOLS]) {
  blk_load_issue(sm, i, lane, v);
  blk_load_wait(sm, i, v);
}
__device__ __forceinline__ void blk_store(const Sm& sm, int i, int lane, const float v[TCOLS]) {
  const int b = sm.blk(i);
  if (!sm.spills || b < sm.tmn) {
    tm_store(sm.tm + (uint32_t)(TCOLS * b), v);
  } else {
    float4* r = const_cast<float4*>(spill_row(sm, b, lane));
#pragma unroll
    for (int c = 0; c < TCOLS / 4; ++c) r[c ^ (lane & 7)] = make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
  }
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

__device__ __forceinline__ double wcost(const KParams& P, int j) {
  return j < 9 ? P.wq[j] : (j < 18 ? P.wqd[j - 9] : P.wf[j - 18]);
}

// Ruiz-scaled P diagonal of node i, var j: w_j dt_i e_j^2 (mpc.cpp:81-103).
__device__ __forceinline__ float phat(const KParams& P, const Sm& sm, int i, int j) {
  const float e = sm.V(i, V_E)[j];
  return (float)(wcost(P, j) * P.dt[i]) * e * e;
}

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
  float acc0 = Op::id(), acc1 = Op::id();
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
    if (k & 1) acc1 = Op::comb(acc1, c, v);
    else acc0 = Op::comb(acc0, c, v);
  }
  return Op::red(acc0, acc1);
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

// ------------------------------------------------------------------------- stage: setup
// Lane i < NT builds node i of the QP (build_qp, mpc.cpp:64-238) in FP64 and stores the
// unscaled coefficients, bounds and q in shared memory.  Returns false if the linearization
// point is non-finite (StructuralError, mpc.cpp:70-72).
// Warp 0's share: lane i < NT builds node i's integration, contact, box and initial-state rows
// (setup_dynamics below builds the base-dynamics rows and q^ on warp 1).
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
    float4* rw = sm.R(i);
    const double dt = P.dt[i];

    Frames F;
    fk_frames(P, gq, gqd, F);
    double Jx[4][9], Jz[4][9];
#pragma unroll
    for (int c = 0; c < 4; ++c) contact_jac(F, c, Jx[c], Jz[c]);

    if (i + 1 < NT) {
#pragma unroll
      for (int k = 0; k < 9; ++k) {  // integration (mpc.cpp:138-148)
        cf[C_A1 + k] = 1.f;
        cf[C_A2 + k] = -1.f;
        cf[C_A3 + k] = to_f(-dt);
        const double r = -(nq[k] - gq[k] - dt * nqd[k]);
        set_row(rw + k, r, r);
      }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {  // contacts (mpc.cpp:181-218)
      const double fx = gF[2 * c], fz = gF[2 * c + 1];
      float4* r0 = rw + 12 + 4 * c;
      if ((bits >> c) & 1u) {
        cf[C_FORCE + 4 * c + 0] = 1.f;
        cf[C_FORCE + 4 * c + 1] = to_f(-P.mu);
        cf[C_FORCE + 4 * c + 2] = -1.f;
        cf[C_FORCE + 4 * c + 3] = to_f(-P.mu);
        set_row(r0, -1e30, -(fx - P.mu * fz));
        set_row(r0 + 1, -1e30, -(-fx - P.mu * fz));
        if (i > 0) {
          double v0 = 0.0, v1 = 0.0;
#pragma unroll
          for (int k = 0; k < 9; ++k) {
            v0 += Jx[c][k] * gqd[k];
            v1 += Jz[c][k] * gqd[k];
            cf[C_JA + 9 * c + k] = to_f(Jx[c][k]);
            cf[C_JB + 9 * c + k] = to_f(Jz[c][k]);
          }
          set_row(r0 + 2, -v0, -v0);
          set_row(r0 + 3, -v1, -v1);
        }
      } else {
        cf[C_FORCE + 4 * c + 0] = 1.f;
        cf[C_FORCE + 4 * c + 3] = 1.f;
        set_row(r0, -fx, -fx);
        set_row(r0 + 1, -fz, -fz);
        if (i > 0) {
          const double h = bezier_height(swt[c], P.z_swing, P.v_to, P.v_td);
          const double r = h - F.con[c].pz;
#pragma unroll
          for (int k = 0; k < 9; ++k) cf[C_JAQ + 9 * c + k] = to_f(Jz[c][k]);
          set_row(r0 + 2, r, r);
        }
      }
    }
    if (i > 0) {  // joint boxes (mpc.cpp:220-232)
#pragma unroll
      for (int m = 0; m < 6; ++m) {
        cf[C_BOX + m] = 1.f;
        set_row(rw + 28 + m, P.jlo[m] - gq[3 + m], P.jhi[m] - gq[3 + m]);
        cf[C_BOX + 6 + m] = 1.f;
        set_row(rw + 34 + m, -P.qdlim[m] - gqd[3 + m], P.qdlim[m] - gqd[3 + m]);
      }
    } else {  // initial state (mpc.cpp:126-136), rows in block -1
      float4* ri = sm.R(-1) + INIT0;
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        cf[C_INIT + k] = 1.f;
        cf[C_INIT + 9 + k] = 1.f;
        const double rq = st.q[k] - gq[k], rqd = st.qd[k] - gqd[k];
        set_row(ri + k, rq, rq);
        set_row(ri + 9 + k, rqd, rqd);
      }
    }
  }
  return __all_sync(FULL, ok);
}

// Warp 1's share of the setup: the base-dynamics rows of every interval with qdd eliminated
// (mpc.cpp:150-175), one lane per (node, row b), and q^ = w dt (guess - desired)
// (mpc.cpp:81-103), one lane per node.
__device__ bool setup_dynamics(const KParams& P, const Sm& sm, int lane, const rmpc_state& st,
                               const rmpc_command& cmd, const rmpc_gait& gait, bool warm,
                               const float* pz) {
  const int NT = P.NT;
  bool ok = true;
  uint32_t* bits_of = reinterpret_cast<uint32_t*>(sm.scr);  // scratch is free until Ruiz
  for (int i = lane; i < NT; i += 32) {
    double swt[4];
    bits_of[i] = node_schedule(P, gait, i, swt);
  }
  __syncwarp();
  // one lane per (node, row) while that fits the warp, else one lane per node (FK once)
  const bool split = 3 * (NT - 1) <= 32;
#pragma unroll 1
  for (int t = lane; t < (split ? 3 : 1) * (NT - 1); t += 32) {
    const int i = t % (NT - 1);
    const int b0 = split ? t / (NT - 1) : 0, b1 = split ? b0 + 1 : 3;
    const uint32_t bits = bits_of[i], bits_n = bits_of[i + 1];
    double gq[9], gqd[9], gF[8], nq[9], nqd[9], nF[8];
    node_guess(P, i, warm, pz, st, bits, gq, gqd, gF);
    node_guess(P, i + 1, warm, pz, st, bits_n, nq, nqd, nF);
#pragma unroll
    for (int k = 0; k < 9; ++k) ok = ok && isfinite(gq[k]) && isfinite(gqd[k]);
    Frames F;
    fk_frames(P, gq, gqd, F);
    const double dt_inv = 1.0 / P.dt[i];
#pragma unroll 1
    for (int b = b0; b < b1; ++b) {
    double Mr[9], hr;
    base_dynamics_row(P, gqd, F, b, Mr, hr);
    double mq = 0.0;
#pragma unroll
    for (int k = 0; k < 9; ++k) mq += Mr[k] * (nqd[k] - gqd[k]);
    // column b of the contact Jacobians: b = 0, 1 base translation, b = 2 pitch (robot.cpp:98)
    double jbf = 0.0, jx[4], jz[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      jx[c] = b == 0 ? 1.0 : (b == 1 ? 0.0 : -(F.con[c].pz - F.piv[2].pz));
      jz[c] = b == 0 ? 0.0 : (b == 1 ? 1.0 : F.con[c].px - F.piv[2].px);
      jbf += jx[c] * gF[2 * c] + jz[c] * gF[2 * c + 1];
    }
    const double resid = mq * dt_inv + hr - jbf;
    float* cf = sm.C(i);
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      const double mv = Mr[k] * dt_inv;
      cf[C_DYNU + 12 * b + k] = to_f(mv);
      cf[C_DYNV + 20 * b + k] = to_f(-mv);
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      cf[C_DYNV + 20 * b + 9 + 2 * c] = to_f(-jx[c]);
      cf[C_DYNV + 20 * b + 10 + 2 * c] = to_f(-jz[c]);
    }
    set_row(sm.R(i) + 9 + b, -resid, -resid);
    }
  }
#pragma unroll 1
  for (int i = lane; i < NT; i += 32) {
    float* qh = sm.V(i, V_QH);
#pragma unroll 1
    for (int j = 0; j < NV; ++j) {
      double g, des;
      guess_and_target(P, i, j, warm, pz, st, cmd, bits_of[i], g, des);
      qh[j] = to_f(wcost(P, j) * P.dt[i] * (g - des));
    }
  }
  return __all_sync(FULL, ok);
}

// ------------------------------------------------------------------------- stage: Ruiz
// AdmmSolver::equilibrate (qp.cpp:64-95) + ruiz_equilibrate (ruiz.cpp:7-36) on
// [[P, A^T], [A, 0]]: each pass takes delta = 1/sqrt(inf-norm) of every row/column of the
// current scaled matrix (1 for empty ones), then d *= delta (rows), e *= delta (columns).
// Row deltas are parked in row.z, column deltas in V_S until the pass is applied.
__device__ void ruiz(const KParams& P, const Sm& sm, int lane, int warp) {
  const int NT = P.NT;
  Terms T;
  build_terms(lane, T);
  TermBytes B;
  term_bytes<TV_D>(T, B);
  // Double-buffered scales: pass p reads (d, e) from one copy and writes d delta, e delta to
  // the other, so one barrier per pass suffices.  The second d lives in the scratch region,
  // the second e in V_S.
  const int nd = (NT + 1) * NSLOT;
  for (int r = lane + 32 * warp; r < nd; r += 64) sm.scr[r] = sm.dsc[r];
  pair_sync(sm);
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
    auto update_rows = [&](int i, const Norms& n) {  // writes only the destination copies
      const float* d = src.D(i);
      float* dn = dst + (i + 1) * NSLOT;
      dn[lane] = d[lane] * inv_sqrt1(d[lane] * n.o0);
      if (lane < 8) dn[32 + lane] = d[32 + lane] * inv_sqrt1(d[32 + lane] * n.o1);
      if (i == 0 && lane < NINIT) {
        const float* d0 = src.D(-1) + INIT0;
        dst[INIT0 + lane] = d0[lane] * inv_sqrt1(d0[lane] * n.o2);
      }
    };
    auto update_cols = [&](int i, const Norms& n) {
      if (lane < NV) {
        const float e = sm.V(i, es)[lane];
        const float pd = wl * (float)P.dt[i];
        sm.V(i, ed)[lane] = e * inv_sqrt1(e * fmaxf(fabsf(pd) * e, n.cv));
      }
    };
    auto update = [&](int i, const Norms& n) {
      update_rows(i, n);
      update_cols(i, n);
    };
    // nodes are independent within a pass: two per iteration, all loads ahead of the stores;
    // for odd T the last node is split: warp 0 its row scales, warp 1 its column scales
    const int ne = NT & ~1;
    int i = warp;
#pragma unroll 1
    for (; i + 2 < ne; i += 4) {
      const Norms a = norms(i), b = norms(i + 2);
      update(i, a);
      update(i + 2, b);
    }
    if (i < ne) update(i, norms(i));
    if (NT & 1) {
      Norms n;
      if (warp == 0) {
        row_view<OpMax>(src, NT - 1, lane, es, n.o0, n.o1, n.o2);
        update_rows(NT - 1, n);
      } else {
        n.cv = col_view<OpMax, TV_D>(src, NT - 1, T, B);
        update_cols(NT - 1, n);
      }
    }
    pair_sync(sm);  // every norm of the next pass uses the scales of this one
  }
  if (P.ruiz_iters & 1) {  // the last pass wrote the second copies
    for (int r = lane + 32 * warp; r < nd; r += 64) sm.dsc[r] = sm.scr[r];
    for (int i = warp; i < NT; i += 2)
      if (lane < NV) sm.V(i, V_E)[lane] = sm.V(i, V_S)[lane];
    pair_sync(sm);
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

// ------------------------------------------------------------------------- kernel
__device__ __forceinline__ void prof_mark(const KParams& P, int lane, int stage, long long& t0) {
  if (P.profile) {
    const long long t1 = clock64();
    if (lane == 0) atomicAdd(P.prof + stage, (unsigned long long)(t1 - t0));
    t0 = t1;
  }
}

// One agent on one warp pair of the CTA: its shared-memory block at `base`, its TMEM node
// blocks at `tm`, named barrier `bar`.
template <bool SPILL>
__device__ __forceinline__ void solve_agent(const KParams& P, float* base, uint32_t tm, int tmn, int bar,
                                            int agent, int lane, int warp) {
  const int NT = P.NT;
  const Layout L = make_layout(NT, P.spill_nodes);
  Sm sm;
  sm.scr = base + L.scr;
  sm.coef = base + L.coef;
  sm.vec = base + L.vec;
  sm.row = reinterpret_cast<float4*>(base + L.row);
  sm.tt = base + L.tt;
  sm.dsc = base + L.dsc;
  sm.bc = base + L.bc;
  sm.flags = reinterpret_cast<uint32_t*>(base + L.flags);
  sm.NT = NT;
  sm.mid = mid_node(NT);
  sm.tm = tm;
  sm.tmn = tmn;
  sm.spills = SPILL;
  sm.spill = base + L.spill + warp * P.spill_nodes * SPILL_BLK;
  sm.bar = bar;
  const int tid = warp * 32 + lane;
  long long t0 = P.profile ? clock64() : 0;

  // zero coefficients (incl. block -1), rows, vectors; d = e = 1
  for (int k = tid; k < (NT + 1) * C_SIZE; k += 64) sm.coef[k] = 0.f;
  for (int r = tid; r < (NT + 1) * NSLOT; r += 64) {
    sm.row[r] = make_float4(0.f, 0.f, 0.f, 0.f);
    sm.tt[r] = 0.f;
    sm.dsc[r] = 1.f;
  }
  for (int k = tid; k < NT * V_NUM * V_STRIDE; k += 64) sm.vec[k] = 0.f;
  pair_sync(sm);
  for (int i = warp; i < NT; i += 2)
    if (lane < NV) sm.V(i, V_E)[lane] = 1.f;
  sm.bc[tid] = 0.f;

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
  prof_mark(P, tid, 0, t0);
  pair_sync(sm);

  int ok = 1;
  ok = (warp == 0 ? setup_nodes(P, sm, lane, st, cmd, gait, warm, pz)
                  : setup_dynamics(P, sm, lane, st, cmd, gait, warm, pz)) && st_ok;
  ok = pair_and(sm, ok);
  prof_mark(P, tid, 2, t0);
  if (!ok) {
    out.status = RMPC_STATUS_NONFINITE_INPUT;
  } else {
    if (P.ruiz_iters > 0) ruiz(P, sm, lane, warp);
    apply_scaling(P, sm, lane, warp);
    prof_mark(P, tid, 3, t0);
    const int good = factorize(P, sm, lane, warp);
    if (!good) {
      out.status = RMPC_STATUS_SINGULAR;
    } else {
      prof_mark(P, tid, 4, t0);
      const int bad_it = admm(P, sm, lane, warp);
      prof_mark(P, tid, 5, t0);
      if (bad_it >= 0) {
        out.status = RMPC_STATUS_DIVERGED;
        out.fail_iter = bad_it;
      }
    }
  }
  if (out.status == RMPC_STATUS_OK) {  // (pair-uniform) residuals, objective, z*: nodes split
                                       // between the warps; inverse dynamics on warp 0
    // unscaled residuals (qp.cpp:192-200): prim = |A^x - z| / d, dual = |P^x + q^ + A^T y| / e
    Terms T;
    build_terms(lane, T);
    TermBytes B;
    term_bytes<TV_Y>(T, B);
    float prim = 0.f, dual = 0.f, dinf = 0.f;
    double obj = 0.0;
    const float rho = (float)P.rho;
#pragma unroll 1
    for (int i = warp; i < NT; i += 2) {
      float o0, o1, o2;
      row_view<OpSum>(sm, i, lane, V_X, o0, o1, o2);
      const float4* rw = sm.R(i);
      const float* d = sm.D(i);
      prim = fmaxf(prim, fabsf(o0 - rw[lane].z) / d[lane]);
      if (lane < 8) prim = fmaxf(prim, fabsf(o1 - rw[32 + lane].z) / d[32 + lane]);
      if (i == 0 && lane < NINIT)
        prim = fmaxf(prim, fabsf(o2 - sm.R(-1)[INIT0 + lane].z) / sm.D(-1)[INIT0 + lane]);
      if (P.act_out) {  // active set of the final iterate (scaled space, where the clamp acts)
        uint8_t* ao = P.act_out + (size_t)agent * (NT + 1) * NSLOT;
        auto code = [](float4 r) -> uint8_t { return r.x == r.y ? 3 : (r.z == r.x ? 1 : (r.z == r.y ? 2 : 0)); };
        ao[(i + 1) * NSLOT + lane] = code(rw[lane]);
        if (lane < 8) ao[(i + 1) * NSLOT + 32 + lane] = code(rw[32 + lane]);
        if (i == 0 && lane < NSLOT) ao[lane] = code(sm.R(-1)[lane < NSLOT ? lane : 0]);
        if (i == 0 && lane < NSLOT - 32) ao[32 + lane] = code(sm.R(-1)[32 + lane]);
      }
      const float aty = col_view<OpSum, TV_Y>(sm, i, T, B, rho);
      const uint32_t bits = sm.flags[i];
      if (lane < NV) {
        const float x = sm.V(i, V_X)[lane], e = sm.V(i, V_E)[lane];
        dual = fmaxf(dual, fabsf(phat(P, sm, i, lane) * x + sm.V(i, V_QH)[lane] + aty) / e);
        // objective on the unscaled problem in FP64: 1/2 w dt dz^2 + w dt (g - des) dz
        double g, des;
        guess_and_target(P, i, lane, warm, pz, st, cmd, bits, g, des);
        const double w = wcost(P, lane) * P.dt[i];
        const double dz = (double)e * (double)x;
        obj += 0.5 * w * dz * dz + w * (g - des) * dz;
        dinf = fmaxf(dinf, fabsf(e * x));
        const double zv = g + dz;  // z* = guess + dz (mpc.cpp:308-314)
        if (P.z_out) P.z_out[((size_t)agent * NT + i) * NV + lane] = (float)zv;
        if (i < 2) reinterpret_cast<double*>(sm.scr)[i * 32 + lane] = zv;
      }
    }
    prim = wmax(prim);
    dual = wmax(dual);
    dinf = wmax(dinf);
    obj = wsumd(obj);
    if (warp == 1 && lane == 0) {
      sm.bc[0] = prim;
      sm.bc[1] = dual;
      sm.bc[2] = dinf;
      reinterpret_cast<double*>(sm.bc)[2] = obj;
    }
    pair_sync(sm);
    if (warp != 0) return;
    prim = fmaxf(prim, sm.bc[0]);
    dual = fmaxf(dual, sm.bc[1]);
    dinf = fmaxf(dinf, sm.bc[2]);
    obj += reinterpret_cast<const double*>(sm.bc)[2];
    out.prim_res = prim;
    out.dual_res = dual;
    out.delta_inf_norm = dinf;
    out.v_mpc = (float)obj;
    __syncwarp();
    if (lane == 0) {  // inverse dynamics at node 0 (mpc.cpp:320-330), FP64
      const double* z0 = reinterpret_cast<const double*>(sm.scr);
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
  } else {
    if (warp != 0) return;
    if (P.z_out != nullptr)
      for (int k = lane; k < NT * NV; k += 32) P.z_out[(size_t)agent * NT * NV + k] = 0.f;
    if (P.act_out != nullptr)
      for (int k = lane; k < (NT + 1) * NSLOT; k += 32) P.act_out[(size_t)agent * (NT + 1) * NSLOT + k] = 3;
  }
  prof_mark(P, lane, 6, t0);
  if (lane == 0) P.out[agent] = out;
}

// CTA = P.agents_per_cta warp pairs.  Warp w uses TMEM lanes [32 (w % 4), +32) (the quarter
// tcgen05.ld/st of warp w can reach) and columns [(w / 4) tmn 32, +tmn 32), tmn = the node
// blocks its quarter's share holds (tm_nodes); further blocks go to its shared-memory spill.
template <bool SPILL>
__global__ void __launch_bounds__(64 * MAX_AGENTS, 1) rti_kernel(const KParams P) {
  extern __shared__ __align__(16) float smem[];
  __shared__ uint32_t tmem_base;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tmem_base)),
                 "r"(P.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = tmem_base;
  const int pair = w >> 1;
  const int b = blockIdx.x;
  const int agent = b < P.full_ctas ? b * P.agents_per_cta + pair
                                    : (pair < P.tail_agents ? P.full_ctas * P.agents_per_cta +
                                                                   (b - P.full_ctas) * P.tail_agents + pair
                                                             : P.n_agents);
  if (agent < P.n_agents) {
    const int tmn = tm_nodes(P.NT, P.agents_per_cta, w & 3);
    const uint32_t tm = tb + ((uint32_t)(32 * (w & 3)) << 16) + (uint32_t)((w >> 2) * tmn * TCOLS);
    solve_agent<SPILL>(P, smem + pair * make_layout(P.NT, P.spill_nodes).total, tm, tmn, 1 + pair, agent, lane,
                       w & 1);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (w == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(P.tmem_cols) : "memory");
}

}  // namespace rmpc_dev

int rmpc_kernel_setup(int) {
  const int bytes = 227 * 1024 - 128;  // static smem: the TMEM base
  int rc = (int)cudaFuncSetAttribute(rmpc_dev::rti_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (rc == 0)
    rc = (int)cudaFuncSetAttribute(rmpc_dev::rti_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  return rc;
}

int rmpc_launch_rti(const rmpc_dev::KParams& params, void* stream) {
  if (params.n_agents <= 0) return 0;
  const rmpc_dev::CtaShape c = rmpc_dev::cta_shape(params.NT);
  rmpc_dev::KParams P = params;
  P.agents_per_cta = c.agents;
  P.spill_nodes = c.spill_nodes;
  P.tmem_cols = c.tmem_cols;
  // Whole waves of full CTAs (one CTA per SM), then the remainder spread over the SMs at
  // ceil(R / SMs) agents per CTA: a partial wave of fewer agents per SM runs faster than a
  // partial wave of full CTAs on a subset of the SMs.
  static int sms[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && sms[dev] == 0) cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev);
  const int nsm = dev < 64 && sms[dev] > 0 ? sms[dev] : 148;
  const int wave = nsm * c.agents;
  const int full_waves = P.n_agents / wave;
  const int rem = P.n_agents - full_waves * wave;
  int tail = 0, tail_ctas = 0;
  if (rem > 0) {
    tail = (rem + nsm - 1) / nsm;
    tail_ctas = (rem + tail - 1) / tail;
  }
  P.full_ctas = full_waves * nsm;
  P.tail_agents = tail;
  const int grid = P.full_ctas + tail_ctas;
  if (c.spill_nodes > 0)
    rmpc_dev::rti_kernel<true><<<grid, 64 * c.agents, c.smem_bytes, (cudaStream_t)stream>>>(P);
  else
    rmpc_dev::rti_kernel<false><<<grid, 64 * c.agents, c.smem_bytes, (cudaStream_t)stream>>>(P);
  return (int)cudaGetLastError();
}
