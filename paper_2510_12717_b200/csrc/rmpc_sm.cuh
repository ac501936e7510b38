// rmpc_sm.cuh — per-agent shared-memory view (Sm), warp helpers, pair barriers, TMEM access and the node-block store (TMEM or swizzled shared-memory spill).
// Part of the fused solve kernel: included once, in order, by rmpc_kernel.cu.
#pragma once

#include "rmpc_device.cuh"
#include "rmpc_kin.cuh"

namespace rmpc_dev {

#ifndef FULL
#define FULL 0xffffffffu
#endif

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

}  // namespace rmpc_dev
