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
// meets at the middle node only.  Six agents (warp pairs) share a CTA / SM (eight, under a
// 128-register cap, for horizons <= 8: rti_kernel<SPILL, MAXA>).
//
// Precision: gait, guess, linearization, constraint right-hand sides, the objective and the
// inverse dynamics in FP64; Ruiz, H, S^-1 and the ADMM iterations in FP32.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <atomic>

#include "rmpc_device.cuh"
#include "rmpc_kin.cuh"

#include "rmpc_sm.cuh"
#include "rmpc_views.cuh"
#include "rmpc_model.cuh"
#include "rmpc_setup.cuh"
#include "rmpc_ruiz.cuh"
#include "rmpc_factor.cuh"
#include "rmpc_admm.cuh"

namespace rmpc_dev {

// ------------------------------------------------------------------------- kernel
__device__ __forceinline__ void prof_mark(const KParams& P, int lane, int stage, long long& t0) {
  if (P.profile) {
    const long long t1 = clock64();
    if (lane == 0) {
      const unsigned long long d = (unsigned long long)(t1 - t0);
      atomicAdd(P.prof + stage, d);
      atomicAdd(P.prof + RMPC_NUM_STAGES + stage, d * d);
    }
    t0 = t1;
  }
}

// ------------------------------------------------------------------------- schedule store
// Mode 1: after the factorization of a schedule's representative agent, copy everything the
// rest of the solve reads from the schedule-dependent part -- the scaled coefficient blocks
// (with the G_dd entries factorize left in them), e, d, the stance flags and the factor's
// node blocks (each warp its own, as TMEM rows) -- into the store entry `st`.
__device__ void dump_schedule(const KParams& P, const Sm& sm, float* st, int lane, int warp, int status) {
  const int NT = P.NT, tid = warp * 32 + lane;
  const StoreLayout SL = store_layout(NT);
  const float4* c4 = reinterpret_cast<const float4*>(sm.coef);
  float4* o4 = reinterpret_cast<float4*>(st + SL.coef);
  for (int k = tid; k < (NT + 1) * C_SIZE / 4; k += 64) o4[k] = c4[k];
  const float4* d4 = reinterpret_cast<const float4*>(sm.dsc);
  float4* od = reinterpret_cast<float4*>(st + SL.d);
  for (int k = tid; k < (NT + 1) * NSLOT / 4; k += 64) od[k] = d4[k];
  for (int k = tid; k < NT * NV; k += 64) st[SL.e + k] = sm.V(k / NV, V_E)[k % NV];
  int32_t* fl = reinterpret_cast<int32_t*>(st + SL.flags);
  for (int i = tid; i < NT; i += 64) fl[i] = (int32_t)sm.flags[i];
  if (tid == 0) fl[NT] = status;
  const int m = sm.mid;
  for (int i = warp == 0 ? 0 : m + 1; i <= (warp == 0 ? m : NT - 1); ++i) {
    float v[TCOLS];
    blk_load(sm, i, lane, v);
    float4* r = reinterpret_cast<float4*>(st + SL.blocks + (size_t)(i * 32 + lane) * TCOLS);
#pragma unroll
    for (int q = 0; q < TCOLS / 4; ++q) r[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  }
}

// Mode 0, shared schedule: load the entry instead of Ruiz + scaling + factorize, and scale this
// agent's bounds and q by d / e exactly as apply_scaling does.  Returns the factorization
// status (1 ok, 0 singular).  The results are bit-identical to the agent's own factorization.
__device__ int load_schedule(const KParams& P, const Sm& sm, const float* st, int lane, int warp) {
  const int NT = P.NT, tid = warp * 32 + lane;
  const StoreLayout SL = store_layout(NT);
  const float4* c4 = reinterpret_cast<const float4*>(st + SL.coef);
  float4* s4 = reinterpret_cast<float4*>(sm.coef);
  for (int k = tid; k < (NT + 1) * C_SIZE / 4; k += 64) s4[k] = c4[k];
  const float4* d4 = reinterpret_cast<const float4*>(st + SL.d);
  float4* sd = reinterpret_cast<float4*>(sm.dsc);
  for (int k = tid; k < (NT + 1) * NSLOT / 4; k += 64) sd[k] = d4[k];
  for (int k = tid; k < NT * NV; k += 64) sm.V(k / NV, V_E)[k % NV] = st[SL.e + k];
  const int m = sm.mid;
  for (int i = warp == 0 ? 0 : m + 1; i <= (warp == 0 ? m : NT - 1); ++i) {
    const float4* r = reinterpret_cast<const float4*>(st + SL.blocks + (size_t)(i * 32 + lane) * TCOLS);
    float v[TCOLS];
#pragma unroll
    for (int q = 0; q < TCOLS / 4; ++q) {
      const float4 w = r[q];
      v[4 * q] = w.x; v[4 * q + 1] = w.y; v[4 * q + 2] = w.z; v[4 * q + 3] = w.w;
    }
    blk_store(sm, i, lane, v);
  }
  pair_sync(sm);
  for (int i = warp; i < NT; i += 2)
    if (lane < NV) sm.V(i, V_QH)[lane] *= sm.V(i, V_E)[lane];
  for (int r = tid; r < (NT + 1) * NSLOT; r += 64) {
    float4 rd = sm.row[r];
    const float dr = sm.dsc[r];
    rd.x *= dr;
    rd.y *= dr;
    sm.row[r] = rd;
  }
  pair_sync(sm);
  return reinterpret_cast<const int32_t*>(st + SL.flags)[NT];
}

// One agent on one warp pair of the CTA: its shared-memory block at `base`, its TMEM node
// blocks at `tm`, named barrier `bar`.  `sched` is the schedule id the pair builds in mode 1.
template <bool SPILL>
__device__ __forceinline__ void solve_agent(const KParams& P, float* base, uint32_t tm, int tmn, int bar,
                                            int agent, int sched, int lane, int warp) {
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
  if (P.mode == 1 && !ok) {  // cannot happen for a representative (finite inputs); unshared
    if (tid == 0) reinterpret_cast<int32_t*>(P.store + (size_t)sched * P.store_stride + store_layout(NT).flags)[NT] = -1;
    return;
  }
  if (!ok) {
    out.status = RMPC_STATUS_NONFINITE_INPUT;
  } else {
    // the schedule's precomputed entry, if any (mode 0); a flag mismatch (hash collision) or an
    // invalid entry falls back to the agent's own factorization
    const float* entry = nullptr;
    if (P.mode == 0 && P.slot_of != nullptr) {
      const int sl = P.slot_of[agent];
      const int sid = sl >= 0 ? P.slot_id[sl] : -1;
      if (sid >= 0 && sid < P.store_cap) {
        entry = P.store + (size_t)sid * P.store_stride;
        const int32_t* fl = reinterpret_cast<const int32_t*>(entry + store_layout(NT).flags);
        bool same = fl[NT] >= 0;
        for (int i = tid; i < NT; i += 64) same = same && (uint32_t)fl[i] == sm.flags[i];
        if (!pair_and(sm, same)) entry = nullptr;
      }
    }
    int good;
    if (entry != nullptr) {
      good = load_schedule(P, sm, entry, lane, warp);
      prof_mark(P, tid, 3, t0);
    } else {
      if (P.ruiz_iters > 0) ruiz(P, sm, lane, warp);
      apply_scaling(P, sm, lane, warp);
      prof_mark(P, tid, 3, t0);
      good = factorize(P, sm, lane, warp);
      if (P.mode == 1) {
        dump_schedule(P, sm, P.store + (size_t)sched * P.store_stride, lane, warp, good ? 1 : 0);
        return;
      }
    }
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
template <bool SPILL, int MAXA>
__global__ void __launch_bounds__(64 * MAXA, 1) rti_kernel(const KParams P) {
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
  int agent, sched = -1;
  if (P.mode == 1) {  // schedule store: pair -> schedule id -> its representative agent
    sched = b * P.agents_per_cta + pair;
    const int ns = min(*P.n_sched, P.store_cap);
    agent = sched < ns ? P.rep_list[sched] : P.n_agents;
  } else {
    agent = b < P.full_ctas ? b * P.agents_per_cta + pair
                            : (pair < P.tail_agents ? P.full_ctas * P.agents_per_cta +
                                                           (b - P.full_ctas) * P.tail_agents + pair
                                                     : P.n_agents);
  }
  if (agent < P.n_agents) {
    const int tmn = tm_nodes(P.NT, P.agents_per_cta, w & 3);
    const uint32_t tm = tb + ((uint32_t)(32 * (w & 3)) << 16) + (uint32_t)((w >> 2) * tmn * TCOLS);
    solve_agent<SPILL>(P, smem + pair * make_layout(P.NT, P.spill_nodes).total, tm, tmn, 1 + pair, agent, sched,
                       lane, w & 1);
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
  const cudaFuncAttribute a = cudaFuncAttributeMaxDynamicSharedMemorySize;
  int rc = (int)cudaFuncSetAttribute(rmpc_dev::rti_kernel<false, rmpc_dev::MAX_AGENTS>, a, bytes);
  if (rc == 0) rc = (int)cudaFuncSetAttribute(rmpc_dev::rti_kernel<true, rmpc_dev::MAX_AGENTS>, a, bytes);
  if (rc == 0) rc = (int)cudaFuncSetAttribute(rmpc_dev::rti_kernel<false, rmpc_dev::DENSE_AGENTS>, a, bytes);
  return rc;
}

static int launch_variant(const rmpc_dev::KParams& P, const rmpc_dev::CtaShape& c, int grid, cudaStream_t st) {
  if (grid <= 0) return 0;
  if (c.dense)
    rmpc_dev::rti_kernel<false, rmpc_dev::DENSE_AGENTS><<<grid, 64 * c.agents, c.smem_bytes, st>>>(P);
  else if (c.spill_nodes > 0)
    rmpc_dev::rti_kernel<true, rmpc_dev::MAX_AGENTS><<<grid, 64 * c.agents, c.smem_bytes, st>>>(P);
  else
    rmpc_dev::rti_kernel<false, rmpc_dev::MAX_AGENTS><<<grid, 64 * c.agents, c.smem_bytes, st>>>(P);
  return (int)cudaGetLastError();
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
  // SM count per device, cached; several host threads (one per shard) may launch at once
  static std::atomic<int> sms[64];
  int dev = 0;
  cudaGetDevice(&dev);
  int nsm = dev < 64 ? sms[dev].load(std::memory_order_relaxed) : 0;
  if (nsm == 0) {
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (nsm <= 0) nsm = 148;
    if (dev < 64) sms[dev].store(nsm, std::memory_order_relaxed);
  }
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
  return launch_variant(P, c, P.full_ctas + tail_ctas, (cudaStream_t)stream);
}

namespace rmpc_dev {

__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {  // splitmix64 finalizer
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

// One thread per agent: the stance schedule (node_schedule, the same FP64 code the solve's setup
// runs) as the hash key; the first agent to claim a key's slot becomes its representative and
// draws the schedule id.  Agents with a non-finite input are left unshared (their own setup
// reports the failure, as the reference's build_qp does).
__global__ void sched_key_kernel(const KParams P, RmpcSchedBuffers b) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= P.n_agents) return;
  const rmpc_state st = P.states[a];
  const rmpc_command cmd = P.cmds[a];
  const rmpc_gait g = P.gaits[a];
  bool fin = isfinite(cmd.height) && isfinite(cmd.vx) && isfinite(cmd.wpitch) && isfinite(g.phase) &&
             isfinite(g.period) && isfinite(g.phase_switch);
#pragma unroll
  for (int k = 0; k < 9; ++k) fin = fin && isfinite(st.q[k]) && isfinite(st.qd[k]);
#pragma unroll
  for (int c = 0; c < 4; ++c) fin = fin && isfinite(g.offsets[c]);
  if (!fin) {
    b.slot_of[a] = -1;
    return;
  }
  unsigned long long k0 = 0, k1 = 0;  // 4 bits per node, nodes 0..15 and 16..31
  for (int i = 0; i < P.NT; ++i) {
    double sw[4];
    const unsigned long long bits = node_schedule(P, g, i, sw);
    if (i < 16) k0 |= bits << (4 * i); else k1 |= bits << (4 * (i - 16));
  }
  unsigned long long h = mix64(k0 ^ mix64(k1 + 0x9e3779b97f4a7c15ull));
  if (h == ~0ull) h = ~0ull - 1;
  unsigned int slot = (unsigned int)h & (unsigned int)(b.slots - 1);
  for (;;) {
    const unsigned long long prev = atomicCAS(b.table + slot, ~0ull, h);
    if (prev == ~0ull) {
      const int id = atomicAdd(b.n_sched, 1);
      b.slot_id[slot] = id < b.cap ? id : -1;
      if (id < b.cap) b.rep_list[id] = a;
      break;
    }
    if (prev == h) break;
    slot = (slot + 1) & (unsigned int)(b.slots - 1);
  }
  b.slot_of[a] = (int)slot;
}

}  // namespace rmpc_dev

int rmpc_launch_sched(const rmpc_dev::KParams& params, const RmpcSchedBuffers& b, void* stream,
                      rmpc_dev::KParams* params_out) {
  *params_out = params;
  if (params.n_agents <= 0 || params.n_agents > b.agents) return 0;
  const cudaStream_t st = (cudaStream_t)stream;
  int rc = (int)cudaMemsetAsync(b.table, 0xFF, (size_t)b.slots * sizeof(unsigned long long), st);
  if (rc == 0) rc = (int)cudaMemsetAsync(b.n_sched, 0, sizeof(int32_t), st);
  if (rc != 0) return rc;
  rmpc_dev::sched_key_kernel<<<(params.n_agents + 255) / 256, 256, 0, st>>>(params, b);
  rc = (int)cudaGetLastError();
  if (rc != 0) return rc;
  const rmpc_dev::CtaShape c = rmpc_dev::cta_shape(params.NT);
  rmpc_dev::KParams F = params;
  F.mode = 1;
  F.rep_list = b.rep_list;
  F.n_sched = b.n_sched;
  F.store = b.store;
  F.store_cap = b.cap;
  F.store_stride = rmpc_dev::store_layout(params.NT).total;
  F.slot_of = nullptr;
  F.out = nullptr;
  F.z_out = nullptr;
  F.act_out = nullptr;
  F.profile = 0;
  F.agents_per_cta = c.agents;
  F.spill_nodes = c.spill_nodes;
  F.tmem_cols = c.tmem_cols;
  const int grid = (b.cap + c.agents - 1) / c.agents;
  F.full_ctas = grid;
  F.tail_agents = 0;
  rc = launch_variant(F, c, grid, st);
  if (rc != 0) return rc;
  rmpc_dev::KParams& P = *params_out;
  P.mode = 0;
  P.slot_of = b.slot_of;
  P.slot_id = b.slot_id;
  P.store = b.store;
  P.store_cap = b.cap;
  P.store_stride = F.store_stride;
  return 0;
}
