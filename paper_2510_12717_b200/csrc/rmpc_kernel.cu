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
#include "rmpc_squad.cuh"
#include "rmpc_squad4.cuh"

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

// Residuals and objective on the unscaled problem (qp.cpp:192-200), z* = guess + dz and the
// inverse dynamics at node 0 (mpc.cpp:305-330), the active set (optional), the record.
__device__ __forceinline__ void finish_agent(const KParams& P, const Sm& sm, int agent, int lane, int warp,
                                             rmpc_solution& out, const rmpc_state& st, const rmpc_command& cmd,
                                             bool warm, const float* pz, long long& t0) {
  const int NT = P.NT;
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
  for (int k = tid; k < NT * NV; k += 64) {
    st[SL.e + k] = sm.V(k / NV, V_E)[k % NV];
    st[SL.qh + k] = sm.V(k / NV, V_QH)[k % NV];
  }
  float2* rw = reinterpret_cast<float2*>(st + SL.rows);
  for (int r = tid; r < (NT + 1) * NSLOT; r += 64) rw[r] = make_float2(sm.row[r].x, sm.row[r].y);
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

// One agent on one warp pair of the CTA: its shared-memory block at `base`, its TMEM node
// blocks at `tm`, named barrier `bar`.  `sched` is the schedule id the pair builds in mode 1.
__device__ __forceinline__ Sm make_sm(const KParams& P, float* base, uint32_t tm, int tmn, int bar, int warp,
                                      bool spills) {
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
  sm.spills = spills;
  sm.spill = base + L.spill + warp * P.spill_nodes * SPILL_BLK;
  sm.bar = bar;
  return sm;
}

// One agent per CTA (the schedule store's representative, or a per-agent batch of at most one
// agent per SM): warps 2.. of the CTA help the agent's warp pair with the Ruiz passes -- the only
// stage whose work splits by node without changing a single operation (ruiz(): nodes are
// independent within a pass), so the results are bit-identical.  `go` is set by the pair.
__device__ __forceinline__ void ruiz_helper(const KParams& P, float* base, int lane, int w, const int* go) {
  const int nw = (int)(blockDim.x >> 5);
  asm volatile("bar.sync %0, %1;" ::"r"(RUIZ_BAR), "r"((int)blockDim.x) : "memory");  // the pair's setup is done
  if (*go == 0) return;
  const Sm sm = make_sm(P, base, 0u, 0, 1, 0, false);
  ruiz(P, sm, lane, w, nw, (int)blockDim.x);
}

template <bool SPILL>
__device__ __forceinline__ void solve_agent(const KParams& P, float* base, uint32_t tm, int tmn, int bar,
                                            int agent, int sched, int lane, int warp, int* go = nullptr) {
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

  rmpc_state st;
  rmpc_command cmd;
  if (P.mode == 1 && P.synth_rep) {  // the schedule alone matters: the nominal pose at rest
#pragma unroll
    for (int k = 0; k < RMPC_NQ; ++k) {
      st.q[k] = P.nominal[k];
      st.qd[k] = 0.0;
    }
    cmd.height = cmd.vx = cmd.wpitch = 0.0;
  } else {
    st = P.states[agent];
    cmd = P.cmds[agent];
  }
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
  const int nw_cta = (int)(blockDim.x >> 5);
  const bool helped = nw_cta > 2 && go != nullptr;
  if (helped) {  // hand the setup to the helper warps for the Ruiz passes
    if (tid == 0) *go = ok && P.ruiz_iters > 0;
    asm volatile("bar.sync %0, %1;" ::"r"(RUIZ_BAR), "r"((int)blockDim.x) : "memory");
  }
  if (P.mode == 1 && !ok) {  // cannot happen for a representative (finite inputs); unshared
    if (tid == 0) reinterpret_cast<int32_t*>(P.store + (size_t)sched * P.store_stride + store_layout(NT).flags)[NT] = -1;
    return;
  }
  if (!ok) {
    out.status = RMPC_STATUS_NONFINITE_INPUT;
  } else {
    if (P.ruiz_iters > 0) ruiz(P, sm, lane, warp, helped ? nw_cta : 2, helped ? (int)blockDim.x : 64);
    apply_scaling(P, sm, lane, warp);
    prof_mark(P, tid, 3, t0);
    const int good = factorize(P, sm, lane, warp);
    if (P.mode == 1) {
      dump_schedule(P, sm, P.store + (size_t)sched * P.store_stride, lane, warp, good ? 1 : 0);
      return;
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
  finish_agent(P, sm, agent, lane, warp, out, st, cmd, warm, pz, t0);
}

// CTA = P.agents_per_cta warp pairs.  Warp w uses TMEM lanes [32 (w % 4), +32) (the quarter
// tcgen05.ld/st of warp w can reach) and columns [(w / 4) tmn 32, +tmn 32), tmn = the node
// blocks its quarter's share holds (tm_nodes); further blocks go to its shared-memory spill.
template <bool SPILL, int MAXA>
__global__ void __launch_bounds__(64 * MAXA, 1) rti_kernel(const KParams P) {
  extern __shared__ __align__(16) float smem[];
  __shared__ uint32_t tmem_base;
  __shared__ int s_go;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = w >> 1;
  const int b = blockIdx.x;
  int agent, sched = -1;
  if (P.mode == 1) {  // schedule store: one schedule per CTA, built by pair 0 (the other pairs
                      // help with its Ruiz passes: ruiz_helper)
    const int ns = min(*P.n_sched, P.store_cap);
    if (b >= ns) return;  // whole CTA idle
    sched = b;
    agent = pair == 0 ? P.rep_list[sched] : -1;
  } else if (P.agent_list != nullptr) {  // an agent list (unshared agents of a shared solve)
    const int nl = *P.n_list;
    if (b * P.agents_per_cta >= nl) return;
    const int idx = b * P.agents_per_cta + pair;
    agent = idx < nl ? P.agent_list[idx] : P.n_agents;
  } else {
    agent = b < P.full_ctas ? b * P.agents_per_cta + pair
                            : (pair < P.tail_agents ? P.full_ctas * P.agents_per_cta +
                                                           (b - P.full_ctas) * P.tail_agents + pair
                                                     : P.n_agents);
  }
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
  // one agent per CTA (the schedule store; a per-agent batch of at most one agent per SM): the
  // other pairs run the agent's Ruiz passes with it
  const bool helpers = P.mode == 1 || (P.agent_list == nullptr && P.full_ctas == 0 && P.tail_agents == 1);
  if (helpers && pair > 0) {
    ruiz_helper(P, smem, lane, w, &s_go);
  } else if (agent < P.n_agents) {
    const int tmn = tm_nodes(P.NT, P.agents_per_cta, w & 3);
    const uint32_t tm = tb + ((uint32_t)(32 * (w & 3)) << 16) + (uint32_t)((w >> 2) * tmn * TCOLS);
    float* base = smem + pair * make_layout(P.NT, P.spill_nodes).total;
    // (one straight-line call: a loop around the inlined solve -- e.g. a looping wave over the
    // agent list -- doubles the ADMM loop's spills, measured 2x slower)
    solve_agent<SPILL>(P, base, tm, tmn, 1 + pair, agent, sched, lane, w & 1, helpers ? &s_go : nullptr);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (w == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(P.tmem_cols) : "memory");
}

// ------------------------------------------------------------------------- shared schedule
// One agent of a shared-schedule CTA: the coefficient blocks, d, the flags and the factor are
// the CTA's (one copy for every pair); this agent brings its own bounds -- the schedule's
// scaled rows with its initial-state and swing-height rows replaced -- and q^, computed in
// FP64 by exactly the operations setup_nodes / setup_dynamics / apply_scaling use, so the
// solve is bit-identical to the agent's own factorization.  An agent whose stance flags differ
// from the group's (a 64-bit hash collision) is handed to rti_kernel's list instead.
__device__ __forceinline__ void solve_agent_shared(const KParams& P, float* cta, float* base, const float* entry,
                                                const double* con_pz, uint32_t tm, int bar, int agent, int lane,
                                                int warp) {
  const int NT = P.NT;
  const LayoutShared L = make_layout_shared(NT);
  const StoreLayout SL = store_layout(NT);
  Sm sm;
  sm.scr = base + L.scr;
  sm.coef = cta + L.coef;
  sm.vec = base + L.vec;
  sm.row = reinterpret_cast<float4*>(base + L.row);
  sm.tt = base + L.tt;
  sm.dsc = cta + L.d;
  sm.bc = base + L.bc;
  sm.flags = reinterpret_cast<uint32_t*>(cta + L.flags);
  sm.NT = NT;
  sm.mid = mid_node(NT);
  sm.tm = tm;
  sm.tmn = nodes_per_warp(NT);
  sm.spills = false;
  sm.spill = nullptr;
  sm.bar = bar;
  const int tid = warp * 32 + lane;
  long long t0 = P.profile ? clock64() : 0;

  // the schedule's scaled bounds, zero z / t / vectors, e
  const float2* er = reinterpret_cast<const float2*>(entry + SL.rows);
  for (int r = tid; r < (NT + 1) * NSLOT; r += 64) {
    const float2 lh = er[r];
    sm.row[r] = make_float4(lh.x, lh.y, 0.f, 0.f);
    sm.tt[r] = 0.f;
  }
  for (int k = tid; k < NT * V_NUM * V_STRIDE; k += 64) sm.vec[k] = 0.f;
  pair_sync(sm);
  for (int k = tid; k < NT * NV; k += 64) sm.V(k / NV, V_E)[k % NV] = entry[SL.e + k];
  sm.bc[tid] = 0.f;
  const rmpc_state st = P.states[agent];
  const rmpc_command cmd = P.cmds[agent];
  const rmpc_gait gait = P.gaits[agent];
  rmpc_solution out;
  {
    float* o = reinterpret_cast<float*>(&out);
    for (int k = 0; k < 33; ++k) o[k] = 0.f;
    out.status = RMPC_STATUS_OK;
    out.fail_iter = -1;
  }
  prof_mark(P, tid, 0, t0);
  pair_sync(sm);
  bool same = true;
  if (warp == 0) {
    // initial-state rows (setup_nodes, mpc.cpp:126-136): guess = nominal at the measured x
    if (lane < NQ) {
      const int k = lane;
      const double gq = k == 0 ? st.q[0] : P.nominal[k];
      const double rq = st.q[k] - gq, rqd = st.qd[k] - 0.0;
      float4* ri = sm.R(-1) + INIT0;
      const float* di = sm.D(-1) + INIT0;
      const float a = bound_f(rq) * di[k], c = bound_f(rqd) * di[9 + k];
      ri[k] = make_float4(a, a, 0.f, 0.f);
      ri[9 + k] = make_float4(c, c, 0.f, 0.f);
    }
    // swing-height rows (mpc.cpp:210-216) of nodes >= 1
#pragma unroll 1
    for (int i = lane; i < NT; i += 32) {
      double swt[4];
      const uint32_t bits = node_schedule(P, gait, i, swt);
      same = same && bits == sm.flags[i];
      if (i > 0) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if ((bits >> c) & 1u) continue;
          const double h = bezier_height(swt[c], P.z_swing, P.v_to, P.v_td);
          const double r = h - con_pz[c];
          const float v = bound_f(r) * sm.D(i)[14 + 4 * c];
          sm.R(i)[14 + 4 * c] = make_float4(v, v, 0.f, 0.f);
        }
      }
    }
  } else {
    // q^ = e w dt (guess - desired) (setup_dynamics, mpc.cpp:81-103, then apply_scaling)
#pragma unroll 1
    for (int i = lane; i < NT; i += 32) {
      double swt[4];
      const uint32_t bits = node_schedule(P, gait, i, swt);
      float* qh = sm.V(i, V_QH);
      const float* ei = sm.V(i, V_E);
#pragma unroll 1
      for (int j = 0; j < NV; ++j) {
        double g, des;
        guess_and_target(P, i, j, false, nullptr, st, cmd, bits, g, des);
        qh[j] = to_f(wcost(P, j) * P.dt[i] * (g - des)) * ei[j];
      }
    }
  }
  same = __all_sync(FULL, same);
  if (!pair_and(sm, same)) {  // not this CTA's schedule: solve it in rti_kernel's list
    if (tid == 0) P.list_out[atomicAdd(P.n_list, 1)] = agent;
    return;
  }
  prof_mark(P, tid, 2, t0);  // (Ruiz and the factorization ran once per schedule, unprofiled)
  const int status = reinterpret_cast<const int32_t*>(entry + SL.flags)[NT];
  if (status != 1) {
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
  finish_agent(P, sm, agent, lane, warp, out, st, cmd, false, nullptr, t0);
}

// CTA = up to agents_per_cta agents of one schedule group (grp_cta / grp_first / order).  The
// CTA loads the group's store entry once: coefficients, d and flags into shared memory, the
// factor's node blocks into TMEM -- top half (nodes 0..m) in lane quarters 0 and 2, bottom half
// in 1 and 3, the quarters of the pairs' even and odd warps -- then every pair solves its agent.
template <int MAXA>
__global__ void __launch_bounds__(64 * MAXA, 1) rti_shared_kernel(const KParams P) {
  extern __shared__ __align__(16) float smem[];
  __shared__ uint32_t tmem_base;
  __shared__ int s_g, s_first, s_cnt;
  __shared__ double s_con[4];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int NT = P.NT;
  if (tid == 0) {
    const int ng = min(*P.n_sched, P.store_cap);
    int g = -1, first = 0, cnt = 0;
    if (ng > 0 && (int)blockIdx.x < P.grp_cta[ng]) {
      int lo = 0, hi = ng - 1;  // last group whose first CTA is <= blockIdx.x
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (P.grp_cta[mid] <= (int)blockIdx.x) lo = mid; else hi = mid - 1;
      }
      g = lo;
      const int k = (int)blockIdx.x - P.grp_cta[g];
      first = P.grp_first[g] + k * P.agents_per_cta;
      cnt = min(P.agents_per_cta, P.grp_count[g] - k * P.agents_per_cta);
    }
    s_g = g;
    s_first = first;
    s_cnt = cnt;
  }
  __syncthreads();
  if (s_cnt <= 0) return;  // whole CTA idle
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tmem_base)),
                 "r"(P.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  const LayoutShared L = make_layout_shared(NT);
  const StoreLayout SL = store_layout(NT);
  const float* entry = P.store + (size_t)s_g * P.store_stride;
  {  // the CTA region: coefficients, d, flags
    const float4* c4 = reinterpret_cast<const float4*>(entry + SL.coef);
    float4* s4 = reinterpret_cast<float4*>(smem + L.coef);
    for (int k = tid; k < (NT + 1) * C_SIZE / 4; k += blockDim.x) s4[k] = c4[k];
    const float4* d4 = reinterpret_cast<const float4*>(entry + SL.d);
    float4* sd = reinterpret_cast<float4*>(smem + L.d);
    for (int k = tid; k < (NT + 1) * NSLOT / 4; k += blockDim.x) sd[k] = d4[k];
    const int32_t* fl = reinterpret_cast<const int32_t*>(entry + SL.flags);
    for (int k = tid; k < NT; k += blockDim.x) reinterpret_cast<int32_t*>(smem + L.flags)[k] = fl[k];
  }
  if (tid < 4) s_con[tid] = P.con_pz[tid];  // contact heights of the nominal pose (sched_key_kernel)
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = tmem_base;
  if (w < 4) {  // warp w fills lane quarter w with its half of the factor
    const uint32_t tq = tb + ((uint32_t)(32 * w) << 16);
    const int m = mid_node(NT);
    const bool top = (w & 1) == 0;
    for (int i = top ? 0 : m + 1; i <= (top ? m : NT - 1); ++i) {
      const int blk = top ? i : i - m - 1;
      const float4* r = reinterpret_cast<const float4*>(entry + SL.blocks + (size_t)(i * 32 + lane) * TCOLS);
      float v[TCOLS];
#pragma unroll
      for (int q = 0; q < TCOLS / 4; ++q) {
        const float4 x = r[q];
        v[4 * q] = x.x; v[4 * q + 1] = x.y; v[4 * q + 2] = x.z; v[4 * q + 3] = x.w;
      }
      tm_store(tq + (uint32_t)(TCOLS * blk), v);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int pair = w >> 1;
  if (pair < s_cnt) {
    const int agent = P.order[s_first + pair];
    const uint32_t tm = tb + ((uint32_t)(32 * (w & 3)) << 16);
    solve_agent_shared(P, smem, smem + L.cta_total + pair * L.total, entry, s_con, tm, 1 + pair, agent, lane, w & 1);
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
  if (rc == 0) rc = (int)cudaFuncSetAttribute(rmpc_dev::rti_shared_kernel<rmpc_dev::SHARED_AGENTS>, a, bytes);
  if (rc == 0) rc = (int)cudaFuncSetAttribute(rmpc_dev::rti_shared_kernel<rmpc_dev::MAX_AGENTS>, a, bytes);
  if (rc == 0) rc = (int)cudaFuncSetAttribute(rmpc_dev::rti_squad_kernel, a, bytes);
  if (rc == 0) rc = (int)cudaFuncSetAttribute(rmpc_dev::rti_squad4_kernel, a, bytes);
  return rc;
}

// Kernels of the solve path launched by this process (rmpc_kernel_launches): the bench's
// gpu_launches is the difference over its timed region.
static std::atomic<long long> g_launches{0};

// SM count of the current device, cached (several host threads, one per shard, may launch at once)
static int sm_count() {
  static std::atomic<int> sms[64];
  int dev = 0;
  cudaGetDevice(&dev);
  int nsm = dev < 64 ? sms[dev].load(std::memory_order_relaxed) : 0;
  if (nsm == 0) {
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (nsm <= 0) nsm = 148;
    if (dev < 64) sms[dev].store(nsm, std::memory_order_relaxed);
  }
  return nsm;
}

namespace rmpc_dev {
// The per-agent list of a shared solve (over-capacity schedules, non-finite inputs, schedule
// hash collisions found by the squads) is known only on the device: this one-thread kernel reads
// its length and tail-launches rti_kernel over exactly ceil(n_list / A) CTAs (none when the list
// is empty -- an upper-bound grid of idle CTAs cost ~12 us per tick).  The tail launch runs after
// this grid and before anything later in the stream.
__global__ void list_dispatch_kernel(const KParams U, int variant, int threads, int smem) {
  const int nl = *U.n_list;
  if (nl <= 0) return;
  const int grid = (nl + U.agents_per_cta - 1) / U.agents_per_cta;
  if (variant == 0) rti_kernel<false, DENSE_AGENTS><<<grid, threads, smem, cudaStreamTailLaunch>>>(U);
  else if (variant == 1) rti_kernel<true, MAX_AGENTS><<<grid, threads, smem, cudaStreamTailLaunch>>>(U);
  else rti_kernel<false, MAX_AGENTS><<<grid, threads, smem, cudaStreamTailLaunch>>>(U);
}
}  // namespace rmpc_dev

static int launch_variant(const rmpc_dev::KParams& P, const rmpc_dev::CtaShape& c, int grid, cudaStream_t st,
                          int threads = 0) {
  if (grid <= 0) return 0;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  const int nt = threads > 0 ? threads : 64 * c.agents;
  if (c.dense)
    rmpc_dev::rti_kernel<false, rmpc_dev::DENSE_AGENTS><<<grid, nt, c.smem_bytes, st>>>(P);
  else if (c.spill_nodes > 0)
    rmpc_dev::rti_kernel<true, rmpc_dev::MAX_AGENTS><<<grid, nt, c.smem_bytes, st>>>(P);
  else
    rmpc_dev::rti_kernel<false, rmpc_dev::MAX_AGENTS><<<grid, nt, c.smem_bytes, st>>>(P);
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
  const int nsm = sm_count();
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
__device__ __forceinline__ bool state_cmd_finite(const rmpc_state& st, const rmpc_command& cmd) {
  bool fin = isfinite(cmd.height) && isfinite(cmd.vx) && isfinite(cmd.wpitch);
#pragma unroll
  for (int k = 0; k < 9; ++k) fin = fin && isfinite(st.q[k]) && isfinite(st.qd[k]);
  return fin;
}

// The schedule pass's state for a new tick in one launch (instead of four memsets): the hash
// table empty, the counters and group sizes zero.
__global__ void __launch_bounds__(256) sched_init_kernel(RmpcSchedBuffers b) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (int k = t; k < b.slots; k += nt) b.table[k] = ~0ull;
  for (int k = t; k < b.cap; k += nt) b.cnt[k] = 0;
  if (t == 0) {
    *b.n_sched = 0;
    *b.n_unshared = 0;
  }
}

__global__ void sched_key_kernel(const KParams P, RmpcSchedBuffers b) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a == 0) {  // contact heights of the nominal pose (the cold guess of every node), once for
                 // every group CTA of the solve
    double gq[9], gqd[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      gq[k] = P.nominal[k];
      gqd[k] = 0.0;
    }
    Frames F;
    fk_frames(P, gq, gqd, F);
#pragma unroll
    for (int c = 0; c < 4; ++c) b.con[c] = F.con[c].pz;
  }
  if (a >= P.n_agents) return;
  const rmpc_gait g = P.gaits[a];
  bool fin = isfinite(g.phase) && isfinite(g.period) && isfinite(g.phase_switch);
  if (!P.synth_rep) fin = fin && state_cmd_finite(P.states[a], P.cmds[a]);  // (else: the count kernel)
#pragma unroll
  for (int c = 0; c < 4; ++c) fin = fin && isfinite(g.offsets[c]);
  if (!fin) {
    b.slot_of[a] = -1;
    return;
  }
  unsigned long long k0 = 0, k1 = 0;  // 4 bits per node, nodes 0..15 and 16..31
  double shift = 0.0;  // node_schedule's cumulative shift, the same additions in the same order
  for (int i = 0; i < P.NT; ++i) {
    unsigned long long bits = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (wrap01(g.phase + shift + g.offsets[c]) < g.phase_switch) bits |= 1ull << c;
    if (i < 16) k0 |= bits << (4 * i); else k1 |= bits << (4 * (i - 16));
    shift += P.dt[i] / g.period;
  }
  unsigned long long h = mix64(k0 ^ mix64(k1 + 0x9e3779b97f4a7c15ull));
  if (h == ~0ull) h = ~0ull - 1;
  // one insert per distinct key of the warp (thousands of agents share a handful of schedules:
  // a CAS per agent serialises on a few table slots), and a plain read before the CAS
  const unsigned act = __activemask();
  const unsigned peers = __match_any_sync(act, h);
  const int leader = __ffs(peers) - 1;
  unsigned int slot = (unsigned int)h & (unsigned int)(b.slots - 1);
  if ((threadIdx.x & 31) == leader) {
    for (;;) {
      unsigned long long prev = *(volatile unsigned long long*)(b.table + slot);
      if (prev == ~0ull) prev = atomicCAS(b.table + slot, ~0ull, h);
      if (prev == ~0ull) {
        const int id = atomicAdd(b.n_sched, 1);
        b.slot_id[slot] = id < b.cap ? id : -1;
        if (id < b.cap) b.rep_list[id] = a;
        break;
      }
      if (prev == h) break;
      slot = (slot + 1) & (unsigned int)(b.slots - 1);
    }
  }
  slot = __shfl_sync(peers, slot, leader);
  b.slot_of[a] = (int)slot;
}

// One thread per agent: its group position (atomic per schedule id; the order inside a group
// does not matter, every agent's result is independent of it) or the unshared list.
__global__ void sched_count_kernel(const KParams P, RmpcSchedBuffers b) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= P.n_agents) return;
  const int sl = b.slot_of[a];
  int id = sl >= 0 ? b.slot_id[sl] : -1;
  if (id >= 0 && P.synth_rep && !state_cmd_finite(P.states[a], P.cmds[a])) id = -1;  // its own solve fails it
  if (id >= 0) {  // warp-aggregated: one atomic per schedule id of the warp
    const unsigned peers = __match_any_sync(__activemask(), id);
    const int leader = __ffs(peers) - 1, lane = threadIdx.x & 31;
    int base = 0;
    if (lane == leader) base = atomicAdd(b.cnt + id, __popc(peers));
    base = __shfl_sync(peers, base, leader);
    b.pos[a] = base + __popc(peers & ((1u << lane) - 1u));
  } else {
    b.pos[a] = -1;
    b.ulist[atomicAdd(b.n_unshared, 1)] = a;
  }
}

// One CTA of 1024 threads (cap <= 1024 groups): exclusive prefix sums of the group sizes and of
// their CTA counts (ceil(count / A)).
__global__ void sched_scan_kernel(RmpcSchedBuffers b, int A) {
  __shared__ int wsum[2][32];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int ng = min(*b.n_sched, b.cap);
  const int c = t < ng ? b.cnt[t] : 0;
  int v0 = c, v1 = (c + A - 1) / A;  // agents, CTAs
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y0 = __shfl_up_sync(FULL, v0, o), y1 = __shfl_up_sync(FULL, v1, o);
    if (lane >= o) { v0 += y0; v1 += y1; }
  }
  if (lane == 31) { wsum[0][wid] = v0; wsum[1][wid] = v1; }
  __syncthreads();
  if (wid == 0) {
    int s0 = wsum[0][lane], s1 = wsum[1][lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y0 = __shfl_up_sync(FULL, s0, o), y1 = __shfl_up_sync(FULL, s1, o);
      if (lane >= o) { s0 += y0; s1 += y1; }
    }
    wsum[0][lane] = s0;
    wsum[1][lane] = s1;
  }
  __syncthreads();
  const int base0 = wid > 0 ? wsum[0][wid - 1] : 0, base1 = wid > 0 ? wsum[1][wid - 1] : 0;
  const int incl0 = v0 + base0, incl1 = v1 + base1;
  if (t < ng) {
    b.grp_first[t] = incl0 - c;
    b.grp_cta[t] = incl1 - (c + A - 1) / A;
  }
  if (t == (ng > 0 ? ng - 1 : 0)) b.grp_cta[ng] = ng > 0 ? incl1 : 0;
}

__global__ void sched_scatter_kernel(const KParams P, RmpcSchedBuffers b) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= P.n_agents) return;
  const int p = b.pos[a];
  if (p >= 0) b.order[b.grp_first[b.slot_id[b.slot_of[a]]] + p] = a;
}

}  // namespace rmpc_dev

int rmpc_launch_shared(const rmpc_dev::KParams& params_in, const RmpcSchedBuffers& b, void* stream, int variant,
                       const RmpcCopyOut* co, void* ev_inputs) {
  using namespace rmpc_dev;
  if (params_in.n_agents <= 0) return 0;
  if (params_in.n_agents > b.agents) return (int)cudaErrorInvalidValue;
  const cudaStream_t st = (cudaStream_t)stream;
  const int n = params_in.n_agents, NT = params_in.NT;
  const int blocks = (n + 255) / 256;
  // squads: two per CTA for T <= 10 (rmpc_squad.cuh), one long squad of four warps per CTA for
  // T = 11..20 (rmpc_squad4.cuh)
  const bool long_sq = variant == 2 && sq4_supported(NT) && b.sqpack != nullptr;
  const bool squads = (variant == 2 && sq_supported(NT) && b.sqpack != nullptr) || long_sq;
  const int spc = long_sq ? 1 : 2;  // squads per CTA
  static const int synth_env = [] {  // RMPC_SYNTH_REP=0: build the store from the representative's own state
    const char* e = getenv("RMPC_SYNTH_REP");
    return e ? atoi(e) : 1;
  }();
  KParams params = params_in;
  params.synth_rep = squads && synth_env != 0;
  if (!params.synth_rep && ev_inputs)  // the whole pass reads the states: wait for them here
    cudaStreamWaitEvent(st, (cudaEvent_t)ev_inputs, 0);
  static const int solo = [] {  // debugging: one squad per CTA (RMPC_SQUAD_SOLO=1: slot 0, 2: slot 1)
    const char* e = getenv("RMPC_SQUAD_SOLO");
    return e ? atoi(e) : 0;
  }();
  // host outputs: a split pays only where a second wave of squad CTAs follows the first; else
  // the solve writes the mapped host buffers itself
  if (co && !(squads && !solo && (n + 31) / 32 + std::min(b.cap, n) > spc * co->sms)) {
    KParams Q = params_in;
    Q.out = co->h_out;
    Q.z_out = co->h_z;
    return rmpc_launch_shared(Q, b, stream, variant, nullptr, params.synth_rep ? ev_inputs : nullptr);
  }
  sched_init_kernel<<<64, 256, 0, st>>>(b);
  sched_key_kernel<<<blocks, 256, 0, st>>>(params, b);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  int rc = 0;
  // fork: the grouping pass (count, scan, scatter) needs only the keys; it runs on the side
  // stream while the store build (which needs only the representatives) runs here
  const cudaStream_t side = b.side ? (cudaStream_t)b.side : st;
  if (side != st) {
    cudaEventRecord((cudaEvent_t)b.ev_fork, st);
    cudaStreamWaitEvent(side, (cudaEvent_t)b.ev_fork, 0);
  }
  // host outputs: the schedule count to the host (side stream), so the squad launch below knows
  // whether a second wave follows the first
  const bool ask_nsched = co != nullptr && b.h_nsched != nullptr && b.ev_nsched != nullptr && side != st;
  if (ask_nsched) {
    cudaMemcpyAsync(b.h_nsched, b.n_sched, sizeof(int32_t), cudaMemcpyDeviceToHost, side);
    cudaEventRecord((cudaEvent_t)b.ev_nsched, side);
  }
  if (params.synth_rep && ev_inputs)  // the count kernel is the first to read the states
    cudaStreamWaitEvent(side, (cudaEvent_t)ev_inputs, 0);
  sched_count_kernel<<<blocks, 256, 0, side>>>(params, b);
  g_launches.fetch_add(2, std::memory_order_relaxed);
  // the store: setup + Ruiz + factorization of each schedule's representative (mode 1), one
  // warp pair per CTA (the few schedules' latency chains run alone on their SMs)
  const CtaShape c = cta_shape(NT);
  CtaShape c1 = c;
  c1.agents = 1;
  c1.spill_nodes = 0;
  c1.dense = false;
  c1.tmem_cols = 32;
  while (c1.tmem_cols < nodes_per_warp(NT) * TCOLS) c1.tmem_cols *= 2;
  c1.smem_bytes = smem_bytes(NT, 0);
  KParams F = params;
  F.mode = 1;
  F.rep_list = b.rep_list;
  F.n_sched = b.n_sched;
  F.store = b.store;
  F.store_cap = b.cap;
  F.store_stride = store_layout(NT).total;
  F.out = nullptr;
  F.z_out = nullptr;
  F.act_out = nullptr;
  F.profile = 0;
  F.agents_per_cta = 1;
  F.spill_nodes = 0;
  F.tmem_cols = c1.tmem_cols;
  F.full_ctas = b.cap;
  F.tail_agents = 0;
  // one CTA per schedule: the representative's warp pair plus helper warps for its Ruiz passes
  rc = launch_variant(F, c1, F.full_ctas, st, 64 * MAX_AGENTS);
  if (rc != 0) return rc;
  const CtaShapeShared cs = cta_shape_shared(NT, shared_agents_cap(NT));
  // the groups: one schedule per CTA (grid: an upper bound of sum ceil(count / A))
  KParams S = params;
  S.mode = 0;
  S.n_sched = b.n_sched;
  S.store = b.store;
  S.store_cap = b.cap;
  S.store_stride = F.store_stride;
  S.order = b.order;
  S.grp_cta = b.grp_cta;
  S.grp_first = b.grp_first;
  S.grp_count = b.cnt;
  S.con_pz = b.con;
  S.n_list = b.n_unshared;
  S.list_out = b.ulist;
  S.agents_per_cta = cs.agents;
  S.tmem_cols = cs.tmem_cols;
  const int grid_s = (n + cs.agents - 1) / cs.agents + std::min(b.cap, n);
  bool single_wave = false;
  if (squads) {  // lane-per-agent squads, two per CTA (grid: an upper bound of sum ceil(count / 32) / 2)
    S.agents_per_cta = 32;
    S.sqpack = b.sqpack;
    sq_pack_kernel<<<dim3(b.cap, SQ_PACK_SLICES), 256, 0, st>>>(S);  // (needs only the store)
    g_launches.fetch_add(1, std::memory_order_relaxed);
  }
  sched_scan_kernel<<<1, 1024, 0, side>>>(b, squads ? 32 : cs.agents);
  sched_scatter_kernel<<<blocks, 256, 0, side>>>(params, b);
  if (side != st) {  // join before the group solve
    cudaEventRecord((cudaEvent_t)b.ev_join, side);
    cudaStreamWaitEvent(st, (cudaEvent_t)b.ev_join, 0);
  }
  g_launches.fetch_add(3, std::memory_order_relaxed);  // + the group kernel below
  if (squads) {
    const int nsq = (n + 31) / 32 + std::min(b.cap, n);
    S.pad2_ = solo;
    const int grid = (solo || long_sq) ? nsq : (nsq + 1) / 2;
    const int smem = long_sq ? sq4_smem_bytes(NT) : sq_smem_bytes(NT);
    auto launch_sq = [&](int g) {
      if (long_sq) rti_squad4_kernel<<<g, 128, smem, st>>>(S);
      else rti_squad_kernel<<<g, 128, smem, st>>>(S);
    };
    // host outputs with every squad in the first wave (known once the key kernel has counted the
    // schedules; the host waits for that ~10 us copy while the store build runs): one launch into
    // the device buffers, then copy-engine transfers of the whole contiguous outputs (56 vs 47
    // GB/s of SM-issued mapped writes) after the per-agent list
    if (co && ask_nsched && !solo) {
      cudaEventSynchronize((cudaEvent_t)b.ev_nsched);
      const int ns = std::min(std::max(*b.h_nsched, 0), b.cap);
      single_wave = (n + 31) / 32 + ns <= spc * co->sms;
    }
    if (co && !single_wave) {  // split: first wave, its copy-out beside the second launch
      S.sq_cta_base = 0;
      launch_sq(co->sms);
      cudaEventRecord((cudaEvent_t)co->ev_a, st);
      cudaStreamWaitEvent((cudaStream_t)co->stream2, (cudaEvent_t)co->ev_a, 0);
      sq_copyout_kernel<<<64, 256, 0, (cudaStream_t)co->stream2>>>(S, 0, co->sms, 0, co->h_out, co->h_z, spc);
      cudaEventRecord((cudaEvent_t)co->ev_b, (cudaStream_t)co->stream2);
      S.sq_cta_base = co->sms;  // the second launch writes the mapped host buffers itself: its
      S.out = co->h_out;        // CTAs are the last ones, nothing waits for their SMs
      S.z_out = co->h_z;
      launch_sq(grid - co->sms);
      g_launches.fetch_add(2, std::memory_order_relaxed);
    } else {
      launch_sq(grid);
    }
  } else if (cs.agents > MAX_AGENTS)
    rti_shared_kernel<SHARED_AGENTS><<<grid_s, 64 * cs.agents, cs.smem_bytes, st>>>(S);
  else
    rti_shared_kernel<MAX_AGENTS><<<grid_s, 64 * cs.agents, cs.smem_bytes, st>>>(S);
  rc = (int)cudaGetLastError();
  if (rc != 0) return rc;
  // the rest (over-capacity schedules, non-finite inputs, hash collisions): per-agent solves
  KParams U = params;
  U.mode = 0;
  U.agent_list = b.ulist;
  U.n_list = b.n_unshared;
  U.agents_per_cta = c.agents;
  U.spill_nodes = c.spill_nodes;
  U.tmem_cols = c.tmem_cols;
  U.full_ctas = (n + c.agents - 1) / c.agents;  // (the largest list)
  U.tail_agents = 0;
  if (co && !single_wave) {
    // the per-agent list writes the mapped host buffers too, after the first wave's copy-out: a
    // fallback agent of the first wave is in both, and its list record must land last
    cudaStreamWaitEvent(st, (cudaEvent_t)co->ev_b, 0);
    U.out = co->h_out;
    U.z_out = co->h_z;
  }
  list_dispatch_kernel<<<1, 1, 0, st>>>(U, c.dense ? 0 : (c.spill_nodes > 0 ? 1 : 2), 64 * c.agents, c.smem_bytes);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (single_wave) {  // every record and z* row is in the device buffers: two contiguous copies
    cudaMemcpyAsync(co->h_out, params.out, (size_t)n * sizeof(rmpc_solution), cudaMemcpyDefault, st);
    if (co->h_z && params.z_out)
      cudaMemcpyAsync(co->h_z, params.z_out, (size_t)n * NT * NV * sizeof(float), cudaMemcpyDefault, st);
  }
  return (int)cudaGetLastError();
}

namespace rmpc_dev {

// rmpc_solve_soa's unpack: thread a reads column a of the 28 component rows (each warp-wide row
// read is one coalesced 128-byte transaction) and writes agent a's FP64 records.  float -> double
// is exact, so the solve sees exactly the values the caller's FP32 block holds.
__global__ void __launch_bounds__(256) soa_unpack_kernel(const float* __restrict__ soa, long long ld, int n,
                                                         rmpc_state* states, rmpc_command* cmds, rmpc_gait* gaits,
                                                         int part) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= n) return;
  const float* c = soa + a;
  if (part != 1) {  // the state and command rows
    rmpc_state st;
#pragma unroll
    for (int k = 0; k < RMPC_NQ; ++k) {
      st.q[k] = (double)__ldg(c + (RMPC_SOA_Q + k) * ld);
      st.qd[k] = (double)__ldg(c + (RMPC_SOA_QD + k) * ld);
    }
    rmpc_command cm;
    cm.height = (double)__ldg(c + RMPC_SOA_HEIGHT * ld);
    cm.vx = (double)__ldg(c + RMPC_SOA_VX * ld);
    cm.wpitch = (double)__ldg(c + RMPC_SOA_WPITCH * ld);
    states[a] = st;
    cmds[a] = cm;
  }
  if (part != 2) {  // the gait rows
    rmpc_gait g;
    g.phase = (double)__ldg(c + RMPC_SOA_PHASE * ld);
    g.period = (double)__ldg(c + RMPC_SOA_PERIOD * ld);
    g.phase_switch = (double)__ldg(c + RMPC_SOA_PHASE_SWITCH * ld);
#pragma unroll
    for (int k = 0; k < RMPC_NC; ++k) g.offsets[k] = (double)__ldg(c + (RMPC_SOA_OFFSETS + k) * ld);
    gaits[a] = g;
  }
}

}  // namespace rmpc_dev

int rmpc_launch_soa_unpack(const float* soa, long long ld, int n, rmpc_state* states, rmpc_command* cmds,
                           rmpc_gait* gaits, void* stream, int part) {
  if (n <= 0) return 0;
  rmpc_dev::soa_unpack_kernel<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(soa, ld, n, states, cmds, gaits,
                                                                                  part);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return (int)cudaGetLastError();
}

extern "C" int64_t rmpc_kernel_launches(void) { return (int64_t)g_launches.load(std::memory_order_relaxed); }
