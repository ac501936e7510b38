// rmpc_setup.cuh — stage f_KKT: build_qp (mpc.cpp:64-238) into the padded per-node layout, FP64, split over the warp pair.
// Part of the fused solve kernel: included once, in order, by rmpc_kernel.cu.
#pragma once

#include "rmpc_device.cuh"
#include "rmpc_kin.cuh"

namespace rmpc_dev {

#ifndef FULL
#define FULL 0xffffffffu
#endif

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

}  // namespace rmpc_dev
