// rmpc_oracle.hpp — TEST INFRASTRUCTURE ONLY.
//
// Plain-C++ CPU restatement of the reference's batched RTI-MPC hot path
// (/root/reference/proj/src/{gait,robot,mpc,csc,ruiz,qp,ldl,batch}.cpp), used as the parity
// checker for the CUDA solver and as the CPU baseline in bench.py.  It is never linked
// into, imported by, or called from the product library (paper_2510_12717_b200/).
//
// Templated on the scalar type: double = parity oracle (the reference is FP64 throughout),
// float = FP32 sensitivity probe, Counted<double> = FLOP instrumentation (oracle_flops.hpp).
//
// Deviations from the reference, all rounding-level only:
//   * Eigen's AMDOrdering (ldl.cpp:14-35) is replaced by an exact minimum-degree ordering on
//     the same symmetric pattern (min_degree_ordering below).  Eigen is absent from this
//     image; the permutation changes only rounding, not the mathematics.  The exact AMD
//     permutation is therefore "parity unpinned".
//   * Eigen fixed-size products are written as explicit loops (same terms, possibly a
//     different summation order).
#pragma once

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../include/rmpc_b200.h"
#include "rmpc_oracle_ordering.hpp"

namespace oracle {

constexpr double kInf = 1e30;  // types.hpp:15
constexpr int kNq = 9, kNj = 6, kNc = 4, kNf = 8, kNv = 26;

struct StructuralError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct SingularityError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DivergenceError : std::runtime_error {
  DivergenceError(const std::string& w, int it) : std::runtime_error(w), iteration(it) {}
  int iteration;
};

// Stage attribution for the FLOP counter (MpcStage, mpc.hpp:79-88).
enum Stage { kInit = 0, kParam, kKkt, kRuiz, kFactor, kAdmm, kRnea, kNumStages };
inline thread_local int g_stage = kInit;

using std::abs;
using std::cos;
using std::sin;
using std::sqrt;

// ---------------------------------------------------------------- defaults
inline void model_default(rmpc_model* p) {  // robot.hpp:24-50
  std::memset(p, 0, sizeof(*p));
  p->torso_mass = 10.0; p->torso_len = 0.4; p->torso_inertia = 10.0 * 0.4 * 0.4 / 12.0;
  p->thigh_mass = 2.5; p->thigh_len = 0.4; p->thigh_inertia = 2.5 * 0.4 * 0.4 / 12.0;
  p->shank_mass = 1.5; p->shank_len = 0.4; p->shank_inertia = 1.5 * 0.4 * 0.4 / 12.0;
  p->foot_mass = 0.5; p->foot_half_len = 0.09; p->foot_inertia = 0.5 * 0.18 * 0.18 / 12.0;
  p->ankle_drop = 0.05;
  const double lo[6] = {-1.5, 0.05, -1.2, -1.5, 0.05, -1.2};
  const double hi[6] = {1.5, 2.4, 1.2, 1.5, 2.4, 1.2};
  const double tl[6] = {60.0, 60.0, 30.0, 60.0, 60.0, 30.0};
  for (int j = 0; j < 6; ++j) {
    p->joint_lo[j] = lo[j]; p->joint_hi[j] = hi[j];
    p->qd_limit[j] = 20.0; p->tau_limit[j] = tl[j];
    p->kp[j] = 30.0; p->kd[j] = 1.0;
  }
  p->mu = 0.8; p->gravity = 9.81;
  p->nominal_stagger = 0.15; p->nominal_drop = 0.75;
}

inline void settings_default(rmpc_settings* s, int horizon) {  // mpc.hpp:16-57, qp.hpp:29-36
  std::memset(s, 0, sizeof(*s));
  s->horizon = horizon;
  for (int i = 0; i < RMPC_MAX_HORIZON; ++i) s->dt_schedule[i] = i < horizon ? 0.05 : 0.0;
  const double wq[9] = {0.0, 500.0, 300.0, 5.0, 5.0, 5.0, 5.0, 5.0, 5.0};
  const double wqd[9] = {100.0, 100.0, 50.0, 0.1, 0.1, 0.1, 0.1, 0.1, 0.1};
  for (int k = 0; k < 9; ++k) { s->w_q[k] = wq[k]; s->w_qd[k] = wqd[k]; }
  for (int k = 0; k < 8; ++k) s->w_f[k] = 1e-3;
  s->gait_period = 0.8; s->phase_switch = 0.5;
  s->phase_offsets[0] = 0.5; s->phase_offsets[1] = 0.5;
  s->phase_offsets[2] = 0.0; s->phase_offsets[3] = 0.0;
  s->z_swing = 0.075; s->v_to = 0.2; s->v_td = -0.3;
  s->n_qp = 25; s->mu = 0.6; s->sigma = 1e-6; s->rho = 0.1; s->over_relax = 1.6;
  s->warm_start = 0; s->ruiz_iters = 10;
}

inline double total_mass(const rmpc_model& p) {
  return p.torso_mass + 2.0 * (p.thigh_mass + p.shank_mass + p.foot_mass);
}
inline double nominal_height(const rmpc_model& p) {
  return p.ankle_drop + p.nominal_drop + 0.5 * p.torso_len;
}

// ---------------------------------------------------------------- kinematics (robot.cpp)
// Link order torso, L thigh, L shank, L foot, R thigh, R shank, R foot; each link's CoM
// moves with the angle coordinates of its chain (robot.cpp:18-21).
constexpr int kChain[7][4] = {{2, -1, -1, -1}, {2, 3, -1, -1}, {2, 3, 4, -1}, {2, 3, 4, 5},
                              {2, 6, -1, -1},  {2, 6, 7, -1},  {2, 6, 7, 8}};

template <class T>
struct Pt {  // position and velocity of a point in the sagittal plane
  T px, pz, vx, vz;
};

template <class T>
struct Kin {
  Pt<T> com[7];
  T com_jac[7][2][kNq];
  T com_jdq[7][2];  // J-dot * qd of each CoM
  Pt<T> c[kNc];     // contact points
  T c_jac[kNc][2][kNq];
};

// Point rigidly attached to `from`, offset (x, z) in the frame rotated by `ang`, spinning at
// `w`: p = from + R(ang)(x,z), v = from.v + w * perp(R(ang)(x,z)), perp(a,b) = (-b, a).
template <class T>
inline Pt<T> attach(const Pt<T>& from, const T& ang, const T& w, const T& x, const T& z) {
  const T c = cos(ang), s = sin(ang);
  const T rx = c * x - s * z;
  const T rz = s * x + c * z;
  return {from.px + rx, from.pz + rz, from.vx - w * rz, from.vz + w * rx};
}

// robot.cpp:29-148
template <class T>
Kin<T> kinematics(const rmpc_model& p, const T* q, const T* qd) {
  Kin<T> k;
  const Pt<T> base{q[0], q[1], qd[0], qd[1]};
  const T th = q[2];
  const Pt<T> hip = attach(base, th, qd[2], T(0.0), T(-0.5 * p.torso_len));
  Pt<T> knee[2], ankle[2];
  T ang[2][3], om[2][3];
  for (int leg = 0; leg < 2; ++leg) {  // leg 0 = left (coords 3..5), 1 = right (6..8)
    const int h = 3 + 3 * leg;
    ang[leg][0] = th + q[h];
    ang[leg][1] = ang[leg][0] + q[h + 1];
    ang[leg][2] = ang[leg][1] + q[h + 2];
    om[leg][0] = qd[2] + qd[h];
    om[leg][1] = om[leg][0] + qd[h + 1];
    om[leg][2] = om[leg][1] + qd[h + 2];
    knee[leg] = attach(hip, ang[leg][0], om[leg][0], T(0.0), T(-p.thigh_len));
    ankle[leg] = attach(knee[leg], ang[leg][1], om[leg][1], T(0.0), T(-p.shank_len));
  }
  Pt<T> pivot[kNq];
  pivot[2] = base;
  pivot[3] = hip; pivot[4] = knee[0]; pivot[5] = ankle[0];
  pivot[6] = hip; pivot[7] = knee[1]; pivot[8] = ankle[1];

  k.com[0] = base;
  for (int leg = 0; leg < 2; ++leg) {
    k.com[1 + 3 * leg] = attach(hip, ang[leg][0], om[leg][0], T(0.0), T(-0.5 * p.thigh_len));
    k.com[2 + 3 * leg] =
        attach(knee[leg], ang[leg][1], om[leg][1], T(0.0), T(-0.5 * p.shank_len));
    k.com[3 + 3 * leg] = attach(ankle[leg], ang[leg][2], om[leg][2], T(0.0), T(-p.ankle_drop));
  }
  auto jacobian = [&](const Pt<T>& pt, int link, T (*J)[kNq]) {
    for (int r = 0; r < 2; ++r)
      for (int c = 0; c < kNq; ++c) J[r][c] = T(0.0);
    J[0][0] = T(1.0);
    J[1][1] = T(1.0);
    for (int s = 0; s < 4; ++s) {
      const int a = kChain[link][s];
      if (a < 0) break;
      J[0][a] = -(pt.pz - pivot[a].pz);
      J[1][a] = pt.px - pivot[a].px;
    }
  };
  for (int l = 0; l < 7; ++l) {
    jacobian(k.com[l], l, k.com_jac[l]);
    T ax = T(0.0), az = T(0.0);
    for (int s = 0; s < 4; ++s) {
      const int a = kChain[l][s];
      if (a < 0) break;
      ax += qd[a] * (-(k.com[l].vz - pivot[a].vz));
      az += qd[a] * (k.com[l].vx - pivot[a].vx);
    }
    k.com_jdq[l][0] = ax;
    k.com_jdq[l][1] = az;
  }
  // contacts (R toe, R heel, L toe, L heel), robot.cpp:131-146
  for (int c = 0; c < kNc; ++c) {
    const int leg = c < 2 ? 1 : 0;
    const int link = c < 2 ? 6 : 3;
    const double xo = (c % 2 == 0) ? p.foot_half_len : -p.foot_half_len;
    k.c[c] = attach(ankle[leg], ang[leg][2], om[leg][2], T(xo), T(-p.ankle_drop));
    jacobian(k.c[c], link, k.c_jac[c]);
  }
  return k;
}

inline void link_params(const rmpc_model& p, double* m, double* I) {  // robot.cpp:152-161
  const double mm[7] = {p.torso_mass, p.thigh_mass, p.shank_mass, p.foot_mass,
                        p.thigh_mass, p.shank_mass, p.foot_mass};
  const double ii[7] = {p.torso_inertia, p.thigh_inertia, p.shank_inertia, p.foot_inertia,
                        p.thigh_inertia, p.shank_inertia, p.foot_inertia};
  for (int l = 0; l < 7; ++l) { m[l] = mm[l]; I[l] = ii[l]; }
}

inline bool in_chain(int link, int a) {
  for (int s = 0; s < 4; ++s)
    if (kChain[link][s] == a) return true;
  return false;
}

// M = sum_l m_l J_l^T J_l + I_l w_l w_l^T  (robot.cpp:169-178)
template <class T>
void mass_matrix(const rmpc_model& p, const Kin<T>& k, T M[kNq][kNq]) {
  double m[7], I[7];
  link_params(p, m, I);
  for (int i = 0; i < kNq; ++i)
    for (int j = 0; j < kNq; ++j) M[i][j] = T(0.0);
  for (int l = 0; l < 7; ++l)
    for (int i = 0; i < kNq; ++i)
      for (int j = 0; j < kNq; ++j) {
        T acc = k.com_jac[l][0][i] * k.com_jac[l][0][j] + k.com_jac[l][1][i] * k.com_jac[l][1][j];
        M[i][j] += T(m[l]) * acc;
        if (in_chain(l, i) && in_chain(l, j)) M[i][j] += T(I[l]);
      }
}

// h = sum_l m_l J_l^T (Jdot_l qd + g)  (robot.cpp:184-195)
template <class T>
void bias_forces(const rmpc_model& p, const Kin<T>& k, T h[kNq]) {
  double m[7], I[7];
  link_params(p, m, I);
  for (int i = 0; i < kNq; ++i) h[i] = T(0.0);
  for (int l = 0; l < 7; ++l) {
    const T ax = k.com_jdq[l][0];
    const T az = k.com_jdq[l][1] + T(p.gravity);
    for (int i = 0; i < kNq; ++i)
      h[i] += T(m[l]) * (k.com_jac[l][0][i] * ax + k.com_jac[l][1][i] * az);
  }
}

// gen = M qdd + h - J^T F; tau = gen[3:9], base residual = gen[0:3]  (robot.cpp:211-233)
template <class T>
void inverse_dynamics(const rmpc_model& p, const T* q, const T* qd, const T* qdd, const T* F,
                      T tau[kNj], T base_res[3]) {
  const Kin<T> k = kinematics<T>(p, q, qd);
  double m[7], I[7];
  link_params(p, m, I);
  T gen[kNq];
  for (int i = 0; i < kNq; ++i) gen[i] = T(0.0);
  for (int l = 0; l < 7; ++l) {
    T ax = k.com_jdq[l][0], az = k.com_jdq[l][1] + T(p.gravity);
    T wdot = T(0.0);
    for (int j = 0; j < kNq; ++j) {
      ax += k.com_jac[l][0][j] * qdd[j];
      az += k.com_jac[l][1][j] * qdd[j];
      if (in_chain(l, j)) wdot += qdd[j];
    }
    for (int i = 0; i < kNq; ++i) {
      gen[i] += T(m[l]) * (k.com_jac[l][0][i] * ax + k.com_jac[l][1][i] * az);
      if (in_chain(l, i)) gen[i] += T(I[l]) * wdot;
    }
  }
  for (int c = 0; c < kNc; ++c)
    for (int i = 0; i < kNq; ++i)
      gen[i] -= k.c_jac[c][0][i] * F[2 * c] + k.c_jac[c][1][i] * F[2 * c + 1];
  for (int b = 0; b < 3; ++b) base_res[b] = gen[b];
  for (int j = 0; j < kNj; ++j) tau[j] = gen[3 + j];
}

// clamp(Kp (q_des - q_j) + Kd (qd_des - qd_j) + tau_ff, +-tau_limit)  (robot.cpp:235-241)
inline void pd_torque(const rmpc_model& p, const double* q_des, const double* qd_des,
                      const double* q, const double* qd, const double* tau_ff, double* out) {
  for (int j = 0; j < kNj; ++j) {
    const double t = p.kp[j] * (q_des[j] - q[3 + j]) + p.kd[j] * (qd_des[j] - qd[3 + j]) + tau_ff[j];
    out[j] = std::min(std::max(t, -p.tau_limit[j]), p.tau_limit[j]);
  }
}

// Standing pose: 2-link IK per leg for a flat foot, ankles at +-stagger shifted until the
// CoM is over the contact centroid (60-iteration fixed point).  robot.cpp:245-279.  FP64.
inline void nominal_pose(const rmpc_model& p, double q[kNq]) {
  auto leg_angles = [&](double x_off, double out[3]) {
    const double l1 = p.thigh_len, l2 = p.shank_len;
    const double hyp = std::hypot(x_off, p.nominal_drop);
    const double ck = (hyp * hyp - l1 * l1 - l2 * l2) / (2.0 * l1 * l2);
    const double knee = std::acos(std::min(1.0, std::max(-1.0, ck)));
    const double gamma = std::atan2(x_off, p.nominal_drop);
    const double beta = std::atan2(l2 * std::sin(knee), l1 + l2 * std::cos(knee));
    const double a1 = gamma - beta;
    out[0] = a1;
    out[1] = knee;
    out[2] = -(a1 + knee);
  };
  double m[7], I[7];
  link_params(p, m, I);
  double shift = 0.0;
  for (int it = 0; it < 60; ++it) {
    double l[3], r[3];
    leg_angles(shift + p.nominal_stagger, l);
    leg_angles(shift - p.nominal_stagger, r);
    q[0] = 0.0; q[1] = nominal_height(p); q[2] = 0.0;
    q[3] = l[0]; q[4] = l[1]; q[5] = l[2];
    q[6] = r[0]; q[7] = r[1]; q[8] = r[2];
    double zero[kNq] = {0};
    const Kin<double> k = kinematics<double>(p, q, zero);
    double cx = 0.0, tot = 0.0;
    for (int i = 0; i < 7; ++i) { cx += m[i] * k.com[i].px; tot += m[i]; }
    cx /= tot;
    if (std::abs(cx - shift) < 1e-14) break;
    shift = cx;
  }
}

// ---------------------------------------------------------------- gait (gait.cpp), FP64
inline double wrap01(double x) {
  const double w = std::fmod(x, 1.0);
  return w < 0.0 ? w + 1.0 : w;
}

// Stance flags and swing progress; node i uses the cumulative dt of nodes < i
// (gait.cpp:37-63).
inline void horizon_schedule(const rmpc_gait& g, const double* dt, int T,
                             std::array<bool, kNc>* stance, std::array<double, kNc>* swing_t) {
  double shift = 0.0;
  for (int i = 0; i < T; ++i) {
    for (int c = 0; c < kNc; ++c) {
      const double ph = wrap01(g.phase + shift + g.offsets[c]);
      stance[i][c] = ph < g.phase_switch;
      swing_t[i][c] = (ph >= g.phase_switch && g.phase_switch < 1.0)
                          ? (ph - g.phase_switch) / (1.0 - g.phase_switch)
                          : 0.0;
    }
    shift += dt[i] / g.period;
  }
}

// Quintic Bezier through (0, z_swing at t=1/2, 0) with end slopes v_to, v_td and P2 = P3
// (gait.cpp:65-99).  Returns height; slope through *vel.
inline double bezier_swing(double t_sw, double z_swing, double v_to, double v_td,
                           double* vel = nullptr) {
  const double t = std::min(1.0, std::max(0.0, t_sw));
  const double P[6] = {0.0, v_to / 5.0, 0.0, 0.0, -v_td / 5.0, 0.0};
  double pts[6];
  std::memcpy(pts, P, sizeof(pts));
  pts[2] = pts[3] = (32.0 * z_swing - 5.0 * (pts[1] + pts[4])) / 20.0;
  const double s = 1.0 - t;
  const double b[6] = {s * s * s * s * s,         5.0 * s * s * s * s * t, 10.0 * s * s * s * t * t,
                       10.0 * s * s * t * t * t, 5.0 * s * t * t * t * t,   t * t * t * t * t};
  double h = 0.0;
  for (int i = 0; i < 6; ++i) h += b[i] * pts[i];
  if (vel) {
    const double c[5] = {s * s * s * s, 4.0 * s * s * s * t, 6.0 * s * s * t * t,
                         4.0 * s * t * t * t, t * t * t * t};
    double v = 0.0;
    for (int i = 0; i < 5; ++i) v += c[i] * 5.0 * (pts[i + 1] - pts[i]);
    *vel = v;
  }
  return h;
}

// ---------------------------------------------------------------- sparse CSC (csc.cpp)
template <class T>
struct Csc {
  int nrows = 0, ncols = 0;
  std::vector<int> colptr, rowidx;
  std::vector<T> val;
  int nnz() const { return (int)val.size(); }
};

template <class T>
struct Trip {
  int r, c;
  T v;
};

// Canonical CSC from triplets: per-column row sort, duplicates summed, explicit zeros kept
// (csc.cpp:35-91).
template <class T>
Csc<T> csc_from_triplets(const std::vector<Trip<T>>& ts, int nrows, int ncols) {
  for (const auto& t : ts)
    if (t.r < 0 || t.r >= nrows || t.c < 0 || t.c >= ncols)
      throw StructuralError("csc_from_triplets: entry outside matrix");
  Csc<T> m;
  m.nrows = nrows;
  m.ncols = ncols;
  std::vector<int> cnt(ncols + 1, 0);
  for (const auto& t : ts) ++cnt[t.c + 1];
  for (int j = 0; j < ncols; ++j) cnt[j + 1] += cnt[j];
  std::vector<int> order(ts.size());
  {
    std::vector<int> next(cnt.begin(), cnt.end() - 1);
    for (int p = 0; p < (int)ts.size(); ++p) order[next[ts[p].c]++] = p;
  }
  m.colptr.assign(ncols + 1, 0);
  m.rowidx.reserve(ts.size());
  m.val.reserve(ts.size());
  for (int j = 0; j < ncols; ++j) {
    std::stable_sort(order.begin() + cnt[j], order.begin() + cnt[j + 1],
                     [&](int a, int b) { return ts[a].r < ts[b].r; });
    const int start = (int)m.rowidx.size();
    for (int s = cnt[j]; s < cnt[j + 1]; ++s) {
      const auto& t = ts[order[s]];
      if ((int)m.rowidx.size() > start && m.rowidx.back() == t.r) {
        m.val.back() += t.v;
      } else {
        m.rowidx.push_back(t.r);
        m.val.push_back(t.v);
      }
    }
    m.colptr[j + 1] = (int)m.rowidx.size();
  }
  return m;
}

template <class T>
void gemv(const Csc<T>& a, const std::vector<T>& x, std::vector<T>& y) {  // csc.cpp:149-155
  y.assign(a.nrows, T(0.0));
  for (int j = 0; j < a.ncols; ++j)
    for (int p = a.colptr[j]; p < a.colptr[j + 1]; ++p) y[a.rowidx[p]] += a.val[p] * x[j];
}
template <class T>
void gemv_t(const Csc<T>& a, const std::vector<T>& x, std::vector<T>& y) {  // csc.cpp:157-164
  y.assign(a.ncols, T(0.0));
  for (int j = 0; j < a.ncols; ++j) {
    T acc = T(0.0);
    for (int p = a.colptr[j]; p < a.colptr[j + 1]; ++p) acc += a.val[p] * x[a.rowidx[p]];
    y[j] = acc;
  }
}
template <class T>
void symv_upper(const Csc<T>& u, const std::vector<T>& x, std::vector<T>& y) {  // csc.cpp:166-177
  y.assign(u.nrows, T(0.0));
  for (int j = 0; j < u.ncols; ++j)
    for (int p = u.colptr[j]; p < u.colptr[j + 1]; ++p) {
      const int i = u.rowidx[p];
      y[i] += u.val[p] * x[j];
      if (i != j) y[j] += u.val[p] * x[i];
    }
}

// ---------------------------------------------------------------- Ruiz (ruiz.cpp:7-36)
// Symmetric Ruiz passes on an upper-stored square matrix: delta_i = 1/sqrt(||row_i||_inf),
// empty rows keep 1.  Scales in place; returns the accumulated scaling.
template <class T>
std::vector<T> ruiz_equilibrate(Csc<T>& a, int passes) {
  if (a.nrows != a.ncols) throw StructuralError("ruiz_equilibrate: matrix must be square");
  if (passes < 1) throw StructuralError("ruiz_equilibrate: max_iters must be >= 1");
  const int n = a.ncols;
  std::vector<T> scale(n, T(1.0)), norm(n), delta(n);
  for (int pass = 0; pass < passes; ++pass) {
    std::fill(norm.begin(), norm.end(), T(0.0));
    for (int j = 0; j < n; ++j)
      for (int p = a.colptr[j]; p < a.colptr[j + 1]; ++p) {
        const T v = abs(a.val[p]);
        const int i = a.rowidx[p];
        if (v > norm[i]) norm[i] = v;
        if (v > norm[j]) norm[j] = v;
      }
    for (int i = 0; i < n; ++i) delta[i] = norm[i] > T(0.0) ? T(1.0) / sqrt(norm[i]) : T(1.0);
    for (int j = 0; j < n; ++j)
      for (int p = a.colptr[j]; p < a.colptr[j + 1]; ++p) a.val[p] *= delta[a.rowidx[p]] * delta[j];
    for (int i = 0; i < n; ++i) scale[i] *= delta[i];
  }
  return scale;
}

// ---------------------------------------------------------------- sparse LDL^T (ldl.cpp)
// Up-looking LDL^T of a symmetric quasi-definite matrix (upper stored), no pivoting, with a
// fill-reducing symmetric permutation: P A P^T = L D L^T, (P x)[k] = x[perm[k]].
template <class T>
struct Ldl {
  int n = 0;
  std::vector<int> perm, iperm;
  Csc<T> B;                 // permuted upper copy
  std::vector<int> src;     // B.val[k] = A.val[src[k]]
  std::vector<int> parent;  // elimination tree
  std::vector<int> Lp, Li;  // strictly lower L (CSC)
  std::vector<T> Lx, D, Dinv;

  Ldl(const Csc<T>& a, bool use_ordering = true) {
    if (a.nrows != a.ncols)
      throw StructuralError("SparseLdl: matrix must be square (upper triangle stored)");
    for (int j = 0; j < a.ncols; ++j)
      for (int p = a.colptr[j]; p < a.colptr[j + 1]; ++p)
        if (a.rowidx[p] > j)
          throw StructuralError("SparseLdl: entries below the diagonal; store the upper triangle");
    n = a.ncols;
    if (use_ordering && n > 1) {
      perm = min_degree_ordering(n, a.colptr, a.rowidx);
    } else {
      perm.resize(n);
      for (int k = 0; k < n; ++k) perm[k] = k;
    }
    iperm.resize(n);
    for (int k = 0; k < n; ++k) iperm[perm[k]] = k;
    permute(a);
    symbolic();
    numeric(a);
  }

  // ldl.cpp:65-94: B = upper(P A P^T) with a source map.
  void permute(const Csc<T>& a) {
    std::vector<Trip<int>> ent;
    ent.reserve(a.nnz());
    for (int j = 0; j < a.ncols; ++j)
      for (int p = a.colptr[j]; p < a.colptr[j + 1]; ++p) {
        int bi = iperm[a.rowidx[p]], bj = iperm[j];
        if (bi > bj) std::swap(bi, bj);
        ent.push_back({bi, bj, p});
      }
    std::sort(ent.begin(), ent.end(), [](const Trip<int>& x, const Trip<int>& y) {
      return x.c != y.c ? x.c < y.c : x.r < y.r;
    });
    B.nrows = B.ncols = n;
    B.colptr.assign(n + 1, 0);
    B.rowidx.resize(ent.size());
    B.val.assign(ent.size(), T(0.0));
    src.resize(ent.size());
    for (size_t k = 0; k < ent.size(); ++k) {
      ++B.colptr[ent[k].c + 1];
      B.rowidx[k] = ent[k].r;
      src[k] = ent[k].v;
    }
    for (int j = 0; j < n; ++j) B.colptr[j + 1] += B.colptr[j];
  }

  // ldl.cpp:96-121: elimination tree and column counts.
  void symbolic() {
    parent.assign(n, -1);
    std::vector<int> flag(n), cnt(n, 0);
    for (int k = 0; k < n; ++k) {
      flag[k] = k;
      for (int p = B.colptr[k]; p < B.colptr[k + 1]; ++p) {
        for (int i = B.rowidx[p]; i < k && flag[i] != k; i = parent[i]) {
          if (parent[i] == -1) parent[i] = k;
          ++cnt[i];
          flag[i] = k;
        }
      }
    }
    Lp.assign(n + 1, 0);
    for (int k = 0; k < n; ++k) Lp[k + 1] = Lp[k] + cnt[k];
    Li.assign(Lp[n], 0);
    Lx.assign(Lp[n], T(0.0));
    D.assign(n, T(0.0));
    Dinv.assign(n, T(0.0));
  }

  // ldl.cpp:123-167: row k of L from the sparse triangular solve along the etree reach.
  void numeric(const Csc<T>& a) {
    for (size_t k = 0; k < src.size(); ++k) B.val[k] = a.val[src[k]];
    std::vector<T> y(n, T(0.0));
    std::vector<int> flag(n, -1), fill(n, 0), stack(n);
    for (int k = 0; k < n; ++k) {
      int top = n;
      flag[k] = k;
      for (int p = B.colptr[k]; p < B.colptr[k + 1]; ++p) {
        int i = B.rowidx[p];
        if (i > k) continue;
        y[i] += B.val[p];
        int len = 0;
        for (; flag[i] != k; i = parent[i]) {
          stack[len++] = i;
          flag[i] = k;
        }
        while (len > 0) stack[--top] = stack[--len];
      }
      D[k] = y[k];
      y[k] = T(0.0);
      for (; top < n; ++top) {
        const int i = stack[top];
        const T yi = y[i];
        y[i] = T(0.0);
        const int pend = Lp[i] + fill[i];
        for (int p = Lp[i]; p < pend; ++p) y[Li[p]] -= Lx[p] * yi;
        const T lki = yi / D[i];
        D[k] -= lki * yi;
        Li[pend] = k;
        Lx[pend] = lki;
        ++fill[i];
      }
      if (D[k] == T(0.0))
        throw SingularityError("SparseLdl: exact zero pivot at column " + std::to_string(perm[k]) +
                               " (permuted column " + std::to_string(k) + ")");
      Dinv[k] = T(1.0) / D[k];
    }
  }

  // ldl.cpp:176-192
  void solve_inplace(std::vector<T>& b, std::vector<T>& w) const {
    if ((int)b.size() != n) throw StructuralError("SparseLdl::solve: dimension mismatch");
    w.resize(n);
    for (int k = 0; k < n; ++k) w[k] = b[perm[k]];
    for (int k = 0; k < n; ++k) {
      const T wk = w[k];
      for (int p = Lp[k]; p < Lp[k + 1]; ++p) w[Li[p]] -= Lx[p] * wk;
    }
    for (int k = 0; k < n; ++k) w[k] *= Dinv[k];
    for (int k = n - 1; k >= 0; --k) {
      T acc = w[k];
      for (int p = Lp[k]; p < Lp[k + 1]; ++p) acc -= Lx[p] * w[Li[p]];
      w[k] = acc;
    }
    for (int k = 0; k < n; ++k) b[perm[k]] = w[k];
  }
};

// ---------------------------------------------------------------- QP + ADMM (qp.cpp)
template <class T>
struct Qp {
  Csc<T> P;  // n x n upper
  std::vector<T> q;
  Csc<T> A;  // m x n
  std::vector<T> lo, hi;
  std::vector<int> tag;  // per row: (node + 1) * 40 + slot of the device's padded layout
  int n() const { return P.ncols; }
  int m() const { return A.nrows; }
};

struct AdmmSettings {  // qp.hpp:29-36
  double sigma = 1e-6, rho = 0.1, alpha = 1.6;
  int iters = 25, ruiz_iters = 10;
  double eps_exit = 0.0;
};

template <class T>
struct QpResult {
  std::vector<T> x, y, z;
  // final iterate per row: 1 at lo, 2 at hi, 0 between (scaled space, where the clamp acts),
  // 3 for an equality row; margin = distance of the unclamped value to the nearer bound
  std::vector<int8_t> act;
  std::vector<T> margin;
  T prim = T(0.0), dual = T(0.0), obj = T(0.0), obj_quad = T(0.0), obj_lin = T(0.0);
  int iters_run = 0;
  int ldl_nnz = 0;
};

// Upper [[P + sigma I, A^T], [., -1/rho I]]  (qp.cpp:11-34)
template <class T>
Csc<T> assemble_kkt(const Csc<T>& P, const Csc<T>& A, double sigma, double rho) {
  const int n = P.ncols, m = A.nrows;
  if (P.nrows != n) throw StructuralError("assemble_kkt: P must be square");
  if (A.ncols != n) throw StructuralError("assemble_kkt: A column count != P dimension");
  std::vector<Trip<T>> ts;
  ts.reserve(P.nnz() + A.nnz() + n + m);
  for (int j = 0; j < n; ++j) {
    for (int p = P.colptr[j]; p < P.colptr[j + 1]; ++p) {
      if (P.rowidx[p] > j) throw StructuralError("assemble_kkt: P has entries below the diagonal");
      ts.push_back({P.rowidx[p], j, P.val[p]});
    }
    ts.push_back({j, j, T(sigma)});
  }
  for (int j = 0; j < n; ++j)
    for (int p = A.colptr[j]; p < A.colptr[j + 1]; ++p) ts.push_back({j, n + A.rowidx[p], A.val[p]});
  for (int i = 0; i < m; ++i) ts.push_back({n + i, n + i, T(-1.0 / rho)});
  return csc_from_triplets(ts, n + m, n + m);
}

template <class T>
T qp_value(const Qp<T>& qp, const std::vector<T>& x) {  // qp.cpp:46-50
  std::vector<T> px;
  symv_upper(qp.P, x, px);
  T a = T(0.0), b = T(0.0);
  for (int i = 0; i < qp.n(); ++i) { a += x[i] * px[i]; b += qp.q[i] * x[i]; }
  return T(0.5) * a + b;
}

// AdmmSolver::{equilibrate, assemble, factorize, run} (qp.cpp:52-202), cold start x=y=z=0
// unless warm (x0, y0) is given.
template <class T>
QpResult<T> admm_solve(const Qp<T>& qp, const AdmmSettings& st, const std::vector<T>* x0 = nullptr,
                       const std::vector<T>* y0 = nullptr, bool use_ordering = true,
                       double* stage_s = nullptr) {
  using Clock = std::chrono::steady_clock;
  Clock::time_point tmark = stage_s ? Clock::now() : Clock::time_point();
  auto lap = [&](int stage) {  // accumulate wall time into stage_s[stage]
    if (!stage_s) return;
    const Clock::time_point t = Clock::now();
    stage_s[stage] += std::chrono::duration<double>(t - tmark).count();
    tmark = t;
  };
  const int n = qp.n(), m = qp.m();
  if (qp.A.ncols != n || (int)qp.lo.size() != m || (int)qp.hi.size() != m || (int)qp.q.size() != n)
    throw StructuralError("AdmmSolver: inconsistent problem dimensions");
  if (st.iters < 1) throw StructuralError("AdmmSolver: n_iters must be >= 1");

  // equilibrate (qp.cpp:64-95)
  g_stage = kRuiz;
  std::vector<T> e(n, T(1.0)), d(m, T(1.0));
  Csc<T> Ps = qp.P, As = qp.A;
  std::vector<T> qs = qp.q, los = qp.lo, his = qp.hi;
  const bool scaled = st.ruiz_iters > 0;
  if (scaled) {
    std::vector<Trip<T>> ts;
    ts.reserve(qp.P.nnz() + qp.A.nnz());
    for (int j = 0; j < n; ++j)
      for (int p = qp.P.colptr[j]; p < qp.P.colptr[j + 1]; ++p) ts.push_back({qp.P.rowidx[p], j, qp.P.val[p]});
    for (int j = 0; j < n; ++j)
      for (int p = qp.A.colptr[j]; p < qp.A.colptr[j + 1]; ++p) ts.push_back({j, n + qp.A.rowidx[p], qp.A.val[p]});
    Csc<T> pat = csc_from_triplets(ts, n + m, n + m);
    const std::vector<T> s = ruiz_equilibrate(pat, st.ruiz_iters);
    for (int i = 0; i < n; ++i) e[i] = s[i];
    for (int i = 0; i < m; ++i) d[i] = s[n + i];
    for (int j = 0; j < n; ++j)
      for (int p = Ps.colptr[j]; p < Ps.colptr[j + 1]; ++p) Ps.val[p] *= e[Ps.rowidx[p]] * e[j];
    for (int j = 0; j < n; ++j)
      for (int p = As.colptr[j]; p < As.colptr[j + 1]; ++p) As.val[p] *= d[As.rowidx[p]] * e[j];
    for (int i = 0; i < n; ++i) qs[i] = qp.q[i] * e[i];
    for (int i = 0; i < m; ++i) { los[i] = qp.lo[i] * d[i]; his[i] = qp.hi[i] * d[i]; }
  }
  lap(kRuiz);
  // assemble + factorize (qp.cpp:97-102)
  g_stage = kKkt;
  const Csc<T> K = assemble_kkt(Ps, As, st.sigma, st.rho);
  lap(kKkt);
  g_stage = kFactor;
  const Ldl<T> ldl(K, use_ordering);
  lap(kFactor);

  g_stage = kAdmm;
  std::vector<T> x(n, T(0.0)), y(m, T(0.0)), z(m, T(0.0)), b(n + m), w, zt(m);
  if (x0 && y0) {  // qp.cpp:126-136
    for (int i = 0; i < n; ++i) x[i] = (*x0)[i] / e[i];
    for (int i = 0; i < m; ++i) y[i] = (*y0)[i] / d[i];
    gemv(As, x, z);
    for (int i = 0; i < m; ++i) z[i] = std::min(std::max(z[i], los[i]), his[i]);
  }
  const T rho = T(st.rho), alpha = T(st.alpha), rho_inv = T(1.0 / st.rho), sigma = T(st.sigma);
  QpResult<T> res;
  auto recover = [&]() {
    res.x.resize(n); res.y.resize(m); res.z.resize(m);
    for (int i = 0; i < n; ++i) res.x[i] = x[i] * e[i];
    for (int i = 0; i < m; ++i) { res.y[i] = y[i] * d[i]; res.z[i] = z[i] / d[i]; }
  };
  auto residuals = [&](T& pr, T& dr) {
    std::vector<T> ax, px, aty;
    gemv(qp.A, res.x, ax);
    symv_upper(qp.P, res.x, px);
    gemv_t(qp.A, res.y, aty);
    pr = T(0.0);
    dr = T(0.0);
    for (int i = 0; i < m; ++i) { const T v = abs(ax[i] - res.z[i]); if (v > pr) pr = v; }
    for (int i = 0; i < n; ++i) { const T v = abs(px[i] + qp.q[i] + aty[i]); if (v > dr) dr = v; }
  };
  int it = 0;
  for (; it < st.iters; ++it) {  // qp.cpp:156-190
    for (int i = 0; i < n; ++i) b[i] = sigma * x[i] - qs[i];
    for (int i = 0; i < m; ++i) b[n + i] = z[i] - y[i] / rho;
    ldl.solve_inplace(b, w);
    for (int i = 0; i < n + m; ++i)
      if (!std::isfinite((double)b[i]))
        throw DivergenceError("admm: non-finite iterate at iteration " + std::to_string(it), it);
    for (int i = 0; i < m; ++i) zt[i] = z[i] + rho_inv * (b[n + i] - y[i]);
    for (int i = 0; i < n; ++i) x[i] = alpha * b[i] + (T(1.0) - alpha) * x[i];
    const bool last = it + 1 == st.iters;
    if (last) {
      res.act.assign(m, 0);
      res.margin.assign(m, T(0.0));
    }
    for (int i = 0; i < m; ++i) {
      const T wv = alpha * zt[i] + (T(1.0) - alpha) * z[i];
      T zn = wv + rho_inv * y[i];
      if (last) {
        res.act[i] = los[i] == his[i] ? 3 : (zn <= los[i] ? 1 : (zn >= his[i] ? 2 : 0));
        res.margin[i] = std::min(abs(zn - los[i]), abs(zn - his[i]));
      }
      zn = std::min(std::max(zn, los[i]), his[i]);
      z[i] = zn;
      y[i] += rho * (wv - zn);
    }
    if (st.eps_exit > 0.0) {
      recover();
      T pr, dr;
      residuals(pr, dr);
      if (pr < T(st.eps_exit) && dr < T(st.eps_exit)) { ++it; break; }
    }
  }
  g_stage = kRnea;
  recover();
  res.iters_run = it;
  residuals(res.prim, res.dual);
  res.obj = qp_value(qp, res.x);
  {
    std::vector<T> px;
    symv_upper(qp.P, res.x, px);
    T a = T(0.0), b = T(0.0);
    for (int i = 0; i < n; ++i) { a += res.x[i] * px[i]; b += qp.q[i] * res.x[i]; }
    res.obj_quad = T(0.5) * a;
    res.obj_lin = b;
  }
  res.ldl_nnz = ldl.Lp[ldl.n];
  lap(kAdmm);
  return res;
}

// ---------------------------------------------------------------- MPC (mpc.cpp)
template <class T>
struct Traj {  // DecisionTrajectory: T rows x (9 | 9 | 8)
  int T_ = 0;
  std::vector<T> q, qd, F;
  void resize(int n) {
    T_ = n;
    q.assign((size_t)n * kNq, T(0.0));
    qd.assign((size_t)n * kNq, T(0.0));
    F.assign((size_t)n * kNf, T(0.0));
  }
};

struct Reference {  // MpcReference (mpc.hpp:75-80), FP64
  int T_ = 0;
  std::vector<double> q_des, qd_des, F_des;
  std::vector<std::array<bool, kNc>> stance;
  std::vector<std::array<double, kNc>> swing_height;
};

inline int n_active(const std::array<bool, kNc>& s) {
  int k = 0;
  for (bool b : s) k += b ? 1 : 0;
  return k;
}

// desired_trajectory (mpc.cpp:28-62)
inline Reference desired_trajectory(const rmpc_command& cmd, const rmpc_gait& gait,
                                    const rmpc_settings& st, const rmpc_model& model,
                                    const double* nominal) {
  const int T = st.horizon;
  Reference r;
  r.T_ = T;
  r.q_des.assign((size_t)T * kNq, 0.0);
  r.qd_des.assign((size_t)T * kNq, 0.0);
  r.F_des.assign((size_t)T * kNf, 0.0);
  r.stance.resize(T);
  r.swing_height.resize(T);
  std::vector<std::array<double, kNc>> swing_t(T);
  horizon_schedule(gait, st.dt_schedule, T, r.stance.data(), swing_t.data());
  const double weight = total_mass(model) * model.gravity;
  for (int i = 0; i < T; ++i) {
    for (int k = 0; k < kNq; ++k) r.q_des[i * kNq + k] = nominal[k];
    r.q_des[i * kNq + 0] = 0.0;
    r.q_des[i * kNq + 1] = cmd.height;
    r.q_des[i * kNq + 2] = 0.0;
    r.qd_des[i * kNq + 0] = cmd.vx;
    r.qd_des[i * kNq + 2] = cmd.wpitch;
    const int na = n_active(r.stance[i]);
    for (int c = 0; c < kNc; ++c) {
      if (r.stance[i][c]) {
        r.F_des[i * kNf + 2 * c + 1] = na > 0 ? weight / na : 0.0;
        r.swing_height[i][c] = 0.0;
      } else {
        r.swing_height[i][c] = bezier_swing(swing_t[i][c], st.z_swing, st.v_to, st.v_td);
      }
    }
  }
  return r;
}

inline bool finite_all(const double* v, int n) {
  for (int i = 0; i < n; ++i)
    if (!std::isfinite(v[i])) return false;
  return true;
}

// build_qp (mpc.cpp:64-238): rows ordered initial state; integration per interval; base
// dynamics per interval; contact rows per node; joint boxes from node 1.
template <class T>
Qp<T> build_qp(const rmpc_state& state, const Traj<T>& g, const Reference& ref,
               const rmpc_settings& st, const rmpc_model& model) {
  const int NT = st.horizon;
  for (int i = 0; i < NT * kNq; ++i)
    if (!std::isfinite((double)g.q[i]) || !std::isfinite((double)g.qd[i]))
      throw StructuralError("build_qp: non-finite linearization point");
  for (int i = 0; i < NT * kNf; ++i)
    if (!std::isfinite((double)g.F[i])) throw StructuralError("build_qp: non-finite linearization point");
  if (!finite_all(state.q, kNq) || !finite_all(state.qd, kNq))
    throw StructuralError("build_qp: non-finite linearization point");

  const int n = NT * kNv;
  auto vq = [](int i, int k) { return i * kNv + k; };
  auto vqd = [](int i, int k) { return i * kNv + kNq + k; };
  auto vf = [](int i, int k) { return i * kNv + 2 * kNq + k; };
  Qp<T> qp;
  {  // cost (mpc.cpp:81-103)
    std::vector<Trip<T>> pts;
    qp.q.assign(n, T(0.0));
    for (int i = 0; i < NT; ++i) {
      const double dt = st.dt_schedule[i];
      for (int k = 0; k < kNq; ++k) {
        const T wq = T(st.w_q[k] * dt), wqd = T(st.w_qd[k] * dt);
        pts.push_back({vq(i, k), vq(i, k), wq});
        pts.push_back({vqd(i, k), vqd(i, k), wqd});
        qp.q[vq(i, k)] = wq * (g.q[i * kNq + k] - T(ref.q_des[i * kNq + k]));
        qp.q[vqd(i, k)] = wqd * (g.qd[i * kNq + k] - T(ref.qd_des[i * kNq + k]));
      }
      for (int k = 0; k < kNf; ++k) {
        const T wf = T(st.w_f[k] * dt);
        pts.push_back({vf(i, k), vf(i, k), wf});
        qp.q[vf(i, k)] = wf * (g.F[i * kNf + k] - T(ref.F_des[i * kNf + k]));
      }
    }
    qp.P = csc_from_triplets(pts, n, n);
  }
  std::vector<Kin<T>> kin(NT);
  std::vector<std::array<std::array<T, kNq>, 3>> Mb(NT);
  std::vector<std::array<T, 3>> hb(NT);
  for (int i = 0; i < NT; ++i) {  // mpc.cpp:105-115
    kin[i] = kinematics<T>(model, &g.q[i * kNq], &g.qd[i * kNq]);
    T M[kNq][kNq], h[kNq];
    mass_matrix(model, kin[i], M);
    bias_forces(model, kin[i], h);
    for (int b = 0; b < 3; ++b) {
      for (int k = 0; k < kNq; ++k) Mb[i][b][k] = M[b][k];
      hb[i][b] = h[b];
    }
  }
  std::vector<Trip<T>> at;
  std::vector<T> lo, hi;
  int row = 0;
  std::vector<int> tag;
  int cur_tag = 0;  // set before each bound(); slots as in the device layout (rmpc_device.cuh)
  auto bound = [&](T l, T h) { lo.push_back(l); hi.push_back(h); tag.push_back(cur_tag); ++row; };
  const T inf = T(kInf);
  for (int k = 0; k < kNq; ++k) {  // initial state (mpc.cpp:126-136)
    at.push_back({row, vq(0, k), T(1.0)});
    const T r = T(state.q[k]) - g.q[k];
    cur_tag = 12 + k;
    bound(r, r);
  }
  for (int k = 0; k < kNq; ++k) {
    at.push_back({row, vqd(0, k), T(1.0)});
    const T r = T(state.qd[k]) - g.qd[k];
    cur_tag = 21 + k;
    bound(r, r);
  }
  for (int i = 0; i + 1 < NT; ++i) {  // integration (mpc.cpp:138-148)
    const T dt = T(st.dt_schedule[i]);
    for (int k = 0; k < kNq; ++k) {
      at.push_back({row, vq(i + 1, k), T(1.0)});
      at.push_back({row, vq(i, k), T(-1.0)});
      at.push_back({row, vqd(i + 1, k), -dt});
      const T r = -(g.q[(i + 1) * kNq + k] - g.q[i * kNq + k] - dt * g.qd[(i + 1) * kNq + k]);
      cur_tag = (i + 1) * 40 + k;
      bound(r, r);
    }
  }
  for (int i = 0; i + 1 < NT; ++i) {  // base dynamics (mpc.cpp:150-175)
    const T dti = T(1.0 / st.dt_schedule[i]);
    T res[3];
    for (int b = 0; b < 3; ++b) {
      T mq = T(0.0);
      for (int k = 0; k < kNq; ++k) mq += Mb[i][b][k] * (g.qd[(i + 1) * kNq + k] - g.qd[i * kNq + k]);
      T jf = T(0.0);
      for (int c = 0; c < kNc; ++c)
        jf += kin[i].c_jac[c][0][b] * g.F[i * kNf + 2 * c] + kin[i].c_jac[c][1][b] * g.F[i * kNf + 2 * c + 1];
      res[b] = mq * dti + hb[i][b] - jf;
    }
    for (int b = 0; b < 3; ++b) {
      for (int k = 0; k < kNq; ++k) {
        const T mv = Mb[i][b][k] * dti;
        if (mv != T(0.0)) {
          at.push_back({row, vqd(i + 1, k), mv});
          at.push_back({row, vqd(i, k), -mv});
        }
      }
      for (int c = 0; c < kNc; ++c) {
        at.push_back({row, vf(i, 2 * c), -kin[i].c_jac[c][0][b]});
        at.push_back({row, vf(i, 2 * c + 1), -kin[i].c_jac[c][1][b]});
      }
      cur_tag = (i + 1) * 40 + 9 + b;
      bound(-res[b], -res[b]);
    }
  }
  const T mu = T(st.mu);
  for (int i = 0; i < NT; ++i) {  // contacts (mpc.cpp:181-218)
    for (int c = 0; c < kNc; ++c) {
      const T fx = g.F[i * kNf + 2 * c], fz = g.F[i * kNf + 2 * c + 1];
      int t_ = 0;
      auto ctag = [&]() { cur_tag = (i + 1) * 40 + 12 + 4 * c + t_++; };
      if (ref.stance[i][c]) {
        at.push_back({row, vf(i, 2 * c), T(1.0)});
        at.push_back({row, vf(i, 2 * c + 1), -mu});
        ctag();
        bound(-inf, -(fx - mu * fz));
        at.push_back({row, vf(i, 2 * c), T(-1.0)});
        at.push_back({row, vf(i, 2 * c + 1), -mu});
        ctag();
        bound(-inf, -(-fx - mu * fz));
        if (i == 0) continue;
        for (int ax = 0; ax < 2; ++ax) {
          T r = T(0.0);
          for (int k = 0; k < kNq; ++k) r += kin[i].c_jac[c][ax][k] * g.qd[i * kNq + k];
          r = -r;
          for (int k = 0; k < kNq; ++k) {
            const T j = kin[i].c_jac[c][ax][k];
            if (j != T(0.0)) at.push_back({row, vqd(i, k), j});
          }
          ctag();
          bound(r, r);
        }
      } else {
        at.push_back({row, vf(i, 2 * c), T(1.0)});
        ctag();
        bound(-fx, -fx);
        at.push_back({row, vf(i, 2 * c + 1), T(1.0)});
        ctag();
        bound(-fz, -fz);
        if (i == 0) continue;
        const T r = T(ref.swing_height[i][c]) - kin[i].c[c].pz;
        for (int k = 0; k < kNq; ++k) {
          const T j = kin[i].c_jac[c][1][k];
          if (j != T(0.0)) at.push_back({row, vq(i, k), j});
        }
        ctag();
        bound(r, r);
      }
    }
  }
  for (int i = 1; i < NT; ++i) {  // joint boxes (mpc.cpp:220-232)
    for (int k = 0; k < kNj; ++k) {
      at.push_back({row, vq(i, 3 + k), T(1.0)});
      cur_tag = (i + 1) * 40 + 28 + k;
      bound(T(model.joint_lo[k]) - g.q[i * kNq + 3 + k], T(model.joint_hi[k]) - g.q[i * kNq + 3 + k]);
    }
    for (int k = 0; k < kNj; ++k) {
      at.push_back({row, vqd(i, 3 + k), T(1.0)});
      cur_tag = (i + 1) * 40 + 34 + k;
      bound(T(-model.qd_limit[k]) - g.qd[i * kNq + 3 + k], T(model.qd_limit[k]) - g.qd[i * kNq + 3 + k]);
    }
  }
  qp.A = csc_from_triplets(at, row, n);
  qp.lo = lo;
  qp.hi = hi;
  qp.tag = tag;
  return qp;
}

// FP64 output record of one agent (MpcSolution, mpc.hpp:100-116).
struct Solution {
  int status = RMPC_STATUS_OK;
  int fail_iter = -1;
  std::string message;
  std::vector<double> z_star;  // T x 26 (q | qd | F per node)
  double tau_ff[kNj] = {0}, q_set[kNj] = {0}, qd_set[kNj] = {0}, f0[kNf] = {0};
  double v_mpc = 0, prim_res = 0, dual_res = 0, delta_inf = 0, base_res[3] = {0};
  double v_quad = 0, v_lin = 0;
  double stage_s[kNumStages] = {0};
  int m = 0, n = 0, ldl_nnz = 0;
  // active set of the final iterate on the device's (node + 1, slot) grid ((T+1) x 40):
  // 0 inactive, 1 at lo, 2 at hi, 3 equality row or no row; margin as in QpResult
  std::vector<int8_t> act;
  std::vector<double> act_margin;
};

// MpcController::rti_step (mpc.cpp:248-338).  `prev_z` (T x 26) is read only when
// settings.warm_start and prev_ok.
template <class T>
Solution rti_step(const rmpc_model& model, const rmpc_settings& st, const double* nominal,
                  const rmpc_state& state, const rmpc_command& cmd, const rmpc_gait& gait,
                  const double* prev_z = nullptr, bool prev_ok = false, bool timed = false);

}  // namespace oracle

#include "rmpc_oracle_rti.hpp"
