// rmpc_kin.cuh — FP64 planar-biped kinematics on the device (compute_kinematics,
// /root/reference/proj/src/robot.cpp:29-148), shared by the solve kernel (linearization,
// inverse dynamics) and the simulator step (rmpc_env.cu).
#pragma once

namespace rmpc_dev {

struct Fr {
  double px, pz, vx, vz;
};

// Point attached to `f` at offset (x, z) in the frame rotated by an angle with sine/cosine
// (s, c), spinning at `w` (robot.cpp:39-43).
__device__ __forceinline__ Fr attach(const Fr& f, double s, double c, double w, double x, double z) {
  const double rx = c * x - s * z, rz = s * x + c * z;
  Fr o;
  o.px = f.px + rx;
  o.pz = f.pz + rz;
  o.vx = f.vx - w * rz;
  o.vz = f.vz + w * rx;
  return o;
}

// Kinematic chains of the 7 links (robot.cpp:18-21): coordinate indices, -1 padded.
__device__ __forceinline__ int kchain(int l, int s) {
  const int t[7][4] = {{2, -1, -1, -1}, {2, 3, -1, -1}, {2, 3, 4, -1}, {2, 3, 4, 5},
                       {2, 6, -1, -1},  {2, 6, 7, -1},  {2, 6, 7, 8}};
  return t[l][s];
}

// Frames of the planar biped at (q, qd) with base x taken as 0: Jacobians, J-dot qd and
// masses depend only on position differences (robot.cpp:98), contact heights only on z.
struct Frames {
  Fr piv[9];  // pivots of angle coordinates 2..8
  Fr com[7];
  Fr con[4];
};

// Each of the 7 absolute angles (pitch, then hip/knee/ankle of each leg) gets one sincos.
// The 7 absolute angles (pitch, then hip/knee/ankle of each leg) fk_frames rotates by.
__device__ __forceinline__ double fk_angle(const double* q, int k) {
  if (k == 0) return q[2];
  const int h = k <= 3 ? 3 : 6, n = k <= 3 ? k : k - 3;
  double a = q[2] + q[h];
  if (n > 1) a = a + q[h + 1];
  if (n > 2) a = a + q[h + 2];
  return a;
}

// fk_frames with the sines / cosines of the 7 angles given (sc[k] = {sin, cos} of fk_angle k),
// so a warp can compute them on 7 lanes.
template <class Geo>
__device__ void fk_frames_sc(const Geo& P, const double* q, const double* qd, const double sc[7][2], Frames& F,
                             double base_x = 0.0) {
  Fr base;
  base.px = base_x;  // 0 for the solve: Jacobians use position differences only
  base.pz = q[1];
  base.vx = qd[0];
  base.vz = qd[1];
  const Fr hip = attach(base, sc[0][0], sc[0][1], qd[2], 0.0, -0.5 * P.torso_len);
  F.piv[2] = base;
  F.piv[3] = hip;
  F.piv[6] = hip;
  F.com[0] = base;
#pragma unroll
  for (int leg = 0; leg < 2; ++leg) {  // 0 = left (3..5), 1 = right (6..8)
    const int h = 3 + 3 * leg, a = 1 + 3 * leg;
    const double w1 = qd[2] + qd[h], w2 = w1 + qd[h + 1], w3 = w2 + qd[h + 2];
    const Fr knee = attach(hip, sc[a][0], sc[a][1], w1, 0.0, -P.thigh_len);
    const Fr ankle = attach(knee, sc[a + 1][0], sc[a + 1][1], w2, 0.0, -P.shank_len);
    F.piv[h + 1] = knee;
    F.piv[h + 2] = ankle;
    F.com[1 + 3 * leg] = attach(hip, sc[a][0], sc[a][1], w1, 0.0, -0.5 * P.thigh_len);
    F.com[2 + 3 * leg] = attach(knee, sc[a + 1][0], sc[a + 1][1], w2, 0.0, -0.5 * P.shank_len);
    F.com[3 + 3 * leg] = attach(ankle, sc[a + 2][0], sc[a + 2][1], w3, 0.0, -P.ankle_drop);
    const int k0 = leg == 0 ? 2 : 0;  // contacts (R toe, R heel, L toe, L heel)
    F.con[k0] = attach(ankle, sc[a + 2][0], sc[a + 2][1], w3, P.foot_half, -P.ankle_drop);
    F.con[k0 + 1] = attach(ankle, sc[a + 2][0], sc[a + 2][1], w3, -P.foot_half, -P.ankle_drop);
  }
}

// Each of the 7 absolute angles gets one sincos.
template <class Geo>  // torso_len, thigh_len, shank_len, foot_half, ankle_drop
__device__ void fk_frames(const Geo& P, const double* q, const double* qd, Frames& F, double base_x = 0.0) {
  double sc[7][2];
#pragma unroll
  for (int k = 0; k < 7; ++k) sincos(fk_angle(q, k), &sc[k][0], &sc[k][1]);
  fk_frames_sc(P, q, qd, sc, F, base_x);
}

// Contact Jacobian rows (2 x 9) of contact c (robot.cpp:91-101,137-146).
__device__ __forceinline__ void contact_jac(const Frames& F, int c, double Jx[9], double Jz[9]) {
#pragma unroll
  for (int k = 0; k < 9; ++k) Jx[k] = Jz[k] = 0.0;
  Jx[0] = 1.0;
  Jz[1] = 1.0;
  const int h = c < 2 ? 6 : 3;
  const int chain[4] = {2, h, h + 1, h + 2};
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const int a = chain[s];
    Jx[a] = -(F.con[c].pz - F.piv[a].pz);
    Jz[a] = F.con[c].px - F.piv[a].px;
  }
}

}  // namespace rmpc_dev
