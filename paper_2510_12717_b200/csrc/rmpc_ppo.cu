// rmpc_ppo.cu — the PPO batch on sm_100a (second half), FP64 like the
// reference (/root/reference/proj/src/ppo.cpp):
//
//   rmpc_ppo_loss_device    ppo_loss (ppo.cpp:79-135): policy_forward with the cache
//                           (policy.cpp:85-102), gaussian_log_prob (policy.cpp:168-176), the
//                           clipped surrogate / value / entropy terms and mlp_backward
//                           (ppo.cpp:63-77) summed over the batch
//   rmpc_gae_device         gae_advantages (ppo.cpp:28-45)
//   rmpc_ppo_update_device  ppo_update (ppo.cpp:195-276): GAE, advantage normalisation, epochs x
//                           minibatches of {Fisher-Yates shuffle, ppo_loss, gradient-norm clip,
//                           AdamOptimizer::step (ppo.cpp:179-193)}
//
// Loss kernel.  The batch gradient is a sum over samples of outer products delta_l post_l^T,
// i.e. per layer a (out x n) . (n x in) product with a long reduction dimension: the kernel is
// split-K over the samples.  Grid = (chunks, 2): blockIdx.y picks the trunk (pi / value, which
// are independent given the batch), blockIdx.x a contiguous chunk of samples.  A block keeps its
// trunk's weights in shared memory and walks its chunk in tiles of 32 samples: forward
// (activations and ELU derivatives cached in shared memory), the per-sample loss head (warp =
// sample), backward layer by layer, then the gradient update, whose per-thread share stays in
// registers for the whole chunk; the per-chunk partial gradients are summed in a fixed order by
// a second kernel (deterministic, no atomics).  Two implementations of the block:
//   loss_kernel_mma  every product on the FP64 tensor cores (mma.sync.m8n8k4.f64 -- tcgen05 has
//                    no FP64 kind; TF32/BF16 would miss the FP64 reference by orders of
//                    magnitude), operands straight from shared memory in 8x8 blocks
//   loss_kernel<TL>  CUDA-core FMAs for shapes beyond the tensor-core layout (obs > 32 or
//                    shared memory), thread = neuron x TL/8 samples, paired double2 loads
// The FP64 work is ~0.11 MFLOP per sample.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <new>
#include <vector>

#include "rmpc_policy.cuh"

namespace rmpc_ppo_dev {

using rmpc_policy_dev::MAXH;
using rmpc_policy_dev::MAXIO;
using rmpc_policy_dev::Net;
using rmpc_policy_dev::PolicyParams;

constexpr int THREADS = 512, TILE = 32, WARPS = THREADS / 32;
constexpr double kLogSqrt2Pi = 0.91893853320467274178032973640562;

struct TrunkSm {
  int ld[4];        // padded column stride of W_l in shared memory (odd)
  int w[4], b[4];   // shared-memory offsets of W_l and b_l
  int wr[4], br[4]; // offsets of W_l and b_l relative to the trunk's first parameter
  int wtotal;       // doubles of the shared weight region
};

struct LossParams {
  PolicyParams P;
  TrunkSm ts[2];
  int n, chunk, nch;    // samples, samples per block, blocks per trunk
  int pst, dst, ost;    // per-sample strides of the activation / delta / output tiles
  int part_stride;      // doubles per (trunk, chunk) partial
  double clip_eps, value_coef, inv_n;
  const double* w;      // parameters (flatten_policy order)
  const double* obs;
  const double* act;
  const double* old_logp;
  const double* adv;
  const double* ret;
  const int32_t* idx;   // optional gather: sample s of the batch is row idx[s]
  double* part;
};

// expm1(z) for z <= 0 (the ELU branch), ~1 ulp: z = k ln2 + r (Cody-Waite), |r| <= ln2 / 2,
// expm1(r) by a degree-12 Taylor polynomial (remainder < 2e-17), then
// expm1(z) = 2^k expm1(r) + (2^k - 1).  About half the instructions of the general routine.
__device__ __forceinline__ double expm1_neg(double z) {
  if (z < -40.0) return -1.0;
  const double k = rint(z * 1.4426950408889634074);
  const double r = fma(k, -1.9082149292705877000e-10, fma(k, -6.93147180369123816490e-01, z));
  double p = 2.08767569878680989792e-09;  // 1/12!
  p = fma(p, r, 2.50521083854417187751e-08);  // 1/11!
  p = fma(p, r, 2.75573192239858906526e-07);
  p = fma(p, r, 2.75573192239858906526e-06);
  p = fma(p, r, 2.48015873015873015873e-05);
  p = fma(p, r, 1.98412698412698412698e-04);
  p = fma(p, r, 1.38888888888888888889e-03);
  p = fma(p, r, 8.33333333333333333333e-03);
  p = fma(p, r, 4.16666666666666666667e-02);
  p = fma(p, r, 1.66666666666666666667e-01);
  p = fma(p, r, 0.5);
  p = fma(p * r, r, r);  // r + r^2 (1/2 + r/6 + ...)
  const int ki = (int)k;
  const double sc = __hiloint2double((ki + 1023) << 20, 0);  // 2^k, k in [-58, 0]
  return fma(sc, p, sc - 1.0);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Tile layouts, per sample (every segment starts at an even offset, so pairs load as double2):
// activations [post_0 = obs | post_1 | post_2 | post_3 | 1] and deltas [d_0 | d_1 | d_2 | d_3]
// (d_l holds ELU'(z_l) after the forward pass, then the delta).
__device__ __forceinline__ int even_up(int x) { return (x + 1) & ~1; }
__device__ __forceinline__ int poff(const PolicyParams& P, int l) {
  return l == 0 ? 0 : even_up(P.obs) + (l - 1) * even_up(P.hidden);
}
__device__ __forceinline__ int doff(const PolicyParams& P, int l) { return l * even_up(P.hidden); }

template <int TL>
__global__ void __launch_bounds__(THREADS, 1) loss_kernel(const LossParams L) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double lstd[MAXIO], lsd[MAXIO];  // log_std and exp(log_std), once per block
  __shared__ double wred[WARPS];
  const int trunk = blockIdx.y, chunk = blockIdx.x;
  const PolicyParams& P = L.P;
  const Net& N = trunk == 0 ? P.pi : P.vf;
  const TrunkSm& S = L.ts[trunk];
  double* W = sm;
  double* post = W + S.wtotal;
  double* del = post + TL * L.pst;
  double* out = del + TL * L.dst;  // TL x ost trunk outputs
  double* red = post;                // WARPS x MAXIO log_std partials (after the last tile)
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;

  for (int l = 0; l < 4; ++l) {
    const int rows = N.out[l], cols = N.in[l];
    for (int e = t; e < rows * cols; e += THREADS) W[S.w[l] + (e / rows) * S.ld[l] + e % rows] = L.w[N.w[l] + e];
    for (int i = t; i < rows; i += THREADS) W[S.b[l] + i] = L.w[N.b[l] + i];
  }
  if (t < P.act) {
    lstd[t] = L.w[P.total + t];
    lsd[t] = exp(lstd[t]);
  }
  // pads stay zero (the paired loads read them)
  for (int e = t; e < TL * (L.pst + L.dst); e += THREADS) post[e] = 0.0;

  // Gradient ownership: thread (i, kg) accumulates W_l(i, k) for k in [8 kg, 8 kg + 8) of every
  // layer and, for kg = 0, b_l(i): delta_l(s, i) is loaded once per sample and layer, the 8
  // activations as 4 broadcast double2.
  const int i = t & 63, kg = t >> 6, sg = kg;  // sg: sample group (samples sg + 8 q) elsewhere
  double accW[4][8], accB[4];
#pragma unroll
  for (int l = 0; l < 4; ++l) {
    accB[l] = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) accW[l][j] = 0.0;
  }
  double lsg0 = 0.0, lsg1 = 0.0, lsum = 0.0;  // log_std gradient (lanes j, j + 32), loss term
  const int c0 = chunk * L.chunk, c1 = min(L.n, c0 + L.chunk);
  __syncthreads();

  for (int base = c0; base < c1; base += TL) {
    // ---- load the tile (rows past the chunk are zero: zero delta, zero contribution)
    for (int e = t; e < TL * P.obs; e += THREADS) {
      const int s = e / P.obs, k = e % P.obs, g = base + s;
      double v = 0.0;
      if (g < c1) v = L.obs[(size_t)(L.idx ? L.idx[g] : g) * P.obs + k];
      post[s * L.pst + k] = v;
    }
    __syncthreads();
    // ---- forward (mlp_forward, policy.cpp:15-31): z = W h + b, ELU on the hidden layers;
    // thread = neuron i x samples sg + 8 q, input pairs as broadcast double2
    for (int l = 0; l < 4; ++l) {
      const int rows = N.out[l], cols = N.in[l];
      if (i < rows) {
        const double* Wl = W + S.w[l] + i;
        const int ld = S.ld[l];
        const double2* x = reinterpret_cast<const double2*>(post + sg * L.pst + poff(P, l));
        const int xs = 4 * L.pst;  // 8 samples, in double2
        double a[(TL / 8)];
#pragma unroll
        for (int q = 0; q < (TL / 8); ++q) a[q] = 0.0;
#pragma unroll 2
        for (int k2 = 0; k2 < cols / 2; ++k2) {
          const double w0 = Wl[2 * k2 * ld], w1 = Wl[(2 * k2 + 1) * ld];
#pragma unroll
          for (int q = 0; q < (TL / 8); ++q) {
            const double2 u = x[q * xs + k2];
            a[q] = fma(w1, u.y, fma(w0, u.x, a[q]));
          }
        }
        if (cols & 1) {
          const double w0 = Wl[(cols - 1) * ld];
#pragma unroll
          for (int q = 0; q < (TL / 8); ++q) a[q] = fma(w0, x[q * xs + cols / 2].x, a[q]);
        }
        const double bi = W[S.b[l] + i];
#pragma unroll
        for (int q = 0; q < (TL / 8); ++q) {
          const int s = sg + 8 * q;
          const double z = a[q] + bi;
          if (l < 3) {
            const double em = expm1(fmin(z, 0.0));  // ELU and ELU' = exp(z) = expm1(z) + 1
            post[s * L.pst + poff(P, l + 1) + i] = z > 0.0 ? z : em;
            del[s * L.dst + doff(P, l) + i] = z > 0.0 ? 1.0 : em + 1.0;  // elu_grad, ppo.cpp:12
          } else {
            out[s * L.ost + i] = z;
          }
        }
      }
      __syncthreads();
    }
    // ---- loss head (ppo.cpp:92-126), warp = sample
    for (int s = warp; s < TL; s += WARPS) {
      const int g = base + s;
      const bool valid = g < c1;
      const size_t row = valid ? (size_t)(L.idx ? L.idx[g] : g) : 0;
      double* d3 = del + s * L.dst + doff(P, 3);
      if (trunk == 0) {
        const int A = P.act;
        double z0 = 0.0, z1 = 0.0, sd0 = 1.0, sd1 = 1.0, lp = 0.0;
        if (lane < A) {
          sd0 = lsd[lane];
          z0 = (L.act[row * A + lane] - out[s * L.ost + lane]) / sd0;
          lp += -0.5 * z0 * z0 - lstd[lane] - kLogSqrt2Pi;
        }
        if (lane + 32 < A) {
          sd1 = lsd[lane + 32];
          z1 = (L.act[row * A + lane + 32] - out[s * L.ost + lane + 32]) / sd1;
          lp += -0.5 * z1 * z1 - lstd[lane + 32] - kLogSqrt2Pi;
        }
        lp = warp_sum(lp);
        const double adv = valid ? L.adv[row] : 0.0;
        const double ratio = exp(lp - (valid ? L.old_logp[row] : 0.0));
        const double surr1 = ratio * adv;
        const double clipped = fmin(fmax(ratio, 1.0 - L.clip_eps), 1.0 + L.clip_eps) * adv;
        if (lane == 0 && valid) lsum += -fmin(surr1, clipped) * L.inv_n;
        const double g_r = surr1 <= clipped ? -adv * L.inv_n : 0.0;
        const bool on = valid && g_r != 0.0;
        const double g_logp = g_r * ratio;
        if (lane < A) {
          d3[lane] = on ? g_logp * z0 / sd0 : 0.0;
          if (on) lsg0 += g_logp * (z0 * z0 - 1.0);
        }
        if (lane + 32 < A) {
          d3[lane + 32] = on ? g_logp * z1 / sd1 : 0.0;
          if (on) lsg1 += g_logp * (z1 * z1 - 1.0);
        }
        if (lane == 0 && (A & 1)) d3[A] = 0.0;  // pad of the paired loads
      } else if (lane == 0) {
        const double verr = valid ? out[s * L.ost] - L.ret[row] : 0.0;
        if (valid) lsum += 0.5 * verr * verr * L.inv_n;
        d3[0] = valid ? L.value_coef * verr * L.inv_n : 0.0;
        d3[1] = 0.0;  // pad of the paired loads
      }
    }
    __syncthreads();
    // ---- backward (mlp_backward, ppo.cpp:63-77): delta_{l-1} = (W_l^T delta_l) .* ELU'(z_{l-1});
    // thread = column i x samples sg + 8 q, delta pairs as broadcast double2
    for (int l = 3; l > 0; --l) {
      const int rows = N.out[l], cols = N.in[l];
      if (i < cols) {
        const double* Wl = W + S.w[l] + i * S.ld[l];
        const double2* e = reinterpret_cast<const double2*>(del + sg * L.dst + doff(P, l));
        const int es = 4 * L.dst;  // 8 samples, in double2
        double b[(TL / 8)];
#pragma unroll
        for (int q = 0; q < (TL / 8); ++q) b[q] = 0.0;
#pragma unroll 2
        for (int r2 = 0; r2 < (rows + 1) / 2; ++r2) {
          const double w0 = Wl[2 * r2], w1 = 2 * r2 + 1 < rows ? Wl[2 * r2 + 1] : 0.0;
#pragma unroll
          for (int q = 0; q < (TL / 8); ++q) {
            const double2 u = e[q * es + r2];
            b[q] = fma(w1, u.y, fma(w0, u.x, b[q]));
          }
        }
#pragma unroll
        for (int q = 0; q < (TL / 8); ++q) del[(sg + 8 * q) * L.dst + doff(P, l - 1) + i] *= b[q];
      }
      __syncthreads();
    }
    // ---- gradient: W_l += delta_l post_l^T, b_l += delta_l over the tile
#pragma unroll 1
    for (int s = 0; s < TL; ++s) {
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        const int rows = N.out[l], cols = N.in[l];
        if (i < rows) {
          const double d = del[s * L.dst + doff(P, l) + i];
          if (kg == 0) accB[l] += d;
          if (8 * kg < cols) {
            const double2* pp = reinterpret_cast<const double2*>(post + s * L.pst + poff(P, l) + 8 * kg);
#pragma unroll
            for (int j2 = 0; j2 < 4; ++j2) {
              const double2 u = pp[j2];
              accW[l][2 * j2] = fma(d, u.x, accW[l][2 * j2]);
              accW[l][2 * j2 + 1] = fma(d, u.y, accW[l][2 * j2 + 1]);
            }
          }
        }
      }
    }
    __syncthreads();
  }
  // ---- per-chunk partials: gradient entries, log_std gradient (pi), loss term
  double* part = L.part + (size_t)(trunk * L.nch + chunk) * L.part_stride;
#pragma unroll
  for (int l = 0; l < 4; ++l) {
    const int rows = N.out[l], cols = N.in[l];
    if (i < rows) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (8 * kg + j < cols) part[S.wr[l] + (8 * kg + j) * rows + i] = accW[l][j];
      if (kg == 0) part[S.br[l] + i] = accB[l];
    }
  }
  if (trunk == 0) {
    red[warp * MAXIO + lane] = lsg0;
    red[warp * MAXIO + lane + 32] = lsg1;
  }
  if (lane == 0) wred[warp] = lsum;
  __syncthreads();
  if (trunk == 0 && t < P.act) {
    double v = 0.0;
    for (int w = 0; w < WARPS; ++w) v += red[w * MAXIO + t];
    part[N.total + t] = v;
  }
  if (t == 0) {
    double v = 0.0;
    for (int w = 0; w < WARPS; ++w) v += wred[w];
    part[N.total + MAXIO] = v;
  }
}

// ------------------------------------------------------------------------- FP64 tensor-core path
// The same loss and gradient with every matrix product on the FP64 tensor cores
// (mma.sync.m8n8k4.f64; tcgen05 has no FP64 kind).  Per tile of 32 samples: forward
// Z = X W^T + b, backward delta_{l-1} = (delta_l W) .* ELU', gradient G_l += delta_l^T X_l, all
// as 8x8 output blocks with k-steps of 4, operands straight from shared memory (row strides
// = 4 mod 16 doubles: conflict-free fragment loads).  A thread's gradient blocks stay in its
// registers for the whole chunk (C fragments).  Measured peak of the unit on this GPU ~36 TFLOP/s,
// the same as the FP64 FMA pipe: the gain is 8-16x fewer shared-memory loads per FLOP.
constexpr int MAXB = 14;  // gradient blocks per warp (obs <= 32, hidden <= 64, act <= 64)

struct MmaTrunk {
  int K[4], N[4];    // layer in / out
  int Kp[4], Np[4];  // padded to 8
  int ldw[4];        // shared row stride of W_l (one row per input k): = 4 mod 16, >= Np
  int w[4], b[4];    // shared offsets of W_l, b_l
  int wr[4], br[4];  // parameter offsets relative to the trunk
  int nblk[4];       // gradient blocks of layer l: (Np / 8) x (Kp / 8)
  int wtotal;
};

struct MmaParams {
  PolicyParams P;
  MmaTrunk tr[2];
  int ldx[4], xo[4];  // activation X_l = input of layer l: TILE x ldx_l at xo_l
  int ldd[4], dd[4];  // delta_l: TILE x ldd_l at dd_l (ELU' first, then the delta)
  int xtotal, dtotal;
  int n, chunk, nch, part_stride;
  double clip_eps, value_coef, inv_n;
  const double* w;
  const double* obs;
  const double* act;
  const double* old_logp;
  const double* adv;
  const double* ret;
  const int32_t* idx;
  double* part;
};

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(THREADS, 1) loss_kernel_mma(const MmaParams L) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double lstd[MAXIO], lsd[MAXIO];  // log_std and exp(log_std), once per block
  __shared__ double wred[WARPS];
  const int trunk = blockIdx.y, chunk = blockIdx.x;
  const PolicyParams& P = L.P;
  const Net& N = trunk == 0 ? P.pi : P.vf;
  const MmaTrunk& T = L.tr[trunk];
  double* W = sm;
  double* X = W + T.wtotal;
  double* D = X + L.xtotal;
  double* red = X;  // WARPS x MAXIO log_std partials (after the last tile)
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, g = lane >> 2, q = lane & 3;

  for (int e = t; e < T.wtotal + L.xtotal + L.dtotal; e += THREADS) sm[e] = 0.0;  // pads stay 0
  __syncthreads();
  for (int l = 0; l < 4; ++l) {
    const int rows = N.out[l], cols = N.in[l];
    for (int e = t; e < rows * cols; e += THREADS) W[T.w[l] + (e / rows) * T.ldw[l] + e % rows] = L.w[N.w[l] + e];
    for (int i = t; i < rows; i += THREADS) W[T.b[l] + i] = L.w[N.b[l] + i];
  }
  if (t < P.act) {
    lstd[t] = L.w[P.total + t];
    lsd[t] = exp(lstd[t]);
  }

  double acc[MAXB][2];
  // this warp's gradient blocks, decoded once: delta / activation fragment offsets | layer << 30
  uint32_t gblk[MAXB];
#pragma unroll
  for (int r = 0; r < MAXB; ++r) {
    acc[r][0] = acc[r][1] = 0.0;
    int j = warp + WARPS * r, l = 0;
    while (l < 4 && j >= T.nblk[l]) j -= T.nblk[l++];
    gblk[r] = 0xffffffffu;
    if (l < 4) {
      const int nbk = T.Kp[l] / 8, nb = j / nbk, kb = j % nbk;
      const uint32_t doff = L.dd[l] + q * L.ldd[l] + 8 * nb + g, xoff = L.xo[l] + q * L.ldx[l] + 8 * kb + g;
      gblk[r] = doff | (xoff << 15) | ((uint32_t)l << 30);
    }
  }
  // bias gradient entry of this thread: layer bl, row bn (flat over the trunk's biases)
  int bl = -1, bn = 0;
  {
    int e = t;
    for (int l = 0; l < 4 && bl < 0; ++l) {
      if (e < N.out[l]) { bl = l; bn = e; }
      else e -= N.out[l];
    }
  }
  double accB = 0.0;
  double lsg0 = 0.0, lsg1 = 0.0, lsum = 0.0;
  const int c0 = chunk * L.chunk, c1 = min(L.n, c0 + L.chunk);
  __syncthreads();

  for (int base = c0; base < c1; base += TILE) {
    // ---- load the tile into X_0 (rows past the chunk stay zero)
    for (int e = t; e < TILE * P.obs; e += THREADS) {
      const int s = e / P.obs, k = e % P.obs, gi = base + s;
      X[L.xo[0] + s * L.ldx[0] + k] = gi < c1 ? L.obs[(size_t)(L.idx ? L.idx[gi] : gi) * P.obs + k] : 0.0;
    }
    __syncthreads();
    // ---- forward: Z_l = X_l W_l^T (+ b), unit = (M block mb, N blocks nb0, nb0 + 1)
    for (int l = 0; l < 4; ++l) {
      const int nbN = T.Np[l] / 8, units = 4 * ((nbN + 1) / 2);
      const double* Wl = W + T.w[l];
      const double* Xl = X + L.xo[l];
      const int ldw = T.ldw[l], ldx = L.ldx[l];
      for (int u = warp; u < units; u += WARPS) {
        const int mb = u & 3, nb0 = 2 * (u >> 2);
        const bool two = nb0 + 1 < nbN;
        double z00 = 0.0, z01 = 0.0, z10 = 0.0, z11 = 0.0;
        const double* xa = Xl + (8 * mb + g) * ldx + q;
        const double* wb = Wl + q * ldw + 8 * nb0 + g;
#pragma unroll 4
        for (int k4 = 0; k4 < T.Kp[l] / 4; ++k4) {
          const double a = xa[4 * k4];
          dmma(z00, z01, a, wb[4 * k4 * ldw]);
          if (two) dmma(z10, z11, a, wb[4 * k4 * ldw + 8]);
        }
        const int s = 8 * mb + g;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (h == 1 && !two) break;
          const int n = 8 * (nb0 + h) + 2 * q;
          const double za = (h ? z10 : z00) + W[T.b[l] + n], zb = (h ? z11 : z01) + W[T.b[l] + n + 1];
          if (l < 3) {
            double* xo = X + L.xo[l + 1] + s * L.ldx[l + 1] + n;
            double* eo = D + L.dd[l] + s * L.ldd[l] + n;
            // one transcendental per element: ELU = expm1(z), ELU' = exp(z) = expm1(z) + 1 (z <= 0)
            const double ea = expm1_neg(fmin(za, 0.0)), eb = expm1_neg(fmin(zb, 0.0));
            xo[0] = za > 0.0 ? za : ea;
            xo[1] = zb > 0.0 ? zb : eb;
            eo[0] = za > 0.0 ? 1.0 : ea + 1.0;  // elu_grad, ppo.cpp:12
            eo[1] = zb > 0.0 ? 1.0 : eb + 1.0;
          } else {
            double* zo = D + L.dd[3] + s * L.ldd[3] + n;  // trunk outputs, overwritten by the head
            zo[0] = za;
            zo[1] = zb;
          }
        }
      }
      __syncthreads();
    }
    // ---- loss head (ppo.cpp:92-126), warp = sample
    for (int s = warp; s < TILE; s += WARPS) {
      const int gi = base + s;
      const bool valid = gi < c1;
      const size_t row = valid ? (size_t)(L.idx ? L.idx[gi] : gi) : 0;
      double* d3 = D + L.dd[3] + s * L.ldd[3];
      if (trunk == 0) {
        const int A = P.act;
        double z0 = 0.0, z1 = 0.0, sd0 = 1.0, sd1 = 1.0, lp = 0.0;
        if (lane < A) {
          sd0 = lsd[lane];
          z0 = (L.act[row * A + lane] - d3[lane]) / sd0;
          lp += -0.5 * z0 * z0 - lstd[lane] - kLogSqrt2Pi;
        }
        if (lane + 32 < A) {
          sd1 = lsd[lane + 32];
          z1 = (L.act[row * A + lane + 32] - d3[lane + 32]) / sd1;
          lp += -0.5 * z1 * z1 - lstd[lane + 32] - kLogSqrt2Pi;
        }
        lp = warp_sum(lp);
        const double adv = valid ? L.adv[row] : 0.0;
        const double ratio = exp(lp - (valid ? L.old_logp[row] : 0.0));
        const double surr1 = ratio * adv;
        const double clipped = fmin(fmax(ratio, 1.0 - L.clip_eps), 1.0 + L.clip_eps) * adv;
        if (lane == 0 && valid) lsum += -fmin(surr1, clipped) * L.inv_n;
        const double g_r = surr1 <= clipped ? -adv * L.inv_n : 0.0;
        const bool on = valid && g_r != 0.0;
        const double g_logp = g_r * ratio;
        __syncwarp();
        if (lane < A) {
          d3[lane] = on ? g_logp * z0 / sd0 : 0.0;
          if (on) lsg0 += g_logp * (z0 * z0 - 1.0);
        }
        if (lane + 32 < A) {
          d3[lane + 32] = on ? g_logp * z1 / sd1 : 0.0;
          if (on) lsg1 += g_logp * (z1 * z1 - 1.0);
        }
      } else {
        const double verr = valid ? d3[0] - L.ret[row] : 0.0;
        __syncwarp();
        if (lane == 0) {
          if (valid) lsum += 0.5 * verr * verr * L.inv_n;
          d3[0] = valid ? L.value_coef * verr * L.inv_n : 0.0;
        }
      }
      // padded output rows carry a zero delta
      for (int j = N.out[3] + lane; j < T.Np[3]; j += 32) d3[j] = 0.0;
    }
    __syncthreads();
    // ---- backward: delta_{l-1} = (delta_l W_l) .* ELU'(z_{l-1}), unit = (mb, kb0, kb0 + 1)
    for (int l = 3; l > 0; --l) {
      const int nbK = T.Kp[l] / 8, units = 4 * ((nbK + 1) / 2);
      const double* Wl = W + T.w[l];
      const double* Dl = D + L.dd[l];
      const int ldw = T.ldw[l], ldd = L.ldd[l];
      for (int u = warp; u < units; u += WARPS) {
        const int mb = u & 3, kb0 = 2 * (u >> 2);
        const bool two = kb0 + 1 < nbK;
        double b00 = 0.0, b01 = 0.0, b10 = 0.0, b11 = 0.0;
        const double* da = Dl + (8 * mb + g) * ldd + q;
        const double* wb = Wl + (8 * kb0 + g) * ldw + q;
#pragma unroll 4
        for (int n4 = 0; n4 < T.Np[l] / 4; ++n4) {
          const double a = da[4 * n4];
          dmma(b00, b01, a, wb[4 * n4]);
          if (two) dmma(b10, b11, a, wb[4 * n4 + 8 * ldw]);
        }
        const int s = 8 * mb + g;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (h == 1 && !two) break;
          double* eo = D + L.dd[l - 1] + s * L.ldd[l - 1] + 8 * (kb0 + h) + 2 * q;
          eo[0] *= h ? b10 : b00;
          eo[1] *= h ? b11 : b01;
        }
      }
      __syncthreads();
    }
    // ---- gradient: G_l += delta_l^T X_l over the tile (8 k-steps of 4 samples); biases
#pragma unroll
    for (int r = 0; r < MAXB; ++r) {
      if (gblk[r] != 0xffffffffu) {
        const int l = gblk[r] >> 30;
        const double* da = D + (gblk[r] & 0x7fffu);
        const double* xb = X + ((gblk[r] >> 15) & 0x7fffu);
        const int sd = 4 * L.ldd[l], sx = 4 * L.ldx[l];
#pragma unroll
        for (int k4 = 0; k4 < TILE / 4; ++k4) dmma(acc[r][0], acc[r][1], da[k4 * sd], xb[k4 * sx]);
      }
    }
    if (bl >= 0) {
      const double* db = D + L.dd[bl] + bn;
      double v = 0.0;
#pragma unroll 8
      for (int s = 0; s < TILE; ++s) v += db[s * L.ldd[bl]];
      accB += v;
    }
    __syncthreads();
  }
  // ---- per-chunk partials
  double* part = L.part + (size_t)(trunk * L.nch + chunk) * L.part_stride;
#pragma unroll
  for (int r = 0; r < MAXB; ++r) {
    int j = warp + WARPS * r, l = 0;
    while (l < 4 && j >= T.nblk[l]) j -= T.nblk[l++];
    if (l < 4) {
      const int nbk = T.Kp[l] / 8, n = 8 * (j / nbk) + g, k = 8 * (j % nbk) + 2 * q;
      if (n < T.N[l]) {
        if (k < T.K[l]) part[T.wr[l] + k * T.N[l] + n] = acc[r][0];
        if (k + 1 < T.K[l]) part[T.wr[l] + (k + 1) * T.N[l] + n] = acc[r][1];
      }
    }
  }
  if (bl >= 0) part[T.br[bl] + bn] = accB;
  if (trunk == 0) {
    red[warp * MAXIO + lane] = lsg0;
    red[warp * MAXIO + lane + 32] = lsg1;
  }
  if (lane == 0) wred[warp] = lsum;
  __syncthreads();
  if (trunk == 0 && t < P.act) {
    double v = 0.0;
    for (int w = 0; w < WARPS; ++w) v += red[w * MAXIO + t];
    part[N.total + t] = v;
  }
  if (t == 0) {
    double v = 0.0;
    for (int w = 0; w < WARPS; ++w) v += wred[w];
    part[N.total + MAXIO] = v;
  }
}

// policy_forward (policy.cpp:85-102) on the same tensor-core layout: the forward phase of
// loss_kernel_mma alone, trunk outputs straight to global memory (mean n x act, value n).
__global__ void __launch_bounds__(THREADS, 1) forward_kernel_mma(const MmaParams L, double* mean, double* value) {
  extern __shared__ __align__(16) double sm[];
  const int trunk = blockIdx.y, chunk = blockIdx.x;
  if ((trunk == 0 && !mean) || (trunk == 1 && !value)) return;
  const PolicyParams& P = L.P;
  const Net& N = trunk == 0 ? P.pi : P.vf;
  const MmaTrunk& T = L.tr[trunk];
  double* W = sm;
  double* X = W + T.wtotal;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, g = lane >> 2, q = lane & 3;
  for (int e = t; e < T.wtotal + L.xtotal; e += THREADS) sm[e] = 0.0;
  __syncthreads();
  for (int l = 0; l < 4; ++l) {
    const int rows = N.out[l], cols = N.in[l];
    for (int e = t; e < rows * cols; e += THREADS) W[T.w[l] + (e / rows) * T.ldw[l] + e % rows] = L.w[N.w[l] + e];
    for (int i = t; i < rows; i += THREADS) W[T.b[l] + i] = L.w[N.b[l] + i];
  }
  const int c0 = chunk * L.chunk, c1 = min(L.n, c0 + L.chunk);
  __syncthreads();
  for (int base = c0; base < c1; base += TILE) {
    for (int e = t; e < TILE * P.obs; e += THREADS) {
      const int s = e / P.obs, k = e % P.obs, gi = base + s;
      X[L.xo[0] + s * L.ldx[0] + k] = gi < c1 ? L.obs[(size_t)gi * P.obs + k] : 0.0;
    }
    __syncthreads();
    for (int l = 0; l < 4; ++l) {
      const int nbN = T.Np[l] / 8, units = 4 * ((nbN + 1) / 2);
      const double* Wl = W + T.w[l];
      const double* Xl = X + L.xo[l];
      const int ldw = T.ldw[l], ldx = L.ldx[l];
      for (int u = warp; u < units; u += WARPS) {
        const int mb = u & 3, nb0 = 2 * (u >> 2);
        const bool two = nb0 + 1 < nbN;
        double z00 = 0.0, z01 = 0.0, z10 = 0.0, z11 = 0.0;
        const double* xa = Xl + (8 * mb + g) * ldx + q;
        const double* wb = Wl + q * ldw + 8 * nb0 + g;
#pragma unroll 4
        for (int k4 = 0; k4 < T.Kp[l] / 4; ++k4) {
          const double a = xa[4 * k4];
          dmma(z00, z01, a, wb[4 * k4 * ldw]);
          if (two) dmma(z10, z11, a, wb[4 * k4 * ldw + 8]);
        }
        const int s = 8 * mb + g;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (h == 1 && !two) break;
          const int n = 8 * (nb0 + h) + 2 * q;
          const double za = (h ? z10 : z00) + W[T.b[l] + n], zb = (h ? z11 : z01) + W[T.b[l] + n + 1];
          if (l < 3) {
            double* xo = X + L.xo[l + 1] + s * L.ldx[l + 1] + n;
            xo[0] = za > 0.0 ? za : expm1_neg(fmin(za, 0.0));
            xo[1] = zb > 0.0 ? zb : expm1_neg(fmin(zb, 0.0));
          } else if (base + s < c1) {
            const size_t row = (size_t)(base + s);
            if (trunk == 0) {
              if (n < P.act) mean[row * P.act + n] = za;
              if (n + 1 < P.act) mean[row * P.act + n + 1] = zb;
            } else if (n == 0) {
              value[row] = za;
            }
          }
        }
      }
      __syncthreads();
    }
  }
}

// Fixed-order sum of the chunk partials into the flatten_grads vector and the loss info.
// Block = 32 parameters (lane) x 8 warps, warp w summing chunks w, w + 8, ...; the eight
// warp sums are then added in warp order: a fixed order, and ~nch / 8 loads in flight per thread
// instead of a serial walk over all chunks.
constexpr int RED_PARAMS = 32, RED_WARPS = 8;
__global__ void __launch_bounds__(32 * RED_WARPS) reduce_kernel(const PolicyParams P, int nch, int part_stride,
                                                                 const double* __restrict__ part, double entropy_coef,
                                                                 double value_coef, const double* __restrict__ w,
                                                                 double* grads, rmpc_ppo_loss_info* info,
                                                                 double* sq) {
  __shared__ double sh[RED_WARPS][RED_PARAMS];
  const int np = P.total + P.act, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int p = blockIdx.x * RED_PARAMS + lane;
  double v = 0.0;
  if (p < np) {
    int tr = 0, e = p;
    if (p >= P.pi.total && p < P.total) {
      tr = 1;
      e = p - P.pi.total;
    } else if (p >= P.total) {
      e = P.pi.total + (p - P.total);
    }
    const double* q = part + (size_t)tr * nch * part_stride + e;
    for (int c = warp; c < nch; c += RED_WARPS) v += q[(size_t)c * part_stride];
  }
  sh[warp][lane] = v;
  __syncthreads();
  if (warp == 0) {
    double s = 0.0;
    if (p < np) {
      for (int k = 0; k < RED_WARPS; ++k) s += sh[k][lane];
      if (p >= P.total && entropy_coef != 0.0) s -= entropy_coef;
      if (grads) grads[p] = s;
    }
    if (sq) {  // this block's share of |g|^2 for the clip (fixed butterfly order)
      double q = p < np ? s * s : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
      if (lane == 0) sq[blockIdx.x] = q;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && info) {
    double sur = 0.0, vl = 0.0, ent = 0.0;
    for (int c = 0; c < nch; ++c) sur += part[(size_t)c * part_stride + P.pi.total + MAXIO];
    for (int c = 0; c < nch; ++c) vl += part[(size_t)(nch + c) * part_stride + P.vf.total + MAXIO];
    for (int j = 0; j < P.act; ++j) ent += w[P.total + j] + kLogSqrt2Pi + 0.5;
    info->surrogate = sur;
    info->value_loss = vl;
    info->entropy = ent;
    info->total = sur + value_coef * vl - entropy_coef * ent;
  }
}

// gae_advantages (ppo.cpp:28-45): one thread per env, the backward recursion over the steps.
__global__ void gae_kernel(int T, int E, const double* __restrict__ rew, const double* __restrict__ val,
                           const double* __restrict__ done, const double* __restrict__ boot, double gamma,
                           double lam, double* adv, double* ret) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  double running = 0.0;
  for (int t = T - 1; t >= 0; --t) {
    const size_t k = (size_t)t * E + e;
    const double not_done = 1.0 - done[k];
    const double next_value = t == T - 1 ? boot[e] : val[k + E];
    const double delta = rew[k] + gamma * next_value * not_done - val[k];
    running = delta + gamma * lam * not_done * running;
    adv[k] = running;
    ret[k] = running + val[k];
  }
}

constexpr int RED_THREADS = 1024;

// Fixed-order block sum (every thread gets the total).
__device__ double block_sum(double v, double* sh) {
  const int t = threadIdx.x;
  sh[t] = v;
  __syncthreads();
  for (int o = RED_THREADS / 2; o > 0; o >>= 1) {
    if (t < o) sh[t] += sh[t + o];
    __syncthreads();
  }
  const double r = sh[0];
  __syncthreads();
  return r;
}

// Advantage normalisation of ppo_update (ppo.cpp:201-204), one block.
__global__ void __launch_bounds__(RED_THREADS) normalize_kernel(int N, double* adv) {
  __shared__ double sh[RED_THREADS];
  double s = 0.0;
  for (int k = threadIdx.x; k < N; k += RED_THREADS) s += adv[k];
  const double mean = block_sum(s, sh) / N;
  double q = 0.0;
  for (int k = threadIdx.x; k < N; k += RED_THREADS) q += (adv[k] - mean) * (adv[k] - mean);
  const double var = block_sum(q, sh) / N;
  const double inv_std = 1.0 / sqrt(var + 1e-8);
  for (int k = threadIdx.x; k < N; k += RED_THREADS) adv[k] = (adv[k] - mean) * inv_std;
}

// Gradient-norm clip (ppo.cpp:252-256) + AdamOptimizer::step (ppo.cpp:179-193), one thread per
// parameter; every block sums the reduce kernel's |g|^2 partials in the same fixed order.
constexpr int ADAM_THREADS = 256;
__global__ void __launch_bounds__(ADAM_THREADS) adam_kernel(int np, const double* __restrict__ g,
                                                            const double* __restrict__ sq, int nsq, double* m,
                                                            double* v, double* w, double max_norm, double lr,
                                                            double b1, double b2, double eps, double bc1,
                                                            double bc2) {
  __shared__ double sh[ADAM_THREADS];
  const int t = threadIdx.x;
  double q = 0.0;
  for (int k = t; k < nsq; k += ADAM_THREADS) q += sq[k];
  sh[t] = q;
  __syncthreads();
  for (int o = ADAM_THREADS / 2; o > 0; o >>= 1) {
    if (t < o) sh[t] += sh[t + o];
    __syncthreads();
  }
  const double norm = sqrt(sh[0]);
  const bool clip = max_norm > 0.0 && norm > max_norm;
  const double scale = clip ? max_norm / norm : 1.0;
  const int k = blockIdx.x * ADAM_THREADS + t;
  if (k < np) {
    const double gk = clip ? g[k] * scale : g[k];
    const double mk = b1 * m[k] + (1.0 - b1) * gk;
    const double vk = b2 * v[k] + (1.0 - b2) * (gk * gk);
    m[k] = mk;
    v[k] = vk;
    w[k] -= lr * (mk / bc1) / (sqrt(vk / bc2) + eps);
  }
}

TrunkSm trunk_sm(const Net& N) {
  TrunkSm S{};
  int off = 0;
  for (int l = 0; l < 4; ++l) {
    S.ld[l] = N.out[l] | 1;
    S.w[l] = off;
    off += N.in[l] * S.ld[l];
    S.b[l] = off;
    off += N.out[l];
    S.wr[l] = N.w[l] - N.w[0];
    S.br[l] = N.b[l] - N.w[0];
  }
  S.wtotal = (off + 1) & ~1;
  return S;
}

int ld4(int n) { return n + ((4 - n % 16) + 16) % 16; }  // >= n, = 4 mod 16
int up8(int n) { return (n + 7) & ~7; }

// The tensor-core layout; false if the shapes exceed it (then the CUDA-core kernel runs).
bool mma_layout(const PolicyParams& P, MmaParams& M, int& smem) {
  M.P = P;
  int xo = 0, dd = 0;
  for (int l = 0; l < 4; ++l) {
    const int kp = l == 0 ? up8(P.obs) : up8(P.hidden), np = l < 3 ? up8(P.hidden) : up8(std::max(P.act, 1));
    M.ldx[l] = ld4(kp);
    M.xo[l] = xo;
    xo += TILE * M.ldx[l];
    M.ldd[l] = ld4(np);
    M.dd[l] = dd;
    dd += TILE * M.ldd[l];
  }
  M.xtotal = xo;
  M.dtotal = dd;
  int wmax = 0, blocks = 0;
  for (int tr = 0; tr < 2; ++tr) {
    const Net& N = tr == 0 ? P.pi : P.vf;
    MmaTrunk& T = M.tr[tr];
    int off = 0, nb = 0;
    for (int l = 0; l < 4; ++l) {
      T.K[l] = N.in[l];
      T.N[l] = N.out[l];
      T.Kp[l] = up8(N.in[l]);
      T.Np[l] = l < 3 ? up8(N.out[l]) : up8(std::max(P.act, 1));  // both trunks share delta_3's shape
      T.ldw[l] = ld4(T.Np[l]);
      T.w[l] = off;
      off += T.Kp[l] * T.ldw[l];
      T.b[l] = off;
      off += T.Np[l];
      T.wr[l] = N.w[l] - N.w[0];
      T.br[l] = N.b[l] - N.w[0];
      T.nblk[l] = (T.Np[l] / 8) * (T.Kp[l] / 8);
      nb += T.nblk[l];
    }
    T.wtotal = (off + 1) & ~1;
    wmax = std::max(wmax, T.wtotal);
    blocks = std::max(blocks, nb);
  }
  smem = (int)sizeof(double) * (wmax + M.xtotal + M.dtotal);
  return P.hidden <= MAXH && P.obs <= MAXIO && P.act <= MAXIO && blocks <= WARPS * MAXB &&
         smem <= 227 * 1024 - 1024;
}

// One ppo_loss over n samples (optionally gathered through idx) into grads / info.
int launch_loss(rmpc_policy* p, int n, const double* obs, const double* act, const double* old_logp,
                const double* adv, const double* ret, const int32_t* idx, const rmpc_ppo_config& cfg, double* grads,
                rmpc_ppo_loss_info* info, cudaStream_t st, double* sq = nullptr) {
  const PolicyParams& P = p->P;
  LossParams L{};
  L.P = P;
  L.ts[0] = trunk_sm(P.pi);
  L.ts[1] = trunk_sm(P.vf);
  L.n = n;
  L.nch = std::max(1, std::min(p->sms / 2, (n + TILE - 1) / TILE));
  L.chunk = (n + L.nch - 1) / L.nch;
  const int ob2 = (P.obs + 1) & ~1, h2 = (P.hidden + 1) & ~1;
  L.pst = ob2 + 3 * h2 + 2;
  L.dst = 3 * h2 + ((P.act + 1) & ~1);
  L.ost = (P.act + 1) & ~1;
  L.part_stride = std::max(P.pi.total, P.vf.total) + 2 * MAXIO;
  L.clip_eps = cfg.clip_eps;
  L.value_coef = cfg.value_coef;
  L.inv_n = 1.0 / n;
  L.w = p->d_w;
  L.obs = obs;
  L.act = act;
  L.old_logp = old_logp;
  L.adv = adv;
  L.ret = ret;
  L.idx = idx;
  const size_t need = (size_t)2 * L.nch * L.part_stride;
  if (need > p->part_cap) {
    cudaFree(p->d_part);
    p->d_part = nullptr;
    p->part_cap = 0;
    if (cudaMalloc(&p->d_part, need * sizeof(double)) != cudaSuccess) return RMPC_ERR_CUDA;
    p->part_cap = need;
  }
  L.part = p->d_part;
  MmaParams M{};
  int msmem = 0;
  if (mma_layout(P, M, msmem)) {  // FP64 tensor cores
    M.n = L.n;
    M.chunk = L.chunk;
    M.nch = L.nch;
    M.part_stride = L.part_stride;
    M.clip_eps = L.clip_eps;
    M.value_coef = L.value_coef;
    M.inv_n = L.inv_n;
    M.w = L.w;
    M.obs = obs;
    M.act = act;
    M.old_logp = old_logp;
    M.adv = adv;
    M.ret = ret;
    M.idx = idx;
    M.part = L.part;
    if (cudaFuncSetAttribute(loss_kernel_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, msmem) != cudaSuccess)
      return RMPC_ERR_CUDA;
    loss_kernel_mma<<<dim3(L.nch, 2), THREADS, msmem, st>>>(M);
  } else {  // CUDA cores (shapes beyond the tensor-core layout): 32- or 16-sample tiles
    const int wmax = std::max(L.ts[0].wtotal, L.ts[1].wtotal);
    auto smem_for = [&](int tl) { return (int)sizeof(double) * (wmax + tl * (L.pst + L.dst + L.ost)); };
    const int limit = 227 * 1024 - 1024;
    if (smem_for(32) <= limit) {
      if (cudaFuncSetAttribute(loss_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_for(32)) !=
          cudaSuccess)
        return RMPC_ERR_CUDA;
      loss_kernel<32><<<dim3(L.nch, 2), THREADS, smem_for(32), st>>>(L);
    } else if (smem_for(16) <= limit) {
      if (cudaFuncSetAttribute(loss_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_for(16)) !=
          cudaSuccess)
        return RMPC_ERR_CUDA;
      loss_kernel<16><<<dim3(L.nch, 2), THREADS, smem_for(16), st>>>(L);
    } else {
      return RMPC_ERR_STRUCTURAL;
    }
  }
  const int np = P.total + P.act;
  reduce_kernel<<<(np + RED_PARAMS - 1) / RED_PARAMS, 32 * RED_WARPS, 0, st>>>(
      P, L.nch, L.part_stride, L.part, cfg.entropy_coef, cfg.value_coef, p->d_w, grads, info, sq);
  return cudaGetLastError() == cudaSuccess ? RMPC_OK : RMPC_ERR_CUDA;
}

// policy_forward on the tensor cores; false when the shapes exceed the layout (the caller then
// runs the CUDA-core kernel of rmpc_policy.cu).
bool launch_forward_mma(rmpc_policy* p, int n, const double* obs, double* mean, double* value, cudaStream_t st,
                        int* rc) {
  MmaParams M{};
  int smem = 0;
  if (!mma_layout(p->P, M, smem)) return false;
  const int wmax = std::max(M.tr[0].wtotal, M.tr[1].wtotal);
  smem = (int)sizeof(double) * (wmax + M.xtotal);
  M.n = n;
  M.nch = std::max(1, std::min(p->sms / 2, (n + TILE - 1) / TILE));
  M.chunk = (n + M.nch - 1) / M.nch;
  M.w = p->d_w;
  M.obs = obs;
  if (cudaFuncSetAttribute(forward_kernel_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) {
    *rc = RMPC_ERR_CUDA;
    return true;
  }
  forward_kernel_mma<<<dim3(M.nch, 2), THREADS, smem, st>>>(M, mean, value);
  *rc = cudaGetLastError() == cudaSuccess ? RMPC_OK : RMPC_ERR_CUDA;
  return true;
}

// xoshiro256++ (rng.hpp:15-43): seeding and uniform_int for the minibatch shuffles.
uint64_t splitmix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
uint64_t next_u64(uint64_t s[4]) {
  const uint64_t r = rotl(s[0] + s[3], 23) + s[0];
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl(s[3], 45);
  return r;
}

}  // namespace rmpc_ppo_dev

struct rmpc_adam {
  rmpc_policy* policy = nullptr;
  double lr = 3e-4, beta1 = 0.9, beta2 = 0.999, eps = 1e-8;
  int t = 0;
  double* d_m = nullptr;
  double* d_v = nullptr;
  double* d_sq = nullptr;  // per reduce block |g|^2 partials
  // ppo_update workspace
  double* d_adv = nullptr;
  double* d_ret = nullptr;
  int32_t* d_order = nullptr;
  rmpc_ppo_loss_info* d_info = nullptr;
  int32_t* h_order = nullptr;  // pinned
  size_t adv_cap = 0, ret_cap = 0, order_cap = 0, info_cap = 0;
};

extern "C" {

void rmpc_ppo_config_default(rmpc_ppo_config* c) {  // PpoConfig, ppo.hpp:14-24
  if (!c) return;
  c->gamma = 0.99;
  c->lam_gae = 0.95;
  c->clip_eps = 0.2;
  c->epochs = 4;
  c->minibatches = 4;
  c->lr = 3e-4;
  c->entropy_coef = 0.0;
  c->value_coef = 0.5;
  c->max_grad_norm = 1.0;
}

void rmpc_rng_seed(uint64_t seed, uint64_t stream, uint64_t state[4]) {  // Rng(seed, stream)
  uint64_t x = seed ^ rmpc_ppo_dev::splitmix(stream + 0x9e3779b97f4a7c15ULL);
  for (int k = 0; k < 4; ++k) {
    x += 0x9e3779b97f4a7c15ULL;
    state[k] = rmpc_ppo_dev::splitmix(x);
  }
}

int32_t rmpc_ppo_loss_device(rmpc_policy* p, int32_t n, const double* obs, const double* act, const double* old_logp,
                             const double* adv, const double* ret, const rmpc_ppo_config* cfg, double* grads,
                             rmpc_ppo_loss_info* info, void* stream) {
  if (!p || !cfg || n < 0) return RMPC_ERR_INVALID_ARG;
  if (n == 0) return RMPC_ERR_STRUCTURAL;  // ppo_loss: empty batch (ppo.cpp:82)
  if (!obs || !act || !old_logp || !adv || !ret) return RMPC_ERR_INVALID_ARG;
  if (cudaSetDevice(p->device) != cudaSuccess) return RMPC_ERR_CUDA;
  return rmpc_ppo_dev::launch_loss(p, n, obs, act, old_logp, adv, ret, nullptr, *cfg, grads, info,
                                   stream ? (cudaStream_t)stream : cudaStreamLegacy);
}

int32_t rmpc_gae_device(int32_t T, int32_t E, const double* rew, const double* val, const double* done,
                        const double* boot, double gamma, double lam, double* adv, double* ret, void* stream) {
  if (T < 0 || E < 0 || ((size_t)T * E > 0 && (!rew || !val || !done || !boot || !adv || !ret)))
    return RMPC_ERR_INVALID_ARG;
  if ((size_t)T * E == 0) return RMPC_OK;
  rmpc_ppo_dev::gae_kernel<<<(E + 127) / 128, 128, 0, stream ? (cudaStream_t)stream : cudaStreamLegacy>>>(
      T, E, rew, val, done, boot, gamma, lam, adv, ret);
  return cudaGetLastError() == cudaSuccess ? RMPC_OK : RMPC_ERR_CUDA;
}

int32_t rmpc_adam_create(rmpc_policy* p, double lr, rmpc_adam** out) {
  if (!p || !out) return RMPC_ERR_INVALID_ARG;
  *out = nullptr;
  if (cudaSetDevice(p->device) != cudaSuccess) return RMPC_ERR_CUDA;
  rmpc_adam* a = new (std::nothrow) rmpc_adam;
  if (!a) return RMPC_ERR_CUDA;
  a->policy = p;
  a->lr = lr;
  const size_t np = (size_t)(p->P.total + p->P.act);
  if (cudaMalloc(&a->d_m, np * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&a->d_v, np * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&a->d_sq, ((np + rmpc_ppo_dev::RED_PARAMS - 1) / rmpc_ppo_dev::RED_PARAMS) * sizeof(double)) !=
          cudaSuccess ||
      cudaMemset(a->d_m, 0, np * sizeof(double)) != cudaSuccess ||
      cudaMemset(a->d_v, 0, np * sizeof(double)) != cudaSuccess) {
    cudaFree(a->d_m);
    cudaFree(a->d_v);
    cudaFree(a->d_sq);
    delete a;
    return RMPC_ERR_CUDA;
  }
  *out = a;
  return RMPC_OK;
}

void rmpc_adam_destroy(rmpc_adam* a) {
  if (!a) return;
  cudaSetDevice(a->policy->device);
  cudaFree(a->d_m);
  cudaFree(a->d_v);
  cudaFree(a->d_sq);
  cudaFree(a->d_adv);
  cudaFree(a->d_ret);
  cudaFree(a->d_order);
  cudaFree(a->d_info);
  cudaFreeHost(a->h_order);
  delete a;
}

int32_t rmpc_ppo_update_device(rmpc_policy* p, rmpc_adam* a, int32_t T, int32_t E, const double* obs,
                               const double* act, const double* logp, const double* values, const double* rewards,
                               const double* dones, const double* boot, const rmpc_ppo_config* cfg,
                               uint64_t rng[4], rmpc_ppo_update_stats* stats, void* stream) {
  using namespace rmpc_ppo_dev;
  if (!p || !a || a->policy != p || !cfg || !rng || !stats || T < 1 || E < 1) return RMPC_ERR_INVALID_ARG;
  if (!obs || !act || !logp || !values || !rewards || !dones || !boot) return RMPC_ERR_INVALID_ARG;
  if (cudaSetDevice(p->device) != cudaSuccess) return RMPC_ERR_CUDA;
  const cudaStream_t st = stream ? (cudaStream_t)stream : cudaStreamLegacy;
  const int N = T * E;
  const int epochs = std::max(0, cfg->epochs), mbc = std::max(1, cfg->minibatches);
  const int np = p->P.total + p->P.act;
  const int nsq = (np + RED_PARAMS - 1) / RED_PARAMS;
  auto grow = [](auto*& ptr, size_t& cap, size_t need, size_t elem) {
    if (need <= cap) return true;
    cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
    if (cudaMalloc(&ptr, need * elem) != cudaSuccess) return false;
    cap = need;
    return true;
  };
  if (!grow(a->d_adv, a->adv_cap, (size_t)N, sizeof(double)) || !grow(a->d_ret, a->ret_cap, (size_t)N, sizeof(double)))
    return RMPC_ERR_CUDA;
  const size_t norder = (size_t)std::max(epochs, 1) * N;
  if (norder > a->order_cap) {
    cudaFree(a->d_order);
    cudaFreeHost(a->h_order);
    a->d_order = nullptr;
    a->h_order = nullptr;
    a->order_cap = 0;
    if (cudaMalloc(&a->d_order, norder * sizeof(int32_t)) != cudaSuccess ||
        cudaMallocHost(&a->h_order, norder * sizeof(int32_t)) != cudaSuccess)
      return RMPC_ERR_CUDA;
    a->order_cap = norder;
  }
  if (!grow(a->d_info, a->info_cap, (size_t)std::max(epochs * mbc, 1), sizeof(rmpc_ppo_loss_info)))
    return RMPC_ERR_CUDA;
  if (!p->d_grads && cudaMalloc(&p->d_grads, np * sizeof(double)) != cudaSuccess) return RMPC_ERR_CUDA;
  cudaStreamSynchronize(st);  // h_order may still feed a previous call's copy
  gae_kernel<<<(E + 127) / 128, 128, 0, st>>>(T, E, rewards, values, dones, boot, cfg->gamma, cfg->lam_gae, a->d_adv,
                                               a->d_ret);
  normalize_kernel<<<1, RED_THREADS, 0, st>>>(N, a->d_adv);
  // per epoch: the host draws the shuffle (the Rng advances exactly as the reference's loop)
  // while the device still runs the previous epoch's minibatches
  std::vector<int32_t> order(N);
  for (int k = 0; k < N; ++k) order[k] = k;
  const int mb = (N + mbc - 1) / mbc;
  int count = 0;
  for (int ep = 0; ep < epochs; ++ep) {
    for (int k = N - 1; k > 0; --k) std::swap(order[k], order[next_u64(rng) % (uint64_t)(k + 1)]);
    int32_t* h = a->h_order + (size_t)ep * N;
    std::copy(order.begin(), order.end(), h);
    if (cudaMemcpyAsync(a->d_order + (size_t)ep * N, h, (size_t)N * sizeof(int32_t), cudaMemcpyHostToDevice, st) !=
        cudaSuccess)
      return RMPC_ERR_CUDA;
    for (int b = 0; b < mbc; ++b) {
      const int lo = b * mb, hi = std::min(N, lo + mb);
      if (lo >= hi) continue;
      const int rc = launch_loss(p, hi - lo, obs, act, logp, a->d_adv, a->d_ret, a->d_order + (size_t)ep * N + lo, *cfg,
                                 p->d_grads, a->d_info + count, st, a->d_sq);
      if (rc != RMPC_OK) return rc;
      ++a->t;
      const double bc1 = 1.0 - std::pow(a->beta1, a->t), bc2 = 1.0 - std::pow(a->beta2, a->t);
      adam_kernel<<<(np + ADAM_THREADS - 1) / ADAM_THREADS, ADAM_THREADS, 0, st>>>(
          np, p->d_grads, a->d_sq, nsq, a->d_m, a->d_v, p->d_w, cfg->max_grad_norm, a->lr, a->beta1, a->beta2, a->eps,
          bc1, bc2);
      ++count;
    }
  }
  std::vector<rmpc_ppo_loss_info> infos(std::max(count, 1));
  if (count > 0 && cudaMemcpyAsync(infos.data(), a->d_info, count * sizeof(rmpc_ppo_loss_info),
                                   cudaMemcpyDeviceToHost, st) != cudaSuccess)
    return RMPC_ERR_CUDA;
  if (cudaStreamSynchronize(st) != cudaSuccess || cudaGetLastError() != cudaSuccess) return RMPC_ERR_CUDA;
  rmpc_ppo_update_stats s{0.0, 0.0, 0.0, 0.0};
  for (int k = 0; k < count; ++k) {
    s.loss += infos[k].total;
    s.surrogate += infos[k].surrogate;
    s.value_loss += infos[k].value_loss;
    s.entropy = infos[k].entropy;
  }
  if (count > 0) {
    s.loss /= count;
    s.surrogate /= count;
    s.value_loss /= count;
  }
  *stats = s;
  return RMPC_OK;
}

}  // extern "C"
