// rmpc_policy.cu — the residual policy forward on sm_100a:
// policy_forward (/root/reference/proj/src/policy.cpp:85-102) = mlp_forward (policy.cpp:15-31)
// of the pi and value trunks, FP64 like the reference.
//
// The default path is forward_kernel_mma in rmpc_ppo.cu: the PPO loss kernel's forward phase on
// the FP64 tensor cores (mma.sync m8n8k4 f64; TF32/BF16 would miss the FP64 reference by 1e-3).
// This file keeps the policy handle and the CUDA-core fallback for shapes beyond that layout:
// one warp per agent, lane j owns output neurons j and j + 32 of every layer, all weights of both
// trunks resident in shared memory as Eigen stores them (column-major, so a layer's column is
// 64 consecutive doubles: conflict-free 8-byte loads across the warp), the layer input staged
// per warp in shared memory and broadcast.  Persistent CTAs of 8 warps stride over the agents.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <new>
#include <vector>

#include "rmpc_policy.cuh"

namespace rmpc_policy_dev {

constexpr int WARPS = 8;

// One trunk for the agent held by this warp; x (per-warp smem, MAXIO) holds the input and is
// overwritten layer by layer.  Returns, in lane j, outputs j (o0) and j + 32 (o1).
__device__ __forceinline__ void trunk(const Net& N, const double* W, double* x, int lane, double& o0,
                                      double& o1) {
#pragma unroll 1
  for (int l = 0; l < 4; ++l) {
    const int ni = N.in[l], no = N.out[l];
    const double* Wl = W + N.w[l];
    double a0 = lane < no ? W[N.b[l] + lane] : 0.0;
    double a1 = lane + 32 < no ? W[N.b[l] + lane + 32] : 0.0;
    const int j0 = lane < no ? lane : 0, j1 = lane + 32 < no ? lane + 32 : 0;
#pragma unroll 4
    for (int k = 0; k < ni; ++k) {  // column k of W (column-major, out rows)
      const double xk = x[k];
      a0 = fma(Wl[k * no + j0], xk, a0);
      a1 = fma(Wl[k * no + j1], xk, a1);
    }
    if (l < 3) {  // ELU on the hidden layers (policy.cpp:13)
      a0 = a0 > 0.0 ? a0 : expm1(a0);
      a1 = a1 > 0.0 ? a1 : expm1(a1);
    }
    __syncwarp();
    if (lane < no) x[lane] = a0;
    if (lane + 32 < no) x[lane + 32] = a1;
    __syncwarp();
    o0 = a0;
    o1 = a1;
  }
}

__global__ void __launch_bounds__(32 * WARPS) forward_kernel(const PolicyParams P, const double* __restrict__ gw,
                                                             int n, const double* __restrict__ obs,
                                                             double* mean, double* value) {
  extern __shared__ __align__(16) double sw[];
  double* W = sw;                        // both trunks, P.total doubles
  double* xs = sw + P.total;             // per warp: MAXIO input staging
  for (int k = threadIdx.x; k < P.total; k += blockDim.x) W[k] = gw[k];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* x = xs + warp * MAXIO;
  for (int a = blockIdx.x * WARPS + warp; a < n; a += gridDim.x * WARPS) {
    const double* o = obs + (size_t)a * P.obs;
    double o0, o1;
    if (mean) {
      for (int k = lane; k < P.obs; k += 32) x[k] = o[k];
      __syncwarp();
      trunk(P.pi, W, x, lane, o0, o1);
      if (lane < P.act) mean[(size_t)a * P.act + lane] = o0;
    }
    if (value) {
      __syncwarp();
      for (int k = lane; k < P.obs; k += 32) x[k] = o[k];
      __syncwarp();
      trunk(P.vf, W, x, lane, o0, o1);
      if (lane == 0) value[a] = o0;
    }
    __syncwarp();
  }
}

}  // namespace rmpc_policy_dev

extern "C" {

int32_t rmpc_policy_create(int32_t obs_dim, int32_t act_dim, int32_t hidden, const double* params,
                           int32_t n_params, int32_t device, rmpc_policy** out) {
  using namespace rmpc_policy_dev;
  if (!out || !params) return RMPC_ERR_INVALID_ARG;
  *out = nullptr;
  if (obs_dim < 1 || obs_dim > MAXIO || act_dim < 1 || act_dim > MAXH || hidden < 1 || hidden > MAXH)
    return RMPC_ERR_STRUCTURAL;
  const rmpc_policy_dev::PolicyParams P = rmpc_policy_dev::policy_shape(obs_dim, act_dim, hidden);
  if (n_params != P.total + act_dim) return RMPC_ERR_STRUCTURAL;  // + log_std
  if (cudaSetDevice(device) != cudaSuccess) return RMPC_ERR_CUDA;
  rmpc_policy* p = new (std::nothrow) rmpc_policy;
  if (!p) return RMPC_ERR_CUDA;
  p->device = device;
  p->P = P;
  p->smem = (P.total + WARPS * MAXIO) * (int)sizeof(double);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  p->grid = sms;
  p->sms = sms;
  if (cudaMalloc(&p->d_w, (P.total + act_dim) * sizeof(double)) != cudaSuccess ||
      cudaMemcpy(p->d_w, params, (P.total + act_dim) * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaFuncSetAttribute(forward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, p->smem) !=
          cudaSuccess) {
    cudaFree(p->d_w);
    delete p;
    return RMPC_ERR_CUDA;
  }
  *out = p;
  return RMPC_OK;
}

void rmpc_policy_destroy(rmpc_policy* p) {
  if (!p) return;
  cudaSetDevice(p->device);
  cudaFree(p->d_w);
  cudaFree(p->d_part);
  cudaFree(p->d_grads);
  delete p;
}

int32_t rmpc_policy_num_params(const rmpc_policy* p) { return p ? p->P.total + p->P.act : -1; }

int32_t rmpc_policy_get_params(rmpc_policy* p, double* params, int32_t n_params) {
  if (!p || !params) return RMPC_ERR_INVALID_ARG;
  if (n_params != p->P.total + p->P.act) return RMPC_ERR_STRUCTURAL;
  if (cudaSetDevice(p->device) != cudaSuccess ||
      cudaMemcpy(params, p->d_w, n_params * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
    return RMPC_ERR_CUDA;
  return RMPC_OK;
}

int32_t rmpc_policy_set_params(rmpc_policy* p, const double* params, int32_t n_params) {
  if (!p || !params) return RMPC_ERR_INVALID_ARG;
  if (n_params != p->P.total + p->P.act) return RMPC_ERR_STRUCTURAL;
  if (cudaSetDevice(p->device) != cudaSuccess ||
      cudaMemcpy(p->d_w, params, n_params * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess)
    return RMPC_ERR_CUDA;
  return RMPC_OK;
}

int32_t rmpc_policy_forward_device(rmpc_policy* p, int32_t n, const double* obs, double* mean, double* value,
                                   void* stream) {
  if (!p || n < 0 || (n > 0 && !obs)) return RMPC_ERR_INVALID_ARG;
  if (n == 0 || (!mean && !value)) return RMPC_OK;
  if (cudaSetDevice(p->device) != cudaSuccess) return RMPC_ERR_CUDA;
  int rc = RMPC_OK;
  if (rmpc_ppo_dev::launch_forward_mma(p, n, obs, mean, value, stream ? (cudaStream_t)stream : cudaStreamLegacy, &rc))
    return rc;
  const int need = (n + rmpc_policy_dev::WARPS - 1) / rmpc_policy_dev::WARPS;
  rmpc_policy_dev::forward_kernel<<<need < p->grid ? need : p->grid, 32 * rmpc_policy_dev::WARPS, p->smem,
                                    stream ? (cudaStream_t)stream : cudaStreamLegacy>>>(p->P, p->d_w, n, obs,
                                                                                         mean, value);
  return cudaGetLastError() == cudaSuccess ? RMPC_OK : RMPC_ERR_CUDA;
}

}  // extern "C"
