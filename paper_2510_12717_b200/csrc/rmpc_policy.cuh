// rmpc_policy.cuh — the residual policy's device-side shape and handle, shared by the forward
// (rmpc_policy.cu) and the PPO batch (rmpc_ppo.cu).  Parameters live on the device as one FP64
// vector in flatten_policy order (/root/reference/proj/src/ppo.cpp:144-153): per trunk and
// layer W (out x in, column-major as Eigen stores it) then b; pi, then value, then log_std.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/rmpc_b200_env.h"

namespace rmpc_policy_dev {

constexpr int MAXH = 64, MAXIO = 64;  // hidden / obs / act limits (one neuron pair per lane)

struct Net {
  int in[4], out[4];  // layer shapes
  int w[4], b[4];     // offsets (doubles) into the parameter vector
  int total;          // doubles of this trunk
};

struct PolicyParams {
  int obs, act, hidden;
  int total;  // doubles of both trunks (log_std excluded); log_std starts here
  Net pi, vf;
};

// init_policy's trunk shapes (policy.cpp:57-83): obs -> hidden -> hidden -> hidden -> out.
inline PolicyParams policy_shape(int obs, int act, int hidden) {
  PolicyParams P{};
  P.obs = obs;
  P.act = act;
  P.hidden = hidden;
  int off = 0;
  auto net = [&](Net& N, int out_dim) {
    const int sizes[5] = {obs, hidden, hidden, hidden, out_dim};
    const int base = off;
    for (int l = 0; l < 4; ++l) {
      N.in[l] = sizes[l];
      N.out[l] = sizes[l + 1];
      N.w[l] = off;
      off += sizes[l] * sizes[l + 1];
      N.b[l] = off;
      off += sizes[l + 1];
    }
    N.total = off - base;
  };
  net(P.pi, act);
  net(P.vf, 1);
  P.total = off;
  return P;
}

}  // namespace rmpc_policy_dev

struct rmpc_policy;
namespace rmpc_ppo_dev {
// policy_forward on the FP64 tensor cores (rmpc_ppo.cu); false if the shapes exceed its layout.
bool launch_forward_mma(rmpc_policy* p, int n, const double* obs, double* mean, double* value, cudaStream_t st,
                        int* rc);
}  // namespace rmpc_ppo_dev

struct rmpc_policy {
  int device = 0;
  rmpc_policy_dev::PolicyParams P{};
  double* d_w = nullptr;  // P.total + act doubles (log_std last)
  int smem = 0, grid = 0, sms = 148;
  // PPO workspace (rmpc_ppo.cu), grown on demand
  double* d_part = nullptr;
  size_t part_cap = 0;  // doubles
  double* d_grads = nullptr;
};
