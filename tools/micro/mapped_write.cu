// Mapped-host write throughput for z*-shaped outputs (the end-to-end tail of a squad solve):
// A: one 26-float row (104 B) per warp store, as the squad finish writes z* node by node
// B: an agent's 1040 B as float2 words, lanes on consecutive words (the copy-out kernel)
// C: B with float4 words;  D: the copy engine (cudaMemcpyAsync D2H of the same bytes)
#include <cstdio>
#include <cuda_runtime.h>
constexpr int NV = 26, NT = 10;
__global__ void rows(float* dst, const float* src, int agents) {
  const int lane = threadIdx.x & 31, w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int a = w; a < agents; a += nw)
    for (int i = 0; i < NT; ++i)
      if (lane < NV) dst[((size_t)a * NT + i) * NV + lane] = src[((size_t)a * NT + i) * NV + lane];
}
__global__ void words2(float* dst, const float* src, int agents) {
  const int lane = threadIdx.x & 31, w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int a = w; a < agents; a += nw) {
    const float2* s = reinterpret_cast<const float2*>(src + (size_t)a * NT * NV);
    float2* d = reinterpret_cast<float2*>(dst + (size_t)a * NT * NV);
    for (int k = lane; k < NT * NV / 2; k += 32) d[k] = s[k];
  }
}
__global__ void words4(float* dst, const float* src, int agents) {
  const int lane = threadIdx.x & 31, w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int a = w; a < agents; a += nw) {
    const float4* s = reinterpret_cast<const float4*>(src + (size_t)a * NT * NV);
    float4* d = reinterpret_cast<float4*>(dst + (size_t)a * NT * NV);
    for (int k = lane; k < NT * NV / 4; k += 32) d[k] = s[k];
  }
}
int main() {
  const int agents_list[3] = {6912, 9472, 16384};
  float *h, *dh, *d;
  const size_t maxb = (size_t)16384 * NT * NV * 4;
  cudaHostAlloc(&h, maxb, cudaHostAllocMapped);
  cudaHostGetDevicePointer(&dh, h, 0);
  cudaMalloc(&d, maxb);
  cudaMemset(d, 0, maxb);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int ai = 0; ai < 3; ++ai) {
    const int agents = agents_list[ai];
    const size_t bytes = (size_t)agents * NT * NV * 4;
    for (int v = 0; v < 4; ++v) {
      for (int grid : {108, 148, 296}) {
        if (v == 3 && grid != 148) continue;
        float best = 1e9f;
        for (int r = 0; r < 6; ++r) {
          cudaEventRecord(e0);
          if (v == 0) rows<<<grid, 128>>>(dh, d, agents);
          if (v == 1) words2<<<grid, 128>>>(dh, d, agents);
          if (v == 2) words4<<<grid, 128>>>(dh, d, agents);
          if (v == 3) cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          if (r > 0 && ms < best) best = ms;
        }
        const char* nm[4] = {"rows104", "float2", "float4", "memcpy"};
        printf("agents %5d %-8s grid %3d: %.3f ms  %.1f GB/s\n", agents, nm[v], grid, best, bytes / best / 1e6);
      }
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
