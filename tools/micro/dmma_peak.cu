// FP64 tensor-core (mma.sync m8n8k4 f64) vs FP64 FMA throughput on this GPU.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_peak dmma_peak.cu && ./dmma_peak
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[u][0]), "+d"(c[u][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
  for (int u = 0; u < 8; ++u) s += c[u][0] + c[u][1];
  if (s == 1.2345) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double x[8];
  for (int u = 0; u < 8; ++u) x[u] = threadIdx.x * 1e-7 + u;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = fma(x[u], 0.999, 1e-6);
  }
  double s = 0;
  for (int u = 0; u < 8; ++u) s += x[u];
  if (s == 1.2345) out[0] = s;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  cudaMalloc(&d, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps : {4, 8, 16, 32}) {
    const int threads = 32 * warps, iters = 2048;
    dmma_loop<<<sms, threads>>>(d, 16);
    cudaEventRecord(e0);
    dmma_loop<<<sms, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = 2.0 * 256 * 8 * (double)iters * warps * sms;  // 256 FMA per mma per warp
    printf("dmma  warps/SM %2d: %.1f TFLOP/s\n", warps, fl / (ms * 1e-3) / 1e12);
    dfma_loop<<<sms, threads>>>(d, 16);
    cudaEventRecord(e0);
    dfma_loop<<<sms, threads>>>(d, iters / 4);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl2 = 2.0 * 16 * 8 * (double)(iters / 4) * threads * sms;
    printf("dfma  warps/SM %2d: %.1f TFLOP/s\n", warps, fl2 / (ms * 1e-3) / 1e12);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
