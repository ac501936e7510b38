// Microtest (run once on a B200): a 12-warp CTA allocates 512 TMEM columns; warp w owns lane
// quarter w % 4 and column block (w / 4) * 160 -- the layout rti_kernel uses.  Checks that each
// warp reads back exactly what it stored and times tcgen05.ld.32x32b.x32.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tq tools/micro/tmem_quarters.cu
// TMEM microtest: 12-warp CTA, 512 columns, warp w -> lane quarter w%4, column block (w/4)*160.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define X32_REGS(v) "=f"(v[0]),"=f"(v[1]),"=f"(v[2]),"=f"(v[3]),"=f"(v[4]),"=f"(v[5]),"=f"(v[6]),"=f"(v[7]),"=f"(v[8]),"=f"(v[9]),"=f"(v[10]),"=f"(v[11]),"=f"(v[12]),"=f"(v[13]),"=f"(v[14]),"=f"(v[15]),"=f"(v[16]),"=f"(v[17]),"=f"(v[18]),"=f"(v[19]),"=f"(v[20]),"=f"(v[21]),"=f"(v[22]),"=f"(v[23]),"=f"(v[24]),"=f"(v[25]),"=f"(v[26]),"=f"(v[27]),"=f"(v[28]),"=f"(v[29]),"=f"(v[30]),"=f"(v[31])
#define X32_IN(v) "f"(v[0]),"f"(v[1]),"f"(v[2]),"f"(v[3]),"f"(v[4]),"f"(v[5]),"f"(v[6]),"f"(v[7]),"f"(v[8]),"f"(v[9]),"f"(v[10]),"f"(v[11]),"f"(v[12]),"f"(v[13]),"f"(v[14]),"f"(v[15]),"f"(v[16]),"f"(v[17]),"f"(v[18]),"f"(v[19]),"f"(v[20]),"f"(v[21]),"f"(v[22]),"f"(v[23]),"f"(v[24]),"f"(v[25]),"f"(v[26]),"f"(v[27]),"f"(v[28]),"f"(v[29]),"f"(v[30]),"f"(v[31])
__device__ __forceinline__ void tm_ld32(uint32_t a, float v[32]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
               : X32_REGS(v) : "r"(a));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tm_st32(uint32_t a, const float v[32]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
               :: "r"(a), X32_IN(v) : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__global__ void __launch_bounds__(384, 1) k(float* out, int iters, long long* cyc) {
  __shared__ uint32_t base;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"((uint32_t)__cvta_generic_to_shared(&base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = base + ((uint32_t)(32 * (w & 3)) << 16) + (w >> 2) * 160;
  for (int n = 0; n < 5; ++n) {
    float v[32];
    for (int c = 0; c < 32; ++c) v[c] = blockIdx.x * 1e6f + w * 1e4f + n * 1e3f + lane * 32 + c;
    tm_st32(tb + 32 * n, v);
  }
  __syncwarp();
  int bad = 0;
  for (int n = 0; n < 5; ++n) {
    float v[32];
    tm_ld32(tb + 32 * n, v);
    for (int c = 0; c < 32; ++c) bad += v[c] != blockIdx.x * 1e6f + w * 1e4f + n * 1e3f + lane * 32 + c;
  }
  // throughput: iters x (ld x32 + 32 FMA)
  float acc = 0.f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float v[32];
    tm_ld32(tb + 32 * (it % 5), v);
#pragma unroll
    for (int c = 0; c < 32; ++c) acc = fmaf(v[c], 1.0001f, acc);
  }
  long long t1 = clock64();
  if (lane == 0 && blockIdx.x == 0) cyc[w] = t1 - t0;
  out[blockIdx.x * 384 + threadIdx.x] = bad + acc * 1e-30f;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(base));
}
int main() {
  float* out; long long* cyc;
  const int nb = 148 * 2;
  cudaMalloc(&out, nb * 384 * 4); cudaMalloc(&cyc, 12 * 8);
  k<<<nb, 384>>>(out, 1000, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  printf("err %s\n", cudaGetErrorString(e));
  float* h = new float[nb * 384]; cudaMemcpy(h, out, nb * 384 * 4, cudaMemcpyDeviceToHost);
  double bad = 0; for (int i = 0; i < nb * 384; ++i) bad += (int)h[i];
  long long c[12]; cudaMemcpy(c, cyc, 96, cudaMemcpyDeviceToHost);
  printf("mismatches %.0f\n", bad);
  for (int w = 0; w < 12; ++w) printf("w%d %.1f cyc/iter\n", w, c[w] / 1000.0);
}
