// Microbenchmark: MUFU.EX2 and FFMA2 throughput per SM per clock on this GPU.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mufu_bw tools/mufu_bw.cu && tools/mufu_bw
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int MODE>
__global__ void k(float* out, int iters, long long* clk) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i * 1e-4f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) a[i] = ex2(a[i]) * -0.5f;          // MUFU + FMUL
      if (MODE == 1) a[i] = fmaf(a[i], 0.999f, 1e-3f);  // FFMA
    }
  }
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

int main() {
  float* out;
  long long* clk;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMallocManaged(&clk, 8);
  const int iters = 4096;
  for (int mode = 0; mode < 2; ++mode)
    for (int threads : {128, 256, 512, 1024}) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (mode == 0) k<0><<<148, threads>>>(out, iters, clk);
        else k<1><<<148, threads>>>(out, iters, clk);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
      }
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double ops_per_sm = double(threads) * iters * 8;
      printf("%s threads=%4d  %.3f ms  clk=%lld  ops/clk/SM=%.2f\n", mode == 0 ? "ex2 " : "ffma", threads, ms, *clk,
             ops_per_sm / double(*clk));
    }
  return 0;
}
