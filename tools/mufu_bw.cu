// Microbenchmark: MUFU.EX2 and FFMA2 throughput per SM per clock on this GPU.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mufu_bw tools/mufu_bw.cu && tools/mufu_bw
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint32_t ex2_bf16x2(uint32_t x) {
  uint32_t y;
  asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ uint32_t ex2_f16x2(uint32_t x) {
  uint32_t y;
  asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x));
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
      if (MODE == 2) a[i] = __uint_as_float(ex2_bf16x2(__float_as_uint(a[i])) ^ 0x80008000u);  // 2 results
      if (MODE == 3) a[i] = __uint_as_float(ex2_f16x2(__float_as_uint(a[i])) ^ 0x80008000u);
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
  for (int mode = 0; mode < 4; ++mode)
    for (int threads : {128, 256, 512, 1024}) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (mode == 0) k<0><<<148, threads>>>(out, iters, clk);
        else if (mode == 1) k<1><<<148, threads>>>(out, iters, clk);
        else if (mode == 2) k<2><<<148, threads>>>(out, iters, clk);
        else k<3><<<148, threads>>>(out, iters, clk);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
      }
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double ops_per_sm = double(threads) * iters * 8 * (mode >= 2 ? 2 : 1);
      const char* names[] = {"ex2.f32   ", "ffma      ", "ex2.bf16x2", "ex2.f16x2 "};
      printf("%s threads=%4d  %.3f ms  clk=%lld  results/clk/SM=%.2f\n", names[mode], threads, ms, *clk,
             ops_per_sm / double(*clk));
    }
  return 0;
}
