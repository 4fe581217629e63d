// tools/pipe_bw.cu — microbenchmark: issue/pipe throughput per SMSP of the K5 softmax
// instruction classes (FFMA, FFMA2, FADD2, FMNMX, FMNMX3, F2FP bf16 pack, IMAD, MUFU.EX2) and
// of mixes, with 1 or 2 warps per SMSP and 8 independent chains per thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pipe_bw tools/pipe_bw.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t f2fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t f2add(uint64_t a, uint64_t b) {
  uint64_t d;
  asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ float ffma(float a, float b, float c) {
  float d;
  asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm volatile("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
__device__ __forceinline__ float fmax2(float a, float b) {
  float d;
  asm volatile("max.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
  return d;
}
__device__ __forceinline__ uint32_t cvt_bf16x2(float a, float b) {
  uint32_t d;
  asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(a), "f"(b));
  return d;
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ uint32_t shladd(uint32_t a, uint32_t c) {
  uint32_t d;
  asm volatile("shl.b32 %0, %1, 23;\n\tadd.u32 %0, %0, %2;" : "=r"(d) : "r"(a), "r"(c));
  return d;
}

// ops per inner iteration per thread: 8 instructions of the class (mixes: see names)
template <int MODE>
__global__ void k(float* out, int iters, long long* clk) {
  float a[8];
  uint64_t p[8];
  uint32_t u[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    a[i] = threadIdx.x * 1e-3f + i * 1e-4f;
    p[i] = (uint64_t(__float_as_uint(a[i])) << 32) | __float_as_uint(a[i] + 1.f);
    u[i] = threadIdx.x + i;
  }
  const uint64_t c1 = (uint64_t(__float_as_uint(0.999f)) << 32) | __float_as_uint(0.999f);
  const uint64_t c2 = (uint64_t(__float_as_uint(1e-3f)) << 32) | __float_as_uint(1e-3f);
  const float s1 = a[3] * 0.5f, s2 = a[5] * 0.25f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) a[i] = ffma(a[i], 0.999f, s1);
      if (MODE == 1) p[i] = f2fma(p[i], c1, c2);
      if (MODE == 2) p[i] = f2add(p[i], c2);
      if (MODE == 3) a[i] = fmax2(a[i], s1);
      if (MODE == 4) a[i] = fmax3(a[i], s1, s2);
      if (MODE == 5) u[i] = cvt_bf16x2(__uint_as_float(u[i]), s1);
      if (MODE == 6) u[i] = imad(u[i], 0x800000u, u[(i + 1) & 7]);
      if (MODE == 7) a[i] = ex2(a[i]);
      if (MODE == 8) {  // 1 MUFU + 1 FFMA2 per step (co-issue?)
        a[i] = ex2(a[i]);
        p[i] = f2fma(p[i], c1, c2);
      }
      if (MODE == 9) {  // 1 MUFU + 3 FFMA2
        a[i] = ex2(a[i]);
        p[i] = f2fma(p[i], c1, c2);
        p[i] = f2fma(p[i], c1, c2);
        p[i] = f2fma(p[i], c1, c2);
      }
      if (MODE == 10) {  // 1 FFMA2 + 1 FMNMX (fma + alu pipes)
        p[i] = f2fma(p[i], c1, c2);
        a[i] = fmax2(a[i], s1);
      }
      if (MODE == 11) u[i] = shladd(u[i], u[(i + 1) & 7]);
      if (MODE == 12) {  // 1 MUFU + 1 F2FP (shared XU pipe?)
        a[i] = ex2(a[i]);
        u[i] = cvt_bf16x2(__uint_as_float(u[i]), s1);
      }
      if (MODE == 13) {  // 1 MUFU + 2 F2FP
        a[i] = ex2(a[i]);
        u[i] = cvt_bf16x2(__uint_as_float(u[i]), s1);
        u[i] = cvt_bf16x2(__uint_as_float(u[i]), s2);
      }
      if (MODE == 14) {  // 1 F2FP + 1 FFMA2
        u[i] = cvt_bf16x2(__uint_as_float(u[i]), s1);
        p[i] = f2fma(p[i], c1, c2);
      }
      if (MODE == 15) {  // 1 F2FP + 1 FMNMX3
        u[i] = cvt_bf16x2(__uint_as_float(u[i]), s1);
        a[i] = fmax3(a[i], s1, s2);
      }
    }
  }
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i] + __uint_as_float(uint32_t(p[i])) + __uint_as_float(u[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

int main() {
  float* out;
  long long* clk;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMallocManaged(&clk, 8);
  const int iters = 2048;
  const char* names[] = {"FFMA", "FFMA2", "FADD2", "FMNMX", "FMNMX3", "F2FP.BF16", "IMAD", "MUFU.EX2",
                         "EX2+FFMA2", "EX2+3xFFMA2", "FFMA2+FMNMX", "SHL+IADD", "EX2+F2FP", "EX2+2xF2FP", "F2FP+FFMA2", "F2FP+FMNMX3"};
  using KF = void (*)(float*, int, long long*);
  KF ks[] = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>, k<6>, k<7>, k<8>, k<9>, k<10>, k<11>, k<12>, k<13>, k<14>, k<15>};
  for (int mode = 0; mode < 16; ++mode)
    for (int threads : {256}) {
      for (int rep = 0; rep < 2; ++rep) ks[mode]<<<148, threads>>>(out, iters, clk);
      cudaDeviceSynchronize();
      const double warps_per_smsp = threads / 128.0;
      const double steps = double(iters) * 8 * warps_per_smsp;  // per SMSP
      printf("%-12s warps/SMSP=%.0f  %.2f clk per step per SMSP  (%s)\n", names[mode], warps_per_smsp,
             double(*clk) / steps, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
