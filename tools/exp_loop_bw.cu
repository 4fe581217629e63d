// tools/exp_loop_bw.cu — microbenchmark: K5's per-block softmax exponential loop in
// isolation (64 logits per thread, register-resident, 2 warps per SMSP as in K5), in SM
// cycles per block, for variants of the MUFU / FMA-polynomial split and the bf16 packing.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/exp_loop_bw tools/exp_loop_bw.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2605_23445_b200/csrc/sm100.cuh"
using namespace dfsgpu::sm100;

__device__ __forceinline__ uint32_t pack_trunc(float lo, float hi) {  // bf16 by truncation (1 PRMT)
  return __byte_perm(__float_as_uint(lo), __float_as_uint(hi), 0x7632);
}
// POLY: 38 = pairs 1,4,7 of 8; n = every n-th pair; 0 none. PACK: 0 cvt.rn, 1 PRMT truncation
template <int POLY, int PACK>
__device__ __forceinline__ bool poly_at(int i) {
  if constexpr (POLY == 0) return false;
  else if constexpr (POLY == 38) return (0x92u >> (i % 8)) & 1u;
  else return i % POLY == POLY - 1;
}
template <int POLY, int PACK>
__global__ void __launch_bounds__(256, 1) k(uint32_t* out, int iters, long long* clk, float scale) {
  // K5's softmax data path: per block, S slice TMEM -> registers (2 x32 loads), exp2 of the
  // 64 logits, packed bf16 P back to TMEM (2 x16 stores), row sum; 2 warps per SMSP.
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, wg = warp >> 2;
  if (warp == 0) tmem_alloc<512>(&tbase);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase, lane_addr = uint32_t((warp & 3) * 32) << 16;
  {  // S = small logits
    uint32_t z[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) z[i] = __float_as_uint(-0.01f * float((lane + i) & 63));
    tmem_st32(tmem + lane_addr + wg * 64, z);
    tmem_st32(tmem + lane_addr + wg * 64 + 32, z);
    tmem_wait_st();
  }
  uint64_t lsum[2] = {0, 0};
  float m = 0.5f;
  __syncwarp();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t sv[64];
    tmem_ld32(tmem + lane_addr + wg * 64, *reinterpret_cast<uint32_t(*)[32]>(sv));
    tmem_ld32(tmem + lane_addr + wg * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(sv + 32));
    tmem_wait_ld();
    const uint64_t sc2 = f2_pack(scale, scale), nm2 = f2_pack(-m, -m);
    uint32_t pk[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      float x0, x1;
      f2_unpack(f2_fma(f2_pack(__uint_as_float(sv[2 * i]), __uint_as_float(sv[2 * i + 1])), sc2, nm2), x0, x1);
      float p0, p1;
      if (poly_at<POLY, PACK>(i)) {
        f2_unpack(ex2_poly2(x0, x1), p0, p1);
      } else {
        p0 = ex2(x0);
        p1 = ex2(x1);
      }
      lsum[i & 1] = f2_add(lsum[i & 1], f2_pack(p0, p1));
      pk[i] = PACK ? pack_trunc(p0, p1) : pack_bf16(p0, p1);
    }
    tmem_st16(tmem + lane_addr + 256 + wg * 32, *reinterpret_cast<const uint32_t(*)[16]>(pk));
    tmem_st16(tmem + lane_addr + 256 + wg * 32 + 16, *reinterpret_cast<const uint32_t(*)[16]>(pk + 16));
    tmem_wait_st();
    m = m * 1.0000001f;  // loop-carried, like the running max
  }
  const long long t1 = clock64();
  float a, b;
  f2_unpack(f2_add(lsum[0], lsum[1]), a, b);
  out[blockIdx.x * blockDim.x + threadIdx.x] = __float_as_uint(a + b + m);
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

int main() {
  uint32_t* out;
  long long* clk;
  cudaMalloc(&out, 148 * 256 * 4);
  cudaMallocManaged(&clk, 8);
  const int iters = 2000;
  using KF = void (*)(uint32_t*, int, long long*, float);
  struct V { const char* name; KF f; } vs[] = {
      {"all MUFU, cvt.rn", k<0, 0>}, {"poly 1,4,7/8, cvt.rn", k<38, 0>}, {"poly every 3rd, cvt.rn", k<3, 0>},
      {"poly every 2nd, cvt.rn", k<2, 0>}, {"all MUFU, PRMT trunc", k<0, 1>}, {"poly 1,4,7/8, PRMT trunc", k<38, 1>},
      {"poly every 3rd, PRMT", k<3, 1>}, {"poly every 2nd, PRMT", k<2, 1>}};
  for (auto& v : vs)
    for (int threads : {256}) {
      for (int rep = 0; rep < 2; ++rep) v.f<<<148, threads>>>(out, iters, clk, 0.1f);
      cudaDeviceSynchronize();
      printf("%-26s warps/SMSP=%d: %.0f cycles per block (64 logits/thread)  %s\n", v.name, threads / 128,
             double(*clk) / iters, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
