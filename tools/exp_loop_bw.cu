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
// FEAT bits: 16 = column-split TMEM shapes (32x32b: thread = lane, 64 consecutive columns),
// 32 = cheap threshold test (x max over the polynomial pairs only + block-sum check), 1 = threshold test (x max over the block, shuffle, vote) as K5's row-split loop,
// 2 = mbarrier protocol (try_wait on an already-completed phase, fence, syncwarp, lane-0
// arrive), 4 = per-block LUT load + partial-block bound (as K5), 8 = second warpgroup offset
// by half a block (a dummy pass first)
template <int POLY, int PACK, int FEAT = 0>
__global__ void __launch_bounds__(256, 1) k(uint32_t* out, int iters, long long* clk, float scale, const int* lut) {
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bars[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, wg = warp >> 2;
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], (1u << 20) - 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&tbase);
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) mbar_arrive(&bars[0]);  // phase 0 completes: later waits on parity 0 return at once
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase, lane_addr = uint32_t((warp & 3) * 32 + wg * 16) << 16;
  {  // S = small logits
    uint32_t z[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) z[i] = __float_as_uint(-0.01f * float((lane + i) & 63));
    tmem_st16x2_x32<32>(tmem + lane_addr, z);
    tmem_st16x2_x32<32>(tmem + lane_addr + 64, z);
    tmem_wait_st();
  }
  uint64_t lsum[2] = {0, 0};
  float m = 0.5f;
  int vb_next = 0, valid_acc = 0;
  const uint32_t bar0 = pin_u32(smem_u32(&bars[0])), bar1 = pin_u32(smem_u32(&bars[1]));
  __syncwarp();
  const long long t0 = clock64();
  for (int it = 0; it < iters + ((FEAT & 8) && wg ? 0 : 0); ++it) {
    int vb = 0;
    if constexpr (FEAT & 4) {
      vb = vb_next;
      vb_next = __ldg(lut + ((it + 1) & 1023));
    }
    if constexpr (FEAT & 2) mbar_wait_a(bar0, 0);
    tc_fence_after();
    uint32_t sv[64];
    if constexpr (FEAT & 16) {
      tmem_ld32(tmem + (lane_addr & 0xffe00000u) + wg * 64, *reinterpret_cast<uint32_t(*)[32]>(sv));
      tmem_ld32(tmem + (lane_addr & 0xffe00000u) + wg * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(sv + 32));
    } else {
      tmem_ld16x2_x64<64>(tmem + lane_addr, sv);
    }
    tmem_wait_ld();
    if constexpr (FEAT & 4) {
      const int valid = min(128, 118800 - vb * 128) - (lane >> 4) * 64;
      if (valid < 64) {
#pragma unroll
        for (int i = 0; i < 64; ++i)
          if (i >= valid) sv[i] = __float_as_uint(-INFINITY);
      }
    }
    const uint64_t sc2 = f2_pack(scale, scale), nm2 = f2_pack(-m, -m);
    uint32_t pk[32];
    float xm[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      float x0, x1;
      f2_unpack(f2_fma(f2_pack(__uint_as_float(sv[2 * i]), __uint_as_float(sv[2 * i + 1])), sc2, nm2), x0, x1);
      if constexpr (FEAT & 1) xm[i & 3] = fmaxf(xm[i & 3], fmaxf(x0, x1));
      if constexpr (FEAT & 32)
        if (poly_at<POLY, PACK>(i)) xm[i & 3] = fmaxf(xm[i & 3], fmaxf(x0, x1));
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
    if constexpr (FEAT & 1) {
      float xmax = fmaxf(fmaxf(xm[0], xm[1]), fmaxf(xm[2], xm[3]));
      xmax = fmaxf(xmax, __shfl_xor_sync(0xffffffffu, xmax, 16));
      if (__any_sync(0xffffffffu, xmax > 1e30f)) m += 1.f;  // never taken
    }
    if constexpr (FEAT & 32) {
      float xmax = fmaxf(fmaxf(xm[0], xm[1]), fmaxf(xm[2], xm[3]));
      float a0, a1;
      f2_unpack(f2_add(lsum[0], lsum[1]), a0, a1);
      if (__any_sync(0xffffffffu, xmax > 20.f || !(a0 + a1 <= 1048576.f))) m += 1.f;  // never taken
    }
    if constexpr (FEAT & 16) {
      tmem_st16(tmem + (lane_addr & 0xffe00000u) + 256 + wg * 32, *reinterpret_cast<const uint32_t(*)[16]>(pk));
      tmem_st16(tmem + (lane_addr & 0xffe00000u) + 256 + wg * 32 + 16, *reinterpret_cast<const uint32_t(*)[16]>(pk + 16));
    } else {
      tmem_st16x2_x32<32>(tmem + lane_addr + 256, pk);
    }
    tmem_wait_st();
    if constexpr (FEAT & 2) {
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_a(bar1);
    }
    m = m * 1.0000001f;  // loop-carried, like the running max
    if constexpr (FEAT & 4) valid_acc += vb;
  }
  const long long t1 = clock64();
  float a, b;
  f2_unpack(f2_add(lsum[0], lsum[1]), a, b);
  out[blockIdx.x * blockDim.x + threadIdx.x] = __float_as_uint(a + b + m) + valid_acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(tmem);
}


// NL logits per thread (64 or 32) with 128 * WPS threads: WPS warps per SMSP. NL = 32: warp pairs
// of a row group take column halves (16x32bx2.x32 at columns 32 * half + {0, 64}).
template <int NL, int WPS>
__global__ void __launch_bounds__(128 * WPS, 1) kw(uint32_t* out, int iters, long long* clk, float scale) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc<512>(&tbase);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const int grp = warp >> 2;                   // 0 .. WPS-1
  const int hf = NL == 64 ? grp : (grp >> 1);  // row half
  const int cs = NL == 64 ? 0 : (grp & 1);     // column half (NL = 32)
  const uint32_t tmem = tbase, lane_addr = uint32_t((warp & 3) * 32 + hf * 16) << 16;
  uint64_t lsum[2] = {0, 0};
  float m = 0.5f;
  __syncwarp();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t sv[NL];
    if constexpr (NL == 64)
      tmem_ld16x2_x64<64>(tmem + lane_addr, sv);
    else
      tmem_ld16x2_x32<64>(tmem + lane_addr + cs * 32, sv);
    tmem_wait_ld();
    const uint64_t sc2 = f2_pack(scale, scale), nm2 = f2_pack(-m, -m);
    uint32_t pk[NL / 2];
#pragma unroll
    for (int i = 0; i < NL / 2; ++i) {
      float x0, x1;
      f2_unpack(f2_fma(f2_pack(__uint_as_float(sv[2 * i]), __uint_as_float(sv[2 * i + 1])), sc2, nm2), x0, x1);
      float p0, p1;
      if (poly_at<38, 0>(i)) {
        f2_unpack(ex2_poly2(x0, x1), p0, p1);
      } else {
        p0 = ex2(x0);
        p1 = ex2(x1);
      }
      lsum[i & 1] = f2_add(lsum[i & 1], f2_pack(p0, p1));
      pk[i] = pack_bf16(p0, p1);
    }
    if constexpr (NL == 64)
      tmem_st16x2_x32<32>(tmem + lane_addr + 256, pk);
    else
      tmem_st16x2_x16<32>(tmem + lane_addr + 256 + cs * 16, pk);
    tmem_wait_st();
    m = m * 1.0000001f;
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


// Ping-pong candidate: one thread per row (32x32b: 32 lanes of the warp's quadrant), 128 logits
// per thread per block in 4 chunks of 32 (TMEM load of chunk c + 1 in flight while chunk c is
// exponentiated), P stored per chunk; WPS independent warps per SMSP (different tiles).
// MMA > 0: one extra warp (id 4 * WPS, SMSP 0) issues K5's MMA pattern (QK + PV, both operands
// from shared memory / TMEM, on TMEM columns 256-511) back to back while the softmax warps run.
template <int WPS, int MMA = 0>
__global__ void __launch_bounds__(128 * WPS + 32 * MMA, 1) kp(uint32_t* out, int iters, long long* clk, float scale) {
  __shared__ uint32_t tbase;
  __shared__ volatile int done;
  extern __shared__ __align__(1024) uint8_t smem_dyn[];
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) done = 0;
  if (warp == 0) tmem_alloc<512>(&tbase);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (MMA && warp == 4 * WPS) {
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
    const uint32_t a = smem_u32(sm), b = a + 32768;
    const uint32_t idqk = idesc_bf16_f32(128, 128, false, false), idpv = idesc_bf16_f32(128, 128, false, true);
    if ((threadIdx.x & 31) == 0) {
      while (!done) {
#pragma unroll
        for (int st = 0; st < 8; ++st) {
          const uint32_t off = (st >> 2) * 16384 + (st & 3) * 32;
          umma_f16(tbase + 256, smem_desc_sw128(a + off, 16, 1024), smem_desc_sw128(b + off, 16, 1024), idqk, st > 0);
        }
#pragma unroll
        for (int st = 0; st < 8; ++st)
          umma_f16_ts(tbase + 384, tbase + 256 + st * 8, smem_desc_sw128(b + st * 16 * 128, 16384, 1024), idpv, 1);
      }
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc<512>(tbase);
    return;
  }
  const int tile = warp >> 2;  // which tile's S / P this warp works on
  const uint32_t tmem = tbase + tile * 256, lane_addr = uint32_t((warp & 3) * 32) << 16;
  uint64_t lsum[2] = {0, 0};
  float m = 0.5f;
  __syncwarp();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const uint64_t sc2 = f2_pack(scale, scale), nm2 = f2_pack(-m, -m);
    uint32_t sa[32], sb[32];
    tmem_ld32(tmem + lane_addr, sa);
    tmem_wait_ld();
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t(&cur)[32] = (c & 1) ? sb : sa;
      uint32_t(&nxt)[32] = (c & 1) ? sa : sb;
      if (c < 3) tmem_ld32(tmem + lane_addr + (c + 1) * 32, nxt);
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        float x0, x1;
        f2_unpack(f2_fma(f2_pack(__uint_as_float(cur[2 * i]), __uint_as_float(cur[2 * i + 1])), sc2, nm2), x0, x1);
        float p0, p1;
        if (poly_at<38, 0>(i + 16 * c)) {
          f2_unpack(ex2_poly2(x0, x1), p0, p1);
        } else {
          p0 = ex2(x0);
          p1 = ex2(x1);
        }
        lsum[i & 1] = f2_add(lsum[i & 1], f2_pack(p0, p1));
        pk[i] = pack_bf16(p0, p1);
      }
      tmem_st16(tmem + lane_addr + 128 + c * 16, pk);
      if (c < 3) tmem_wait_ld();
    }
    tmem_wait_st();
    m = m * 1.0000001f;
  }
  const long long t1 = clock64();
  float a, b;
  f2_unpack(f2_add(lsum[0], lsum[1]), a, b);
  out[blockIdx.x * blockDim.x + threadIdx.x] = __float_as_uint(a + b + m);
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
  if (threadIdx.x == 0) done = 1;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(tbase);
}

int main() {
  uint32_t* out;
  long long* clk;
  int* lut;
  cudaMalloc(&out, 148 * 256 * 4);
  cudaMallocManaged(&clk, 8);
  cudaMalloc(&lut, 1024 * 4);
  cudaMemset(lut, 0, 1024 * 4);
  const int iters = 2000;
  using KF = void (*)(uint32_t*, int, long long*, float, const int*);
  struct V { const char* name; KF f; } vs[] = {
      {"32x32b ld+exp+st", k<38, 0, 16>},
      {"ld+exp+st (poly 1,4,7/8)", k<38, 0, 0>},
      {"+ cheap threshold test", k<38, 0, 32>},
      {"cheap test + mbar + LUT", k<38, 0, 32 | 6>},
      {"32x32b + cheap + mbar + LUT", k<38, 0, 32 | 16 | 6>},
      {"+ threshold test", k<38, 0, 1>},
      {"+ mbarrier protocol", k<38, 0, 2>},
      {"+ LUT load / bound", k<38, 0, 4>},
      {"all of K5's loop", k<38, 0, 7>},
      {"all, every 3rd poly", k<3, 0, 7>},
      {"all, all MUFU", k<0, 0, 7>}};
  {
    using KW = void (*)(uint32_t*, int, long long*, float);
    struct W { const char* name; KW f; int threads; } ws[] = {
        {"2 warps/SMSP x 64 logits", kw<64, 2>, 256}, {"4 warps/SMSP x 32 logits", kw<32, 4>, 512}};
    for (auto& w : ws) {
      for (int rep = 0; rep < 2; ++rep) w.f<<<148, w.threads>>>(out, iters, clk, 0.1f);
      cudaDeviceSynchronize();
      printf("%-28s: %.0f cycles per block (4096 exps per SMSP)  %s\n", w.name, double(*clk) / iters,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  for (int cfg = 0; cfg < 4; ++cfg) {
    const int wps = cfg & 1 ? 2 : 1, mma = cfg >> 1;
    using KP = void (*)(uint32_t*, int, long long*, float);
    KP f = cfg == 0 ? kp<1, 0> : cfg == 1 ? kp<2, 0> : cfg == 2 ? kp<1, 1> : kp<2, 1>;
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 66560);
    for (int rep = 0; rep < 2; ++rep) f<<<148, 128 * wps + 32 * mma, 66560>>>(out, iters, clk, 0.1f);
    cudaDeviceSynchronize();
    printf("ping-pong: %d warp(s)/SMSP x 128 logits (chunks of 32)%s: %.0f cycles per block per warp  %s\n", wps,
           mma ? " + MMA warp" : "", double(*clk) / iters, cudaGetErrorString(cudaGetLastError()));
  }
  for (auto& v : vs) {
    for (int rep = 0; rep < 2; ++rep) v.f<<<148, 256>>>(out, iters, clk, 0.1f, lut);
    cudaDeviceSynchronize();
    printf("%-28s 2 warps/SMSP (16 rows each): %.0f cycles per block  %s\n", v.name, double(*clk) / iters,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
