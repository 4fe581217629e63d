// tools/gather4_bw.cu — L2->SMEM bandwidth of TMA tile::gather4 row gathers (the K/V reorder
// fused into K5) against plain tile loads of a pre-permuted copy. 148 persistent CTAs stream
// 128 x 128 bf16 tiles (32 KB) of random key blocks of ONE head (the L2-resident working set
// K5 has while it walks a head) into a 4-stage ring; a consumer warp only waits and frees.
//   gather: rows token*24 + h of a raster [118800*24, 128] map, 64 gather4 per tile (2 per lane)
//   tile:   2 boxes of 128 x 64 from a [24*118800, 128] head-major copy
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/gather4_bw tools/gather4_bw.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include "../paper_2605_23445_b200/csrc/sm100.cuh"
using namespace dfsgpu::sm100;

constexpr int kN = 118800, kH = 24, kD = 128, kStages = 4, kTiles = 256;

__global__ void __launch_bounds__(64, 1) k(const __grid_constant__ CUtensorMap gmap, const __grid_constant__ CUtensorMap tmap,
                                            const int* perm, int mode, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* s = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[kStages], empty[kStages];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const unsigned long long t0 = clock64();
  const int h = 3;
  if (warp == 0) {
    for (int t = 0; t < kTiles; ++t) {
      const int slot = t % kStages, use = t / kStages;
      mbar_wait(&empty[slot], (use & 1) ^ 1);
      const int blk = (blockIdx.x * 7919 + t * 104729) % 928;
      uint8_t* dst = s + slot * 32768;
      if (mode == 0) {
        int rr[4];
        for (int q = 0; q < 4; ++q) rr[q] = perm[blk * 128 + 4 * lane + q] * kH + h;
        if (elect_one()) mbar_expect_tx(&full[slot], 32768);
        __syncwarp();
        for (int c = 0; c < 2; ++c) tma_gather4(dst + c * 16384 + lane * 512, &gmap, &full[slot], c * 64, rr[0], rr[1], rr[2], rr[3]);
        __syncwarp();
      } else {
        if (elect_one()) {
          mbar_expect_tx(&full[slot], 32768);
          for (int c = 0; c < 2; ++c)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                    smem_u32(dst + c * 16384)),
                "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(smem_u32(&full[slot])), "r"(c * 64), "r"(h * kN + blk * 128)
                : "memory");
        }
        __syncwarp();
      }
    }
  } else {
    for (int t = 0; t < kTiles; ++t) {
      const int slot = t % kStages, use = t / kStages;
      mbar_wait(&full[slot], use & 1);
      if (elect_one()) mbar_arrive(&empty[slot]);
      __syncwarp();
    }
    if (lane == 0 && blockIdx.x == 0) cyc[mode] = clock64() - t0;
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  void* ptr = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)ptr;
  const size_t rows = size_t(kN) * kH;
  void *dr, *dp;
  cudaMalloc(&dr, rows * kD * 2);
  cudaMalloc(&dp, rows * kD * 2);
  cudaMemset(dr, 0, rows * kD * 2);
  cudaMemset(dp, 0, rows * kD * 2);
  int* hperm = (int*)malloc(sizeof(int) * kN);
  for (int i = 0; i < kN; ++i) hperm[i] = i;
  srand(1);
  for (int i = kN - 1; i > 0; --i) {  // blocks of 128 tokens spread like a 3D Hilbert block over the raster
    int j = rand() % (i + 1);
    int t = hperm[i]; hperm[i] = hperm[j]; hperm[j] = t;
  }
  int* dperm;
  cudaMalloc(&dperm, sizeof(int) * kN);
  cudaMemcpy(dperm, hperm, sizeof(int) * kN, cudaMemcpyHostToDevice);
  unsigned long long* dc;
  cudaMalloc(&dc, 16);
  CUtensorMap gmap, tmap;
  cuuint64_t gd[2] = {(cuuint64_t)kD, (cuuint64_t)rows}, gs[1] = {(cuuint64_t)kD * 2};
  cuuint32_t gb[2] = {64, 1}, tb[2] = {64, 128}, es[2] = {1, 1};
  enc(&gmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dr, gd, gs, gb, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dp, gd, gs, tb, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = kStages * 32768 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 3; ++rep) k<<<148, 64, smem>>>(gmap, tmap, dperm, mode, dc);
    cudaDeviceSynchronize();
    unsigned long long c[2];
    cudaMemcpy(c, dc, 16, cudaMemcpyDeviceToHost);
    printf("%s: %llu cycles for %d tiles -> %.1f B/clk/SM (%s)\n", mode ? "tile loads (permuted copy)" : "gather4 (raster rows)",
           c[mode], kTiles, kTiles * 32768.0 / c[mode], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
