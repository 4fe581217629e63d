// tools/tma_bw.cu — microbenchmark: L2 -> SMEM bandwidth with TMA tile loads, the
// access pattern of K5 (128 x 64 bf16 SWIZZLE_128B boxes, 2 per 32 KB tile) from
// an L2-resident per-head K/V working set. Standalone: nvcc -gencode
// arch=compute_100a,code=sm_100a -O3 -o tools/tma_bw tools/tma_bw.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include "../paper_2605_23445_b200/csrc/sm100.cuh"

using namespace dfsgpu::sm100;

template <int STAGES>
__global__ void __launch_bounds__(64, 1) tma_bw_kernel(const __grid_constant__ CUtensorMap map, int rows_total,
                                                         int tiles_per_cta, int heads, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * 32768);
  uint64_t* empty = full + STAGES;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const unsigned long long t0 = clock64();
  const int warp = threadIdx.x >> 5;
  uint32_t seed = blockIdx.x * 2654435761u;
  if (warp == 0 && threadIdx.x == 0) {
    for (int t = 0; t < tiles_per_cta; ++t) {
      const int slot = t % STAGES, use = t / STAGES;
      mbar_wait(&empty[slot], (use & 1) ^ 1);
      mbar_expect_tx(&full[slot], 32768);
      seed = seed * 1664525u + 1013904223u;
      const int blk = (seed >> 8) % (rows_total / 128);
      const int h = (seed >> 4) % heads;
      tma_load_3d(smem + slot * 32768, &map, &full[slot], 0, blk * 128, h);
      tma_load_3d(smem + slot * 32768 + 16384, &map, &full[slot], 64, blk * 128, h);
    }
  } else if (warp == 1 && threadIdx.x == 32) {
    for (int t = 0; t < tiles_per_cta; ++t) {
      const int slot = t % STAGES, use = t / STAGES;
      mbar_wait(&full[slot], use & 1);
      mbar_arrive(&empty[slot]);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) cycles[blockIdx.x] = clock64() - t0;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int STAGES>
void run(EncodeFn enc, void* buf, int rows, int heads, int ctas, int tiles) {
  CUtensorMap map;
  cuuint64_t dims[3] = {128, (cuuint64_t)rows, (cuuint64_t)heads};
  cuuint64_t strides[2] = {256, (cuuint64_t)rows * 256};
  cuuint32_t box[3] = {64, 128, 1}, es[3] = {1, 1, 1};
  enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = STAGES * 32768 + 1024 + 256;
  cudaFuncSetAttribute(tma_bw_kernel<STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* cyc;
  cudaMalloc(&cyc, sizeof(unsigned long long) * ctas);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  tma_bw_kernel<STAGES><<<ctas, 64, smem>>>(map, rows, tiles, heads, cyc);
  cudaEventRecord(a);
  tma_bw_kernel<STAGES><<<ctas, 64, smem>>>(map, rows, tiles, heads, cyc);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double bytes = double(ctas) * tiles * 32768.0;
  printf("stages=%d ctas=%d working_set=%.0fMB: %.3f ms, %.2f TB/s (%.1f B/clk/SM @1.9GHz) err=%s\n", STAGES, ctas,
         double(rows) * heads * 256 / 1e6, ms, bytes / ms / 1e9, bytes / ms / 1e9 * 1e3 / 1.9e9 / ctas * 1e3 / 1e3,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(cyc);
}

int main() {
  void* ptr = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)ptr;
  const int rows = 118912, heads = 24;  // one HY K tensor (730 MB) ...
  void* buf;
  cudaMalloc(&buf, size_t(rows) * heads * 256);
  cudaMemset(buf, 0, size_t(rows) * heads * 256);
  // L2-resident: 2 heads (61 MB) vs DRAM-streaming: 24 heads
  for (int h : {1, 2, 24}) {
    run<2>(enc, buf, rows, h, 148, 4000);
    run<4>(enc, buf, rows, h, 148, 4000);
    run<6>(enc, buf, rows, h, 148, 4000);
    run<3>(enc, buf, rows, h, 296, 2000);
  }
  return 0;
}
