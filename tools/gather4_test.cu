// tools/gather4_test.cu — does a TMA tile::gather4 row gather (2D map, box {64, 1},
// SWIZZLE_128B, 32 x 4 rows) produce the same shared-memory image as a plain tile
// load of the pre-permuted rows (box {64, 128})? The K5 reorder fusion depends on it.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/gather4_test tools/gather4_test.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include "../paper_2605_23445_b200/csrc/sm100.cuh"

using namespace dfsgpu::sm100;

__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int r0, int r1,
                                            int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__global__ void k(const __grid_constant__ CUtensorMap gmap, const __grid_constant__ CUtensorMap tmap,
                  const int* idx, int* mismatches) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* s = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
  uint8_t* a = s;            // gathered: 2 chunks x 128 rows x 128 B
  uint8_t* b = s + 32768;    // plain tile of the permuted copy
  __shared__ uint64_t bar[2];
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bar[0], 32768);
    for (int c = 0; c < 2; ++c)
      for (int g = 0; g < 32; ++g)
        tma_gather4(a + c * 16384 + g * 512, &gmap, &bar[0], c * 64, idx[4 * g], idx[4 * g + 1], idx[4 * g + 2],
                    idx[4 * g + 3]);
    mbar_expect_tx(&bar[1], 32768);
    for (int c = 0; c < 2; ++c) tma_load_2d(b + c * 16384, &tmap, &bar[1], c * 64, 0);
  }
  mbar_wait(&bar[0], 0);
  mbar_wait(&bar[1], 0);
  int bad = 0;
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x)
    bad += reinterpret_cast<const uint32_t*>(a)[i] != reinterpret_cast<const uint32_t*>(b)[i];
  atomicAdd(mismatches, bad);
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  void* ptr = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)ptr;
  const int R = 4096, D = 128;
  unsigned short* h = (unsigned short*)malloc(size_t(R) * D * 2);
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < D; ++c) h[r * D + c] = (unsigned short)((r * 131 + c * 7) & 0xffff);
  int hidx[128];
  for (int i = 0; i < 128; ++i) hidx[i] = (i * 977 + 13) % R;
  unsigned short* hp = (unsigned short*)malloc(128 * D * 2);
  for (int i = 0; i < 128; ++i)
    for (int c = 0; c < D; ++c) hp[i * D + c] = h[hidx[i] * D + c];
  void *dg, *dp;
  int *didx, *dbad;
  cudaMalloc(&dg, size_t(R) * D * 2);
  cudaMalloc(&dp, 128 * D * 2);
  cudaMalloc(&didx, sizeof(hidx));
  cudaMalloc(&dbad, 4);
  cudaMemcpy(dg, h, size_t(R) * D * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dp, hp, 128 * D * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(didx, hidx, sizeof(hidx), cudaMemcpyHostToDevice);
  cudaMemset(dbad, 0, 4);
  CUtensorMap gmap, tmap;
  cuuint64_t gd[2] = {(cuuint64_t)D, (cuuint64_t)R}, gs[1] = {(cuuint64_t)D * 2};
  cuuint32_t gb[2] = {64, 1}, es[2] = {1, 1};
  CUresult r1 = enc(&gmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dg, gd, gs, gb, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cuuint64_t td[2] = {(cuuint64_t)D, 128}, ts[1] = {(cuuint64_t)D * 2};
  cuuint32_t tb[2] = {64, 128};
  CUresult r2 = enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dp, td, ts, tb, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  k<<<1, 128, 65536 + 1024>>>(gmap, tmap, didx, dbad);
  int bad = -1;
  cudaError_t e = cudaMemcpy(&bad, dbad, 4, cudaMemcpyDeviceToHost);
  printf("encode gather=%d tile=%d  kernel=%s  mismatching words=%d (of 8192)\n", int(r1), int(r2),
         cudaGetErrorString(e), bad);
  return bad == 0 ? 0 : 1;
}
