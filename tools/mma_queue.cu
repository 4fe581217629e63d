// tools/mma_queue.cu — microbenchmark: how deep is the tcgen05.mma issue queue? One thread issues
// 16 M=128 N=128 K=16 MMAs into an idle tensor pipe and records clock64 after each issue
// (issue returns once the instruction is accepted; a full queue makes it wait for execution).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mma_queue tools/mma_queue.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2605_23445_b200/csrc/sm100.cuh"
using namespace dfsgpu::sm100;

__global__ void __launch_bounds__(128, 1) k(unsigned long long* out, int ts) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tbase;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&tbase);
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = a + 32768;
    const uint32_t idesc = idesc_bf16_f32(128, 128, false, false);
    unsigned long long t[17];
    t[0] = clock64();
#pragma unroll
    for (int s = 0; s < 16; ++s) {
      const uint32_t off = ((s & 7) >> 2) * 16384 + (s & 3) * 32;
      if (ts)
        umma_f16_ts(tmem + 128, tmem + 384 + (s & 7) * 8, smem_desc_sw128(b + off, 16, 1024), idesc, s > 0);
      else
        umma_f16(tmem, smem_desc_sw128(a + off, 16, 1024), smem_desc_sw128(b + off, 16, 1024), idesc, s > 0);
      t[s + 1] = clock64();
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    const unsigned long long done = clock64();
    if (blockIdx.x == 0) {
      for (int s = 0; s <= 16; ++s) out[s] = t[s] - t[0];
      out[17] = done - t[0];
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 32 * sizeof(unsigned long long));
  const int smem = 65536 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int ts : {0, 1}) {
    for (int rep = 0; rep < 3; ++rep) k<<<148, 128, smem>>>(d, ts);
    unsigned long long h[18];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%s: clock after each of 16 issues:", ts ? "TS (A from TMEM)" : "SS");
    for (int s = 1; s <= 16; ++s) printf(" %llu", h[s]);
    printf(" | all complete %llu  (%s)\n", h[17], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
