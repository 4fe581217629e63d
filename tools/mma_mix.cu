// tools/mma_mix.cu — microbenchmark: cost of row-sum MMAs (P x ones, N = 16) next to the PV
// MMAs (N = 128) in one issuing thread. Mode 0: 8 PV (N = 128) per block; 1: each PV followed
// by an N = 16 MMA; 2: 8 PV then 8 N = 16; 3: 8 MMAs with N = 144; 4: 8 N=16 alone. A from TMEM
// (as K5's P), B from smem; 64 blocks back to back; clock64 of the whole sequence per CTA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mma_mix tools/mma_mix.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "../paper_2605_23445_b200/csrc/sm100.cuh"
using namespace dfsgpu::sm100;

__global__ void __launch_bounds__(128, 1) k(unsigned long long* out, int mode) {
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
    const uint32_t b = smem_u32(smem);
    const uint32_t id128 = idesc_bf16_f32(128, 128, false, true);
    const uint32_t id16 = idesc_bf16_f32(128, 16, false, true);
    const uint32_t id144 = idesc_bf16_f32(128, 144, false, true);
    const unsigned long long t0 = clock64();
    for (int blk = 0; blk < 64; ++blk) {
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const uint64_t bd = smem_desc_sw128(b + s * 16 * 128, 16384, 1024);
        if (mode == 0 || mode == 1 || mode == 2)
          umma_f16_ts(tmem + 256, tmem + (s & 7) * 8, bd, id128, blk + s > 0);
        if (mode == 3) umma_f16_ts(tmem + 256, tmem + (s & 7) * 8, smem_desc_sw128(b + s * 16 * 128, 16384, 1024), id144, blk + s > 0);
        if (mode == 1 || mode == 4) umma_f16_ts(tmem + 448, tmem + (s & 7) * 8, bd, id16, blk + s > 0);
      }
      if (mode == 2) {
#pragma unroll
        for (int s = 0; s < 8; ++s)
          umma_f16_ts(tmem + 448, tmem + (s & 7) * 8, smem_desc_sw128(b + s * 16 * 128, 16384, 1024), id16, blk + s > 0);
      }
    }
    const unsigned long long t1 = clock64();
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    const unsigned long long done = clock64();
    if (blockIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = done - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

// operand modes: 64 blocks x 8 MMAs (K = 16 each) of one shape; ts = A from TMEM
__global__ void __launch_bounds__(128, 1) k2(unsigned long long* out, int ts, int n, int bmn, int dcol = 0, int acol = 256) {
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
  for (int i = threadIdx.x; i < 131072 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = a + 32768;
    const uint32_t idesc = idesc_bf16_f32(128, n, false, bmn != 0);
    const unsigned long long t0 = clock64();
    for (int blk = 0; blk < 64; ++blk) {
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const uint32_t koff = ((s >> 2) * 16384 + (s & 3) * 32);
        const uint64_t bd = bmn ? smem_desc_sw128(b + s * 16 * 128, 16384, 1024) : smem_desc_sw128(b + koff, 16, 1024);
        if (ts)
          umma_f16_ts(tmem + dcol, tmem + acol + s * 8, bd, idesc, blk + s > 0);
        else
          umma_f16(tmem + dcol, smem_desc_sw128(a + koff, 16, 1024), bd, idesc, blk + s > 0);
      }
    }
    const unsigned long long t1 = clock64();
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    const unsigned long long done = clock64();
    if (blockIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = done - t0;
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
  if (getenv("MIX_ORDER")) {  // interleave: does the per-MMA cost drift with the run (power) or the kernel?
    cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072 + 1024);
    for (int it = 0; it < 4; ++it) {
      unsigned long long h[2];
      for (int rep = 0; rep < 3; ++rep) k<<<148, 128, smem>>>(d, 0);
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      printf("k  mode 0 (TS N=128 MN): per MMA %.1f\n", h[1] / 512.0);
      for (int rep = 0; rep < 3; ++rep) k2<<<148, 128, 131072 + 1024>>>(d, 1, 128, 1, 256, 0);
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      printf("k2 TS N=128 MN D 256 A 0: per MMA %.1f\n", h[1] / 512.0);
    }
    return 0;
  }
  const char* names[] = {"8 PV N=128", "8 x (PV N=128, sum N=16)", "8 PV N=128 then 8 sum N=16", "8 PV N=144",
                         "8 sum N=16 alone"};
  for (int mode = 0; mode < 5; ++mode) {
    for (int rep = 0; rep < 3; ++rep) k<<<148, 128, smem>>>(d, mode);
    unsigned long long h[2];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-28s: per block issue %.1f cycles, complete %.1f cycles (%s)\n", names[mode], h[0] / 64.0, h[1] / 64.0,
           cudaGetErrorString(cudaGetLastError()));
  }
  cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072 + 1024);
  const int cfg[][3] = {{0, 128, 0}, {1, 128, 0}, {0, 128, 1}, {1, 128, 1}, {1, 64, 1}, {0, 64, 1}, {1, 256, 0},
                        {0, 256, 0}, {1, 256, 1}, {1, 64, 0}, {0, 64, 0}};
  for (auto& c : cfg) {
    for (int rep = 0; rep < 3; ++rep) k2<<<148, 128, 131072 + 1024>>>(d, c[0], c[1], c[2]);
    unsigned long long h[2];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%s N=%3d B %s: per MMA %.1f cycles (ideal %d) (%s)\n", c[0] ? "TS" : "SS", c[1], c[2] ? "MN-major" : "K-major ",
           h[1] / 512.0, c[1] / 2, cudaGetErrorString(cudaGetLastError()));
  }
  const int pl[][2] = {{0, 256}, {256, 0}, {0, 384}, {256, 384}, {128, 384}, {384, 0}, {0, 128}, {128, 0}};
  for (auto& q : pl) {
    for (int n : {128, 256}) {
      if (n == 256 && (q[0] == 384 || q[0] == 128 && q[1] < 384)) continue;
      for (int rep = 0; rep < 3; ++rep) k2<<<148, 128, 131072 + 1024>>>(d, 1, n, 1, q[0], q[1]);
      unsigned long long h[2];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      printf("TS N=%d D col %3d, A col %3d: per MMA %.1f cycles (%s)\n", n, q[0], q[1], h[1] / 512.0,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
