// tools/tmem_contention.cu — microbenchmark: does softmax-side TMEM traffic (tcgen05.ld of S,
// tcgen05.st of P) slow the tensor pipe? One warp issues K5's per-block MMA pattern (QK with
// A = Q from TMEM, PV with A = P from TMEM, B operands from smem) back to back; eight other
// warps optionally stream tcgen05.ld 16x32bx2.x64 + tcgen05.st 16x32bx2.x32 over the S columns,
// with `spin` cycles of ALU work between blocks to set their rate.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tmem_contention tools/tmem_contention.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2605_23445_b200/csrc/sm100.cuh"
using namespace dfsgpu::sm100;

template <int kMmaWarp>
__global__ void __launch_bounds__(320, 1) k(int iters, int traffic, int spin, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tbase;
  __shared__ uint64_t bar;
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
    done = 0;
  }
  if (warp == kMmaWarp) tmem_alloc<512>(&tbase);
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  if (warp == kMmaWarp) {
    unsigned long long t0 = clock64();
    if (lane == 0) {
      const uint32_t kslot = smem_u32(smem), vslot = kslot + 32768;
      const uint32_t idqk = idesc_bf16_f32(128, 128, false, false), idpv = idesc_bf16_f32(128, 128, false, true);
      for (int it = 0; it < iters; ++it) {
        const uint32_t sq = ((it + 2) % 2) * 128, sp = (it % 2) * 128;
#pragma unroll
        for (int s = 0; s < 8; ++s)
          umma_f16_ts(tmem + 256, tmem + sp + s * 8, smem_desc_sw128(vslot + s * 16 * 128, 16384, 1024), idpv, 1);
#pragma unroll
        for (int s = 0; s < 8; ++s) {
          const uint32_t off = (s >> 2) * 16384 + (s & 3) * 32;
          umma_f16_ts(tmem + sq, tmem + 384 + s * 8, smem_desc_sw128(kslot + off, 16, 1024), idqk, s > 0);
        }
      }
      umma_commit(&bar);
      mbar_wait(&bar, 0);
      out[blockIdx.x] = clock64() - t0;
      done = 1;
    }
    __syncwarp();
  } else if (warp >= 1 && warp != kMmaWarp && warp <= 9 && traffic == 3) {
    // pure FMA work on every SMSP: iterations completed while the MMAs run, per warp
    float a = threadIdx.x * 1e-3f, b2 = a + 1.f, c = a + 2.f, e = a + 3.f;
    unsigned long long n = 0;
    while (!done) {
      if (spin) {  // one dependent chain: ~25 % issue per warp, ~50 % per SMSP
#pragma unroll
        for (int i = 0; i < 256; ++i) a = fmaf(a, 0.999f, 1e-3f);
      } else {
#pragma unroll
        for (int i = 0; i < 64; ++i) {
          a = fmaf(a, 0.999f, 1e-3f);
          b2 = fmaf(b2, 0.999f, 1e-3f);
          c = fmaf(c, 0.999f, 1e-3f);
          e = fmaf(e, 0.999f, 1e-3f);
        }
      }
      ++n;
    }
    if (lane == 0) out[200 + blockIdx.x * 16 + warp] = n;
    if (a + b2 + c + e == 0.123f) out[1000] = 1;
  } else if (warp >= 2 && warp != kMmaWarp && traffic) {
    const int w = warp - 2, hf = w >> 2;
    const uint32_t lane_addr = uint32_t((warp & 3) * 32 + hf * 16) << 16;
    uint32_t acc = 0;
    int b = 0;
    while (!done) {
      uint32_t sv[64];
      tmem_ld16x2_x64<64>(tmem + lane_addr + (b & 1) * 128, sv);
      tmem_wait_ld();
      uint32_t pk[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) pk[i] = sv[2 * i] ^ sv[2 * i + 1] ^ acc;
      for (int i = 0; i < spin; ++i) acc = acc * 1664525u + 1013904223u;
      if (traffic > 1) {
        tmem_st16x2_x32<32>(tmem + lane_addr + (b & 1) * 128, pk);
        tmem_wait_st();
      }
      acc ^= pk[lane & 31];
      ++b;
    }
    if (acc == 0x12345678u) out[1000] = acc;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == kMmaWarp) tmem_dealloc<512>(tmem);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 4000 * sizeof(unsigned long long));
  const int smem = 65536 + 1024, iters = 4000;
  for (int mw : {1, 9}) {
    auto kern = mw == 1 ? k<1> : k<9>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int traffic : {0, 3, 4}) {
      const int spin = traffic == 4;
      if (traffic == 4) traffic = 3;
      kern<<<148, 320, smem>>>(iters, traffic, spin, d);
      kern<<<148, 320, smem>>>(iters, traffic, spin, d);
      unsigned long long c;
      cudaMemcpy(&c, d, sizeof(c), cudaMemcpyDeviceToHost);
      printf("MMA warp %d, %s: %.1f cycles per block of 16 MMAs (ideal 1024)  %s\n", mw,
             traffic ? (spin ? "8 latency-bound FMA warps (~50 % SMSP issue)" : "8 FMA-bound warps alongside") : "alone", double(c) / iters, cudaGetErrorString(cudaGetLastError()));
      if (traffic == 3) {
        unsigned long long w[16];
        cudaMemcpy(w, d + 200, sizeof(w), cudaMemcpyDeviceToHost);
        printf("  FMA loop iterations per warp (SMSP = warp %% 4):");
        for (int i = 1; i < 10; ++i)
          if (i != mw) printf(" w%d:%llu", i, w[i]);
        printf("\n");
      }
    }
  }
  return 0;
}
