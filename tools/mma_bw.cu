// tools/mma_bw.cu — microbenchmark: tcgen05.mma throughput per SM for the K5 shapes
// (M=128, N=128, K=16 bf16; SS = both operands in smem, TS = A in TMEM), with and
// without concurrent TMA traffic into shared memory.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mma_bw tools/mma_bw.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>

#include "../paper_2605_23445_b200/csrc/sm100.cuh"

using namespace dfsgpu::sm100;

template <int mode, int n_dim>
__global__ void __launch_bounds__(128, 1) mma_kernel(int iters, unsigned long long* out,
                                                       const __grid_constant__ CUtensorMap map, int tma) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tbase;
  __shared__ uint64_t bar, tbar[2];
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&tbar[0], 1);
    mbar_init(&tbar[1], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&tbase);
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  const uint32_t a = smem_u32(smem), b = a + 32768;
  const uint32_t idesc = idesc_bf16_f32(128, n_dim, false, false);
  unsigned long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (mode == 12) {  // mode 10 with Q resident in TMEM (QK as TS: A = Q from TMEM cols 256..319), 2 S buffers
        const uint32_t sq = ((it + 2) % 2) * 128, sp = (it % 2) * 128;
        const uint32_t ring = a + 32768;
        const uint32_t kslot = ring + uint32_t((2 * it) % 5) * 32768, vslot = ring + uint32_t((2 * it + 1) % 5) * 32768;
#pragma unroll
        for (int s = 0; s < 8; ++s) {
          const uint32_t off = (s >> 2) * 16384 + (s & 3) * 32;
          umma_f16_ts(tmem + sq, tmem + 256 + s * 8, smem_desc_sw128(kslot + off, 16, 1024), idesc, s > 0);
        }
#pragma unroll
        for (int s = 0; s < 8; ++s)
          umma_f16_ts(tmem + 384, tmem + sp + s * 8, smem_desc_sw128(vslot + s * 16 * 128, 16384, 1024),
                      idesc_bf16_f32(128, n_dim, false, true), 1);
        continue;
      }
      if (mode == 10 || mode == 11) {  // mode 8's order with K/V operands rotating through 5 ring slots of 32 KB
        const uint32_t sq = ((it + 2) % 3) * 128, sp = (it % 3) * 128;
        const uint32_t ring = a + 32768;  // Q at a (32 KB), ring after it
        const uint32_t kslot = ring + uint32_t((2 * it) % 5) * 32768, vslot = ring + uint32_t((2 * it + 1) % 5) * 32768;
#pragma unroll
        for (int s = 0; s < 8; ++s) {
          const uint32_t off = (s >> 2) * 16384 + (s & 3) * 32;
          umma_f16(tmem + sq, smem_desc_sw128(a + off, 16, 1024), smem_desc_sw128(kslot + off, 16, 1024), idesc, s > 0);
        }
        if (mode == 11) {  // K5 commits two mbarriers after every group (kv_empty + s_full / o_done)
          umma_commit(&tbar[0]);
          umma_commit(&tbar[1]);
        }
#pragma unroll
        for (int s = 0; s < 8; ++s)
          umma_f16_ts(tmem + 384, tmem + sp + s * 8, smem_desc_sw128(vslot + s * 16 * 128, 16384, 1024),
                      idesc_bf16_f32(128, n_dim, false, true), 1);
        if (mode == 11) {
          umma_commit(&tbar[0]);
          umma_commit(&tbar[1]);
        }
        continue;
      }
      if (mode == 8 || mode == 9) {  // 3 S buffers: QK_{j+2} -> S[(j+2)%3], PV_j reads P_j from S[j%3]
        const uint32_t sq = ((it + 2) % 3) * 128, sp = (it % 3) * 128;
        if (mode == 8) {  // K5 r1 order: QK_{j+2} then PV_j (the next QK overwrites the buffer PV_j just read)
#pragma unroll
          for (int s = 0; s < 8; ++s) {
            const uint32_t off = (s >> 2) * 16384 + (s & 3) * 32;
            umma_f16(tmem + sq, smem_desc_sw128(a + off, 16, 1024), smem_desc_sw128(b + off, 16, 1024), idesc, s > 0);
          }
#pragma unroll
          for (int s = 0; s < 8; ++s)
            umma_f16_ts(tmem + 384, tmem + sp + s * 8, smem_desc_sw128(b + s * 16 * 128, 16384, 1024),
                        idesc_bf16_f32(128, n_dim, false, true), 1);
        } else {  // PV_j then QK_{j+2}
#pragma unroll
          for (int s = 0; s < 8; ++s)
            umma_f16_ts(tmem + 384, tmem + sp + s * 8, smem_desc_sw128(b + s * 16 * 128, 16384, 1024),
                        idesc_bf16_f32(128, n_dim, false, true), 1);
#pragma unroll
          for (int s = 0; s < 8; ++s) {
            const uint32_t off = (s >> 2) * 16384 + (s & 3) * 32;
            umma_f16(tmem + sq, smem_desc_sw128(a + off, 16, 1024), smem_desc_sw128(b + off, 16, 1024), idesc, s > 0);
          }
        }
        continue;
      }
      if (mode == 7) {  // K5 order, unrolled: 8 SS (QK into S[it&1]) then 8 TS (PV into O), per iteration
#pragma unroll
        for (int s = 0; s < 8; ++s) {
          const uint32_t off = (s >> 2) * 16384 + (s & 3) * 32;
          umma_f16(tmem + (it & 1) * 128, smem_desc_sw128(a + off, 16, 1024), smem_desc_sw128(b + off, 16, 1024),
                   idesc, s > 0);
        }
#pragma unroll
        for (int s = 0; s < 8; ++s)
          umma_f16_ts(tmem + 256, tmem + (it & 1) * 128 + s * 8, smem_desc_sw128(b + s * 16 * 128, 16384, 1024),
                      idesc_bf16_f32(128, n_dim, false, true), 1);
        continue;
      }
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const uint32_t off = (s >> 2) * 16384 + (s & 3) * 32;
        if (mode == 0)
          umma_f16(tmem + (it & 1) * 128, smem_desc_sw128(a + off, 16, 1024), smem_desc_sw128(b + off, 16, 1024), idesc,
                   s > 0);
        else if (mode == 1)
          umma_f16_ts(tmem + (it & 1) * 128, tmem + 384 + s * 8, smem_desc_sw128(b + off, 16, 1024), idesc, s > 0);
        else if (mode == 2)  // two independent SS accumulation chains, interleaved
          umma_f16(tmem + (s & 1) * 128, smem_desc_sw128(a + off, 16, 1024), smem_desc_sw128(b + off, 16, 1024), idesc,
                   s > 1);
        else if (mode == 3) {  // K5 pattern: SS (QK into S) interleaved with TS (PV into O)
          if (s & 1)
            umma_f16_ts(tmem + 256, tmem + 384 + s * 8, smem_desc_sw128(b + off, 16, 1024), idesc, s > 1);
          else
            umma_f16(tmem + (it & 1) * 128, smem_desc_sw128(a + off, 16, 1024), smem_desc_sw128(b + off, 16, 1024),
                     idesc, s > 1);
        } else if (mode == 5) {  // TS with an MN-major B operand (K5's V: 64-col chunks, LBO = 16 KB)
          const uint32_t vb = b + s * 16 * 128;
          umma_f16_ts(tmem + (it & 1) * 128, tmem + 384 + s * 8, smem_desc_sw128(vb, 16384, 1024),
                      idesc_bf16_f32(128, n_dim, false, true), s > 0);
        } else if (mode == 6) {  // SS with an MN-major B operand
          const uint32_t vb = b + s * 16 * 128;
          umma_f16(tmem + (it & 1) * 128, smem_desc_sw128(a + off, 16, 1024), smem_desc_sw128(vb, 16384, 1024),
                   idesc_bf16_f32(128, n_dim, false, true), s > 0);
        } else {  // mode 4: 8 SS into S then 8 TS into O (current K5 issue order), per pair of its
          if (it & 1)
            umma_f16_ts(tmem + 256, tmem + 384 + s * 8, smem_desc_sw128(b + off, 16, 1024), idesc, s > 0);
          else
            umma_f16(tmem + 128 * ((it >> 1) & 1), smem_desc_sw128(a + off, 16, 1024), smem_desc_sw128(b + off, 16, 1024),
                     idesc, s > 0);
        }
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  } else if (threadIdx.x == 32 && tma) {
    // concurrent TMA stream into a separate 2 x 32 KB region (L2-resident source)
    uint8_t* dst = smem + 65536;
    for (int t = 0; t < tma; ++t) {
      const int slot = t & 1;
      if (t >= 2) mbar_wait(&tbar[slot], ((t >> 1) - 1) & 1);
      mbar_expect_tx(&tbar[slot], 32768);
      tma_load_3d(dst + slot * 32768, &map, &tbar[slot], 0, (t * 7 % 900) * 128, 0);
      tma_load_3d(dst + slot * 32768 + 16384, &map, &tbar[slot], 64, (t * 7 % 900) * 128, 0);
    }
    for (int t = (tma > 2 ? tma - 2 : 0); t < tma; ++t) mbar_wait(&tbar[t & 1], (t >> 1) & 1);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

using KFn = void (*)(int, unsigned long long*, const CUtensorMap, int);
template <int M>
KFn pick_n(int n) {
  if (n == 64) return mma_kernel<M, 64>;
  if (n == 128) return mma_kernel<M, 128>;
  return mma_kernel<M, 256>;
}
KFn pick(int mode, int n) {
  switch (mode) {
    case 0: return pick_n<0>(n);
    case 1: return pick_n<1>(n);
    case 2: return pick_n<2>(n);
    case 3: return pick_n<3>(n);
    case 4: return pick_n<4>(n);
    case 5: return pick_n<5>(n);
    case 6: return pick_n<6>(n);
    case 7: return pick_n<7>(n);
    case 8: return pick_n<8>(n);
    case 9: return pick_n<9>(n);
    case 10: return pick_n<10>(n);
    case 11: return pick_n<11>(n);
    default: return pick_n<12>(n);
  }
}

int main() {
  void* ptr = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)ptr;
  void* buf;
  const int rows = 118912;
  cudaMalloc(&buf, size_t(rows) * 256);
  cudaMemset(buf, 0, size_t(rows) * 256);
  CUtensorMap map;
  cuuint64_t dims[3] = {128, (cuuint64_t)rows, 1};
  cuuint64_t strides[2] = {256, (cuuint64_t)rows * 256};
  cuuint32_t box[3] = {64, 128, 1}, es[3] = {1, 1, 1};
  enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  unsigned long long* d;
  cudaMalloc(&d, 148 * sizeof(unsigned long long));
  const int smem = 32768 * 6 + 1024;
  const int iters = 4000;
  for (int mode = 0; mode < 13; ++mode)
    for (int n : {64, 128, 256})
      for (int tma : {0, 4000, 8000, 16000}) {
        if (mode == 11 && tma) continue;  // its commits share tbar with the TMA stream
        if (tma == 16000 && mode < 10) continue;
        if (n == 256 && mode >= 2 && mode < 5) continue;
        if (n == 256 && mode >= 5) continue;
        if (tma && !(mode >= 7 || mode == 0) ) continue;
        if (n != 128 && tma) continue;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        auto kern = pick(mode, n);
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        kern<<<148, 128, smem>>>(iters, d, map, tma);
        cudaEventRecord(e0);
        kern<<<148, 128, smem>>>(iters, d, map, tma);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long c[148];
        cudaMemcpy(c, d, sizeof(c), cudaMemcpyDeviceToHost);
        const double flops = 2.0 * 128 * n * 16 * 8.0 * iters * 148 * (mode >= 7 ? 2 : 1);
        printf("%s N=%d tma_tiles=%d: %.1f cyc/MMA (clk64), %.3f ms, %.0f TFLOP/s  err=%s\n", (const char*[]){"SS", "TS", "SSx2", "SS+TS", "SS8+TS8", "TS-MNmajorB", "SS-MNmajorB", "K5:SS8,TS8(P=S)", "3buf:QK(j+2),PV(j)", "3buf:PV(j),QK(j+2)", "3buf+5 ring slots", "3buf+ring+commits", "Q-in-TMEM(TS QK)+ring"}[mode], n, tma,
               double(c[0]) / (iters * 8 * (mode >= 7 ? 2 : 1)), ms, flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
