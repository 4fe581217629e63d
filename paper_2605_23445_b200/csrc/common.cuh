// common.cuh — shared device/host helpers for the sm_100a kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <nvtx3/nvToolsExt.h>

#include <string>

#include "dfs_gpu.h"

namespace dfsgpu {

// thread-local error message behind dfs_last_error()
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);

#define DFS_CUDA_CHECK(expr)                                 \
  do {                                                       \
    cudaError_t _e = (expr);                                 \
    if (_e != cudaSuccess) return ::dfsgpu::cuda_fail(_e, #expr); \
  } while (0)

#define DFS_LAUNCH_CHECK(where)                                       \
  do {                                                                \
    cudaError_t _e = cudaGetLastError();                              \
    if (_e != cudaSuccess) return ::dfsgpu::cuda_fail(_e, where);     \
  } while (0)

inline cudaStream_t as_stream(dfs_stream s) { return reinterpret_cast<cudaStream_t>(s); }

// NVTX range over a C-ABI entry point (header-only NVTX3: free unless a profiler
// such as nsys / ncu --nvtx is attached); names the stage in timelines and lets
// ncu filter launches by range (--nvtx-include "dfs_run_step/").
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

constexpr int kNumSMs = 148;

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---- element access over both dtypes -------------------------------------
template <typename T>
__device__ __forceinline__ float to_f32(T x);
template <>
__device__ __forceinline__ float to_f32<float>(float x) { return x; }
template <>
__device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }

template <typename T>
__device__ __forceinline__ T from_f32(float x);
template <>
__device__ __forceinline__ float from_f32<float>(float x) { return x; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

// row address of (head h, token i) in NHD [N,H,d] or HND [H,N,d]
__host__ __device__ __forceinline__ int64_t row_offset(int layout, int64_t n, int64_t heads, int64_t d,
                                                       int64_t h, int64_t i) {
  return layout == DFS_NHD ? (i * heads + h) * d : (h * n + i) * d;
}

// ---- warp / block reductions ---------------------------------------------
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace dfsgpu
