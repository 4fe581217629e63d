// permute.cu — K2 (gather + fused mean-pool + finite check) and K6 (scatter).
//
// apply_permutation (curve.cpp:166-176) is a row gather out[i] = x[fwd[i]];
// here it runs for every head at once and converts [N,H,d] raster activations
// to the path's head-major [H,N,d] reordered layout. Pure data movement:
// HBM-bound, so every access is a 16-byte vector, the source row (H*d*2 bytes
// per token, 6 KB at HunyuanVideo) is read by consecutive threads, and each
// thread keeps `kUnroll` independent row loads in flight.
//
// When the destination rows are also needed as sub-block means for scoring
// (mask_builder.cpp:12-28 mean_pool: fp64 accumulate, divide by B_s even for
// the zero-padded last group, fp32 store) the CTA owns whole pooling groups and
// emits the pooled rows from registers: the scores never re-read Q/K.
#include <algorithm>

#include "common.cuh"

#ifndef DFS_PERMUTE_BATCH
#define DFS_PERMUTE_BATCH 8  // independent 16-byte row loads in flight per thread
#endif
#ifndef DFS_PERMUTE_CTA
#define DFS_PERMUTE_CTA 128  // most (head, 16-byte chunk) slots per CTA before splitting over blockIdx.y
#endif

namespace dfsgpu {

namespace {

template <typename T>
struct Vec;  // 16-byte vector of T
template <>
struct Vec<float> {
  static constexpr int N = 4;
};
template <>
struct Vec<__nv_bfloat16> {
  static constexpr int N = 8;
};

template <typename T>
__device__ __forceinline__ void unpack(const uint4& u, float (&x)[Vec<T>::N]);
template <>
__device__ __forceinline__ void unpack<float>(const uint4& u, float (&x)[4]) {
  x[0] = __uint_as_float(u.x);
  x[1] = __uint_as_float(u.y);
  x[2] = __uint_as_float(u.z);
  x[3] = __uint_as_float(u.w);
}
template <>
__device__ __forceinline__ void unpack<__nv_bfloat16>(const uint4& u, float (&x)[8]) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    x[2 * j] = __uint_as_float(w[j] << 16);
    x[2 * j + 1] = __uint_as_float(w[j] & 0xffff0000u);
  }
}

// One CTA = `rows` consecutive destination rows (a pooling group when pooling)
// x all heads. Thread slots walk (head, 16B column chunk).
// kPeer: the source is sequence-sharded over the ranks (dfs_peer_table, Ulysses): token
// si of head h lives in rank si / n_local's [n_local, H, d] shard, row si % n_local,
// head h0 + h — read over NVLink from the peer's memory (plain loads: no .nc on peers).
template <typename T, bool kPool, bool kScatter, bool kPeer = false>
__global__ void __launch_bounds__(1024) permute_kernel(const T* __restrict__ src, int src_layout,
                                                      T* __restrict__ dst, int dst_layout,
                                                      const uint32_t* __restrict__ idx, int64_t n,
                                                      int64_t heads, int64_t d, int rows,
                                                      float* __restrict__ pooled, int64_t pool,
                                                      int32_t* __restrict__ nonfinite,
                                                      const dfs_peer_table* __restrict__ peers = nullptr) {
  constexpr int V = Vec<T>::N;
  // independent 16-byte row loads in flight per thread, with the (head, chunk) slots split
  // over 128-thread CTAs (DFS_PERMUTE_CTA): more, smaller CTAs per SM and 8 loads each beat
  // 384-thread CTAs with 4 (round 2, tools/permute_bench.py: HY 0.693 -> 0.647 ms for the three
  // passes, W4 0.342 -> 0.311, C 0.131 -> 0.120; 16 in flight: 0.911; 384-thread CTAs with 8
  // in flight had lost to occupancy in round 1)
  constexpr int kBatch = kPeer ? 4 : DFS_PERMUTE_BATCH;  // the peer-pointer variant spills at 8
  const int64_t vec_per_row = d / V;
  const int64_t slots = heads * vec_per_row;
  const int64_t r0 = int64_t(blockIdx.x) * rows;
  // the CTA's row indices once in shared memory (rows <= 64): the per-row loads of the
  // slots below then have no dependent index load in front of them
  __shared__ int64_t s_src[64], s_dst[64];
  for (int t = threadIdx.x; t < rows; t += blockDim.x) {  // blockDim may be < rows for narrow rows
    const int64_t i = r0 + t;
    int64_t si = -1, di = -1;
    if (i < n) {
      si = kScatter ? i : int64_t(idx[i]);
      di = kScatter ? int64_t(idx[i]) : i;
      if (si >= n || di >= n) si = di = -1;  // invalid permutation entry: no wild access
    }
    if (kPeer && si >= 0) {  // absolute address of the row's head-group start in its owner's shard
      const int64_t r = si / peers->n_local;
      si = int64_t(reinterpret_cast<uintptr_t>(static_cast<const T*>(peers->ptr[r]) +
                                               ((si - r * peers->n_local) * peers->heads_total + peers->h0) * d));
    }
    s_src[t] = si;
    s_dst[t] = di;
  }
  __syncthreads();
  bool bad = false;
  // slots split over blockIdx.y when one CTA would need more than DFS_PERMUTE_CTA threads
  // (HY: 24 heads x 16 chunks = 384 slots -> 3 x 128)
  for (int64_t s = int64_t(blockIdx.y) * blockDim.x + threadIdx.x; s < slots; s += int64_t(gridDim.y) * blockDim.x) {
    const int64_t h = s / vec_per_row;
    const int64_t c = (s % vec_per_row) * V;
#ifdef DFS_PERMUTE_POOL_F32  // experiment builds only: fp32 sums (not the reference's rounding)
    using Acc = float;
#else
    using Acc = double;
#endif
    Acc acc[kPool ? V : 1];
    if (kPool) {
#pragma unroll
      for (int j = 0; j < V; ++j) acc[j] = 0.0;
    }
    for (int rb = 0; rb < rows; rb += kBatch) {
      uint4 u[kBatch];
#pragma unroll
      for (int k = 0; k < kBatch; ++k) {
        const int64_t si = rb + k < rows ? s_src[rb + k] : -1;
        if constexpr (kPeer)
          u[k] = si >= 0 ? *reinterpret_cast<const uint4*>(reinterpret_cast<const T*>(si) + h * d + c)
                         : make_uint4(0u, 0u, 0u, 0u);
        else
          u[k] = si >= 0 ? __ldg(reinterpret_cast<const uint4*>(src + row_offset(src_layout, n, heads, d, h, si) + c))
                         : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int k = 0; k < kBatch; ++k) {
        if (rb + k >= rows) break;
        const int64_t di = s_dst[rb + k];
        if (di < 0) continue;
        if (dst) *reinterpret_cast<uint4*>(dst + row_offset(dst_layout, n, heads, d, h, di) + c) = u[k];
        if (kPool || nonfinite) {
          float x[V];
          unpack<T>(u[k], x);
#pragma unroll
          for (int j = 0; j < V; ++j) {
            if (kPool) acc[j] += Acc(x[j]);
            bad |= !isfinite(x[j]);
          }
        }
      }
    }
    if (kPool) {
      const int64_t g = r0 / pool;
      float* out = pooled + (h * ceil_div(n, pool) + g) * d + c;
#pragma unroll
      for (int j = 0; j < V; ++j) out[j] = float(acc[j] / Acc(pool));
    }
  }
  if (nonfinite && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(nonfinite, 1);
}

// scalar fallback for d not a multiple of the 16-byte vector (drop-in shapes)
template <typename T, bool kScatter>
__global__ void permute_scalar_kernel(const T* __restrict__ src, int src_layout, T* __restrict__ dst,
                                      int dst_layout, const uint32_t* __restrict__ idx, int64_t n,
                                      int64_t heads, int64_t d, float* __restrict__ pooled,
                                      int64_t pool, int32_t* __restrict__ nonfinite) {
  // one CTA per pooling group (or per 16 rows), one thread per (head, column)
  const int64_t rows = pooled ? pool : 16;
  const int64_t r0 = int64_t(blockIdx.x) * rows;
  bool bad = false;
  for (int64_t s = threadIdx.x; s < heads * d; s += blockDim.x) {
    const int64_t h = s / d, c = s % d;
    double acc = 0.0;
    for (int64_t r = 0; r < rows; ++r) {
      const int64_t i = r0 + r;
      if (i >= n) break;
      const int64_t si = kScatter ? i : int64_t(idx[i]);
      const int64_t di = kScatter ? int64_t(idx[i]) : i;
      if (si >= n || di >= n) continue;
      const T x = src[row_offset(src_layout, n, heads, d, h, si) + c];
      if (dst) dst[row_offset(dst_layout, n, heads, d, h, di) + c] = x;
      const float xf = to_f32<T>(x);
      acc += double(xf);
      bad |= !isfinite(xf);
    }
    if (pooled) pooled[(h * ceil_div(n, pool) + r0 / pool) * d + c] = float(acc / double(pool));
  }
  if (nonfinite && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(nonfinite, 1);
}

template <typename T, bool kScatter>
int launch(const void* src, int src_layout, void* dst, int dst_layout, const uint32_t* idx, int64_t n,
           int64_t heads, int64_t d, float* pooled, int64_t pool, int32_t* nonfinite, cudaStream_t stream) {
  const T* s = static_cast<const T*>(src);
  T* o = static_cast<T*>(dst);
  // dst == NULL: read-only pass (pooled rows and/or the finite check of a gathered order)
  const bool vec_ok = d % Vec<T>::N == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0 &&
                      (reinterpret_cast<uintptr_t>(dst) & 15) == 0 && (!pooled || pool <= 64);
  // (rows per CTA: the pooling group, or 16; both <= 64 as the kernel's index cache requires)
  const int64_t rows = pooled ? pool : 16;
  const int64_t grid = ceil_div(n, rows);
  if (grid > int64_t(INT32_MAX)) return fail(DFS_E_UNSUPPORTED, "permute: too many rows");
  if (vec_ok) {
    // one thread per (head, 16-byte column chunk) slot when that fits a CTA: every thread
    // then walks the CTA's rows once (no second round for a remainder of slots)
    const int64_t slots = heads * (d / Vec<T>::N);
    const int64_t ysplit = ceil_div(slots, int64_t(DFS_PERMUTE_CTA));
    const int threads = int(ceil_div(ceil_div(slots, ysplit), 32) * 32);
    const dim3 g{unsigned(grid), unsigned(ysplit), 1u};
    if (ysplit > 65535) return fail(DFS_E_UNSUPPORTED, "permute: rows too wide");
    if (pooled)
      permute_kernel<T, true, kScatter><<<g, threads, 0, stream>>>(s, src_layout, o, dst_layout, idx, n, heads, d,
                                                                  int(rows), pooled, pool, nonfinite);
    else
      permute_kernel<T, false, kScatter><<<g, threads, 0, stream>>>(s, src_layout, o, dst_layout, idx, n, heads, d,
                                                                   int(rows), nullptr, 1, nonfinite);
  } else {
    permute_scalar_kernel<T, kScatter><<<unsigned(grid), 256, 0, stream>>>(
        s, src_layout, o, dst_layout, idx, n, heads, d, pooled, pool, nonfinite);
  }
  DFS_LAUNCH_CHECK("permute_rows");
  return DFS_OK;
}

template <typename T>
__global__ void finite_kernel(const T* __restrict__ x, int64_t count, int32_t* __restrict__ flag) {
  bool bad = false;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x)
    bad |= !isfinite(to_f32<T>(x[i]));
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// fp32 -> bf16 (RNE) with the finite check of the source folded in; 8 elements per
// thread as two 16-byte loads and one 16-byte store
__global__ void cast_f32_bf16_kernel(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst, int64_t count,
                                     int32_t* __restrict__ nonfinite) {
  bool bad = false;
  const int64_t n8 = count / 8;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n8; i += stride) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(src) + 2 * i);
    const float4 b = __ldg(reinterpret_cast<const float4*>(src) + 2 * i + 1);
    const float x[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      bad |= !isfinite(x[2 * j]) || !isfinite(x[2 * j + 1]);
      const __nv_bfloat162 p = __floats2bfloat162_rn(x[2 * j], x[2 * j + 1]);
      w[j] = *reinterpret_cast<const uint32_t*>(&p);
    }
    reinterpret_cast<uint4*>(dst)[i] = make_uint4(w[0], w[1], w[2], w[3]);
  }
  for (int64_t i = n8 * 8 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count; i += stride) {
    bad |= !isfinite(src[i]);
    dst[i] = __float2bfloat16_rn(src[i]);
  }
  if (nonfinite && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(nonfinite, 1);
}

__global__ void cast_bf16_f32_kernel(const __nv_bfloat16* __restrict__ src, float* __restrict__ dst, int64_t count,
                                     int32_t* __restrict__ nonfinite) {
  bool bad = false;
  const int64_t n8 = count / 8;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n8; i += stride) {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(src) + i);
    float x[8];
    unpack<__nv_bfloat16>(u, x);
#pragma unroll
    for (int j = 0; j < 8; ++j) bad |= !isfinite(x[j]);
    reinterpret_cast<float4*>(dst)[2 * i] = make_float4(x[0], x[1], x[2], x[3]);
    reinterpret_cast<float4*>(dst)[2 * i + 1] = make_float4(x[4], x[5], x[6], x[7]);
  }
  for (int64_t i = n8 * 8 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count; i += stride) {
    const float x = __bfloat162float(src[i]);
    bad |= !isfinite(x);
    dst[i] = x;
  }
  if (nonfinite && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(nonfinite, 1);
}

// K2 with the QK-norm / RoPE prologue (dfs_qk_prologue): bf16 [N, H, d] raster rows,
// RMS-normalised and rotated in registers, rounded to bf16, written to `dst` (reordered
// [H, N, d], or raster [N, H, d] for a dense step) and pooled. One thread per (head,
// 16-byte chunk) slot; a row's d/8 chunks sit in consecutive lanes, so the row's sum of
// squares and the rotate_half partner exchange are warp shuffles.
__global__ void __launch_bounds__(1024) prologue_kernel(const __nv_bfloat16* __restrict__ src,
                                                       __nv_bfloat16* __restrict__ dst, int dst_layout,
                                                       const uint32_t* __restrict__ idx, int64_t n, int64_t heads,
                                                       int64_t d, int rows, float* __restrict__ pooled,
                                                       int64_t pool, int32_t* __restrict__ nonfinite,
                                                       const float* __restrict__ nw, float eps, int rope_layout,
                                                       const float* __restrict__ cos_t,
                                                       const float* __restrict__ sin_t) {
  const int vpr = int(d / 8);  // 8 or 16 chunks per row: a power of two that divides 32
  const int64_t slots = heads * vpr;
  const int64_t s = int64_t(blockIdx.y) * blockDim.x + threadIdx.x;
  const bool active = s < slots;
  const int64_t h = active ? s / vpr : 0;
  const int c = int(s % vpr) * 8;
  const int64_t r0 = int64_t(blockIdx.x) * rows;
  __shared__ int64_t s_src[64], s_dst[64];
  for (int t = threadIdx.x; t < rows; t += blockDim.x) {
    const int64_t i = r0 + t;
    int64_t si = -1;
    if (i < n) si = idx ? int64_t(idx[i]) : i;
    if (si >= n) si = -1;
    s_src[t] = si;
    s_dst[t] = si >= 0 ? i : -1;
  }
  __syncthreads();
  float w[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) w[j] = nw && active ? nw[c + j] : 1.f;
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  bool bad = false;
  const int half = int(d / 2);
  for (int r = 0; r < rows; ++r) {
    const int64_t si = s_src[r], di = s_dst[r];
    if (si < 0) continue;  // CTA-uniform
    const uint4 u = active ? __ldg(reinterpret_cast<const uint4*>(src + (si * heads + h) * d + c))
                           : make_uint4(0u, 0u, 0u, 0u);
    float x[8];
    unpack<__nv_bfloat16>(u, x);
#pragma unroll
    for (int j = 0; j < 8; ++j) bad |= !isfinite(x[j]);
    if (nw) {
      float ss = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) ss = fmaf(x[j], x[j], ss);
      for (int o = vpr / 2; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      const float rs = 1.f / sqrtf(ss / float(d) + eps);
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = x[j] * rs * w[j];
    }
    if (rope_layout == DFS_ROPE_INTERLEAVED) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float co = active ? __ldg(cos_t + si * half + c / 2 + i) : 0.f;
        const float sn = active ? __ldg(sin_t + si * half + c / 2 + i) : 0.f;
        const float a = x[2 * i], b = x[2 * i + 1];
        x[2 * i] = a * co - b * sn;
        x[2 * i + 1] = a * sn + b * co;
      }
    } else if (rope_layout == DFS_ROPE_HALF) {
      float y[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) y[j] = __shfl_xor_sync(0xffffffffu, x[j], vpr / 2);
      const bool lo = c < half;
      const int t0 = lo ? c : c - half;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float co = active ? __ldg(cos_t + si * half + t0 + j) : 0.f;
        const float sn = active ? __ldg(sin_t + si * half + t0 + j) : 0.f;
        x[j] = lo ? x[j] * co - y[j] * sn : x[j] * co + y[j] * sn;
      }
    }
    uint32_t pk[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const __nv_bfloat162 p2 = __floats2bfloat162_rn(x[2 * j], x[2 * j + 1]);
      pk[j] = *reinterpret_cast<const uint32_t*>(&p2);
      if (pooled) {
        acc[2 * j] += double(__low2float(p2));
        acc[2 * j + 1] += double(__high2float(p2));
      }
    }
    if (active && dst)
      *reinterpret_cast<uint4*>(dst + row_offset(dst_layout, n, heads, d, h, di) + c) =
          make_uint4(pk[0], pk[1], pk[2], pk[3]);
  }
  if (pooled && active) {
    float* out = pooled + (h * ceil_div(n, pool) + r0 / pool) * d + c;
#pragma unroll
    for (int j = 0; j < 8; ++j) out[j] = float(acc[j] / double(pool));
  }
  if (nonfinite && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(nonfinite, 1);
}

}  // namespace

int prologue_permute_impl(const void* src, void* dst, int dst_layout, const uint32_t* idx, int64_t n, int64_t heads,
                          int64_t d, float* pooled, int64_t pool, int32_t* nonfinite, const float* norm_weight,
                          float eps, int rope_layout, const float* cos_t, const float* sin_t, cudaStream_t stream) {
  if (d % 16 || d / 8 > 32) return fail(DFS_E_UNSUPPORTED, "qk prologue: d must be a multiple of 16, <= 256");
  if ((pooled && (pool < 1 || pool > 64)) || (reinterpret_cast<uintptr_t>(src) & 15) ||
      (reinterpret_cast<uintptr_t>(dst) & 15))
    return fail(DFS_E_UNSUPPORTED, "qk prologue: pool <= 64 and 16-byte aligned buffers");
  if (rope_layout != DFS_ROPE_NONE && (!cos_t || !sin_t))
    return fail(DFS_E_INVALID, "qk prologue: RoPE tables missing");
  const int64_t rows = pooled ? pool : 16;
  const int64_t grid = ceil_div(n, rows);
  const int64_t slots = heads * (d / 8);
  const int64_t ysplit = ceil_div(slots, 512);
  const int threads = int(ceil_div(ceil_div(slots, ysplit), 32) * 32);
  if (grid > int64_t(INT32_MAX) || ysplit > 65535) return fail(DFS_E_UNSUPPORTED, "qk prologue: too many rows");
  prologue_kernel<<<dim3(unsigned(grid), unsigned(ysplit)), threads, 0, stream>>>(
      static_cast<const __nv_bfloat16*>(src), static_cast<__nv_bfloat16*>(dst), dst_layout, idx, n, heads, d,
      int(rows), pooled, pool, nonfinite, norm_weight, eps, rope_layout, cos_t, sin_t);
  DFS_LAUNCH_CHECK("qk_prologue");
  return DFS_OK;
}

// K2 over sequence-sharded peers (Ulysses): gather + pool + finite check of this rank's
// head group, bf16 only, destination [heads, n, d] (HND) or NULL (read-only pooling pass)
int permute_rows_peer_impl(const dfs_peer_table* peers_dev, int64_t heads_total, void* dst, const uint32_t* idx,
                           int64_t n, int64_t heads, int64_t d, float* pooled, int64_t pool, int32_t* nonfinite,
                           cudaStream_t stream) {
  using T = __nv_bfloat16;
  if (d % 8 || (pooled && pool > 64) || (reinterpret_cast<uintptr_t>(dst) & 15))
    return fail(DFS_E_UNSUPPORTED, "alltoall: d must be a multiple of 8 and pool <= 64");
  const int64_t rows = pooled ? pool : 16;
  const int64_t grid = ceil_div(n, rows);
  const int64_t slots = heads * (d / 8);
  const int64_t ysplit = ceil_div(slots, int64_t(DFS_PERMUTE_CTA));
  const int threads = int(ceil_div(ceil_div(slots, ysplit), 32) * 32);
  if (grid > int64_t(INT32_MAX) || ysplit > 65535) return fail(DFS_E_UNSUPPORTED, "alltoall: too many rows");
  (void)heads_total;
  const dim3 g{unsigned(grid), unsigned(ysplit), 1u};
  if (pooled)
    permute_kernel<T, true, false, true><<<g, threads, 0, stream>>>(nullptr, DFS_NHD, static_cast<T*>(dst), DFS_HND,
                                                                   idx, n, heads, d, int(rows), pooled, pool,
                                                                   nonfinite, peers_dev);
  else
    permute_kernel<T, false, false, true><<<g, threads, 0, stream>>>(nullptr, DFS_NHD, static_cast<T*>(dst),
                                                                    DFS_HND, idx, n, heads, d, int(rows), nullptr, 1,
                                                                    nonfinite, peers_dev);
  DFS_LAUNCH_CHECK("permute_rows_peer");
  return DFS_OK;
}

int cast_impl(const void* src, int src_dtype, void* dst, int dst_dtype, int64_t count, int32_t* nonfinite,
              cudaStream_t stream) {
  if (count < 0) return fail(DFS_E_INVALID, "cast: negative count");
  if (count == 0) return DFS_OK;
  if ((reinterpret_cast<uintptr_t>(src) & 15) || (reinterpret_cast<uintptr_t>(dst) & 15))
    return fail(DFS_E_UNSUPPORTED, "cast: buffers must be 16-byte aligned");
  const int64_t blocks = std::min<int64_t>(ceil_div(ceil_div(count, 8), 256), 16 * kNumSMs);
  if (src_dtype == DFS_F32 && dst_dtype == DFS_BF16)
    cast_f32_bf16_kernel<<<unsigned(blocks), 256, 0, stream>>>(static_cast<const float*>(src),
                                                               static_cast<__nv_bfloat16*>(dst), count, nonfinite);
  else if (src_dtype == DFS_BF16 && dst_dtype == DFS_F32)
    cast_bf16_f32_kernel<<<unsigned(blocks), 256, 0, stream>>>(static_cast<const __nv_bfloat16*>(src),
                                                               static_cast<float*>(dst), count, nonfinite);
  else
    return fail(DFS_E_INVALID, "cast: only f32 <-> bf16");
  DFS_LAUNCH_CHECK("cast");
  return DFS_OK;
}

// attention.cpp:19-20 (non-finite input is an error) for the dense-step path
int finite_check_impl(const void* x, int64_t count, int dtype, int32_t* flag, cudaStream_t stream) {
  const int64_t blocks = ceil_div(count, 256) < 8 * kNumSMs ? ceil_div(count, 256) : 8 * kNumSMs;
  if (dtype == DFS_BF16)
    finite_kernel<<<unsigned(blocks), 256, 0, stream>>>(static_cast<const __nv_bfloat16*>(x), count, flag);
  else
    finite_kernel<<<unsigned(blocks), 256, 0, stream>>>(static_cast<const float*>(x), count, flag);
  DFS_LAUNCH_CHECK("finite_check");
  return DFS_OK;
}

int permute_rows_impl(const void* src, int src_layout, void* dst, int dst_layout, int dtype,
                      const uint32_t* idx, int64_t n, int64_t heads, int64_t d, float* pooled,
                      int64_t pool, int32_t* nonfinite, bool scatter, cudaStream_t stream) {
  if (n < 1 || heads < 1 || d < 1) return fail(DFS_E_INVALID, "permute_rows: empty input");
  if (pooled && pool < 1) return fail(DFS_E_INVALID, "mean_pool: pool must be >= 1");
  if (pooled && scatter) return fail(DFS_E_INVALID, "permute_rows: pooling only on gather");
  if (dtype == DFS_BF16)
    return scatter ? launch<__nv_bfloat16, true>(src, src_layout, dst, dst_layout, idx, n, heads, d, pooled,
                                                 pool, nonfinite, stream)
                   : launch<__nv_bfloat16, false>(src, src_layout, dst, dst_layout, idx, n, heads, d,
                                                  pooled, pool, nonfinite, stream);
  if (dtype == DFS_F32)
    return scatter ? launch<float, true>(src, src_layout, dst, dst_layout, idx, n, heads, d, pooled, pool,
                                         nonfinite, stream)
                   : launch<float, false>(src, src_layout, dst, dst_layout, idx, n, heads, d, pooled, pool,
                                          nonfinite, stream);
  return fail(DFS_E_INVALID, "permute_rows: unknown dtype");
}

}  // namespace dfsgpu
