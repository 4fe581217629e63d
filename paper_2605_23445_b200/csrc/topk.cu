// topk.cu — K4: per-row top-K block selection (mask_builder.cpp:82-113).
//
// The reference stable-sorts each score row by (value desc, index asc), keeps
// K and re-sorts ascending (top_indices, mask_builder.cpp:91-102). On device
// that is a rank selection, done per (head, query block) by one CTA entirely
// in shared memory:
//   1. map each fp64 score to an order-preserving u64 key (+0.0 for zeros so
//      -0.0 ties +0.0 like the reference's `!=` comparison);
//   2. MSB-first 8-bit radix select finds the K-th largest key T and how many
//      elements equal to T are still needed (`need`);
//   3. selected = key > T, or key == T among the first `need` such indices —
//      exactly the stable sort's tie rule;
//   4. a block scan over index order compacts the selection ascending into the
//      LUT row (and a 0/1 byte row when the BlockMask payload is requested).
// Given identical scores the output is bit-identical to the reference.
#include "common.cuh"

namespace dfsgpu {

namespace {

constexpr int kThreads = 256;

// order_key on the raw bits: -0.0 maps like +0.0
__device__ __forceinline__ uint64_t order_key_bits(uint64_t b) {
  if ((b << 1) == 0) b = 0;
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__device__ __forceinline__ uint64_t order_key(double x) {
  if (x == 0.0) x = 0.0;
  const uint64_t b = static_cast<uint64_t>(__double_as_longlong(x));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__device__ __forceinline__ int block_excl_scan(int v, int* warp_buf, int* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_buf[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int w = lane < kThreads / 32 ? warp_buf[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < kThreads / 32) warp_buf[lane] = w;
  }
  __syncthreads();
  const int excl = (wid ? warp_buf[wid - 1] : 0) + x - v;
  if (total) *total = warp_buf[kThreads / 32 - 1];
  __syncthreads();
  return excl;
}

__global__ void __launch_bounds__(kThreads) topk_kernel(const double* __restrict__ scores, int m, int k,
                                                        int32_t* __restrict__ lut, uint8_t* __restrict__ sel) {
  extern __shared__ uint64_t keys[];  // [m]
  __shared__ int hist[256];
  __shared__ int warp_buf[kThreads / 32];
  __shared__ uint64_t s_prefix;
  __shared__ int s_need;
  const int64_t row = blockIdx.x;  // h * m + u
  const double* srow = scores + row * m;
  for (int i = threadIdx.x; i < m; i += kThreads) keys[i] = order_key(srow[i]);
  if (threadIdx.x == 0) {
    s_prefix = 0;
    s_need = k;
  }
  __syncthreads();

  uint64_t prefix = 0, pmask = 0;
  for (int digit = 7; digit >= 0; --digit) {
    for (int i = threadIdx.x; i < 256; i += kThreads) hist[i] = 0;
    __syncthreads();
    const int shift = digit * 8;
    for (int i = threadIdx.x; i < m; i += kThreads) {
      const uint64_t key = keys[i];
      if ((key & pmask) == prefix) atomicAdd(&hist[(key >> shift) & 255], 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int need = s_need, cum = 0, b = 255;
      for (; b > 0; --b) {
        if (cum + hist[b] >= need) break;
        cum += hist[b];
      }
      s_need = need - cum;  // elements still needed from bucket b downward
      s_prefix = prefix | (uint64_t(b) << shift);
    }
    __syncthreads();
    prefix = s_prefix;
    pmask |= uint64_t(255) << shift;
  }
  const uint64_t T = prefix;
  const int need_eq = s_need;  // how many keys equal to T are selected (lowest indices first)

  // contiguous index chunk per thread keeps the scans in index order
  const int chunk = (m + kThreads - 1) / kThreads;
  const int lo = threadIdx.x * chunk, hi = min(lo + chunk, m);
  int eq = 0;
  for (int i = lo; i < hi; ++i) eq += keys[i] == T;
  int eq_before = block_excl_scan(eq, warp_buf, nullptr);
  int cnt = 0;
  for (int i = lo; i < hi; ++i) {
    const uint64_t key = keys[i];
    cnt += key > T || (key == T && eq_before++ < need_eq);
  }
  int pos = block_excl_scan(cnt, warp_buf, nullptr);
  eq_before -= eq;  // rewind for the write pass
  int32_t* lrow = lut ? lut + row * k : nullptr;
  uint8_t* brow = sel ? sel + row * m : nullptr;
  for (int i = lo; i < hi; ++i) {
    const uint64_t key = keys[i];
    const bool take = key > T || (key == T && eq_before++ < need_eq);
    if (take && lrow) lrow[pos] = i;
    pos += take;
    if (brow) brow[i] = take;
  }
}


// ---- warp-per-row path (M <= 32 * CH): keys live in registers ------------------
// Lane l holds the keys of blocks l, l + 32, ..., so a 32-wide chunk is one
// coalesced row segment and a ballot over a chunk is in index order. The K-th
// largest key T is found by bisection over the 64 key bits (MSB first), with an
// early exit as soon as exactly K keys lie at or above the probe (then the
// selection is those keys and no tie rule applies). Compaction: a ballot per
// chunk gives each selected block its ascending slot.
template <int CH>
__global__ void __launch_bounds__(128) topk_warp_kernel(const double* __restrict__ scores, int64_t rows, int m, int k,
                                                        int32_t* __restrict__ lut, uint8_t* __restrict__ sel) {
  const int lane = threadIdx.x & 31;
  const int64_t row = int64_t(blockIdx.x) * 4 + (threadIdx.x >> 5);
  if (row >= rows) return;
  const double* srow = scores + row * m;
  // all CH loads issued before any key is formed (a per-element load -> compare chain
  // serialised the row's L2 latency 32 times); keys from the raw bits with integer ops
  uint64_t key[CH];
  const unsigned long long* rbits = reinterpret_cast<const unsigned long long*>(srow);
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const int i = c * 32 + lane;
    key[c] = i < m ? __ldg(rbits + i) : 0ull;
  }
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    // padding (0) sorts below every real key: real keys have bit 63 set or are ~b of a
    // negative double, never 0 for finite input
    if (c * 32 + lane < m) key[c] = order_key_bits(key[c]);
  }
  // largest T with count(key >= T) >= k, built MSB-first; stop early once count == k at
  // the probe. Two 32-bit phases instead of one 64-bit pass: the high words decide almost
  // every row (sign, exponent and 20 mantissa bits), and a 32-bit compare is one
  // instruction where a 64-bit one is two.
  uint32_t hi[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) hi[c] = uint32_t(key[c] >> 32);
  // T lies between the smallest and the largest real key, so it shares every high bit above
  // the highest bit in which those two differ: start the bisection below that bit (block
  // scores are probabilities — sign and most exponent bits are common to a whole row)
  uint32_t hmin = 0xffffffffu, hmax = 0u;
#pragma unroll
  for (int c = 0; c < CH; ++c)
    if (c * 32 + lane < m) {
      hmin = min(hmin, hi[c]);
      hmax = max(hmax, hi[c]);
    }
  hmin = __reduce_min_sync(0xffffffffu, hmin);
  hmax = __reduce_max_sync(0xffffffffu, hmax);
  const uint32_t diff = hmin ^ hmax;
  const int top = diff ? 31 - __clz(diff) : -1;  // highest differing bit (-1: all high words equal)
  uint32_t t_hi = top < 0 ? hmin : top >= 31 ? 0u : hmin & ~((2u << top) - 1u);
  bool exact = false;
  for (int bit = top; bit >= 0; --bit) {
    const uint32_t cand = t_hi | (1u << bit);
    int c = 0;
#pragma unroll
    for (int j = 0; j < CH; ++j) c += hi[j] >= cand;
    c = __reduce_add_sync(0xffffffffu, c);
    if (c >= k) {
      t_hi = cand;
      if (c == k) {
        exact = true;
        break;
      }
    }
  }
  uint32_t t_lo = 0;
  if (!exact) {
    // count(hi > t_hi) < k <= count(hi >= t_hi): the rest is decided among hi == t_hi
    int gt = 0;
    uint32_t eq = 0;  // bit j: hi[j] == t_hi
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      gt += hi[j] > t_hi;
      eq |= uint32_t(hi[j] == t_hi) << j;
    }
    const int need = k - __reduce_add_sync(0xffffffffu, gt);
    for (int bit = 31; bit >= 0; --bit) {
      const uint32_t cand = t_lo | (1u << bit);
      int c = 0;
#pragma unroll
      for (int j = 0; j < CH; ++j) c += ((eq >> j) & 1u) && uint32_t(key[j]) >= cand;
      c = __reduce_add_sync(0xffffffffu, c);
      if (c >= need) {
        t_lo = cand;
        if (c == need) {
          exact = true;
          break;
        }
      }
    }
  }
  const uint64_t T = (uint64_t(t_hi) << 32) | t_lo;
  int need_eq = k;  // keys equal to T taken, lowest indices first (stable-sort tie rule)
  if (!exact) {
    int gt = 0;
#pragma unroll
    for (int j = 0; j < CH; ++j) gt += key[j] > T;
    need_eq = k - __reduce_add_sync(0xffffffffu, gt);
  }
  int32_t* lrow = lut ? lut + row * k : nullptr;
  uint8_t* brow = sel ? sel + row * m : nullptr;
  const uint32_t lt_mask = (1u << lane) - 1u;
  int pos = 0, eq_seen = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const int i = c * 32 + lane;
    bool take;
    if (exact) {
      take = i < m && key[c] >= T;
    } else {
      const bool eq = i < m && key[c] == T;
      const uint32_t eqb = __ballot_sync(0xffffffffu, eq);
      take = (i < m && key[c] > T) || (eq && eq_seen + __popc(eqb & lt_mask) < need_eq);
      eq_seen += __popc(eqb);
    }
    const uint32_t tb = __ballot_sync(0xffffffffu, take);
    if (take && lrow) lrow[pos + __popc(tb & lt_mask)] = i;
    if (brow && i < m) brow[i] = take;
    pos += __popc(tb);
  }
}

// BlockMask payload: bit (u, v) at idx = u*M + v, MSB-first (block_mask.hpp:36-48)
__global__ void pack_bits_kernel(const uint8_t* __restrict__ sel, int64_t m, int64_t bytes,
                                 uint8_t* __restrict__ bits) {
  const int64_t h = blockIdx.y;
  const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= bytes) return;
  const uint8_t* s = sel + h * m * m;
  uint8_t out = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int64_t idx = b * 8 + j;
    if (idx < m * m && s[idx]) out |= uint8_t(1u << (7 - j));
  }
  bits[h * bytes + b] = out;
}

// CSR from BlockMask payloads: one CTA per (head, row): count + ascending list
__global__ void bits_to_csr_count(const uint8_t* __restrict__ bits, int64_t m, int64_t bytes,
                                  int32_t* __restrict__ counts) {
  const int64_t row = blockIdx.x;
  const int64_t h = row / m, u = row % m;
  const uint8_t* b = bits + h * bytes;
  int c = 0;
  for (int64_t v = threadIdx.x; v < m; v += blockDim.x) {
    const int64_t idx = u * m + v;
    c += (b[idx >> 3] >> (7 - (idx & 7))) & 1;
  }
  c = __reduce_add_sync(0xffffffffu, c);
  __shared__ int part[8];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) t += part[w];
    counts[row] = t;
  }
}

__global__ void __launch_bounds__(1024) excl_scan_kernel(const int32_t* __restrict__ counts, int64_t rows,
                                                         int32_t* __restrict__ ptr, int32_t* __restrict__ empty) {
  __shared__ int buf[1024];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < rows; base += 1024) {
    const int64_t i = base + threadIdx.x;
    const int v = i < rows ? counts[i] : 0;
    if (i < rows && v == 0) atomicOr(empty, 1);
    buf[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
      const int y = threadIdx.x >= o ? buf[threadIdx.x - o] : 0;
      __syncthreads();
      buf[threadIdx.x] += y;
      __syncthreads();
    }
    if (i < rows) ptr[i] = carry + buf[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry += buf[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0) ptr[rows] = carry;
}

__global__ void bits_to_csr_fill(const uint8_t* __restrict__ bits, int64_t m, int64_t bytes,
                                 const int32_t* __restrict__ ptr, int32_t* __restrict__ idx_out) {
  const int64_t row = blockIdx.x;
  const int64_t h = row / m, u = row % m;
  if (threadIdx.x != 0) return;  // rows are short (M <= a few thousand): one ordered writer
  const uint8_t* b = bits + h * bytes;
  int32_t p = ptr[row];
  for (int64_t v = 0; v < m; ++v) {
    const int64_t idx = u * m + v;
    if ((b[idx >> 3] >> (7 - (idx & 7))) & 1) idx_out[p++] = int32_t(v);
  }
}

__global__ void lut_ptr_kernel(int64_t rows, int64_t k, int32_t* __restrict__ ptr) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i <= rows) ptr[i] = int32_t(i * k);
}

}  // namespace

int64_t topk_max_m() { return (200 * 1024) / 8; }

// rows independent rows of length n: the k best (desc value, asc index), ascending
// (mask_builder.cpp:91-102 top_indices); sel (optional) gets a 0/1 byte per element.
int top_indices_impl(const double* values, int64_t rows, int64_t n, int64_t k, int32_t* out, uint8_t* sel,
                     cudaStream_t stream) {
  if (n < 1 || k < 1 || k > n) return fail(DFS_E_INVALID, "top_indices: need 1 <= k <= n");
  if (n > topk_max_m()) return fail(DFS_E_UNSUPPORTED, "top_indices: row too long for the smem kernel");
  const int64_t m = n;
  int32_t* lut = out;
  const unsigned wgrid = unsigned(ceil_div(rows, 4));
  if (m <= 32 * 8) {
    topk_warp_kernel<8><<<wgrid, 128, 0, stream>>>(values, rows, int(m), int(k), lut, sel);
  } else if (m <= 32 * 32) {
    topk_warp_kernel<32><<<wgrid, 128, 0, stream>>>(values, rows, int(m), int(k), lut, sel);
  } else {
    const size_t smem = size_t(m) * sizeof(uint64_t);
    if (smem > 48 * 1024)
      DFS_CUDA_CHECK(cudaFuncSetAttribute(topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    topk_kernel<<<unsigned(rows), kThreads, smem, stream>>>(values, int(m), int(k), lut, sel);
  }
  DFS_LAUNCH_CHECK("topk_select");
  return DFS_OK;
}

int topk_select_impl(const double* scores, int64_t heads, int64_t m, int64_t k, int32_t* lut, uint8_t* sel,
                     uint8_t* bits, cudaStream_t stream) {
  if (m < 1 || k < 1 || k > m) return fail(DFS_E_INVALID, "topk_select: need 1 <= K <= M");
  if (int rc = top_indices_impl(scores, heads * m, m, k, lut, sel, stream)) return rc;
  if (bits) {
    const int64_t bytes = (m * m + 7) / 8;
    dim3 g(unsigned(ceil_div(bytes, 256)), unsigned(heads));
    pack_bits_kernel<<<g, 256, 0, stream>>>(sel, m, bytes, bits);
    DFS_LAUNCH_CHECK("pack_bits");
  }
  return DFS_OK;
}

int mask_bits_to_csr_impl(const uint8_t* bits, int64_t heads, int64_t m, int32_t* blk_ptr, int32_t* blk_idx,
                          int32_t* counts_ws, int32_t* flag_ws, int64_t* nnz_host, cudaStream_t stream) {
  const int64_t bytes = (m * m + 7) / 8;
  const int64_t rows = heads * m;
  bits_to_csr_count<<<unsigned(rows), 128, 0, stream>>>(bits, m, bytes, counts_ws);
  DFS_CUDA_CHECK(cudaMemsetAsync(flag_ws, 0, sizeof(int32_t), stream));
  excl_scan_kernel<<<1, 1024, 0, stream>>>(counts_ws, rows, blk_ptr, flag_ws);
  bits_to_csr_fill<<<unsigned(rows), 32, 0, stream>>>(bits, m, bytes, blk_ptr, blk_idx);
  DFS_LAUNCH_CHECK("mask_bits_to_csr");
  int32_t host[2] = {0, 0};
  DFS_CUDA_CHECK(cudaMemcpyAsync(&host[0], flag_ws, sizeof(int32_t), cudaMemcpyDeviceToHost, stream));
  DFS_CUDA_CHECK(cudaMemcpyAsync(&host[1], blk_ptr + rows, sizeof(int32_t), cudaMemcpyDeviceToHost, stream));
  DFS_CUDA_CHECK(cudaStreamSynchronize(stream));
  if (nnz_host) *nnz_host = host[1];
  if (host[0]) return fail(DFS_E_INVALID, "block_sparse_attention: empty mask row leaves softmax undefined");
  return DFS_OK;
}

int lut_row_ptr_impl(int64_t heads, int64_t m, int64_t k, int32_t* blk_ptr, cudaStream_t stream) {
  const int64_t rows = heads * m;
  lut_ptr_kernel<<<unsigned(ceil_div(rows + 1, 256)), 256, 0, stream>>>(rows, k, blk_ptr);
  DFS_LAUNCH_CHECK("lut_row_ptr");
  return DFS_OK;
}

}  // namespace dfsgpu
