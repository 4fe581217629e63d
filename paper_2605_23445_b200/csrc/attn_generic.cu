// attn_generic.cu — K5, geometry-generic SIMT path (any B, d <= 256, fp32 or bf16).
//
// block_sparse_attention (attention.cpp:125-159) and full_attention_output
// (attention.cpp:95-103) for shapes outside the tcgen05 kernel's contract —
// the drop-in dfs:: API accepts arbitrary B and d (test_attention.cpp uses
// d = 1..16, B = 1..9). One CTA per (head, query block), one thread per query
// row, keys streamed through shared memory 32 at a time, per-key online
// softmax in fp32 (the reference attends one row at a time in fp64,
// attention.cpp:32-60). Keys come from the CSR block list in ascending order
// and are clipped to nk, so padded keys never participate and padded query
// rows are never written (attention.cpp:146-152).
#include "common.cuh"

namespace dfsgpu {

namespace {

constexpr int kKT = 32;  // keys per smem tile

template <typename T, int DMAX>
__global__ void __launch_bounds__(128) attn_generic_kernel(dfs_attn_args a, int64_t mq, float scale) {
  extern __shared__ float sm[];
  const int64_t d = a.d;
  float* sk = sm;             // [kKT][d]
  float* sv = sm + kKT * d;   // [kKT][d]
  const int64_t h = blockIdx.y;
  const int64_t u = blockIdx.x;
  const int64_t B = a.block;
  const T* q = static_cast<const T*>(a.q);
  const T* k = static_cast<const T*>(a.k);
  const T* v = static_cast<const T*>(a.v);
  T* o = static_cast<T*>(a.o);
  // CSR block list, or every key block when blk_ptr is NULL (dense / cross attention)
  const int64_t mk = ceil_div(a.nk, B);
  const int32_t beg = a.blk_ptr ? a.blk_ptr[h * mq + u] : 0;
  const int32_t end = a.blk_ptr ? a.blk_ptr[h * mq + u + 1] : int32_t(mk);

  for (int64_t r0 = 0; r0 < B; r0 += blockDim.x) {
    const int64_t i = u * B + r0 + threadIdx.x;
    const bool active = (r0 + threadIdx.x) < B && i < a.nq;
    float qr[DMAX], acc[DMAX];
#pragma unroll
    for (int c = 0; c < DMAX; ++c) {
      qr[c] = (active && c < d)
                  ? to_f32<T>(q[(a.in_rows ? row_offset(DFS_NHD, a.nq, a.heads, d, h, int64_t(a.in_rows[i]))
                                            : row_offset(a.in_layout, a.nq, a.heads, d, h, i)) + c]) * scale
                  : 0.f;
      acc[c] = 0.f;
    }
    float mrun = -INFINITY, l = 0.f;
    for (int32_t e = beg; e < end; ++e) {
      const int64_t vb = a.blk_idx ? a.blk_idx[e] : e;
      const int64_t klo = vb * B, khi = min(klo + B, a.nk);
      for (int64_t k0 = klo; k0 < khi; k0 += kKT) {
        const int64_t cnt = min(int64_t(kKT), khi - k0);
        __syncthreads();
        for (int64_t t = threadIdx.x; t < cnt * d; t += blockDim.x) {
          const int64_t r = t / d, c = t % d;
          const int64_t off = row_offset(a.in_layout, a.nk, a.heads, d, h, k0 + r) + c;
          sk[r * d + c] = to_f32<T>(k[off]);
          sv[r * d + c] = to_f32<T>(v[off]);
        }
        __syncthreads();
        if (!active) continue;
        for (int64_t j = 0; j < cnt; ++j) {
          float s = 0.f;
#pragma unroll
          for (int c = 0; c < DMAX; ++c)
            if (c < d) s = fmaf(qr[c], sk[j * d + c], s);
          if (s > mrun) {
            const float corr = __expf(mrun - s);
            l *= corr;
#pragma unroll
            for (int c = 0; c < DMAX; ++c) acc[c] *= corr;
            mrun = s;
          }
          const float p = __expf(s - mrun);
          l += p;
#pragma unroll
          for (int c = 0; c < DMAX; ++c)
            if (c < d) acc[c] = fmaf(p, sv[j * d + c], acc[c]);
        }
      }
    }
    if (active) {
      const int64_t orow = a.out_rows ? int64_t(a.out_rows[i]) : i;
      T* dst = o + row_offset(a.out_layout, a.nq, a.heads, d, h, orow);
      const float inv = l > 0.f ? 1.f / l : 0.f;  // empty key list -> zero row
#pragma unroll
      for (int c = 0; c < DMAX; ++c)
        if (c < d) dst[c] = from_f32<T>(acc[c] * inv);
    }
  }
}

template <typename T, int DMAX>
int launch(const dfs_attn_args& a, int64_t mq, float scale, cudaStream_t stream) {
  const size_t smem = size_t(2 * kKT * a.d) * sizeof(float);
  if (smem > 48 * 1024)
    DFS_CUDA_CHECK(cudaFuncSetAttribute(attn_generic_kernel<T, DMAX>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  const int threads = a.block >= 128 ? 128 : int(((a.block + 31) / 32) * 32);
  dim3 grid(unsigned(mq), unsigned(a.heads));
  attn_generic_kernel<T, DMAX><<<grid, threads, smem, stream>>>(a, mq, scale);
  DFS_LAUNCH_CHECK("sparse_attn_generic");
  return DFS_OK;
}

template <typename T>
int dispatch_d(const dfs_attn_args& a, int64_t mq, float scale, cudaStream_t stream) {
  if (a.d <= 16) return launch<T, 16>(a, mq, scale, stream);
  if (a.d <= 32) return launch<T, 32>(a, mq, scale, stream);
  if (a.d <= 64) return launch<T, 64>(a, mq, scale, stream);
  if (a.d <= 128) return launch<T, 128>(a, mq, scale, stream);
  if (a.d <= 256) return launch<T, 256>(a, mq, scale, stream);
  return fail(DFS_E_UNSUPPORTED, "sparse_attn: d > 256");
}


// ---- fp32 drop-in path: the reference's fp64 arithmetic -------------------------
// For DFS_F32 inputs (the dfs::Matrix API) the softmax and the weighted sum run in
// fp64 like attend_row (attention.cpp:32-60): one warp per query row, lanes split
// the head dim (DPL = d/32 rounded up values each), every logit is a warp-reduced
// fp64 dot product. Pass 1 keeps an online (max, sum); pass 2 recomputes each
// logit, forms p = exp(l - max) / z and accumulates p * v in fp64; the result is
// rounded to fp32 once, as the reference does. Keys come from the CSR block list
// in ascending order and are clipped to nk.
template <int DPL>
__global__ void __launch_bounds__(128) attn_f64_kernel(dfs_attn_args a, int64_t mq, double scale) {
  const int lane = threadIdx.x & 31;
  const int64_t row = int64_t(blockIdx.x) * 4 + (threadIdx.x >> 5);
  const int64_t h = blockIdx.y;
  if (row >= a.nq) return;
  const int64_t d = a.d, dv = a.dv > 0 ? a.dv : a.d, B = a.block, u = row / B;
  const float* q = static_cast<const float*>(a.q);
  const float* k = static_cast<const float*>(a.k);
  const float* v = static_cast<const float*>(a.v);
  const int64_t mk = ceil_div(a.nk, B);
  const int32_t beg = a.blk_ptr ? a.blk_ptr[h * mq + u] : 0;
  const int32_t end = a.blk_ptr ? a.blk_ptr[h * mq + u + 1] : int32_t(mk);
  double qv[DPL];
  const float* qrow = q + (a.in_rows ? row_offset(DFS_NHD, a.nq, a.heads, d, h, int64_t(a.in_rows[row]))
                                     : row_offset(a.in_layout, a.nq, a.heads, d, h, row));
#pragma unroll
  for (int t = 0; t < DPL; ++t) {
    const int64_t c = lane + 32 * t;
    qv[t] = c < d ? double(qrow[c]) : 0.0;
  }
  auto logit = [&](int64_t j) {
    const float* krow = k + row_offset(a.in_layout, a.nk, a.heads, d, h, j);
    double acc = 0.0;
#pragma unroll
    for (int t = 0; t < DPL; ++t) {
      const int64_t c = lane + 32 * t;
      if (c < d) acc += qv[t] * double(krow[c]);
    }
    return warp_sum_d(acc) * scale;
  };
  double mx = -INFINITY, z = 0.0;
  for (int32_t e = beg; e < end; ++e) {
    const int64_t vb = a.blk_idx ? a.blk_idx[e] : e;
    const int64_t hi = min((vb + 1) * B, a.nk);
    for (int64_t j = vb * B; j < hi; ++j) {
      const double l = logit(j);
      if (l > mx) {
        z = z * exp(mx - l);
        mx = l;
      }
      z += exp(l - mx);
    }
  }
  double acc[DPL];
#pragma unroll
  for (int t = 0; t < DPL; ++t) acc[t] = 0.0;
  for (int32_t e = beg; e < end; ++e) {
    const int64_t vb = a.blk_idx ? a.blk_idx[e] : e;
    const int64_t hi = min((vb + 1) * B, a.nk);
    for (int64_t j = vb * B; j < hi; ++j) {
      const double p = exp(logit(j) - mx) / z;
      const float* vrow = v + row_offset(a.in_layout, a.nk, a.heads, dv, h, j);
#pragma unroll
      for (int t = 0; t < DPL; ++t) {
        const int64_t c = lane + 32 * t;
        if (c < dv) acc[t] += p * double(vrow[c]);
      }
    }
  }
  const int64_t orow = a.out_rows ? int64_t(a.out_rows[row]) : row;
  float* dst = static_cast<float*>(a.o) + row_offset(a.out_layout, a.nq, a.heads, dv, h, orow);
#pragma unroll
  for (int t = 0; t < DPL; ++t) {
    const int64_t c = lane + 32 * t;
    if (c < dv) dst[c] = z > 0.0 ? float(acc[t]) : 0.f;  // empty key list -> zero row
  }
}

template <int DPL>
int launch_f64(const dfs_attn_args& a, int64_t mq, double scale, cudaStream_t stream) {
  dim3 grid(unsigned(ceil_div(a.nq, 4)), unsigned(a.heads));
  attn_f64_kernel<DPL><<<grid, 128, 0, stream>>>(a, mq, scale);
  DFS_LAUNCH_CHECK("sparse_attn_f64");
  return DFS_OK;
}

}  // namespace

int sparse_attn_generic(const dfs_attn_args& a, float scale, cudaStream_t stream) {
  if (a.dv > 0 && a.dv != a.d && a.dtype != DFS_F32)
    return fail(DFS_E_UNSUPPORTED, "sparse_attn: dv != d only on the fp32 path");
  const int64_t mq = ceil_div(a.nq, a.block);
  if (mq > 2147483647LL || a.heads > 65535) return fail(DFS_E_UNSUPPORTED, "sparse_attn: grid too large");
  if (a.dtype == DFS_F32) {
    // fp64 softmax and accumulation (the reference's arithmetic); the scale is recomputed
    // in fp64 when the caller asked for the default 1/sqrt(d)
    const double sc = a.scale > 0.f ? double(a.scale) : 1.0 / sqrt(double(a.d));
    if (a.heads > 65535 || ceil_div(a.nq, 4) > 2147483647LL) return fail(DFS_E_UNSUPPORTED, "sparse_attn: grid too large");
    const int64_t dmax = a.dv > a.d ? a.dv : a.d;
    if (dmax <= 32) return launch_f64<1>(a, mq, sc, stream);
    if (dmax <= 64) return launch_f64<2>(a, mq, sc, stream);
    if (dmax <= 128) return launch_f64<4>(a, mq, sc, stream);
    if (dmax <= 256) return launch_f64<8>(a, mq, sc, stream);
    return fail(DFS_E_UNSUPPORTED, "sparse_attn: d > 256");
  }
  if (a.dtype == DFS_BF16) return dispatch_d<__nv_bfloat16>(a, mq, scale, stream);
  return fail(DFS_E_INVALID, "sparse_attn: unknown dtype");
}

}  // namespace dfsgpu
