// dropin.cu — the Matrix-level C ABI behind the dfs:: drop-in shim: dense
// softmax scores, tile aggregation, row top-k, mask expansion and recall.
//
// These are the reference's small-shape / analysis companions of the hot path
// (attention.cpp:105-123 attention_scores, :161-190 masked_scores /
// attention_recall; mask_builder.cpp:64-102 aggregate_scores / top_indices)
// that the shim needs so reference callers relink unchanged. All of them run
// on the device; the arithmetic is the reference's (fp64 sums, fp32 storage).
#include "common.cuh"

namespace dfsgpu {

int softmax_scores_impl(const float* q, const float* k, int64_t heads, int64_t qvalid, int64_t qrows,
                        int64_t kvalid, int64_t kcols, int64_t d, double scale, float* P, cudaStream_t stream);
int aggregate_scores_impl(const float* P, int64_t heads, int64_t mq, int64_t mk, int64_t subs, double* S,
                          cudaStream_t stream);
int top_indices_impl(const double* values, int64_t rows, int64_t n, int64_t k, int32_t* out, uint8_t* sel,
                     cudaStream_t stream);
int finite_check_impl(const void* x, int64_t count, int dtype, int32_t* flag, cudaStream_t stream);

namespace {

__device__ __forceinline__ bool mask_get(const uint8_t* bits, int64_t m, int64_t u, int64_t v) {
  const int64_t idx = u * m + v;
  return (bits[idx >> 3] >> (7 - (idx & 7))) & 1;
}

// out[i][j] = scores[i][j] if mask(i / b, j / b) else 0 (attention.cpp:161-173)
__global__ void masked_scores_kernel(const float* __restrict__ scores, int64_t rows, int64_t cols,
                                     const uint8_t* __restrict__ bits, int64_t m, int64_t b,
                                     float* __restrict__ out) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= rows * cols) return;
  const int64_t i = t / cols, j = t % cols;
  out[t] = mask_get(bits, m, i / b, j / b) ? scores[t] : 0.0f;
}

// one CTA per score row: fp64 sums of |A| kept and total (attention.cpp:175-190)
__global__ void recall_rows_kernel(const float* __restrict__ scores, int64_t cols, const uint8_t* __restrict__ bits,
                                   int64_t m, int64_t b, double* __restrict__ kept, double* __restrict__ total) {
  const int64_t i = blockIdx.x;
  double k = 0.0, t = 0.0;
  for (int64_t j = threadIdx.x; j < cols; j += blockDim.x) {
    const double a = fabs(double(scores[i * cols + j]));
    t += a;
    if (mask_get(bits, m, i / b, j / b)) k += a;
  }
  k = warp_sum_d(k);
  t = warp_sum_d(t);
  __shared__ double sk[8], st[8];
  if ((threadIdx.x & 31) == 0) {
    sk[threadIdx.x >> 5] = k;
    st[threadIdx.x >> 5] = t;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, c = 0.0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) {
      a += sk[w];
      c += st[w];
    }
    kept[i] = a;
    total[i] = c;
  }
}

// ordered final reduction over rows (one thread: deterministic, rows <= 4096)
__global__ void recall_final_kernel(const double* __restrict__ kept, const double* __restrict__ total, int64_t rows,
                                    double* __restrict__ out) {
  double a = 0.0, c = 0.0;
  for (int64_t i = 0; i < rows; ++i) {
    a += kept[i];
    c += total[i];
  }
  *out = c == 0.0 ? 0.0 : a / c;
}

}  // namespace
}  // namespace dfsgpu

using namespace dfsgpu;

extern "C" {

int dfs_softmax_scores(const float* q, const float* k, int64_t heads, int64_t q_valid, int64_t q_rows,
                       int64_t k_valid, int64_t k_cols, int64_t d, double scale, float* probs, dfs_stream stream) {
  if (!q || !k || !probs) return fail(DFS_E_INVALID, "softmax_scores: null pointer");
  if (heads < 1 || q_valid < 0 || k_valid < 1 || d < 1 || q_rows < q_valid || k_cols < k_valid)
    return fail(DFS_E_INVALID, "attention: empty input");
  if (scale <= 0.0) scale = 1.0 / sqrt(double(d));
  return softmax_scores_impl(q, k, heads, q_valid, q_rows, k_valid, k_cols, d, scale, probs, as_stream(stream));
}

int dfs_aggregate_scores(const float* probs, int64_t heads, int64_t mq, int64_t mk, int64_t subs, double* scores,
                         dfs_stream stream) {
  if (!probs || !scores || heads < 1 || mq < 1 || mk < 1 || subs < 1)
    return fail(DFS_E_INVALID, "aggregate_scores: bad arguments");
  return aggregate_scores_impl(probs, heads, mq, mk, subs, scores, as_stream(stream));
}

int dfs_top_indices(const double* values, int64_t rows, int64_t n, int64_t k, int32_t* out, dfs_stream stream) {
  if (!values || !out || rows < 1) return fail(DFS_E_INVALID, "top_indices: bad arguments");
  return top_indices_impl(values, rows, n, k, out, nullptr, as_stream(stream));
}

int dfs_masked_scores(const float* scores, int64_t rows, int64_t cols, const uint8_t* bits, int64_t m, int64_t block,
                      float* out, dfs_stream stream) {
  if (!scores || !bits || !out || block < 1) return fail(DFS_E_INVALID, "masked_scores: bad arguments");
  if (ceil_div(rows, block) != m || ceil_div(cols, block) != m)
    return fail(DFS_E_INVALID, "block mask geometry inconsistent with sequence length");
  if (rows * cols == 0) return DFS_OK;
  masked_scores_kernel<<<unsigned(ceil_div(rows * cols, 256)), 256, 0, as_stream(stream)>>>(scores, rows, cols, bits,
                                                                                           m, block, out);
  DFS_LAUNCH_CHECK("masked_scores");
  return DFS_OK;
}

int dfs_check_finite(const void* x, int64_t count, int dtype, int* nonfinite_host, dfs_stream stream) {
  if (!nonfinite_host || (count > 0 && !x)) return fail(DFS_E_INVALID, "check_finite: bad arguments");
  *nonfinite_host = 0;
  if (count < 1) return DFS_OK;
  cudaStream_t s = as_stream(stream);
  int32_t* flag = nullptr;
  DFS_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&flag), sizeof(int32_t), s));
  int rc = DFS_OK;
  cudaError_t e = cudaMemsetAsync(flag, 0, sizeof(int32_t), s);
  if (e == cudaSuccess) rc = finite_check_impl(x, count, dtype, flag, s);
  int32_t host = 0;
  if (e == cudaSuccess && rc == DFS_OK) e = cudaMemcpyAsync(&host, flag, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && rc == DFS_OK) e = cudaStreamSynchronize(s);
  cudaFreeAsync(flag, s);
  if (rc) return rc;
  if (e != cudaSuccess) return cuda_fail(e, "check_finite");
  *nonfinite_host = host != 0;
  return DFS_OK;
}

int dfs_attention_recall(const float* scores, int64_t rows, int64_t cols, const uint8_t* bits, int64_t m,
                         int64_t block, double* recall_host, dfs_stream stream) {
  if (!scores || !bits || !recall_host || block < 1) return fail(DFS_E_INVALID, "attention_recall: bad arguments");
  if (ceil_div(rows, block) != m || ceil_div(cols, block) != m)
    return fail(DFS_E_INVALID, "block mask geometry inconsistent with sequence length");
  cudaStream_t s = as_stream(stream);
  if (rows < 1) {
    *recall_host = 0.0;
    return DFS_OK;
  }
  double* ws = nullptr;
  DFS_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&ws), sizeof(double) * size_t(2 * rows + 1), s));
  recall_rows_kernel<<<unsigned(rows), 256, 0, s>>>(scores, cols, bits, m, block, ws, ws + rows);
  recall_final_kernel<<<1, 1, 0, s>>>(ws, ws + rows, rows, ws + 2 * rows);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(recall_host, ws + 2 * rows, sizeof(double), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFreeAsync(ws, s);
  if (e != cudaSuccess) return cuda_fail(e, "attention_recall");
  return DFS_OK;
}

}  // extern "C"
