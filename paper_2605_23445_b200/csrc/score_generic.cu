// score_generic.cu — K3, geometry-generic path (any d <= 256, any B_s | B).
//
// mask_builder.cpp:30-80 subblock_scores + aggregate_scores for the drop-in
// dfs:: API's arbitrary shapes. fp64 logits / exp / normalisation (the
// reference's own precision, attention.cpp:64-68,83-86), each probability
// rounded to fp32 (attention.cpp:120), then fp64 tile sums in the reference's
// (i, j) order. Two launches per batch of heads:
//   1. softmax_rows: one CTA per 32 pooled query rows; pass 1 streams the key
//      tiles for the row max and partition sum, pass 2 recomputes and writes
//      the fp32 probabilities P [qrows, kcols] (padded key columns = 0, padded
//      query rows = zero vectors -> uniform over the valid keys).
//   2. aggregate: one thread per (u, v) sums its subs x subs tile of P.
// The tensor-core path for B=128/d in {64,128} is score_sm100.cu.
#include "common.cuh"

namespace dfsgpu {

namespace {

constexpr int kRows = 32;   // pooled query rows per CTA
constexpr int kKeys = 32;   // pooled keys per tile

__global__ void __launch_bounds__(256) softmax_rows_kernel(const float* __restrict__ pq,
                                                           const float* __restrict__ pk, int64_t qvalid,
                                                           int64_t qrows, int64_t kvalid, int64_t kcols,
                                                           int64_t d, double scale,
                                                           float* __restrict__ P) {
  extern __shared__ float smem[];
  const int64_t ld = d + 1;  // pad: lanes read different keys at the same column
  float* sq = smem;
  float* sk = smem + kRows * ld;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t h = blockIdx.y;
  const int64_t row0 = int64_t(blockIdx.x) * kRows;
  const float* q = pq + h * qvalid * d;
  const float* k = pk + h * kvalid * d;
  float* out = P + h * qrows * kcols;

  for (int64_t t = threadIdx.x; t < kRows * d; t += blockDim.x) {
    const int64_t r = t / d, c = t % d;
    const int64_t gr = row0 + r;
    sq[r * ld + c] = gr < qvalid ? q[gr * d + c] : 0.0f;  // padded rows pool to zero
  }
  double m[4], z[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    m[j] = -INFINITY;
    z[j] = 0.0;
  }
  for (int pass = 0; pass < 2; ++pass) {
    for (int64_t k0 = 0; k0 < kvalid; k0 += kKeys) {
      __syncthreads();
      for (int64_t t = threadIdx.x; t < kKeys * d; t += blockDim.x) {
        const int64_t r = t / d, c = t % d;
        sk[r * ld + c] = k0 + r < kvalid ? k[(k0 + r) * d + c] : 0.0f;
      }
      __syncthreads();
      const int64_t key = k0 + lane;
      double l[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float* qr = sq + (warp * 4 + j) * ld;
        const float* kr = sk + lane * ld;
        double acc = 0.0;
        for (int64_t c = 0; c < d; ++c) acc += double(qr[c]) * double(kr[c]);
        l[j] = acc * scale;
      }
      if (pass == 0) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          double tile_max = key < kvalid ? l[j] : -INFINITY;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) tile_max = fmax(tile_max, __shfl_xor_sync(0xffffffffu, tile_max, o));
          const double nm = fmax(m[j], tile_max);
          double e = key < kvalid ? exp(l[j] - nm) : 0.0;
          e = warp_sum_d(e);
          z[j] = z[j] * exp(m[j] - nm) + e;
          m[j] = nm;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int64_t gr = row0 + warp * 4 + j;
          if (gr < qrows && key < kvalid) out[gr * kcols + key] = float(exp(l[j] - m[j]) / z[j]);
        }
      }
    }
  }
  // padded key columns stay zero (mask_builder.cpp:50-60)
  for (int j = 0; j < 4; ++j) {
    const int64_t gr = row0 + warp * 4 + j;
    if (gr >= qrows) continue;
    for (int64_t c = kvalid + lane; c < kcols; c += 32) out[gr * kcols + c] = 0.0f;
  }
}

// S[u][v] = sum of the subs x subs tile (u, v) of P, fp64 in the reference's (i, j)
// order (mask_builder.cpp:64-80); mq x mk blocks, P is [mq*subs, mk*subs] per head.
__global__ void aggregate_kernel(const float* __restrict__ P, int64_t mq, int64_t mk, int64_t subs,
                                 double* __restrict__ S) {
  const int64_t h = blockIdx.y;
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= mq * mk) return;
  const int64_t u = t / mk, v = t % mk;
  const int64_t kcols = mk * subs;
  const float* p = P + h * mq * subs * kcols;
  double acc = 0.0;
  for (int64_t i = u * subs; i < (u + 1) * subs; ++i)
    for (int64_t j = v * subs; j < (v + 1) * subs; ++j) acc += double(p[i * kcols + j]);
  S[h * mq * mk + t] = acc;
}

}  // namespace

// pq [H, qvalid, d], pk [H, kvalid, d] (qvalid == kvalid == ceil(n/Bs)); S [H, M, M].
// P_ws must hold heads_per_batch * qrows * kcols floats.
int score_blocks_generic(const float* pq, const float* pk, int64_t heads, int64_t n, int64_t d, int64_t block,
                         int64_t sub_block, double* S, float* P_ws, int64_t P_ws_floats,
                         cudaStream_t stream) {
  if (d > 256) return fail(DFS_E_UNSUPPORTED, "score_blocks: generic path needs d <= 256");
  const int64_t subs = block / sub_block;
  const int64_t m = ceil_div(n, block);
  const int64_t qrows = m * subs, kcols = qrows;
  const int64_t valid = ceil_div(n, sub_block);
  const int64_t per_head = qrows * kcols;
  const int64_t batch = P_ws_floats / per_head;
  if (batch < 1) return fail(DFS_E_INTERNAL, "score_blocks: workspace too small");
  const size_t smem = size_t(2 * kRows * (d + 1)) * sizeof(float);
  if (smem > 48 * 1024) {
    DFS_CUDA_CHECK(cudaFuncSetAttribute(softmax_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        int(smem)));
  }
  const double scale = 1.0 / sqrt(double(d));
  for (int64_t h0 = 0; h0 < heads; h0 += batch) {
    const int64_t hb = heads - h0 < batch ? heads - h0 : batch;
    dim3 g1(unsigned(ceil_div(qrows, kRows)), unsigned(hb));
    softmax_rows_kernel<<<g1, 256, smem, stream>>>(pq + h0 * valid * d, pk + h0 * valid * d, valid, qrows, valid,
                                                   kcols, d, scale, P_ws);
    dim3 g2(unsigned(ceil_div(m * m, 256)), unsigned(hb));
    aggregate_kernel<<<g2, 256, 0, stream>>>(P_ws, m, m, subs, S + h0 * m * m);
    DFS_LAUNCH_CHECK("score_blocks_generic");
  }
  return DFS_OK;
}

// Row softmax of q k^T * scale (attention.cpp:105-123 attention_scores, and the
// pooled form inside subblock_scores, mask_builder.cpp:30-62): q [H, qvalid, d],
// k [H, kvalid, d] fp32 -> P [H, qrows, kcols] fp32 with fp64 logits/exp/sum.
// Rows >= qvalid are zero vectors (uniform over the valid keys), columns >= kvalid
// stay 0.
int softmax_scores_impl(const float* q, const float* k, int64_t heads, int64_t qvalid, int64_t qrows,
                        int64_t kvalid, int64_t kcols, int64_t d, double scale, float* P, cudaStream_t stream) {
  if (d > 256) return fail(DFS_E_UNSUPPORTED, "attention_scores: d > 256");
  if (heads > 65535) return fail(DFS_E_UNSUPPORTED, "attention_scores: too many heads");
  const size_t smem = size_t(2 * kRows * (d + 1)) * sizeof(float);
  if (smem > 48 * 1024)
    DFS_CUDA_CHECK(cudaFuncSetAttribute(softmax_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        int(smem)));
  dim3 g1(unsigned(ceil_div(qrows, kRows)), unsigned(heads));
  softmax_rows_kernel<<<g1, 256, smem, stream>>>(q, k, qvalid, qrows, kvalid, kcols, d, scale, P);
  DFS_LAUNCH_CHECK("softmax_scores");
  return DFS_OK;
}

int aggregate_scores_impl(const float* P, int64_t heads, int64_t mq, int64_t mk, int64_t subs, double* S,
                          cudaStream_t stream) {
  dim3 g2(unsigned(ceil_div(mq * mk, 256)), unsigned(heads));
  aggregate_kernel<<<g2, 256, 0, stream>>>(P, mq, mk, subs, S);
  DFS_LAUNCH_CHECK("aggregate_scores");
  return DFS_OK;
}

}  // namespace dfsgpu
