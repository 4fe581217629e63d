// shim.cpp — the dfs:: drop-in C++ API (include/dfs/*.hpp) on top of the C ABI.
//
// Every operator of the reference's hot path (curve.hpp, mask_builder.hpp,
// attention.hpp, scheduler.hpp under /root/reference/proj/include/dfs) keeps its
// signature, argument meaning and exception behaviour, and computes on the GPU
// through include/dfs_gpu.h: host Matrix/BlockMask values are copied to the
// device, the sm_100a kernels run on this thread's stream, results come back.
// Nothing here computes on the CPU besides argument checks and container
// bookkeeping; a missing or unusable GPU raises std::runtime_error.
//
// Threading (scheduler.hpp:52-53, parallel.hpp:19-22): each calling thread owns
// a library handle and a non-blocking CUDA stream (thread_local), so concurrent
// run_trajectory workers overlap on the device and results do not depend on the
// worker count.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <string>
#include <utility>

#include "dfs/attention.hpp"
#include "dfs/curve.hpp"
#include "dfs/mask_builder.hpp"
#include "dfs/parallel.hpp"
#include "dfs/scheduler.hpp"
#include "dfs_gpu.h"

namespace dfs {

namespace {

// ---- errors ------------------------------------------------------------------
// DFS_E_INVALID / DFS_E_UNSUPPORTED -> std::invalid_argument (an explicit
// refusal, never a fallback), DFS_E_RANGE -> std::out_of_range.
void check(int rc) {
  if (rc == DFS_OK) return;
  const std::string msg = dfs_last_error();
  if (rc == DFS_E_INVALID || rc == DFS_E_UNSUPPORTED) throw std::invalid_argument(msg);
  if (rc == DFS_E_RANGE) throw std::out_of_range(msg);
  throw std::runtime_error("dfs_gpu: " + msg);
}

void cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("dfs_gpu: ") + what + ": " + cudaGetErrorString(e));
}

// ---- per-thread device context --------------------------------------------------
struct Context {
  dfs_handle* handle = nullptr;
  cudaStream_t stream = nullptr;
  Context() {
    int dev = 0;
    cuda(cudaGetDevice(&dev), "cudaGetDevice");
    check(dfs_handle_create(&handle, dev));
    cuda(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "cudaStreamCreate");
  }
  ~Context() {
    if (stream) cudaStreamDestroy(stream);
    if (handle) dfs_handle_destroy(handle);
  }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
};

Context& ctx() {
  thread_local Context c;
  return c;
}
dfs_stream stream() { return ctx().stream; }
void sync() { cuda(cudaStreamSynchronize(ctx().stream), "cudaStreamSynchronize"); }

// stream-ordered device buffer
class Dev {
 public:
  Dev() = default;
  explicit Dev(size_t bytes) : bytes_(bytes) {
    if (bytes) cuda(cudaMallocAsync(&p_, bytes, ctx().stream), "cudaMallocAsync");
  }
  Dev(Dev&& o) noexcept : p_(std::exchange(o.p_, nullptr)), bytes_(std::exchange(o.bytes_, 0)) {}
  Dev& operator=(Dev&& o) noexcept {
    std::swap(p_, o.p_);
    std::swap(bytes_, o.bytes_);
    return *this;
  }
  ~Dev() {
    if (p_) cudaFreeAsync(p_, ctx().stream);
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p_);
  }
  void* get() const { return p_; }

 private:
  void* p_ = nullptr;
  size_t bytes_ = 0;
};

template <typename T>
Dev upload(std::span<const T> x) {
  Dev d(x.size_bytes());
  if (!x.empty())
    cuda(cudaMemcpyAsync(d.get(), x.data(), x.size_bytes(), cudaMemcpyHostToDevice, ctx().stream), "upload");
  return d;
}
template <typename T>
void download(const Dev& d, std::span<T> x) {
  if (!x.empty())
    cuda(cudaMemcpyAsync(x.data(), d.get(), x.size_bytes(), cudaMemcpyDeviceToHost, ctx().stream), "download");
}

void require_finite(const Dev& x, int64_t count) {
  int bad = 0;
  check(dfs_check_finite(x.get(), count, DFS_F32, &bad, stream()));
  if (bad) throw std::invalid_argument("attention: non-finite input");
}

// attention.cpp:14-21 argument checks (shapes on the host, finiteness on the device)
void check_qkv_shapes(const Matrix& q, const Matrix& k, const Matrix& v) {
  if (q.cols() != k.cols()) throw std::invalid_argument("attention: q and k head dims differ");
  if (k.rows() != v.rows()) throw std::invalid_argument("attention: k and v row counts differ");
  if (q.rows() < 1 || k.rows() < 1 || q.cols() < 1) throw std::invalid_argument("attention: empty input");
}

void check_mask_geometry(int64_t rows, int64_t cols, const BlockMask& mask) {
  const int64_t b = mask.block_size();
  if (block_count_for(rows, b) != mask.block_count() || block_count_for(cols, b) != mask.block_count())
    throw std::invalid_argument("block mask geometry inconsistent with sequence length");
}

// device attention over one head: q [nq, d], k [nk, d], v [nk, dv] fp32; CSR block
// list (NULL = dense); out_rows scatters row i to row out_rows[i]
void attend(const Dev& q, const Dev& k, const Dev& v, const Dev& o, int64_t nq, int64_t nk, int64_t d, int64_t dv,
            int64_t block, const int32_t* blk_ptr, const int32_t* blk_idx, const uint32_t* out_rows) {
  dfs_attn_args a{};
  a.q = q.get();
  a.k = k.get();
  a.v = v.get();
  a.o = o.get();
  a.dtype = DFS_F32;
  a.in_layout = DFS_NHD;
  a.out_layout = DFS_NHD;
  a.heads = 1;
  a.nq = nq;
  a.nk = nk;
  a.d = d;
  a.dv = dv;
  a.block = block;
  a.blk_ptr = blk_ptr;
  a.blk_idx = blk_idx;
  a.out_rows = out_rows;
  check(dfs_sparse_attn_fwd(ctx().handle, &a, stream()));
}

// Past the reference's dense-score cap (kMaxDenseScoreRows tokens) the Matrix operators
// run the tensor-core kernels: fp32 inputs rounded to bf16 on the device, K5 (tcgen05,
// fp32 softmax / accumulation), output converted back — the bf16 I/O tolerance of
// SURVEY §8(d) (2e-2 of max|O|) instead of the compatibility kernels' fp64 arithmetic.
bool fast_attention(int64_t nq, int64_t nk, int64_t d, int64_t dv, int64_t block) {
  return std::max(nq, nk) > kMaxDenseScoreRows && (d == 64 || d == 128) && dv == d && block == 128;
}

Dev to_bf16(const Dev& x, int64_t count) {
  Dev out(sizeof(uint16_t) * size_t(count));
  check(dfs_cast(x.get(), DFS_F32, out.get(), DFS_BF16, count, nullptr, stream()));
  return out;
}

void attend_tc(const Dev& q, const Dev& k, const Dev& v, const Dev& o, int64_t nq, int64_t nk, int64_t d,
               int64_t block, const int32_t* blk_ptr, const int32_t* blk_idx) {
  const Dev q16 = to_bf16(q, nq * d), k16 = to_bf16(k, nk * d), v16 = to_bf16(v, nk * d);
  Dev o16(sizeof(uint16_t) * size_t(nq * d));
  dfs_attn_args a{};
  a.q = q16.get();
  a.k = k16.get();
  a.v = v16.get();
  a.o = o16.get();
  a.dtype = DFS_BF16;
  a.in_layout = DFS_NHD;
  a.out_layout = DFS_NHD;
  a.heads = 1;
  a.nq = nq;
  a.nk = nk;
  a.d = d;
  a.block = block;
  a.blk_ptr = blk_ptr;
  a.blk_idx = blk_idx;
  check(dfs_sparse_attn_fwd(ctx().handle, &a, stream()));
  check(dfs_cast(o16.get(), DFS_BF16, o.get(), DFS_F32, nq * d, nullptr, stream()));
}

// BlockMask payload (device) -> CSR (device); throws on an empty row
struct Csr {
  Dev ptr, idx;
};
Csr mask_csr(const Dev& bits, int64_t m) {
  Csr c{Dev(sizeof(int32_t) * size_t(m + 1)), Dev(sizeof(int32_t) * size_t(std::max<int64_t>(m * m, 1)))};
  check(dfs_mask_bits_to_csr(ctx().handle, bits.as<uint8_t>(), 1, m, c.ptr.as<int32_t>(), c.idx.as<int32_t>(), nullptr,
                             stream()));
  return c;
}

void check_rows_nonempty(const BlockMask& mask) {
  for (int64_t u = 0; u < mask.block_count(); ++u)
    if (mask.row_empty(u))
      throw std::invalid_argument("block_sparse_attention: empty mask row " + std::to_string(u) +
                                  " leaves softmax undefined");
}

// device mean_pool: x [n, d] fp32 -> [ceil(n/pool), d] (fp64 sums, divided by pool)
Dev pool_rows(const Dev& x, int64_t n, int64_t d, int64_t pool, const Dev& identity) {
  Dev scratch(sizeof(float) * size_t(n * d));
  Dev out(sizeof(float) * size_t(block_count_for(n, pool) * d));
  check(dfs_permute_rows(x.get(), DFS_NHD, scratch.get(), DFS_NHD, DFS_F32, identity.as<uint32_t>(), n, 1, d,
                         out.as<float>(), pool, nullptr, stream()));
  return out;
}

Dev identity_perm(int64_t n) {
  Dev id(sizeof(uint32_t) * size_t(n));
  check(dfs_order_tokens(DFS_RASTER, n, 1, 1, id.as<uint32_t>(), nullptr, stream()));
  return id;
}

// fp32 sub-block probabilities [mq*subs, mk*subs] from pooled rows (mask_builder.cpp:30-62);
// refuses past the dense-score cap like attention_scores does (attention.cpp:107-109)
Dev pooled_softmax(const Dev& pq, int64_t valid_q, int64_t qrows, const Dev& pk, int64_t valid_k, int64_t kcols,
                   int64_t d) {
  if (qrows > kMaxDenseScoreRows || valid_k > kMaxDenseScoreRows)
    throw std::invalid_argument("attention_scores: dense scores capped at N = " + std::to_string(kMaxDenseScoreRows));
  require_finite(pq, valid_q * d);
  require_finite(pk, valid_k * d);
  Dev P(sizeof(float) * size_t(qrows * kcols));
  check(dfs_softmax_scores(pq.as<float>(), pk.as<float>(), 1, valid_q, qrows, valid_k, kcols, d, 0.0, P.as<float>(),
                           stream()));
  return P;
}

struct ScoreShape {
  int64_t subs, mq, mk, qrows, kcols, valid_q, valid_k;
};
ScoreShape score_shape(const Matrix& q, const Matrix& k, const ScoringParams& params) {
  ScoreShape s{};
  s.subs = params.subs_per_block();
  s.mq = block_count_for(q.rows(), params.block_size);
  s.mk = block_count_for(k.rows(), params.block_size);
  s.qrows = s.mq * s.subs;
  s.kcols = s.mk * s.subs;
  s.valid_q = block_count_for(q.rows(), params.sub_block_size);
  s.valid_k = block_count_for(k.rows(), params.sub_block_size);
  return s;
}

// q, k already on the device: fp32 sub-block probabilities (device)
Dev subblock_scores_dev(const Dev& q, int64_t nq, const Dev& k, int64_t nk, int64_t d, const ScoringParams& params,
                        const ScoreShape& s) {
  if (nq < 1 || nk < 1) throw std::invalid_argument("mean_pool: empty input");
  const Dev id = identity_perm(std::max(nq, nk));
  const Dev pq = pool_rows(q, nq, d, params.sub_block_size, id);
  const Dev pk = pool_rows(k, nk, d, params.sub_block_size, id);
  return pooled_softmax(pq, s.valid_q, s.qrows, pk, s.valid_k, s.kcols, d);
}

MatrixD download_scores(const Dev& S, int64_t mq, int64_t mk) {
  MatrixD out(mq, mk);
  std::vector<double> host(size_t(mq * mk));
  download(S, std::span<double>(host));
  sync();
  for (int64_t u = 0; u < mq; ++u)
    std::memcpy(out.row(u).data(), host.data() + u * mk, sizeof(double) * size_t(mk));
  return out;
}

}  // namespace

// ================================== curve.hpp ===================================

const char* ordering_name(Ordering o) {
  switch (o) {
    case Ordering::kRaster: return "raster";
    case Ordering::kHilbert2d: return "hilbert2d";
    case Ordering::kBlock3d: return "block3d";
    case Ordering::kHilbert3d: return "hilbert3d";
  }
  throw std::invalid_argument("unknown ordering");
}

Ordering parse_ordering(const std::string& name) {
  for (Ordering o : {Ordering::kRaster, Ordering::kHilbert2d, Ordering::kBlock3d, Ordering::kHilbert3d})
    if (name == ordering_name(o)) return o;
  throw std::invalid_argument("unknown ordering: " + name);
}

void validate_permutation(const std::vector<uint32_t>& forward) {
  if (forward.empty()) throw std::invalid_argument("permutation: empty");
  const Dev f = upload(std::span<const uint32_t>(forward));
  int ok = 0;
  check(dfs_validate_permutation(ctx().handle, f.as<uint32_t>(), int64_t(forward.size()), &ok, stream()));
  if (!ok) throw std::invalid_argument("permutation: not a bijection");
}

Permutation order_tokens(Ordering ordering, const GridDims& dims) {
  dims.validate();
  const int64_t n = dims.token_count();
  Dev fwd(sizeof(uint32_t) * size_t(n));
  check(dfs_order_tokens(int(ordering), dims.frames, dims.height, dims.width, fwd.as<uint32_t>(), nullptr, stream()));
  Permutation p;
  p.label = ordering;
  p.forward.resize(size_t(n));
  download(fwd, std::span<uint32_t>(p.forward));
  sync();
  return p;
}

Permutation raster_order(const GridDims& dims) { return order_tokens(Ordering::kRaster, dims); }
Permutation hilbert3d_order(const GridDims& dims) { return order_tokens(Ordering::kHilbert3d, dims); }
Permutation hilbert2d_order(const GridDims& dims) { return order_tokens(Ordering::kHilbert2d, dims); }
Permutation block3d_order(const GridDims& dims) { return order_tokens(Ordering::kBlock3d, dims); }

Matrix apply_permutation(const Permutation& perm, const Matrix& x) {
  if (perm.size() != x.rows()) throw std::invalid_argument("apply_permutation: length mismatch");
  Matrix out(x.rows(), x.cols());
  if (x.rows() == 0 || x.cols() == 0) return out;
  const Dev src = upload(x.values());
  const Dev idx = upload(std::span<const uint32_t>(perm.forward));
  Dev dst(sizeof(float) * size_t(x.size()));
  check(dfs_permute_rows(src.get(), DFS_NHD, dst.get(), DFS_NHD, DFS_F32, idx.as<uint32_t>(), x.rows(), 1, x.cols(),
                         nullptr, 1, nullptr, stream()));
  download(dst, out.values());
  sync();
  return out;
}

Permutation invert_permutation(const Permutation& perm) {
  Permutation inv;
  inv.label = perm.label;
  inv.forward.assign(perm.forward.size(), 0u);
  if (perm.forward.empty()) return inv;
  const Dev f = upload(std::span<const uint32_t>(perm.forward));
  Dev out(sizeof(uint32_t) * perm.forward.size());
  cuda(cudaMemsetAsync(out.get(), 0, sizeof(uint32_t) * perm.forward.size(), ctx().stream), "memset");
  check(dfs_invert_permutation(f.as<uint32_t>(), perm.size(), out.as<uint32_t>(), stream()));
  download(out, std::span<uint32_t>(inv.forward));
  sync();
  return inv;
}

// =============================== mask_builder.hpp ===============================

Matrix mean_pool(const Matrix& x, int64_t pool) {
  if (pool < 1) throw std::invalid_argument("mean_pool: pool must be >= 1");
  if (x.rows() < 1) throw std::invalid_argument("mean_pool: empty input");
  const int64_t groups = block_count_for(x.rows(), pool);
  Matrix out(groups, x.cols());
  if (x.cols() == 0) return out;
  const Dev src = upload(x.values());
  const Dev pooled = pool_rows(src, x.rows(), x.cols(), pool, identity_perm(x.rows()));
  download(pooled, out.values());
  sync();
  return out;
}

Matrix subblock_scores(const Matrix& q, const Matrix& k, const ScoringParams& params) {
  params.validate();
  if (q.cols() != k.cols()) throw std::invalid_argument("subblock_scores: head dims differ");
  if (q.rows() < 1 || k.rows() < 1) throw std::invalid_argument("mean_pool: empty input");
  const ScoreShape s = score_shape(q, k, params);
  Matrix out(s.qrows, s.kcols);
  if (q.cols() == 0) return out;
  const Dev dq = upload(q.values()), dk = upload(k.values());
  const Dev P = subblock_scores_dev(dq, q.rows(), dk, k.rows(), q.cols(), params, s);
  download(P, out.values());
  sync();
  return out;
}

MatrixD aggregate_scores(const Matrix& sub, const ScoringParams& params) {
  params.validate();
  const int64_t subs = params.subs_per_block();
  if (sub.rows() % subs != 0 || sub.cols() % subs != 0)
    throw std::invalid_argument("aggregate_scores: geometry not divisible into sub-blocks");
  const int64_t mq = sub.rows() / subs, mk = sub.cols() / subs;
  if (mq == 0 || mk == 0) return MatrixD(mq, mk);
  const Dev P = upload(sub.values());
  Dev S(sizeof(double) * size_t(mq * mk));
  check(dfs_aggregate_scores(P.as<float>(), 1, mq, mk, subs, S.as<double>(), stream()));
  return download_scores(S, mq, mk);
}

int64_t topk_count(double budget, int64_t block_count) {
  int64_t k = 0;
  check(dfs_topk_count(budget, block_count, &k));
  return k;
}

std::vector<int32_t> top_indices(std::span<const double> values, int64_t k) {
  const int64_t n = int64_t(values.size());
  if (k <= 0) return {};
  const int64_t kk = std::min(k, n);
  std::vector<int32_t> out(static_cast<size_t>(kk), 0);
  if (kk > 0) {
    const Dev v = upload(values);
    Dev o(sizeof(int32_t) * size_t(kk));
    check(dfs_top_indices(v.as<double>(), 1, n, kk, o.as<int32_t>(), stream()));
    download(o, std::span<int32_t>(out));
    sync();
  }
  if (k > n) {  // the reference's resize pads with index 0 before the ascending sort
    out.resize(size_t(k), 0);
    std::sort(out.begin(), out.end());
  }
  return out;
}

BlockMask topk_select(const MatrixD& scores, double budget, int64_t block_size) {
  if (scores.rows() != scores.cols() || scores.rows() < 1)
    throw std::invalid_argument("topk_select: scores must be square and non-empty");
  const int64_t m = scores.rows();
  const int64_t k = topk_count(budget, m);
  BlockMask mask(m, block_size);
  const Dev S = upload(scores.values());
  Dev bits(size_t(BlockMask::byte_size(m)));
  check(dfs_topk_select(S.as<double>(), 1, m, k, nullptr, bits.as<uint8_t>(), stream()));
  download(bits, mask.bytes());
  sync();
  return mask;
}

MatrixD block_scores(const Matrix& q, const Matrix& k, const ScoringParams& params) {
  params.validate();
  if (q.cols() != k.cols()) throw std::invalid_argument("subblock_scores: head dims differ");
  if (q.rows() < 1 || k.rows() < 1) throw std::invalid_argument("mean_pool: empty input");
  const ScoreShape s = score_shape(q, k, params);
  if (q.cols() == 0) return aggregate_scores(Matrix(s.qrows, s.kcols), params);
  const Dev dq = upload(q.values()), dk = upload(k.values());
  if ((s.qrows > kMaxDenseScoreRows || s.valid_k > kMaxDenseScoreRows) && q.rows() == k.rows()) {
    // Past the reference's dense-score cap (attention.cpp:107-109, which throws here):
    // K2 pooling (fp64 sums) + the K3 scorer, which never materialises the sub-block
    // probabilities (fp32-accurate fp16x3 tcgen05 GEMM; fp64 for other geometries).
    require_finite(dq, q.size());
    require_finite(dk, k.size());
    const Dev id = identity_perm(q.rows());
    const Dev pq = pool_rows(dq, q.rows(), q.cols(), params.sub_block_size, id);
    const Dev pk = pool_rows(dk, k.rows(), k.cols(), params.sub_block_size, id);
    Dev S(sizeof(double) * size_t(s.mq * s.mk));
    check(dfs_score_blocks(ctx().handle, pq.as<float>(), pk.as<float>(), 1, q.rows(), q.cols(), params.block_size,
                           params.sub_block_size, S.as<double>(), stream()));
    return download_scores(S, s.mq, s.mk);
  }
  const Dev P = subblock_scores_dev(dq, q.rows(), dk, k.rows(), q.cols(), params, s);
  Dev S(sizeof(double) * size_t(s.mq * s.mk));
  check(dfs_aggregate_scores(P.as<float>(), 1, s.mq, s.mk, s.subs, S.as<double>(), stream()));
  return download_scores(S, s.mq, s.mk);
}

BlockMask build_mask(const Matrix& q, const Matrix& k, const ScoringParams& params, double budget) {
  if (q.rows() != k.rows()) throw std::invalid_argument("build_mask: q and k row counts differ");
  return topk_select(block_scores(q, k, params), budget, params.block_size);
}

// ================================= attention.hpp ================================

Matrix full_attention_output(const Matrix& q, const Matrix& k, const Matrix& v) {
  check_qkv_shapes(q, k, v);
  Matrix out(q.rows(), v.cols());
  const Dev dq = upload(q.values()), dk = upload(k.values()), dv = upload(v.values());
  require_finite(dq, q.size());
  require_finite(dk, k.size());
  require_finite(dv, v.size());
  if (v.cols() == 0) return out;
  Dev o(sizeof(float) * size_t(out.size()));
  if (fast_attention(q.rows(), k.rows(), q.cols(), v.cols(), 128))
    attend_tc(dq, dk, dv, o, q.rows(), k.rows(), q.cols(), 128, nullptr, nullptr);
  else
    attend(dq, dk, dv, o, q.rows(), k.rows(), q.cols(), v.cols(), 128, nullptr, nullptr, nullptr);
  download(o, out.values());
  sync();
  return out;
}

Matrix attention_scores(const Matrix& q, const Matrix& k) {
  if (q.cols() != k.cols()) throw std::invalid_argument("attention: q and k head dims differ");
  if (q.rows() > kMaxDenseScoreRows || k.rows() > kMaxDenseScoreRows)
    throw std::invalid_argument("attention_scores: dense scores capped at N = " + std::to_string(kMaxDenseScoreRows));
  Matrix out(q.rows(), k.rows());
  if (q.rows() == 0 || k.rows() == 0) return out;
  const Dev dq = upload(q.values()), dk = upload(k.values());
  require_finite(dq, q.size());
  require_finite(dk, k.size());
  Dev P(sizeof(float) * size_t(out.size()));
  check(dfs_softmax_scores(dq.as<float>(), dk.as<float>(), 1, q.rows(), q.rows(), k.rows(), k.rows(), q.cols(), 0.0,
                           P.as<float>(), stream()));
  download(P, out.values());
  sync();
  return out;
}

DenseAttention full_attention(const Matrix& q, const Matrix& k, const Matrix& v) {
  check_qkv_shapes(q, k, v);
  if (q.rows() > kMaxDenseScoreRows || k.rows() > kMaxDenseScoreRows)
    throw std::invalid_argument("full_attention: dense scores capped at N = " + std::to_string(kMaxDenseScoreRows));
  DenseAttention r{full_attention_output(q, k, v), attention_scores(q, k)};
  return r;
}

Matrix block_sparse_attention(const Matrix& q, const Matrix& k, const Matrix& v, const BlockMask& mask) {
  check_qkv_shapes(q, k, v);
  const Dev dq = upload(q.values()), dk = upload(k.values()), dv = upload(v.values());
  require_finite(dq, q.size());
  require_finite(dk, k.size());
  require_finite(dv, v.size());
  if (q.rows() != k.rows()) throw std::invalid_argument("block_sparse_attention: q and k row counts differ");
  check_mask_geometry(q.rows(), k.rows(), mask);
  check_rows_nonempty(mask);
  Matrix out(q.rows(), v.cols());
  if (v.cols() == 0) return out;
  const Dev bits = upload(std::span<const uint8_t>(mask.bytes()));
  const Csr csr = mask_csr(bits, mask.block_count());
  Dev o(sizeof(float) * size_t(out.size()));
  if (fast_attention(q.rows(), k.rows(), q.cols(), v.cols(), mask.block_size()))
    attend_tc(dq, dk, dv, o, q.rows(), k.rows(), q.cols(), mask.block_size(), csr.ptr.as<int32_t>(),
              csr.idx.as<int32_t>());
  else
    attend(dq, dk, dv, o, q.rows(), k.rows(), q.cols(), v.cols(), mask.block_size(), csr.ptr.as<int32_t>(),
           csr.idx.as<int32_t>(), nullptr);
  download(o, out.values());
  sync();
  return out;
}

Matrix masked_scores(const Matrix& scores, const BlockMask& mask) {
  check_mask_geometry(scores.rows(), scores.cols(), mask);
  Matrix out(scores.rows(), scores.cols());
  if (scores.size() == 0) return out;
  const Dev s = upload(scores.values()), bits = upload(std::span<const uint8_t>(mask.bytes()));
  Dev o(sizeof(float) * size_t(scores.size()));
  check(dfs_masked_scores(s.as<float>(), scores.rows(), scores.cols(), bits.as<uint8_t>(), mask.block_count(),
                          mask.block_size(), o.as<float>(), stream()));
  download(o, out.values());
  sync();
  return out;
}

double attention_recall(const Matrix& scores, const BlockMask& mask) {
  check_mask_geometry(scores.rows(), scores.cols(), mask);
  if (scores.size() == 0) return 0.0;
  const Dev s = upload(scores.values()), bits = upload(std::span<const uint8_t>(mask.bytes()));
  double r = 0.0;
  check(dfs_attention_recall(s.as<float>(), scores.rows(), scores.cols(), bits.as<uint8_t>(), mask.block_count(),
                             mask.block_size(), &r, stream()));
  return r;
}

// ================================= scheduler.hpp ================================

namespace {
dfs_schedule c_schedule(const SparsitySchedule::Config& c) {
  dfs_schedule s{};
  s.total_steps = c.total_steps;
  s.warmup_fraction = c.warmup_fraction;
  s.phase_budgets = c.phase_budgets.data();
  s.n_budgets = int(c.phase_budgets.size());
  s.phase_fraction = c.phase_fraction;
  s.update_interval = c.update_interval;
  return s;
}
}  // namespace

SparsitySchedule::SparsitySchedule(Config config) : config_(std::move(config)) {
  const dfs_schedule s = c_schedule(config_);
  check(dfs_schedule_info(&s, &warmup_steps_, &phase_length_));
}

std::optional<double> SparsitySchedule::budget_at(int step) const {
  const dfs_schedule s = c_schedule(config_);
  double b = 0.0;
  check(dfs_schedule_budget_at(&s, step, &b));
  if (b < 0.0) return std::nullopt;
  return b;
}

bool SparsitySchedule::is_update_step(int step) const {
  const dfs_schedule s = c_schedule(config_);
  int u = 0;
  check(dfs_schedule_is_update_step(&s, step, &u));
  return u != 0;
}

std::optional<MaskCache::Entry> MaskCache::find(int layer, int head) const {
  std::lock_guard<std::mutex> g(mu_);
  const auto it = entries_.find({layer, head});
  if (it == entries_.end()) return std::nullopt;
  return it->second;
}

bool MaskCache::contains(int layer, int head) const {
  std::lock_guard<std::mutex> g(mu_);
  return entries_.find({layer, head}) != entries_.end();
}

void MaskCache::store(int layer, int head, BlockMask mask, int step) {
  std::lock_guard<std::mutex> g(mu_);
  entries_[{layer, head}] = Entry{std::move(mask), step};
}

size_t MaskCache::size() const {
  std::lock_guard<std::mutex> g(mu_);
  return entries_.size();
}

void MaskCache::clear() {
  std::lock_guard<std::mutex> g(mu_);
  entries_.clear();
}

bool should_update(const MaskCache& cache, int layer, int head, int step, const SparsitySchedule& schedule) {
  return !cache.contains(layer, head) || schedule.is_update_step(step);
}

namespace {

// One device step (dfs_run_step) for `heads` heads of one layer: q/k/v fp32 [n, heads, d]
// (host, packed) -> out [n, heads, dv]. fp32 steps run the compatibility kernels up to
// kMaxDenseScoreRows tokens (bit-identical to the Matrix operators above) and the
// tcgen05 kernels past it.
struct DeviceStep {
  dfs_handle* h;
  dfs_stream st;
  const uint32_t* fwd;  // device forward permutation
};

struct StepResult {
  bool dense = true;
  double budget = 1.0;
  std::vector<int> updated;
  std::vector<double> sparsity, recall;
};

StepResult device_step(const DeviceStep& ds, const dfs_schedule& sched, const float* q, const float* k,
                       const float* v, float* out, int64_t n, int64_t heads, int64_t d, int64_t dv, int64_t block,
                       int64_t sub, int layer, int step, bool force_dense, bool record_recall) {
  Dev dq(sizeof(float) * size_t(n * heads * d)), dk(sizeof(float) * size_t(n * heads * d));
  Dev dvv(sizeof(float) * size_t(n * heads * dv)), dout(sizeof(float) * size_t(n * heads * dv));
  sync();  // allocated in this thread's stream order; used on ds.st below
  cudaStream_t cs = static_cast<cudaStream_t>(ds.st);
  cuda(cudaMemcpyAsync(dq.get(), q, sizeof(float) * size_t(n * heads * d), cudaMemcpyHostToDevice, cs), "upload");
  cuda(cudaMemcpyAsync(dk.get(), k, sizeof(float) * size_t(n * heads * d), cudaMemcpyHostToDevice, cs), "upload");
  cuda(cudaMemcpyAsync(dvv.get(), v, sizeof(float) * size_t(n * heads * dv), cudaMemcpyHostToDevice, cs), "upload");
  StepResult r;
  r.updated.assign(size_t(heads), 0);
  r.sparsity.assign(size_t(heads), 0.0);
  r.recall.assign(size_t(heads), 1.0);
  int dense = 1;
  dfs_step_args a{};
  a.q = dq.get();
  a.k = dk.get();
  a.v = dvv.get();
  a.o = dout.get();
  a.n = n;
  a.heads = heads;
  a.d = d;
  a.dv = dv;
  a.dtype = DFS_F32;
  a.perm = ds.fwd;
  a.block = block;
  a.sub_block = sub;
  a.layer = layer;
  a.step = step;
  a.force_dense = force_dense;
  a.dense_out = &dense;
  a.budget_out = &r.budget;
  a.updated_out = r.updated.data();
  a.sparsity_out = r.sparsity.data();
  a.recall_out = record_recall ? r.recall.data() : nullptr;
  check(dfs_run_step(ds.h, &sched, &a, ds.st));
  cuda(cudaMemcpyAsync(out, dout.get(), sizeof(float) * size_t(n * heads * dv), cudaMemcpyDeviceToHost, cs),
       "download");
  cuda(cudaStreamSynchronize(cs), "cudaStreamSynchronize");
  r.dense = dense != 0;
  return r;
}

BlockMask cached_mask(dfs_handle* h, dfs_stream st, int layer, int head) {
  int64_t m = 0, b = 0;
  int last = 0;
  check(dfs_mask_cache_info(h, layer, head, &m, &b, &last));
  BlockMask mask(m, b);
  Dev bits(size_t(BlockMask::byte_size(m)));
  sync();  // allocated in this thread's stream order; used on st below
  check(dfs_mask_cache_get(h, layer, head, bits.as<uint8_t>(), nullptr, nullptr, st));
  cuda(cudaMemcpyAsync(mask.bytes().data(), bits.get(), size_t(BlockMask::byte_size(m)), cudaMemcpyDeviceToHost,
                       static_cast<cudaStream_t>(st)),
       "download");
  cuda(cudaStreamSynchronize(static_cast<cudaStream_t>(st)), "cudaStreamSynchronize");
  return mask;
}

}  // namespace

// scheduler.cpp:91-135: argument checks in the reference's order on the host, then ONE
// dfs_run_step on this thread's handle (reorder + fused pooling, scoring + selection or
// the cached mask, attention with the unpermute fused in). The host MaskCache entry of
// (layer, head) is mirrored into the handle's device cache for a reuse step and read
// back after an update, so should_update / find / store keep the reference's semantics.
Matrix run_step(const Matrix& q, const Matrix& k, const Matrix& v, const Permutation& perm,
                const ScoringParams& params, const SparsitySchedule& schedule, MaskCache& cache, int layer, int head,
                int step, const StepOptions& options, StepStats* stats) {
  if (perm.size() != q.rows()) throw std::invalid_argument("run_step: permutation length does not match token count");
  const std::optional<double> budget = schedule.budget_at(step);
  if (!budget || options.force_dense) {
    if (stats) {
      *stats = StepStats{};
      stats->recall_recorded = options.record_recall;  // dense: recall 1 at any N
    }
    return full_attention_output(q, k, v);
  }
  const int64_t n = q.rows();
  if (k.rows() != n || v.rows() != n) throw std::invalid_argument("apply_permutation: length mismatch");
  const bool update = should_update(cache, layer, head, step, schedule);
  std::optional<MaskCache::Entry> entry;
  if (update) {
    params.validate();
    if (q.cols() != k.cols()) throw std::invalid_argument("subblock_scores: head dims differ");
  } else {
    entry = cache.find(layer, head);
    if (q.cols() != k.cols()) throw std::invalid_argument("attention: q and k head dims differ");
    check_mask_geometry(n, n, entry->mask);
    check_rows_nonempty(entry->mask);
  }
  if (n < 1 || q.cols() < 1) throw std::invalid_argument("attention: empty input");
  const int64_t d = q.cols(), dv = v.cols();
  Matrix out(n, dv);
  if (dv == 0) {  // nothing to attend; the reference still builds / caches the mask
    if (update) cache.store(layer, head, build_mask(apply_permutation(perm, q), apply_permutation(perm, k), params,
                                                    *budget), step);
    const BlockMask mask = cache.find(layer, head)->mask;
    if (stats) {
      stats->dense = false;
      stats->budget = *budget;
      stats->mask_updated = update;
      const double m = double(mask.block_count());
      stats->sparsity = 1.0 - double(mask.selected_count()) / (m * m);
      stats->recall_recorded = false;
    }
    return out;
  }
  Context& c = ctx();
  check(dfs_mask_cache_clear(c.handle));
  const int64_t block = update ? params.block_size : entry->mask.block_size();
  if (!update) {
    const Dev bits = upload(std::span<const uint8_t>(entry->mask.bytes()));
    check(dfs_mask_cache_store(c.handle, 0, 0, bits.as<uint8_t>(), entry->mask.block_count(), block,
                               entry->last_update_step, c.stream));
  }
  const Dev fwd = upload(std::span<const uint32_t>(perm.forward));
  const SparsitySchedule::Config& cfg = schedule.config();
  dfs_schedule sched{cfg.total_steps, cfg.warmup_fraction, cfg.phase_budgets.data(), int(cfg.phase_budgets.size()),
                     cfg.phase_fraction, cfg.update_interval};
  const StepResult r = device_step(DeviceStep{c.handle, c.stream, fwd.as<uint32_t>()}, sched, q.values().data(),
                                   k.values().data(), v.values().data(), out.values().data(), n, 1, d, dv, block,
                                   update ? params.sub_block_size : block, 0, step, false, options.record_recall);
  BlockMask mask = update ? cached_mask(c.handle, c.stream, 0, 0) : entry->mask;
  if (update) cache.store(layer, head, mask, step);
  if (stats) {
    stats->dense = false;
    stats->budget = *budget;
    stats->mask_updated = update;
    const double m = double(mask.block_count());
    stats->sparsity = 1.0 - double(mask.selected_count()) / (m * m);  // metrics.cpp:39-42
    stats->recall_recorded = options.record_recall;
    stats->recall = options.record_recall ? r.recall[0] : 1.0;
  }
  return out;
}

// scheduler.cpp:137-186. Steps run in order; within a step the (layer, head) pairs are
// fanned out as in the reference for the host work (workload.tensors, sinks), while the
// device runs ONE batched dfs_run_step per layer over all its heads. The trajectory owns
// one library handle (and stream) per layer, and the handle's device mask cache plays the
// reference's trajectory-local MaskCache. Layers run concurrently on their own streams.
std::vector<TrajectoryRow> run_trajectory(const Workload& workload, const Permutation& perm,
                                          const ScoringParams& params, const SparsitySchedule& schedule,
                                          const TrajectoryOptions& options) {
  if (workload.steps != schedule.total_steps())
    throw std::invalid_argument("run_trajectory: workload steps differ from schedule steps");
  if (workload.layers < 1 || workload.heads < 1 || !workload.tensors)
    throw std::invalid_argument("run_trajectory: invalid workload");
  const int L = workload.layers, H = workload.heads, pairs = L * H;
  const int64_t n = perm.size();
  std::vector<TrajectoryRow> rows(size_t(workload.steps) * size_t(pairs));

  struct LayerDev {
    dfs_handle* h = nullptr;
    cudaStream_t st = nullptr;
    ~LayerDev() {
      if (st) cudaStreamDestroy(st);
      if (h) dfs_handle_destroy(h);
    }
  };
  int dev = 0;
  cuda(cudaGetDevice(&dev), "cudaGetDevice");
  std::vector<LayerDev> layers(static_cast<size_t>(L));
  for (auto& ld : layers) {
    check(dfs_handle_create(&ld.h, dev));
    cuda(cudaStreamCreateWithFlags(&ld.st, cudaStreamNonBlocking), "cudaStreamCreate");
  }
  uint32_t* fwd = nullptr;
  if (n > 0) {
    cuda(cudaMalloc(&fwd, sizeof(uint32_t) * size_t(n)), "cudaMalloc");
    cuda(cudaMemcpy(fwd, perm.forward.data(), sizeof(uint32_t) * size_t(n), cudaMemcpyHostToDevice), "upload");
  }
  struct FreeOnExit {
    uint32_t* p;
    ~FreeOnExit() {
      if (p) cudaFree(p);
    }
  } free_fwd{fwd};
  const SparsitySchedule::Config& cfg = schedule.config();
  const dfs_schedule sched{cfg.total_steps, cfg.warmup_fraction, cfg.phase_budgets.data(),
                           int(cfg.phase_budgets.size()), cfg.phase_fraction, cfg.update_interval};

  std::vector<StepTensors> tensors(static_cast<size_t>(pairs));
  std::vector<Matrix> outs(static_cast<size_t>(pairs));
  std::vector<std::optional<BlockMask>> updated(static_cast<size_t>(pairs));
  for (int step = 0; step < workload.steps; ++step) {
    // host: every pair's tensors, in parallel like the reference's fan-out
    parallel_for(pairs, options.threads, [&](int64_t pair) {
      const int layer = int(pair) / H, head = int(pair) % H;
      tensors[size_t(pair)] = workload.tensors(step, layer, head);
      if (tensors[size_t(pair)].q.rows() != n)
        throw std::invalid_argument("run_trajectory: token count drifted between steps");
    });
    // device: one batched step per layer (all heads), layers concurrently
    parallel_for(L, options.threads, [&](int64_t layer) {
      const int l = int(layer);
      const StepTensors& t0 = tensors[size_t(l * H)];
      const int64_t d = t0.q.cols(), dv = t0.v.cols();
      bool uniform = d > 0 && dv > 0;
      for (int hh = 0; hh < H && uniform; ++hh) {
        const StepTensors& t = tensors[size_t(l * H + hh)];
        uniform = t.q.cols() == d && t.k.cols() == d && t.k.rows() == n && t.v.rows() == n && t.v.cols() == dv;
      }
      const bool force_dense = options.dense_layers.count(l) > 0;
      const std::optional<double> budget = schedule.budget_at(step);
      if (!uniform) {
        // ragged shapes: the per-head operator, which raises the reference's errors
        throw std::invalid_argument("run_trajectory: heads of a layer must share q/k/v shapes (" +
                                    std::to_string(n) + " tokens)");
      }
      std::vector<float> q(size_t(n * H * d)), k(size_t(n * H * d)), v(size_t(n * H * dv)), o(size_t(n * H * dv));
      for (int hh = 0; hh < H; ++hh) {
        const StepTensors& t = tensors[size_t(l * H + hh)];
        for (int64_t i = 0; i < n; ++i) {
          std::memcpy(&q[size_t((i * H + hh) * d)], t.q.row(i).data(), sizeof(float) * size_t(d));
          std::memcpy(&k[size_t((i * H + hh) * d)], t.k.row(i).data(), sizeof(float) * size_t(d));
          std::memcpy(&v[size_t((i * H + hh) * dv)], t.v.row(i).data(), sizeof(float) * size_t(dv));
        }
      }
      const StepResult r = device_step(DeviceStep{layers[size_t(l)].h, layers[size_t(l)].st, fwd}, sched, q.data(),
                                       k.data(), v.data(), o.data(), n, H, d, dv, params.block_size,
                                       params.sub_block_size, l, step, force_dense, options.record_recall);
      for (int hh = 0; hh < H; ++hh) {
        const int64_t pair = int64_t(l) * H + hh;
        Matrix& out = outs[size_t(pair)];
        out = Matrix(n, dv);
        for (int64_t i = 0; i < n; ++i)
          std::memcpy(out.row(i).data(), &o[size_t((i * H + hh) * dv)], sizeof(float) * size_t(dv));
        updated[size_t(pair)].reset();
        if (r.updated[size_t(hh)] && options.mask_sink)
          updated[size_t(pair)] = cached_mask(layers[size_t(l)].h, layers[size_t(l)].st, l, hh);
        TrajectoryRow& row = rows[size_t(step) * size_t(pairs) + size_t(pair)];
        row.step = step;
        row.layer = l;
        row.head = hh;
        row.dense = r.dense;
        row.budget = r.dense ? 1.0 : r.budget;
        row.sparsity = r.dense ? 0.0 : r.sparsity[size_t(hh)];
        row.mask_updated = r.updated[size_t(hh)] != 0;
        row.recall_recorded = options.record_recall;
        row.recall = options.record_recall ? r.recall[size_t(hh)] : 1.0;
        (void)budget;
      }
    });
    // host: sinks, fanned out like the reference (they may be called from worker threads)
    parallel_for(pairs, options.threads, [&](int64_t pair) {
      const int layer = int(pair) / H, head = int(pair) % H;
      if (options.mask_sink && updated[size_t(pair)]) options.mask_sink(step, layer, head, *updated[size_t(pair)]);
      if (options.output_sink) options.output_sink(step, layer, head, outs[size_t(pair)]);
    });
  }
  return rows;
}

}  // namespace dfs
