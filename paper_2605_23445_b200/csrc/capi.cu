// capi.cu — the extern "C" boundary (include/dfs_gpu.h): handle, workspaces,
// permutation cache, device mask cache and the Alg. 1 step driver.
//
// Host logic restated from the reference:
//   SparsitySchedule  scheduler.cpp:18-56 (floor warmup, ceil phase length,
//                     last phase absorbs, update every Delta sparse steps)
//   MaskCache         scheduler.cpp:58-83 (per (layer, head), keeps the K of
//                     its update step across phase changes — test_cli.cpp:279-283)
//   should_update     scheduler.cpp:85-89
//   run_step          scheduler.cpp:91-135 (dense steps skip the reorder)
// The per-head loop of the reference becomes one batched launch per kernel over
// all H heads of the layer; the unpermute is fused into the attention epilogue.
#include <cuda.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "common.cuh"

namespace dfsgpu {

// ---- kernels implemented in the other translation units -------------------
int order_tokens_impl(int ordering, int64_t f, int64_t h, int64_t w, uint32_t* fwd, uint32_t* inv,
                      int* scratch, int64_t scratch_ints, cudaStream_t stream);
int64_t order_tokens_scratch_ints(int ordering, int64_t f, int64_t h, int64_t w);
int invert_permutation_impl(const uint32_t* fwd, int64_t n, uint32_t* inv, cudaStream_t stream);
int validate_permutation_impl(const uint32_t* fwd, int64_t n, int* seen, int* bad, int* ok_host,
                              cudaStream_t stream);
int permute_rows_impl(const void* src, int src_layout, void* dst, int dst_layout, int dtype,
                      const uint32_t* idx, int64_t n, int64_t heads, int64_t d, float* pooled,
                      int64_t pool, int32_t* nonfinite, bool scatter, cudaStream_t stream);
int finite_check_impl(const void* x, int64_t count, int dtype, int32_t* flag, cudaStream_t stream);
int cast_impl(const void* src, int src_dtype, void* dst, int dst_dtype, int64_t count, int32_t* nonfinite,
              cudaStream_t stream);
int permute_rows_peer_impl(const dfs_peer_table* peers_dev, int64_t heads_total, void* dst, const uint32_t* idx,
                           int64_t n, int64_t heads, int64_t d, float* pooled, int64_t pool, int32_t* nonfinite,
                           cudaStream_t stream);
int prologue_permute_impl(const void* src, void* dst, int dst_layout, const uint32_t* idx, int64_t n, int64_t heads,
                          int64_t d, float* pooled, int64_t pool, int32_t* nonfinite, const float* norm_weight,
                          float eps, int rope_layout, const float* cos_t, const float* sin_t, cudaStream_t stream);
int score_blocks_generic(const float* pq, const float* pk, int64_t heads, int64_t n, int64_t d, int64_t block,
                         int64_t sub_block, double* S, float* P_ws, int64_t P_ws_floats, cudaStream_t stream);
int score_blocks_sm100(const float* pq, const float* pk, int64_t heads, int64_t n, int64_t d, int64_t block,
                       int64_t sub_block, double* S, void* ws, int64_t ws_bytes, cudaStream_t stream);
bool score_sm100_supports(int64_t d, int64_t block, int64_t sub_block);
int64_t score_sm100_ws_bytes(int64_t heads, int64_t n, int64_t d, int64_t block, int64_t sub_block);
int topk_select_impl(const double* scores, int64_t heads, int64_t m, int64_t k, int32_t* lut, uint8_t* sel,
                     uint8_t* bits, cudaStream_t stream);
int64_t topk_max_m();
int mask_bits_to_csr_impl(const uint8_t* bits, int64_t heads, int64_t m, int32_t* blk_ptr, int32_t* blk_idx,
                          int32_t* counts_ws, int32_t* flag_ws, int64_t* nnz_host, cudaStream_t stream);
int lut_row_ptr_impl(int64_t heads, int64_t m, int64_t k, int32_t* blk_ptr, cudaStream_t stream);
int sparse_attn_generic(const dfs_attn_args& a, float scale, cudaStream_t stream);
int sparse_attn_sm100(const dfs_attn_args& a, float scale, cudaStream_t stream);
bool attn_sm100_supports(const dfs_attn_args& a);
bool recall_sm100_supports(int64_t d);
int block_recall_sm100(const void* q, const void* k, int layout, const uint32_t* q_rows, int64_t heads, int64_t n,
                       int64_t d, const int32_t* blk_ptr, const int32_t* blk_idx, float* mass, double* recall,
                       cudaStream_t stream);

// ---- errors ----------------------------------------------------------------
namespace {
thread_local std::string g_error;
}
void set_error(const std::string& msg) { g_error = msg; }
int fail(int code, const std::string& msg) {
  g_error = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* where) {
  g_error = std::string(where) + ": " + cudaGetErrorString(e);
  return DFS_E_CUDA;
}

// ---- device buffers ---------------------------------------------------------
struct Buf {
  void* p = nullptr;
  size_t bytes = 0;
  Buf() = default;
  Buf(const Buf&) = delete;
  Buf& operator=(const Buf&) = delete;
  Buf(Buf&& o) noexcept : p(o.p), bytes(o.bytes) {
    o.p = nullptr;
    o.bytes = 0;
  }
  Buf& operator=(Buf&& o) noexcept {
    if (this != &o) {
      if (p) cudaFree(p);
      p = o.p;
      bytes = o.bytes;
      o.p = nullptr;
      o.bytes = 0;
    }
    return *this;
  }
  ~Buf() {
    if (p) cudaFree(p);
  }
  int ensure(size_t need) {
    if (need <= bytes) return DFS_OK;
    if (p) {
      cudaFree(p);
      p = nullptr;
      bytes = 0;
    }
    if (need == 0) return DFS_OK;
    DFS_CUDA_CHECK(cudaMalloc(&p, need));
    bytes = need;
    return DFS_OK;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

}  // namespace dfsgpu

using namespace dfsgpu;

struct PermEntry {
  Buf fwd, inv;
  int64_t n = 0;
};

struct HeadMask {
  bool valid = false;
  int last_update_step = 0;
  int64_t nnz = 0;
};

// One layer's device-resident masks: a CSR over (head, query block).
struct LayerMasks {
  int64_t heads = 0, m = 0, block = 0;
  Buf ptr, idx;  // ptr [heads*m+1], idx [cap]
  std::vector<HeadMask> head;
  std::vector<int64_t> head_off;  // start of each head's rows in idx
};

struct dfs_handle {
  int device = 0;
  int opt_generic_score = 0;  // DFS_OPT_GENERIC_SCORE
  int opt_generic_attn = 0;   // DFS_OPT_GENERIC_ATTN
  std::map<std::tuple<int, int64_t, int64_t, int64_t>, PermEntry> perms;
  std::map<int, LayerMasks> masks;  // keyed by layer
  // workspaces
  Buf scratch_i32, flag;
  Buf k_hnd, v_hnd, pooled_q, pooled_k, scores, score_ws, lut, sel, counts;
  Buf tmp_ptr, tmp_idx, recall_ws;
  Buf step_flag;                         // the step's non-finite flag (dfs_step_args.nonfinite == NULL)
  Buf q16, k16, v16, o16;                // DFS_F32 steps past the compatibility cap: bf16 copies
  Buf f32_q, f32_k, f32_v, probs, bits;  // DFS_F32 compatibility steps: reordered fp32 [H, N, d]
  Buf peer_tabs;                         // Ulysses: q/k/v/o dfs_peer_table on the device
  // side stream for the V reorder (only K5 needs it: it runs under K3/K4) + its events
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_v = nullptr;
  ~dfs_handle() {
    if (host_flag) cudaFreeHost(host_flag);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_v) cudaEventDestroy(ev_v);
    if (aux) cudaStreamDestroy(aux);
  }
  int32_t* host_flag = nullptr;  // pinned read-back slot of the step's non-finite flag
  int ensure_aux() {
    if (aux) return DFS_OK;
    DFS_CUDA_CHECK(cudaStreamCreateWithFlags(&aux, cudaStreamNonBlocking));
    DFS_CUDA_CHECK(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    DFS_CUDA_CHECK(cudaEventCreateWithFlags(&ev_v, cudaEventDisableTiming));
    return DFS_OK;
  }
  int64_t total_bytes() const {
    int64_t t = 0;
    for (const Buf* b : {&scratch_i32, &flag, &k_hnd, &v_hnd, &pooled_q, &pooled_k, &scores, &score_ws,
                         &lut, &sel, &counts, &tmp_ptr, &tmp_idx, &recall_ws, &step_flag, &q16, &k16, &v16,
                         &o16, &f32_q, &f32_k, &f32_v, &probs, &bits, &peer_tabs})
      t += int64_t(b->bytes);
    return t;
  }
};

namespace capi_detail {

int check_handle(dfs_handle* h) {
  if (!h) return fail(DFS_E_INVALID, "null dfs_handle");
  DFS_CUDA_CHECK(cudaSetDevice(h->device));
  return DFS_OK;
}

int schedule_validate(const dfs_schedule* s, int* warmup, int* phase_len) {
  constexpr double kEps = 1e-9;  // scheduler.cpp:10-13
  if (!s) return fail(DFS_E_INVALID, "null schedule");
  if (s->total_steps < 1) return fail(DFS_E_INVALID, "SparsitySchedule: total_steps must be >= 1");
  if (s->warmup_fraction < 0.0 || s->warmup_fraction > 1.0)
    return fail(DFS_E_INVALID, "SparsitySchedule: warmup_fraction must lie in [0, 1]");
  if (s->phase_fraction < 0.0 || s->phase_fraction > 1.0)
    return fail(DFS_E_INVALID, "SparsitySchedule: phase_fraction must lie in [0, 1]");
  if (s->update_interval < 1) return fail(DFS_E_INVALID, "SparsitySchedule: update_interval must be >= 1");
  for (int i = 0; i < s->n_budgets; ++i)
    if (!(s->phase_budgets[i] > 0.0) || s->phase_budgets[i] > 1.0)
      return fail(DFS_E_INVALID, "SparsitySchedule: budgets must lie in (0, 1]");
  if (s->warmup_fraction + double(s->n_budgets) * s->phase_fraction > 1.0 + kEps)
    return fail(DFS_E_INVALID, "SparsitySchedule: warmup + phases exceed the step range");
  const double t = double(s->total_steps);
  int w = int(std::floor(s->warmup_fraction * t + kEps));
  if (w > s->total_steps) w = s->total_steps;
  if (w < s->total_steps && s->n_budgets == 0)
    return fail(DFS_E_INVALID, "SparsitySchedule: sparse steps exist but no phase budgets given");
  int pl = int(std::ceil(s->phase_fraction * t - kEps));
  if (pl < 1) pl = 1;
  if (warmup) *warmup = w;
  if (phase_len) *phase_len = pl;
  return DFS_OK;
}

int get_perm(dfs_handle* h, int ordering, int64_t f, int64_t hh, int64_t w, cudaStream_t stream,
             const PermEntry** out) {
  auto key = std::make_tuple(ordering, f, hh, w);
  auto it = h->perms.find(key);
  if (it == h->perms.end()) {
    if (f < 1 || hh < 1 || w < 1) return fail(DFS_E_INVALID, "GridDims: extents must be >= 1");
    PermEntry e;
    e.n = f * hh * w;
    int rc;
    if ((rc = e.fwd.ensure(sizeof(uint32_t) * size_t(e.n)))) return rc;
    if ((rc = e.inv.ensure(sizeof(uint32_t) * size_t(e.n)))) return rc;
    const int64_t sc = order_tokens_scratch_ints(ordering, f, hh, w);
    if ((rc = h->scratch_i32.ensure(sizeof(int) * size_t(sc)))) return rc;
    if ((rc = order_tokens_impl(ordering, f, hh, w, e.fwd.as<uint32_t>(), e.inv.as<uint32_t>(),
                                h->scratch_i32.as<int>(), sc, stream)))
      return rc;
    it = h->perms.emplace(key, std::move(e)).first;
  }
  *out = &it->second;
  return DFS_OK;
}

float resolve_scale(float scale, int64_t d) { return scale > 0.f ? scale : float(1.0 / std::sqrt(double(d))); }

int attn_dispatch(dfs_handle* h, const dfs_attn_args& a, cudaStream_t stream) {
  const float scale = resolve_scale(a.scale, a.d);
  if (a.out_peers && (a.force_generic || h->opt_generic_attn || !attn_sm100_supports(a)))
    return fail(DFS_E_UNSUPPORTED, "sparse_attn: peer-scattered output needs the tcgen05 kernel");
  if (!a.force_generic && !h->opt_generic_attn && attn_sm100_supports(a)) return sparse_attn_sm100(a, scale, stream);
  // bf16 is the performance path: geometry outside the tcgen05 kernel's contract is an
  // explicit refusal, never a silent ~20x slower SIMT fallback. The SIMT
  // kernel serves fp32 (the drop-in Matrix path, fp64 arithmetic) and callers that ask
  // for it (force_generic / DFS_OPT_GENERIC_ATTN).
  if (a.dtype == DFS_BF16 && !a.force_generic && !h->opt_generic_attn)
    return fail(DFS_E_UNSUPPORTED,
                "sparse_attn: the bf16 tensor-core kernel needs B in {64, 128}, d in {64, 128}, dv == d and "
                "16-byte aligned q/k/v/o (got B = " + std::to_string(a.block) + ", d = " + std::to_string(a.d) +
                "); set force_generic / DFS_OPT_GENERIC_ATTN for the SIMT kernel");
  return sparse_attn_generic(a, scale, stream);
}

int score_dispatch(dfs_handle* h, const float* pq, const float* pk, int64_t heads, int64_t n, int64_t d,
                   int64_t block, int64_t sub, double* S, cudaStream_t stream) {
  int rc;
  if (!h->opt_generic_score && score_sm100_supports(d, block, sub)) {
    const int64_t need = score_sm100_ws_bytes(heads, n, d, block, sub);
    if ((rc = h->score_ws.ensure(size_t(need)))) return rc;
    return score_blocks_sm100(pq, pk, heads, n, d, block, sub, S, h->score_ws.p, need, stream);
  }
  const int64_t subs = block / sub;
  const int64_t rows = ceil_div(n, block) * subs;
  const int64_t per_head = rows * rows;
  // batch as many heads as fit in 1 GiB of probability workspace (>= 1)
  int64_t batch = (int64_t(1) << 28) / (per_head > 0 ? per_head : 1);
  if (batch < 1) batch = 1;
  if (batch > heads) batch = heads;
  if ((rc = h->score_ws.ensure(sizeof(float) * size_t(batch * per_head)))) return rc;
  return score_blocks_generic(pq, pk, heads, n, d, block, sub, S, h->score_ws.as<float>(),
                              int64_t(h->score_ws.bytes / sizeof(float)), stream);
}

}  // namespace capi_detail
using namespace capi_detail;

extern "C" {

const char* dfs_last_error(void) { return g_error.c_str(); }
int dfs_abi_version(void) { return DFS_ABI_VERSION; }

int dfs_handle_create(dfs_handle** out, int device) {
  if (!out) return fail(DFS_E_INVALID, "null out");
  int count = 0;
  DFS_CUDA_CHECK(cudaGetDeviceCount(&count));
  if (device < 0 || device >= count) return fail(DFS_E_INVALID, "no such CUDA device");
  DFS_CUDA_CHECK(cudaSetDevice(device));
  cudaDeviceProp prop;
  DFS_CUDA_CHECK(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(DFS_E_UNSUPPORTED, "this library is compiled for sm_100a (B200) only");
  auto* h = new dfs_handle;
  h->device = device;
  if (int rc = h->flag.ensure(64)) {
    delete h;
    return rc;
  }
  *out = h;
  return DFS_OK;
}

int dfs_handle_destroy(dfs_handle* h) {
  if (h) {
    cudaSetDevice(h->device);
    delete h;
  }
  return DFS_OK;
}

int dfs_handle_set_option(dfs_handle* h, int option, int value) {
  if (!h) return fail(DFS_E_INVALID, "null handle");
  switch (option) {
    case DFS_OPT_GENERIC_SCORE:
      h->opt_generic_score = value;
      return DFS_OK;
    case DFS_OPT_GENERIC_ATTN:
      h->opt_generic_attn = value;
      return DFS_OK;
    default:
      return fail(DFS_E_INVALID, "unknown handle option");
  }
}

int dfs_handle_workspace_bytes(dfs_handle* h, int64_t* bytes) {
  if (!h || !bytes) return fail(DFS_E_INVALID, "null argument");
  *bytes = h->total_bytes();
  return DFS_OK;
}

// ---------------------------------------------------------------- K1 -------
int dfs_order_tokens(int ordering, int64_t f, int64_t h, int64_t w, uint32_t* fwd, uint32_t* inv,
                     dfs_stream stream) {
  if (f < 1 || h < 1 || w < 1) return fail(DFS_E_INVALID, "GridDims: extents must be >= 1");
  if (f > (int64_t(1) << 31) / h / w) return fail(DFS_E_INVALID, "GridDims: token count overflows index range");
  if (!fwd) return fail(DFS_E_INVALID, "null forward buffer");
  const int64_t sc = order_tokens_scratch_ints(ordering, f, h, w);
  int* scratch = nullptr;
  DFS_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&scratch), sizeof(int) * size_t(sc), as_stream(stream)));
  const int rc = order_tokens_impl(ordering, f, h, w, fwd, inv, scratch, sc, as_stream(stream));
  cudaFreeAsync(scratch, as_stream(stream));
  return rc;
}

int dfs_invert_permutation(const uint32_t* fwd, int64_t n, uint32_t* inv, dfs_stream stream) {
  if (!fwd || !inv || n < 1) return fail(DFS_E_INVALID, "invert_permutation: bad arguments");
  return invert_permutation_impl(fwd, n, inv, as_stream(stream));
}

int dfs_validate_permutation(dfs_handle* h, const uint32_t* fwd, int64_t n, int* ok_host, dfs_stream stream) {
  if (int rc = check_handle(h)) return rc;
  if (!ok_host) return fail(DFS_E_INVALID, "null ok_host");
  if (n < 1) {
    *ok_host = 0;
    return DFS_OK;
  }
  if (int rc = h->counts.ensure(sizeof(int) * size_t(n))) return rc;
  return validate_permutation_impl(fwd, n, h->counts.as<int>(), h->flag.as<int>(), ok_host, as_stream(stream));
}

// ------------------------------------------------------------- K2 / K6 -----
int dfs_permute_rows(const void* src, int src_layout, void* dst, int dst_layout, int dtype, const uint32_t* idx,
                     int64_t n, int64_t heads, int64_t d, float* pooled, int64_t pool, int32_t* nonfinite,
                     dfs_stream stream) {
  NvtxRange nvtx("dfs_permute_rows");
  if (!src || !idx || (!dst && !pooled && !nonfinite)) return fail(DFS_E_INVALID, "permute_rows: null pointer");
  return permute_rows_impl(src, src_layout, dst, dst_layout, dtype, idx, n, heads, d, pooled, pool, nonfinite,
                           false, as_stream(stream));
}

int dfs_unpermute_rows(const void* src, int src_layout, void* dst, int dst_layout, int dtype, const uint32_t* idx,
                       int64_t n, int64_t heads, int64_t d, dfs_stream stream) {
  if (!src || !dst || !idx) return fail(DFS_E_INVALID, "unpermute_rows: null pointer");
  return permute_rows_impl(src, src_layout, dst, dst_layout, dtype, idx, n, heads, d, nullptr, 1, nullptr, true,
                           as_stream(stream));
}

// ------------------------------------------------------------- K3 / K4 -----
int dfs_score_blocks(dfs_handle* h, const float* pq, const float* pk, int64_t heads, int64_t n, int64_t d,
                     int64_t block, int64_t sub_block, double* scores, dfs_stream stream) {
  NvtxRange nvtx("dfs_score_blocks");
  if (int rc = check_handle(h)) return rc;
  if (sub_block < 1 || block < sub_block)
    return fail(DFS_E_INVALID, "ScoringParams: need 1 <= sub_block_size <= block_size");
  if (block % sub_block) return fail(DFS_E_INVALID, "ScoringParams: sub_block_size must divide block_size");
  if (n < 1 || heads < 1 || d < 1) return fail(DFS_E_INVALID, "score_blocks: empty input");
  return score_dispatch(h, pq, pk, heads, n, d, block, sub_block, scores, as_stream(stream));
}

int dfs_topk_count(double budget, int64_t m, int64_t* k) {
  if (!(budget > 0.0) || budget > 1.0) return fail(DFS_E_INVALID, "budget must lie in (0, 1]");
  if (!k) return fail(DFS_E_INVALID, "null k");
  int64_t kk = std::llround(budget * double(m));  // mask_builder.cpp:85, half away from zero
  if (kk < 1) kk = 1;
  if (kk > m) kk = m;
  *k = kk;
  return DFS_OK;
}

int dfs_topk_select(const double* scores, int64_t heads, int64_t m, int64_t k, int32_t* lut, uint8_t* bits,
                    dfs_stream stream) {
  NvtxRange nvtx("dfs_topk_select");
  if (!scores || m < 1 || heads < 1) return fail(DFS_E_INVALID, "topk_select: scores must be square and non-empty");
  uint8_t* sel = nullptr;
  cudaStream_t s = as_stream(stream);
  if (bits) DFS_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&sel), size_t(heads * m * m), s));
  const int rc = topk_select_impl(scores, heads, m, k, lut, sel, bits, s);
  if (sel) cudaFreeAsync(sel, s);
  return rc;
}

int dfs_mask_bits_to_csr(dfs_handle* h, const uint8_t* bits, int64_t heads, int64_t m, int32_t* blk_ptr,
                         int32_t* blk_idx, int64_t* nnz_host, dfs_stream stream) {
  if (int rc = check_handle(h)) return rc;
  if (int rc = h->counts.ensure(sizeof(int32_t) * size_t(heads * m))) return rc;
  return mask_bits_to_csr_impl(bits, heads, m, blk_ptr, blk_idx, h->counts.as<int32_t>(), h->flag.as<int32_t>(),
                               nnz_host, as_stream(stream));
}

int dfs_lut_row_ptr(int64_t heads, int64_t m, int64_t k, int32_t* blk_ptr, dfs_stream stream) {
  return lut_row_ptr_impl(heads, m, k, blk_ptr, as_stream(stream));
}

// ---------------------------------------------------------------- K5 -------
int dfs_sparse_attn_fwd(dfs_handle* h, const dfs_attn_args* a, dfs_stream stream) {
  NvtxRange nvtx("dfs_sparse_attn_fwd");
  if (int rc = check_handle(h)) return rc;
  if (!a || !a->q || !a->k || !a->v || !a->o) return fail(DFS_E_INVALID, "sparse_attn: null pointer");
  if (a->nq < 1 || a->nk < 1 || a->d < 1 || a->heads < 1)
    return fail(DFS_E_INVALID, "attention: empty input");
  if (a->block < 1) return fail(DFS_E_INVALID, "block_size must be >= 1");
  if ((a->blk_ptr == nullptr) != (a->blk_idx == nullptr))
    return fail(DFS_E_INVALID, "sparse_attn: blk_ptr and blk_idx must both be set or both be NULL");
  return attn_dispatch(h, *a, as_stream(stream));
}

// ---------------------------------------------------------- schedule -------
int dfs_schedule_info(const dfs_schedule* s, int* warmup_steps, int* phase_length) {
  return schedule_validate(s, warmup_steps, phase_length);
}

int dfs_schedule_budget_at(const dfs_schedule* s, int step, double* budget) {
  int w, pl;
  if (int rc = schedule_validate(s, &w, &pl)) return rc;
  if (step < 0 || step >= s->total_steps) return fail(DFS_E_RANGE, "budget_at: step out of range");
  if (step < w) {
    *budget = -1.0;
    return DFS_OK;
  }
  int phase = (step - w) / pl;
  if (phase > s->n_budgets - 1) phase = s->n_budgets - 1;
  *budget = s->phase_budgets[phase];
  return DFS_OK;
}

int dfs_schedule_is_update_step(const dfs_schedule* s, int step, int* is_update) {
  int w, pl;
  if (int rc = schedule_validate(s, &w, &pl)) return rc;
  *is_update = step >= w && ((step - w) % s->update_interval) == 0;
  return DFS_OK;
}

// ---------------------------------------------------------- mask cache -----
int dfs_mask_cache_clear(dfs_handle* h) {
  if (!h) return fail(DFS_E_INVALID, "null handle");
  h->masks.clear();
  return DFS_OK;
}

int dfs_mask_cache_contains(dfs_handle* h, int layer, int head, int* found) {
  if (!h || !found) return fail(DFS_E_INVALID, "null argument");
  auto it = h->masks.find(layer);
  *found = it != h->masks.end() && head >= 0 && head < int(it->second.head.size()) &&
           it->second.head[size_t(head)].valid;
  return DFS_OK;
}

int dfs_mask_cache_size(dfs_handle* h, int64_t* n) {
  if (!h || !n) return fail(DFS_E_INVALID, "null argument");
  int64_t c = 0;
  for (auto& kv : h->masks)
    for (auto& hm : kv.second.head) c += hm.valid;
  *n = c;
  return DFS_OK;
}

}  // extern "C"

namespace capi_detail {

__global__ void csr_to_bits_kernel(const int32_t* __restrict__ ptr, const int32_t* __restrict__ idx, int64_t m,
                                   int64_t row0, uint8_t* __restrict__ sel) {
  const int64_t u = blockIdx.x;
  const int32_t b = ptr[row0 + u], e = ptr[row0 + u + 1];
  for (int32_t t = b + threadIdx.x; t < e; t += blockDim.x) sel[u * m + idx[t]] = 1;
}

__global__ void pack_sel_kernel(const uint8_t* __restrict__ sel, int64_t total, uint8_t* __restrict__ bits) {
  const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b * 8 >= total) return;
  uint8_t o = 0;
  for (int j = 0; j < 8; ++j)
    if (b * 8 + j < total && sel[b * 8 + j]) o |= uint8_t(1u << (7 - j));
  bits[b] = o;
}

__global__ void fill_kernel(int32_t* __restrict__ dst, int64_t count, int32_t value) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < count) dst[i] = value;
}

__global__ void rebase_ptr_kernel(const int32_t* __restrict__ src, int64_t count, int32_t delta,
                                  int32_t* __restrict__ dst) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < count) dst[i] = src[i] + delta;
}

// Rebuild layer L's CSR so that head `hh` holds (ptr_h [m+1] relative, idx_h [nnz]) and
// every other valid head keeps its rows. Rare path (explicit stores, partial updates).
int layer_replace_heads(dfs_handle* h, LayerMasks& L, const std::vector<int>& heads_new,
                        const std::vector<const int32_t*>& ptr_new, const std::vector<const int32_t*>& idx_new,
                        const std::vector<int64_t>& nnz_new, cudaStream_t s) {
  const int64_t H = L.heads, m = L.m;
  std::vector<int64_t> nnz(size_t(H), 0);
  std::vector<int> src(size_t(H), -1);  // index into heads_new, or -1 = keep old
  for (size_t j = 0; j < heads_new.size(); ++j) src[size_t(heads_new[j])] = int(j);
  int64_t total = 0;
  for (int64_t hh = 0; hh < H; ++hh) {
    if (src[size_t(hh)] >= 0)
      nnz[size_t(hh)] = nnz_new[size_t(src[size_t(hh)])];
    else
      nnz[size_t(hh)] = L.head[size_t(hh)].valid ? L.head[size_t(hh)].nnz : 0;
    total += nnz[size_t(hh)];
  }
  Buf nptr, nidx;
  int rc;
  if ((rc = nptr.ensure(sizeof(int32_t) * size_t(H * m + 1)))) return rc;
  if ((rc = nidx.ensure(sizeof(int32_t) * size_t(total > 0 ? total : 1)))) return rc;
  DFS_CUDA_CHECK(cudaMemsetAsync(nptr.p, 0, sizeof(int32_t) * size_t(H * m + 1), s));
  std::vector<int64_t> off(size_t(H), 0);
  int64_t o = 0;
  for (int64_t hh = 0; hh < H; ++hh) {
    off[size_t(hh)] = o;
    const int j = src[size_t(hh)];
    if (j >= 0) {
      rebase_ptr_kernel<<<unsigned(ceil_div(m + 1, 256)), 256, 0, s>>>(ptr_new[size_t(j)], m + 1, int32_t(o),
                                                                         nptr.as<int32_t>() + hh * m);
      if (nnz[size_t(hh)])
        DFS_CUDA_CHECK(cudaMemcpyAsync(nidx.as<int32_t>() + o, idx_new[size_t(j)],
                                       sizeof(int32_t) * size_t(nnz[size_t(hh)]), cudaMemcpyDeviceToDevice, s));
    } else if (L.head[size_t(hh)].valid) {
      const int64_t old = L.head_off[size_t(hh)];
      rebase_ptr_kernel<<<unsigned(ceil_div(m + 1, 256)), 256, 0, s>>>(
          L.ptr.as<int32_t>() + hh * m, m + 1, int32_t(o - old), nptr.as<int32_t>() + hh * m);
      if (nnz[size_t(hh)])
        DFS_CUDA_CHECK(cudaMemcpyAsync(nidx.as<int32_t>() + o, L.idx.as<int32_t>() + old,
                                       sizeof(int32_t) * size_t(nnz[size_t(hh)]), cudaMemcpyDeviceToDevice, s));
    } else {
      // empty head: all its row pointers equal o (keeps the CSR monotone)
      fill_kernel<<<unsigned(ceil_div(m + 1, 256)), 256, 0, s>>>(nptr.as<int32_t>() + hh * m, m + 1, int32_t(o));
    }
    o += nnz[size_t(hh)];
  }
  DFS_LAUNCH_CHECK("layer_replace_heads");
  DFS_CUDA_CHECK(cudaStreamSynchronize(s));  // old buffers are freed below
  std::swap(L.ptr.p, nptr.p);
  std::swap(L.ptr.bytes, nptr.bytes);
  std::swap(L.idx.p, nidx.p);
  std::swap(L.idx.bytes, nidx.bytes);
  L.head_off = off;
  for (int64_t hh = 0; hh < H; ++hh) L.head[size_t(hh)].nnz = nnz[size_t(hh)];
  (void)h;
  return DFS_OK;
}

}  // namespace capi_detail
using namespace capi_detail;

extern "C" {

int dfs_mask_cache_store(dfs_handle* h, int layer, int head, const uint8_t* bits, int64_t m, int64_t block,
                         int step, dfs_stream stream) {
  if (int rc = check_handle(h)) return rc;
  if (head < 0 || m < 1 || !bits) return fail(DFS_E_INVALID, "mask_cache_store: bad arguments");
  cudaStream_t s = as_stream(stream);
  LayerMasks& L = h->masks[layer];
  if (L.m != 0 && (L.m != m || L.block != block)) {
    // a new geometry for this layer replaces every head's mask
    h->masks.erase(layer);
    return dfs_mask_cache_store(h, layer, head, bits, m, block, step, stream);
  }
  if (L.m == 0) {
    L.m = m;
    L.block = block;
  }
  if (int64_t(head) >= L.heads) {
    // grow the head range; existing rows are preserved by the rebuild below
    const int64_t H = int64_t(head) + 1;
    LayerMasks grown;
    grown.heads = H;
    grown.m = m;
    grown.block = block;
    grown.head = L.head;
    grown.head.resize(size_t(H));
    grown.head_off = L.head_off;
    grown.head_off.resize(size_t(H), 0);
    if (L.heads > 0) {
      // carry the old CSR into the grown layout by treating old heads as "new"
      std::vector<int> hs;
      std::vector<const int32_t*> ps, is;
      std::vector<int64_t> ns;
      Buf tmp_ptrs;
      for (int64_t hh = 0; hh < L.heads; ++hh)
        if (L.head[size_t(hh)].valid) {
          hs.push_back(int(hh));
          ps.push_back(L.ptr.as<int32_t>() + hh * m);  // absolute offsets; rebased below
          is.push_back(L.idx.as<int32_t>());
          ns.push_back(L.head[size_t(hh)].nnz);
        }
      // absolute pointers: rebasing by 0 and copying the whole old idx per head
      // would be wrong, so rebuild through relative copies
      std::vector<Buf> rel_ptr(hs.size());
      for (size_t j = 0; j < hs.size(); ++j) {
        const int64_t hh = hs[j];
        if (int rc = rel_ptr[j].ensure(sizeof(int32_t) * size_t(m + 1))) return rc;
        rebase_ptr_kernel<<<unsigned(ceil_div(m + 1, 256)), 256, 0, s>>>(
            L.ptr.as<int32_t>() + hh * m, m + 1, -int32_t(L.head_off[size_t(hh)]), rel_ptr[j].as<int32_t>());
        ps[j] = rel_ptr[j].as<int32_t>();
        is[j] = L.idx.as<int32_t>() + L.head_off[size_t(hh)];
      }
      for (auto& hm : grown.head) hm.valid = false;
      if (int rc = layer_replace_heads(h, grown, hs, ps, is, ns, s)) return rc;
      for (size_t j = 0; j < hs.size(); ++j) grown.head[size_t(hs[j])] = L.head[size_t(hs[j])];
      for (int64_t hh = 0; hh < H; ++hh)
        if (!grown.head[size_t(hh)].valid) grown.head[size_t(hh)].nnz = 0;
    } else {
      if (int rc = grown.ptr.ensure(sizeof(int32_t) * size_t(H * m + 1))) return rc;
      DFS_CUDA_CHECK(cudaMemsetAsync(grown.ptr.p, 0, sizeof(int32_t) * size_t(H * m + 1), s));
      if (int rc = grown.idx.ensure(sizeof(int32_t))) return rc;
    }
    L = std::move(grown);
  }
  // bits -> relative CSR for this head
  Buf ptr1, idx1;
  int64_t nnz = 0;
  if (int rc = ptr1.ensure(sizeof(int32_t) * size_t(m + 1))) return rc;
  if (int rc = idx1.ensure(sizeof(int32_t) * size_t(m * m))) return rc;
  if (int rc = dfs_mask_bits_to_csr(h, bits, 1, m, ptr1.as<int32_t>(), idx1.as<int32_t>(), &nnz, stream)) return rc;
  if (int rc = layer_replace_heads(h, L, {head}, {ptr1.as<int32_t>()}, {idx1.as<int32_t>()}, {nnz}, s)) return rc;
  L.head[size_t(head)].valid = true;
  L.head[size_t(head)].last_update_step = step;
  return DFS_OK;
}

int dfs_mask_cache_get(dfs_handle* h, int layer, int head, uint8_t* bits, int* last_update_step, int64_t* m,
                       dfs_stream stream) {
  if (int rc = check_handle(h)) return rc;
  auto it = h->masks.find(layer);
  if (it == h->masks.end() || head < 0 || head >= int(it->second.head.size()) ||
      !it->second.head[size_t(head)].valid)
    return fail(DFS_E_INVALID, "mask_cache_get: no entry for (layer, head)");
  LayerMasks& L = it->second;
  if (m) *m = L.m;
  if (last_update_step) *last_update_step = L.head[size_t(head)].last_update_step;
  if (!bits) return DFS_OK;
  cudaStream_t s = as_stream(stream);
  uint8_t* sel = nullptr;
  DFS_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&sel), size_t(L.m * L.m), s));
  DFS_CUDA_CHECK(cudaMemsetAsync(sel, 0, size_t(L.m * L.m), s));
  csr_to_bits_kernel<<<unsigned(L.m), 64, 0, s>>>(L.ptr.as<int32_t>(), L.idx.as<int32_t>(), L.m,
                                                 int64_t(head) * L.m, sel);
  const int64_t bytes = (L.m * L.m + 7) / 8;
  pack_sel_kernel<<<unsigned(ceil_div(bytes, 256)), 256, 0, s>>>(sel, L.m * L.m, bits);
  cudaFreeAsync(sel, s);
  DFS_LAUNCH_CHECK("mask_cache_get");
  return DFS_OK;
}

// ------------------------------------------------------------- recall ------
int dfs_block_recall(dfs_handle* h, const void* q, const void* k, int layout, const uint32_t* q_rows, int64_t heads,
                     int64_t n, int64_t d, const int32_t* blk_ptr, const int32_t* blk_idx, double* recall_host,
                     dfs_stream stream) {
  NvtxRange nvtx("dfs_block_recall");
  if (int rc = check_handle(h)) return rc;
  if (!q || !k || !blk_ptr || !blk_idx || !recall_host || heads < 1 || n < 1)
    return fail(DFS_E_INVALID, "block_recall: bad arguments");
  if (!recall_sm100_supports(d)) return fail(DFS_E_UNSUPPORTED, "block_recall: d must be 64 or 128");
  cudaStream_t s = as_stream(stream);
  if (int rc = h->recall_ws.ensure(sizeof(float) * size_t(heads * n) + sizeof(double) * size_t(heads) + 256))
    return rc;
  float* mass = h->recall_ws.as<float>();
  double* rec = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(mass + heads * n) + 255) & ~uintptr_t(255));
  if (int rc = block_recall_sm100(q, k, layout, q_rows, heads, n, d, blk_ptr, blk_idx, mass, rec, s)) return rc;
  DFS_CUDA_CHECK(cudaMemcpyAsync(recall_host, rec, sizeof(double) * size_t(heads), cudaMemcpyDeviceToHost, s));
  DFS_CUDA_CHECK(cudaStreamSynchronize(s));
  return DFS_OK;
}

// ------------------------------------------------------------- misc --------
int dfs_cast(const void* src, int src_dtype, void* dst, int dst_dtype, int64_t count, int32_t* nonfinite,
             dfs_stream stream) {
  if (!src || !dst) return fail(DFS_E_INVALID, "cast: null pointer");
  return cast_impl(src, src_dtype, dst, dst_dtype, count, nonfinite, as_stream(stream));
}

int dfs_qk_prologue_apply(const dfs_qk_prologue* p, int which, const void* src, void* dst, int dst_layout,
                          const uint32_t* idx, int64_t n, int64_t heads, int64_t d, dfs_stream stream) {
  if (!p || !src || !dst || (which != 0 && which != 1)) return fail(DFS_E_INVALID, "qk_prologue: bad arguments");
  if (n < 1 || heads < 1 || d < 1) return fail(DFS_E_INVALID, "qk_prologue: empty input");
  return prologue_permute_impl(src, dst, dst_layout, idx, n, heads, d, nullptr, 1, nullptr,
                               which ? p->k_norm_weight : p->q_norm_weight, p->eps, p->rope_layout, p->rope_cos,
                               p->rope_sin, as_stream(stream));
}

int dfs_mask_cache_info(dfs_handle* h, int layer, int head, int64_t* m, int64_t* block, int* last_update_step) {
  if (!h) return fail(DFS_E_INVALID, "null handle");
  auto it = h->masks.find(layer);
  if (it == h->masks.end() || head < 0 || head >= int(it->second.head.size()) ||
      !it->second.head[size_t(head)].valid)
    return fail(DFS_E_INVALID, "mask_cache_info: no entry for (layer, head)");
  if (m) *m = it->second.m;
  if (block) *block = it->second.block;
  if (last_update_step) *last_update_step = it->second.head[size_t(head)].last_update_step;
  return DFS_OK;
}

}  // extern "C"

namespace capi_detail {

// Reads the step's non-finite flag back (one stream sync, before anything is scored or
// cached): the reference throws from check_qkv / attention_scores before build_mask
// stores a mask (attention.cpp:19-20, scheduler.cpp:114-116), so a NaN step leaves the
// cache and the output untouched here too.
// Both step flags (q/k at flag[0], v at flag[1]) in one read-back on `s`; the caller decides
// when each is reported.
int check_flags2(dfs_handle* h, const int32_t* flag, cudaStream_t s) {
  if (!h->host_flag) DFS_CUDA_CHECK(cudaMallocHost(&h->host_flag, 64));
  DFS_CUDA_CHECK(cudaMemcpyAsync(h->host_flag, flag, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  DFS_CUDA_CHECK(cudaStreamSynchronize(s));
  if (h->host_flag[0]) return fail(DFS_E_INVALID, "attention: non-finite input");
  return DFS_OK;
}

// The read-back goes to pinned memory: a pageable D2H copy is staged by the driver and held
// back the kernels launched right after it (traced: ~175 us of GPU idle per update step).
int check_flag(dfs_handle* h, const int32_t* flag, cudaStream_t s) {
  if (!h->host_flag) DFS_CUDA_CHECK(cudaMallocHost(&h->host_flag, 64));
  DFS_CUDA_CHECK(cudaMemcpyAsync(h->host_flag, flag, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  DFS_CUDA_CHECK(cudaStreamSynchronize(s));
  if (*h->host_flag) return fail(DFS_E_INVALID, "attention: non-finite input");
  return DFS_OK;
}

// attention_recall(attention_scores(rq, rk), mask) per head on the fp32 compatibility
// path (scheduler.cpp:129-131 at n <= kMaxDenseScoreRows): fp64 logits, fp32
// probabilities, the reference's recall sums (dropin.cu), the head's mask taken from the
// layer's device CSR.
int compat_recall(dfs_handle* h, const LayerMasks& L, const float* rq, const float* rk, int64_t H, int64_t n,
                  int64_t d, double* recall_out, cudaStream_t s) {
  int rc;
  const int64_t m = L.m;
  if ((rc = h->probs.ensure(sizeof(float) * size_t(n * n))) || (rc = h->sel.ensure(size_t(m * m))) ||
      (rc = h->bits.ensure(size_t((m * m + 7) / 8))))
    return rc;
  for (int64_t hh = 0; hh < H; ++hh) {
    if ((rc = dfs_softmax_scores(rq + hh * n * d, rk + hh * n * d, 1, n, n, n, n, d, 0.0, h->probs.as<float>(), s)))
      return rc;
    DFS_CUDA_CHECK(cudaMemsetAsync(h->sel.p, 0, size_t(m * m), s));
    csr_to_bits_kernel<<<unsigned(m), 64, 0, s>>>(L.ptr.as<int32_t>(), L.idx.as<int32_t>(), m, hh * m,
                                                  h->sel.as<uint8_t>());
    pack_sel_kernel<<<unsigned(ceil_div((m * m + 7) / 8, 256)), 256, 0, s>>>(h->sel.as<uint8_t>(), m * m,
                                                                           h->bits.as<uint8_t>());
    DFS_LAUNCH_CHECK("compat_recall");
    if ((rc = dfs_attention_recall(h->probs.as<float>(), n, n, h->bits.as<uint8_t>(), m, L.block,
                                   recall_out + hh, s)))
      return rc;
  }
  return DFS_OK;
}

// the compatibility scorer, batched over heads: subblock_scores (fp64 logits, fp32
// probabilities, padded rows uniform; mask_builder.cpp:30-62, attention.cpp:105-123) then
// aggregate_scores (fp64 tile sums, mask_builder.cpp:64-80) — the kernels behind
// dfs::block_scores at n <= kMaxDenseScoreRows
int compat_scores(dfs_handle* h, const float* pq, const float* pk, int64_t H, int64_t n, int64_t d, int64_t B,
                  int64_t Bs, double* S, cudaStream_t s) {
  const int64_t subs = B / Bs, m = ceil_div(n, B), valid = ceil_div(n, Bs), rows = m * subs;
  int64_t batch = (int64_t(1) << 26) / (rows * rows);  // <= 256 MB of probabilities per launch
  batch = batch < 1 ? 1 : (batch > H ? H : batch);
  int rc;
  if ((rc = h->probs.ensure(sizeof(float) * size_t(batch * rows * rows)))) return rc;
  for (int64_t h0 = 0; h0 < H; h0 += batch) {
    const int64_t hb = H - h0 < batch ? H - h0 : batch;
    if ((rc = dfs_softmax_scores(pq + h0 * valid * d, pk + h0 * valid * d, hb, valid, rows, valid, rows, d, 0.0,
                                 h->probs.as<float>(), s)) ||
        (rc = dfs_aggregate_scores(h->probs.as<float>(), hb, m, m, subs, S + h0 * m * m, s)))
      return rc;
  }
  return DFS_OK;
}

// Scoring (K3, or the compatibility scorer), top-K (K4) and the commit of the new masks
// of heads `need` into the layer's device CSR (scheduler.cpp:113-116 build_mask +
// cache.store). Runs only after the step's non-finite check passed.
// K3: block scores of every head into h->scores (scratch: nothing is committed yet)
int score_phase(dfs_handle* h, int64_t H, int64_t m, int64_t n, int64_t d, int64_t B, int64_t Bs, bool compat,
                const float* pq, const float* pk, cudaStream_t s) {
  int rc;
  if ((rc = h->scores.ensure(sizeof(double) * size_t(H * m * m)))) return rc;
  if (compat) return compat_scores(h, pq, pk, H, n, d, B, Bs, h->scores.as<double>(), s);
  return score_dispatch(h, pq, pk, H, n, d, B, Bs, h->scores.as<double>(), s);
}

// K4 over h->scores and the commit of the selected masks into the layer's device CSR cache
int select_commit(dfs_handle* h, int layer, int step, const std::vector<int>& need, int64_t H, int64_t m,
                  int64_t B, double budget, LayerMasks** Lout, cudaStream_t s) {
  int rc;
  int64_t K;
  if ((rc = dfs_topk_count(budget, m, &K))) return rc;
  if (m > topk_max_m()) return fail(DFS_E_UNSUPPORTED, "topk_select: M too large");
  if (int64_t(need.size()) == H) {
    // common case: every head refreshes -> the LUT becomes the layer's CSR in place
    LayerMasks& NL = h->masks[layer];
    NL.heads = H;
    NL.m = m;
    NL.block = B;
    NL.head.assign(size_t(H), HeadMask{});
    NL.head_off.resize(size_t(H));
    if ((rc = NL.ptr.ensure(sizeof(int32_t) * size_t(H * m + 1))) ||
        (rc = NL.idx.ensure(sizeof(int32_t) * size_t(H * m * K))))
      return rc;
    if ((rc = topk_select_impl(h->scores.as<double>(), H, m, K, NL.idx.as<int32_t>(), nullptr, nullptr, s)))
      return rc;
    if ((rc = lut_row_ptr_impl(H, m, K, NL.ptr.as<int32_t>(), s))) return rc;
    for (int64_t hh = 0; hh < H; ++hh) {
      NL.head[size_t(hh)] = HeadMask{true, step, m * K};
      NL.head_off[size_t(hh)] = hh * m * K;
    }
    *Lout = &NL;
    return DFS_OK;
  }
  if ((rc = h->lut.ensure(sizeof(int32_t) * size_t(H * m * K))) ||
      (rc = h->tmp_ptr.ensure(sizeof(int32_t) * size_t(H * m + 1))))
    return rc;
  if ((rc = topk_select_impl(h->scores.as<double>(), H, m, K, h->lut.as<int32_t>(), nullptr, nullptr, s))) return rc;
  if ((rc = lut_row_ptr_impl(1, m, K, h->tmp_ptr.as<int32_t>(), s))) return rc;
  LayerMasks& NL = h->masks[layer];
  if (NL.m == 0) {
    NL.heads = H;
    NL.m = m;
    NL.block = B;
    NL.head.assign(size_t(H), HeadMask{});
    NL.head_off.assign(size_t(H), 0);
    if ((rc = NL.ptr.ensure(sizeof(int32_t) * size_t(H * m + 1)))) return rc;
    DFS_CUDA_CHECK(cudaMemsetAsync(NL.ptr.p, 0, sizeof(int32_t) * size_t(H * m + 1), s));
  }
  std::vector<const int32_t*> ps, is;
  std::vector<int64_t> ns;
  for (int hh : need) {
    ps.push_back(h->tmp_ptr.as<int32_t>());
    is.push_back(h->lut.as<int32_t>() + int64_t(hh) * m * K);
    ns.push_back(m * K);
  }
  if ((rc = layer_replace_heads(h, NL, need, ps, is, ns, s))) return rc;
  for (int hh : need) {
    NL.head[size_t(hh)].valid = true;
    NL.head[size_t(hh)].last_update_step = step;
  }
  *Lout = &NL;
  return DFS_OK;
}

int build_and_commit(dfs_handle* h, int layer, int step, const std::vector<int>& need, int64_t H, int64_t m,
                     int64_t n, int64_t d, int64_t B, int64_t Bs, double budget, bool compat, const float* pq,
                     const float* pk, LayerMasks** Lout, cudaStream_t s) {
  if (int rc = score_phase(h, H, m, n, d, B, Bs, compat, pq, pk, s)) return rc;
  return select_commit(h, layer, step, need, H, m, B, budget, Lout, s);
}

int attn_simple(dfs_handle* h, const void* q, const void* k, const void* v, void* o, int dtype, int in_layout,
                const uint32_t* in_rows, int out_layout, const uint32_t* out_rows, int64_t H, int64_t n, int64_t d,
                int64_t dv, int64_t B, const int32_t* blk_ptr, const int32_t* blk_idx, cudaStream_t s) {
  dfs_attn_args at{};
  at.q = q;
  at.k = k;
  at.v = v;
  at.o = o;
  at.dtype = dtype;
  at.in_layout = in_layout;
  at.in_rows = in_rows;
  at.out_layout = out_layout;
  at.out_rows = out_rows;
  at.heads = H;
  at.nq = n;
  at.nk = n;
  at.d = d;
  at.dv = dv == d ? 0 : dv;
  at.block = B;
  at.blk_ptr = blk_ptr;
  at.blk_idx = blk_idx;
  return attn_dispatch(h, at, s);
}

}  // namespace capi_detail
using namespace capi_detail;

extern "C" {

// ------------------------------------------------------------ run_step -----
// scheduler.cpp:91-135 run_step for all heads of a layer. Three input regimes:
//   bf16            the performance path: K2 (pool / permute), K3 tcgen05, K4, K5 tcgen05
//                   with the Q gather and the unpermute fused in;
//   fp32, n <= cap  compatibility kernels (fp64 softmax arithmetic) bit-identical to the
//                   dfs:: Matrix operators the reference's unit suites pin at 1e-5;
//   fp32, n > cap   pooling and scoring from the fp32 values (tcgen05 fp16x3 = fp32
//                   accurate), inputs rounded to bf16 for K5, output converted back.
int dfs_run_step(dfs_handle* h, const dfs_schedule* sched, const dfs_step_args* a, dfs_stream stream) {
  NvtxRange nvtx("dfs_run_step");
  if (int rc = check_handle(h)) return rc;
  if (!a || !a->q || !a->k || !a->v || !a->o) return fail(DFS_E_INVALID, "run_step: null pointer");
  cudaStream_t s = as_stream(stream);
  const int64_t n = a->n, H = a->heads, d = a->d, B = a->block, Bs = a->sub_block;
  const int64_t dv = a->dv > 0 ? a->dv : d;
  const int dtype = a->dtype;
  if (dtype != DFS_BF16 && dtype != DFS_F32) return fail(DFS_E_INVALID, "run_step: dtype must be bf16 or f32");
  if (n < 1 || H < 1 || d < 1) return fail(DFS_E_INVALID, "attention: empty input");
  if (Bs < 1 || B < Bs) return fail(DFS_E_INVALID, "ScoringParams: need 1 <= sub_block_size <= block_size");
  if (B % Bs) return fail(DFS_E_INVALID, "ScoringParams: sub_block_size must divide block_size");
  // the tcgen05 attention kernel's geometry contract, checked before anything runs
  auto tc_ok = [&](const void* q, const void* k, const void* v, const void* o) {
    dfs_attn_args pr{};
    pr.q = q;
    pr.k = k;
    pr.v = v;
    pr.o = const_cast<void*>(o);
    pr.dtype = DFS_BF16;
    pr.heads = H;
    pr.nq = n;
    pr.nk = n;
    pr.d = d;
    pr.dv = dv == d ? 0 : dv;
    pr.block = B;
    pr.in_rows = reinterpret_cast<const uint32_t*>(a->q);  // the sparse step gathers Q rows
    return attn_sm100_supports(pr);
  };
  // fp32 inputs: compatibility kernels up to the cap, and for any geometry the tensor-core
  // kernels do not cover (the drop-in Matrix API accepts every shape the reference does)
  const bool compat = dtype == DFS_F32 && (n <= DFS_COMPAT_MAX_ROWS || dv != d || !tc_ok(h, h, h, h));
  if (dtype == DFS_BF16 && !h->opt_generic_attn && !tc_ok(a->q, a->k, a->v, a->o))
    return fail(DFS_E_UNSUPPORTED,
                "run_step: bf16 steps run the tensor-core kernels (B in {64, 128}, d in {64, 128}, 16-byte aligned "
                "[N, H, d] tensors); got B = " + std::to_string(B) + ", d = " + std::to_string(d) +
                " (DFS_OPT_GENERIC_ATTN selects the SIMT kernel)");
  if (dv != d && !compat)
    return fail(DFS_E_UNSUPPORTED, "run_step: dv != d only on the fp32 compatibility path");
  const dfs_qk_prologue* pro = a->prologue;
  if (pro && (dtype != DFS_BF16 || d % 16))
    return fail(DFS_E_UNSUPPORTED, "run_step: the QK-norm / RoPE prologue runs on bf16 steps with d % 16 == 0");
  if (pro && pro->rope_layout != DFS_ROPE_NONE && pro->rope_layout != DFS_ROPE_INTERLEAVED &&
      pro->rope_layout != DFS_ROPE_HALF)
    return fail(DFS_E_INVALID, "run_step: unknown RoPE layout");
  double budget;
  if (int rc = dfs_schedule_budget_at(sched, a->step, &budget)) return rc;
  const int64_t m = ceil_div(n, B);
  int rc;
  int32_t* flag = a->nonfinite;
  if ((rc = h->step_flag.ensure(2 * sizeof(int32_t)))) return rc;
  int32_t* flag_v = h->step_flag.as<int32_t>() + 1;  // V's, when its reorder runs on the side stream
  if (!flag) {
    flag = h->step_flag.as<int32_t>();
    DFS_CUDA_CHECK(cudaMemsetAsync(flag, 0, 2 * sizeof(int32_t), s));
  } else {
    DFS_CUDA_CHECK(cudaMemsetAsync(flag_v, 0, sizeof(int32_t), s));
  }
  bool v_aside = false;  // V reordered on h->aux (joined before K5)
  bool v_late = false;   // V's finite flag (flag_v) is checked after the mask commit
  // q or k through the prologue: raster -> dst (reordered by idx, or raster for idx == NULL)
  auto prologue = [&](const void* x, void* dst, int layout, const uint32_t* idx, float* pooled, const float* w) {
    return prologue_permute_impl(x, dst, layout, idx, n, H, d, pooled, Bs, flag, w, pro->eps, pro->rope_layout,
                                 pro->rope_cos, pro->rope_sin, s);
  };
  const size_t tok16 = sizeof(__nv_bfloat16) * size_t(n * H * d);
  // fp32 inputs past the cap: bf16 copies for the tensor-core kernels (finite check folded in)
  auto cast_inputs = [&]() -> int {
    int r;
    if ((r = h->q16.ensure(tok16)) || (r = h->k16.ensure(tok16)) || (r = h->v16.ensure(tok16))) return r;
    if ((r = cast_impl(a->q, DFS_F32, h->q16.p, DFS_BF16, n * H * d, flag, s)) ||
        (r = cast_impl(a->k, DFS_F32, h->k16.p, DFS_BF16, n * H * d, flag, s)) ||
        (r = cast_impl(a->v, DFS_F32, h->v16.p, DFS_BF16, n * H * d, flag, s)))
      return r;
    return DFS_OK;
  };

  if (budget < 0.0 || a->force_dense) {  // scheduler.cpp:99-105: dense, raster order, no reorder
    if (pro) {  // normalised / rotated q and k in raster order, then dense attention
      if ((rc = h->q16.ensure(tok16)) || (rc = h->k16.ensure(tok16))) return rc;
      if ((rc = prologue(a->q, h->q16.p, DFS_NHD, nullptr, nullptr, pro->q_norm_weight)) ||
          (rc = prologue(a->k, h->k16.p, DFS_NHD, nullptr, nullptr, pro->k_norm_weight)) ||
          (rc = finite_check_impl(a->v, n * H * d, DFS_BF16, flag, s)) || (rc = check_flag(h, flag, s)))
        return rc;
      if ((rc = attn_simple(h, h->q16.p, h->k16.p, a->v, a->o, DFS_BF16, DFS_NHD, nullptr, DFS_NHD, nullptr, H, n, d,
                            d, B, nullptr, nullptr, s)))
        return rc;
    } else if (dtype == DFS_BF16 || compat) {
      const int64_t c[3] = {n * H * d, n * H * d, n * H * dv};
      const void* x[3] = {a->q, a->k, a->v};
      for (int t = 0; t < 3; ++t)
        if ((rc = finite_check_impl(x[t], c[t], dtype, flag, s))) return rc;
      if ((rc = check_flag(h, flag, s))) return rc;
      if ((rc = attn_simple(h, a->q, a->k, a->v, a->o, dtype, DFS_NHD, nullptr, DFS_NHD, nullptr, H, n, d, dv, B,
                            nullptr, nullptr, s)))
        return rc;
    } else {
      if ((rc = cast_inputs()) || (rc = check_flag(h, flag, s))) return rc;
      if ((rc = h->o16.ensure(tok16))) return rc;
      if ((rc = attn_simple(h, h->q16.p, h->k16.p, h->v16.p, h->o16.p, DFS_BF16, DFS_NHD, nullptr, DFS_NHD, nullptr,
                            H, n, d, d, B, nullptr, nullptr, s)) ||
          (rc = cast_impl(h->o16.p, DFS_BF16, a->o, DFS_F32, n * H * d, nullptr, s)))
        return rc;
    }
    if (a->dense_out) *a->dense_out = 1;
    if (a->budget_out) *a->budget_out = 1.0;
    if (a->recall_out)
      for (int64_t hh = 0; hh < H; ++hh) a->recall_out[hh] = 1.0;  // StepStats{} default (scheduler.hpp:78-85)
    for (int64_t hh = 0; hh < H; ++hh) {
      if (a->updated_out) a->updated_out[hh] = 0;
      if (a->sparsity_out) a->sparsity_out[hh] = 0.0;
    }
    return DFS_OK;
  }

  // sparse: reorder
  const uint32_t* fwd = a->perm;
  if (!fwd) {
    const PermEntry* pe;
    if ((rc = get_perm(h, DFS_HILBERT3D, a->frames, a->height, a->width, s, &pe))) return rc;
    if (pe->n != n) return fail(DFS_E_INVALID, "run_step: permutation length does not match token count");
    fwd = pe->fwd.as<uint32_t>();
  }
  // which heads need a fresh mask (scheduler.cpp:85-89)
  int is_upd = 0;
  dfs_schedule_is_update_step(sched, a->step, &is_upd);
  LayerMasks* L = nullptr;
  {
    auto it = h->masks.find(a->layer);
    if (it != h->masks.end()) {
      if (it->second.m != m || it->second.block != B || it->second.heads != H)
        h->masks.erase(it);  // geometry changed: nothing reusable
      else
        L = &it->second;
    }
  }
  std::vector<int> need;
  for (int64_t hh = 0; hh < H; ++hh)
    if (is_upd || !L || !L->head[size_t(hh)].valid) need.push_back(int(hh));
  const bool update_any = !need.empty();

  const int64_t pv = ceil_div(n, Bs);
  float* pq = nullptr;
  float* pk = nullptr;
  if (update_any) {
    if ((rc = h->pooled_q.ensure(sizeof(float) * size_t(H * pv * d))) ||
        (rc = h->pooled_k.ensure(sizeof(float) * size_t(H * pv * d))))
      return rc;
    pq = h->pooled_q.as<float>();
    pk = h->pooled_k.as<float>();
  }
  // attention operands after the reorder
  const void *att_q = a->q, *att_k = nullptr, *att_v = nullptr;
  if (compat) {
    // reorder q, k, v into fp32 [H, N, d] (pooled rows of q and k fused in)
    if ((rc = h->f32_q.ensure(sizeof(float) * size_t(n * H * d))) ||
        (rc = h->f32_k.ensure(sizeof(float) * size_t(n * H * d))) ||
        (rc = h->f32_v.ensure(sizeof(float) * size_t(n * H * dv))))
      return rc;
    if ((rc = permute_rows_impl(a->q, DFS_NHD, h->f32_q.p, DFS_HND, DFS_F32, fwd, n, H, d, pq, update_any ? Bs : 1,
                                flag, false, s)) ||
        (rc = permute_rows_impl(a->k, DFS_NHD, h->f32_k.p, DFS_HND, DFS_F32, fwd, n, H, d, pk, update_any ? Bs : 1,
                                flag, false, s)) ||
        (rc = permute_rows_impl(a->v, DFS_NHD, h->f32_v.p, DFS_HND, DFS_F32, fwd, n, H, dv, nullptr, 1, flag_v, false,
                                s)))
      return rc;
    v_late = true;
    att_q = h->f32_q.p;
    att_k = h->f32_k.p;
    att_v = h->f32_v.p;
  } else {
    // Reorder: Q is gathered by K5 itself (TMA tile::gather4 by `fwd`, once per query
    // tile), so an update step only reads q for its pooled sub-block rows; K and V are
    // re-read by every query block that selects them, so they get one permuted [H, N, d]
    // copy each (K with the pooled rows fused in).
    if ((rc = h->k_hnd.ensure(tok16)) || (rc = h->v_hnd.ensure(tok16))) return rc;
    att_k = h->k_hnd.p;
    att_v = h->v_hnd.p;
    const void *q = a->q, *k = a->k, *v = a->v;
    if (dtype == DFS_F32) {
      // pooled rows from the fp32 values (what dfs::build_mask scores), then bf16 copies
      if (update_any &&
          ((rc = permute_rows_impl(a->q, DFS_NHD, nullptr, DFS_HND, DFS_F32, fwd, n, H, d, pq, Bs, nullptr, false, s)) ||
           (rc = permute_rows_impl(a->k, DFS_NHD, nullptr, DFS_HND, DFS_F32, fwd, n, H, d, pk, Bs, nullptr, false, s))))
        return rc;
      if ((rc = cast_inputs())) return rc;
      q = h->q16.p;
      k = h->k16.p;
      v = h->v16.p;
      att_q = q;
      pq = pk = nullptr;  // already pooled
    }
    // V's reordered copy is read only by K5: on the bf16 path it runs on the side stream from
    // the start of the step, next to the q and k passes (the q pass alone does not saturate
    // HBM) and under the flag read-back and K3/K4
    if (!pro && dtype == DFS_BF16) {
      if ((rc = h->ensure_aux())) return rc;
      DFS_CUDA_CHECK(cudaEventRecord(h->ev_fork, s));  // after the flag reset
      DFS_CUDA_CHECK(cudaStreamWaitEvent(h->aux, h->ev_fork, 0));
      if ((rc = permute_rows_impl(v, DFS_NHD, h->v_hnd.p, DFS_HND, DFS_BF16, fwd, n, H, d, nullptr, 1, flag_v, false,
                                  h->aux)))
        return rc;
      DFS_CUDA_CHECK(cudaEventRecord(h->ev_v, h->aux));
      v_aside = v_late = true;
    }
    if (pro) {
      // QK-norm / RoPE fused into the reorder: the transformed q gets a reordered copy
      // (K5 then loads Q tiles instead of gathering raster rows), k goes to k_hnd
      if ((rc = h->q16.ensure(tok16))) return rc;
      if ((rc = prologue(q, h->q16.p, DFS_HND, fwd, pq, pro->q_norm_weight)) ||
          (rc = prologue(k, h->k_hnd.p, DFS_HND, fwd, pk, pro->k_norm_weight)) ||
          (rc = permute_rows_impl(v, DFS_NHD, h->v_hnd.p, DFS_HND, DFS_BF16, fwd, n, H, d, nullptr, 1, flag, false, s)))
        return rc;
      att_q = h->q16.p;
      k = v = nullptr;  // done
    } else if (pq) {
      if ((rc = permute_rows_impl(q, DFS_NHD, nullptr, DFS_HND, DFS_BF16, fwd, n, H, d, pq, Bs, flag, false, s)))
        return rc;
    } else if (dtype == DFS_BF16 && (rc = finite_check_impl(q, n * H * d, DFS_BF16, flag, s))) {
      return rc;
    }
    if (!pro && (rc = permute_rows_impl(k, DFS_NHD, h->k_hnd.p, DFS_HND, DFS_BF16, fwd, n, H, d, pk, pk ? Bs : 1,
                                        flag, false, s)))
      return rc;
    if (!pro && !v_aside && (rc = permute_rows_impl(v, DFS_NHD, h->v_hnd.p, DFS_HND, DFS_BF16, fwd, n, H, d, nullptr,
                                                    1, flag, false, s)))
      return rc;
  }
  if (v_aside && update_any && flag + 1 == flag_v) {
    // The non-finite read-back overlaps K3: both flags are copied on the side stream once K2
    // (main stream) and V's reorder (side stream) are done, K3 is launched, and the host waits
    // for the copy while the scorer runs. K3 writes scratch only; K4 and the mask commit are
    // launched after the check (the reference throws before build_mask stores anything).
    DFS_CUDA_CHECK(cudaEventRecord(h->ev_fork, s));
    DFS_CUDA_CHECK(cudaStreamWaitEvent(h->aux, h->ev_fork, 0));
    if ((rc = score_phase(h, H, m, n, d, B, Bs, false, h->pooled_q.as<float>(), h->pooled_k.as<float>(), s)))
      return rc;
    if ((rc = check_flags2(h, flag, h->aux))) return rc;  // q, k (slot 0) and v (slot 1)
    if ((rc = select_commit(h, a->layer, a->step, need, H, m, B, budget, &L, s))) return rc;
    if (h->host_flag[1]) return fail(DFS_E_INVALID, "attention: non-finite input");  // after the commit, as v's
    DFS_CUDA_CHECK(cudaStreamWaitEvent(s, h->ev_v, 0));
    v_late = false;
  } else {
    if ((rc = check_flag(h, flag, s))) return rc;  // nothing scored, cached or written yet
    if (update_any && (rc = build_and_commit(h, a->layer, a->step, need, H, m, n, d, B, Bs, budget, compat,
                                               h->pooled_q.as<float>(), h->pooled_k.as<float>(), &L, s)))
      return rc;
  }

  if (v_late) {
    // V is checked like the reference's block_sparse_attention checks it: after build_mask
    // stored the mask (scheduler.cpp:113-122), before any output is produced
    if ((rc = check_flag(h, flag_v, v_aside ? h->aux : s))) return rc;
    if (v_aside) DFS_CUDA_CHECK(cudaStreamWaitEvent(s, h->ev_v, 0));
  }
  // attention over the selected blocks; output row i -> raster row fwd[i] (scheduler.cpp:134)
  if (compat) {
    rc = attn_simple(h, att_q, att_k, att_v, a->o, DFS_F32, DFS_HND, nullptr, DFS_NHD, fwd, H, n, d, dv, B,
                     L->ptr.as<int32_t>(), L->idx.as<int32_t>(), s);
  } else if (dtype == DFS_F32) {
    if ((rc = h->o16.ensure(tok16))) return rc;
    rc = attn_simple(h, att_q, att_k, att_v, h->o16.p, DFS_BF16, DFS_HND, fwd, DFS_NHD, fwd, H, n, d, d, B,
                     L->ptr.as<int32_t>(), L->idx.as<int32_t>(), s);
    if (!rc) rc = cast_impl(h->o16.p, DFS_BF16, a->o, DFS_F32, n * H * d, nullptr, s);
  } else {
    rc = attn_simple(h, att_q, att_k, att_v, a->o, DFS_BF16, DFS_HND, pro ? nullptr : fwd, DFS_NHD, fwd, H, n, d, d, B,
                     L->ptr.as<int32_t>(), L->idx.as<int32_t>(), s);
  }
  if (rc) return rc;

  if (a->recall_out) {  // scheduler.cpp:129-131; past the reference's 4096-row cap via the streamed kernel
    if (compat)
      rc = compat_recall(h, *L, h->f32_q.as<float>(), h->f32_k.as<float>(), H, n, d, a->recall_out, s);
    else
      rc = dfs_block_recall(h, att_q, h->k_hnd.p, DFS_HND, pro ? nullptr : fwd, H, n, d, L->ptr.as<int32_t>(),
                            L->idx.as<int32_t>(),
                            a->recall_out, stream);
    if (rc) return rc;
  }
  if (a->dense_out) *a->dense_out = 0;
  if (a->budget_out) *a->budget_out = budget;
  for (int64_t hh = 0; hh < H; ++hh) {
    const bool upd = std::find(need.begin(), need.end(), int(hh)) != need.end();
    if (a->updated_out) a->updated_out[hh] = upd;
    if (a->sparsity_out) a->sparsity_out[hh] = 1.0 - double(L->head[size_t(hh)].nnz) / (double(m) * double(m));
  }
  return DFS_OK;
}

// ------------------------------------------------------------ Ulysses ------
}  // extern "C"

namespace capi_detail {
// cuMemGetAddressRange through the runtime's driver entry point (the library does not
// link libcuda directly, so it loads on machines without a driver: the CPU test suite)
int mem_range(const void* p, CUdeviceptr* base, size_t* size) {
  using Fn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static Fn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &ptr, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return fail(DFS_E_CUDA, "cuMemGetAddressRange unavailable");
    fn = reinterpret_cast<Fn>(ptr);
  }
  if (fn(base, size, reinterpret_cast<CUdeviceptr>(p)) != CUDA_SUCCESS)
    return fail(DFS_E_INVALID, "alltoall: not a device allocation");
  return DFS_OK;
}
}  // namespace capi_detail

extern "C" {

int dfs_alltoall_export(const void* dev_ptr, dfs_peer_handle* out) {
  static_assert(sizeof(out->bytes) == sizeof(cudaIpcMemHandle_t), "IPC handle size");
  if (!dev_ptr || !out) return fail(DFS_E_INVALID, "alltoall_export: null argument");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (int rc = mem_range(dev_ptr, &base, &size)) return rc;
  cudaIpcMemHandle_t hd;
  DFS_CUDA_CHECK(cudaIpcGetMemHandle(&hd, reinterpret_cast<void*>(base)));
  std::memcpy(out->bytes, &hd, sizeof(hd));
  out->offset = int64_t(reinterpret_cast<CUdeviceptr>(dev_ptr) - base);
  return DFS_OK;
}

namespace {
struct Mapped {
  void* base;
  int refs;
};
std::mutex g_ipc_mu;
std::map<std::string, Mapped> g_ipc;  // handle bytes -> mapping
}  // namespace

int dfs_alltoall_import(const dfs_peer_handle* handle, void** dev_ptr) {
  if (!handle || !dev_ptr) return fail(DFS_E_INVALID, "alltoall_import: null argument");
  std::lock_guard<std::mutex> g(g_ipc_mu);
  const std::string key(reinterpret_cast<const char*>(handle->bytes), sizeof(handle->bytes));
  auto it = g_ipc.find(key);
  if (it == g_ipc.end()) {
    cudaIpcMemHandle_t hd;
    std::memcpy(&hd, handle->bytes, sizeof(hd));
    void* base = nullptr;
    DFS_CUDA_CHECK(cudaIpcOpenMemHandle(&base, hd, cudaIpcMemLazyEnablePeerAccess));
    it = g_ipc.emplace(key, Mapped{base, 0}).first;
  }
  ++it->second.refs;
  *dev_ptr = static_cast<char*>(it->second.base) + handle->offset;
  return DFS_OK;
}

int dfs_alltoall_close(void* dev_ptr) {
  if (!dev_ptr) return fail(DFS_E_INVALID, "alltoall_close: null pointer");
  std::lock_guard<std::mutex> g(g_ipc_mu);
  for (auto it = g_ipc.begin(); it != g_ipc.end(); ++it) {
    CUdeviceptr base = 0;
    size_t size = 0;
    if (mem_range(it->second.base, &base, &size)) continue;
    const auto p = reinterpret_cast<CUdeviceptr>(dev_ptr);
    if (p < base || p >= base + size) continue;
    if (--it->second.refs == 0) {
      cudaIpcCloseMemHandle(it->second.base);
      g_ipc.erase(it);
    }
    return DFS_OK;
  }
  return fail(DFS_E_INVALID, "alltoall_close: pointer was not imported");
}

// scheduler.cpp:91-135 for the rank's head group on sequence-sharded activations: the
// seq->head all-to-all is K2's P2P gather, the head->seq all-to-all K5's P2P epilogue.
int dfs_alltoall_run_step(dfs_handle* h, const dfs_schedule* sched, const dfs_alltoall_step_args* a,
                          dfs_stream stream) {
  NvtxRange nvtx("dfs_alltoall_run_step");
  if (int rc = check_handle(h)) return rc;
  if (!a) return fail(DFS_E_INVALID, "alltoall_run_step: null arguments");
  const int P = a->world;
  if (P < 1 || P > DFS_MAX_PEERS || a->rank < 0 || a->rank >= P)
    return fail(DFS_E_INVALID, "alltoall_run_step: world must be 1..16 and 0 <= rank < world");
  if (a->heads < 1 || a->heads % P) return fail(DFS_E_INVALID, "alltoall_run_step: heads must split over the ranks");
  const int64_t nl = a->n_local, n = nl * P, Ht = a->heads, Hl = Ht / P, d = a->d, B = a->block, Bs = a->sub_block;
  if (nl < 1 || a->frames * a->height * a->width != n)
    return fail(DFS_E_INVALID, "alltoall_run_step: world * n_local must equal the lattice's token count");
  for (int r = 0; r < P; ++r)
    if (!a->q[r] || !a->k[r] || !a->v[r] || !a->o[r]) return fail(DFS_E_INVALID, "alltoall_run_step: null shard");
  if (Bs < 1 || B < Bs || B % Bs) return fail(DFS_E_INVALID, "ScoringParams: sub_block_size must divide block_size");
  if (B != 128 || (d != 64 && d != 128))
    return fail(DFS_E_UNSUPPORTED, "alltoall_run_step: the fused exchange runs on the tcgen05 kernels (B = 128, d = 64|128)");
  cudaStream_t s = as_stream(stream);
  double budget;
  int rc;
  if ((rc = dfs_schedule_budget_at(sched, a->step, &budget))) return rc;
  const int64_t m = ceil_div(n, B);
  const int64_t h0 = int64_t(a->rank) * Hl;

  // peer tables: q, k, v, o (device, read by K2 and K5's epilogue)
  dfs_peer_table tab[4] = {};
  for (int t = 0; t < 4; ++t) {
    tab[t].n_local = nl;
    tab[t].heads_total = Ht;
    tab[t].h0 = h0;
  }
  for (int r = 0; r < P; ++r) {
    tab[0].ptr[r] = a->q[r];
    tab[1].ptr[r] = a->k[r];
    tab[2].ptr[r] = a->v[r];
    tab[3].ptr[r] = a->o[r];
  }
  if ((rc = h->peer_tabs.ensure(sizeof(tab)))) return rc;
  DFS_CUDA_CHECK(cudaMemcpyAsync(h->peer_tabs.p, tab, sizeof(tab), cudaMemcpyHostToDevice, s));
  DFS_CUDA_CHECK(cudaStreamSynchronize(s));  // tab is on the host stack
  const dfs_peer_table* dtab = h->peer_tabs.as<dfs_peer_table>();

  if ((rc = h->step_flag.ensure(sizeof(int32_t)))) return rc;
  int32_t* flag = h->step_flag.as<int32_t>();
  DFS_CUDA_CHECK(cudaMemsetAsync(flag, 0, sizeof(int32_t), s));
  const size_t tok16 = sizeof(__nv_bfloat16) * size_t(n * Hl * d);
  if ((rc = h->q16.ensure(tok16)) || (rc = h->k_hnd.ensure(tok16)) || (rc = h->v_hnd.ensure(tok16))) return rc;

  const bool dense = budget < 0.0 || a->force_dense;
  const PermEntry* pe;
  // dense steps run in raster order (scheduler.cpp:99-105): the identity gather
  if ((rc = get_perm(h, dense ? DFS_RASTER : DFS_HILBERT3D, dense ? n : a->frames, dense ? 1 : a->height,
                     dense ? 1 : a->width, s, &pe)))
    return rc;
  const uint32_t* fwd = pe->fwd.as<uint32_t>();

  std::vector<int> need;
  LayerMasks* L = nullptr;
  if (!dense) {
    int is_upd = 0;
    dfs_schedule_is_update_step(sched, a->step, &is_upd);
    auto it = h->masks.find(a->layer);
    if (it != h->masks.end()) {
      if (it->second.m != m || it->second.block != B || it->second.heads != Hl)
        h->masks.erase(it);
      else
        L = &it->second;
    }
    for (int64_t hh = 0; hh < Hl; ++hh)
      if (is_upd || !L || !L->head[size_t(hh)].valid) need.push_back(int(hh));
  }
  const bool update_any = !need.empty();
  const int64_t pv = ceil_div(n, Bs);
  if (update_any && ((rc = h->pooled_q.ensure(sizeof(float) * size_t(Hl * pv * d))) ||
                     (rc = h->pooled_k.ensure(sizeof(float) * size_t(Hl * pv * d)))))
    return rc;
  float* pq = update_any ? h->pooled_q.as<float>() : nullptr;
  float* pk = update_any ? h->pooled_k.as<float>() : nullptr;
  // K2 over the peers: this rank's heads of every token, reordered, pooled, finite-checked
  if ((rc = permute_rows_peer_impl(dtab + 0, Ht, h->q16.p, fwd, n, Hl, d, pq, pq ? Bs : 1, flag, s)) ||
      (rc = permute_rows_peer_impl(dtab + 1, Ht, h->k_hnd.p, fwd, n, Hl, d, pk, pk ? Bs : 1, flag, s)) ||
      (rc = permute_rows_peer_impl(dtab + 2, Ht, h->v_hnd.p, fwd, n, Hl, d, nullptr, 1, flag, s)))
    return rc;
  if ((rc = check_flag(h, flag, s))) return rc;
  if (update_any &&
      (rc = build_and_commit(h, a->layer, a->step, need, Hl, m, n, d, B, Bs, budget, false, pq, pk, &L, s)))
    return rc;

  dfs_attn_args at{};
  at.q = h->q16.p;
  at.k = h->k_hnd.p;
  at.v = h->v_hnd.p;
  at.o = a->o[a->rank];
  at.dtype = DFS_BF16;
  at.in_layout = DFS_HND;
  at.out_layout = DFS_NHD;
  at.heads = Hl;
  at.nq = n;
  at.nk = n;
  at.d = d;
  at.block = B;
  at.blk_ptr = dense ? nullptr : L->ptr.as<int32_t>();
  at.blk_idx = dense ? nullptr : L->idx.as<int32_t>();
  at.out_rows = dense ? nullptr : fwd;
  at.out_peers = dtab + 3;
  if (!attn_sm100_supports(at) || h->opt_generic_attn)
    return fail(DFS_E_UNSUPPORTED, "alltoall_run_step: shards must be 16-byte aligned for the tcgen05 kernel");
  if ((rc = sparse_attn_sm100(at, resolve_scale(0.f, d), s))) return rc;

  if (a->dense_out) *a->dense_out = dense;
  if (a->budget_out) *a->budget_out = dense ? 1.0 : budget;
  for (int64_t hh = 0; hh < Hl; ++hh) {
    const bool upd = std::find(need.begin(), need.end(), int(hh)) != need.end();
    if (a->updated_out) a->updated_out[hh] = upd;
    if (a->sparsity_out)
      a->sparsity_out[hh] = dense ? 0.0 : 1.0 - double(L->head[size_t(hh)].nnz) / (double(m) * double(m));
  }
  return DFS_OK;
}

}  // extern "C"
