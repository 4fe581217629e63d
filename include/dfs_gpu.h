/* include/dfs_gpu.h — the drop-in C ABI of the B200-native DFSAttn hot path.
 *
 * Plain C: POD arguments, raw device pointers, sizes and a cudaStream_t passed
 * as void*. No torch / C++ types cross this boundary. The C++ drop-in shim
 * (include/dfs/*.hpp, namespace dfs::) is implemented on top of these entry
 * points; Python (paper_2605_23445_b200/_capi.py) binds them with ctypes.
 *
 * Reference interfaces replaced (paths relative to /root/reference/proj):
 *   reorder      include/dfs/curve.hpp:28-54        (curve.cpp:27-185)
 *   score/mask   include/dfs/mask_builder.hpp:27-57 (mask_builder.cpp:12-124)
 *   sparse-attn  include/dfs/attention.hpp:20-33    (attention.cpp:95-159)
 *   mask cache   include/dfs/scheduler.hpp:20-140   (scheduler.cpp:18-186)
 *
 * Conventions
 *   - Status: 0 ok; negative on error. DFS_E_INVALID mirrors the reference's
 *     std::invalid_argument, DFS_E_RANGE its std::out_of_range. The message is
 *     thread-local: dfs_last_error().
 *   - Every entry point is reentrant; a dfs_handle owns workspaces and the
 *     device mask cache and must not be used by two threads at once (one
 *     handle per thread or per stream). Nothing else is global.
 *   - Token tensors on device are either
 *       NHD: [N, H, d] token-major (raster order; the caller's activations), or
 *       HND: [H, N, d] head-major (reordered; the path's internal layout).
 *     dtype is DFS_BF16 (performance path) or DFS_F32 (drop-in Matrix path).
 *   - Block masks are CSR over (head, query block): blk_ptr[H*M+1] and
 *     blk_idx[nnz] ascending key-block indices, or BlockMask bit payloads
 *     (M*M bits row-major, MSB-first, block_mask.hpp:15-80).
 *   - No CPU fallback: unsupported geometry returns DFS_E_UNSUPPORTED.
 */
#ifndef DFS_GPU_H
#define DFS_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DFS_ABI_VERSION 2

/* attention.hpp:16 kMaxDenseScoreRows: up to this many tokens a DFS_F32 step runs the
 * compatibility kernels (fp64 softmax arithmetic, the reference's 1e-5 tolerances);
 * past it, fp32 inputs are rounded to bf16 for the tcgen05 kernels (2e-2 tolerance). */
#define DFS_COMPAT_MAX_ROWS 4096

enum dfs_status {
  DFS_OK = 0,
  DFS_E_INVALID = -1,     /* std::invalid_argument in the reference */
  DFS_E_RANGE = -2,       /* std::out_of_range in the reference */
  DFS_E_UNSUPPORTED = -3, /* geometry outside the compiled kernels' contract */
  DFS_E_CUDA = -4,        /* CUDA runtime / launch failure */
  DFS_E_INTERNAL = -5
};

enum dfs_dtype { DFS_BF16 = 0, DFS_F32 = 1 };
enum dfs_layout { DFS_NHD = 0, DFS_HND = 1 };
/* curve.hpp:12 Ordering, same numeric values as the enum's declaration order */
enum dfs_ordering { DFS_RASTER = 0, DFS_HILBERT2D = 1, DFS_BLOCK3D = 2, DFS_HILBERT3D = 3 };

typedef struct dfs_handle dfs_handle;
typedef void* dfs_stream; /* cudaStream_t */

const char* dfs_last_error(void);
int dfs_abi_version(void);

/* ---- handle: workspaces + per-geometry permutation cache + mask cache ---- */
int dfs_handle_create(dfs_handle** out, int device);
int dfs_handle_destroy(dfs_handle* h);

/* ======================= K1: token ordering (curve.hpp) =================== */
/* curve.hpp:31-48 order_tokens / hilbert3d_order / ...: forward[i] = raster
 * index of the token at reordered position i. inv may be NULL; when given,
 * inv[forward[i]] = i (curve.hpp:53 invert_permutation). Device outputs. */
int dfs_order_tokens(int ordering, int64_t frames, int64_t height, int64_t width, uint32_t* fwd,
                     uint32_t* inv, dfs_stream stream);
/* curve.hpp:53 invert_permutation on device. */
int dfs_invert_permutation(const uint32_t* fwd, int64_t n, uint32_t* inv, dfs_stream stream);
/* curve.hpp:27 validate_permutation: *ok_host = 1 iff fwd is a bijection on [0,n).
 * Synchronises the stream. */
int dfs_validate_permutation(dfs_handle* h, const uint32_t* fwd, int64_t n, int* ok_host,
                             dfs_stream stream);

/* ================ K2/K6: permute / unpermute (curve.hpp:50,53) ============== */
/* dst row i <- src row idx[i] for every head (curve.cpp:166 apply_permutation),
 * converting layout src_layout -> dst_layout. dst may be NULL (read-only pass)
 * when pooled and/or nonfinite is given. With pooled != NULL also emits
 * the sub-block means of the DESTINATION rows (mask_builder.cpp:12 mean_pool,
 * zero-padded last group divided by pool) as fp32 [H, ceil(n/pool), d].
 * With nonfinite != NULL atomically ORs 1 into *nonfinite when any element is
 * NaN/Inf (attention.cpp:19-20 check). */
int dfs_permute_rows(const void* src, int src_layout, void* dst, int dst_layout, int dtype,
                     const uint32_t* idx, int64_t n, int64_t heads, int64_t d, float* pooled,
                     int64_t pool, int32_t* nonfinite, dfs_stream stream);
/* Element type conversion of `count` elements (DFS_F32 <-> DFS_BF16, round to
 * nearest even); ORs 1 into *nonfinite (optional, device) when a source element
 * is NaN/Inf. Used to feed fp32 Matrix inputs to the bf16 tensor-core kernels. */
int dfs_cast(const void* src, int src_dtype, void* dst, int dst_dtype, int64_t count, int32_t* nonfinite,
             dfs_stream stream);
/* Inverse direction: dst row idx[i] <- src row i (scatter), i.e.
 * apply_permutation(invert_permutation(p), x) without materialising inv. */
int dfs_unpermute_rows(const void* src, int src_layout, void* dst, int dst_layout, int dtype,
                       const uint32_t* idx, int64_t n, int64_t heads, int64_t d,
                       dfs_stream stream);

/* ================= K3/K4: hierarchical scoring + selection ================ */
/* mask_builder.cpp:30-80,115-117 block_scores from POOLED inputs:
 * pq [H, M*subs, d] fp32 (zero rows past ceil(n/Bs)), pk [H, ceil(n/Bs), d]
 * fp32; S [H, M, M] fp64, rows sum to subs. fp32-accurate tensor-core GEMM +
 * fp32 softmax with fp64 tile sums. */
int dfs_score_blocks(dfs_handle* h, const float* pq, const float* pk, int64_t heads, int64_t n,
                     int64_t d, int64_t block, int64_t sub_block, double* scores,
                     dfs_stream stream);
/* mask_builder.cpp:82-87 topk_count (host). */
int dfs_topk_count(double budget, int64_t m, int64_t* k);
/* mask_builder.cpp:91-113 topk_select on device, per (head, row): the K best
 * key blocks under (score desc, index asc), ascending. scores [H, M, M] fp64;
 * lut [H, M, K] int32 (may be NULL); bits [H, ceil(M*M/8)] BlockMask payloads
 * (may be NULL; zeroed by the call). Bit-exact with the reference given the
 * same scores. */
int dfs_topk_select(const double* scores, int64_t heads, int64_t m, int64_t k, int32_t* lut,
                    uint8_t* bits, dfs_stream stream);
/* BlockMask payloads [H][ceil(M*M/8)] -> CSR (blk_ptr [H*M+1], blk_idx cap
 * H*M*M). Returns DFS_E_INVALID (after a stream sync) if a row is empty
 * (attention.cpp:133-136). nnz_host may be NULL. */
int dfs_mask_bits_to_csr(dfs_handle* h, const uint8_t* bits, int64_t heads, int64_t m,
                         int32_t* blk_ptr, int32_t* blk_idx, int64_t* nnz_host,
                         dfs_stream stream);
/* Uniform-K LUT [H, M, K] -> CSR row pointers blk_ptr [H*M+1] (blk_idx = lut). */
int dfs_lut_row_ptr(int64_t heads, int64_t m, int64_t k, int32_t* blk_ptr, dfs_stream stream);

/* ===================== K5: block-sparse attention forward ================= */
/* attention.cpp:125-159 block_sparse_attention (and :95-103
 * full_attention_output with a full mask, nq != nk allowed). Per head h and
 * query block u the keys are the union of blocks blk_idx[blk_ptr[h*M+u] ..
 * blk_ptr[h*M+u+1]) clipped to nk (padded keys excluded); query rows >= nq are
 * not produced. q [.., nq, ..], k/v [.., nk, ..] in `in_layout`; o in
 * `out_layout`. When out_rows != NULL, output row i is written to row
 * out_rows[i] (fused unpermute: pass the forward permutation).
 * scale <= 0 means 1/sqrt(d). fp32 softmax and accumulation. */
typedef struct {
  const void* q;
  const void* k;
  const void* v;
  void* o;
  int dtype;      /* DFS_BF16 | DFS_F32 (f32 uses the generic kernel) */
  int in_layout;  /* DFS_HND | DFS_NHD */
  int out_layout; /* DFS_HND | DFS_NHD */
  int64_t heads;
  int64_t nq;
  int64_t nk;
  int64_t d;
  int64_t block; /* B, query and key block size */
  const int32_t* blk_ptr;
  const int32_t* blk_idx;
  const uint32_t* out_rows;
  float scale;
  int force_generic; /* 1: use the SIMT kernel even when the tcgen05 one applies */
  int64_t dv;        /* head dim of v / o; 0 = d (dv != d: fp32 kernel only) */
  /* Fused query reorder: when non-NULL, q is the [nq, H, d] raster-order (NHD)
   * tensor and logical query row i is its row in_rows[i], gathered by TMA inside
   * the kernel (curve.cpp:166 apply_permutation without a permuted copy of Q);
   * k and v keep `in_layout`. */
  const uint32_t* in_rows;
  /* ABI 2. Peer-scattered output (device pointer to a dfs_peer_table, or NULL): output
   * row i (after out_rows) is raster token t = out_rows[i], written to rank
   * t / n_local's [n_local, heads_total, dv] shard at row t % n_local, head
   * h0 + h — the reverse Ulysses all-to-all fused into the epilogue (tcgen05 K5 only). */
  const void* out_peers;
} dfs_attn_args;
int dfs_sparse_attn_fwd(dfs_handle* h, const dfs_attn_args* a, dfs_stream stream);

/* ======================= K7: mask cache + Alg.1 step ====================== */
/* scheduler.hpp:20-50 SparsitySchedule (host, identical rules). */
typedef struct {
  int total_steps;
  double warmup_fraction;
  const double* phase_budgets;
  int n_budgets;
  double phase_fraction;
  int update_interval;
} dfs_schedule;
/* budget_at: *budget = -1 for a dense step; DFS_E_RANGE outside [0,T). */
int dfs_schedule_budget_at(const dfs_schedule* s, int step, double* budget);
int dfs_schedule_is_update_step(const dfs_schedule* s, int step, int* is_update);
int dfs_schedule_info(const dfs_schedule* s, int* warmup_steps, int* phase_length);

/* scheduler.hpp:54-71 MaskCache, device resident, owned by the handle, keyed
 * by (layer, head). */
int dfs_mask_cache_clear(dfs_handle* h);
int dfs_mask_cache_contains(dfs_handle* h, int layer, int head, int* found);
/* Copies the cached mask of (layer, head) out as a BlockMask payload (device
 * pointer, ceil(M*M/8) bytes) and reports its last update step / block count. */
int dfs_mask_cache_get(dfs_handle* h, int layer, int head, uint8_t* bits, int* last_update_step,
                       int64_t* m, dfs_stream stream);
/* Stores a BlockMask payload (device pointer) for (layer, head) at `step`. */
int dfs_mask_cache_store(dfs_handle* h, int layer, int head, const uint8_t* bits, int64_t m,
                         int64_t block, int step, dfs_stream stream);
int dfs_mask_cache_size(dfs_handle* h, int64_t* n);
/* Geometry of the cached (layer, head) mask: block count m, block size and last
 * update step (any pointer may be NULL). DFS_E_INVALID when absent. */
int dfs_mask_cache_info(dfs_handle* h, int layer, int head, int64_t* m, int64_t* block, int* last_update_step);

/* Optional prologue fused into K2 (§8(f) row 1; PAPER.md:852 — the paper's end-to-end
 * runs use fused QK-norm / RoPE kernels): each (token, head) row of q and of k is
 * RMS-normalised over d, x * weight / sqrt(mean(x^2) + eps), then rotated by RoPE, in
 * the same pass that reorders and pools it — so the DiT's separate norm / rotary pass
 * over q and k (read + write of both tensors) disappears. The transformed rows are
 * rounded to bf16 and are what the step scores and attends. */
enum dfs_rope_layout {
  DFS_ROPE_NONE = 0,
  DFS_ROPE_INTERLEAVED = 1, /* pairs (2i, 2i+1) rotated by angle i (complex-multiply form) */
  DFS_ROPE_HALF = 2         /* pairs (i, i + d/2) (rotate_half form) */
};
typedef struct {
  const float* q_norm_weight; /* device [d] fp32, or NULL: q is not normalised */
  const float* k_norm_weight; /* device [d] fp32, or NULL */
  float eps;                  /* RMSNorm epsilon */
  int rope_layout;            /* dfs_rope_layout */
  const float* rope_cos;      /* device [N, d/2] fp32 by raster token (3D RoPE tables), or NULL */
  const float* rope_sin;      /* device [N, d/2] fp32 */
} dfs_qk_prologue;

/* The prologue alone: q (which = 0, q_norm_weight) or k (which = 1, k_norm_weight) bf16
 * [N, H, d] raster -> dst bf16, row i = transformed source row idx[i] (idx NULL: raster),
 * in dst_layout. */
int dfs_qk_prologue_apply(const dfs_qk_prologue* p, int which, const void* src, void* dst, int dst_layout,
                          const uint32_t* idx, int64_t n, int64_t heads, int64_t d, dfs_stream stream);

/* scheduler.cpp:91-135 run_step for ALL heads of one layer at once.
 * q, k, v, o: [N, H, d] bf16 raster-order activations (the DiT layout).
 * Dense steps (warmup or force_dense) run full attention in raster order;
 * sparse steps reorder (forward permutation `perm`, device u32[N]), build or
 * reuse the cached (layer, head) masks, attend, and scatter back to raster
 * order. Per-head stats go to the host arrays when non-NULL. */
typedef struct {
  const void* q;
  const void* k;
  const void* v;
  void* o;
  int64_t n;
  int64_t heads;
  int64_t d;
  const uint32_t* perm; /* device forward permutation; NULL = hilbert3d of dims */
  int64_t frames, height, width;
  int64_t block;
  int64_t sub_block;
  int layer;
  int step;
  int force_dense;
  /* Non-finite input is an error (attention.cpp:19-20), in the reference's order:
   * flags are ORed in the passes that read q/k/v anyway (K2, or a check pass on dense
   * / reuse steps); a non-finite q or k returns DFS_E_INVALID before anything is
   * scored or cached (build_mask -> attention_scores throws), a non-finite v after
   * the new masks are stored (block_sparse_attention throws after cache.store,
   * scheduler.cpp:113-122); no output is written in either case. `nonfinite`
   * optionally names the device flag for q/k (caller-zeroed); NULL = the handle's. */
  int32_t* nonfinite;
  /* outputs (host, optional) */
  int* dense_out;        /* 1 if the step ran dense */
  double* budget_out;    /* budget (1.0 when dense) */
  int* updated_out;      /* [H] mask_updated per head */
  double* sparsity_out;  /* [H] realized sparsity per head (metrics.cpp:39) */
  /* [H] host, optional: attention recall of each head's mask on sparse steps
   * (scheduler.cpp:129-131 record_recall), streamed without the N x N matrix, so
   * it is available past the reference's 4096-row cap (dfs_block_recall). */
  double* recall_out;
  /* ABI 2. dtype of q/k/v/o: DFS_BF16 (0, the performance path) or DFS_F32 (the
   * drop-in Matrix path: n <= DFS_COMPAT_MAX_ROWS runs fp64-arithmetic compatibility
   * kernels bit-identical to dfs::build_mask / block_sparse_attention; larger n pools
   * and scores from the fp32 values (fp32-accurate tcgen05 scorer) and attends in bf16
   * through K5, output converted back to fp32). */
  int dtype;
  int64_t dv; /* head dim of v / o; 0 = d (dv != d: DFS_F32 with n <= DFS_COMPAT_MAX_ROWS only) */
  const dfs_qk_prologue* prologue; /* host pointer or NULL; bf16 steps with d % 16 == 0 only */
} dfs_step_args;
int dfs_run_step(dfs_handle* h, const dfs_schedule* s, const dfs_step_args* a, dfs_stream stream);

/* ================ Ulysses: the all-to-all fused into K2 and K5 ================ */
/* a DiT that keeps q/k/v/o sequence-sharded ([N/P, H, d] per rank,
 * rank r holding raster tokens [r*N/P, (r+1)*N/P)) runs the step for its head
 * group [r*H/P, (r+1)*H/P) straight on its peers' shards over NVLink: K2 pulls the
 * token rows of its heads from every peer (P2P loads — the seq->head all-to-all
 * and its unpack are the gather's addressing) and K5's epilogue stores every output
 * row into the shard of the rank that owns the token (P2P stores — the head->seq
 * all-to-all and its pack). No exchange pass, no pack/unpack copies, no NCCL call on
 * the data path. Buffers are shared once per allocation with CUDA IPC. */
#define DFS_MAX_PEERS 16
typedef struct {
  unsigned char bytes[64]; /* cudaIpcMemHandle_t of the allocation that holds the buffer */
  int64_t offset;          /* byte offset of the buffer inside that allocation */
} dfs_peer_handle;
/* IPC handle of any device buffer (e.g. a sub-allocation of a caching allocator). */
int dfs_alltoall_export(const void* dev_ptr, dfs_peer_handle* out);
/* Maps a peer's buffer into this process (peer access enabled lazily over NVLink); an
 * allocation exported several times is mapped once and reference counted. */
int dfs_alltoall_import(const dfs_peer_handle* handle, void** dev_ptr);
/* Releases a pointer returned by dfs_alltoall_import. */
int dfs_alltoall_close(void* dev_ptr);
/* Device-resident table of the ranks' shard pointers (what K2/K5 index by token). */
typedef struct {
  const void* ptr[DFS_MAX_PEERS];
  int64_t n_local;     /* tokens per rank shard */
  int64_t heads_total; /* H of the [n_local, H, d] shards */
  int64_t h0;          /* first head of this rank's group */
} dfs_peer_table;
/* One Alg. 1 step (scheduler.cpp:91-135) for this rank's head group on
 * sequence-sharded bf16 activations. q/k/v[r] and o[r]: rank r's [n_local, H, d] shard
 * as mapped in THIS process (own shard = local pointer). Every rank calls it with the
 * same step; callers synchronise the ranks (barrier) before the step — peers' inputs
 * written — and after it — this rank's output rows written by the peers. Stats are
 * per local head. */
typedef struct {
  const void* q[DFS_MAX_PEERS];
  const void* k[DFS_MAX_PEERS];
  const void* v[DFS_MAX_PEERS];
  void* o[DFS_MAX_PEERS];
  int world;
  int rank;
  int64_t n_local;
  int64_t heads; /* H (all ranks); H % world == 0 */
  int64_t d;
  int64_t frames, height, width; /* token lattice, frames*height*width = world*n_local */
  int64_t block;
  int64_t sub_block;
  int layer;
  int step;
  int force_dense;
  int* dense_out;
  double* budget_out;
  int* updated_out;     /* [H / world] */
  double* sparsity_out; /* [H / world] */
} dfs_alltoall_step_args;
int dfs_alltoall_run_step(dfs_handle* h, const dfs_schedule* s, const dfs_alltoall_step_args* a, dfs_stream stream);

/* ============ Matrix-level companions used by the dfs:: drop-in shim =========== */
/* attention.cpp:105-123 attention_scores (and the pooled softmax inside
 * mask_builder.cpp:30-62 subblock_scores): row-softmax(q k^T * scale) with fp64
 * logits/exp/sum, fp32 probabilities. q [H, q_valid, d], k [H, k_valid, d] fp32
 * device; probs [H, q_rows, k_cols]. Rows >= q_valid are zero vectors (uniform
 * over the valid keys), columns >= k_valid are 0. scale <= 0 means 1/sqrt(d). */
int dfs_softmax_scores(const float* q, const float* k, int64_t heads, int64_t q_valid, int64_t q_rows,
                       int64_t k_valid, int64_t k_cols, int64_t d, double scale, float* probs,
                       dfs_stream stream);
/* mask_builder.cpp:64-80 aggregate_scores: S [H, mq, mk] fp64 tile sums of
 * probs [H, mq*subs, mk*subs]. */
int dfs_aggregate_scores(const float* probs, int64_t heads, int64_t mq, int64_t mk, int64_t subs,
                         double* scores, dfs_stream stream);
/* mask_builder.cpp:91-102 top_indices for `rows` independent rows of length n:
 * out [rows, k] ascending indices of the k best (value desc, index asc). */
int dfs_top_indices(const double* values, int64_t rows, int64_t n, int64_t k, int32_t* out,
                    dfs_stream stream);
/* attention.cpp:161-173 masked_scores (scores [rows, cols] fp32, BlockMask
 * payload bits of an m x m mask with block size `block`). */
int dfs_masked_scores(const float* scores, int64_t rows, int64_t cols, const uint8_t* bits, int64_t m,
                      int64_t block, float* out, dfs_stream stream);
/* attention.cpp:19-20 (non-finite input is an error): *nonfinite_host = 1 when
 * any of `count` elements (dtype) is NaN/Inf. Synchronises the stream. */
int dfs_check_finite(const void* x, int64_t count, int dtype, int* nonfinite_host, dfs_stream stream);
/* attention.cpp:175-190 attention_recall -> *recall_host (synchronises). */
int dfs_attention_recall(const float* scores, int64_t rows, int64_t cols, const uint8_t* bits, int64_t m,
                         int64_t block, double* recall_host, dfs_stream stream);

/* attention.cpp:175-190 attention_recall(attention_scores(q, k), mask) for H
 * heads at any N: sum |A o M| / sum |A| with A = row-softmax(q k^T / sqrt(d)),
 * computed by streaming every key block through the tensor cores (no N x N
 * storage). q, k: bf16 in `layout` (q_rows != NULL: q is raster NHD and logical
 * row i is its row q_rows[i], as dfs_attn_args.in_rows); the mask is a CSR over
 * (head, query block) with B = 128. recall_host [H] (synchronises). d in {64,128}. */
int dfs_block_recall(dfs_handle* h, const void* q, const void* k, int layout, const uint32_t* q_rows,
                     int64_t heads, int64_t n, int64_t d, const int32_t* blk_ptr, const int32_t* blk_idx,
                     double* recall_host, dfs_stream stream);

/* Per-handle kernel selection (A/B tests): route scoring / attention through
 * the geometry-generic kernels even where the tcgen05 ones apply. */
enum dfs_option { DFS_OPT_GENERIC_SCORE = 1, DFS_OPT_GENERIC_ATTN = 2 };
int dfs_handle_set_option(dfs_handle* h, int option, int value);

/* Device mem introspection for the bench (bytes of workspace held). */
int dfs_handle_workspace_bytes(dfs_handle* h, int64_t* bytes);

#ifdef __cplusplus
}
#endif
#endif /* DFS_GPU_H */
