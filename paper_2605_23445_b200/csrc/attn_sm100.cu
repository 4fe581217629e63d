// attn_sm100.cu — K5: block-sparse FlashAttention forward on tcgen05 / TMEM / TMA.
//
// block_sparse_attention (attention.cpp:125-159) for B = 128, d in {64, 128},
// bf16 I/O, fp32 softmax and accumulation. Persistent CTAs (one per SM) walk
// (head, query block) tiles; a tile visits ONLY the key blocks of its CSR list
// (top-K LUT, or every block for dense / cross attention), so masked blocks
// cost neither bytes nor FLOPs.
//
// Warp roles (192 threads):
//   warp 0      TMA producer: Q tile, then K_0, K_1, V_0, K_2, V_1, ... into a
//               ring of kStages smem slots (SWIZZLE_128B boxes of 128 x 64).
//   warp 1      MMA issuer (one thread): S = Q K^T into a double-buffered TMEM
//               S (so QK of block j+1 overlaps the softmax of block j), then
//               O += P V with O resident in TMEM.
//   warps 2-5   softmax + correction + epilogue: thread r owns query row r
//               (TMEM lane r). Online softmax in the log2 domain; O is rescaled
//               in TMEM only when the running max grows by > 2^8 (the final
//               normalisation uses the same stale max for O and l, so this is
//               exact). P goes to smem in the UMMA K-major SW128 layout. The
//               epilogue writes each output row straight to its raster position
//               out_rows[i] — the unpermute (scheduler.cpp:134) is fused here.
// Padded keys of the last partial block get -inf logits; padded query rows
// are computed on TMA zero-fill and never stored (attention.cpp:146-152).
#include <cuda.h>

#include "common.cuh"
#include "sm100.cuh"

namespace dfsgpu {

namespace {

using namespace sm100;

constexpr int kBM = 128;         // query rows per tile (= TMEM lanes)
constexpr int kBN = 128;         // keys per block
constexpr int kThreads = 192;
constexpr uint32_t kTmemCols = 512;
constexpr float kRescaleThreshold = 8.0f;  // log2 units

template <int D>
struct Cfg {
  static constexpr int kChunks = D / 64;                 // 128-byte swizzle chunks per row
  static constexpr int kTileBytes = kBM * D * 2;         // one Q / K / V tile
  static constexpr int kChunkBytes = kBM * 128;          // one 128 x 64 bf16 TMA box
  static constexpr int kStages = D == 64 ? 8 : 4;
  static constexpr int kPBytes = kBM * kBN * 2;
  static constexpr int kQOff = 0;
  static constexpr int kRingOff = kQOff + kTileBytes;
  static constexpr int kPOff = kRingOff + kStages * kTileBytes;
  static constexpr int kBarOff = kPOff + kPBytes;
  static constexpr int kSmem = kBarOff + 256 + 1024;     // barriers + alignment slack
  static constexpr uint32_t kIdescQK = idesc_bf16_f32(kBM, kBN, false, false);
  static constexpr uint32_t kIdescPV = idesc_bf16_f32(kBM, D, false, true);
  static constexpr uint32_t kOCol = 256;                  // TMEM: S0 [0,128) S1 [128,256) O [256,256+D)
};

struct Params {
  int64_t heads, nq, nk, mq, mk;
  const int32_t* blk_ptr;  // NULL = dense
  const int32_t* blk_idx;
  const uint32_t* out_rows;
  __nv_bfloat16* out;
  int out_layout;
  int in_nhd;  // 1: inputs are [N, H, d] (tensor-map coordinates (col, head, row))
  float scale_log2;
  int64_t tiles;
};

struct Bars {
  uint64_t q_full, q_empty;
  uint64_t s_full[2], s_free[2];
  uint64_t p_full, o_done;
  uint64_t kv_full[8], kv_empty[8];
  uint32_t tmem_base;
};

__device__ __forceinline__ void tile_list(const Params& p, int64_t tile, int64_t& h, int64_t& u, int32_t& beg,
                                          int32_t& cnt) {
  h = tile / p.mq;
  u = tile % p.mq;
  if (p.blk_ptr) {
    beg = p.blk_ptr[tile];
    cnt = p.blk_ptr[tile + 1] - beg;
  } else {
    beg = 0;
    cnt = int32_t(p.mk);
  }
}

__device__ __forceinline__ int32_t block_at(const Params& p, int32_t beg, int32_t j) {
  return p.blk_ptr ? p.blk_idx[beg + j] : j;
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    attn_sm100_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                      const __grid_constant__ CUtensorMap tm_v, const Params p) {
  using C = Cfg<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem + C::kQOff;
  uint8_t* sRing = smem + C::kRingOff;
  uint8_t* sP = smem + C::kPOff;
  Bars* bars = reinterpret_cast<Bars*>(smem + C::kBarOff);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    mbar_init(&bars->q_full, 1);
    mbar_init(&bars->q_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars->s_full[i], 1);
      mbar_init(&bars->s_free[i], 128);
    }
    mbar_init(&bars->p_full, 128);
    mbar_init(&bars->o_done, 1);
    for (int i = 0; i < C::kStages; ++i) {
      mbar_init(&bars->kv_full[i], 1);
      mbar_init(&bars->kv_empty[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tm_q);
    prefetch_tmap(&tm_k);
    prefetch_tmap(&tm_v);
  }
  if (warp == 1) tmem_alloc<kTmemCols>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  if (warp == 0) {
    // ================================ TMA producer ==============================
    if (lane == 0) {
      uint32_t q_phase = 0, ring = 0;
      auto load_tile = [&](const CUtensorMap* map, int64_t h, int64_t row0) {
        const uint32_t slot = ring % C::kStages;
        const uint32_t use = ring / C::kStages;
        mbar_wait(&bars->kv_empty[slot], (use & 1) ^ 1);
        mbar_expect_tx(&bars->kv_full[slot], C::kTileBytes);
        uint8_t* dst = sRing + slot * C::kTileBytes;
#pragma unroll
        for (int c = 0; c < C::kChunks; ++c)
          tma_load_3d(dst + c * C::kChunkBytes, map, &bars->kv_full[slot], c * 64, p.in_nhd ? int(h) : int(row0),
                      p.in_nhd ? int(row0) : int(h));
        ++ring;
      };
      for (int64_t tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
        int64_t h, u;
        int32_t beg, cnt;
        tile_list(p, tile, h, u, beg, cnt);
        mbar_wait(&bars->q_empty, q_phase ^ 1);
        q_phase ^= 1;
        mbar_expect_tx(&bars->q_full, C::kTileBytes);
#pragma unroll
        for (int c = 0; c < C::kChunks; ++c)
          tma_load_3d(sQ + c * C::kChunkBytes, &tm_q, &bars->q_full, c * 64, p.in_nhd ? int(h) : int(u * kBM),
                      p.in_nhd ? int(u * kBM) : int(h));
        // consumption order of the MMA warp: K0, K1, V0, K2, V1, ..., V_{n-1}
        load_tile(&tm_k, h, int64_t(block_at(p, beg, 0)) * kBN);
        for (int32_t j = 1; j < cnt; ++j) {
          load_tile(&tm_k, h, int64_t(block_at(p, beg, j)) * kBN);
          load_tile(&tm_v, h, int64_t(block_at(p, beg, j - 1)) * kBN);
        }
        load_tile(&tm_v, h, int64_t(block_at(p, beg, cnt - 1)) * kBN);
      }
    }
  } else if (warp == 1) {
    // ================================ MMA issuer ================================
    if (lane == 0) {
      uint32_t q_phase = 0, ring = 0, s_iter = 0, pv_iter = 0;
      const uint32_t q_base = smem_u32(sQ), p_base = smem_u32(sP);
      auto next_slot = [&](uint32_t& slot) {
        slot = ring % C::kStages;
        mbar_wait(&bars->kv_full[slot], (ring / C::kStages) & 1);
        ++ring;
      };
      auto issue_qk = [&]() {
        uint32_t slot;
        next_slot(slot);
        const uint32_t sb = s_iter & 1;
        mbar_wait(&bars->s_free[sb], ((s_iter >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t k_base = smem_u32(sRing + slot * C::kTileBytes);
#pragma unroll
        for (int s = 0; s < D / 16; ++s) {
          const uint32_t off = (s >> 2) * C::kChunkBytes + (s & 3) * 32;
          umma_f16(tmem + sb * 128, smem_desc_sw128(q_base + off, 16, 1024), smem_desc_sw128(k_base + off, 16, 1024),
                   C::kIdescQK, s > 0);
        }
        umma_commit(&bars->kv_empty[slot]);
        umma_commit(&bars->s_full[sb]);
        ++s_iter;
      };
      auto issue_pv = [&](bool first) {
        uint32_t slot;
        next_slot(slot);
        mbar_wait(&bars->p_full, pv_iter & 1);
        tc_fence_after();
        const uint32_t v_base = smem_u32(sRing + slot * C::kTileBytes);
#pragma unroll
        for (int s = 0; s < kBN / 16; ++s) {
          const uint32_t a_off = (s >> 2) * (kBM * 128) + (s & 3) * 32;  // P: K-major, 64-key chunks
          const uint32_t b_off = s * 16 * 128;                             // V: MN-major, 16 keys per step
          umma_f16(tmem + C::kOCol, smem_desc_sw128(p_base + a_off, 16, 1024),
                   smem_desc_sw128(v_base + b_off, C::kChunkBytes, 1024), C::kIdescPV, (!first || s > 0) ? 1u : 0u);
        }
        umma_commit(&bars->kv_empty[slot]);
        umma_commit(&bars->o_done);
        ++pv_iter;
      };
      for (int64_t tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
        int64_t h, u;
        int32_t beg, cnt;
        tile_list(p, tile, h, u, beg, cnt);
        mbar_wait(&bars->q_full, q_phase);
        q_phase ^= 1;
        issue_qk();
        if (cnt == 1) umma_commit(&bars->q_empty);
        for (int32_t j = 1; j < cnt; ++j) {
          issue_qk();
          if (j == cnt - 1) umma_commit(&bars->q_empty);
          issue_pv(j == 1);
        }
        issue_pv(cnt == 1);
      }
    }
  } else {
    // ============================ softmax / epilogue ============================
    const int r = (warp & 3) * 32 + lane;              // query row within the tile == TMEM lane
    const uint32_t lane_addr = uint32_t((warp & 3) * 32) << 16;
    uint32_t s_iter = 0, o_phase = 0;
    uint8_t* prow = sP + r * 128;                      // row r inside each 64-key chunk
    for (int64_t tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
      int64_t h, u;
      int32_t beg, cnt;
      tile_list(p, tile, h, u, beg, cnt);
      float m = -INFINITY, l = 0.f;
      for (int32_t j = 0; j < cnt; ++j) {
        const uint32_t sb = s_iter & 1;
        mbar_wait(&bars->s_full[sb], (s_iter >> 1) & 1);
        tc_fence_after();
        uint32_t sv[4][32];
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld32(tmem + lane_addr + sb * 128 + c * 32, sv[c]);
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(&bars->s_free[sb]);
        ++s_iter;
        // padded keys of a partial last block (attention.cpp:146-152)
        const int64_t vb = block_at(p, beg, j);
        const int valid = int(min(int64_t(kBN), p.nk - vb * kBN));
        float mx = -INFINITY;
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            float x = __uint_as_float(sv[c][i]);
            if (c * 32 + i >= valid) x = -INFINITY;
            sv[c][i] = __float_as_uint(x);
            mx = fmaxf(mx, x);
          }
        const float m_new = fmaxf(m, mx * p.scale_log2);
        if (j > 0) {
          mbar_wait(&bars->o_done, o_phase);  // PV_{j-1} complete: P buffer free, O stable
          o_phase ^= 1;
          tc_fence_after();
        }
        // tcgen05.ld/st are warp-collective (.sync.aligned): the rescale decision
        // must be warp-uniform, so one lagging row rescales its whole warp
        if (j == 0) {
          m = m_new;
        } else if (__any_sync(0xffffffffu, m_new - m > kRescaleThreshold)) {
          const float alpha = ex2(m - m_new);
          l *= alpha;
          m = m_new;
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            uint32_t ov[32];
            tmem_ld32(tmem + lane_addr + C::kOCol + c * 32, ov);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
            tmem_st32(tmem + lane_addr + C::kOCol + c * 32, ov);
          }
          tmem_wait_st();
        }
        const float neg_m = -m;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float p0 = ex2(fmaf(__uint_as_float(sv[c][2 * i]), p.scale_log2, neg_m));
            const float p1 = ex2(fmaf(__uint_as_float(sv[c][2 * i + 1]), p.scale_log2, neg_m));
            l += p0 + p1;
            pk[i] = pack_bf16(p0, p1);
          }
          // keys [32c, 32c+32): chunk c/2, 16-byte units 4*(c&1) .. +3, swizzled by row
          uint8_t* base = prow + (c >> 1) * (kBM * 128);
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            const int unit = ((c & 1) * 4 + q4) ^ (r & 7);
            *reinterpret_cast<uint4*>(base + unit * 16) =
                make_uint4(pk[4 * q4], pk[4 * q4 + 1], pk[4 * q4 + 2], pk[4 * q4 + 3]);
          }
        }
        fence_proxy_async_smem();
        tc_fence_before();
        mbar_arrive(&bars->p_full);
      }
      // epilogue: wait for the last PV, normalise, scatter the row to its raster slot
      mbar_wait(&bars->o_done, o_phase);
      o_phase ^= 1;
      tc_fence_after();
      const int64_t i = u * kBM + r;
      const float inv_l = 1.f / l;
      uint32_t ov[D / 32][32];
#pragma unroll
      for (int c = 0; c < D / 32; ++c) tmem_ld32(tmem + lane_addr + C::kOCol + c * 32, ov[c]);
      tmem_wait_ld();
      tc_fence_before();
      if (i < p.nq) {
        const int64_t orow = p.out_rows ? int64_t(p.out_rows[i]) : i;
        __nv_bfloat16* dst = p.out + row_offset(p.out_layout, p.nq, p.heads, D, h, orow);
#pragma unroll
        for (int c = 0; c < D / 32; ++c)
#pragma unroll
          for (int q8 = 0; q8 < 4; ++q8) {
            uint4 w;
            w.x = pack_bf16(__uint_as_float(ov[c][8 * q8 + 0]) * inv_l, __uint_as_float(ov[c][8 * q8 + 1]) * inv_l);
            w.y = pack_bf16(__uint_as_float(ov[c][8 * q8 + 2]) * inv_l, __uint_as_float(ov[c][8 * q8 + 3]) * inv_l);
            w.z = pack_bf16(__uint_as_float(ov[c][8 * q8 + 4]) * inv_l, __uint_as_float(ov[c][8 * q8 + 5]) * inv_l);
            w.w = pack_bf16(__uint_as_float(ov[c][8 * q8 + 6]) * inv_l, __uint_as_float(ov[c][8 * q8 + 7]) * inv_l);
            *reinterpret_cast<uint4*>(dst + c * 32 + q8 * 8) = w;
          }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<kTmemCols>(tmem);
}

// ---- host ------------------------------------------------------------------------

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn get_encode() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(ptr);
  }
  return fn;
}

// 3D map over a token tensor so that box (64 cols, 128 rows, 1 head) is one
// SWIZZLE_128B operand chunk; rows past n are zero-filled.
int make_map(CUtensorMap* map, const void* base, int layout, int64_t n, int64_t heads, int64_t d) {
  EncodeFn enc = get_encode();
  if (!enc) return fail(DFS_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3], strides[2];
  cuuint32_t box[3], estr[3] = {1, 1, 1};
  if (layout == DFS_HND) {  // [H, N, d]: dims (d, N, H)
    dims[0] = cuuint64_t(d);
    dims[1] = cuuint64_t(n);
    dims[2] = cuuint64_t(heads);
    strides[0] = cuuint64_t(d) * 2;
    strides[1] = cuuint64_t(n) * cuuint64_t(d) * 2;
    box[0] = 64;
    box[1] = 128;
    box[2] = 1;
  } else {  // [N, H, d]: dims (d, H, N), box (64, 1, 128)
    dims[0] = cuuint64_t(d);
    dims[1] = cuuint64_t(heads);
    dims[2] = cuuint64_t(n);
    strides[0] = cuuint64_t(d) * 2;
    strides[1] = cuuint64_t(heads) * cuuint64_t(d) * 2;
    box[0] = 64;
    box[1] = 1;
    box[2] = 128;
  }
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DFS_E_CUDA, "cuTensorMapEncodeTiled failed");
  return DFS_OK;
}

template <int D>
int launch(const dfs_attn_args& a, float scale, cudaStream_t stream, int layout_hint) {
  using C = Cfg<D>;
  CUtensorMap mq, mk, mv;
  int rc;
  if ((rc = make_map(&mq, a.q, a.in_layout, a.nq, a.heads, D))) return rc;
  if ((rc = make_map(&mk, a.k, a.in_layout, a.nk, a.heads, D))) return rc;
  if ((rc = make_map(&mv, a.v, a.in_layout, a.nk, a.heads, D))) return rc;
  (void)layout_hint;
  Params p;
  p.heads = a.heads;
  p.nq = a.nq;
  p.nk = a.nk;
  p.mq = ceil_div(a.nq, kBM);
  p.mk = ceil_div(a.nk, kBN);
  p.blk_ptr = a.blk_ptr;
  p.blk_idx = a.blk_idx;
  p.out_rows = a.out_rows;
  p.out = static_cast<__nv_bfloat16*>(a.o);
  p.out_layout = a.out_layout;
  p.in_nhd = a.in_layout == DFS_NHD;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.tiles = p.mq * a.heads;
  static bool attr_set = false;
  if (!attr_set) {
    DFS_CUDA_CHECK(cudaFuncSetAttribute(attn_sm100_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
    attr_set = true;
  }
  const int64_t grid = p.tiles < kNumSMs ? p.tiles : kNumSMs;
  attn_sm100_kernel<D><<<unsigned(grid), kThreads, C::kSmem, stream>>>(mq, mk, mv, p);
  DFS_LAUNCH_CHECK("attn_sm100");
  return DFS_OK;
}

}  // namespace

// [H, rows, d] fp16 operand map for the scorer (score_sm100.cu): box 64 x 128 x 1, SW128
int make_map_f16(CUtensorMap* map, const void* base, int64_t rows, int64_t heads, int64_t d) {
  EncodeFn enc = get_encode();
  if (!enc) return fail(DFS_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {cuuint64_t(d), cuuint64_t(rows), cuuint64_t(heads)};
  cuuint64_t strides[2] = {cuuint64_t(d) * 2, cuuint64_t(rows) * cuuint64_t(d) * 2};
  cuuint32_t box[3] = {64, 128, 1}, estr[3] = {1, 1, 1};
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DFS_E_CUDA, "cuTensorMapEncodeTiled (f16) failed");
  return DFS_OK;
}

bool attn_sm100_supports(const dfs_attn_args& a) {
  if (a.dtype != DFS_BF16 || a.block != 128 || (a.d != 64 && a.d != 128)) return false;
  const void* ptrs[4] = {a.q, a.k, a.v, a.o};
  for (const void* ptr : ptrs)
    if (reinterpret_cast<uintptr_t>(ptr) & 15) return false;
  if (a.nq >= (int64_t(1) << 31) || a.nk >= (int64_t(1) << 31)) return false;
  return true;
}

int sparse_attn_sm100(const dfs_attn_args& a, float scale, cudaStream_t stream) {
  if (a.d == 128) return launch<128>(a, scale, stream, 0);
  if (a.d == 64) return launch<64>(a, scale, stream, 0);
  return fail(DFS_E_UNSUPPORTED, "attn_sm100: d must be 64 or 128");
}

}  // namespace dfsgpu
