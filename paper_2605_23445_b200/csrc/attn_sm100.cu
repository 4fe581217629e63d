// attn_sm100.cu — K5: block-sparse FlashAttention forward on tcgen05 / TMEM / TMA.
//
// block_sparse_attention (attention.cpp:125-159) for B = 128, d in {64, 128},
// bf16 I/O, fp32 softmax and accumulation. Persistent CTAs (one per SM) walk
// (head, query block) tiles; a tile visits ONLY the key blocks of its CSR list
// (top-K LUT, or every block for dense / cross attention), so masked blocks
// cost neither bytes nor FLOPs.
//
// Warp roles (320 threads):
//   warp 0      TMA producer: Q tile, then K_0, K_1, V_0, K_2, V_1, ... into a
//               ring of kStages smem slots (SWIZZLE_128B boxes of 128 x 64).
//   warp 1      MMA issuer (one thread): S_j = Q K_j^T into a double-buffered
//               TMEM S (QK of block j+1 overlaps the softmax of block j), then
//               O += P_j V_j with P_j read straight from TMEM (it overwrites
//               S_j in place, bf16) and O resident in TMEM.
//   warps 2-9   softmax / correction / epilogue, two warpgroups that split the
//               128 key columns of every query row (TMEM lane): each thread
//               handles 64 logits per block, the row max is exchanged through
//               shared memory with one named barrier per block. Online softmax
//               in the log2 domain; O is rescaled in TMEM only when the
//               running max grows by > 2^8 (the final normalisation uses the
//               same stale max for O and l, so this is exact). The epilogue
//               writes each output row straight to its raster position
//               out_rows[i] — the unpermute (scheduler.cpp:134) is fused here.
// Padded keys of the last partial block get -inf logits; padded query rows
// are computed on TMA zero-fill and never stored (attention.cpp:146-152).
#include <cuda.h>

#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "sm100.cuh"

namespace dfsgpu {

namespace {

using namespace sm100;

constexpr int kBM = 128;         // query rows per tile (= TMEM lanes)
constexpr int kBN = 128;         // keys per block
constexpr int kWG = 4;                     // softmax warpgroups (32 key columns each)
constexpr int kSoftmaxThreads = 128 * kWG;
constexpr int kThreads = 64 + kSoftmaxThreads;
constexpr uint32_t kTmemCols = 512;
constexpr float kRescaleThreshold = 8.0f;  // log2 units
constexpr uint32_t kBarMax = 1;            // named barrier ids (0 = __syncthreads)

template <int D>
struct Cfg {
  static constexpr int kChunks = D / 64;                 // 128-byte swizzle chunks per row
  static constexpr int kTileBytes = kBM * D * 2;         // one Q / K / V tile
  static constexpr int kChunkBytes = kBM * 128;          // one 128 x 64 bf16 TMA box
  static constexpr int kStages = D == 64 ? 12 : 5;
  static constexpr int kQOff = 0;
  static constexpr int kRingOff = kQOff + kTileBytes;
  static constexpr int kRedOff = kRingOff + kStages * kTileBytes;   // float max[2][kWG][128], sum[kWG][128]
  static constexpr int kBarOff = kRedOff + 3 * kWG * kBM * 4;
  static constexpr int kSmem = kBarOff + 512 + 1024;     // barriers + alignment slack
  static constexpr uint32_t kIdescQK = idesc_bf16_f32(kBM, kBN, false, false);
  static constexpr uint32_t kIdescPV = idesc_bf16_f32(kBM, D, false, true);
  static constexpr int kSBufs = 3;         // TMEM: S0/P0 [0,128) S1/P1 [128,256) S2/P2 [256,384) O [384,384+D)
  static constexpr uint32_t kOCol = 384;
  static constexpr int kOColsPerWG = D / kWG;
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
  unsigned long long* trace;  // debug timeline (DFS_ATTN_TRACE), NULL in production
  int exp_mode;               // debug (DFS_ATTN_EXP): 1 skip QK, 2 skip PV, 4 skip softmax math
  int64_t tiles;
};

struct Bars {
  uint64_t q_full, q_empty;
  uint64_t s_full[3];
  uint64_t p_full, o_done;
  uint64_t kv_full[12], kv_empty[12];
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

__device__ __forceinline__ void trace(const Params& p, int ev, uint32_t idx) {
  if (p.trace && blockIdx.x == 0 && idx < 256) p.trace[ev * 256 + idx] = clock64();
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
  float* red = reinterpret_cast<float*>(smem + C::kRedOff);  // [parity][wg][row]
  Bars* bars = reinterpret_cast<Bars*>(smem + C::kBarOff);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    mbar_init(&bars->q_full, 1);
    mbar_init(&bars->q_empty, 1);
    for (int i = 0; i < 3; ++i) mbar_init(&bars->s_full[i], 1);
    mbar_init(&bars->p_full, kSoftmaxThreads);
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
        // consumption order of the MMA warp (QK runs two blocks ahead of PV):
        // K0, K1, K2, V0, K3, V1, ..., K_{n-1}, V_{n-3}, V_{n-2}, V_{n-1}
        load_tile(&tm_k, h, int64_t(block_at(p, beg, 0)) * kBN);
        if (cnt > 1) load_tile(&tm_k, h, int64_t(block_at(p, beg, 1)) * kBN);
        for (int32_t j = 0; j < cnt; ++j) {
          if (j + 2 < cnt) load_tile(&tm_k, h, int64_t(block_at(p, beg, j + 2)) * kBN);
          load_tile(&tm_v, h, int64_t(block_at(p, beg, j)) * kBN);
        }
      }
    }
  } else if (warp == 1) {
    // ================================ MMA issuer ================================
    if (lane == 0) {
      uint32_t q_phase = 0, ring = 0, s_iter = 0, pv_iter = 0;
      const uint32_t q_base = smem_u32(sQ);
      auto next_slot = [&](uint32_t& slot) {
        slot = ring % C::kStages;
        trace(p, 0, ring);
        mbar_wait(&bars->kv_full[slot], (ring / C::kStages) & 1);
        trace(p, 1, ring);
        ++ring;
      };
      // Three S/P buffers: QK_{j+2} overwrites S[(j+2)%3], whose P_{j-1} was consumed by
      // PV_{j-1}, issued earlier into the in-order tcgen05 pipe — so QK never waits for the
      // softmax, and the tensor pipe always has the next QK queued behind each PV.
      auto issue_qk = [&]() {
        uint32_t slot;
        next_slot(slot);
        const uint32_t sb = s_iter % C::kSBufs;
        tc_fence_after();
        const uint32_t k_base = smem_u32(sRing + slot * C::kTileBytes);
#pragma unroll
        for (int s = 0; s < D / 16; ++s) {
          const uint32_t off = (s >> 2) * C::kChunkBytes + (s & 3) * 32;
          if (!(p.exp_mode & 1))
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
        trace(p, 2, pv_iter);
        mbar_wait(&bars->p_full, pv_iter & 1);
        trace(p, 3, pv_iter);
        tc_fence_after();
        const uint32_t v_base = smem_u32(sRing + slot * C::kTileBytes);
        const uint32_t p_tmem = tmem + (pv_iter % C::kSBufs) * 128;  // P_j aliases S_j (bf16 pairs)
#pragma unroll
        for (int s = 0; s < kBN / 16; ++s)
          if (!(p.exp_mode & 2))
            umma_f16_ts(tmem + C::kOCol, p_tmem + s * 8, smem_desc_sw128(v_base + s * 16 * 128, C::kChunkBytes, 1024),
                        C::kIdescPV, (!first || s > 0) ? 1u : 0u);
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
        if (cnt > 1) issue_qk();
        if (cnt <= 2) umma_commit(&bars->q_empty);  // Q smem free once the last QK read it
        for (int32_t j = 0; j < cnt; ++j) {
          if (j + 2 < cnt) {
            issue_qk();
            if (j + 3 == cnt) umma_commit(&bars->q_empty);
          }
          issue_pv(j == 0);
        }
      }
    }
  } else {
    // ============================ softmax / epilogue ============================
    // kWG warpgroups split the 128 key columns of each block (32 per group); a thread
    // owns one query row (TMEM lane) of its 32-column slice.
    const int wg = (warp - 2) >> 2;                    // key columns [32*wg, 32*wg + 32)
    const int r = (warp & 3) * 32 + lane;              // query row within the tile == TMEM lane
    const uint32_t lane_addr = uint32_t((warp & 3) * 32) << 16;
    uint32_t s_iter = 0, o_phase = 0;
    float* red_max = red;                              // [parity][kWG][kBM]
    float* red_sum = red + 2 * kWG * kBM;              // [kWG][kBM]
    for (int64_t tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
      int64_t h, u;
      int32_t beg, cnt;
      tile_list(p, tile, h, u, beg, cnt);
      float m = -INFINITY;
      uint64_t lsum[2] = {0, 0};  // packed fp32x2 partial row sums (2 independent chains)
      int32_t vb_next = block_at(p, beg, 0);
      for (int32_t j = 0; j < cnt; ++j) {
        const int32_t vb = vb_next;
        if (j + 1 < cnt) vb_next = block_at(p, beg, j + 1);  // prefetch: keeps the LUT load off the critical path
        const uint32_t sb = s_iter % C::kSBufs;
        const uint32_t s_phase = (s_iter / C::kSBufs) & 1;
        float* red_par = red_max + (s_iter & 1) * kWG * kBM;
        const bool tr = (threadIdx.x == 64 || threadIdx.x == 192);
        if (tr) trace(p, 4 + (wg & 1) * 4, s_iter);
        mbar_wait(&bars->s_full[sb], s_phase);
        if (tr) trace(p, 5 + (wg & 1) * 4, s_iter);
        tc_fence_after();
        const uint32_t s_addr = tmem + lane_addr + sb * 128 + wg * 32;
        if (p.exp_mode & 4) {  // debug: S -> P plumbing only
          ++s_iter;
          if (j > 0) {
            mbar_wait(&bars->o_done, o_phase);
            o_phase ^= 1;
          }
          tc_fence_before();
          mbar_arrive(&bars->p_full);
          continue;
        }
        uint32_t sv[32];
        tmem_ld32(s_addr, sv);
        tmem_wait_ld();
        ++s_iter;
        // padded keys of a partial last block (attention.cpp:146-152); warp-uniform branch
        const int valid = int(min(int64_t(kBN), p.nk - int64_t(vb) * kBN)) - wg * 32;
        if (valid < 32) {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (i >= valid) sv[i] = __float_as_uint(-INFINITY);
        }
        float mq[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int i = 0; i < 32; ++i) mq[i & 3] = fmaxf(mq[i & 3], __uint_as_float(sv[i]));
        float mx = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3]));
        red_par[wg * kBM + r] = mx;
        named_bar_sync(kBarMax, kSoftmaxThreads);      // every slice loaded S and published its max
        if (tr) trace(p, 6 + (wg & 1) * 4, s_iter - 1);
#pragma unroll
        for (int w = 0; w < kWG; ++w) mx = fmaxf(mx, red_par[w * kBM + r]);
        const float m_new = fmaxf(m, mx * p.scale_log2);
        bool waited = false;
        // tcgen05.ld/st are warp-collective: the rescale decision is warp-uniform
        // (the partner warps cover the same rows, so they decide identically)
        if (j == 0) {
          m = m_new;
        } else if (__any_sync(0xffffffffu, m_new - m > kRescaleThreshold)) {
          mbar_wait(&bars->o_done, o_phase);            // PV_{j-1} complete: O stable
          o_phase ^= 1;
          waited = true;
          tc_fence_after();
          const float alpha = ex2(m - m_new);
          const uint64_t a2 = f2_pack(alpha, alpha);
          lsum[0] = f2_mul(lsum[0], a2);
          lsum[1] = f2_mul(lsum[1], a2);
          m = m_new;
          const uint32_t o_addr = tmem + lane_addr + C::kOCol + wg * C::kOColsPerWG;
          if constexpr (C::kOColsPerWG == 32) {
            uint32_t ov[32];
            tmem_ld32(o_addr, ov);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
            tmem_st32(o_addr, ov);
          } else {
            uint32_t ov[16];
            tmem_ld16(o_addr, ov);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
            tmem_st16(o_addr, ov);
          }
        }
        // p = 2^(s*scale - m): 3 of every 4 pairs on MUFU, 1 on the FMA pipe (balances the pipes)
        const uint64_t sc2 = f2_pack(p.scale_log2, p.scale_log2), nm2 = f2_pack(-m, -m);
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          float x0, x1;
          f2_unpack(f2_fma(f2_pack(__uint_as_float(sv[2 * i]), __uint_as_float(sv[2 * i + 1])), sc2, nm2), x0, x1);
          float p0, p1;
          if ((i & 3) == 3) {
            p0 = ex2_poly(x0);
            p1 = ex2_poly(x1);
          } else {
            p0 = ex2(x0);
            p1 = ex2(x1);
          }
          lsum[i & 1] = f2_add(lsum[i & 1], f2_pack(p0, p1));
          pk[i] = pack_bf16(p0, p1);
        }
        // P_j (bf16 pairs) over the first 64 columns of S[sb]: this slice's 32 keys -> 16 columns
        tmem_st16(tmem + lane_addr + sb * 128 + wg * 16, pk);
        tmem_wait_st();
        if (j > 0 && !waited) {
          mbar_wait(&bars->o_done, o_phase);            // keep o_done phases in lock-step
          o_phase ^= 1;
        }
        tc_fence_before();
        if (tr) trace(p, 7 + (wg & 1) * 4, s_iter - 1);
        mbar_arrive(&bars->p_full);
      }
      float l;
      {
        float a, b;
        f2_unpack(f2_add(lsum[0], lsum[1]), a, b);
        l = a + b;
      }
      // epilogue: wait for the last PV, combine the slices' row sums, normalise,
      // scatter this slice's columns of the row to its raster slot
      mbar_wait(&bars->o_done, o_phase);
      o_phase ^= 1;
      tc_fence_after();
      red_sum[wg * kBM + r] = l;   // dedicated slots: the max slots may still be read by peers
      named_bar_sync(kBarMax, kSoftmaxThreads);
      float l_tot = 0.f;
#pragma unroll
      for (int w = 0; w < kWG; ++w) l_tot += red_sum[w * kBM + r];
      const int64_t i = u * kBM + r;
      const float inv_l = 1.f / l_tot;
      constexpr int kOC = C::kOColsPerWG;
      uint32_t ov[kOC];
      if constexpr (kOC == 32)
        tmem_ld32(tmem + lane_addr + C::kOCol + wg * kOC, *reinterpret_cast<uint32_t(*)[32]>(ov));
      else
        tmem_ld16(tmem + lane_addr + C::kOCol + wg * kOC, *reinterpret_cast<uint32_t(*)[16]>(ov));
      tmem_wait_ld();
      tc_fence_before();
      if (i < p.nq) {
        const int64_t orow = p.out_rows ? int64_t(p.out_rows[i]) : i;
        __nv_bfloat16* dst = p.out + row_offset(p.out_layout, p.nq, p.heads, D, h, orow) + wg * kOC;
#pragma unroll
        for (int q8 = 0; q8 < kOC / 8; ++q8) {
          uint4 w;
          w.x = pack_bf16(__uint_as_float(ov[8 * q8 + 0]) * inv_l, __uint_as_float(ov[8 * q8 + 1]) * inv_l);
          w.y = pack_bf16(__uint_as_float(ov[8 * q8 + 2]) * inv_l, __uint_as_float(ov[8 * q8 + 3]) * inv_l);
          w.z = pack_bf16(__uint_as_float(ov[8 * q8 + 4]) * inv_l, __uint_as_float(ov[8 * q8 + 5]) * inv_l);
          w.w = pack_bf16(__uint_as_float(ov[8 * q8 + 6]) * inv_l, __uint_as_float(ov[8 * q8 + 7]) * inv_l);
          *reinterpret_cast<uint4*>(dst + q8 * 8) = w;
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
  p.trace = nullptr;
  const char* trace_path = getenv("DFS_ATTN_TRACE");
  p.exp_mode = getenv("DFS_ATTN_EXP") ? atoi(getenv("DFS_ATTN_EXP")) : 0;
  if (trace_path) DFS_CUDA_CHECK(cudaMalloc(&p.trace, 16 * 256 * sizeof(unsigned long long)));
  if (p.trace) DFS_CUDA_CHECK(cudaMemsetAsync(p.trace, 0, 16 * 256 * sizeof(unsigned long long), stream));
  static bool attr_set = false;
  if (!attr_set) {
    DFS_CUDA_CHECK(cudaFuncSetAttribute(attn_sm100_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
    attr_set = true;
  }
  const int64_t grid = p.tiles < kNumSMs ? p.tiles : kNumSMs;
  attn_sm100_kernel<D><<<unsigned(grid), kThreads, C::kSmem, stream>>>(mq, mk, mv, p);
  DFS_LAUNCH_CHECK("attn_sm100");
  if (p.trace) {
    unsigned long long host[16 * 256];
    DFS_CUDA_CHECK(cudaMemcpyAsync(host, p.trace, sizeof(host), cudaMemcpyDeviceToHost, stream));
    DFS_CUDA_CHECK(cudaStreamSynchronize(stream));
    if (FILE* f = fopen(trace_path, "wb")) {
      fwrite(host, sizeof(host), 1, f);
      fclose(f);
    }
    cudaFree(p.trace);
  }
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
