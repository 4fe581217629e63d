// attn_b64.cu — K5 for B = 64: block-sparse FlashAttention forward on tcgen05 / TMEM / TMA
// with 64-token query and key blocks (SURVEY §8(b) contract B in {64, 128}; config T).
//
// block_sparse_attention (attention.cpp:125-159) at B = 64 with the B = 128 kernel's
// machinery (attn_sm100.cu: warp roles, TMA ring, three TMEM S buffers, online softmax
// split over two warpgroups, fused unpermute): a 128-row tile holds the two query blocks
// 2t and 2t+1 (one M = 128 MMA), and walks the UNION of their key lists in 64-key blocks
// (N = 64 MMAs). A pre-pass merges the two ascending CSR rows into one list whose
// entries carry an ownership mask (bit 28: block 2t, bit 29: block 2t+1); the softmax
// warps of a half that does not own a block write P = 0 for it, so each query row
// attends exactly its own block list (padded keys of the last block excluded, rows past
// N never stored). Kept as a separate kernel so the B = 128 kernel's code stays the
// tuned one (the generalised template measured +2.9 % SM cycles at HY, ncu).
#include <cuda.h>

#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "sm100.cuh"

namespace dfsgpu {

namespace {

using namespace sm100;

constexpr int kBM = 128;         // query rows per tile (= TMEM lanes)
// Key block = MMA N: 128 (B = 128), or 64 (B = 64: a tile then holds the two query blocks
// 2t, 2t+1 and walks the union of their key lists; each entry carries an ownership
// mask in bits 28-29 and the rows of a half that does not own a block get P = 0).
constexpr int32_t kBlkMask = 0x0fffffff;
#ifndef DFS_ATTN_WG
#define DFS_ATTN_WG 2
#endif
constexpr int kWG = DFS_ATTN_WG;           // softmax warpgroups splitting the 128 key columns
constexpr int kSoftmaxThreads = 128 * kWG;
constexpr int kThreads = 64 + kSoftmaxThreads;
constexpr uint32_t kTmemCols = 512;
#ifndef DFS_ATTN_RESCALE_LOG2
#define DFS_ATTN_RESCALE_LOG2 8.0f
#endif
constexpr float kRescaleThreshold = DFS_ATTN_RESCALE_LOG2;  // log2 units
constexpr uint32_t kBarRows = 2;           // named barriers 2..5: one per 32-row group (0 = __syncthreads)

template <int D, int BN>
struct Cfg {
  static constexpr int kCPT = BN / kWG;                  // key columns (logits) per softmax thread per block
  static constexpr int kChunks = D / 64;                 // 128-byte swizzle chunks per row
  static constexpr int kTileBytes = kBM * D * 2;         // the Q tile
  static constexpr int kChunkBytes = kBM * 128;          // one 128 x 64 bf16 TMA box (Q)
  static constexpr int kKVTileBytes = BN * D * 2;        // one K / V block
  static constexpr int kKVChunkBytes = BN * 128;         // one BN x 64 bf16 TMA box (K / V)
  static constexpr int kStages = D == 64 ? 12 : (BN == 128 ? 5 : 10);
  static constexpr int kQOff = 0;
  static constexpr int kRingOff = kQOff + kTileBytes;
  static constexpr int kRedOff = kRingOff + kStages * kKVTileBytes;  // float max[2][kWG][128], sum[kWG][128]
  static constexpr int kBarOff = kRedOff + 3 * kWG * kBM * 4;
  static constexpr int kSmem = kBarOff + 512 + 1024;     // barriers + alignment slack
  static constexpr uint32_t kIdescQK = idesc_bf16_f32(kBM, BN, false, false);
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
  int out_v8;  // output 32-byte aligned: 32-byte epilogue stores
  int in_nhd;  // 1: inputs are [N, H, d] (tensor-map coordinates (col, head, row))
  float scale_log2;
  const uint32_t* in_rows;  // fused Q reorder: logical query row i = raster token in_rows[i] (NULL: tiles)
  int64_t mq_blk;           // B = 64: query blocks per head (two per tile)
  const int32_t* u_cnt;     // B = 64: per tile, the length of the union list at blk_idx[blk_ptr[h*mq_blk+2t]]
  int64_t tiles;
};

struct Bars {
  uint64_t q_full, q_empty;
  uint64_t s_full[3];
  uint64_t p_full[3], o_done[3];  // per S/P buffer: the softmax may run a block ahead of PV
  uint64_t kv_full[12], kv_empty[12];
  uint32_t tmem_base;
};

// (begin, count) of a tile's key-block list, loaded one tile ahead by every role so the
// list pointers, the first list entry and the epilogue's output-row index are not a
// chain of dependent global loads on each tile boundary
struct TileMeta {
  int32_t beg, cnt;
};
template <int BN>
__device__ __forceinline__ TileMeta load_meta(const Params& p, int64_t tile) {
  TileMeta t{0, 0};
  if (tile < p.tiles) {
    if (p.blk_ptr && BN == 64) {  // union list of query blocks 2t, 2t+1, stored over their CSR rows
      const int64_t h = tile / p.mq, u = tile - h * p.mq;
      t.beg = __ldg(p.blk_ptr + h * p.mq_blk + 2 * u);
      t.cnt = __ldg(p.u_cnt + tile);
    } else if (p.blk_ptr) {
      t.beg = __ldg(p.blk_ptr + tile);
      t.cnt = __ldg(p.blk_ptr + tile + 1) - t.beg;
    } else {
      t.cnt = int32_t(p.mk);
    }
  }
  return t;
}


__device__ __forceinline__ int32_t block_at(const Params& p, int32_t beg, int32_t j) {
  return p.blk_ptr ? p.blk_idx[beg + j] : j;
}

// which exp2 pairs of a thread's row slice go to the FMA-pipe polynomial: POLY = n < 10
// is every n-th pair (0 = none); POLY = 38 is pairs 1, 4, 7 of every 8
template <int POLY>
__device__ __forceinline__ constexpr bool use_poly(int i) {
  if constexpr (POLY == 0) {
    return false;
  } else if constexpr (POLY == 38) {
    return (0x92u >> (i % 8)) & 1u;  // pairs 1, 4, 7 of each 8
  } else {
    return i % POLY == POLY - 1;
  }
}

template <int D, int POLY, int BN>
__global__ void __launch_bounds__(kThreads, 1)
    attn_b64_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                      const __grid_constant__ CUtensorMap tm_v, const Params p) {
  using C = Cfg<D, BN>;
  constexpr int kBN = BN;
  constexpr int kCPT = C::kCPT;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment (SWIZZLE_128B atoms) by offset, so the pointer keeps its shared state space
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem + C::kQOff;
  uint8_t* sRing = smem + C::kRingOff;
  float* red = reinterpret_cast<float*>(smem + C::kRedOff);  // [parity][wg][row]
  Bars* bars = reinterpret_cast<Bars*>(smem + C::kBarOff);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    mbar_init(&bars->q_full, 1);
    mbar_init(&bars->q_empty, 1);
    for (int i = 0; i < 3; ++i) {
      mbar_init(&bars->s_full[i], 1);
      mbar_init(&bars->p_full[i], kSoftmaxThreads / 32);  // one arrive per softmax warp
      mbar_init(&bars->o_done[i], 1);
    }
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
    // The whole warp runs the loop (so the control state is warp-uniform) and one
    // elected lane issues; the key-block list is read 32 entries at a time by the
    // warp (one coalesced load) and broadcast with shuffles, keeping the LUT's
    // global-load latency off the per-block issue path.
    uint32_t q_phase = 0, ring = 0;
    // Fused Q reorder (p.in_rows != NULL): Q's map is 2D over the raster [N*H, d]
    // activations and a 128-row tile is 32 tile::gather4 loads per 64-column chunk, one
    // per lane; lane l fetches logical rows 4l..4l+3 = raster tokens in_rows[row0+4l..].
    // Rows past n (partial last block) repeat a valid token (padded queries are never
    // stored). K/V are not gathered: each K/V tile is re-read by ~K query blocks, and
    // gather4 moves only ~7 B/clk/SM (measured), so their reorder stays a one-time copy.
    // The raster row indices are loaded before waiting for the ring slot, so their
    // latency overlaps the wait.
    auto gather_rows = [&](int64_t h, int64_t row0, int (&rr)[4]) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        int64_t i = row0 + 4 * lane + k;
        i = i < p.nq ? i : p.nq - 1;
        rr[k] = int(int64_t(__ldg(p.in_rows + i)) * p.heads + h);
      }
    };
    auto issue_tile = [&](const CUtensorMap* map, int64_t h, int64_t row0, uint8_t* dst, uint64_t* bar,
                          const int (&rr)[4], bool gather, uint32_t bytes, uint32_t chunk_bytes) {
      if constexpr (BN == 128) {  // Q and K/V tiles share one geometry
        bytes = C::kTileBytes;
        chunk_bytes = C::kChunkBytes;
      }
      if (gather) {
        if (elect_one()) mbar_expect_tx(bar, C::kTileBytes);
        __syncwarp();
#pragma unroll
        for (int c = 0; c < C::kChunks; ++c)
          tma_gather4(dst + c * C::kChunkBytes + lane * 512, map, bar, c * 64, rr[0], rr[1], rr[2], rr[3]);
        __syncwarp();
        return;
      }
      if (elect_one()) {
        mbar_expect_tx(bar, bytes);
#pragma unroll
        for (int c = 0; c < C::kChunks; ++c)
          tma_load_3d(dst + c * chunk_bytes, map, bar, c * 64, p.in_nhd ? int(h) : int(row0),
                      p.in_nhd ? int(row0) : int(h));
      }
      __syncwarp();
    };
    auto load_tile = [&](const CUtensorMap* map, int64_t h, int64_t row0) {
      const uint32_t slot = ring % C::kStages;
      const uint32_t use = ring / C::kStages;
      const int rr[4] = {0, 0, 0, 0};
      mbar_wait(&bars->kv_empty[slot], (use & 1) ^ 1);
      issue_tile(map, h, row0, sRing + slot * C::kKVTileBytes, &bars->kv_full[slot], rr, false, C::kKVTileBytes,
                 C::kKVChunkBytes);
      ++ring;
    };
    TileMeta nxt = load_meta<BN>(p, blockIdx.x);
    for (int64_t tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
      const int64_t h = tile / p.mq, u = tile % p.mq;
      const int32_t beg = nxt.beg, cnt = nxt.cnt;
      nxt = load_meta<BN>(p, tile + gridDim.x);
      {
        int rr[4] = {0, 0, 0, 0};
        if (p.in_rows) gather_rows(h, u * kBM, rr);  // row indices fetched while Q's slot drains
        mbar_wait(&bars->q_empty, q_phase ^ 1);
        q_phase ^= 1;
        issue_tile(&tm_q, h, u * kBM, sQ, &bars->q_full, rr, p.in_rows != nullptr, C::kTileBytes, C::kChunkBytes);
      }
      // key-block list window: entries [win, win + 32) held one per lane
      int32_t win = -64, lut_reg = 0;
      auto blk = [&](int32_t j) -> int32_t {
        if (!p.blk_ptr) return j;
        const int32_t w = j & ~31;
        if (w != win) {
          win = w;
          lut_reg = (w + lane < cnt) ? p.blk_idx[beg + w + lane] : 0;
        }
        const int32_t e = __shfl_sync(0xffffffffu, lut_reg, j & 31);
        return BN == 64 ? e & kBlkMask : e;
      };
      // consumption order of the MMA warp (QK runs two blocks ahead of PV):
      // K0, K1, K2, V0, K3, V1, ..., K_{n-1}, V_{n-3}, V_{n-2}, V_{n-1}
      if (cnt > 0) load_tile(&tm_k, h, int64_t(blk(0)) * kBN);
      if (cnt > 1) load_tile(&tm_k, h, int64_t(blk(1)) * kBN);
      for (int32_t j = 0; j < cnt; ++j) {
        if (j + 2 < cnt) load_tile(&tm_k, h, int64_t(blk(j + 2)) * kBN);
        load_tile(&tm_v, h, int64_t(blk(j)) * kBN);
      }
    }
  } else if (warp == 1) {
    // ================================ MMA issuer ================================
    // Warp-uniform control flow, one elected lane issues. Descriptors are kept as
    // 32-bit halves: per K step only the low word moves (one uniform add), which
    // keeps the issue path to a handful of instructions per UMMA — this warp shares
    // its scheduler with four softmax warps, so its instruction count sets the
    // tensor pipe's feed rate.
    uint32_t q_phase = 0, ring = 0, s_iter = 0, pv_iter = 0;
    constexpr uint32_t kHiK = desc_sw128_hi(1024);  // K-major SW128: LBO 16 B (unused), SBO 1024 B
    const uint32_t q_lo = desc_sw128_lo(smem_u32(sQ), 16);
    const uint32_t ring_lo = desc_sw128_lo(smem_u32(sRing), 16);
    const uint32_t ring_lo_v = desc_sw128_lo(smem_u32(sRing), C::kKVChunkBytes);  // V: MN-major, LBO = chunk
    auto next_slot = [&]() -> uint32_t {
      const uint32_t slot = ring % C::kStages;
      mbar_wait(&bars->kv_full[slot], (ring / C::kStages) & 1);
      ++ring;
      return slot;
    };
    // Three S/P buffers: QK_{j+2} overwrites S[(j+2)%3], whose P_{j-1} was consumed by
    // PV_{j-1}, issued earlier into the in-order tcgen05 pipe — so QK never waits for the
    // softmax, and the tensor pipe always has the next QK queued behind each PV.
    auto issue_qk = [&]() {
      const uint32_t slot = next_slot();
      const uint32_t sb = s_iter % C::kSBufs;
      tc_fence_after();
      const uint32_t k_lo = ring_lo + slot * (C::kKVTileBytes >> 4);
      if (elect_one()) {
#pragma unroll
        for (int s = 0; s < D / 16; ++s) {
          const uint32_t off = ((s >> 2) * C::kChunkBytes + (s & 3) * 32) >> 4;
          const uint32_t off_k = ((s >> 2) * C::kKVChunkBytes + (s & 3) * 32) >> 4;
          umma_ss(tmem + sb * 128, q_lo + off, kHiK, k_lo + off_k, kHiK, C::kIdescQK, s > 0);
        }
        umma_commit(&bars->kv_empty[slot]);
        umma_commit(&bars->s_full[sb]);
      }
      __syncwarp();
      ++s_iter;
    };
    auto issue_pv = [&](bool first) {
      const uint32_t slot = next_slot();
      const uint32_t pb = pv_iter % C::kSBufs;
      mbar_wait(&bars->p_full[pb], (pv_iter / C::kSBufs) & 1);
      tc_fence_after();
      const uint32_t v_lo = ring_lo_v + slot * (C::kKVTileBytes >> 4);
      const uint32_t p_tmem = tmem + pb * 128;  // P_j aliases S_j (bf16 pairs)
      if (elect_one()) {
#pragma unroll
        for (int s = 0; s < kBN / 16; ++s) {
          umma_ts(tmem + C::kOCol, p_tmem + s * 8, v_lo + ((s * 16 * 128) >> 4), kHiK, C::kIdescPV,
                  (!first || s > 0) ? 1u : 0u);
        }
        umma_commit(&bars->kv_empty[slot]);
        umma_commit(&bars->o_done[pb]);
      }
      __syncwarp();
      ++pv_iter;
    };
    TileMeta nxt = load_meta<BN>(p, blockIdx.x);
    for (int64_t tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
      const int32_t cnt = nxt.cnt;
      nxt = load_meta<BN>(p, tile + gridDim.x);
      mbar_wait(&bars->q_full, q_phase);
      q_phase ^= 1;
      if (cnt > 0) issue_qk();
      if (cnt > 1) issue_qk();
      auto release_q = [&]() {  // Q smem free once the last QK read it
        if (elect_one()) umma_commit(&bars->q_empty);
        __syncwarp();
      };
      if (cnt <= 2) release_q();
      for (int32_t j = 0; j < cnt; ++j) {
        if (j + 2 < cnt) {
          issue_qk();
          if (j + 3 == cnt) release_q();
        }
        issue_pv(j == 0);
      }
    }
  } else {
    // ============================ softmax / epilogue ============================
    // kWG warpgroups split the 128 key columns of each block (128 / kWG each); a thread
    // owns one query row (TMEM lane) of its 32-column slice.
    const int wg = (warp - 2) >> 2;                    // key columns [kCPT*wg, kCPT*wg + kCPT)
    const int r = (warp & 3) * 32 + lane;              // query row within the tile == TMEM lane
    const uint32_t lane_addr = uint32_t((warp & 3) * 32) << 16;
    // A row's max / sum exchange involves only the kWG warps holding that row's slices
    // (same warp & 3): each 32-row group synchronises on its own named barrier, so a
    // slow warp stalls three peers instead of all sixteen softmax warps.
    const uint32_t bar_rows = kBarRows + uint32_t(warp & 3);
    uint32_t s_iter = 0;
    float* red_max = red;                              // [parity][kWG][kBM]
    float* red_sum = red + 2 * kWG * kBM;              // [kWG][kBM]
    // PV number g (CTA-global block counter) completes phase (g / 3) & 1 of o_done[g % 3].
    // Waiting on it by parity is safe: S_{g+1} (or S_g at the epilogue) being ready implies
    // PV_{g-3} completed (in-order tcgen05 pipe, QK_{g+1} is issued after PV_{g-2}), so the
    // barrier is never more than one phase behind the one waited for.
    auto wait_pv = [&](uint32_t g) { mbar_wait(&bars->o_done[g % C::kSBufs], (g / C::kSBufs) & 1); };
    TileMeta nxt = load_meta<BN>(p, blockIdx.x);
    int32_t vb_first = nxt.cnt > 0 ? block_at(p, nxt.beg, 0) : 0;
    // B = 64: rows 0-63 (warps & 3 in {0, 1}) are query block 2t (ownership bit 0), rows
    // 64-127 query block 2t+1 (bit 1)
    const int own_bit = ((warp & 3) >> 1) + 28;
    for (int64_t tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
      const int64_t h = tile / p.mq, u = tile % p.mq;
      const int32_t beg = nxt.beg, cnt = nxt.cnt;
      nxt = load_meta<BN>(p, tile + gridDim.x);
      const int64_t i_row = u * kBM + r;  // this thread's query row, and its raster slot
      const int64_t orow = i_row < p.nq && p.out_rows ? int64_t(__ldg(p.out_rows + i_row)) : i_row;
      float m = -INFINITY;
      uint64_t lsum[2] = {0, 0};  // packed fp32x2 partial row sums (2 independent chains)
      int32_t vb_next = vb_first;
      for (int32_t j = 0; j < cnt; ++j) {
        const int32_t entry = vb_next;
        const int32_t vb = BN == 64 ? entry & kBlkMask : entry;
        if (j + 1 < cnt) vb_next = block_at(p, beg, j + 1);  // prefetch: keeps the LUT load off the critical path
        const uint32_t sb = s_iter % C::kSBufs;
        const uint32_t s_phase = (s_iter / C::kSBufs) & 1;
        float* red_par = red_max + (s_iter & 1) * kWG * kBM;
        mbar_wait(&bars->s_full[sb], s_phase);
        tc_fence_after();
        if (BN == 64 && p.blk_ptr && !((entry >> own_bit) & 1)) {
          // a block of the partner query block only: this half's P is zero (warp-uniform;
          // the partner warps of these rows skip it the same way, so no exchange)
          uint32_t zero[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) zero[i] = 0u;
#pragma unroll
          for (int c = 0; c < kCPT / 32; ++c) tmem_st16(tmem + lane_addr + sb * 128 + wg * (kCPT / 2) + c * 16, zero);
          tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bars->p_full[sb]);
          ++s_iter;
          continue;
        }
        uint32_t sv[kCPT];
#pragma unroll
        for (int c = 0; c < kCPT / 32; ++c)
          tmem_ld32(tmem + lane_addr + sb * 128 + wg * kCPT + c * 32, *reinterpret_cast<uint32_t(*)[32]>(sv + 32 * c));
        tmem_wait_ld();
        // padded keys of a partial last block (attention.cpp:146-152); warp-uniform branch
        const int valid = int(min(int64_t(kBN), p.nk - int64_t(vb) * kBN)) - wg * kCPT;
        if (valid < kCPT) {
#pragma unroll
          for (int i = 0; i < kCPT; ++i)
            if (i >= valid) sv[i] = __float_as_uint(-INFINITY);
        }
        float mq[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int i = 0; i < kCPT; ++i) mq[i & 3] = fmaxf(mq[i & 3], __uint_as_float(sv[i]));
        float mx = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3]));
        red_par[wg * kBM + r] = mx;
        named_bar_sync(bar_rows, kWG * 32);            // every slice of these rows published its max
#pragma unroll
        for (int w = 0; w < kWG; ++w) mx = fmaxf(mx, red_par[w * kBM + r]);
        const float m_new = fmaxf(m, mx * p.scale_log2);
        // tcgen05.ld/st are warp-collective: the rescale decision is warp-uniform
        // (the partner warps cover the same rows, so they decide identically)
        if (j == 0 || (BN == 64 && m == -INFINITY)) {  // first block this row attends
          m = m_new;
        } else if (__any_sync(0xffffffffu, m_new - m > kRescaleThreshold)) {
          wait_pv(s_iter - 1);                          // PV_{j-1} complete: O stable
          tc_fence_after();
          const float alpha = ex2(m - m_new);
          const uint64_t a2 = f2_pack(alpha, alpha);
          lsum[0] = f2_mul(lsum[0], a2);
          lsum[1] = f2_mul(lsum[1], a2);
          m = m_new;
          const uint32_t o_addr = tmem + lane_addr + C::kOCol + wg * C::kOColsPerWG;
          if constexpr (C::kOColsPerWG >= 32) {
#pragma unroll
            for (int c = 0; c < C::kOColsPerWG; c += 32) {
              uint32_t ov[32];
              tmem_ld32(o_addr + c, ov);
              tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
              tmem_st32(o_addr + c, ov);
            }
          } else {
            uint32_t ov[16];
            tmem_ld16(o_addr, ov);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
            tmem_st16(o_addr, ov);
          }
        }
        // p = 2^(s*scale - m); the use_poly<POLY> pairs on the FMA pipe (offloads MUFU)
        const uint64_t sc2 = f2_pack(p.scale_log2, p.scale_log2), nm2 = f2_pack(-m, -m);
        uint32_t pk[kCPT / 2];
#pragma unroll
        for (int i = 0; i < kCPT / 2; ++i) {
          float x0, x1;
          f2_unpack(f2_fma(f2_pack(__uint_as_float(sv[2 * i]), __uint_as_float(sv[2 * i + 1])), sc2, nm2), x0, x1);
          float p0, p1;
          if (use_poly<POLY>(i)) {
            f2_unpack(ex2_poly2(x0, x1), p0, p1);
          } else {
            p0 = ex2(x0);
            p1 = ex2(x1);
          }
          lsum[i & 1] = f2_add(lsum[i & 1], f2_pack(p0, p1));
          pk[i] = pack_bf16(p0, p1);
        }
        // P_j (bf16 pairs) over the first 64 columns of S[sb]: this slice's kCPT keys -> kCPT/2 columns
#pragma unroll
        for (int c = 0; c < kCPT / 32; ++c)
          tmem_st16(tmem + lane_addr + sb * 128 + wg * (kCPT / 2) + c * 16,
                    *reinterpret_cast<const uint32_t(*)[16]>(pk + 16 * c));
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();  // every lane's P store has completed (tcgen05.wait::st above)
        if (lane == 0) mbar_arrive(&bars->p_full[sb]);
        ++s_iter;
      }
      vb_first = nxt.cnt > 0 ? block_at(p, nxt.beg, 0) : 0;  // lands during the epilogue
      float l;
      {
        float a, b;
        f2_unpack(f2_add(lsum[0], lsum[1]), a, b);
        l = a + b;
      }
      // epilogue: wait for the last PV, combine the slices' row sums, normalise,
      // scatter this slice's columns of the row to its raster slot
      if (cnt > 0) wait_pv(s_iter - 1);
      tc_fence_after();
      red_sum[wg * kBM + r] = l;   // dedicated slots: the max slots may still be read by peers
      named_bar_sync(bar_rows, kWG * 32);
      float l_tot = 0.f;
#pragma unroll
      for (int w = 0; w < kWG; ++w) l_tot += red_sum[w * kBM + r];
      const int64_t i = i_row;
      // an empty key list (possible only through a caller-built CSR; the BlockMask entry
      // points refuse it like attention.cpp:133-136) yields a zero row, never stale TMEM
      // (B = 64: a half that owns none of the tile's blocks also gets a zero row)
      const float inv_l = cnt > 0 && (BN == 128 || l_tot > 0.f) ? 1.f / l_tot : 0.f;
      constexpr int kOC = C::kOColsPerWG;
      uint32_t ov[kOC];
      if constexpr (kOC >= 32) {
#pragma unroll
        for (int c = 0; c < kOC; c += 32)
          tmem_ld32(tmem + lane_addr + C::kOCol + wg * kOC + c, *reinterpret_cast<uint32_t(*)[32]>(ov + c));
      } else {
        tmem_ld16(tmem + lane_addr + C::kOCol + wg * kOC, *reinterpret_cast<uint32_t(*)[16]>(ov));
      }
      tmem_wait_ld();
      tc_fence_before();
      if (cnt == 0) {
#pragma unroll
        for (int c = 0; c < kOC; ++c) ov[c] = 0u;
      }
      if (i < p.nq) {
        __nv_bfloat16* dst = p.out + row_offset(p.out_layout, p.nq, p.heads, D, h, orow) + wg * kOC;
        // 32-byte stores (STG.256): half the store instructions of 16-byte ones; the store
        // issue at the tile boundary is what holds the warps there
        uint32_t w[kOC / 2];
#pragma unroll
        for (int c = 0; c < kOC / 2; ++c)
          w[c] = pack_bf16(__uint_as_float(ov[2 * c]) * inv_l, __uint_as_float(ov[2 * c + 1]) * inv_l);
        if (p.out_v8) {
#pragma unroll
          for (int q = 0; q < kOC / 16; ++q)
            asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst + q * 16),
                         "r"(w[8 * q + 0]), "r"(w[8 * q + 1]), "r"(w[8 * q + 2]), "r"(w[8 * q + 3]),
                         "r"(w[8 * q + 4]), "r"(w[8 * q + 5]), "r"(w[8 * q + 6]), "r"(w[8 * q + 7])
                         : "memory");
        } else {  // output only 16-byte aligned
#pragma unroll
          for (int q = 0; q < kOC / 8; ++q)
            *reinterpret_cast<uint4*>(dst + q * 8) = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
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

}  // namespace

int make_token_map_rows(CUtensorMap* map, const void* base, int layout, int64_t n, int64_t heads, int64_t d,
                        int box_rows);  // attn_sm100.cu
int make_row_gather_map(CUtensorMap* map, const void* base, int64_t rows, int64_t d);

namespace {

template <int D, int POLY, int BN>
int launch_kernel(const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv, const Params& p,
                  cudaStream_t stream) {
  using C = Cfg<D, BN>;
  // per device and race-free: set on every launch (~1 us)
  DFS_CUDA_CHECK(cudaFuncSetAttribute(attn_b64_kernel<D, POLY, BN>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
  const int64_t grid = p.tiles < kNumSMs ? p.tiles : kNumSMs;
  attn_b64_kernel<D, POLY, BN><<<unsigned(grid), kThreads, C::kSmem, stream>>>(mq, mk, mv, p);
  DFS_LAUNCH_CHECK("attn_sm100");
  return DFS_OK;
}

// exp2 split between MUFU and the FMA-pipe polynomial (use_poly): measured per head
// dimension with tools/k5_cycles.sh and the degree-2 polynomial — d = 128: pairs 1, 4, 7
// of every 8 (-1.9 % SM cycles vs every 3rd; the positions matter as much as the
// ratio: pairs 0, 3, 6 gain only 0.5 %), d = 64: every 3rd pair. DFS_ATTN_POLY
// overrides the default for A/B measurements.
template <int D>
constexpr int kDefaultPoly = D == 128 ? 38 : 3;

// B = 64: the union of the key lists of query blocks 2t and 2t+1, written over their
// (adjacent) CSR rows: entry = key block | ownership bits (28: block 2t, 29: block 2t+1).
// One thread per tile, a linear merge of two ascending lists (attention.cpp:146-152's
// per-block key sets, visited once for both blocks).
__global__ void union_pairs_kernel(const int32_t* __restrict__ ptr, const int32_t* __restrict__ idx, int64_t heads,
                                   int64_t mq_blk, int64_t tiles_per_head, int32_t* __restrict__ out,
                                   int32_t* __restrict__ cnt) {
  const int64_t tile = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (tile >= heads * tiles_per_head) return;
  const int64_t h = tile / tiles_per_head, t = tile - h * tiles_per_head;
  const int64_t u0 = h * mq_blk + 2 * t;
  const int32_t ab = ptr[u0], ae = ptr[u0 + 1];
  const bool has_b = 2 * t + 1 < mq_blk;
  const int32_t bb = has_b ? ptr[u0 + 1] : 0, be = has_b ? ptr[u0 + 2] : 0;
  int32_t i = ab, j = bb, o = ab;
  while (i < ae || j < be) {
    const int32_t va = i < ae ? idx[i] : INT32_MAX, vb = j < be ? idx[j] : INT32_MAX;
    if (va == vb) {
      out[o++] = va | (3 << 28);
      ++i;
      ++j;
    } else if (va < vb) {
      out[o++] = va | (1 << 28);
      ++i;
    } else {
      out[o++] = vb | (2 << 28);
      ++j;
    }
  }
  cnt[tile] = o - ab;
}

template <int D, int BN = 128>
int launch(const dfs_attn_args& a, float scale, cudaStream_t stream) {
  CUtensorMap mq, mk, mv;
  int rc;
  if (a.in_rows) {  // Q: 2D row-gather map over the raster [N*H, d] activations
    if ((rc = make_row_gather_map(&mq, a.q, a.nq * a.heads, D))) return rc;
  } else if ((rc = make_token_map_rows(&mq, a.q, a.in_layout, a.nq, a.heads, D, 128))) {
    return rc;
  }
  if ((rc = make_token_map_rows(&mk, a.k, a.in_layout, a.nk, a.heads, D, BN))) return rc;
  if ((rc = make_token_map_rows(&mv, a.v, a.in_layout, a.nk, a.heads, D, BN))) return rc;
  Params p;
  p.heads = a.heads;
  p.nq = a.nq;
  p.nk = a.nk;
  p.mq = ceil_div(a.nq, kBM);
  p.mk = ceil_div(a.nk, BN);
  p.mq_blk = ceil_div(a.nq, BN);
  p.u_cnt = nullptr;
  int32_t* u_buf = nullptr;
  if (BN == 64 && a.blk_ptr) {
    // the union lists live at the CSR offsets of their first query block: buffers of nnz entries
    int32_t nnz = 0;
    DFS_CUDA_CHECK(cudaMemcpyAsync(&nnz, a.blk_ptr + a.heads * p.mq_blk, sizeof(int32_t), cudaMemcpyDeviceToHost,
                                   stream));
    DFS_CUDA_CHECK(cudaStreamSynchronize(stream));
    DFS_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&u_buf),
                                   sizeof(int32_t) * size_t(nnz + 1 + p.mq * a.heads), stream));
    int32_t* cnt = u_buf + nnz + 1;
    const int64_t tiles = p.mq * a.heads;
    union_pairs_kernel<<<unsigned(ceil_div(tiles, 128)), 128, 0, stream>>>(a.blk_ptr, a.blk_idx, a.heads, p.mq_blk,
                                                                         p.mq, u_buf, cnt);
    DFS_LAUNCH_CHECK("union_pairs");
    p.u_cnt = cnt;
  }
  p.blk_ptr = a.blk_ptr;
  p.blk_idx = u_buf ? u_buf : a.blk_idx;
  p.out_rows = a.out_rows;
  p.out = static_cast<__nv_bfloat16*>(a.o);
  p.out_layout = a.out_layout;
  p.out_v8 = (reinterpret_cast<uintptr_t>(a.o) & 31) == 0;
  p.in_nhd = a.in_layout == DFS_NHD;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.in_rows = a.in_rows;
  p.tiles = p.mq * a.heads;
  static_assert(BN == 64, "attn_b64 instantiates the 64-key-block kernel only");
  rc = launch_kernel<D, kDefaultPoly<D>, 64>(mq, mk, mv, p, stream);
  if (u_buf) cudaFreeAsync(u_buf, stream);
  if (rc) return rc;
  return DFS_OK;
}

}  // namespace

int sparse_attn_b64(const dfs_attn_args& a, float scale, cudaStream_t stream) {
  if (a.d == 128) return launch<128, 64>(a, scale, stream);
  if (a.d == 64) return launch<64, 64>(a, scale, stream);
  return fail(DFS_E_UNSUPPORTED, "attn_b64: d must be 64 or 128");
}

}  // namespace dfsgpu
