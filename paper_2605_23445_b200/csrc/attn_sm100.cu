// attn_sm100.cu — K5: block-sparse FlashAttention forward on tcgen05 / TMEM / TMA.
//
// block_sparse_attention (attention.cpp:125-159) for B = 128 (B = 64: attn_b64.cu), d in {64, 128},
// bf16 I/O, fp32 softmax and accumulation. Persistent CTAs (one per SM) walk
// (head, query block) tiles; a tile visits ONLY the key blocks of its CSR list
// (top-K LUT, or every block for dense / cross attention), so masked blocks
// cost neither bytes nor FLOPs.
//
// Warp roles (320 threads):
//   warp 0      TMA producer: the Q tile (TMA tile::gather4 of raster rows when the
//               reorder is fused), then K_0, K_1, ... / V_0, V_1, ... into one ring of
//               kStages smem slots (SWIZZLE_128B boxes of 128 x 64) in the MMA warp's order.
//   warp 9      MMA issuer (one elected lane): Q copied once per tile into TMEM
//               (tcgen05.cp), S_j = Q K_j^T with A from TMEM into one of the TMEM S
//               buffers, O += P_j V_j with P_j read straight from TMEM (bf16, aliasing S_j).
//   warps 1-8   softmax / epilogue. Default (row split): the two warps of a TMEM lane
//               quadrant own 16 query rows each, a thread pair per row (key columns
//               0-63 / 64-127, tcgen05.ld 16x32bx2), so a row's max is one shuffle and no
//               warp waits for another. The running max is stale by design: the
//               exponentials use it directly and a block that raises it by > 2^8 rescales
//               O in TMEM and recomputes (exact: O and l share the stale max). exp2 is
//               split between MUFU and a degree-2 FMA-pipe polynomial. The epilogue writes
//               each output row straight to its raster position out_rows[i] — the
//               unpermute (scheduler.cpp:134) is fused here.
//               DFS_ATTN_ROWSPLIT=0 builds the earlier column split (two warpgroups split
//               the 128 key columns, row max exchanged through shared memory per block).
// TMEM, row split: d = 128: S0/P0 [0,128) S1/P1 [128,256) O [256,384) Q [384,448) [448,512);
// d = 64: S0..S2 [0,384) O [384,448) Q [448,480) [480,512).
// Padded keys of the last partial block get -inf logits; padded query rows
// are computed on TMA zero-fill and never stored (attention.cpp:146-152).
#include <cuda.h>

#include <cstddef>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "sm100.cuh"

namespace dfsgpu {

namespace {

using namespace sm100;

constexpr int kBM = 128;         // query rows per tile (= TMEM lanes)
constexpr int kBN = 128;         // keys per block
#ifndef DFS_ATTN_WG
#define DFS_ATTN_WG 2
#endif
constexpr int kWG = DFS_ATTN_WG;           // softmax warpgroups splitting the 128 key columns
[[maybe_unused]] constexpr int kCPT = 128 / kWG;  // column split: key columns (logits) per softmax thread per block
constexpr int kSoftmaxThreads = 128 * kWG;
constexpr int kThreads = 64 + kSoftmaxThreads;
constexpr int kMmaWarp = kSoftmaxThreads / 32 + 1;  // 9; softmax warps 1 .. kSoftmaxThreads / 32
constexpr uint32_t kTmemCols = 512;
#ifndef DFS_ATTN_RESCALE_LOG2
#define DFS_ATTN_RESCALE_LOG2 8.0f
#endif
[[maybe_unused]] constexpr float kRescaleThreshold = DFS_ATTN_RESCALE_LOG2;  // log2 units
// Row split: the rescale test runs on each half-row's block sum of p instead of the max of
// the exponent arguments (no per-pair max on the ALU pipe): p >= 0, so a sum <= kRescaleSum
// bounds every p of the block by it; a larger sum sends the block down the rare path, which
// takes the block's real row max from S (still intact in TMEM).
#ifndef DFS_ATTN_SUMTEST
#define DFS_ATTN_SUMTEST 1
#endif
constexpr bool kSumTest = DFS_ATTN_SUMTEST;
// row split: S_j read from TMEM as one x64 load per thread, or as 2 / 4 smaller loads
#ifndef DFS_ATTN_LDSPLIT
#define DFS_ATTN_LDSPLIT 2
#endif
constexpr int kLdSplit = DFS_ATTN_LDSPLIT;
#ifndef DFS_ATTN_RESCALE_SUM
#define DFS_ATTN_RESCALE_SUM 4096.0f
#endif
constexpr float kRescaleSum = DFS_ATTN_RESCALE_SUM;
[[maybe_unused]] constexpr uint32_t kBarRows = 2;  // column split: named barriers 2..5: one per 32-row group (0 = __syncthreads)
// d = 64: the two softmax warpgroups run DECOUPLED (no per-block row-max exchange): each
// keeps its own running max / sum for its 64 key columns and its own O accumulator in
// TMEM (O_0 at column 384, O_1 at 448: 3 S buffers + 2 x 64 columns = 512), PV_j is two
// K = 64 MMAs (P_0 V[0:64] -> O_0, P_1 V[64:128] -> O_1) gated by per-warpgroup barriers,
// and the two partial rows are merged once per tile in the epilogue,
// O = (2^(m0-m) O_0 + 2^(m1-m) O_1) / (2^(m0-m) l_0 + 2^(m1-m) l_1). At d = 128 TMEM has
// no room for a second O next to three S buffers, so d = 128 keeps the exchange.
#ifndef DFS_ATTN_SPLIT_O_D64
#define DFS_ATTN_SPLIT_O_D64 1
#endif
// d = 128: Q resident in TMEM (QK^T issued with A from TMEM). Shared memory, not the tensor
// pipe, bounds the MMA side when Q is an smem operand: per 128 x 128 block QK reads Q and K
// (64 KB), PV reads V (32 KB) and TMA writes K and V (64 KB) — 160 KB at ~128 B/clk/SM is
// ~1250 cycles against 1024 tensor cycles (tools/mma_bw.cu; the MMA-only isolation build
// stalls at ~0.8 of peak). With Q copied once per tile into TMEM (tcgen05.cp, 8 x 128x256b)
// a block moves 128 KB of smem. TMEM then holds two S buffers: S0 [0,128) S1 [128,256),
// O [256,384), Q double-buffered at [384,448) / [448,512).
#ifndef DFS_ATTN_QT
#define DFS_ATTN_QT 1
#endif
// d = 128: softmax warps split the tile by ROWS, not key columns. The two warps sharing a TMEM
// lane quadrant (and an SMSP) own 16 rows each; a row's 128 logits are held by a thread pair
// (lanes l and l + 16: tcgen05.ld 16x32bx2, key columns 0-63 / 64-127), so the row max is one
// shuffle and no warp ever waits for another. With the column split both warps of an SMSP
// met at a per-block max exchange and ran in lockstep, so their serial phases (S wait, TMEM
// load, max chain, P store) coincided and the scheduler idled; decoupled, the arbiter's
// priority staggers them and one warp's latency hides under the other's exponentials.
#ifndef DFS_ATTN_ROWSPLIT
#define DFS_ATTN_ROWSPLIT 1
#endif

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
  // Q in TMEM (see DFS_ATTN_QT); at d = 64 its columns are the column-split path's second O
  static constexpr bool kQT = DFS_ATTN_QT && (D == 128 || DFS_ATTN_ROWSPLIT || !DFS_ATTN_SPLIT_O_D64);
  // TMEM: S0/P0 [0,128) S1/P1 [128,256) S2/P2 [256,384) O [384,384+D).
  // kQT, d = 128: two S buffers, O [256,384), Q [384,448) and [448,512);
  // kQT, d = 64: three S buffers, O [384,448), Q [448,480) and [480,512).
  static constexpr int kSBufs = kQT && D == 128 ? 2 : 3;
  static constexpr uint32_t kOCol = kQT && D == 128 ? 256 : 384;
  static constexpr uint32_t kQCol = D == 128 ? 384 : 448;
  static constexpr uint32_t kQStride = D / 2;  // TMEM columns of one Q buffer (bf16 pairs)
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
  unsigned long long* trace;  // debug timeline (DFS_ATTN_TRACE), NULL in production
  int64_t tiles;
  const dfs_peer_table* out_peers;  // Ulysses: rows go to the token owner's shard (kPeerOut instantiation)
};

struct Bars {
  uint64_t q_full, q_empty;
  uint64_t s_full[3];
  uint64_t p_full[3], o_done[3];  // per S/P buffer: the softmax may run a block ahead of PV
  uint64_t kv_full[12], kv_empty[12];
  uint32_t tmem_base;
  uint64_t p_full1[3];  // decoupled d = 64: warpgroup 1's P of each buffer (p_full: warpgroup 0's)
};

// (begin, count) of a tile's key-block list, loaded one tile ahead by every role so the
// list pointers, the first list entry and the epilogue's output-row index are not a
// chain of dependent global loads on each tile boundary
struct TileMeta {
  int32_t beg, cnt;
};
__device__ __forceinline__ TileMeta load_meta(const Params& p, int64_t tile) {
  TileMeta t{0, 0};
  if (tile >= 0 && tile < p.tiles) {
    if (p.blk_ptr) {
      t.beg = __ldg(p.blk_ptr + tile);
      t.cnt = __ldg(p.blk_ptr + tile + 1) - t.beg;
    } else {
      t.cnt = int32_t(p.mk);
    }
  }
  return t;
}

// The it-th tile of this CTA (-1: done). kMcast (dense steps, 2-CTA clusters): the two CTAs
// of a cluster take query blocks (2v, 2v+1) of one head, which walk the same key blocks, so
// the even CTA multicasts every K/V tile into both; with an odd block count the odd CTA
// repeats the head's last block without storing it (a "phantom" tile).
template <bool kMcast>
__device__ __forceinline__ int64_t tile_at(const Params& p, int64_t it) {
  if constexpr (!kMcast) {
    const int64_t t = int64_t(blockIdx.x) + it * gridDim.x;
    return t < p.tiles ? t : -1;
  } else {
    const int64_t pph = (p.mq + 1) / 2, pi = int64_t(blockIdx.x >> 1) + it * (gridDim.x >> 1);
    if (pi >= p.heads * pph) return -1;
    const int64_t u = 2 * (pi % pph) + (blockIdx.x & 1);
    return (pi / pph) * p.mq + (u < p.mq ? u : p.mq - 1);
  }
}
template <bool kMcast>
__device__ __forceinline__ bool phantom_tile(const Params& p, int64_t tile) {
  return kMcast && (blockIdx.x & 1) && (p.mq & 1) && tile % p.mq == p.mq - 1;
}

#ifndef DFS_TRACE_T0
#define DFS_TRACE_T0 64  // traced softmax warps: T0 / 32 and T0 / 32 + 4 (one SMSP)
#endif
#ifdef DFS_ATTN_TRACE_BUILD
__device__ __forceinline__ void trace(const Params& p, int ev, uint32_t idx) {
  if (p.trace && blockIdx.x == 0 && idx < 256) p.trace[ev * 256 + idx] = clock64();
}
#else
__device__ __forceinline__ void trace(const Params&, int, uint32_t) {}
#endif

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
  } else if constexpr (POLY == 516) {
    return (0x2492u >> (i % 16)) & 1u;  // pairs 1, 4, 7, 10, 13 of each 16
  } else {
    return i % POLY == POLY - 1;
  }
}

template <int D, int POLY, bool kPeerOut, bool kMcast>
__global__ void __launch_bounds__(kThreads, 1)
    attn_sm100_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                      const __grid_constant__ CUtensorMap tm_v, const Params p) {
  using C = Cfg<D>;
  constexpr bool kRowSplit = kWG == 2 && DFS_ATTN_ROWSPLIT;
  constexpr bool kSplitO = D == 64 && kWG == 2 && DFS_ATTN_SPLIT_O_D64 && !kRowSplit;
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
      if constexpr (kSplitO) {  // one arrive per warp of the owning warpgroup
        mbar_init(&bars->p_full[i], 4);
        mbar_init(&bars->p_full1[i], 4);
      } else {
        mbar_init(&bars->p_full[i], kSoftmaxThreads / 32);  // one arrive per softmax warp
      }
      mbar_init(&bars->o_done[i], 1);
    }
    for (int i = 0; i < C::kStages; ++i) {
      mbar_init(&bars->kv_full[i], 1);
      mbar_init(&bars->kv_empty[i], kMcast ? 2 : 1);  // kMcast: both CTAs' MMAs release a slot
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tm_q);
    prefetch_tmap(&tm_k);
    prefetch_tmap(&tm_v);
  }
  if (warp == kMmaWarp) tmem_alloc<kTmemCols>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if constexpr (kMcast) cluster_sync();  // the peer's barriers are initialised before any remote arrival
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
                          const int (&rr)[4], bool gather) {
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
        mbar_expect_tx(bar, C::kTileBytes);
#pragma unroll
        for (int c = 0; c < C::kChunks; ++c)
          tma_load_3d(dst + c * C::kChunkBytes, map, bar, c * 64, p.in_nhd ? int(h) : int(row0),
                      p.in_nhd ? int(row0) : int(h));
      }
      __syncwarp();
    };
    auto load_tile = [&](const CUtensorMap* map, int64_t h, int64_t row0) {
      const uint32_t slot = ring % C::kStages;
      const uint32_t use = ring / C::kStages;
      const int rr[4] = {0, 0, 0, 0};
      mbar_wait(&bars->kv_empty[slot], (use & 1) ^ 1);
#ifdef DFS_ATTN_SKIP_TMA  // experiment builds only: K/V never loaded (garbage operands)
      if (elect_one()) mbar_arrive(&bars->kv_full[slot]);
      __syncwarp();
#else
      if constexpr (kMcast) {  // each CTA expects the bytes; the even CTA multicasts them into both
        if (elect_one()) {
          mbar_expect_tx(&bars->kv_full[slot], C::kTileBytes);
          if ((blockIdx.x & 1) == 0) {
#pragma unroll
            for (int c = 0; c < C::kChunks; ++c)
              tma_load_3d_mcast2(sRing + slot * C::kTileBytes + c * C::kChunkBytes, map, &bars->kv_full[slot], c * 64,
                                 p.in_nhd ? int(h) : int(row0), p.in_nhd ? int(row0) : int(h));
          }
        }
        __syncwarp();
      } else {
        issue_tile(map, h, row0, sRing + slot * C::kTileBytes, &bars->kv_full[slot], rr, false);
      }
#endif
      ++ring;
    };
    TileMeta nxt = load_meta(p, tile_at<kMcast>(p, 0));
    for (int64_t it = 0, tile = tile_at<kMcast>(p, 0); tile >= 0; tile = tile_at<kMcast>(p, ++it)) {
      const int64_t h = tile / p.mq, u = tile % p.mq;
      const int32_t beg = nxt.beg, cnt = nxt.cnt;
      nxt = load_meta(p, tile_at<kMcast>(p, it + 1));
      {
        int rr[4] = {0, 0, 0, 0};
        if (p.in_rows) gather_rows(h, u * kBM, rr);  // row indices fetched while Q's slot drains
        mbar_wait(&bars->q_empty, q_phase ^ 1);
        q_phase ^= 1;
        issue_tile(&tm_q, h, u * kBM, sQ, &bars->q_full, rr, p.in_rows != nullptr);
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
        return __shfl_sync(0xffffffffu, lut_reg, j & 31);
      };
      // consumption order of the MMA warp (QK runs two blocks ahead of PV):
      // K0, K1, K2, V0, K3, V1, ..., K_{n-1}, V_{n-3}, V_{n-2}, V_{n-1}
      // (two S buffers, kQT: QK_{j+2} follows PV_j: K0, K1, V0, K2, V1, K3, ...)
      if (cnt > 0) load_tile(&tm_k, h, int64_t(blk(0)) * kBN);
      if (cnt > 1) load_tile(&tm_k, h, int64_t(blk(1)) * kBN);
      for (int32_t j = 0; j < cnt; ++j) {
        if constexpr (C::kSBufs == 2) {
          load_tile(&tm_v, h, int64_t(blk(j)) * kBN);
          if (j + 2 < cnt) load_tile(&tm_k, h, int64_t(blk(j + 2)) * kBN);
        } else {
          if (j + 2 < cnt) load_tile(&tm_k, h, int64_t(blk(j + 2)) * kBN);
          load_tile(&tm_v, h, int64_t(blk(j)) * kBN);
        }
      }
    }
  } else if (warp == kMmaWarp) {
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
    const uint32_t ring_lo_v = desc_sw128_lo(smem_u32(sRing), C::kChunkBytes);  // V: MN-major, LBO = chunk
    auto next_slot = [&]() -> uint32_t {
      const uint32_t slot = ring % C::kStages;
      trace(p, 0, ring);
      mbar_wait(&bars->kv_full[slot], (ring / C::kStages) & 1);
      trace(p, 1, ring);
      ++ring;
      return slot;
    };
    // Three S/P buffers: QK_{j+2} overwrites S[(j+2)%3], whose P_{j-1} was consumed by
    // PV_{j-1}, issued earlier into the in-order tcgen05 pipe — so QK never waits for the
    // softmax, and the tensor pipe always has the next QK queued behind each PV.
    uint32_t q_tm = tmem + C::kQCol;  // kQT: this tile's Q buffer in TMEM
    auto issue_qk = [&]() {
      const uint32_t slot = next_slot();
      const uint32_t sb = s_iter % C::kSBufs;
      tc_fence_after();
      const uint32_t k_lo = ring_lo + slot * (C::kTileBytes >> 4);
      if (elect_one()) {
#pragma unroll
        for (int s = 0; s < D / 16; ++s) {
          const uint32_t off = ((s >> 2) * C::kChunkBytes + (s & 3) * 32) >> 4;
#ifndef DFS_ATTN_SKIP_MMA  // experiment builds only (tools/attn_exp.sh): isolate the softmax side
          if constexpr (C::kQT)
            umma_ts(tmem + sb * 128, q_tm + s * 8, k_lo + off, kHiK, C::kIdescQK, s > 0);
          else
            umma_ss(tmem + sb * 128, q_lo + off, kHiK, k_lo + off, kHiK, C::kIdescQK, s > 0);
#endif
        }
        if constexpr (kMcast) umma_commit_both(&bars->kv_empty[slot]); else umma_commit(&bars->kv_empty[slot]);
        umma_commit(&bars->s_full[sb]);
      }
      __syncwarp();
      trace(p, 17, s_iter);
      ++s_iter;
    };
    auto issue_pv = [&](bool first) {
      const uint32_t slot = next_slot();
      const uint32_t pb = pv_iter % C::kSBufs;
      if constexpr (kSplitO) {  // two K = 64 halves, each as soon as its warpgroup's P is in
        const uint32_t v_lo = ring_lo_v + slot * (C::kTileBytes >> 4);
        const uint32_t p_tmem = tmem + pb * 128;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          mbar_wait(half ? &bars->p_full1[pb] : &bars->p_full[pb], (pv_iter / C::kSBufs) & 1);
          tc_fence_after();
          if (elect_one()) {
#pragma unroll
            for (int s = 4 * half; s < 4 * half + 4; ++s)  // P_1 sits in warpgroup 1's own S columns
              umma_ts(tmem + C::kOCol + half * D, p_tmem + half * 32 + s * 8, v_lo + ((s * 16 * 128) >> 4), kHiK,
                      C::kIdescPV, (!first || s > 4 * half) ? 1u : 0u);
          }
          __syncwarp();
        }
        if (elect_one()) {
          if constexpr (kMcast) umma_commit_both(&bars->kv_empty[slot]); else umma_commit(&bars->kv_empty[slot]);
          umma_commit(&bars->o_done[pb]);
        }
        __syncwarp();
        ++pv_iter;
        return;
      }
      trace(p, 2, pv_iter);
      mbar_wait(&bars->p_full[pb], (pv_iter / C::kSBufs) & 1);
      trace(p, 3, pv_iter);
      tc_fence_after();
      const uint32_t v_lo = ring_lo_v + slot * (C::kTileBytes >> 4);
      const uint32_t p_tmem = tmem + pb * 128;  // P_j aliases S_j (bf16 pairs)
      if (elect_one()) {
#pragma unroll
        for (int s = 0; s < kBN / 16; ++s) {
#ifndef DFS_ATTN_SKIP_MMA
          umma_ts(tmem + C::kOCol, p_tmem + s * 8, v_lo + ((s * 16 * 128) >> 4), kHiK, C::kIdescPV,
                  (!first || s > 0) ? 1u : 0u);
#endif
        }
        if constexpr (kMcast) umma_commit_both(&bars->kv_empty[slot]); else umma_commit(&bars->kv_empty[slot]);
        umma_commit(&bars->o_done[pb]);
      }
      __syncwarp();
      trace(p, 16, pv_iter);
      ++pv_iter;
    };
    TileMeta nxt = load_meta(p, tile_at<kMcast>(p, 0));
    for (int64_t it = 0, tile = tile_at<kMcast>(p, 0); tile >= 0; tile = tile_at<kMcast>(p, ++it)) {
      const int32_t cnt = nxt.cnt;
      nxt = load_meta(p, tile_at<kMcast>(p, it + 1));
      mbar_wait(&bars->q_full, q_phase);
      q_phase ^= 1;
      auto release_q = [&]() {  // Q smem free once the last QK read it (kQT: once copied to TMEM)
        if (elect_one()) umma_commit(&bars->q_empty);
        __syncwarp();
      };
      if constexpr (C::kQT) {
        // Q -> TMEM buffer (tile parity): one 128x256b copy per K step, the same SW128
        // K-major descriptors the SS MMA used. tcgen05.cp and tcgen05.mma execute in issue
        // order, and the buffer's previous user (two tiles back) issued all its QKs before.
        q_tm = tmem + C::kQCol + (q_phase ? 0u : C::kQStride);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int s = 0; s < D / 16; ++s) {
            const uint32_t off = ((s >> 2) * C::kChunkBytes + (s & 3) * 32) >> 4;
            tmem_cp_128x256b(q_tm + s * 8, (uint64_t(kHiK) << 32) | (q_lo + off));
          }
        }
        __syncwarp();
        release_q();
      }
      if (cnt > 0) issue_qk();
      if (cnt > 1) issue_qk();
      if constexpr (C::kSBufs == 2) {
        for (int32_t j = 0; j < cnt; ++j) {
          issue_pv(j == 0);
          if (j + 2 < cnt) issue_qk();
        }
      } else {
        if (!C::kQT && cnt <= 2) release_q();
        for (int32_t j = 0; j < cnt; ++j) {
          if (j + 2 < cnt) {
            issue_qk();
            if (!C::kQT && j + 3 == cnt) release_q();
          }
          issue_pv(j == 0);
        }
      }
    }
  } else if constexpr (kRowSplit) {
    // ============================ softmax / epilogue, row split ===========================
    // warp w (1..8): TMEM lane quadrant w & 3, row half (w - 1) >> 2: rows 32 (w & 3) + 16 half + [0, 16).
    // Lane l: row (l & 15) of those, key columns 64 (l >> 4) + [0, 64) of every block.
    const int hf = (warp - 1) >> 2, ch = lane >> 4;
    const int r = (warp & 3) * 32 + hf * 16 + (lane & 15);  // query row within the tile == TMEM lane
    const uint32_t lane_addr = uint32_t((warp & 3) * 32 + hf * 16) << 16;
    uint32_t s_iter = 0;
    const uint32_t s_full0 = pin_u32(smem_u32(&bars->s_full[0])), p_full0 = s_full0 + 24, o_done0 = s_full0 + 48;
    static_assert(offsetof(Bars, p_full) == offsetof(Bars, s_full) + 24 && offsetof(Bars, o_done) == offsetof(Bars, s_full) + 48,
                  "barrier layout");
    auto wait_pv = [&](uint32_t g) { mbar_wait_a(o_done0 + (g % C::kSBufs) * 8, (g / C::kSBufs) & 1); };
    const int32_t nk32 = int32_t(p.nk);
    TileMeta nxt = load_meta(p, tile_at<kMcast>(p, 0));
    int32_t vb_first = nxt.cnt > 0 ? block_at(p, nxt.beg, 0) : 0;
    for (int64_t it = 0, tile = tile_at<kMcast>(p, 0); tile >= 0; tile = tile_at<kMcast>(p, ++it)) {
      const int64_t h = tile / p.mq, u = tile % p.mq;
      const int32_t beg = nxt.beg, cnt = nxt.cnt;
      nxt = load_meta(p, tile_at<kMcast>(p, it + 1));
      const int64_t i_row = u * kBM + r;
      const int64_t orow = i_row < p.nq && p.out_rows ? int64_t(__ldg(p.out_rows + i_row)) : i_row;
      float m = -INFINITY;
      uint64_t lsum[2] = {0, 0};
      int32_t vb_next = vb_first;
#ifdef DFS_SYNCCHECK_BUILD
  // Unrolled, ptxas addresses the second copy's S wait as [o_done register - 0x30]: the
  // right barrier (checked in the SASS), but compute-sanitizer synccheck reports every such
  // wait as "missing init"; the sanitizer build keeps the loop rolled (same protocol).
#pragma unroll 1
#else
#pragma unroll 2
#endif
      for (int32_t j = 0; j < cnt; ++j) {
        const int32_t vb = vb_next;
        if (j + 1 < cnt) vb_next = block_at(p, beg, j + 1);
        const uint32_t sb = s_iter % C::kSBufs;
        const bool tr = threadIdx.x == DFS_TRACE_T0 || threadIdx.x == DFS_TRACE_T0 + 128;
        if (tr) trace(p, 4 + hf * 4, s_iter);
        mbar_wait_a(s_full0 + sb * 8, (s_iter / C::kSBufs) & 1);
        if (tr) trace(p, 5 + hf * 4, s_iter);
        if (lane == 0) trace(p, 25 + warp, s_iter);  // 26..33: S_j seen by softmax warp 1..8
#ifdef DFS_SYNCCHECK_BUILD
        if (threadIdx.x == 64 && s_iter >= C::kSBufs) wait_pv(s_iter - C::kSBufs);
#endif
        tc_fence_after();
#ifdef DFS_ATTN_SKIP_SOFTMAX  // experiment builds only (tools/k5_isolation.sh): the MMA/TMA side alone
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_a(p_full0 + sb * 8);
        ++s_iter;
        continue;
#endif
        uint32_t sv[64];
        const int valid = min(kBN, nk32 - vb * kBN) - ch * 64;
        auto load_s = [&]() {
          if constexpr (kLdSplit == 4) {  // four x16 loads: each chunk's consumers wait only for their own
#pragma unroll
            for (int c = 0; c < 4; ++c) tmem_ld16x2_x16<64>(tmem + lane_addr + sb * 128 + c * 16, sv + c * 16);
          } else if constexpr (kLdSplit == 2) {
            tmem_ld16x2_x32<64>(tmem + lane_addr + sb * 128, *reinterpret_cast<uint32_t(*)[32]>(sv));
            tmem_ld16x2_x32<64>(tmem + lane_addr + sb * 128 + 32, *reinterpret_cast<uint32_t(*)[32]>(sv + 32));
          } else {
            tmem_ld16x2_x64<64>(tmem + lane_addr + sb * 128, sv);
          }
          tmem_wait_ld();
          if (valid < 64) {  // padded keys of a partial last block (attention.cpp:146-152)
#pragma unroll
            for (int i = 0; i < 64; ++i)
              if (i >= valid) sv[i] = __float_as_uint(-INFINITY);
          }
        };
        load_s();
        if (tr && hf == 0) trace(p, 12, s_iter);
        // The running max m is stale by design (O is rescaled only when a block's p grow too
        // large), so the exponentials of block j need only m, not block j's own max: they
        // start right after the TMEM load, and the test runs on their results — each
        // half-row's block sum of p (kSumTest: sum <= 2^12 bounds every p; costs one FADD2
        // per block, where the max of the arguments x = s * scale - m cost one FMNMX3 per
        // pair: HY K5 -3.9 %, C -5.1 % SM cycles) — off the critical path. A block that fails
        // it (rare) takes its real row max from S, rescales O and recomputes its exponentials
        // before P is stored. The first block of a tile sets m from its own max.
        if (j == 0) {
          float mq[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
          for (int i = 0; i < 64; ++i) mq[i & 3] = fmaxf(mq[i & 3], __uint_as_float(sv[i]));
          const float mx = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3]));
          m = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16)) * p.scale_log2;  // + the row's other 64 keys
        }
        uint32_t pk[32];
        uint64_t lb[2];
        float xmax;
        auto exps = [&]() {
          const uint64_t sc2 = f2_pack(p.scale_log2, p.scale_log2), nm2 = f2_pack(-m, -m);
          lb[0] = lb[1] = 0;
          [[maybe_unused]] float xm[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            float x0, x1;
            f2_unpack(f2_fma(f2_pack(__uint_as_float(sv[2 * i]), __uint_as_float(sv[2 * i + 1])), sc2, nm2), x0, x1);
            if constexpr (!kSumTest) xm[i & 3] = fmaxf(xm[i & 3], fmaxf(x0, x1));
            float p0, p1;
            if (use_poly<POLY>(i)) {
              f2_unpack(ex2_poly2(x0, x1), p0, p1);
            } else {
              p0 = ex2(x0);
              p1 = ex2(x1);
            }
            lb[i & 1] = f2_add(lb[i & 1], f2_pack(p0, p1));
            pk[i] = pack_bf16(p0, p1);
          }
          if constexpr (kSumTest) {
            float a, b;
            f2_unpack(f2_add(lb[0], lb[1]), a, b);
            xmax = a + b;  // this half-row's block sum: bounds every p of it (p >= 0)
          } else {
            xmax = fmaxf(fmaxf(xm[0], xm[1]), fmaxf(xm[2], xm[3]));
          }
        };
        exps();
        if (j > 0) {
          bool big;
          if constexpr (kSumTest) {
            big = __any_sync(0xffffffffu, !(xmax <= kRescaleSum));  // also catches inf / NaN sums
          } else {
            xmax = fmaxf(xmax, __shfl_xor_sync(0xffffffffu, xmax, 16));  // the row's other 64 keys
            big = __any_sync(0xffffffffu, xmax > kRescaleThreshold);
          }
          if (big) {  // warp-uniform (TMEM ops below)
            if constexpr (kSumTest) {  // rare path: the block's own row max (S_j is intact in TMEM)
              load_s();
              float mq[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
              for (int i = 0; i < 64; ++i) mq[i & 3] = fmaxf(mq[i & 3], __uint_as_float(sv[i]));
              const float mx = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3]));
              xmax = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16)) * p.scale_log2 - m;
            }
            const float m_new = m + fmaxf(xmax, 0.f);
            wait_pv(s_iter - 1);  // PV_{j-1} complete: O stable
            tc_fence_after();
            const float alpha = ex2(m - m_new);
            const uint64_t a2 = f2_pack(alpha, alpha);
            lsum[0] = f2_mul(lsum[0], a2);
            lsum[1] = f2_mul(lsum[1], a2);
            m = m_new;
#pragma unroll
            for (int c = 0; c < D / 2; c += 32) {  // this thread's D/2 output columns of the row
              uint32_t ov[32];
              tmem_ld16x2_x32<D / 2>(tmem + lane_addr + C::kOCol + c, ov);
              tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
              tmem_st16x2_x32<D / 2>(tmem + lane_addr + C::kOCol + c, ov);
            }
            load_s();  // S_j is still in TMEM (P not yet stored): reload instead of keeping sv live
            exps();
          }
        }
        lsum[0] = f2_add(lsum[0], lb[0]);
        lsum[1] = f2_add(lsum[1], lb[1]);
        if (tr && hf == 0) trace(p, 14, s_iter);
        // P_j (bf16 pairs) over S columns 0-63 of the row: keys 64 ch + [0, 64) -> columns 32 ch + [0, 32)
        tmem_st16x2_x32<32>(tmem + lane_addr + sb * 128, pk);
        tmem_wait_st();
        tc_fence_before();
        if (tr) trace(p, 7 + hf * 4, s_iter);
        __syncwarp();
        if (lane == 0) {
          trace(p, 17 + warp, s_iter);  // 18..25: P_j arrival of softmax warp 1..8
          mbar_arrive_a(p_full0 + sb * 8);
        }
        ++s_iter;
      }
      vb_first = nxt.cnt > 0 ? block_at(p, nxt.beg, 0) : 0;
      float l;
      {
        float a, b;
        f2_unpack(f2_add(lsum[0], lsum[1]), a, b);
        l = a + b;
      }
      l += __shfl_xor_sync(0xffffffffu, l, 16);
      if (cnt > 0) wait_pv(s_iter - 1);
      tc_fence_after();
      const float inv_l = cnt > 0 ? 1.f / l : 0.f;
      uint32_t ov[D / 2];
      if constexpr (D == 128)
        tmem_ld16x2_x64<64>(tmem + lane_addr + C::kOCol, ov);
      else
        tmem_ld16x2_x32<32>(tmem + lane_addr + C::kOCol, ov);
      tmem_wait_ld();
      tc_fence_before();
      if (i_row < p.nq && !phantom_tile<kMcast>(p, tile)) {  // a phantom tile repeats its peer's
        __nv_bfloat16* dst;
        if constexpr (kPeerOut) {
          const int64_t nl = p.out_peers->n_local, rk = orow / nl;
          dst = static_cast<__nv_bfloat16*>(const_cast<void*>(p.out_peers->ptr[rk])) +
                ((orow - rk * nl) * p.out_peers->heads_total + p.out_peers->h0 + h) * D + ch * (D / 2);
        } else {
          dst = p.out + row_offset(p.out_layout, p.nq, p.heads, D, h, orow) + ch * (D / 2);
        }
        uint32_t w[D / 4];
#pragma unroll
        for (int c = 0; c < D / 4; ++c)
          w[c] = pack_bf16(__uint_as_float(ov[2 * c]) * inv_l, __uint_as_float(ov[2 * c + 1]) * inv_l);
        if (!kPeerOut && p.out_v8) {
#pragma unroll
          for (int q = 0; q < D / 32; ++q)
            asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst + q * 16),
                         "r"(w[8 * q + 0]), "r"(w[8 * q + 1]), "r"(w[8 * q + 2]), "r"(w[8 * q + 3]),
                         "r"(w[8 * q + 4]), "r"(w[8 * q + 5]), "r"(w[8 * q + 6]), "r"(w[8 * q + 7])
                         : "memory");
        } else {
#pragma unroll
          for (int q = 0; q < D / 16; ++q)
            *reinterpret_cast<uint4*>(dst + q * 8) = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
        }
      }
    }
  } else {
    // ============================ softmax / epilogue ============================
    // kWG warpgroups split the 128 key columns of each block (128 / kWG each); a thread
    // owns one query row (TMEM lane) of its 32-column slice.
    constexpr int kOColsPerWG = D / kWG;  // output columns per warpgroup
    const int wg = (warp - 1) >> 2;                    // key columns [kCPT*wg, kCPT*wg + kCPT)
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
    TileMeta nxt = load_meta(p, tile_at<kMcast>(p, 0));
    int32_t vb_first = nxt.cnt > 0 ? block_at(p, nxt.beg, 0) : 0;
    for (int64_t it = 0, tile = tile_at<kMcast>(p, 0); tile >= 0; tile = tile_at<kMcast>(p, ++it)) {
      const int64_t h = tile / p.mq, u = tile % p.mq;
      const int32_t beg = nxt.beg, cnt = nxt.cnt;
      nxt = load_meta(p, tile_at<kMcast>(p, it + 1));
      const int64_t i_row = u * kBM + r;  // this thread's query row, and its raster slot
      const int64_t orow = i_row < p.nq && p.out_rows ? int64_t(__ldg(p.out_rows + i_row)) : i_row;
      float m = -INFINITY;
      uint64_t lsum[2] = {0, 0};  // packed fp32x2 partial row sums (2 independent chains)
      int32_t vb_next = vb_first;
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
#ifdef DFS_SYNCCHECK_BUILD
        // sanitizer builds only (tools/sanitize.sh): observe every o_done phase once, so
        // compute-sanitizer synccheck sees no unobserved phase. S_j ready implies PV_{j-3}
        // — the previous phase of this o_done — completed (in-order tcgen05 pipe), so the
        // production kernel may leave phases unobserved: its parity waits (rescale,
        // epilogue) are never more than one phase behind. (Measured: this one extra probe
        // per block in warp 2 costs ~5 % SM cycles at HY through the row-group barrier.)
        if (threadIdx.x == 64 && s_iter >= C::kSBufs) wait_pv(s_iter - C::kSBufs);
#endif
        tc_fence_after();
#ifdef DFS_ATTN_SKIP_SOFTMAX  // experiment builds only: isolate the MMA/TMA side
        (void)red_par;
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars->p_full[sb]);
        ++s_iter;
        continue;
#endif
        uint32_t sv[kCPT];
#pragma unroll
        for (int c = 0; c < kCPT / 32; ++c)
          tmem_ld32(tmem + lane_addr + sb * 128 + wg * kCPT + c * 32, *reinterpret_cast<uint32_t(*)[32]>(sv + 32 * c));
        tmem_wait_ld();
        if (tr && wg == 0) trace(p, 12, s_iter);
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
        if (tr && wg == 0) trace(p, 13, s_iter);
        if constexpr (!kSplitO) {
          red_par[wg * kBM + r] = mx;
          named_bar_sync(bar_rows, kWG * 32);            // every slice of these rows published its max
          if (tr) trace(p, 6 + (wg & 1) * 4, s_iter);
#pragma unroll
          for (int w = 0; w < kWG; ++w) mx = fmaxf(mx, red_par[w * kBM + r]);
        }
        const float m_new = fmaxf(m, mx * p.scale_log2);
        // tcgen05.ld/st are warp-collective: the rescale decision is warp-uniform
        // (the partner warps cover the same rows, so they decide identically)
        if (j == 0) {
          m = m_new;
        } else if (__any_sync(0xffffffffu, m_new - m > kRescaleThreshold)) {
          wait_pv(s_iter - 1);                          // PV_{j-1} complete: O stable
          tc_fence_after();
          const float alpha = ex2(m - m_new);
          const uint64_t a2 = f2_pack(alpha, alpha);
          lsum[0] = f2_mul(lsum[0], a2);
          lsum[1] = f2_mul(lsum[1], a2);
          m = m_new;
          const uint32_t o_addr = tmem + lane_addr + C::kOCol + wg * (kSplitO ? D : kOColsPerWG);
          if constexpr (kSplitO) {  // this warpgroup's own O: all d columns
#pragma unroll
            for (int c = 0; c < D; c += 32) {
              uint32_t ov[32];
              tmem_ld32(o_addr + c, ov);
              tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
              tmem_st32(o_addr + c, ov);
            }
          } else if constexpr (kOColsPerWG >= 32) {
#pragma unroll
            for (int c = 0; c < kOColsPerWG; c += 32) {
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
        // (decoupled d = 64: a slice whose keys were all padding so far has m = -inf; its p = 0)
        const float m_use = kSplitO && m == -INFINITY ? 0.f : m;
        const uint64_t sc2 = f2_pack(p.scale_log2, p.scale_log2), nm2 = f2_pack(-m_use, -m_use);
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
        if (tr && wg == 0) trace(p, 14, s_iter);
        // P_j (bf16 pairs) over the first 64 columns of S[sb]: this slice's kCPT keys -> kCPT/2 columns.
        // (Decoupled d = 64: there is no exchange barrier proving the partner has loaded its
        // S columns, so each warpgroup writes P into its OWN S columns: 0-31 and 64-95.)
        constexpr int kPStride = kSplitO ? kCPT : kCPT / 2;
#pragma unroll
        for (int c = 0; c < kCPT / 32; ++c)
          tmem_st16(tmem + lane_addr + sb * 128 + wg * kPStride + c * 16,
                    *reinterpret_cast<const uint32_t(*)[16]>(pk + 16 * c));
        tmem_wait_st();
        tc_fence_before();
        if (tr) trace(p, 7 + (wg & 1) * 4, s_iter);
        __syncwarp();  // every lane's P store has completed (tcgen05.wait::st above)
        if (lane == 0) mbar_arrive(kSplitO && wg ? &bars->p_full1[sb] : &bars->p_full[sb]);
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
      float l_tot = 0.f;
      float a_w[2] = {1.f, 1.f};  // decoupled d = 64: weights of O_0, O_1 in the merged row
      if constexpr (kSplitO) {
        red_max[wg * kBM + r] = m;  // the (stale) max each slice's P and O were computed with
        red_sum[wg * kBM + r] = l;
        named_bar_sync(bar_rows, kWG * 32);
        const float m0 = red_max[r], m1 = red_max[kBM + r];
        const float mm = fmaxf(m0, m1);
        a_w[0] = m0 == -INFINITY ? 0.f : ex2(m0 - mm);
        a_w[1] = m1 == -INFINITY ? 0.f : ex2(m1 - mm);
        l_tot = a_w[0] * red_sum[r] + a_w[1] * red_sum[kBM + r];
      } else {
        red_sum[wg * kBM + r] = l;   // dedicated slots: the max slots may still be read by peers
        named_bar_sync(bar_rows, kWG * 32);
#pragma unroll
        for (int w = 0; w < kWG; ++w) l_tot += red_sum[w * kBM + r];
      }
      const int64_t i = i_row;
      // an empty key list (possible only through a caller-built CSR; the BlockMask entry
      // points refuse it like attention.cpp:133-136) yields a zero row, never stale TMEM
      const float inv_l = cnt > 0 ? 1.f / l_tot : 0.f;
      constexpr int kOC = kOColsPerWG;
      uint32_t ov[kOC];
      if constexpr (kSplitO) {  // this warpgroup's output columns of both partial rows, merged
        static_assert(kOC == 32, "decoupled epilogue: 32 output columns per warpgroup");
        uint32_t o1[32];
        tmem_ld32(tmem + lane_addr + C::kOCol + wg * kOC, *reinterpret_cast<uint32_t(*)[32]>(ov));
        tmem_ld32(tmem + lane_addr + C::kOCol + D + wg * kOC, o1);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 32; ++c)
          ov[c] = __float_as_uint(a_w[0] * __uint_as_float(ov[c]) + a_w[1] * __uint_as_float(o1[c]));
        // both warpgroups read both accumulators: neither may let the next tile's first
        // PV (which only waits for its own warpgroup's P) overwrite them before the other read
        named_bar_sync(bar_rows, kWG * 32);
      } else if constexpr (kOC >= 32) {
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
        __nv_bfloat16* dst;
        if constexpr (kPeerOut) {
          const int64_t nl = p.out_peers->n_local, r = orow / nl;
          dst = static_cast<__nv_bfloat16*>(const_cast<void*>(p.out_peers->ptr[r])) +
                ((orow - r * nl) * p.out_peers->heads_total + p.out_peers->h0 + h) * D + wg * kOC;
        } else {
          dst = p.out + row_offset(p.out_layout, p.nq, p.heads, D, h, orow) + wg * kOC;
        }
        // 32-byte stores (STG.256): half the store instructions of 16-byte ones; the store
        // issue at the tile boundary is what holds the warps there
        uint32_t w[kOC / 2];
#pragma unroll
        for (int c = 0; c < kOC / 2; ++c)
          w[c] = pack_bf16(__uint_as_float(ov[2 * c]) * inv_l, __uint_as_float(ov[2 * c + 1]) * inv_l);
        if (!kPeerOut && p.out_v8) {
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
  if constexpr (kMcast) cluster_sync();  // no CTA leaves while its peer may still signal or fill it
  if (warp == kMmaWarp) tmem_dealloc<kTmemCols>(tmem);
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
int make_map(CUtensorMap* map, const void* base, int layout, int64_t n, int64_t heads, int64_t d,
             int box_rows = 128) {
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
    box[1] = cuuint32_t(box_rows);
    box[2] = 1;
  } else {  // [N, H, d]: dims (d, H, N), box (64, 1, 128)
    dims[0] = cuuint64_t(d);
    dims[1] = cuuint64_t(heads);
    dims[2] = cuuint64_t(n);
    strides[0] = cuuint64_t(d) * 2;
    strides[1] = cuuint64_t(heads) * cuuint64_t(d) * 2;
    box[0] = 64;
    box[1] = 1;
    box[2] = cuuint32_t(box_rows);
  }
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DFS_E_CUDA, "cuTensorMapEncodeTiled failed");
  return DFS_OK;
}

// 2D map over rows x d bf16 for tile::gather4: box {64 columns, 1 row}, SWIZZLE_128B
int make_gather_map(CUtensorMap* map, const void* base, int64_t rows, int64_t d) {
  EncodeFn enc = get_encode();
  if (!enc) return fail(DFS_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  if (rows >= (int64_t(1) << 31)) return fail(DFS_E_UNSUPPORTED, "attn_sm100: N*H too large for row gather");
  cuuint64_t dims[2] = {cuuint64_t(d), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(d) * 2};
  cuuint32_t box[2] = {64, 1}, estr[2] = {1, 1};
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DFS_E_CUDA, "cuTensorMapEncodeTiled (gather) failed");
  return DFS_OK;
}

// dense steps (full key list): 2-CTA clusters with K/V tiles multicast into both CTAs
#ifndef DFS_ATTN_MCAST
#define DFS_ATTN_MCAST 1
#endif

template <int D, int POLY, bool kPeerOut = false>
int launch_kernel(const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv, const Params& p,
                  cudaStream_t stream) {
  using C = Cfg<D>;
  if (DFS_ATTN_MCAST && !kPeerOut && !p.blk_ptr && kWG == 2 && DFS_ATTN_ROWSPLIT) {
    auto* kfn = attn_sm100_kernel<D, POLY, kPeerOut, true>;
    DFS_CUDA_CHECK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
    const int64_t pairs = p.heads * ((p.mq + 1) / 2);
    const int64_t grid = 2 * (pairs < kNumSMs / 2 ? pairs : kNumSMs / 2);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(grid));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = C::kSmem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    DFS_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kfn, mq, mk, mv, p));
    DFS_LAUNCH_CHECK("attn_sm100 (dense, multicast)");
    return DFS_OK;
  }
  // per device and race-free: set on every launch (~1 us)
  DFS_CUDA_CHECK(cudaFuncSetAttribute(attn_sm100_kernel<D, POLY, kPeerOut, false>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
  const int64_t grid = p.tiles < kNumSMs ? p.tiles : kNumSMs;
  attn_sm100_kernel<D, POLY, kPeerOut, false><<<unsigned(grid), kThreads, C::kSmem, stream>>>(mq, mk, mv, p);
  DFS_LAUNCH_CHECK("attn_sm100");
  return DFS_OK;
}

// exp2 split between MUFU and the FMA-pipe polynomial (use_poly), measured with
// tools/poly_sweep.sh (K5 SM cycles, degree-2 polynomial, row-split kernel with the block loop
// unrolled by 2): d = 128 runs every 3rd pair (33 %): HY -1.8 % vs pairs 1, 4, 7, 10, 13 of 16
// (which had won by 4 % before the unroll), -2.1 % vs 1, 4, 7 of every 8; d = 64 keeps 1, 4, 7
// of every 8 (every 3rd +3 %, 5 of 16 +1 %, every 2nd +11 %). The placement in the compiler's
// schedule matters as much as the ratio. DFS_ATTN_POLY overrides the default for A/B runs.
template <int D>
constexpr int kDefaultPoly = D == 128 ? 3 : 38;

template <int D>
int launch(const dfs_attn_args& a, float scale, cudaStream_t stream) {
  CUtensorMap mq, mk, mv;
  int rc;
  if (a.in_rows) {  // Q: 2D row-gather map over the raster [N*H, d] activations
    if ((rc = make_gather_map(&mq, a.q, a.nq * a.heads, D))) return rc;
  } else if ((rc = make_map(&mq, a.q, a.in_layout, a.nq, a.heads, D))) {
    return rc;
  }
  if ((rc = make_map(&mk, a.k, a.in_layout, a.nk, a.heads, D))) return rc;
  if ((rc = make_map(&mv, a.v, a.in_layout, a.nk, a.heads, D))) return rc;
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
  p.out_peers = static_cast<const dfs_peer_table*>(a.out_peers);
  p.out_v8 = !a.out_peers && (reinterpret_cast<uintptr_t>(a.o) & 31) == 0;  // peer shards: 16-byte stores
  p.in_nhd = a.in_layout == DFS_NHD;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.in_rows = a.in_rows;
  p.tiles = p.mq * a.heads;
  p.trace = nullptr;
#ifdef DFS_ATTN_TRACE_BUILD
  const char* trace_path = getenv("DFS_ATTN_TRACE");
  if (trace_path) DFS_CUDA_CHECK(cudaMalloc(&p.trace, 40 * 256 * sizeof(unsigned long long)));
  if (p.trace) DFS_CUDA_CHECK(cudaMemsetAsync(p.trace, 0, 40 * 256 * sizeof(unsigned long long), stream));
#endif
  static const int poly = getenv("DFS_ATTN_POLY") ? atoi(getenv("DFS_ATTN_POLY")) : kDefaultPoly<D>;
  // a trajectory runs dense (multicast) and sparse steps: load both kernels on the first call,
  // not inside the first step that needs the other one (lazy module loading costs ~ms)
  static const bool loaded = [] {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, attn_sm100_kernel<D, kDefaultPoly<D>, false, false>);
    cudaFuncGetAttributes(&fa, attn_sm100_kernel<D, kDefaultPoly<D>, false, true>);
    return true;
  }();
  (void)loaded;
  if (a.out_peers) {  // Ulysses: the epilogue stores into the token owners' shards
    rc = launch_kernel<D, kDefaultPoly<D>, true>(mq, mk, mv, p, stream);
  } else {
    switch (poly) {
      case 0: rc = launch_kernel<D, 0>(mq, mk, mv, p, stream); break;
      case 2: rc = launch_kernel<D, 2>(mq, mk, mv, p, stream); break;
      case 3: rc = launch_kernel<D, 3>(mq, mk, mv, p, stream); break;
      case 38: rc = launch_kernel<D, 38>(mq, mk, mv, p, stream); break;
      case 516: rc = launch_kernel<D, 516>(mq, mk, mv, p, stream); break;
      default: rc = launch_kernel<D, 4>(mq, mk, mv, p, stream); break;
    }
  }
  if (rc) return rc;
#ifdef DFS_ATTN_TRACE_BUILD
  if (p.trace) {
    unsigned long long host[40 * 256];
    DFS_CUDA_CHECK(cudaMemcpyAsync(host, p.trace, sizeof(host), cudaMemcpyDeviceToHost, stream));
    DFS_CUDA_CHECK(cudaStreamSynchronize(stream));
    if (FILE* f = fopen(trace_path, "wb")) {
      fwrite(host, sizeof(host), 1, f);
      fclose(f);
    }
    cudaFree(p.trace);
  }
#endif
  return DFS_OK;
}

}  // namespace

// bf16 token-tensor maps shared with the recall kernel (recall_sm100.cu) and the B = 64
// attention kernel (attn_b64.cu)
int make_token_map(CUtensorMap* map, const void* base, int layout, int64_t n, int64_t heads, int64_t d) {
  return make_map(map, base, layout, n, heads, d);
}
int make_token_map_rows(CUtensorMap* map, const void* base, int layout, int64_t n, int64_t heads, int64_t d,
                        int box_rows) {
  return make_map(map, base, layout, n, heads, d, box_rows);
}
int make_row_gather_map(CUtensorMap* map, const void* base, int64_t rows, int64_t d) {
  return make_gather_map(map, base, rows, d);
}

// [H, rows, d] fp16 operand map for the scorer (score_sm100.cu): box 64 x box_rows x 1, SW128
int make_map_f16(CUtensorMap* map, const void* base, int64_t rows, int64_t heads, int64_t d, int box_rows) {
  EncodeFn enc = get_encode();
  if (!enc) return fail(DFS_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {cuuint64_t(d), cuuint64_t(rows), cuuint64_t(heads)};
  cuuint64_t strides[2] = {cuuint64_t(d) * 2, cuuint64_t(rows) * cuuint64_t(d) * 2};
  cuuint32_t box[3] = {64, cuuint32_t(box_rows), 1}, estr[3] = {1, 1, 1};
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DFS_E_CUDA, "cuTensorMapEncodeTiled (f16) failed");
  return DFS_OK;
}

bool attn_sm100_supports(const dfs_attn_args& a) {
  if (a.dtype != DFS_BF16 || (a.block != 128 && a.block != 64) || (a.d != 64 && a.d != 128)) return false;
  if (a.dv > 0 && a.dv != a.d) return false;
  if (a.in_rows && a.nq >= (int64_t(1) << 31) / a.heads) return false;
  const void* ptrs[4] = {a.q, a.k, a.v, a.o};
  for (const void* ptr : ptrs)
    if (reinterpret_cast<uintptr_t>(ptr) & 15) return false;
  if (a.nq >= (int64_t(1) << 31) || a.nk >= (int64_t(1) << 31)) return false;
  return true;
}

int sparse_attn_b64(const dfs_attn_args& a, float scale, cudaStream_t stream);  // attn_b64.cu

int sparse_attn_sm100(const dfs_attn_args& a, float scale, cudaStream_t stream) {
  if (a.block == 64) {
    if (a.out_peers) return fail(DFS_E_UNSUPPORTED, "attn_sm100: peer-scattered output needs B = 128");
    return sparse_attn_b64(a, scale, stream);
  }
  if (a.block != 128) return fail(DFS_E_UNSUPPORTED, "attn_sm100: block must be 64 or 128");
  if (a.d == 128) return launch<128>(a, scale, stream);
  if (a.d == 64) return launch<64>(a, scale, stream);
  return fail(DFS_E_UNSUPPORTED, "attn_sm100: d must be 64 or 128");
}

}  // namespace dfsgpu
