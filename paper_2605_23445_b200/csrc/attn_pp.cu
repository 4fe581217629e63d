// attn_pp.cu — K5, two query tiles per CTA in ping-pong: block_sparse_attention
// (attention.cpp:125-159) for B = 128, d in {64, 128}, bf16 I/O, fp32 softmax and accumulation.
//
// Why a second K5 design. In attn_sm100.cu one query tile per CTA is split over two softmax
// warps per SMSP that work on the SAME key block at the same time: their serial phases (S wait,
// TMEM loads, P store, loop overhead) coincide, and the S buffers chain block j + 2's scores to
// the last warp's P_j through PV_j + QK_{j+2} (traced: ~1.6k cycles), so the loop runs at
// ~1.5k cycles per block for 1024 tensor cycles. Here a CTA owns TWO tiles (streams A and B,
// different query blocks, each with its own key-block list); each stream has one S and one O
// buffer in TMEM and one softmax warpgroup with one thread per query row (128 logits per
// thread per block). The MMA warp alternates the streams — PV_A(k), QK_A(k+1), PV_B(k),
// QK_B(k+1) — so A's softmax runs under B's MMAs and vice versa, and the two softmax warps
// sharing an SMSP are out of phase by construction (the FA4 / cuDNN forward structure).
//
// Warps (320 threads):
//   0     TMA producer: Q_A / Q_B tiles (gather4 of raster rows when the reorder is fused) and
//         one K/V ring in the MMA warp's consumption order.
//   1-4   softmax + epilogue of stream A (TMEM lane quadrant warp & 3, one thread per row)
//   5-8   softmax + epilogue of stream B
//   9     MMA issuer (one elected lane)
// TMEM (512 columns): S_A/P_A [0,128) O_A [128,128+D) S_B/P_B [256,384) O_B [384,384+D).
// Shared memory: Q_A, Q_B, the K/V ring (SWIZZLE_128B 128 x 64 boxes), barriers.
//
// Softmax (per thread = query row, per block): the running max m is stale by design — O is
// rescaled only when a block raises the row max by more than kRescaleLog2 — so the
// exponentials need only m; the first block of a tile takes its max in a separate pass. The
// 128 logits are loaded from TMEM in four 32-column chunks (the next chunk's load in flight
// while the current one is exponentiated); exp2 is split between MUFU and a degree-2 FMA-pipe
// polynomial; P (bf16) is written over S only after the threshold test, so a block that
// crosses it (rare) reloads S, rescales O (S_j ready implies PV_{j-1} completed: the stream
// has one S buffer and QK_j is issued after PV_{j-1}) and recomputes.
#include <cuda.h>

#include <cstddef>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "sm100.cuh"

namespace dfsgpu {

int make_token_map(CUtensorMap* map, const void* base, int layout, int64_t n, int64_t heads, int64_t d);
int make_row_gather_map(CUtensorMap* map, const void* base, int64_t rows, int64_t d);

namespace {

using namespace sm100;

constexpr int kBM = 128;
constexpr int kBN = 128;
constexpr int kThreads = 320;
constexpr int kMmaWarp = 9;
constexpr float kRescaleLog2 = 8.0f;

template <int D>
struct PCfg {
  static constexpr int kChunks = D / 64;             // 128-byte swizzle chunks per row
  static constexpr int kTileBytes = kBM * D * 2;
  static constexpr int kChunkBytes = kBM * 128;
  static constexpr int kStages = D == 64 ? 12 : 5;
  static constexpr int kQOff = 0;                    // Q_A, Q_B
  static constexpr int kRingOff = 2 * kTileBytes;
  static constexpr int kBarOff = kRingOff + kStages * kTileBytes;
  static constexpr int kSmem = kBarOff + 512 + 1024;
  static constexpr uint32_t kIdescQK = idesc_bf16_f32(kBM, kBN, false, false);
  static constexpr uint32_t kIdescPV = idesc_bf16_f32(kBM, D, false, true);
};

struct PParams {
  int64_t heads, nq, nk, mq, mk, tiles;
  const int32_t* blk_ptr;  // NULL = dense
  const int32_t* blk_idx;
  const uint32_t* out_rows;
  const uint32_t* in_rows;
  __nv_bfloat16* out;
  int out_layout, out_v8, in_nhd;
  float scale_log2;
  const dfs_peer_table* out_peers;
  unsigned long long* trace;  // DFS_ATTN_TRACE_BUILD: per-block timeline of CTA 0
};

#ifdef DFS_ATTN_TRACE_BUILD
__device__ __forceinline__ void ptrace(const PParams& p, int ev, uint32_t idx) {
  if (p.trace && blockIdx.x == 0 && idx < 256) p.trace[ev * 256 + idx] = clock64();
}
#else
__device__ __forceinline__ void ptrace(const PParams&, int, uint32_t) {}
#endif

struct PBars {
  uint64_t q_full[2], q_empty[2], s_full[2], p_full[2], o_done[2];
  uint64_t kv_full[12], kv_empty[12];
  uint32_t tmem_base;
};

struct Meta {
  int32_t beg, cnt;
};
__device__ __forceinline__ Meta tile_meta(const PParams& p, int64_t tile) {
  Meta t{0, 0};
  if (tile < p.tiles) {
    if (p.blk_ptr) {
      t.beg = __ldg(p.blk_ptr + tile);
      t.cnt = __ldg(p.blk_ptr + tile + 1) - t.beg;
    } else {
      t.cnt = int32_t(p.mk);
    }
  }
  return t;
}

// A stream's blocks as one flat sequence over its tiles (tile0, tile0 + 2G, ...), skipping
// tiles with an empty list; used identically by the producer and the MMA warp so both
// agree on the consumption order.
struct Cursor {
  int64_t tile, stride;
  int32_t beg, cnt, j;
  int32_t win = -64, lut = 0;  // producer: list entries [win, win + 32) held one per lane
  bool live;
  __device__ __forceinline__ void seek(const PParams& p) {  // to the first non-empty tile from `tile`
    while (tile < p.tiles) {
      const Meta m = tile_meta(p, tile);
      if (m.cnt > 0) {
        beg = m.beg;
        cnt = m.cnt;
        j = 0;
        win = -64;
        live = true;
        return;
      }
      tile += stride;
    }
    live = false;
  }
  __device__ __forceinline__ void init(const PParams& p, int64_t t0, int64_t st) {
    tile = t0;
    stride = st;
    seek(p);
  }
  __device__ __forceinline__ void advance(const PParams& p) {
    if (++j < cnt) return;
    tile += stride;
    seek(p);
  }
  // key block of entry j, read 32 entries per coalesced warp load and broadcast by shuffle
  // (warp-collective: the whole producer warp runs the cursor)
  __device__ __forceinline__ int32_t block(const PParams& p, int lane) {
    if (!p.blk_ptr) return j;
    const int32_t w = j & ~31;
    if (w != win) {
      win = w;
      lut = (w + lane < cnt) ? __ldg(p.blk_idx + beg + w + lane) : 0;
    }
    return __shfl_sync(0xffffffffu, lut, j & 31);
  }
};

template <int POLY>
__device__ __forceinline__ constexpr bool poly_pair(int i) {
  if constexpr (POLY == 38) return (0x92u >> (i % 8)) & 1u;  // pairs 1, 4, 7 of each 8
  else if constexpr (POLY == 0) return false;
  else return i % POLY == POLY - 1;
}

// tcgen05.wait::ld that also "defines" the registers of a load still in flight, so the
// compiler cannot hoist their uses above the wait
__device__ __forceinline__ void wait_ld_into(uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.wait::ld.sync.aligned;"
      : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
        "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15]),
        "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]), "+r"(r[22]), "+r"(r[23]),
        "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]), "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
      :
      : "memory");
}

template <int D, int POLY, bool kPeerOut>
__global__ void __launch_bounds__(kThreads, 1)
    attn_pp_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                   const __grid_constant__ CUtensorMap tm_v, const PParams p) {
  using C = PCfg<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sRing = smem + C::kRingOff;
  PBars* bars = reinterpret_cast<PBars*>(smem + C::kBarOff);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t G = gridDim.x;

  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bars->q_full[s], 1);
      mbar_init(&bars->q_empty[s], 1);
      mbar_init(&bars->s_full[s], 1);
      mbar_init(&bars->p_full[s], 4);  // one arrive per softmax warp of the stream
      mbar_init(&bars->o_done[s], 1);
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
  if (warp == kMmaWarp) tmem_alloc<512>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  if (warp == 0) {
    // ================================ TMA producer ==============================
    uint32_t ring = 0, q_use[2] = {0, 0};
    auto load_kv = [&](const CUtensorMap* map, int64_t h, int64_t row0) {
      const uint32_t slot = ring % C::kStages;
      mbar_wait(&bars->kv_empty[slot], ((ring / C::kStages) & 1) ^ 1);
      if (elect_one()) {
        mbar_expect_tx(&bars->kv_full[slot], C::kTileBytes);
#pragma unroll
        for (int c = 0; c < C::kChunks; ++c)
          tma_load_3d(sRing + slot * C::kTileBytes + c * C::kChunkBytes, map, &bars->kv_full[slot], c * 64,
                      p.in_nhd ? int(h) : int(row0), p.in_nhd ? int(row0) : int(h));
      }
      __syncwarp();
      ++ring;
    };
    auto load_q = [&](int s, int64_t tile) {  // Q of the stream's new tile
      const int64_t h = tile / p.mq, row0 = (tile % p.mq) * kBM;
      uint8_t* dst = smem + C::kQOff + s * C::kTileBytes;
      int rr[4] = {0, 0, 0, 0};
      if (p.in_rows) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          int64_t i = row0 + 4 * lane + k;
          i = i < p.nq ? i : p.nq - 1;
          rr[k] = int(int64_t(__ldg(p.in_rows + i)) * p.heads + h);
        }
      }
      mbar_wait(&bars->q_empty[s], (q_use[s] & 1) ^ 1);
      ++q_use[s];
      if (p.in_rows) {
        if (elect_one()) mbar_expect_tx(&bars->q_full[s], C::kTileBytes);
        __syncwarp();
#pragma unroll
        for (int c = 0; c < C::kChunks; ++c)
          tma_gather4(dst + c * C::kChunkBytes + lane * 512, &tm_q, &bars->q_full[s], c * 64, rr[0], rr[1], rr[2],
                      rr[3]);
      } else if (elect_one()) {
        mbar_expect_tx(&bars->q_full[s], C::kTileBytes);
#pragma unroll
        for (int c = 0; c < C::kChunks; ++c)
          tma_load_3d(dst + c * C::kChunkBytes, &tm_q, &bars->q_full[s], c * 64, p.in_nhd ? int(h) : int(row0),
                      p.in_nhd ? int(row0) : int(h));
      }
      __syncwarp();
    };
    Cursor kc[2], vc[2];
    for (int s = 0; s < 2; ++s) {
      kc[s].init(p, blockIdx.x + s * G, 2 * G);
      vc[s] = kc[s];
    }
    auto load_k = [&](int s) {
      Cursor& c = kc[s];
      if (c.j == 0) load_q(s, c.tile);
      load_kv(&tm_k, c.tile / p.mq, int64_t(c.block(p, lane)) * kBN);
      c.advance(p);
    };
    for (int s = 0; s < 2; ++s)
      if (kc[s].live) load_k(s);
    while (vc[0].live || vc[1].live) {
      for (int s = 0; s < 2; ++s) {
        if (vc[s].live) {
          load_kv(&tm_v, vc[s].tile / p.mq, int64_t(vc[s].block(p, lane)) * kBN);
          vc[s].advance(p);
        }
        if (kc[s].live) load_k(s);
      }
    }
  } else if (warp == kMmaWarp) {
    // ================================ MMA issuer ================================
    uint32_t ring = 0, q_use[2] = {0, 0}, blk[2] = {0, 0}, pv_blk[2] = {0, 0};
    constexpr uint32_t kHiK = desc_sw128_hi(1024);
    const uint32_t ring_lo = desc_sw128_lo(smem_u32(sRing), 16);
    const uint32_t ring_lo_v = desc_sw128_lo(smem_u32(sRing), C::kChunkBytes);
    auto next_slot = [&]() -> uint32_t {
      const uint32_t slot = ring % C::kStages;
      mbar_wait(&bars->kv_full[slot], (ring / C::kStages) & 1);
      ++ring;
      return slot;
    };
    Cursor kc[2], vc[2];
    for (int s = 0; s < 2; ++s) {
      kc[s].init(p, blockIdx.x + s * G, 2 * G);
      vc[s] = kc[s];
    }
    auto issue_qk = [&](int s) {  // S_s = Q_s K^T (S_s free: PV of the previous block issued before)
      Cursor& c = kc[s];
      if (c.j == 0) {
        mbar_wait(&bars->q_full[s], q_use[s] & 1);
        ++q_use[s];
      }
      const uint32_t slot = next_slot();
      tc_fence_after();
      const uint32_t q_lo = desc_sw128_lo(smem_u32(smem + C::kQOff + s * C::kTileBytes), 16);
      const uint32_t k_lo = ring_lo + slot * (C::kTileBytes >> 4);
      if (elect_one()) {
#pragma unroll
        for (int st = 0; st < D / 16; ++st) {
          const uint32_t off = ((st >> 2) * C::kChunkBytes + (st & 3) * 32) >> 4;
          umma_ss(tmem + s * 256, q_lo + off, kHiK, k_lo + off, kHiK, C::kIdescQK, st > 0);
        }
        umma_commit(&bars->kv_empty[slot]);
        umma_commit(&bars->s_full[s]);
        if (c.j + 1 == c.cnt) umma_commit(&bars->q_empty[s]);  // the tile's last QK read Q_s
      }
      __syncwarp();
      ptrace(p, 4 + s, blk[s]);
      ++blk[s];
      c.advance(p);
    };
    auto issue_pv = [&](int s) {  // O_s (+)= P_s V
      Cursor& c = vc[s];
      const uint32_t slot = next_slot();
      ptrace(p, 6 + s, pv_blk[s]);
      mbar_wait(&bars->p_full[s], pv_blk[s] & 1);
      ptrace(p, 0 + s, pv_blk[s]);
      tc_fence_after();
      const uint32_t v_lo = ring_lo_v + slot * (C::kTileBytes >> 4);
      const bool first = c.j == 0;
      if (elect_one()) {
#pragma unroll
        for (int st = 0; st < kBN / 16; ++st)
          umma_ts(tmem + s * 256 + 128, tmem + s * 256 + st * 8, v_lo + ((st * 16 * 128) >> 4), kHiK, C::kIdescPV,
                  (!first || st > 0) ? 1u : 0u);
        umma_commit(&bars->kv_empty[slot]);
        umma_commit(&bars->o_done[s]);
      }
      __syncwarp();
      ptrace(p, 2 + s, pv_blk[s]);
      ++pv_blk[s];
      c.advance(p);
    };
    for (int s = 0; s < 2; ++s)
      if (kc[s].live) issue_qk(s);
    while (vc[0].live || vc[1].live) {
      for (int s = 0; s < 2; ++s) {
        if (vc[s].live) issue_pv(s);
        if (kc[s].live) issue_qk(s);
      }
    }
  } else {
    // ============================ softmax / epilogue ============================
    const int s = (warp - 1) >> 2;                // stream
    const int r = (warp & 3) * 32 + lane;         // query row within the tile == TMEM lane
    const uint32_t lane_addr = uint32_t((warp & 3) * 32) << 16;
    const uint32_t s_tm = tmem + lane_addr + s * 256, o_tm = s_tm + 128;
    const uint32_t s_full = pin_u32(smem_u32(&bars->s_full[s])), p_full = s_full + 16,
                   o_done = s_full + 32;
    static_assert(offsetof(PBars, p_full) == offsetof(PBars, s_full) + 16 &&
                      offsetof(PBars, o_done) == offsetof(PBars, s_full) + 32,
                  "barrier layout");
    const int32_t nk32 = int32_t(p.nk), mk32 = int32_t(p.mk);
    uint32_t g = 0;  // blocks of this stream so far
    for (int64_t tile = blockIdx.x + s * G; tile < p.tiles; tile += 2 * G) {
      const Meta mt = tile_meta(p, tile);
      const int64_t h = tile / p.mq, u = tile % p.mq;
      const int64_t i_row = u * kBM + r;
      const int64_t orow = i_row < p.nq && p.out_rows ? int64_t(__ldg(p.out_rows + i_row)) : i_row;
      float m = -INFINITY;
      uint64_t lsum[2] = {0, 0};
      int32_t vb_next = mt.cnt > 0 ? (p.blk_ptr ? __ldg(p.blk_idx + mt.beg) : 0) : 0;
      for (int32_t j = 0; j < mt.cnt; ++j) {
        const int32_t vb = vb_next;
        if (j + 1 < mt.cnt) vb_next = p.blk_ptr ? __ldg(p.blk_idx + mt.beg + j + 1) : j + 1;
        // keys of a partial last block are padding (attention.cpp:146-152)
        const int valid = vb == mk32 - 1 ? nk32 - vb * kBN : kBN;
        const bool tr = lane == 0 && (warp == 1 || warp == 5);
        if (tr) ptrace(p, 8 + s, g);
        mbar_wait_a(s_full, g & 1);
        if (tr) ptrace(p, 10 + s, g);
        tc_fence_after();
        uint32_t ca[32], cb[32];
        auto mask = [&](uint32_t(&v)[32], int c) {
          if (valid < kBN) {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (32 * c + i >= valid) v[i] = __float_as_uint(-INFINITY);
          }
        };
        if (j == 0) {  // the tile's first block sets m from its own max
          float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            tmem_ld32(s_tm + 32 * c, ca);
            tmem_wait_ld();
            mask(ca, c);
#pragma unroll
            for (int i = 0; i < 32; ++i) mx[i & 3] = fmaxf(mx[i & 3], __uint_as_float(ca[i]));
          }
          m = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])) * p.scale_log2;
        }
        uint32_t pk[64];
        uint64_t lb[2];
        float xmax;
        auto exps = [&]() {  // pk, lb, xmax from S (four chunks, one load in flight)
          const uint64_t sc2 = f2_pack(p.scale_log2, p.scale_log2), nm2 = f2_pack(-m, -m);
          lb[0] = lb[1] = 0;
          float xm[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
          tmem_ld32(s_tm, ca);
          tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t(&cur)[32] = (c & 1) ? cb : ca;
            uint32_t(&nxt)[32] = (c & 1) ? ca : cb;
            if (c < 3) tmem_ld32(s_tm + 32 * (c + 1), nxt);
            mask(cur, c);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              float x0, x1;
              f2_unpack(f2_fma(f2_pack(__uint_as_float(cur[2 * i]), __uint_as_float(cur[2 * i + 1])), sc2, nm2), x0,
                        x1);
              xm[i & 3] = fmaxf(xm[i & 3], fmaxf(x0, x1));
              float p0, p1;
              if (poly_pair<POLY>(16 * c + i)) {
                f2_unpack(ex2_poly2(x0, x1), p0, p1);
              } else {
                p0 = ex2(x0);
                p1 = ex2(x1);
              }
              lb[i & 1] = f2_add(lb[i & 1], f2_pack(p0, p1));
              pk[16 * c + i] = pack_bf16(p0, p1);
            }
            if (c < 3) wait_ld_into(nxt);
          }
          xmax = fmaxf(fmaxf(xm[0], xm[1]), fmaxf(xm[2], xm[3]));
        };
        exps();
        if (j > 0 && __any_sync(0xffffffffu, xmax > kRescaleLog2)) {
          // S_j ready => QK_j done => PV_{j-1} (issued before it) done: O is stable
          const float m_new = m + fmaxf(xmax, 0.f);
          const float alpha = ex2(m - m_new);
          const uint64_t a2 = f2_pack(alpha, alpha);
          lsum[0] = f2_mul(lsum[0], a2);
          lsum[1] = f2_mul(lsum[1], a2);
          m = m_new;
#pragma unroll
          for (int c = 0; c < D; c += 32) {
            uint32_t ov[32];
            tmem_ld32(o_tm + c, ov);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
            tmem_st32(o_tm + c, ov);
          }
          exps();  // S_j is intact: P is written only below
        }
        lsum[0] = f2_add(lsum[0], lb[0]);
        lsum[1] = f2_add(lsum[1], lb[1]);
        if (tr) ptrace(p, 12 + s, g);
        // P_j (bf16 pairs) over S_j's first 64 columns
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_st16(s_tm + 16 * c, *reinterpret_cast<const uint32_t(*)[16]>(pk + 16 * c));
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_a(p_full);
        if (tr) ptrace(p, 14 + s, g);
        ++g;
      }
      // epilogue: wait for the tile's last PV, normalise, store the row at its raster slot
      float l;
      {
        float a, b;
        f2_unpack(f2_add(lsum[0], lsum[1]), a, b);
        l = a + b;
      }
      if (mt.cnt > 0) mbar_wait_a(o_done, (g - 1) & 1);
      tc_fence_after();
      const float inv_l = mt.cnt > 0 ? 1.f / l : 0.f;
      __nv_bfloat16* dst = nullptr;
      if (i_row < p.nq) {
        if constexpr (kPeerOut) {
          const int64_t nl = p.out_peers->n_local, rk = orow / nl;
          dst = static_cast<__nv_bfloat16*>(const_cast<void*>(p.out_peers->ptr[rk])) +
                ((orow - rk * nl) * p.out_peers->heads_total + p.out_peers->h0 + h) * D;
        } else {
          dst = p.out + row_offset(p.out_layout, p.nq, p.heads, D, h, orow);
        }
      }
#pragma unroll
      for (int c = 0; c < D; c += 32) {
        uint32_t ov[32];
        tmem_ld32(o_tm + c, ov);
        tmem_wait_ld();
        uint32_t w[16];
#pragma unroll
        for (int q = 0; q < 16; ++q)  // an empty key list yields a zero row, never stale TMEM
          w[q] = mt.cnt > 0 ? pack_bf16(__uint_as_float(ov[2 * q]) * inv_l, __uint_as_float(ov[2 * q + 1]) * inv_l) : 0u;
        if (dst) {
          if (!kPeerOut && p.out_v8) {
#pragma unroll
            for (int q = 0; q < 2; ++q)
              asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst + c + q * 16),
                           "r"(w[8 * q + 0]), "r"(w[8 * q + 1]), "r"(w[8 * q + 2]), "r"(w[8 * q + 3]),
                           "r"(w[8 * q + 4]), "r"(w[8 * q + 5]), "r"(w[8 * q + 6]), "r"(w[8 * q + 7])
                           : "memory");
          } else {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              *reinterpret_cast<uint4*>(dst + c + q * 8) = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
          }
        }
      }
      tc_fence_before();
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == kMmaWarp) tmem_dealloc<512>(tmem);
}

template <int D, bool kPeerOut>
int launch_pp(const dfs_attn_args& a, float scale, cudaStream_t stream) {
  using C = PCfg<D>;
  CUtensorMap mq, mk, mv;
  int rc;
  if (a.in_rows) {
    if ((rc = make_row_gather_map(&mq, a.q, a.nq * a.heads, D))) return rc;
  } else if ((rc = make_token_map(&mq, a.q, a.in_layout, a.nq, a.heads, D))) {
    return rc;
  }
  if ((rc = make_token_map(&mk, a.k, a.in_layout, a.nk, a.heads, D))) return rc;
  if ((rc = make_token_map(&mv, a.v, a.in_layout, a.nk, a.heads, D))) return rc;
  PParams p;
  p.heads = a.heads;
  p.nq = a.nq;
  p.nk = a.nk;
  p.mq = ceil_div(a.nq, kBM);
  p.mk = ceil_div(a.nk, kBN);
  p.tiles = p.mq * a.heads;
  p.blk_ptr = a.blk_ptr;
  p.blk_idx = a.blk_idx;
  p.out_rows = a.out_rows;
  p.in_rows = a.in_rows;
  p.out = static_cast<__nv_bfloat16*>(a.o);
  p.out_layout = a.out_layout;
  p.out_v8 = !a.out_peers && (reinterpret_cast<uintptr_t>(a.o) & 31) == 0;
  p.in_nhd = a.in_layout == DFS_NHD;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.out_peers = static_cast<const dfs_peer_table*>(a.out_peers);
  p.trace = nullptr;
#ifdef DFS_ATTN_TRACE_BUILD
  const char* trace_path = getenv("DFS_ATTN_TRACE");
  if (trace_path) {
    DFS_CUDA_CHECK(cudaMalloc(&p.trace, 16 * 256 * sizeof(unsigned long long)));
    DFS_CUDA_CHECK(cudaMemsetAsync(p.trace, 0, 16 * 256 * sizeof(unsigned long long), stream));
  }
#endif
  auto kern = attn_pp_kernel<D, 38, kPeerOut>;
  DFS_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
  // two tiles per CTA: at most ceil(tiles / 2) CTAs
  const int64_t grid = (p.tiles + 1) / 2 < kNumSMs ? (p.tiles + 1) / 2 : kNumSMs;
  kern<<<unsigned(grid), kThreads, C::kSmem, stream>>>(mq, mk, mv, p);
  DFS_LAUNCH_CHECK("attn_pp");
#ifdef DFS_ATTN_TRACE_BUILD
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
#endif
  return DFS_OK;
}

}  // namespace

// B = 128, d in {64, 128} (attn_sm100_supports() has checked alignment and sizes)
int sparse_attn_pp(const dfs_attn_args& a, float scale, cudaStream_t stream) {
  if (a.block != 128) return fail(DFS_E_UNSUPPORTED, "attn_pp: block must be 128");
  if (a.d == 128) return a.out_peers ? launch_pp<128, true>(a, scale, stream) : launch_pp<128, false>(a, scale, stream);
  if (a.d == 64) return a.out_peers ? launch_pp<64, true>(a, scale, stream) : launch_pp<64, false>(a, scale, stream);
  return fail(DFS_E_UNSUPPORTED, "attn_pp: d must be 64 or 128");
}

}  // namespace dfsgpu
