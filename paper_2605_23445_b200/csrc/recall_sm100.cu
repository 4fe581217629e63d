// recall_sm100.cu — attention recall of a block mask without the N x N matrix.
//
// attention_recall (attention.cpp:175-190) of attention_scores (attention.cpp:105-123)
// under a BlockMask: recall = sum |A o M| / sum |A|, A = row-softmax(q k^T / sqrt(d)).
// The reference materialises A and refuses N > 4096 (attention.hpp:10); run_step
// records recall only below that cap (scheduler.cpp:129-131). Rows of A sum to 1,
// so recall = (1/N) sum_rows (softmax mass of the row inside its selected blocks):
// this kernel streams every key block once per (head, query block) through the
// tensor cores (S = Q K^T in TMEM, as K5) and keeps, per query row, the online
// softmax normaliser of all keys and of the selected keys only — no V, no O, no
// N x N storage. One launch per call; a second tiny kernel reduces the per-row
// masses to a per-head recall in fp64.
//
// Warp roles (64 + 128 * kWG threads): 0 TMA producer (Q, then every K block in order),
// 1 MMA issuer (S_j into one of kSBufs TMEM buffers; S_{j+kSBufs} waits until the
// softmax has read S_j), 2.. kWG warpgroups splitting each block's 128 key
// columns. Padded keys (partial last block) are excluded, padded query rows are
// not counted.
#include <cuda.h>

#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "sm100.cuh"

namespace dfsgpu {

int make_token_map(CUtensorMap* map, const void* base, int layout, int64_t n, int64_t heads, int64_t d);
int make_row_gather_map(CUtensorMap* map, const void* base, int64_t rows, int64_t d);

namespace {

using namespace sm100;

constexpr int kBM = 128, kBN = 128;
#ifndef DFS_RECALL_WG
#define DFS_RECALL_WG 2
#endif
constexpr int kWG = DFS_RECALL_WG;      // softmax warpgroups splitting each block's 128 key columns
constexpr int kCPT = 128 / kWG;        // key columns per softmax thread
#ifndef DFS_RECALL_SBUFS
#define DFS_RECALL_SBUFS 4
#endif
constexpr int kSBufs = DFS_RECALL_SBUFS;  // TMEM S buffers (no O here: all 512 columns can hold S)
constexpr int kSoftmaxThreads = 128 * kWG;
constexpr int kThreads = 64 + kSoftmaxThreads;
constexpr uint32_t kBarMax = 1;

template <int D>
struct RCfg {
  static constexpr int kChunks = D / 64;
  static constexpr int kTileBytes = kBM * D * 2;
  static constexpr int kChunkBytes = kBM * 128;
  static constexpr int kStages = D == 64 ? 12 : 5;
  static constexpr int kRingOff = kTileBytes;  // Q first
  static constexpr int kRedOff = kRingOff + kStages * kTileBytes;
  static constexpr int kBarOff = kRedOff + 4 * kWG * kBM * 4;  // max[2][kWG][128], zall/zmask[kWG][128]
  static constexpr int kSmem = kBarOff + 512 + 1024;
  static constexpr uint32_t kIdescQK = idesc_bf16_f32(kBM, kBN, false, false);
  static_assert(kSmem <= 227 * 1024, "recall kernel shared memory");
};

struct RParams {
  int64_t heads, n, mq, tiles;
  const int32_t* blk_ptr;
  const int32_t* blk_idx;
  const uint32_t* q_rows;  // optional: Q gathered from raster rows (as K5's in_rows)
  int in_nhd;
  float scale_log2;
  float* mass;             // [heads, n]: softmax mass of each query row inside its mask
};

struct RBars {
  uint64_t q_full, q_empty;
  uint64_t s_full[4], s_free[4];
  uint64_t k_full[12], k_empty[12];
  uint32_t tmem_base;
};

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    recall_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                  const RParams p) {
  using C = RCfg<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem;
  uint8_t* sRing = smem + C::kRingOff;
  float* red = reinterpret_cast<float*>(smem + C::kRedOff);
  RBars* bars = reinterpret_cast<RBars*>(smem + C::kBarOff);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&bars->q_full, 1);
    mbar_init(&bars->q_empty, 1);
    for (int i = 0; i < kSBufs; ++i) {
      mbar_init(&bars->s_full[i], 1);
      mbar_init(&bars->s_free[i], kSoftmaxThreads / 32);
    }
    for (int i = 0; i < C::kStages; ++i) {
      mbar_init(&bars->k_full[i], 1);
      mbar_init(&bars->k_empty[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;
  const int64_t mk = ceil_div(p.n, int64_t(kBN));

  if (warp == 0) {
    // ======================= TMA producer: Q, then K_0 .. K_{M-1} =======================
    uint32_t q_phase = 0, ring = 0;
    for (int64_t tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
      const int64_t h = tile / p.mq, u = tile % p.mq;
      mbar_wait(&bars->q_empty, q_phase ^ 1);
      q_phase ^= 1;
      if (p.q_rows) {
        int rr[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          int64_t i = u * kBM + 4 * lane + k;
          i = i < p.n ? i : p.n - 1;
          rr[k] = int(int64_t(__ldg(p.q_rows + i)) * p.heads + h);
        }
        if (elect_one()) mbar_expect_tx(&bars->q_full, C::kTileBytes);
        __syncwarp();
#pragma unroll
        for (int c = 0; c < C::kChunks; ++c)
          tma_gather4(sQ + c * C::kChunkBytes + lane * 512, &tm_q, &bars->q_full, c * 64, rr[0], rr[1], rr[2], rr[3]);
        __syncwarp();
      } else {
        if (elect_one()) {
          mbar_expect_tx(&bars->q_full, C::kTileBytes);
          for (int c = 0; c < C::kChunks; ++c)
            tma_load_3d(sQ + c * C::kChunkBytes, &tm_q, &bars->q_full, c * 64, p.in_nhd ? int(h) : int(u * kBM),
                        p.in_nhd ? int(u * kBM) : int(h));
        }
        __syncwarp();
      }
      for (int64_t v = 0; v < mk; ++v) {
        const uint32_t slot = ring % C::kStages;
        mbar_wait(&bars->k_empty[slot], ((ring / C::kStages) & 1) ^ 1);
        if (elect_one()) {
          mbar_expect_tx(&bars->k_full[slot], C::kTileBytes);
          for (int c = 0; c < C::kChunks; ++c)
            tma_load_3d(sRing + slot * C::kTileBytes + c * C::kChunkBytes, &tm_k, &bars->k_full[slot], c * 64,
                        p.in_nhd ? int(h) : int(v * kBN), p.in_nhd ? int(v * kBN) : int(h));
        }
        __syncwarp();
        ++ring;
      }
    }
  } else if (warp == 1) {
    // ============ MMA issuer: S_g = Q K_v^T, g counting blocks CTA-globally ============
    uint32_t q_phase = 0, ring = 0, g = 0;
    constexpr uint32_t kHi = desc_sw128_hi(1024);
    const uint32_t q_lo = desc_sw128_lo(smem_u32(sQ), 16);
    const uint32_t ring_lo = desc_sw128_lo(smem_u32(sRing), 16);
    for (int64_t tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
      mbar_wait(&bars->q_full, q_phase);
      q_phase ^= 1;
      for (int64_t v = 0; v < mk; ++v, ++g) {
        const uint32_t sb = g % kSBufs;
        if (g >= kSBufs) mbar_wait(&bars->s_free[sb], ((g / kSBufs) - 1) & 1);  // softmax read S_{g-kSBufs}
        const uint32_t slot = ring % C::kStages;
        mbar_wait(&bars->k_full[slot], (ring / C::kStages) & 1);
        ++ring;
        tc_fence_after();
        const uint32_t k_lo = ring_lo + slot * (C::kTileBytes >> 4);
        if (elect_one()) {
#pragma unroll
          for (int s = 0; s < D / 16; ++s) {
            const uint32_t off = ((s >> 2) * C::kChunkBytes + (s & 3) * 32) >> 4;
            umma_ss(tmem + sb * 128, q_lo + off, kHi, k_lo + off, kHi, C::kIdescQK, s > 0);
          }
          umma_commit(&bars->k_empty[slot]);
          umma_commit(&bars->s_full[sb]);
          if (v == mk - 1) umma_commit(&bars->q_empty);
        }
        __syncwarp();
      }
    }
  } else {
    // ============ softmax sums: all keys and the selected keys, per query row ============
    const int wg = (warp - 2) >> 2;
    const int r = (warp & 3) * 32 + lane;
    const uint32_t lane_addr = uint32_t((warp & 3) * 32) << 16;
    float* red_max = red;                    // [parity][kWG][kBM]
    float* red_za = red + 2 * kWG * kBM;     // [kWG][kBM]
    float* red_zm = red + 3 * kWG * kBM;     // [kWG][kBM]
    uint32_t g = 0;
    for (int64_t tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
      const int64_t h = tile / p.mq, u = tile % p.mq;
      const int32_t beg = p.blk_ptr[tile], cnt = p.blk_ptr[tile + 1] - beg;
      int32_t cur = 0, next_sel = cnt > 0 ? p.blk_idx[beg] : -1;
      float m = -INFINITY, za = 0.f, zm = 0.f;
      for (int64_t v = 0; v < mk; ++v, ++g) {
        const bool sel = next_sel == int32_t(v);  // the list is ascending
        if (sel) {
          ++cur;
          next_sel = cur < cnt ? p.blk_idx[beg + cur] : -1;
        }
        const uint32_t sb = g % kSBufs;
        mbar_wait(&bars->s_full[sb], (g / kSBufs) & 1);
        tc_fence_after();
        uint32_t sv[kCPT];
#pragma unroll
        for (int c = 0; c < kCPT / 32; ++c)
          tmem_ld32(tmem + lane_addr + sb * 128 + wg * kCPT + c * 32, *reinterpret_cast<uint32_t(*)[32]>(sv + 32 * c));
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars->s_free[sb]);  // S_g is in registers: the buffer may be reused
        // every block but the partial last one is full: the per-element bounds test stays
        // out of the hot loop (as a runtime test it is if-converted into selects)
        auto block = [&](auto mask_tag, int valid) {
          constexpr bool kMask = decltype(mask_tag)::value;
          float mq[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
          for (int i = 0; i < kCPT; ++i)
            if (!kMask || i < valid) mq[i & 3] = fmaxf(mq[i & 3], __uint_as_float(sv[i]));
          // each slice keeps its own running max (no P is shared between slices here, unlike
          // K5): no per-block exchange; the slices' (max, sums) merge once per tile
          const float mx = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3]));
          const float m_new = fmaxf(m, mx * p.scale_log2);
          if (m_new > m) {
            const float a = ex2(m - m_new);
            za *= a;
            zm *= a;
            m = m_new;
          }
          // exp2 in packed fp32x2; pairs 1, 4, 7 of every 8 on the FMA-pipe polynomial
          const uint64_t sc2 = f2_pack(p.scale_log2, p.scale_log2), nm2 = f2_pack(-m, -m);
          uint64_t e2 = 0;
#pragma unroll
          for (int i = 0; i < kCPT / 2; ++i) {
            float x0, x1;
            f2_unpack(f2_fma(f2_pack(__uint_as_float(sv[2 * i]), __uint_as_float(sv[2 * i + 1])), sc2, nm2), x0, x1);
            float p0, p1;
            if ((0x92u >> (i % 8)) & 1u) {
              f2_unpack(ex2_poly2(x0, x1), p0, p1);
            } else {
              p0 = ex2(x0);
              p1 = ex2(x1);
            }
            if (kMask) {
              if (2 * i >= valid) p0 = 0.f;
              if (2 * i + 1 >= valid) p1 = 0.f;
            }
            e2 = f2_add(e2, f2_pack(p0, p1));
          }
          float e0, e1;
          f2_unpack(e2, e0, e1);
          return e0 + e1;
        };
        const int valid = int(min(int64_t(kBN), p.n - v * kBN)) - wg * kCPT;
        const float e = valid >= kCPT ? block(std::false_type{}, kCPT) : block(std::true_type{}, valid);
        za += e;
        if (sel) zm += e;
      }
      red_max[wg * kBM + r] = m;
      red_za[wg * kBM + r] = za;
      red_zm[wg * kBM + r] = zm;
      named_bar_sync(kBarMax, kSoftmaxThreads);
      if (wg == 0) {
        float mm = -INFINITY;
#pragma unroll
        for (int w = 0; w < kWG; ++w) mm = fmaxf(mm, red_max[w * kBM + r]);
        float ta = 0.f, tm = 0.f;
#pragma unroll
        for (int w = 0; w < kWG; ++w) {
          const float mw = red_max[w * kBM + r];
          const float sc = mw > -INFINITY ? ex2(mw - mm) : 0.f;
          ta += red_za[w * kBM + r] * sc;
          tm += red_zm[w * kBM + r] * sc;
        }
        const int64_t i = u * kBM + r;
        if (i < p.n) p.mass[h * p.n + i] = tm / ta;
      }
      named_bar_sync(kBarMax, kSoftmaxThreads);  // the sum slots are rewritten by the next tile
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

// recall[h] = sum_i mass[h][i] / n, fp64, one CTA per head (deterministic order)
__global__ void recall_reduce_kernel(const float* __restrict__ mass, int64_t n, double* __restrict__ out) {
  const int64_t h = blockIdx.x;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += double(mass[h * n + i]);
  s = warp_sum_d(s);
  __shared__ double part[32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) t += part[w];
    out[h] = t / double(n);
  }
}

template <int D>
int launch(const void* q, const void* k, int layout, const uint32_t* q_rows, int64_t heads, int64_t n,
           const int32_t* blk_ptr, const int32_t* blk_idx, float* mass, double* recall, cudaStream_t stream) {
  using C = RCfg<D>;
  CUtensorMap mq, mk;
  int rc;
  if (q_rows) {
    if ((rc = make_row_gather_map(&mq, q, n * heads, D))) return rc;
  } else if ((rc = make_token_map(&mq, q, layout, n, heads, D))) {
    return rc;
  }
  if ((rc = make_token_map(&mk, k, layout, n, heads, D))) return rc;
  RParams p;
  p.heads = heads;
  p.n = n;
  p.mq = ceil_div(n, int64_t(kBM));
  p.tiles = p.mq * heads;
  p.blk_ptr = blk_ptr;
  p.blk_idx = blk_idx;
  p.q_rows = q_rows;
  p.in_nhd = layout == DFS_NHD;
  p.scale_log2 = float(1.4426950408889634 / sqrt(double(D)));
  p.mass = mass;
  // per device and race-free: set on every launch (~1 us)
  DFS_CUDA_CHECK(cudaFuncSetAttribute(recall_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
  const int64_t grid = p.tiles < kNumSMs ? p.tiles : kNumSMs;
  recall_kernel<D><<<unsigned(grid), kThreads, C::kSmem, stream>>>(mq, mk, p);
  recall_reduce_kernel<<<unsigned(heads), 256, 0, stream>>>(mass, n, recall);
  DFS_LAUNCH_CHECK("block_recall");
  return DFS_OK;
}

}  // namespace

bool recall_sm100_supports(int64_t d) { return d == 64 || d == 128; }

// mass: caller workspace of heads * n floats; recall: device [heads] fp64
int block_recall_sm100(const void* q, const void* k, int layout, const uint32_t* q_rows, int64_t heads, int64_t n,
                       int64_t d, const int32_t* blk_ptr, const int32_t* blk_idx, float* mass, double* recall,
                       cudaStream_t stream) {
  if (d == 128) return launch<128>(q, k, layout, q_rows, heads, n, blk_ptr, blk_idx, mass, recall, stream);
  if (d == 64) return launch<64>(q, k, layout, q_rows, heads, n, blk_ptr, blk_idx, mass, recall, stream);
  return fail(DFS_E_UNSUPPORTED, "block_recall: d must be 64 or 128");
}

}  // namespace dfsgpu
