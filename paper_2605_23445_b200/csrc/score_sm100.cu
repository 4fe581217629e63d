// score_sm100.cu — K3 tensor-core path: hierarchical block scores on tcgen05.
//
// mask_builder.cpp:30-80 (+ attention.cpp:105-123 as the pooled softmax):
//   S[u][v] = sum over the subs x subs tile (u, v) of softmax_row(Q^ K^T / sqrt(d))
// with Q^, K^ the sub-block means (fp32, from K2's fused pooling). The survey
// (SURVEY.md §0 finding 4) shows scores sit within 1e-4..1e-7 of each other at
// the top-K cut, so the pooled GEMM must be fp32-accurate: bf16/TF32 operands
// flip 0.03-1% of mask bits. Here every fp32 operand is split into two fp16
// halves after a per-head power-of-two scaling (so both halves are normal):
//   a*s = hi + lo * 2^-11,   hi = f16(a*s),  lo = f16((a*s - hi) * 2^11)
//   Q^K^T * sq*sk = Qhi Khi^T + 2^-11 (Qhi Klo^T + Qlo Khi^T)   (+ O(2^-22))
// three fp16 UMMAs at the full 16-bit tensor rate (twice TF32's), fp32
// accumulation in TMEM: D1 = hi*hi, D2 = the two cross terms.
//
// CTA pairs (cta_group::2, cluster of 2): each CTA owns a 128-row stripe of pooled
// queries; the leader issues M = 256 MMAs over both stripes while each CTA loads only
// half of every 128-key tile. One pass over the key tiles: each softmax slice (32 key
// columns) keeps an exact online (max, sum) and writes unnormalised sub-row tile sums
// to an L2-resident per-CTA scratch; the fix-up that turns them into probabilities
// (summed over `subs` rows by shuffles, fp64 S) runs inside the NEXT stripe's tile loop.
// Warp roles as in K5: warp 0 TMA, warp 1 MMA issue (leader), warps 2-17 softmax.
// Padded query rows are zero vectors (uniform over the valid keys, mask_builder
// .cpp:40-49); padded key columns are excluded (:50-60).
#include <cuda.h>
#include <cuda_fp16.h>

#include <type_traits>

#include "common.cuh"
#include "sm100.cuh"

namespace dfsgpu {

int make_map_f16(CUtensorMap* map, const void* base, int64_t rows, int64_t heads, int64_t d, int box_rows = 128);

namespace {

using namespace sm100;

constexpr int kRows = 128;
constexpr int kKeys = 128;
constexpr int kSWG = 4;                   // softmax warpgroups: 32 key columns of each tile apiece
constexpr int kSoftThreads = 128 * kSWG;
constexpr int kThreads = 64 + kSoftThreads;
constexpr float kLoScale = 2048.f;        // 2^11
constexpr float kInvLoScale = 1.f / 2048.f;
// Lazy row max (as in K5): a slice's running max m is set from its first key tile and then
// kept while the tile sums of 2^(l - m) stay <= kLazySum (every p of the tile is bounded by
// its sum); the exponent arguments come straight out of the logit FMAs and no per-tile max
// is computed. A tile whose sum exceeds it (rare) raises m to its own max and recomputes.
// The scratch stores the m each tile used, so the fix-up is unchanged.
#ifndef DFS_SCORE_LAZY
#define DFS_SCORE_LAZY 1
#endif
constexpr bool kLazy = DFS_SCORE_LAZY;
constexpr float kLazySum = 65536.f;
// every kPolyEvery-th exponential pair of the lazy path on the FMA-pipe degree-5 polynomial
// (fp32-accurate, sm100.cuh ex2_poly5x2); 0 = all on MUFU
#ifndef DFS_SCORE_POLY
#define DFS_SCORE_POLY 6
#endif
constexpr int kPolyEvery = DFS_SCORE_POLY;

// CTA pairs (cta_group::2): the pair's MMA is M = 256 (each CTA's own 128-row stripe)
// x N = 128 keys, and each CTA holds only half of every key tile (64 keys) — the pooled
// key operand is read from L2 once per pair instead of once per CTA. The K stream is the
// kernel's L2->SM traffic bound (~5.3 GB per HY call unpaired).
template <int D>
struct SCfg {
  static constexpr int kChunks = D / 64;
  static constexpr int kChunkBytes = 128 * 128;          // A: 128 rows x 64 fp16
  static constexpr int kOpBytes = kRows * D * 2;          // one hi or lo Q stripe
  static constexpr int kHalfKeys = kKeys / 2;             // key rows this CTA supplies
  static constexpr int kBChunkBytes = kHalfKeys * 128;    // B: 64 rows x 64 fp16
  static constexpr int kHalfBytes = kHalfKeys * D * 2;    // one hi or lo key half-tile
  static constexpr int kStages = D == 64 ? 8 : 4;
  static constexpr int kQOff = 0;                         // Qhi, Qlo
  static constexpr int kKOff = 2 * kOpBytes;              // stages x (Khi, Klo) halves
  static constexpr int kRedOff = kKOff + kStages * 2 * kHalfBytes;  // float [2][m | z][kSWG][128]
  static constexpr int kBarOff = kRedOff + 2 * 2 * kSWG * kRows * 4;
  static constexpr int kSmem = kBarOff + 256 + 1024;
};

// kind::f16 with fp16 inputs (formats 0), fp32 accumulation, K-major A and B, M = 256 (pair)
constexpr uint32_t kIdesc = (1u << 4) | (uint32_t(kKeys >> 3) << 17) | (uint32_t(2 * kRows >> 4) << 24);

struct SParams {
  int64_t heads, qvalid, kvalid, m, subs, nrt, nkt;
  int64_t npr, pitems;  // stripe pairs per head (stripes 2i, 2i+1), pairs in total
  const float* fac;   // [H]: scale_log2 / (sq * sk)
  double* S;
  float* tsum;        // per-CTA scratch [gridDim][m][128]: unnormalised row tile sums
  float* tmax;        // per-CTA scratch [gridDim][nkt * kSWG][128]: the max each slice used
};

struct SBars {
  uint64_t q_full, q_empty;
  uint64_t k_full[8], k_empty[8];
  uint64_t acc_full[2], acc_free[2];
  uint32_t tmem_base;
};

// One pass over the pooled keys per 128-row stripe. Each softmax slice keeps an
// exact online (max, sum) and writes, per key block v of its columns, the
// unnormalised sub-row tile sum t_rv = sum_c 2^(l_rc - m_slice) together with the
// slice max it used; after the stripe (max, sum) is merged across the slices and a
// fix-up pass turns t_rv into probabilities, p = t_rv 2^(m_used - m_row) / z_row,
// summed over the SUBS sub-rows of each query block. The per-CTA scratch lives in
// L2 (it is re-read right after it is written), so the second GEMM + exp pass of a
// two-pass softmax is replaced by one L2 round trip of 4 bytes per (row, block).
template <int D, int SUBS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    score_sm100_kernel(const __grid_constant__ CUtensorMap tm_qh, const __grid_constant__ CUtensorMap tm_ql,
                       const __grid_constant__ CUtensorMap tm_kh, const __grid_constant__ CUtensorMap tm_kl,
                       const SParams p) {
  using C = SCfg<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  SBars* bars = reinterpret_cast<SBars*>(smem + C::kBarOff);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();             // 0: leader (issues the pair's MMAs)
  const int64_t cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  if (threadIdx.x == 0) {
    mbar_init(&bars->q_full, 1);
    mbar_init(&bars->q_empty, 1);
    for (int i = 0; i < C::kStages; ++i) {
      mbar_init(&bars->k_full[i], 1);
      mbar_init(&bars->k_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars->acc_full[i], 1);
      mbar_init(&bars->acc_free[i], 2 * kSoftThreads / 32);  // one arrive per softmax warp of the pair
    }
    fence_barrier_init();
  }
  cluster_sync();  // the peer's barriers exist before any remote arrive or TMA signal
  if (warp == 1) tmem_alloc_pair<512>(&bars->tmem_base);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  if (warp == 0) {
    // ============ TMA producer (warp-uniform loop, one elected lane issues) ============
    // Both CTAs load their own Q stripe and their half of each key tile; the bytes are
    // counted on the leader's barriers (the leader posts the pair's expected total).
    uint32_t q_phase = 0, ring = 0;
    for (int64_t pit = cid; pit < p.pitems; pit += ncl) {
      const int h = int(pit / p.npr), rt = int(pit % p.npr) * 2 + int(rank);
      mbar_wait(&bars->q_empty, q_phase ^ 1);
      q_phase ^= 1;
      if (elect_one()) {
        if (rank == 0) mbar_expect_tx(&bars->q_full, 2 * 2 * C::kOpBytes);
        for (int c = 0; c < C::kChunks; ++c) {
          tma_load_3d_pair(smem + C::kQOff + c * C::kChunkBytes, &tm_qh, &bars->q_full, c * 64, rt * kRows, h);
          tma_load_3d_pair(smem + C::kQOff + C::kOpBytes + c * C::kChunkBytes, &tm_ql, &bars->q_full, c * 64,
                           rt * kRows, h);
        }
      }
      __syncwarp();
      for (int kt = 0; kt < p.nkt; ++kt) {
        const uint32_t slot = ring % C::kStages;
        mbar_wait(&bars->k_empty[slot], ((ring / C::kStages) & 1) ^ 1);
#ifdef DFS_SCORE_SKIP_TMA  // experiment builds only: key tiles never loaded (garbage operands)
        if (elect_one() && rank == 0) mbar_arrive(&bars->k_full[slot]);
        __syncwarp();
        ++ring;
        continue;
#endif
        if (elect_one()) {
          if (rank == 0) mbar_expect_tx(&bars->k_full[slot], 2 * 2 * C::kHalfBytes);
          uint8_t* dst = smem + C::kKOff + slot * 2 * C::kHalfBytes;
          const int k0 = kt * kKeys + int(rank) * C::kHalfKeys;
          for (int c = 0; c < C::kChunks; ++c) {
            tma_load_3d_pair(dst + c * C::kBChunkBytes, &tm_kh, &bars->k_full[slot], c * 64, k0, h);
            tma_load_3d_pair(dst + C::kHalfBytes + c * C::kBChunkBytes, &tm_kl, &bars->k_full[slot], c * 64, k0, h);
          }
        }
        __syncwarp();
        ++ring;
      }
    }
  } else if (warp == 1) {
    // ============ MMA issuer (leader only): D1 = Qhi Khi^T, D2 = Qhi Klo^T + Qlo Khi^T ============
    if (rank == 0) {
      uint32_t q_phase = 0, ring = 0, acc_iter = 0;
      constexpr uint32_t kHi = desc_sw128_hi(1024);
      const uint32_t qh_lo = desc_sw128_lo(smem_u32(smem + C::kQOff), 16);
      const uint32_t ql_lo = qh_lo + (C::kOpBytes >> 4);
      const uint32_t k_lo0 = desc_sw128_lo(smem_u32(smem + C::kKOff), 16);
      for (int64_t pit = cid; pit < p.pitems; pit += ncl) {
        mbar_wait(&bars->q_full, q_phase);
        q_phase ^= 1;
        for (int kt = 0; kt < p.nkt; ++kt) {
          const uint32_t slot = ring % C::kStages;
          mbar_wait(&bars->k_full[slot], (ring / C::kStages) & 1);
          ++ring;
          const uint32_t b = acc_iter & 1;
          mbar_wait(&bars->acc_free[b], ((acc_iter >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t kh_lo = k_lo0 + slot * ((2 * C::kHalfBytes) >> 4), kl_lo = kh_lo + (C::kHalfBytes >> 4);
          const uint32_t d1 = tmem + b * 256, d2 = d1 + 128;
          if (elect_one()) {
#pragma unroll
            for (int s = 0; s < D / 16; ++s) {
              const uint32_t oa = ((s >> 2) * C::kChunkBytes + (s & 3) * 32) >> 4;
              const uint32_t ob = ((s >> 2) * C::kBChunkBytes + (s & 3) * 32) >> 4;
#ifndef DFS_SCORE_SKIP_MMA  // experiment builds only: isolate the softmax / TMA side
              umma_ss_pair(d1, qh_lo + oa, kHi, kh_lo + ob, kHi, kIdesc, s > 0);
              umma_ss_pair(d2, qh_lo + oa, kHi, kl_lo + ob, kHi, kIdesc, s > 0);
              umma_ss_pair(d2, ql_lo + oa, kHi, kh_lo + ob, kHi, kIdesc, 1);
#endif
            }
            umma_commit_pair(&bars->k_empty[slot]);
            umma_commit_pair(&bars->acc_full[b]);
            if (kt == p.nkt - 1) umma_commit_pair(&bars->q_empty);
          }
          __syncwarp();
          ++acc_iter;
        }
      }
    }
  } else {
    // kSWG warpgroups split each 128-key tile by columns (32 apiece); a thread owns one
    // pooled query row (TMEM lane) of its slice.
    const int wg = (warp - 2) >> 2;
    const int r = (warp & 3) * 32 + lane;
    const uint32_t lane_addr = uint32_t((warp & 3) * 32) << 16;
    float* red = reinterpret_cast<float*>(smem + C::kRedOff);  // [stripe parity][m | z][kSWG][kRows]
    float* tsum = p.tsum + int64_t(blockIdx.x) * p.m * kRows;            // [v][row]
    float* tmax = p.tmax + int64_t(blockIdx.x) * p.nkt * kSWG * kRows;   // [kt][slice][row]
    constexpr int G = 32 / SUBS;                                           // key blocks per slice per tile
    const int m32 = int(p.m), kvalid32 = int(p.kvalid);                    // (host checks < 2^31 / 128)
    // The fix-up of stripe s runs inside stripe s+1: at tile kt a thread first reads the
    // scratch entries its own slice wrote for tile kt of stripe s (program order: no
    // barrier), turns them into probabilities with stripe s's merged row statistics and
    // then overwrites them. The tensor pipe therefore never idles for a fix-up phase;
    // only the CTA's last stripe is fixed up after the loop.
    struct Prev {
      bool valid = false;
      int64_t h = 0;
      int u = 0;               // S row block of this thread's pooled row in the previous stripe
      float mm = 0.f, inv_z = 0.f;
    } prev;
    // probabilities of (row, key blocks of slice wg in tile kt) for the previous stripe;
    // every lane of the warp takes part (sub-row sums by shuffles)
    auto fix_tile = [&](int kt, const float (&t)[G], float mu) {
      const float e = ex2(mu - prev.mm);
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int v = kt * (kKeys / SUBS) + wg * G + g;
        float pr = t[g] > 0.f ? t[g] * e * prev.inv_z : 0.f;
#pragma unroll
        for (int o = 1; o < SUBS; o <<= 1) pr += __shfl_xor_sync(0xffffffffu, pr, o);
        // S is write-once output: streaming stores keep it from evicting the L2-resident scratch
        if ((lane % SUBS) == 0 && prev.u < m32 && v < m32)
          __stcs(p.S + (prev.h * p.m + prev.u) * p.m + v, double(pr));
      }
    };
    auto load_tile = [&](int kt, float (&t)[G], float& mu) {
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int v = kt * (kKeys / SUBS) + wg * G + g;
        t[g] = v < m32 ? tsum[v * kRows + r] : 0.f;
      }
      mu = tmax[(kt * kSWG + wg) * kRows + r];
    };
    uint32_t acc_iter = 0, parity = 0;
    for (int64_t pit = cid; pit < p.pitems; pit += ncl) {
      const int h = int(pit / p.npr), rt = int(pit % p.npr) * 2 + int(rank);
      const float f = p.fac[h];
      const uint64_t f2 = f2_pack(f, f), g2 = f2_pack(f * kInvLoScale, f * kInvLoScale);
      const int64_t row = int64_t(rt) * kRows + r;     // pooled query row
      float m = -INFINITY, z = 0.f;
      // the previous stripe's scratch entries, fetched one tile ahead (L2 latency hidden
      // behind a whole tile of work)
      float t_nx[G], mu_nx = 0.f;
      if (prev.valid) load_tile(0, t_nx, mu_nx);
      // one key tile; kMask only for the last tile (the one holding the end of the valid
      // keys) — a runtime test here is if-converted into per-element selects every tile
      auto tile = [&](int kt, auto mask_tag) {
        constexpr bool kMask = decltype(mask_tag)::value;
        float t_old[G], mu_old = mu_nx;
#pragma unroll
        for (int g = 0; g < G; ++g) t_old[g] = t_nx[g];
        if (prev.valid && kt + 1 < p.nkt) load_tile(kt + 1, t_nx, mu_nx);
        const uint32_t b = acc_iter & 1;
        mbar_wait(&bars->acc_full[b], (acc_iter >> 1) & 1);
        tc_fence_after();
#ifdef DFS_SCORE_SKIP_SOFTMAX  // experiment builds only (tools/score_exp.sh): isolate the MMA/TMA side
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(&bars->acc_free[b], 0);
        ++acc_iter;
        return;
#endif
        const int cbase = kt * kKeys + wg * 32;
        // logits l = (D1 + D2 / 2^11) * f in packed fp32x2 arithmetic; only the tile holding
        // the end of the valid pooled keys masks (warp-uniform branch)
        uint64_t l2[16];
        // kLazy: x = l - m straight from the FMAs (m of the first tile: 0 here, set below)
        const bool lazy = kLazy && kt > 0;
        const uint64_t nm2 = f2_pack(lazy ? -m : 0.f, lazy ? -m : 0.f);
        {
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            uint32_t a1[16], a2[16];
            tmem_ld16(tmem + lane_addr + b * 256 + wg * 32 + c * 16, a1);
            tmem_ld16(tmem + lane_addr + b * 256 + 128 + wg * 32 + c * 16, a2);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 8; ++i)
              l2[c * 8 + i] = kLazy ? f2_fma(f2_pack(__uint_as_float(a2[2 * i]), __uint_as_float(a2[2 * i + 1])), g2,
                                             f2_fma(f2_pack(__uint_as_float(a1[2 * i]), __uint_as_float(a1[2 * i + 1])), f2, nm2))
                                    : f2_fma(f2_pack(__uint_as_float(a2[2 * i]), __uint_as_float(a2[2 * i + 1])), g2,
                                             f2_mul(f2_pack(__uint_as_float(a1[2 * i]), __uint_as_float(a1[2 * i + 1])), f2));
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(&bars->acc_free[b], 0);  // the leader's barrier
        ++acc_iter;
        const int rem = kvalid32 - cbase;
        if (kMask && rem < 32) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float x0, x1;
            f2_unpack(l2[i], x0, x1);
            if (2 * i >= rem) x0 = -INFINITY;
            if (2 * i + 1 >= rem) x1 = -INFINITY;
            l2[i] = f2_pack(x0, x1);
          }
        }
        float tg[G];
        if (lazy) {  // l2 holds x = l - m
          auto sums = [&](float shift) {  // tile sums of 2^(x - shift)
            const uint64_t sh2 = f2_pack(-shift, -shift);
            float s = 0.f;
#pragma unroll
            for (int g = 0; g < G; ++g) {
              uint64_t t2 = 0;
#pragma unroll
              for (int i = 0; i < SUBS / 2; ++i) {
                float x0, x1;
                f2_unpack(shift != 0.f ? f2_add(l2[g * (SUBS / 2) + i], sh2) : l2[g * (SUBS / 2) + i], x0, x1);
                if (kPolyEvery && (g * (SUBS / 2) + i) % kPolyEvery == kPolyEvery - 1)
                  t2 = f2_add(t2, ex2_poly5x2(x0, x1));  // FMA pipe (offloads MUFU)
                else
                  t2 = f2_add(t2, f2_pack(ex2(x0), ex2(x1)));
              }
              float ta, tb;
              f2_unpack(t2, ta, tb);
              tg[g] = ta + tb;
              s += tg[g];
            }
            return s;
          };
          float s = sums(0.f);
          if (__any_sync(0xffffffffu, !(s <= kLazySum))) {  // rare: raise m to this tile's max
            float mx = -INFINITY;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              float x0, x1;
              f2_unpack(l2[i], x0, x1);
              mx = fmaxf(mx, fmaxf(x0, x1));
            }
            if (mx > 0.f) {
              s = sums(mx);
              z *= ex2(-mx);
              m += mx;
            }
          }
          z += s;
        } else {
        float mx = -INFINITY;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          float x0, x1;
          f2_unpack(l2[i], x0, x1);
          mx = fmaxf(mx, fmaxf(x0, x1));
        }
        const float mn = fmaxf(m, mx);
        if (mn > -INFINITY) {
          const uint64_t nm2 = f2_pack(-mn, -mn);
          float s = 0.f;
#pragma unroll
          for (int g = 0; g < G; ++g) {
            uint64_t t2 = 0;  // two independent fp32 chains per group
#pragma unroll
            for (int i = 0; i < SUBS / 2; ++i) {
              float x0, x1;
              f2_unpack(f2_add(l2[g * (SUBS / 2) + i], nm2), x0, x1);
              t2 = f2_add(t2, f2_pack(ex2(x0), ex2(x1)));
            }
            float ta, tb;
            f2_unpack(t2, ta, tb);
            tg[g] = ta + tb;
            s += tg[g];
          }
          z = z * ex2(m - mn) + s;
          m = mn;
        } else {
#pragma unroll
          for (int g = 0; g < G; ++g) tg[g] = 0.f;
        }
        }
        if (prev.valid) fix_tile(kt, t_old, mu_old);
        // coalesced across the warp: 32 consecutive rows per (v) / (kt, slice) entry
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const int v = (cbase + g * SUBS) / SUBS;
          if (v < m32) tsum[v * kRows + r] = tg[g];
        }
        tmax[(kt * kSWG + wg) * kRows + r] = m;
      };
      for (int kt = 0; kt + 1 < p.nkt; ++kt) tile(kt, std::false_type{});
      tile(int(p.nkt) - 1, std::true_type{});
      // merge the slices' (max, sum) of this row (slots double-buffered by stripe parity)
      float* red_m = red + parity * 2 * kSWG * kRows;
      float* red_z = red_m + kSWG * kRows;
      red_m[wg * kRows + r] = m;
      red_z[wg * kRows + r] = z;
      named_bar_sync(1, kSoftThreads);
      float mm = -INFINITY;
#pragma unroll
      for (int w = 0; w < kSWG; ++w) mm = fmaxf(mm, red_m[w * kRows + r]);
      float zz = 0.f;
#pragma unroll
      for (int w = 0; w < kSWG; ++w) {
        const float mw = red_m[w * kRows + r];
        if (mw > -INFINITY) zz += red_z[w * kRows + r] * ex2(mw - mm);
      }
      prev.valid = true;
      prev.h = h;
      prev.u = int(row / SUBS);
      prev.mm = mm;
      prev.inv_z = 1.f / zz;
      parity ^= 1;
    }
    // the CTA's last stripe: fix-up without a following stripe to hide it in
    if (prev.valid) {
      for (int kt = 0; kt < p.nkt; ++kt) {
        float t_old[G], mu_old;
        load_tile(kt, t_old, mu_old);
        fix_tile(kt, t_old, mu_old);
      }
    }
  }
  tc_fence_before();
  cluster_sync();  // every MMA of the pair has completed and been consumed
  tc_fence_after();
  if (warp == 1) tmem_dealloc_pair<512>(tmem);
}

// ---- operand preparation: per-head power-of-two scale, fp16 hi/lo split ----------

// pooled q (blockIdx.z = 0) and k (1) in one launch each: per-head absmax, then the
// fp16 hi/lo split (16-byte loads); the split's first block of each head also writes
// the logit factor fac[h] = scale_log2 / (s_q s_k)
__global__ void absmax_kernel(const float* __restrict__ xq, const float* __restrict__ xk, int64_t per_head,
                              int heads, unsigned* __restrict__ out) {
  const int h = blockIdx.y;
  const float4* x = reinterpret_cast<const float4*>((blockIdx.z ? xk : xq) + h * per_head);
  float mx = 0.f;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < per_head / 4; i += int64_t(gridDim.x) * blockDim.x) {
    const float4 v = x[i];
    mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
  }
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) atomicMax(out + blockIdx.z * heads + h, __float_as_uint(mx));
}

__device__ __forceinline__ float pow2_scale(unsigned bits) {
  // largest power of two s with max|x| * s <= 2^14 (both halves stay normal fp16)
  const float mx = __uint_as_float(bits);
  if (!(mx > 0.f) || !isfinite(mx)) return 1.f;
  int e;
  frexpf(mx, &e);  // mx = f * 2^e, f in [0.5, 1)
  return ldexpf(1.f, 14 - e);
}

struct SplitOut {
  __half *hi, *lo;
};
__global__ void split_kernel(const float* __restrict__ xq, const float* __restrict__ xk, int64_t per_head,
                             const unsigned* __restrict__ amax, int heads, SplitOut oq, SplitOut ok,
                             float scale_log2, float* __restrict__ fac) {
  const int h = blockIdx.y, z = blockIdx.z;
  if (blockIdx.x == 0 && z == 0 && threadIdx.x == 0)
    fac[h] = scale_log2 / (pow2_scale(amax[h]) * pow2_scale(amax[heads + h]));
  const float s = pow2_scale(amax[z * heads + h]);
  const float4* x = reinterpret_cast<const float4*>((z ? xk : xq) + h * per_head);
  const SplitOut o = z ? ok : oq;
  __half2* hi = reinterpret_cast<__half2*>(o.hi + h * per_head);
  __half2* lo = reinterpret_cast<__half2*>(o.lo + h * per_head);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < per_head / 4; i += int64_t(gridDim.x) * blockDim.x) {
    const float4 v = x[i];
    const float a[4] = {v.x * s, v.y * s, v.z * s, v.w * s};
    __half hh[4], ll[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      hh[j] = __float2half_rn(a[j]);
      ll[j] = __float2half_rn((a[j] - __half2float(hh[j])) * kLoScale);
    }
    hi[2 * i] = __halves2half2(hh[0], hh[1]);
    hi[2 * i + 1] = __halves2half2(hh[2], hh[3]);
    lo[2 * i] = __halves2half2(ll[0], ll[1]);
    lo[2 * i + 1] = __halves2half2(ll[2], ll[3]);
  }
}

template <int D, int SUBS>
int launch(const CUtensorMap* maps, const SParams& p, cudaStream_t stream) {
  using C = SCfg<D>;
  // set on every launch: the attribute is per device and a one-time static flag would be
  // wrong for a second device and racy across host threads (the call costs ~1 us)
  DFS_CUDA_CHECK(cudaFuncSetAttribute(score_sm100_kernel<D, SUBS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      C::kSmem));
  const int64_t grid = 2 * p.pitems < kNumSMs ? 2 * p.pitems : kNumSMs;  // whole pairs (kNumSMs is even)
  score_sm100_kernel<D, SUBS><<<unsigned(grid), kThreads, C::kSmem, stream>>>(maps[0], maps[1], maps[2], maps[3], p);
  DFS_LAUNCH_CHECK("score_sm100");
  return DFS_OK;
}

}  // namespace

bool score_sm100_supports(int64_t d, int64_t block, int64_t sub_block) {
  if (d != 64 && d != 128) return false;
  if (sub_block < 1 || block % sub_block) return false;
  const int64_t subs = block / sub_block;
  return subs == 2 || subs == 4 || subs == 8 || subs == 16 || subs == 32;
}

int64_t score_sm100_ws_bytes(int64_t heads, int64_t n, int64_t d, int64_t block, int64_t sub_block) {
  const int64_t valid = ceil_div(n, sub_block);
  const int64_t m = ceil_div(n, block);
  const int64_t nkt = ceil_div(valid, int64_t(kKeys));
  const int64_t scratch = int64_t(kNumSMs) * (m + nkt * kSWG) * kRows * 4;  // per-CTA tsum + tmax
  return 4 * heads * valid * d * 2 /* qh ql kh kl */ + 2 * heads * 4 /* absmax */ + heads * 4 /* fac */ + 256 +
         scratch + 256;
}

int score_blocks_sm100(const float* pq, const float* pk, int64_t heads, int64_t n, int64_t d, int64_t block,
                       int64_t sub_block, double* S, void* ws, int64_t ws_bytes, cudaStream_t stream) {
  if (ws_bytes < score_sm100_ws_bytes(heads, n, d, block, sub_block))
    return fail(DFS_E_INTERNAL, "score_sm100: workspace too small");
  const int64_t valid = ceil_div(n, sub_block);
  const int64_t per_head = valid * d;
  __half* qh = static_cast<__half*>(ws);
  __half* ql = qh + heads * per_head;
  __half* kh = ql + heads * per_head;
  __half* kl = kh + heads * per_head;
  unsigned* amax = reinterpret_cast<unsigned*>(kl + heads * per_head);
  float* fac = reinterpret_cast<float*>(amax + 2 * heads);
  const uintptr_t sc = (reinterpret_cast<uintptr_t>(fac + heads) + 255) & ~uintptr_t(255);
  float* tsum = reinterpret_cast<float*>(sc);
  const int64_t m_blocks = ceil_div(n, block), nkt_keys = ceil_div(valid, int64_t(kKeys));
  float* tmax = tsum + int64_t(kNumSMs) * m_blocks * kRows;
  (void)nkt_keys;
  DFS_CUDA_CHECK(cudaMemsetAsync(amax, 0, sizeof(unsigned) * size_t(2 * heads), stream));
  dim3 g(unsigned(ceil_div(per_head / 4, 256) < 64 ? ceil_div(per_head / 4, 256) : 64), unsigned(heads), 2u);
  absmax_kernel<<<g, 256, 0, stream>>>(pq, pk, per_head, int(heads), amax);
  const float scale_log2 = float(1.4426950408889634 / sqrt(double(d)));
  split_kernel<<<g, 256, 0, stream>>>(pq, pk, per_head, amax, int(heads), SplitOut{qh, ql}, SplitOut{kh, kl},
                                      scale_log2, fac);
  DFS_LAUNCH_CHECK("score_sm100 prep");

  CUtensorMap maps[4];
  int rc;
  if ((rc = make_map_f16(&maps[0], qh, valid, heads, d)) || (rc = make_map_f16(&maps[1], ql, valid, heads, d)) ||
      (rc = make_map_f16(&maps[2], kh, valid, heads, d, 64)) || (rc = make_map_f16(&maps[3], kl, valid, heads, d, 64)))
    return rc;
  SParams p;
  p.heads = heads;
  p.qvalid = valid;
  p.kvalid = valid;
  p.m = ceil_div(n, block);
  p.subs = block / sub_block;
  p.nrt = ceil_div(p.m * p.subs, kRows);
  p.nkt = ceil_div(valid, kKeys);
  p.npr = ceil_div(p.nrt, int64_t(2));
  p.pitems = heads * p.npr;
  p.fac = fac;
  p.S = S;
  p.tsum = tsum;
  p.tmax = tmax;
  const int subs = int(p.subs);
  if (d == 128) {
    switch (subs) {
      case 2: return launch<128, 2>(maps, p, stream);
      case 4: return launch<128, 4>(maps, p, stream);
      case 8: return launch<128, 8>(maps, p, stream);
      case 16: return launch<128, 16>(maps, p, stream);
      case 32: return launch<128, 32>(maps, p, stream);
    }
  } else {
    switch (subs) {
      case 2: return launch<64, 2>(maps, p, stream);
      case 4: return launch<64, 4>(maps, p, stream);
      case 8: return launch<64, 8>(maps, p, stream);
      case 16: return launch<64, 16>(maps, p, stream);
      case 32: return launch<64, 32>(maps, p, stream);
    }
  }
  return fail(DFS_E_UNSUPPORTED, "score_sm100: unsupported geometry");
}

}  // namespace dfsgpu
