/* oracle/dfs_oracle.c — TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * Independent C11 restatement of the reference hot path; see dfs_oracle.h.
 * fp64 accumulation and fp32 storage exactly where the reference has them, so
 * that on the same host (same libm) the outputs are bit-identical to the
 * reference library — verified by tests/test_oracle.py. Loops over
 * independent rows / query blocks are OpenMP-parallel; every reduction whose
 * order the reference fixes stays sequential inside one thread, so results do
 * not depend on the thread count.
 */
#define _GNU_SOURCE
#include "dfs_oracle.h"

#include <math.h>
#include <omp.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* reorder — curve.cpp                                                        */
/* ------------------------------------------------------------------------ */

static int ceil_log2(int64_t extent) { /* curve.cpp:39-43 bits_for */
  int b = 0;
  while (((int64_t)1 << b) < extent) ++b;
  return b;
}

/* Skilling transpose->axes (curve.cpp:50-81). `nd` axes, `bits` per axis.
 * Step 1 deals the index bits round-robin, most significant group first;
 * step 2 undoes the Gray code; step 3 undoes the per-level rotations. */
static void skilling_axes(uint64_t index, int bits, int nd, uint32_t* x) {
  for (int a = 0; a < nd; ++a) x[a] = 0;
  if (bits == 0) return;
  for (int lvl = 0; lvl < bits; ++lvl) {
    const int shift = (bits - 1 - lvl) * nd;
    const uint64_t group = index >> shift;
    for (int a = 0; a < nd; ++a)
      x[a] |= (uint32_t)((group >> (nd - 1 - a)) & 1u) << (bits - 1 - lvl);
  }
  const uint32_t t = x[nd - 1] >> 1;
  for (int a = nd - 1; a > 0; --a) x[a] ^= x[a - 1];
  x[0] ^= t;
  const uint32_t top = (uint32_t)1 << bits;
  for (uint32_t q = 2; q != top; q <<= 1) {
    const uint32_t p = q - 1;
    for (int a = nd - 1; a >= 0; --a) {
      if (x[a] & q) {
        x[0] ^= p;
      } else {
        const uint32_t s = (x[0] ^ x[a]) & p;
        x[0] ^= s;
        x[a] ^= s;
      }
    }
  }
}

static int check_dims(int64_t f, int64_t h, int64_t w) { /* grid.hpp:21-28 */
  if (f < 1 || h < 1 || w < 1) return -1;
  if (f > ((int64_t)1 << 31) / h / w) return -1;
  return 0;
}

int oracle_order_tokens(int ordering, int64_t f, int64_t h, int64_t w, uint32_t* fwd) {
  if (check_dims(f, h, w)) return -1;
  int64_t pos = 0;
  switch (ordering) {
    case 0: /* raster_order curve.cpp:85-93 */
      for (int64_t i = 0; i < f * h * w; ++i) fwd[i] = (uint32_t)i;
      return 0;
    case 1: { /* hilbert2d_order curve.cpp:114-133: per-frame 2D curve */
      const int bits = ceil_log2(h > w ? h : w);
      const int64_t cells = ((int64_t)1 << bits) * ((int64_t)1 << bits);
      uint32_t a[2];
      for (int64_t t = 0; t < f; ++t)
        for (int64_t dd = 0; dd < cells; ++dd) {
          skilling_axes((uint64_t)dd, bits, 2, a);
          if (a[0] < h && a[1] < w) fwd[pos++] = (uint32_t)((t * h + a[0]) * w + a[1]);
        }
      return 0;
    }
    case 2: /* block3d_order curve.cpp:135-154: 4^3 cubes, local raster */
      for (int64_t ct = 0; ct < f; ct += 4)
        for (int64_t cy = 0; cy < h; cy += 4)
          for (int64_t cx = 0; cx < w; cx += 4)
            for (int64_t t = ct; t < ct + 4 && t < f; ++t)
              for (int64_t y = cy; y < cy + 4 && y < h; ++y)
                for (int64_t x = cx; x < cx + 4 && x < w; ++x)
                  fwd[pos++] = (uint32_t)((t * h + y) * w + x);
      return 0;
    case 3: { /* hilbert3d_order curve.cpp:95-112: enclosing 2^b cube, skip outside */
      int64_t side = f;
      if (h > side) side = h;
      if (w > side) side = w;
      const int bits = ceil_log2(side);
      const int64_t cells = (int64_t)1 << (3 * bits);
      uint32_t a[3];
      for (int64_t dd = 0; dd < cells; ++dd) {
        skilling_axes((uint64_t)dd, bits, 3, a);
        if (a[0] < f && a[1] < h && a[2] < w) fwd[pos++] = (uint32_t)((a[0] * h + a[1]) * w + a[2]);
      }
      return 0;
    }
    default:
      return -1;
  }
}

void oracle_invert_permutation(const uint32_t* fwd, int64_t n, uint32_t* inv) {
  for (int64_t i = 0; i < n; ++i) inv[fwd[i]] = (uint32_t)i; /* curve.cpp:178-185 */
}

int oracle_apply_permutation(const uint32_t* fwd, int64_t n, const float* x, int64_t rows,
                             int64_t cols, float* out) {
  if (n != rows) return -1; /* curve.cpp:167-168 */
  for (int64_t i = 0; i < rows; ++i)
    memcpy(out + i * cols, x + (int64_t)fwd[i] * cols, sizeof(float) * (size_t)cols);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* synthetic inputs — rng.hpp, synthetic.cpp                                 */
/* ------------------------------------------------------------------------ */

static uint64_t sm64(uint64_t* s) { /* rng.hpp:11-17 SplitMix64 */
  uint64_t z = (*s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

uint64_t oracle_derive_seed(uint64_t seed, const uint64_t* path, int npath) { /* rng.hpp:23-31 */
  uint64_t s = seed;
  (void)sm64(&s);
  for (int i = 0; i < npath; ++i) {
    s ^= path[i] + 0x9e3779b97f4a7c15ull + (s << 6) + (s >> 2);
    (void)sm64(&s);
  }
  return s;
}

typedef struct {
  uint64_t state;
  double spare;
  int has_spare;
} gauss_stream;

static double next_gaussian(gauss_stream* g) { /* rng.hpp:57-69 Box-Muller, cached pair */
  if (g->has_spare) {
    g->has_spare = 0;
    return g->spare;
  }
  const double u1 = (double)((sm64(&g->state) >> 11) + 1) * 0x1.0p-53;
  const double u2 = (double)(sm64(&g->state) >> 11) * 0x1.0p-53;
  const double r = sqrt(-2.0 * log(u1));
  const double ang = 2.0 * 3.141592653589793 * u2;
  g->spare = r * sin(ang);
  g->has_spare = 1;
  return r * cos(ang);
}

/* synthetic.cpp:228-263: one boundary-clamped 6-neighbour average (fp64 sum,
 * fp32 store), then re-standardise with a sequential fp64 mean/variance. */
static void smooth_round(float* x, float* tmp, int64_t f, int64_t h, int64_t w, int64_t d) {
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < f; ++t)
    for (int64_t y = 0; y < h; ++y)
      for (int64_t xx = 0; xx < w; ++xx) {
        const int64_t self = (t * h + y) * w + xx;
        const int64_t nb[6] = {
            ((t > 0 ? t - 1 : 0) * h + y) * w + xx,
            ((t + 1 < f ? t + 1 : f - 1) * h + y) * w + xx,
            (t * h + (y > 0 ? y - 1 : 0)) * w + xx,
            (t * h + (y + 1 < h ? y + 1 : h - 1)) * w + xx,
            (t * h + y) * w + (xx > 0 ? xx - 1 : 0),
            (t * h + y) * w + (xx + 1 < w ? xx + 1 : w - 1),
        };
        for (int64_t c = 0; c < d; ++c) {
          double acc = x[self * d + c];
          for (int k = 0; k < 6; ++k) acc += x[nb[k] * d + c];
          tmp[self * d + c] = (float)(acc / 7.0);
        }
      }
  const int64_t total = f * h * w * d;
  double sum = 0.0, sq = 0.0;
  for (int64_t i = 0; i < total; ++i) {
    sum += tmp[i];
    sq += (double)tmp[i] * tmp[i];
  }
  const double nn = (double)total;
  const double var = sq / nn - (sum / nn) * (sum / nn);
  if (var > 0.0) {
    const float inv = (float)(1.0 / sqrt(var));
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < total; ++i) tmp[i] *= inv;
  }
  memcpy(x, tmp, sizeof(float) * (size_t)total);
}

static int field_tensor(int64_t f, int64_t h, int64_t w, int64_t d, double smoothness,
                        uint64_t seed, uint64_t tag, float* x) { /* synthetic.cpp:265-276 */
  const int64_t total = f * h * w * d;
  gauss_stream g = {oracle_derive_seed(seed, &tag, 1), 0.0, 0};
  for (int64_t i = 0; i < total; ++i) x[i] = (float)(1.0 * next_gaussian(&g));
  const long long rounds = llround(smoothness);
  if (rounds > 0) {
    float* tmp = (float*)malloc(sizeof(float) * (size_t)total);
    if (!tmp) return -1;
    for (long long r = 0; r < rounds; ++r) smooth_round(x, tmp, f, h, w, d);
    free(tmp);
  }
  return 0;
}

int oracle_gen_video_field(int64_t f, int64_t h, int64_t w, int64_t d, double smoothness,
                           uint64_t seed, float* q, float* k, float* v) {
  if (check_dims(f, h, w) || d < 1 || smoothness < 0.0) return -1; /* synthetic.cpp:217-221 */
  /* stream tags kTagFieldQ/K/V = 7/8/9 (synthetic.cpp:22-24) */
  if (field_tensor(f, h, w, d, smoothness, seed, 7, q)) return -1;
  if (field_tensor(f, h, w, d, smoothness, seed, 8, k)) return -1;
  if (field_tensor(f, h, w, d, smoothness, seed, 9, v)) return -1;
  return 0;
}

int oracle_trajectory_at(int64_t f, int64_t h, int64_t w, int64_t d, double smoothness,
                         uint64_t seed, int steps, double noise_start, double noise_end, int step,
                         float* q, float* k, float* v) { /* synthetic.cpp:293-321 */
  if (steps < 1 || !(noise_start >= noise_end) || noise_end < 0.0) return -1;
  if (step < 0 || step >= steps) return -2;
  int rc = oracle_gen_video_field(f, h, w, d, smoothness, seed, q, k, v);
  if (rc) return rc;
  double sd = noise_start;
  if (steps > 1) sd = noise_start + (noise_end - noise_start) * ((double)step / (double)(steps - 1));
  if (sd > 0.0) {
    const int64_t total = f * h * w * d;
    float* xs[3] = {q, k, v};
    for (int which = 0; which < 3; ++which) {
      const uint64_t path[3] = {10, (uint64_t)(7 + which), (uint64_t)step}; /* kTagStepNoise */
      gauss_stream g = {oracle_derive_seed(seed, path, 3), 0.0, 0};
      for (int64_t i = 0; i < total; ++i) xs[which][i] += (float)(sd * next_gaussian(&g));
    }
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* score / mask — mask_builder.cpp, attention.cpp:105-123                     */
/* ------------------------------------------------------------------------ */

static int all_finite(const float* x, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (!isfinite(x[i])) return 0;
  return 1;
}

int oracle_mean_pool(const float* x, int64_t rows, int64_t cols, int64_t pool, float* out) {
  if (pool < 1 || rows < 1) return -1; /* mask_builder.cpp:13-14 */
  const int64_t groups = (rows + pool - 1) / pool;
  for (int64_t g = 0; g < groups; ++g) {
    const int64_t lo = g * pool, hi = lo + pool < rows ? lo + pool : rows;
    for (int64_t c = 0; c < cols; ++c) {
      double acc = 0.0;
      for (int64_t i = lo; i < hi; ++i) acc += x[i * cols + c];
      out[g * cols + c] = (float)(acc / (double)pool); /* divides by B_s even when partial */
    }
  }
  return 0;
}

/* attend_row's softmax without V (attention.cpp:32-60 with v == nullptr):
 * fp64 logits, max-subtract, exp, normalise, round each p to fp32. */
static void softmax_row_f32(const float* qrow, const float* keys, int64_t nk, int64_t d,
                            double scale, double* work, float* p) {
  double mx = -INFINITY;
  for (int64_t j = 0; j < nk; ++j) {
    double acc = 0.0;
    for (int64_t c = 0; c < d; ++c) acc += (double)qrow[c] * keys[j * d + c];
    work[j] = acc * scale;
    if (work[j] > mx) mx = work[j];
  }
  double z = 0.0;
  for (int64_t j = 0; j < nk; ++j) {
    work[j] = exp(work[j] - mx);
    z += work[j];
  }
  for (int64_t j = 0; j < nk; ++j) p[j] = (float)(work[j] / z);
}

typedef struct {
  int64_t subs, mq, qrows, kcols, valid_k;
  float* pq; /* [qrows, d], zero padded (mask_builder.cpp:40-49) */
  float* pk; /* [valid_k, d] */
} pooled_t;

static int pool_inputs(const float* q, const float* k, int64_t n, int64_t d, int64_t b,
                       int64_t bs, pooled_t* P) {
  if (bs < 1 || b < bs || b % bs) return -1; /* mask_builder.hpp:17-22 */
  if (!all_finite(q, n * d) || !all_finite(k, n * d)) return -1; /* attention.cpp:110-111 */
  P->subs = b / bs;
  P->mq = (n + b - 1) / b;
  P->qrows = P->mq * P->subs;
  P->kcols = P->qrows; /* q and k have the same length here */
  P->valid_k = (n + bs - 1) / bs;
  P->pq = (float*)calloc((size_t)(P->qrows * d), sizeof(float));
  P->pk = (float*)calloc((size_t)(P->valid_k * d), sizeof(float));
  if (!P->pq || !P->pk) return -1;
  oracle_mean_pool(q, n, d, bs, P->pq);
  oracle_mean_pool(k, n, d, bs, P->pk);
  return 0;
}

int oracle_subblock_scores(const float* q, const float* k, int64_t n, int64_t d, int64_t b,
                           int64_t bs, float* out) { /* mask_builder.cpp:30-62 */
  pooled_t P;
  if (n < 1 || pool_inputs(q, k, n, d, b, bs, &P)) return -1;
  const double scale = 1.0 / sqrt((double)d);
  memset(out, 0, sizeof(float) * (size_t)(P.qrows * P.kcols));
#pragma omp parallel
  {
    double* work = (double*)malloc(sizeof(double) * (size_t)P.valid_k);
#pragma omp for schedule(dynamic, 4)
    for (int64_t i = 0; i < P.qrows; ++i)
      softmax_row_f32(P.pq + i * d, P.pk, P.valid_k, d, scale, work, out + i * P.kcols);
    free(work);
  }
  free(P.pq);
  free(P.pk);
  return 0;
}

/* block_scores = aggregate_scores(subblock_scores) (mask_builder.cpp:64-80,115-117),
 * fused so the P x P matrix is never stored: per query block u the fp64 tile
 * accumulators are fed sub-row by sub-row, column by column — the same
 * addition sequence as aggregate_scores' (i, j) loop. */
int oracle_block_scores(const float* q, const float* k, int64_t n, int64_t d, int64_t b,
                        int64_t bs, double* s) {
  pooled_t P;
  if (n < 1 || pool_inputs(q, k, n, d, b, bs, &P)) return -1;
  const double scale = 1.0 / sqrt((double)d);
  const int64_t mq = P.mq, subs = P.subs;
#pragma omp parallel
  {
    double* work = (double*)malloc(sizeof(double) * (size_t)P.valid_k);
    float* prow = (float*)malloc(sizeof(float) * (size_t)P.valid_k);
#pragma omp for schedule(dynamic, 1)
    for (int64_t u = 0; u < mq; ++u) {
      double* acc = s + u * mq;
      for (int64_t v = 0; v < mq; ++v) acc[v] = 0.0;
      for (int64_t r = 0; r < subs; ++r) {
        const int64_t i = u * subs + r;
        softmax_row_f32(P.pq + i * d, P.pk, P.valid_k, d, scale, work, prow);
        for (int64_t j = 0; j < P.valid_k; ++j) acc[j / subs] += (double)prow[j];
      }
    }
    free(work);
    free(prow);
  }
  free(P.pq);
  free(P.pk);
  return 0;
}

int oracle_topk_count(double budget, int64_t m, int64_t* k) { /* mask_builder.cpp:82-87 */
  if (!(budget > 0.0) || budget > 1.0) return -1;
  long long kk = llround(budget * (double)m);
  if (kk < 1) kk = 1;
  if (kk > m) kk = m;
  *k = kk;
  return 0;
}

typedef struct {
  double v;
  int32_t i;
} scored_t;

static int by_value_desc_index_asc(const void* a, const void* b) { /* mask_builder.cpp:94-98 */
  const scored_t* x = (const scored_t*)a;
  const scored_t* y = (const scored_t*)b;
  if (x->v != y->v) return x->v > y->v ? -1 : 1;
  return x->i < y->i ? -1 : (x->i > y->i);
}

static int by_index(const void* a, const void* b) {
  const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return x < y ? -1 : (x > y);
}

/* topk_select (mask_builder.cpp:91-113): K best per row under (value desc,
 * index asc), reported ascending. bits may be NULL; lut [m, K] may be NULL. */
int oracle_topk_select(const double* s, int64_t m, double budget, uint8_t* bits, int32_t* lut) {
  int64_t K;
  if (m < 1 || oracle_topk_count(budget, m, &K)) return -1;
  if (bits) memset(bits, 0, (size_t)((m * m + 7) / 8));
#pragma omp parallel
  {
    scored_t* row = (scored_t*)malloc(sizeof(scored_t) * (size_t)m);
    int32_t* pick = (int32_t*)malloc(sizeof(int32_t) * (size_t)K);
#pragma omp for schedule(dynamic, 8)
    for (int64_t u = 0; u < m; ++u) {
      for (int64_t v = 0; v < m; ++v) {
        row[v].v = s[u * m + v];
        row[v].i = (int32_t)v;
      }
      qsort(row, (size_t)m, sizeof(scored_t), by_value_desc_index_asc);
      for (int64_t t = 0; t < K; ++t) pick[t] = row[t].i;
      qsort(pick, (size_t)K, sizeof(int32_t), by_index);
      for (int64_t t = 0; t < K; ++t) {
        if (lut) lut[u * K + t] = pick[t];
        if (bits) {
          const int64_t idx = u * m + pick[t];
#pragma omp atomic
          bits[idx >> 3] |= (uint8_t)(1u << (7 - (idx & 7)));
        }
      }
    }
    free(row);
    free(pick);
  }
  return 0;
}

int oracle_build_mask(const float* q, const float* k, int64_t n, int64_t d, int64_t b, int64_t bs,
                      double budget, uint8_t* bits) { /* mask_builder.cpp:119-124 */
  const int64_t m = (n + b - 1) / b;
  double* s = (double*)malloc(sizeof(double) * (size_t)(m * m));
  if (!s) return -1;
  int rc = oracle_block_scores(q, k, n, d, b, bs, s);
  if (!rc) rc = oracle_topk_select(s, m, budget, bits, NULL);
  free(s);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* attention — attention.cpp                                                  */
/* ------------------------------------------------------------------------ */

/* attend_row (attention.cpp:32-60) with an explicit key list. */
static void attend_row(const float* qrow, const float* k, const float* v, const int64_t* keys,
                       int64_t nk, int64_t d, double scale, double* logits, double* acc,
                       float* out) {
  double mx = -INFINITY;
  for (int64_t j = 0; j < nk; ++j) {
    const float* kr = k + keys[j] * d;
    double a = 0.0;
    for (int64_t c = 0; c < d; ++c) a += (double)qrow[c] * kr[c];
    logits[j] = a * scale;
    if (logits[j] > mx) mx = logits[j];
  }
  double z = 0.0;
  for (int64_t j = 0; j < nk; ++j) {
    logits[j] = exp(logits[j] - mx);
    z += logits[j];
  }
  for (int64_t c = 0; c < d; ++c) acc[c] = 0.0;
  for (int64_t j = 0; j < nk; ++j) {
    const double p = logits[j] / z;
    const float* vr = v + keys[j] * d;
    for (int64_t c = 0; c < d; ++c) acc[c] += p * vr[c];
  }
  for (int64_t c = 0; c < d; ++c) out[c] = (float)acc[c];
}

static int mask_get(const uint8_t* bits, int64_t m, int64_t u, int64_t v) {
  const int64_t idx = u * m + v;
  return (bits[idx >> 3] >> (7 - (idx & 7))) & 1;
}

/* block_sparse_attention (attention.cpp:125-159); rows [row_lo, row_hi) only
 * (out is still indexed by absolute row). */
int oracle_block_sparse_attention(const float* q, const float* k, const float* v, int64_t n,
                                  int64_t d, const uint8_t* bits, int64_t m, int64_t b,
                                  int64_t row_lo, int64_t row_hi, float* out) {
  if (n < 1 || d < 1 || b < 1) return -1;
  if (!all_finite(q, n * d) || !all_finite(k, n * d) || !all_finite(v, n * d)) return -1;
  if ((n + b - 1) / b != m) return -1; /* check_mask_geometry :68-73 */
  for (int64_t u = 0; u < m; ++u) {    /* empty rows :133-136 */
    int any = 0;
    for (int64_t vb = 0; vb < m && !any; ++vb) any = mask_get(bits, m, u, vb);
    if (!any) return -1;
  }
  if (row_lo < 0) row_lo = 0;
  if (row_hi > n || row_hi < 0) row_hi = n;
  const double scale = 1.0 / sqrt((double)d);
  const int64_t ublo = row_lo / b, ubhi = (row_hi + b - 1) / b;
#pragma omp parallel
  {
    int64_t* keys = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m * b));
    double* logits = (double*)malloc(sizeof(double) * (size_t)(m * b));
    double* acc = (double*)malloc(sizeof(double) * (size_t)d);
#pragma omp for schedule(dynamic, 1)
    for (int64_t u = ublo; u < ubhi; ++u) {
      int64_t nk = 0;
      for (int64_t vb = 0; vb < m; ++vb) {
        if (!mask_get(bits, m, u, vb)) continue;
        for (int64_t j = vb * b; j < vb * b + b && j < n; ++j) keys[nk++] = j; /* :147-152 */
      }
      for (int64_t i = u * b; i < u * b + b && i < n; ++i) {
        if (i < row_lo || i >= row_hi) continue;
        attend_row(q + i * d, k, v, keys, nk, d, scale, logits, acc, out + i * d);
      }
    }
    free(keys);
    free(logits);
    free(acc);
  }
  return 0;
}

int oracle_full_attention_output(const float* q, int64_t nq, const float* k, const float* v,
                                 int64_t nk, int64_t d, int64_t row_lo, int64_t row_hi,
                                 float* out) { /* attention.cpp:95-103 */
  if (nq < 1 || nk < 1 || d < 1) return -1;
  if (!all_finite(q, nq * d) || !all_finite(k, nk * d) || !all_finite(v, nk * d)) return -1;
  if (row_lo < 0) row_lo = 0;
  if (row_hi > nq || row_hi < 0) row_hi = nq;
  const double scale = 1.0 / sqrt((double)d);
  int64_t* keys = (int64_t*)malloc(sizeof(int64_t) * (size_t)nk);
  for (int64_t j = 0; j < nk; ++j) keys[j] = j;
#pragma omp parallel
  {
    double* logits = (double*)malloc(sizeof(double) * (size_t)nk);
    double* acc = (double*)malloc(sizeof(double) * (size_t)d);
#pragma omp for schedule(dynamic, 16)
    for (int64_t i = row_lo; i < row_hi; ++i)
      attend_row(q + i * d, k, v, keys, nk, d, scale, logits, acc, out + i * d);
    free(logits);
    free(acc);
  }
  free(keys);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* schedule — scheduler.cpp:18-56                                             */
/* ------------------------------------------------------------------------ */

int oracle_schedule(int total, double warmup, const double* budgets, int nb, double phase,
                    int interval, double* budget_out, uint8_t* update_out, int* warmup_steps,
                    int* phase_length) {
  const double eps = 1e-9;
  if (total < 1 || warmup < 0.0 || warmup > 1.0 || phase < 0.0 || phase > 1.0 || interval < 1)
    return -1;
  for (int i = 0; i < nb; ++i)
    if (!(budgets[i] > 0.0) || budgets[i] > 1.0) return -1;
  if (warmup + (double)nb * phase > 1.0 + eps) return -1;
  const double t = (double)total;
  int ws = (int)floor(warmup * t + eps); /* floor, scheduler.cpp:36 */
  if (ws > total) ws = total;
  if (ws < total && nb == 0) return -1;
  int pl = (int)ceil(phase * t - eps);
  if (pl < 1) pl = 1;
  for (int s = 0; s < total; ++s) {
    if (s < ws) {
      budget_out[s] = -1.0;
      update_out[s] = 0;
      continue;
    }
    int ph = (s - ws) / pl;
    if (ph > nb - 1) ph = nb - 1;
    budget_out[s] = budgets[ph];
    update_out[s] = ((s - ws) % interval) == 0;
  }
  *warmup_steps = ws;
  *phase_length = pl;
  return 0;
}

int oracle_threads(void) { return omp_get_max_threads(); }
