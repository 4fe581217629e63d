// oracle/ref_harness.cpp — TEST INFRASTRUCTURE ONLY (never shipped, never on the product path).
//
// A flat extern "C" veneer over the UNMODIFIED reference library built from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libdfsref.so.
// It lets the Python tests, the golden-fixture generator and bench.py's
// reference arm call the reference's own public dfs:: API (curve.hpp,
// mask_builder.hpp, attention.hpp, scheduler.hpp, synthetic.hpp) on plain
// arrays. Every function forwards to exactly one reference entry point (named
// in its comment); nothing here re-implements reference arithmetic.
//
// Status codes mirror include/dfs_gpu.h: 0 ok, -1 invalid_argument,
// -2 out_of_range, -5 anything else. dfsref_last_error() gives the message.

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "dfs/attention.hpp"
#include "dfs/curve.hpp"
#include "dfs/mask_builder.hpp"
#include "dfs/metrics.hpp"
#include "dfs/parallel.hpp"
#include "dfs/rng.hpp"
#include "dfs/scheduler.hpp"
#include "dfs/synthetic.hpp"

using namespace dfs;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return -1;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return -2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -5;
  }
}

Matrix to_matrix(const float* p, int64_t rows, int64_t cols) {
  Matrix m(rows, cols);
  if (rows * cols > 0) std::memcpy(m.values().data(), p, sizeof(float) * rows * cols);
  return m;
}

void from_matrix(const Matrix& m, float* out) {
  std::memcpy(out, m.values().data(), sizeof(float) * m.size());
}

BlockMask to_mask(const uint8_t* bits, int64_t m, int64_t b) {
  BlockMask mask(m, b);
  std::memcpy(mask.bytes().data(), bits, mask.bytes().size());
  return mask;
}

void from_mask(const BlockMask& mask, uint8_t* out) {
  std::memcpy(out, mask.bytes().data(), mask.bytes().size());
}

SparsitySchedule make_schedule(int total, double warmup, const double* budgets, int nb,
                               double phase, int interval) {
  SparsitySchedule::Config c;
  c.total_steps = total;
  c.warmup_fraction = warmup;
  c.phase_budgets.assign(budgets, budgets + nb);
  c.phase_fraction = phase;
  c.update_interval = interval;
  return SparsitySchedule(c);
}

}  // namespace

extern "C" {

const char* dfsref_last_error(void) { return g_err.c_str(); }

// curve.cpp:156 order_tokens (ordering: 0 raster, 1 hilbert2d, 2 block3d, 3 hilbert3d)
int dfsref_order_tokens(int ordering, int64_t f, int64_t h, int64_t w, uint32_t* fwd) {
  return guarded([&] {
    const Permutation p = order_tokens(static_cast<Ordering>(ordering), GridDims{f, h, w});
    std::copy(p.forward.begin(), p.forward.end(), fwd);
  });
}

// curve.cpp:178 invert_permutation
int dfsref_invert_permutation(const uint32_t* fwd, int64_t n, uint32_t* inv) {
  return guarded([&] {
    Permutation p;
    p.forward.assign(fwd, fwd + n);
    const Permutation q = invert_permutation(p);
    std::copy(q.forward.begin(), q.forward.end(), inv);
  });
}

// curve.cpp:166 apply_permutation
int dfsref_apply_permutation(const uint32_t* fwd, int64_t n, const float* x, int64_t rows,
                             int64_t cols, float* out) {
  return guarded([&] {
    Permutation p;
    p.forward.assign(fwd, fwd + n);
    from_matrix(apply_permutation(p, to_matrix(x, rows, cols)), out);
  });
}

// rng.hpp:23 derive_seed (path of up to 4 words)
uint64_t dfsref_derive_seed(uint64_t seed, const uint64_t* path, int npath) {
  uint64_t s = seed;
  (void)splitmix64_next(s);
  // identical to derive_seed's loop; initializer_list cannot be built at run time
  for (int i = 0; i < npath; ++i) {
    s ^= path[i] + 0x9e3779b97f4a7c15ull + (s << 6) + (s >> 2);
    (void)splitmix64_next(s);
  }
  return s;
}

// rng.hpp:35 RandomStream::next_gaussian, n draws from RandomStream(seed)
void dfsref_gaussians(uint64_t seed, int64_t n, double* out) {
  RandomStream s(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = s.next_gaussian();
}

// synthetic.cpp:280 gen_video_field — q, k, v raster [N, d]
int dfsref_gen_video_field(int64_t f, int64_t h, int64_t w, int64_t d, double smoothness,
                           uint64_t seed, float* q, float* k, float* v) {
  return guarded([&] {
    synthetic::FieldParams p;
    p.dims = GridDims{f, h, w};
    p.head_dim = d;
    p.smoothness = smoothness;
    p.seed = seed;
    const auto s = synthetic::gen_video_field(p);
    from_matrix(s.q, q);
    from_matrix(s.k, k);
    from_matrix(s.v, v);
  });
}

// synthetic.cpp:306 DenoisingTrajectory::at
int dfsref_trajectory_at(int64_t f, int64_t h, int64_t w, int64_t d, double smoothness,
                         uint64_t seed, int steps, double noise_start, double noise_end,
                         int step, float* q, float* k, float* v) {
  return guarded([&] {
    synthetic::TrajectoryParams tp;
    tp.field.dims = GridDims{f, h, w};
    tp.field.head_dim = d;
    tp.field.smoothness = smoothness;
    tp.field.seed = seed;
    tp.steps = steps;
    tp.noise_start = noise_start;
    tp.noise_end = noise_end;
    const synthetic::DenoisingTrajectory traj(tp);
    const auto s = traj.at(step);
    from_matrix(s.q, q);
    from_matrix(s.k, k);
    from_matrix(s.v, v);
  });
}

// mask_builder.cpp:12 mean_pool
int dfsref_mean_pool(const float* x, int64_t rows, int64_t cols, int64_t pool, float* out) {
  return guarded([&] { from_matrix(mean_pool(to_matrix(x, rows, cols), pool), out); });
}

// mask_builder.cpp:30 subblock_scores — out [mq*subs, mk*subs]
int dfsref_subblock_scores(const float* q, const float* k, int64_t n, int64_t d, int64_t b,
                           int64_t bs, float* out) {
  return guarded([&] {
    from_matrix(subblock_scores(to_matrix(q, n, d), to_matrix(k, n, d), ScoringParams{b, bs}),
                out);
  });
}

// mask_builder.cpp:115 block_scores — S [M, M] fp64
int dfsref_block_scores(const float* q, const float* k, int64_t n, int64_t d, int64_t b,
                        int64_t bs, double* s) {
  return guarded([&] {
    const MatrixD m = block_scores(to_matrix(q, n, d), to_matrix(k, n, d), ScoringParams{b, bs});
    std::copy(m.values().begin(), m.values().end(), s);
  });
}

// mask_builder.cpp:82 topk_count
int dfsref_topk_count(double budget, int64_t m, int64_t* k) {
  return guarded([&] { *k = topk_count(budget, m); });
}

// mask_builder.cpp:104 topk_select — bits = BlockMask bytes (MSB-first)
int dfsref_topk_select(const double* s, int64_t m, double budget, int64_t b, uint8_t* bits) {
  return guarded([&] {
    MatrixD sc(m, m);
    for (int64_t u = 0; u < m; ++u)
      for (int64_t v = 0; v < m; ++v) sc.at(u, v) = s[u * m + v];
    from_mask(topk_select(sc, budget, b), bits);
  });
}

// mask_builder.cpp:119 build_mask
int dfsref_build_mask(const float* q, const float* k, int64_t n, int64_t d, int64_t b,
                      int64_t bs, double budget, uint8_t* bits) {
  return guarded([&] {
    from_mask(build_mask(to_matrix(q, n, d), to_matrix(k, n, d), ScoringParams{b, bs}, budget),
              bits);
  });
}

// attention.cpp:125 block_sparse_attention
int dfsref_block_sparse_attention(const float* q, const float* k, const float* v, int64_t n,
                                  int64_t d, const uint8_t* bits, int64_t m, int64_t b,
                                  float* out) {
  return guarded([&] {
    from_matrix(block_sparse_attention(to_matrix(q, n, d), to_matrix(k, n, d), to_matrix(v, n, d),
                                       to_mask(bits, m, b)),
                out);
  });
}

// attention.cpp:95 full_attention_output (Nq != Nk allowed)
int dfsref_full_attention_output(const float* q, int64_t nq, const float* k, const float* v,
                                 int64_t nk, int64_t d, float* out) {
  return guarded([&] {
    from_matrix(full_attention_output(to_matrix(q, nq, d), to_matrix(k, nk, d),
                                      to_matrix(v, nk, d)),
                out);
  });
}

// scheduler.cpp:18-56 SparsitySchedule: budget_at (-1 = dense) and is_update_step per step
int dfsref_schedule(int total, double warmup, const double* budgets, int nb, double phase,
                    int interval, double* budget_out, uint8_t* update_out, int* warmup_steps,
                    int* phase_length) {
  return guarded([&] {
    const SparsitySchedule s = make_schedule(total, warmup, budgets, nb, phase, interval);
    for (int t = 0; t < total; ++t) {
      const auto b = s.budget_at(t);
      budget_out[t] = b ? *b : -1.0;
      update_out[t] = s.is_update_step(t) ? 1 : 0;
    }
    *warmup_steps = s.warmup_steps();
    *phase_length = s.phase_length();
  });
}

// scheduler.cpp:137 run_trajectory over cmd_run's synthetic workload
// (commands.cpp:258-272: one DenoisingTrajectory per (layer, head) pair seeded
// derive_seed(seed, {pair})). Per row (step-major, then layer, head):
// budget, sparsity, flags (bit0 dense, bit1 mask_updated). Masks of updated
// rows go to masks[row * mask_bytes]. Outputs of (layer 0, head 0) for every
// step go to out00 [steps, N, d] when non-null.
int dfsref_run_trajectory(int ordering, int64_t f, int64_t h, int64_t w, int64_t d, int layers,
                          int heads, int total, double warmup, const double* budgets, int nb,
                          double phase, int interval, int64_t b, int64_t bs, uint64_t seed,
                          double smoothness, double noise_start, double noise_end, int threads,
                          const int* dense_layers, int n_dense, double* row_budget,
                          double* row_sparsity, uint8_t* row_flags, uint8_t* masks,
                          float* out00) {
  return guarded([&] {
    const GridDims dims{f, h, w};
    const SparsitySchedule schedule = make_schedule(total, warmup, budgets, nb, phase, interval);
    std::vector<synthetic::DenoisingTrajectory> trajs;
    for (int pair = 0; pair < layers * heads; ++pair) {
      synthetic::TrajectoryParams tp;
      tp.field.dims = dims;
      tp.field.head_dim = d;
      tp.field.smoothness = smoothness;
      tp.field.seed = derive_seed(seed, {static_cast<uint64_t>(pair)});
      tp.steps = total;
      tp.noise_start = noise_start;
      tp.noise_end = noise_end;
      trajs.emplace_back(tp);
    }
    Workload wl;
    wl.steps = total;
    wl.layers = layers;
    wl.heads = heads;
    wl.tensors = [&](int step, int layer, int head) {
      const auto s = trajs[static_cast<size_t>(layer * heads + head)].at(step);
      return StepTensors{s.q, s.k, s.v};
    };
    TrajectoryOptions opt;
    opt.record_recall = false;
    opt.threads = threads;
    for (int i = 0; i < n_dense; ++i) opt.dense_layers.insert(dense_layers[i]);
    const int64_t mblocks = block_count_for(dims.token_count(), b);
    const int64_t mbytes = BlockMask::byte_size(mblocks);
    const int pairs = layers * heads;
    opt.mask_sink = [&](int step, int layer, int head, const BlockMask& m) {
      const int64_t row = static_cast<int64_t>(step) * pairs + layer * heads + head;
      std::memcpy(masks + row * mbytes, m.bytes().data(), static_cast<size_t>(mbytes));
    };
    if (out00)
      opt.output_sink = [&](int step, int layer, int head, const Matrix& o) {
        if (layer == 0 && head == 0)
          std::memcpy(out00 + static_cast<int64_t>(step) * o.size(), o.values().data(),
                      sizeof(float) * o.size());
      };
    const auto rows = run_trajectory(wl, order_tokens(static_cast<Ordering>(ordering), dims),
                                     ScoringParams{b, bs}, schedule, opt);
    for (size_t i = 0; i < rows.size(); ++i) {
      row_budget[i] = rows[i].budget;
      row_sparsity[i] = rows[i].sparsity;
      row_flags[i] = (rows[i].dense ? 1 : 0) | (rows[i].mask_updated ? 2 : 0);
    }
  });
}

// ---------------------------------------------------------------------------
// Bounded CPU-baseline sample of the reference path (bench.py reference arm).
//
// A full HunyuanVideo call costs ~2.4 core-hours in the reference, so the
// bench times a sample of (head, query block) units and extrapolates. For one
// unit u of head h the reference arithmetic is reproduced EXACTLY by the
// reference's own public functions:
//   scoring: attention_scores over the unit's pooled query rows against every
//            pooled key (the same attend_row calls subblock_scores makes for
//            those rows, attention.cpp:105), then aggregate over the unit's
//            sub-block tiles;
//   attend:  full_attention_output(q_u, K_sel, V_sel) with K_sel the keys of
//            the unit's selected blocks gathered in ascending order — the key
//            list block_sparse_attention builds (attention.cpp:146-156).
// Per head the harness also runs the full-N reorder (hilbert3d_order,
// apply_permutation x3) and the inverse permute once. Q/K/V are iid normal
// (content does not change the reference's op count).
// dfsref_sample_prepare / _run / _free below implement it.
struct SampleCtx {
  GridDims dims;
  int64_t n = 0, d = 0, b = 0, bs = 0, m = 0, kk = 0, subs = 0;
  std::vector<Matrix> qs, ks, vs;
};

// Inputs for `heads` heads (iid normal, per-head seeds), generated in parallel.
void* dfsref_sample_prepare(int64_t f, int64_t h, int64_t w, int64_t d, int64_t b, int64_t bs, double budget,
                            int heads, int threads) {
  auto* c = new SampleCtx;
  c->dims = GridDims{f, h, w};
  c->n = c->dims.token_count();
  c->d = d;
  c->b = b;
  c->bs = bs;
  c->m = block_count_for(c->n, b);
  c->kk = topk_count(budget, c->m);
  c->subs = b / bs;
  c->qs.resize(static_cast<size_t>(heads));
  c->ks.resize(static_cast<size_t>(heads));
  c->vs.resize(static_cast<size_t>(heads));
  parallel_for(heads, threads, [&](int64_t hh) {
    RandomStream s(derive_seed(7, {static_cast<uint64_t>(hh)}));
    Matrix q(c->n, d), k(c->n, d), v(c->n, d);
    for (float& x : q.values()) x = static_cast<float>(s.next_gaussian());
    for (float& x : k.values()) x = static_cast<float>(s.next_gaussian());
    for (float& x : v.values()) x = static_cast<float>(s.next_gaussian());
    c->qs[static_cast<size_t>(hh)] = std::move(q);
    c->ks[static_cast<size_t>(hh)] = std::move(k);
    c->vs[static_cast<size_t>(hh)] = std::move(v);
  });
  return c;
}

void dfsref_sample_free(void* ctx) { delete static_cast<SampleCtx*>(ctx); }

// One timed sample: per head the full reorder + pooled keys, then
// `units_per_head` query blocks through scoring + selection + attention.
int dfsref_sample_run(void* ctx, int units_per_head, int threads, double* seconds, double* seconds_fixed) {
  return guarded([&] {
    SampleCtx& c = *static_cast<SampleCtx*>(ctx);
    const int heads = static_cast<int>(c.qs.size());
    const int64_t n = c.n, d = c.d, b = c.b, bs = c.bs, m = c.m, kk = c.kk, subs = c.subs;
    const auto t0 = std::chrono::steady_clock::now();
    // per head, once: reorder + inverse (curve.cpp:95,166,178) and the pooled
    // keys every unit of the head scores against (mask_builder.cpp:12)
    std::vector<Matrix> pks(static_cast<size_t>(heads));
    parallel_for(heads, threads, [&](int64_t hh) {
      const Permutation p = hilbert3d_order(c.dims);
      const Matrix rq = apply_permutation(p, c.qs[static_cast<size_t>(hh)]);
      const Matrix rk = apply_permutation(p, c.ks[static_cast<size_t>(hh)]);
      const Matrix rv = apply_permutation(p, c.vs[static_cast<size_t>(hh)]);
      (void)apply_permutation(invert_permutation(p), rv);
      pks[static_cast<size_t>(hh)] = mean_pool(c.ks[static_cast<size_t>(hh)], bs);
    });
    const auto tf = std::chrono::steady_clock::now();
    if (seconds_fixed) *seconds_fixed = std::chrono::duration<double>(tf - t0).count();
    parallel_for(static_cast<int64_t>(heads) * units_per_head, threads, [&](int64_t item) {
      const int hh = static_cast<int>(item / units_per_head);
      const int64_t slot = item % units_per_head;
      const int64_t u = (slot * m) / units_per_head;  // spread the sampled units over the head
      const Matrix& q = c.qs[static_cast<size_t>(hh)];
      const Matrix& k = c.ks[static_cast<size_t>(hh)];
      const Matrix& v = c.vs[static_cast<size_t>(hh)];
      const Matrix& pk = pks[static_cast<size_t>(hh)];
      // scoring for block u (mask_builder.cpp:12,30,64; attention.cpp:105): the
      // unit's pooled query rows, zero rows past the end (mask_builder.cpp:40-49)
      const int64_t qlo = u * b, qhi = std::min(qlo + b, n);
      Matrix xq(qhi - qlo, d);
      for (int64_t i = qlo; i < qhi; ++i)
        for (int64_t cc = 0; cc < d; ++cc) xq.at(i - qlo, cc) = q.at(i, cc);
      const Matrix pq_part = mean_pool(xq, bs);
      Matrix pq(subs, d);
      for (int64_t r = 0; r < pq_part.rows(); ++r)
        for (int64_t cc = 0; cc < d; ++cc) pq.at(r, cc) = pq_part.at(r, cc);
      const Matrix sc = attention_scores(pq, pk);
      std::vector<double> row(static_cast<size_t>(m), 0.0);
      for (int64_t r = 0; r < subs; ++r)
        for (int64_t j = 0; j < pk.rows(); ++j) row[static_cast<size_t>(j / subs)] += sc.at(r, j);
      const auto sel = top_indices(row, kk);
      // attention for block u (attention.cpp:146-156 key list, attend_row)
      std::vector<int64_t> keys;
      for (int32_t vb : sel)
        for (int64_t j = vb * b; j < std::min((vb + 1) * b, n); ++j) keys.push_back(j);
      Matrix ksel(static_cast<int64_t>(keys.size()), d), vsel(static_cast<int64_t>(keys.size()), d);
      for (size_t j = 0; j < keys.size(); ++j)
        for (int64_t cc = 0; cc < d; ++cc) {
          ksel.at(static_cast<int64_t>(j), cc) = k.at(keys[j], cc);
          vsel.at(static_cast<int64_t>(j), cc) = v.at(keys[j], cc);
        }
      (void)full_attention_output(xq, ksel, vsel);
    });
    const auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - tf).count();  // the sampled units only
  });
}

int dfsref_hardware_threads(void) { return auto_threads(0); }

}  // extern "C"
