// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY (never shipped, never timed
// as the product).
//
// A thin extern "C" shim over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled from where it lies by
// oracle/Makefile into oracle/_ref/libsparsim_ref.so). It exposes the
// reference's own functions and its Engine to ctypes so that
//   * the C restatement in oracle/exdyna_oracle.c can be pinned bit for bit
//     against the reference in fp64 mode, and
//   * bench.py --impl reference / cpu_baseline can time the reference's own
//     Engine::step() (engine.cpp:274-350) on the host cores.
// Gradients reach the reference Engine through a replay GradientSource that
// follows the FixedSource pattern of test_engine.cpp:29-48.

#include <algorithm>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "exdyna.h"
#include "sparsim/allocator.hpp"
#include "sparsim/baselines.hpp"
#include "sparsim/collectives.hpp"
#include "sparsim/config.hpp"
#include "sparsim/engine.hpp"
#include "sparsim/partition.hpp"
#include "sparsim/runner.hpp"
#include "sparsim/selector.hpp"
#include "sparsim/threshold.hpp"
#include "sparsim/workloads.hpp"

using namespace sparsim;

namespace {

thread_local std::string g_err;

int fail(int code, const char* what) {
  g_err = what;
  return code;
}

SparsifierConfig to_cfg(const exd_config* c) {
  SparsifierConfig cfg;
  cfg.n = c->n;
  cfg.n_g = c->n_g;
  cfg.n_b = c->n_b;
  cfg.d = c->d;
  cfg.k = c->k;
  if (c->has_delta0) cfg.delta0 = c->delta0;
  cfg.alpha = c->alpha;
  cfg.beta = c->beta;
  cfg.gamma = c->gamma;
  cfg.blk_move = c->blk_move;
  cfg.min_blk = c->min_blk;
  cfg.eta = c->eta;
  cfg.seed = c->seed;
  if (c->has_max_density_cap) cfg.max_density_cap = c->max_density_cap;
  return cfg;
}

void from_topo(const PartitionTopology& t, exd_topology* out) {
  std::memset(out, 0, sizeof(*out));
  out->n = t.partitions();
  out->sz_blk = t.sz_blk;
  for (int i = 0; i < out->n; ++i) {
    out->blk_part[i] = t.blk_part[i];
    out->blk_pos[i] = t.blk_pos[i];
  }
}

PartitionTopology to_topo(const exd_topology* t) {
  PartitionTopology out;
  out.sz_blk = t->sz_blk;
  out.blk_part.assign(t->blk_part, t->blk_part + t->n);
  out.blk_pos.assign(t->blk_pos, t->blk_pos + t->n);
  return out;
}

void fill_record(const IterationRecord& r, exd_record* o) {
  std::memset(o, 0, sizeof(*o));
  o->t = r.t;
  o->k_prime = r.k_prime;
  o->density = r.density;
  o->eps = r.eps;
  o->m_t = r.m_t;
  o->c_t = r.c_t;
  o->f_t = r.f_t;
  o->global_err = r.global_err;
  o->delta = r.delta;
  o->has_loss = r.loss.has_value() ? 1 : 0;
  o->loss = r.loss.value_or(0.0);
  o->duplicates = r.duplicates;
  o->union_count = r.union_count;
  o->n = static_cast<int32_t>(r.k_rank.size());
  o->adjust_moves = r.adjust_moves;
  o->adjust_skips = r.adjust_skips;
  o->cap_hits = r.cap_hits;
  o->idle_workers = r.idle_workers;
  for (size_t i = 0; i < r.k_rank.size() && i < EXD_MAX_WORKERS; ++i) {
    o->k_rank[i] = r.k_rank[i];
  }
}

// Replay source: a pool of P gradient vectors; (t, rank) reads slot
// (t * n + rank) % P. With P == n and the slots rewritten before every step
// this is exactly FixedSource's per-(t, rank) script.
class ReplaySource final : public GradientSource {
 public:
  ReplaySource(Index n_g, int n, int pool)
      : n_g_(n_g), n_(n), pool_(static_cast<size_t>(pool),
                                 std::vector<double>(static_cast<size_t>(n_g))) {}
  Index size() const override { return n_g_; }
  void gradient(long long t, int rank, std::span<const double>,
                std::span<double> out) const override {
    const auto slot = static_cast<size_t>((t * n_ + rank) % static_cast<long long>(pool_.size()));
    std::copy(pool_[slot].begin(), pool_[slot].end(), out.begin());
  }
  std::vector<double>& slot(int s) { return pool_[static_cast<size_t>(s)]; }
  int pool() const { return static_cast<int>(pool_.size()); }

 private:
  Index n_g_;
  int n_;
  std::vector<std::vector<double>> pool_;
};

struct RefEngine {
  std::shared_ptr<ReplaySource> src;
  std::unique_ptr<Engine> engine;
  std::vector<std::vector<Index>> last_sel;  // per-rank selection, last step
  std::vector<Index> last_union;
  EngineOptions opt;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_validate(const exd_config* in, exd_config* out) {
  try {
    const SparsifierConfig v = validate(to_cfg(in));
    *out = *in;
    out->k = v.k;
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(EXD_EINVAL, e.what());
  }
}

int ref_build_topology(int64_t n_g, int64_t n_b, int32_t n, int64_t min_blk,
                       exd_topology* out, char* warning, size_t wlen) {
  try {
    std::string w;
    from_topo(build_topology(n_g, n_b, n, min_blk, &w), out);
    if (warning && wlen) {
      std::strncpy(warning, w.c_str(), wlen - 1);
      warning[wlen - 1] = 0;
    }
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(EXD_EINVAL, e.what());
  }
}

int ref_partition_range(const exd_topology* t, int32_t p, int64_t n_g,
                        int64_t* st, int64_t* end) {
  const IndexRange r = partition_range(to_topo(t), p, n_g);
  *st = r.st;
  *end = r.end;
  return 0;
}

int ref_rotate(const int64_t* k_rank, int64_t t, int32_t n, int64_t* k_part) {
  try {
    PartialK in{std::vector<Count>(k_rank, k_rank + n), KOrdering::RankOrder};
    const PartialK out = rotate_to_partition_order(in, t, n);
    std::copy(out.counts.begin(), out.counts.end(), k_part);
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(EXD_EINVAL, e.what());
  }
}

int ref_adjust(exd_topology* topo, int64_t* k_part, double alpha,
               int64_t blk_move, int64_t min_blk, int64_t n_g, int32_t* moves,
               int32_t* skips) {
  PartitionTopology t = to_topo(topo);
  PartialK k{std::vector<Count>(k_part, k_part + topo->n), KOrdering::PartitionOrder};
  const AdjustStats s = adjust_topology(t, k, alpha, blk_move, min_blk, n_g);
  from_topo(t, topo);
  std::copy(k.counts.begin(), k.counts.end(), k_part);
  *moves = s.moves;
  *skips = s.skips;
  return 0;
}

int ref_allocate(const exd_topology* topo, int64_t t, int32_t rank, int64_t n_g,
                 int32_t* partition, int64_t* st, int64_t* end) {
  const Allocation a = allocate_partition(to_topo(topo), t, rank, n_g);
  *partition = a.partition;
  *st = a.range.st;
  *end = a.range.end;
  return 0;
}

double ref_scale_threshold(int64_t k, int64_t kp, double delta, double beta,
                           double gamma) {
  return scale_threshold(k, kp, delta, beta, gamma);
}

int ref_initial_threshold(const double* mags, int64_t m, double d, double* out) {
  try {
    *out = initial_threshold(std::vector<double>(mags, mags + m), d);
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(EXD_EINVAL, e.what());
  }
}

// topk_select (baselines.cpp:26-41): out gets k indices; returns 0 or EXD_EINVAL.
int ref_topk_select(const double* acc, int64_t n, int64_t k, int64_t* out) {
  try {
    const auto idx = topk_select(std::span<const double>(acc, (size_t)n), k);
    std::copy(idx.begin(), idx.end(), out);
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(EXD_EINVAL, e.what());
  }
}

// hard_threshold_select (baselines.cpp:43-46): out needs n slots; *count set.
int ref_hard_threshold_select(const double* acc, int64_t n, double delta, int64_t* out,
                              int64_t* count) {
  const auto idx = hard_threshold_select(std::span<const double>(acc, (size_t)n), delta);
  std::copy(idx.begin(), idx.end(), out);
  *count = (int64_t)idx.size();
  return 0;
}

// all_gather over n index lists given as (concatenated, counts).
int ref_all_gather(const int64_t* concat, const int64_t* counts, int32_t n,
                   exd_gather_stats* st, int64_t* dups, int64_t* idx_global,
                   int64_t* union_len) {
  try {
    std::vector<SparseBatch> b(static_cast<size_t>(n));
    int64_t off = 0;
    for (int i = 0; i < n; ++i) {
      b[i].indices.assign(concat + off, concat + off + counts[i]);
      b[i].values.assign(static_cast<size_t>(counts[i]), 1.0);
      off += counts[i];
    }
    const GatherResult g = all_gather(b);
    st->k_prime = g.k_prime();
    st->m_t = g.m_t;
    st->c_t = g.c_t;
    st->f_t = g.f_t;
    *dups = g.duplicates;
    *union_len = static_cast<int64_t>(g.idx_global.size());
    if (idx_global) std::copy(g.idx_global.begin(), g.idx_global.end(), idx_global);
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(EXD_EINVAL, e.what());
  }
}

int ref_synthetic_gradient(const exd_stream_spec* s, int64_t t, int32_t rank,
                           double* out) {
  try {
    StreamSpec spec;
    spec.n_g = s->n_g;
    for (int i = 0; i < s->nseg; ++i) {
      spec.segments.push_back({s->seg_length[i], s->seg_scale[i]});
    }
    spec.distribution = s->distribution == 0 ? StreamDistribution::Laplace
                                             : StreamDistribution::LogNormal;
    spec.decay = s->decay;
    if (s->has_decay_step) spec.decay_step = s->decay_step;
    spec.decay_step_factor = s->decay_step_factor;
    spec.seed = s->seed;
    validate(spec);
    synthetic_gradient(spec, t, rank, std::span<double>(out, static_cast<size_t>(s->n_g)));
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(EXD_EINVAL, e.what());
  }
}

// ---- Engine ---------------------------------------------------------------

void* ref_engine_create(const exd_config* c, const exd_options* o, int32_t pool) {
  try {
    auto* h = new RefEngine;
    h->src = std::make_shared<ReplaySource>(c->n_g, c->n, pool);
    EngineOptions opt;
    opt.sparsifier = static_cast<SparsifierKind>(o->sparsifier);
    opt.static_partitions = o->static_partitions != 0;
    opt.fixed_delta = o->fixed_delta;
    opt.parallel_workers = o->parallel_workers != 0;
    opt.verify_replication = o->verify_replication != 0;
    opt.verify_conservation = o->verify_conservation != 0;
    opt.record_loss = o->record_loss != 0;
    h->opt = opt;
    h->engine = std::make_unique<Engine>(to_cfg(c), opt, h->src);
    return h;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_engine_destroy(void* p) { delete static_cast<RefEngine*>(p); }

int ref_engine_pool(void* p) { return static_cast<RefEngine*>(p)->src->pool(); }

int ref_engine_set_slot_f64(void* p, int32_t slot, const double* g) {
  auto* h = static_cast<RefEngine*>(p);
  auto& v = h->src->slot(slot);
  std::copy(g, g + v.size(), v.begin());
  return 0;
}

int ref_engine_set_slot_f32(void* p, int32_t slot, const float* g) {
  auto* h = static_cast<RefEngine*>(p);
  auto& v = h->src->slot(slot);
  for (size_t j = 0; j < v.size(); ++j) v[j] = static_cast<double>(g[j]);
  return 0;
}

// Engine::step(). With capture != 0 the per-rank selections of this step are
// reconstructed afterwards from the reference's own functions (accumulate,
// allocate_partition, select_indices) on a snapshot of the entering residuals.
int ref_engine_step(void* p, exd_record* out, int32_t capture) {
  auto* h = static_cast<RefEngine*>(p);
  Engine& eng = *h->engine;
  const auto& cfg = eng.config();
  try {
    std::vector<std::vector<double>> e_before;
    if (capture) {
      for (const auto& w : eng.workers()) e_before.push_back(w.e);
    }
    const long long t = eng.iteration();
    const IterationRecord rec = eng.step();
    fill_record(rec, out);
    if (capture) {
      h->last_sel.assign(static_cast<size_t>(cfg.n), {});
      h->last_union.clear();
      std::vector<double> grad(static_cast<size_t>(cfg.n_g));
      for (int r = 0; r < cfg.n; ++r) {
        h->src->gradient(t, r, {}, grad);
        const auto acc = accumulate(e_before[static_cast<size_t>(r)], cfg.eta, grad);
        auto& sel = h->last_sel[static_cast<size_t>(r)];
        switch (h->opt.sparsifier) {  // engine.cpp:188-197
          case SparsifierKind::ExDyna: {
            const auto a = allocate_partition(eng.workers()[static_cast<size_t>(r)].topology,
                                              t, r, cfg.n_g);
            sel = select_indices(acc, a.range.st, a.range.end, rec.delta);
            break;
          }
          case SparsifierKind::TopK:
            sel = topk_select(acc, cfg.k);
            break;
          case SparsifierKind::CLTk:
            if (r == cltk_leader(t, cfg.n)) sel = topk_select(acc, cfg.k);
            break;
          case SparsifierKind::HardThreshold:
            sel = hard_threshold_select(acc, h->opt.fixed_delta);
            break;
        }
        h->last_union.insert(h->last_union.end(), h->last_sel[static_cast<size_t>(r)].begin(),
                             h->last_sel[static_cast<size_t>(r)].end());
      }
      std::sort(h->last_union.begin(), h->last_union.end());
      h->last_union.erase(std::unique(h->last_union.begin(), h->last_union.end()),
                          h->last_union.end());
    }
    return 0;
  } catch (const EngineError& e) {
    return fail(EXD_EINVARIANT, e.what());
  } catch (const std::invalid_argument& e) {
    return fail(EXD_EINVAL, e.what());
  } catch (const std::exception& e) {
    return fail(EXD_EINVARIANT, e.what());
  }
}

int64_t ref_engine_iteration(void* p) { return static_cast<RefEngine*>(p)->engine->iteration(); }

int ref_engine_get_vec(void* p, int32_t w, int32_t which, double* out) {
  const auto& ws = static_cast<RefEngine*>(p)->engine->workers()[static_cast<size_t>(w)];
  const auto& v = which == EXD_VEC_X ? ws.x : ws.e;
  std::copy(v.begin(), v.end(), out);
  return 0;
}

int ref_engine_poke_x(void* p, int32_t w, int64_t j, double v) {
  auto& ws = static_cast<RefEngine*>(p)->engine->mutable_workers()[static_cast<size_t>(w)];
  ws.x[static_cast<size_t>(j)] = v;
  return 0;
}

int ref_engine_get_state(void* p, int32_t w, exd_worker_state* out) {
  auto* h = static_cast<RefEngine*>(p);
  const auto& ws = h->engine->workers()[static_cast<size_t>(w)];
  std::memset(out, 0, sizeof(*out));
  out->t = h->engine->iteration();
  out->rank = ws.rank;
  out->delta = ws.delta;
  for (size_t i = 0; i < ws.k_t.counts.size(); ++i) out->k_t[i] = ws.k_t.counts[i];
  from_topo(ws.topology, &out->topology);
  return 0;
}

// selections captured by the last ref_engine_step(capture=1)
int64_t ref_engine_last_selection(void* p, int32_t r, int64_t* out) {
  auto* h = static_cast<RefEngine*>(p);
  const auto& s = h->last_sel[static_cast<size_t>(r)];
  if (out) std::copy(s.begin(), s.end(), out);
  return static_cast<int64_t>(s.size());
}

int64_t ref_engine_last_union(void* p, int64_t* out) {
  auto* h = static_cast<RefEngine*>(p);
  if (out) std::copy(h->last_union.begin(), h->last_union.end(), out);
  return static_cast<int64_t>(h->last_union.size());
}

// format_csv / summarize over records given in the C ABI layout
static IterationRecord to_rec(const exd_record& o) {
  IterationRecord r;
  r.t = o.t;
  r.k_prime = o.k_prime;
  r.density = o.density;
  r.eps = o.eps;
  r.m_t = o.m_t;
  r.c_t = o.c_t;
  r.f_t = o.f_t;
  r.global_err = o.global_err;
  r.delta = o.delta;
  if (o.has_loss) r.loss = o.loss;
  r.duplicates = o.duplicates;
  r.union_count = o.union_count;
  r.k_rank.assign(o.k_rank, o.k_rank + o.n);
  r.adjust_moves = o.adjust_moves;
  r.adjust_skips = o.adjust_skips;
  r.cap_hits = o.cap_hits;
  r.idle_workers = o.idle_workers;
  return r;
}

int64_t ref_format_csv(const exd_record* recs, int64_t count, char* out, int64_t cap) {
  std::vector<IterationRecord> v;
  for (int64_t i = 0; i < count; ++i) v.push_back(to_rec(recs[i]));
  const std::string s = format_csv(v);
  if (out && cap > 0) {
    const int64_t n = std::min<int64_t>(cap - 1, (int64_t)s.size());
    std::memcpy(out, s.data(), (size_t)n);
    out[n] = 0;
  }
  return (int64_t)s.size();
}

int ref_summarize(const exd_record* recs, int64_t count, double* out6, int64_t* out5) {
  std::vector<IterationRecord> v;
  for (int64_t i = 0; i < count; ++i) v.push_back(to_rec(recs[i]));
  const RunStats s = summarize(v);
  out6[0] = s.mean_density;
  out6[1] = s.mean_f;
  out6[2] = s.mean_eps;
  out6[3] = s.mean_idle_workers;
  out6[4] = s.final_delta;
  out6[5] = s.final_global_err;
  out5[0] = s.iterations;
  out5[1] = s.duplicates;
  out5[2] = s.adjust_moves;
  out5[3] = s.adjust_skips;
  out5[4] = s.cap_hits;
  return 0;
}

}  // extern "C"
