// exdyna/engine.hpp — header-only C++ facade over the C ABI (include/exdyna.h)
// with the shape of the reference's sparsifier API (proj/include/sparsim), so
// that sparsim::Engine callers switch by changing a namespace:
//
//   sparsim::SparsifierConfig  -> exdyna::SparsifierConfig   (config.hpp:28-45)
//   sparsim::validate          -> exdyna::validate           (config.cpp:28-51)
//   sparsim::build_topology    -> exdyna::build_topology     (partition.cpp:22-58)
//   sparsim::Engine            -> exdyna::Engine             (engine.hpp:61-105)
//   sparsim::IterationRecord   -> exdyna::IterationRecord    (types.hpp:84-103)
//   sparsim::EngineError       -> exdyna::EngineError        (engine.hpp:47-50)
//   sparsim::topk_select /
//   sparsim::hard_threshold_select -> exdyna::topk_select /
//                                 exdyna::hard_threshold_select (baselines.hpp:25-34)
//
//   sparsim::GradientSource    -> exdyna::GradientSource     (workloads.hpp:77-87, C++20)
//
// Two ways to feed gradients:
//   * the reference's: Engine(cfg, opt, std::shared_ptr<const GradientSource>)
//     with step() / run(T) (engine.hpp:61-64). The source fills host memory;
//     the facade uploads it through pinned, double-buffered staging on the
//     engine's stream (one cudaMemcpyAsync per worker), and in run(T) the
//     source's work for step t+1 overlaps the device's step t whenever the
//     source neither reads x nor reports a loss;
//   * device buffers: step(grads) with one device pointer per local worker.
// The engine works in fp32 (Precision::F32; the source's doubles are rounded
// once to float) or in the reference's fp64 (Precision::F64).
#pragma once

#include <cuda_runtime.h>

#include <cstring>
#include <exception>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>
#if __cplusplus >= 202002L
#include <span>
#endif

#include "exdyna.h"

namespace exdyna {

class EngineError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

class DeviceError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

inline void check(int rc) {
  if (rc == EXD_OK) return;
  const std::string msg = exd_last_error();
  if (rc == EXD_EINVAL) throw std::invalid_argument(msg);
  if (rc == EXD_EINVARIANT) throw EngineError(msg);
  throw DeviceError(msg);
}

struct SparsifierConfig {
  int n = 4;
  int64_t n_g = 1'000'000;
  int64_t n_b = 256;
  double d = 0.001;
  int64_t k = 0;
  std::optional<double> delta0;
  double alpha = 1.25;
  double beta = 1.25;
  double gamma = 0.02;
  int64_t blk_move = 1;
  int64_t min_blk = 2;
  double eta = 1.0;
  uint64_t seed = 42;
  std::optional<double> max_density_cap;

  exd_config to_c() const {
    exd_config c{};
    c.n = n;
    c.n_g = n_g;
    c.n_b = n_b;
    c.d = d;
    c.k = k;
    c.has_delta0 = delta0.has_value();
    c.delta0 = delta0.value_or(0.0);
    c.alpha = alpha;
    c.beta = beta;
    c.gamma = gamma;
    c.blk_move = blk_move;
    c.min_blk = min_blk;
    c.eta = eta;
    c.seed = seed;
    c.has_max_density_cap = max_density_cap.has_value();
    c.max_density_cap = max_density_cap.value_or(0.0);
    return c;
  }
};

inline SparsifierConfig validate(SparsifierConfig cfg) {
  exd_config in = cfg.to_c(), out{};
  check(exd_validate(&in, &out));
  cfg.k = out.k;
  return cfg;
}

using Index = int64_t;
using Count = int64_t;

struct PartitionTopology {
  int64_t sz_blk = 0;
  std::vector<int64_t> blk_part, blk_pos;

  static PartitionTopology from_c(const exd_topology& t) {
    return {t.sz_blk, {t.blk_part, t.blk_part + t.n}, {t.blk_pos, t.blk_pos + t.n}};
  }
  exd_topology to_c() const {
    exd_topology t{};
    t.n = static_cast<int32_t>(blk_part.size());
    t.sz_blk = sz_blk;
    for (size_t i = 0; i < blk_part.size() && i < EXD_MAX_WORKERS; ++i) {
      t.blk_part[i] = blk_part[i];
      t.blk_pos[i] = blk_pos[i];
    }
    return t;
  }
};

// partition.hpp:25-30 / allocator.hpp:37-57
struct IndexRange {
  Index st = 0, end = 0;
  Index length() const { return end - st; }
  friend bool operator==(const IndexRange& a, const IndexRange& b) {
    return a.st == b.st && a.end == b.end;
  }
};
struct Allocation {
  int partition = 0;
  IndexRange range;
};

// allocate_partition, allocator.cpp:92-99
inline Allocation allocate_partition(const PartitionTopology& topo, long long t, int rank,
                                     Index n_g) {
  const exd_topology c = topo.to_c();
  Allocation a;
  int32_t p = 0;
  check(exd_allocate_partition(&c, t, rank, n_g, &p, &a.range.st, &a.range.end));
  a.partition = p;
  return a;
}

inline PartitionTopology build_topology(int64_t n_g, int64_t n_b, int n, int64_t min_blk,
                                        std::string* warning = nullptr) {
  exd_topology t{};
  char w[256] = {0};
  check(exd_build_topology(n_g, n_b, n, min_blk, &t, w, sizeof w));
  if (warning) *warning = w;
  return PartitionTopology::from_c(t);
}

enum class Precision { F32 = EXD_F32, F64 = EXD_F64 };

// engine.hpp:30-32
enum class SparsifierKind {
  ExDyna = EXD_SPARSIFIER_EXDYNA,
  TopK = EXD_SPARSIFIER_TOPK,
  CLTk = EXD_SPARSIFIER_CLTK,
  HardThreshold = EXD_SPARSIFIER_HARD_THRESHOLD,
};

// types.hpp:48-59: k_t in rank order
enum class KOrdering { RankOrder, PartitionOrder };
struct PartialK {
  std::vector<Count> counts;
  KOrdering ordering = KOrdering::RankOrder;
};

// types.hpp:73-80: one worker's replicated state, as a host snapshot
struct WorkerState {
  int rank = 0;
  std::vector<double> x, e;
  double delta = 0.0;
  PartialK k_t;
  PartitionTopology topology;
};

// baselines.hpp:25-34 over a DEVICE vector acc (n_g elements of `precision`);
// the indices come back to the host in ascending order, like the reference's
// std::vector<Index>. `idx_dev` is caller scratch of at least k (top-k) or
// n_g (hard threshold) int32; `stream` is a cudaStream_t (nullptr: default).
inline std::vector<int64_t> topk_select(const void* acc_dev, int64_t n_g, Precision precision,
                                        int64_t k, int32_t* idx_dev, void* stream = nullptr);
inline std::vector<int64_t> hard_threshold_select(const void* acc_dev, int64_t n_g,
                                                  Precision precision, double fixed_delta,
                                                  int32_t* idx_dev, void* stream = nullptr);

// engine.hpp:37-45, plus the B200 knobs (precision, profiling, sync mode)
struct EngineOptions {
  SparsifierKind sparsifier = SparsifierKind::ExDyna;
  bool static_partitions = false;
  double fixed_delta = 0.0;
  bool parallel_workers = true;     // GradientSource calls of local workers on threads
  bool verify_replication = true;
  bool verify_conservation = false;
  bool record_loss = true;          // GradientSource::loss at x_{t+1} (engine.cpp:340)
  Precision precision = Precision::F32;
  bool profile_kernels = false;
  int sync_mode = EXD_SYNC_AUTO;

  exd_options to_c() const {
    exd_options o{};
    o.sparsifier = static_cast<int32_t>(sparsifier);
    o.static_partitions = static_partitions;
    o.fixed_delta = fixed_delta;
    o.parallel_workers = parallel_workers;
    o.verify_replication = verify_replication;
    o.verify_conservation = verify_conservation;
    o.record_loss = record_loss;
    o.dtype = static_cast<int32_t>(precision);
    o.profile_kernels = profile_kernels;
    o.sync_mode = sync_mode;
    return o;
  }
};

struct IterationRecord {
  long long t = 0;
  int64_t k_prime = 0;
  double density = 0.0, eps = 0.0;
  int64_t m_t = 0, c_t = 0;
  double f_t = 1.0, global_err = 0.0, delta = 0.0;
  std::optional<double> loss;
  int64_t duplicates = 0, union_count = 0;
  std::vector<int64_t> k_rank;
  int adjust_moves = 0, adjust_skips = 0, cap_hits = 0, idle_workers = 0;

  static IterationRecord from_c(const exd_record& r) {
    IterationRecord o;
    o.t = r.t;
    o.k_prime = r.k_prime;
    o.density = r.density;
    o.eps = r.eps;
    o.m_t = r.m_t;
    o.c_t = r.c_t;
    o.f_t = r.f_t;
    o.global_err = r.global_err;
    o.delta = r.delta;
    if (r.has_loss) o.loss = r.loss;
    o.duplicates = r.duplicates;
    o.union_count = r.union_count;
    o.k_rank.assign(r.k_rank, r.k_rank + r.n);
    o.adjust_moves = r.adjust_moves;
    o.adjust_skips = r.adjust_skips;
    o.cap_hits = r.cap_hits;
    o.idle_workers = r.idle_workers;
    return o;
  }
};

#if __cplusplus >= 202002L
// workloads.hpp:77-87. gradient() may be called concurrently for different
// ranks (parallel_workers), exactly as the reference does.
class GradientSource {
 public:
  virtual ~GradientSource() = default;
  virtual Index size() const = 0;
  // Stochastic gradient of worker `rank` at iteration t, evaluated at x.
  virtual void gradient(long long t, int rank, std::span<const double> x,
                        std::span<double> out) const = 0;
  virtual std::optional<double> loss(std::span<const double> /*x*/) const {
    return std::nullopt;
  }
  // Optional hints for the device engine (not in the reference interface; the
  // defaults are always correct). reads_x() == false: gradient() ignores x, so
  // the model is not copied back to the host each step; has_loss() == false:
  // loss() is always nullopt. With both false, run(T) overlaps the source's
  // work for step t+1 with the device's step t.
  virtual bool reads_x() const { return true; }
  virtual bool has_loss() const { return true; }
};
#endif

// sparsim::Engine on the B200. All cfg.n workers live in this process on
// `device` (the reference's simulator shape); Engine::rank() builds one rank of
// an n-process job instead (NCCL over NVLink).
class Engine {
 public:
  Engine(SparsifierConfig cfg, EngineOptions opt = {}, int device = 0) : opt_(opt) {
    cfg_ = validate(cfg);
    exd_config c = cfg_.to_c();
    exd_options o = opt.to_c();
    int32_t dev = device;
    check(exd_engine_create(&c, &o, &dev, 1, &h_));
  }
  static Engine rank(SparsifierConfig cfg, EngineOptions opt, int rank, int device,
                     const uint8_t* nccl_id) {
    return Engine(cfg, opt, rank, device, nccl_id);
  }
#if __cplusplus >= 202002L
  // The reference's constructor (engine.hpp:61-62, engine.cpp:51-62).
  Engine(SparsifierConfig cfg, EngineOptions opt, std::shared_ptr<const GradientSource> source,
         int device = 0)
      : opt_(opt) {
    cfg_ = validate(cfg);  // config errors first, as the reference's member init
    if (!source) throw std::invalid_argument("engine: null gradient source");
    if (source->size() != cfg_.n_g) throw std::invalid_argument("engine: workload size != n_g");
    exd_config c = cfg_.to_c();
    exd_options o = opt.to_c();
    int32_t dev = device;
    check(exd_engine_create(&c, &o, &dev, 1, &h_));
    attach(std::move(source), device);
  }
  // One rank of an n-process job fed by a source (it asks for its own rank).
  static Engine rank(SparsifierConfig cfg, EngineOptions opt, int rank, int device,
                     const uint8_t* nccl_id, std::shared_ptr<const GradientSource> source) {
    if (!source) throw std::invalid_argument("engine: null gradient source");
    Engine e(cfg, opt, rank, device, nccl_id);
    if (source->size() != e.cfg_.n_g) throw std::invalid_argument("engine: workload size != n_g");
    e.attach(std::move(source), device);
    return e;
  }
#endif
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;
  Engine(Engine&& o) noexcept
      : cfg_(o.cfg_), opt_(o.opt_), h_(o.h_), stage_(std::move(o.stage_)) {
#if __cplusplus >= 202002L
    src_ = std::move(o.src_);
#endif
    o.h_ = nullptr;
  }
  ~Engine() {
    if (h_) exd_engine_destroy(h_);
  }

#if __cplusplus >= 202002L
  // Engine::step() / run(T) (engine.hpp:63-64): gradients from the source.
  IterationRecord step() { return run(1).back(); }
  std::vector<IterationRecord> run(long long iterations) {
    if (!src_) throw std::invalid_argument("engine: no gradient source attached");
    const bool need_x = src_->reads_x();
    const bool want_loss = opt_.record_loss && src_->has_loss();
    const bool pipelined = !need_x && !want_loss;
    const long long first = iteration();
    std::vector<IterationRecord> out;
    out.reserve(static_cast<size_t>(iterations > 0 ? iterations : 0));
    long long fetched = 0;
    for (long long i = 0; i < iterations; ++i) {
      const long long t = iteration();
      const int slot = static_cast<int>(t & 1);
      Staging& st = *stage_;
      // the host slot is free once the upload of step t-2 finished
      if (cudaEventSynchronize(st.copied[slot]) != cudaSuccess)
        throw DeviceError("gradient staging: event wait failed");
      if (need_x) load_x(st);
      fill(st, t, slot);
      for (int w = 0; w < st.nl; ++w)
        if (cudaMemcpyAsync(st.dev[slot][w], st.host[slot][w], st.bytes, cudaMemcpyHostToDevice,
                            st.stream) != cudaSuccess)
          throw DeviceError("gradient staging: host-to-device copy failed");
      cudaEventRecord(st.copied[slot], st.stream);
      std::vector<const void*> ptrs(st.dev[slot].begin(), st.dev[slot].end());
      if (!pipelined) {
        exd_record r{};
        check(exd_engine_step(h_, ptrs.data(), &r));
        IterationRecord rec = IterationRecord::from_c(r);
        if (want_loss) {
          load_x(st);  // x_{t+1} of local worker 0
          rec.loss = src_->loss(std::span<const double>(st.xd[0]));
        }
        out.push_back(std::move(rec));
        continue;
      }
      check(exd_engine_step_async(h_, ptrs.data()));
      if ((i + 1) % 128 == 0 || i + 1 == iterations) {
        const long long cnt = (i + 1) - fetched;
        std::vector<exd_record> rs(static_cast<size_t>(cnt));
        check(exd_engine_records(h_, first + fetched, cnt, rs.data()));
        for (const auto& r : rs) out.push_back(IterationRecord::from_c(r));
        fetched = i + 1;
      }
    }
    return out;
  }
#endif

  // workers() (engine.hpp:72): a host snapshot of every local worker, refreshed
  // on each call (x and e are copied back from the device).
  const std::vector<WorkerState>& workers() {
    const int nl = local_workers();
    workers_.resize(static_cast<size_t>(nl));
    for (int w = 0; w < nl; ++w) {
      const exd_worker_state s = state(w);
      WorkerState& o = workers_[static_cast<size_t>(w)];
      o.rank = s.rank;
      o.delta = s.delta;
      o.k_t.counts.assign(s.k_t, s.k_t + cfg_.n);
      o.k_t.ordering = KOrdering::RankOrder;
      o.topology = PartitionTopology::from_c(s.topology);
      o.x = as_double(w, EXD_VEC_X);
      o.e = as_double(w, EXD_VEC_E);
    }
    return workers_;
  }

  // Engine::step(): grads[w] is local worker w's device gradient (n_g elements).
  IterationRecord step(const std::vector<const void*>& grads) {
    exd_record r{};
    check(exd_engine_step(h_, grads.data(), &r));
    return IterationRecord::from_c(r);
  }
  // Host-buffer step (what a GradientSource fills, workloads.hpp:77-87).
  IterationRecord step_host(const std::vector<const void*>& host_grads) {
    exd_record r{};
    check(exd_engine_step_host(h_, host_grads.data(), &r));
    return IterationRecord::from_c(r);
  }
  std::vector<IterationRecord> run(long long iterations,
                                   const std::vector<const void*>& grads) {
    std::vector<IterationRecord> out;
    for (long long i = 0; i < iterations; ++i) out.push_back(step(grads));
    return out;
  }

  long long iteration() const { return exd_engine_iteration(h_); }
  const SparsifierConfig& config() const { return cfg_; }
  int local_workers() const { return exd_engine_local_workers(h_); }

  exd_worker_state state(int w = 0) {
    exd_worker_state s{};
    check(exd_engine_get_state(h_, w, &s));
    return s;
  }
  template <typename T>
  std::vector<T> vector(int w, int which) {
    int64_t len = 0;
    check(exd_engine_copy_out(h_, w, which, nullptr, 0, &len));
    std::vector<T> out(static_cast<size_t>(len));
    if (len) check(exd_engine_copy_out(h_, w, which, out.data(), len, &len));
    return out;
  }
  exd_engine* handle() { return h_; }

 private:
  Engine(SparsifierConfig cfg, EngineOptions opt, int rank, int device, const uint8_t* id)
      : opt_(opt) {
    cfg_ = validate(cfg);
    exd_config c = cfg_.to_c();
    exd_options o = opt.to_c();
    check(exd_engine_create_rank(&c, &o, rank, device, id, &h_));
  }

  std::vector<double> as_double(int w, int which) {
    if (opt_.precision == Precision::F64) return vector<double>(w, which);
    const std::vector<float> f = vector<float>(w, which);
    return std::vector<double>(f.begin(), f.end());
  }

  // pinned host + device gradient buffers, two slots (step parity) per worker
  struct Staging {
    int nl = 0;
    size_t bytes = 0;
    bool f32 = true;
    cudaStream_t stream = nullptr;
    std::vector<void*> host[2], dev[2];
    cudaEvent_t copied[2] = {nullptr, nullptr};
    std::vector<std::vector<double>> scratch;  // fp32 mode: the source's doubles
    std::vector<std::vector<double>> xd;       // x as doubles (reads_x / loss)
    ~Staging() {
      for (int s = 0; s < 2; ++s) {
        for (void* p : host[s]) cudaFreeHost(p);
        for (void* p : dev[s]) cudaFree(p);
        if (copied[s]) cudaEventDestroy(copied[s]);
      }
    }
  };

#if __cplusplus >= 202002L
  void attach(std::shared_ptr<const GradientSource> source, int device) {
    src_ = std::move(source);
    auto st = std::make_unique<Staging>();
    st->nl = local_workers();
    st->f32 = opt_.precision == Precision::F32;
    st->bytes = static_cast<size_t>(cfg_.n_g) * (st->f32 ? sizeof(float) : sizeof(double));
    st->stream = static_cast<cudaStream_t>(exd_engine_stream(h_, 0));
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    for (int s = 0; s < 2; ++s) {
      st->host[s].assign(static_cast<size_t>(st->nl), nullptr);
      st->dev[s].assign(static_cast<size_t>(st->nl), nullptr);
      for (int w = 0; w < st->nl; ++w) {
        if (cudaHostAlloc(&st->host[s][w], st->bytes, cudaHostAllocDefault) != cudaSuccess ||
            cudaMalloc(&st->dev[s][w], st->bytes) != cudaSuccess)
          throw DeviceError("gradient staging: allocation failed");
      }
      cudaEventCreateWithFlags(&st->copied[s], cudaEventDisableTiming);
    }
    cudaSetDevice(prev);
    st->scratch.resize(st->f32 ? static_cast<size_t>(st->nl) : 0);
    for (auto& v : st->scratch) v.resize(static_cast<size_t>(cfg_.n_g));
    st->xd.resize(static_cast<size_t>(st->nl));
    stage_ = std::move(st);
  }

  void load_x(Staging& st) {
    for (int w = 0; w < st.nl; ++w) st.xd[w] = as_double(w, EXD_VEC_X);
  }

  // GradientSource::gradient for every local worker (engine.cpp:134), on
  // threads when parallel_workers (engine.cpp:90-117); worker exceptions are
  // rethrown in rank order.
  void fill(Staging& st, long long t, int slot) {
    const int first = exd_engine_first_rank(h_);
    const size_t n_g = static_cast<size_t>(cfg_.n_g);
    auto one = [&](int w) {
      std::span<const double> x;
      if (!st.xd[w].empty()) x = std::span<const double>(st.xd[w]);
      if (st.f32) {
        std::span<double> out(st.scratch[w]);
        src_->gradient(t, first + w, x, out);
        float* dst = static_cast<float*>(st.host[slot][w]);
        for (size_t j = 0; j < n_g; ++j) dst[j] = static_cast<float>(st.scratch[w][j]);
      } else {
        std::span<double> out(static_cast<double*>(st.host[slot][w]), n_g);
        src_->gradient(t, first + w, x, out);
      }
    };
    if (!opt_.parallel_workers || st.nl == 1) {
      for (int w = 0; w < st.nl; ++w) one(w);
      return;
    }
    std::vector<std::exception_ptr> err(static_cast<size_t>(st.nl));
    std::vector<std::thread> th;
    for (int w = 1; w < st.nl; ++w)
      th.emplace_back([&, w] {
        try {
          one(w);
        } catch (...) {
          err[w] = std::current_exception();
        }
      });
    try {
      one(0);
    } catch (...) {
      err[0] = std::current_exception();
    }
    for (auto& x : th) x.join();
    for (auto& e : err)
      if (e) std::rethrow_exception(e);
  }

  std::shared_ptr<const GradientSource> src_;
#endif

  SparsifierConfig cfg_;
  EngineOptions opt_;
  exd_engine* h_ = nullptr;
  std::unique_ptr<Staging> stage_;
  std::vector<WorkerState> workers_;
};

namespace detail {
inline std::vector<int64_t> copy_indices(const int32_t* idx_dev, int64_t count) {
  std::vector<int32_t> h(static_cast<size_t>(count));
  if (count > 0 &&
      cudaMemcpy(h.data(), idx_dev, h.size() * sizeof(int32_t), cudaMemcpyDeviceToHost) !=
          cudaSuccess)
    throw DeviceError("copy of selected indices failed");
  return std::vector<int64_t>(h.begin(), h.end());
}
}  // namespace detail

inline std::vector<int64_t> topk_select(const void* acc_dev, int64_t n_g, Precision precision,
                                        int64_t k, int32_t* idx_dev, void* stream) {
  check(exd_topk_select_device(acc_dev, n_g, static_cast<int32_t>(precision), k, idx_dev,
                               k, stream));
  return detail::copy_indices(idx_dev, k);
}

inline std::vector<int64_t> hard_threshold_select(const void* acc_dev, int64_t n_g,
                                                  Precision precision, double fixed_delta,
                                                  int32_t* idx_dev, void* stream) {
  int64_t count = 0;
  check(exd_hard_threshold_select_device(acc_dev, n_g, static_cast<int32_t>(precision),
                                         fixed_delta, idx_dev, n_g, &count, stream));
  return detail::copy_indices(idx_dev, count);
}

}  // namespace exdyna
