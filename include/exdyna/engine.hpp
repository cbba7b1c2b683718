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
// Differences a caller sees: gradients are DEVICE buffers (one per local
// worker) instead of a host GradientSource callback (step_host() takes the
// host buffers such a source fills); the engine works in fp32
// (Precision::F32) or in the reference's fp64 (Precision::F64).
#pragma once

#include <cuda_runtime.h>

#include <cstring>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

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

struct PartitionTopology {
  int64_t sz_blk = 0;
  std::vector<int64_t> blk_part, blk_pos;
};

inline PartitionTopology build_topology(int64_t n_g, int64_t n_b, int n, int64_t min_blk,
                                        std::string* warning = nullptr) {
  exd_topology t{};
  char w[256] = {0};
  check(exd_build_topology(n_g, n_b, n, min_blk, &t, w, sizeof w));
  if (warning) *warning = w;
  return {t.sz_blk, {t.blk_part, t.blk_part + t.n}, {t.blk_pos, t.blk_pos + t.n}};
}

enum class Precision { F32 = EXD_F32, F64 = EXD_F64 };

// baselines.hpp:25-34 over a DEVICE vector acc (n_g elements of `precision`);
// the indices come back to the host in ascending order, like the reference's
// std::vector<Index>. `idx_dev` is caller scratch of at least k (top-k) or
// n_g (hard threshold) int32; `stream` is a cudaStream_t (nullptr: default).
inline std::vector<int64_t> topk_select(const void* acc_dev, int64_t n_g, Precision precision,
                                        int64_t k, int32_t* idx_dev, void* stream = nullptr);
inline std::vector<int64_t> hard_threshold_select(const void* acc_dev, int64_t n_g,
                                                  Precision precision, double fixed_delta,
                                                  int32_t* idx_dev, void* stream = nullptr);

struct EngineOptions {
  bool static_partitions = false;
  bool verify_replication = true;
  bool verify_conservation = false;
  Precision precision = Precision::F32;
  bool profile_kernels = false;
  int sync_mode = EXD_SYNC_AUTO;

  exd_options to_c() const {
    exd_options o{};
    o.sparsifier = EXD_SPARSIFIER_EXDYNA;
    o.static_partitions = static_partitions;
    o.parallel_workers = 1;
    o.verify_replication = verify_replication;
    o.verify_conservation = verify_conservation;
    o.record_loss = 0;
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
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;
  Engine(Engine&& o) noexcept : cfg_(o.cfg_), opt_(o.opt_), h_(o.h_) { o.h_ = nullptr; }
  ~Engine() {
    if (h_) exd_engine_destroy(h_);
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

  SparsifierConfig cfg_;
  EngineOptions opt_;
  exd_engine* h_ = nullptr;
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
