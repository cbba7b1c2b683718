// The reference's GradientSource-driven Engine (engine.hpp:61-64,
// workloads.hpp:77-87) through the exdyna facade, with only the namespace
// changed on the caller's side:
//   1. the scripted one-iteration trace of test_engine.cpp:79-131 (a
//      FixedSource replaying per-(t, rank) vectors), fp64;
//   2. an x-independent source without a loss (the pipelined run(T) path)
//      against the same source driven one step() at a time with the default
//      hints (the synchronous path): identical records;
//   3. an x-dependent quadratic source with a loss (x copied back every step,
//      loss at x_{t+1} in every record).
// Built and run by tests/test_cpp_facade.py (GPU).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <memory>
#include <span>
#include <vector>

#include "exdyna/engine.hpp"

#define EXPECT(c)                                                          \
  do {                                                                     \
    if (!(c)) {                                                            \
      std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #c); \
      return 1;                                                            \
    }                                                                      \
  } while (0)

namespace {
using exdyna::Index;

// per-(t, rank) script; steps past the end replay the last iteration
class ScriptSource final : public exdyna::GradientSource {
 public:
  ScriptSource(Index n_g, std::vector<std::vector<std::vector<double>>> g)
      : n_g_(n_g), g_(std::move(g)) {}
  Index size() const override { return n_g_; }
  void gradient(long long t, int rank, std::span<const double>,
                std::span<double> out) const override {
    const auto& step = g_[std::min<size_t>(static_cast<size_t>(t), g_.size() - 1)];
    std::copy(step[rank].begin(), step[rank].end(), out.begin());
  }

 private:
  Index n_g_;
  std::vector<std::vector<std::vector<double>>> g_;
};

// deterministic heavy-tailed values from a hash of (t, rank, j)
class HashSource : public exdyna::GradientSource {
 public:
  explicit HashSource(Index n) : n_(n) {}
  Index size() const override { return n_; }
  void gradient(long long t, int rank, std::span<const double>,
                std::span<double> out) const override {
    for (Index j = 0; j < n_; ++j) {
      unsigned long long h = (unsigned long long)t * 0x9e3779b97f4a7c15ULL ^
                             ((unsigned long long)rank << 40) ^ (unsigned long long)j;
      h ^= h >> 31;
      h *= 0xbf58476d1ce4e5b9ULL;
      h ^= h >> 29;
      const double u = ((h >> 11) + 0.5) * (1.0 / 9007199254740992.0);
      out[j] = (u < 0.5 ? 1.0 : -1.0) * -std::log(u < 0.5 ? 2 * u : 2 * (1 - u));
    }
  }

 private:
  Index n_;
};
class HashSourceHinted final : public HashSource {
 public:
  using HashSource::HashSource;
  bool reads_x() const override { return false; }
  bool has_loss() const override { return false; }
};

// f(x) = 1/2 sum (x_j - c_j)^2: gradient x - c reads x; loss at x
class QuadSource final : public exdyna::GradientSource {
 public:
  explicit QuadSource(Index n) : c_(n) {
    for (Index j = 0; j < n; ++j) c_[j] = std::sin(0.37 * j) * (1 + (j % 7));
  }
  Index size() const override { return (Index)c_.size(); }
  void gradient(long long, int, std::span<const double> x, std::span<double> out) const override {
    for (size_t j = 0; j < c_.size(); ++j) out[j] = x[j] - c_[j];
  }
  std::optional<double> loss(std::span<const double> x) const override {
    double s = 0;
    for (size_t j = 0; j < c_.size(); ++j) s += 0.5 * (x[j] - c_[j]) * (x[j] - c_[j]);
    return s;
  }

 private:
  std::vector<double> c_;
};
}  // namespace

int main() {
  using namespace exdyna;
  {  // 1. test_engine.cpp:79-131
    SparsifierConfig cfg;
    cfg.n = 2;
    cfg.n_g = 8;
    cfg.n_b = 2;
    cfg.d = 0.5;
    cfg.min_blk = 1;
    cfg.delta0 = 0.5;
    cfg.eta = 1.0;
    cfg.beta = 2.0;
    cfg.gamma = 0.01;
    const std::vector<double> g0{0.6, 0.1, -0.7, 0.2, 0.05, -0.3, 0.9, -0.05};
    const std::vector<double> g1{-0.4, 0.55, 0.1, -0.6, 0.45, 0.2, -0.1, 0.8};
    auto src = std::make_shared<ScriptSource>(
        8, std::vector<std::vector<std::vector<double>>>{{g0, g1}});
    EngineOptions opt;
    opt.parallel_workers = false;
    opt.verify_conservation = true;
    opt.precision = Precision::F64;
    Engine engine(cfg, opt, src);
    const auto rec = engine.step();
    EXPECT(rec.t == 0 && rec.k_prime == 3 && rec.m_t == 2 && rec.c_t == 2);
    EXPECT(rec.density == 0.375 && rec.eps == 0.125);
    EXPECT(std::fabs(rec.f_t - 4.0 / 3.0) < 1e-15);
    EXPECT(rec.global_err == 0.0 && rec.delta == 0.5 && !rec.loss.has_value());
    EXPECT(rec.duplicates == 0 && rec.union_count == 3);
    EXPECT((rec.k_rank == std::vector<Count>{2, 1}));
    EXPECT(rec.adjust_moves == 0 && rec.adjust_skips == 0 && rec.idle_workers == 0);
    const auto& w0 = engine.workers()[0];
    EXPECT(w0.x[0] == -(0.6 + -0.4) / 2);
    EXPECT(w0.x[2] == -(-0.7 + 0.1) / 2);
    EXPECT(w0.x[7] == -(-0.05 + 0.8) / 2);
    for (int j : {1, 3, 4, 5, 6}) EXPECT(w0.x[static_cast<size_t>(j)] == 0.0);
    EXPECT((w0.e == std::vector<double>{0, 0.1, 0, 0.2, 0.05, -0.3, 0.9, 0}));
    EXPECT((engine.workers()[1].e == std::vector<double>{0, 0.55, 0, -0.6, 0.45, 0.2, -0.1, 0}));
    EXPECT(std::fabs(w0.delta - 0.5 * 1.0025) < 1e-15);
    EXPECT((w0.k_t.counts == std::vector<Count>{2, 1}));
    const auto a = allocate_partition(w0.topology, 1, 0, 8);
    EXPECT((a.range == IndexRange{4, 8}));
    // the source must match n_g (engine.cpp:55-57)
    bool threw = false;
    try {
      Engine bad(cfg, opt, std::make_shared<ScriptSource>(
                               9, std::vector<std::vector<std::vector<double>>>{{g0, g1}}));
    } catch (const std::invalid_argument& e) {
      threw = std::string(e.what()) == "engine: workload size != n_g";
    }
    EXPECT(threw);
    std::printf("PASS scripted trace\n");
  }
  {  // 2. pipelined run(T) == step-by-step
    SparsifierConfig cfg;
    cfg.n = 3;
    cfg.n_g = 300'001;
    cfg.n_b = 24;
    cfg.d = 0.01;
    cfg.seed = 5;
    EngineOptions opt;
    opt.verify_replication = false;
    Engine fast(cfg, opt, std::make_shared<HashSourceHinted>(cfg.n_g));
    Engine slow(cfg, opt, std::make_shared<HashSource>(cfg.n_g));
    const auto rs = fast.run(300);  // crosses the 128-step record batches
    EXPECT(rs.size() == 300);
    for (int t = 0; t < 300; ++t) {
      const auto r = slow.step();
      EXPECT(r.t == t && rs[t].t == t);
      EXPECT(r.k_prime == rs[t].k_prime && r.delta == rs[t].delta && r.k_rank == rs[t].k_rank);
      EXPECT(r.m_t == rs[t].m_t && r.global_err == rs[t].global_err);
      EXPECT(!r.loss.has_value());
    }
    EXPECT(fast.workers()[1].x == slow.workers()[1].x);
    EXPECT(fast.workers()[2].e == slow.workers()[2].e);
    std::printf("PASS pipelined run\n");
  }
  {  // 3. x-dependent source with a loss
    SparsifierConfig cfg;
    cfg.n = 2;
    cfg.n_g = 20'000;
    cfg.n_b = 16;
    cfg.d = 0.05;
    cfg.eta = 0.5;
    EngineOptions opt;
    opt.precision = Precision::F64;
    auto quad = std::make_shared<QuadSource>(cfg.n_g);
    Engine engine2(cfg, opt, quad);
    const auto rs = engine2.run(60);
    EXPECT(rs.size() == 60);
    for (const auto& r : rs) EXPECT(r.loss.has_value());
    // the last record's loss is the source's loss at the final model x_{60}
    const auto& x = engine2.workers()[0].x;
    EXPECT(*rs[59].loss == *quad->loss(std::span<const double>(x)));
    // and x moved: the gradient saw x (x - c differs from -c after step 0)
    EXPECT(*rs[1].loss != *rs[0].loss);
    std::printf("PASS x-dependent source, loss %.6g -> %.6g\n", *rs[0].loss, *rs[59].loss);
  }
  return 0;
}
