// The hand-traced ledger row of the reference (proj/tests/test_engine.cpp:79-131)
// driven through the C++ facade exdyna::Engine, exactly as a sparsim::Engine
// caller would: same config, same scripted gradients, same expectations.
// Built and run by tests/test_cpp_facade.py (GPU).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <vector>

#include "exdyna/engine.hpp"

#define EXPECT(c)                                                   \
  do {                                                              \
    if (!(c)) {                                                     \
      std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #c); \
      return 1;                                                     \
    }                                                               \
  } while (0)

int main() {
  exdyna::SparsifierConfig cfg;  // test_engine.cpp:50-62 trace_config()
  cfg.n = 2;
  cfg.n_g = 8;
  cfg.n_b = 2;
  cfg.d = 0.5;
  cfg.min_blk = 1;
  cfg.delta0 = 0.5;
  cfg.eta = 1.0;
  cfg.beta = 2.0;
  cfg.gamma = 0.01;
  exdyna::EngineOptions opt;
  opt.precision = exdyna::Precision::F64;
  exdyna::Engine engine(cfg, opt);

  const std::vector<double> g0{0.6, 0.1, -0.7, 0.2, 0.05, -0.3, 0.9, -0.05};
  const std::vector<double> g1{-0.4, 0.55, 0.1, -0.6, 0.45, 0.2, -0.1, 0.8};
  double *d0, *d1;
  cudaMalloc(&d0, 8 * sizeof(double));
  cudaMalloc(&d1, 8 * sizeof(double));
  cudaMemcpy(d0, g0.data(), 8 * sizeof(double), cudaMemcpyHostToDevice);
  cudaMemcpy(d1, g1.data(), 8 * sizeof(double), cudaMemcpyHostToDevice);

  const auto rec = engine.step({d0, d1});
  EXPECT(rec.t == 0);
  EXPECT(rec.k_prime == 3);
  EXPECT(rec.density == 0.375);
  EXPECT(rec.eps == 0.125);
  EXPECT(rec.m_t == 2);
  EXPECT(rec.c_t == 2);
  EXPECT(std::fabs(rec.f_t - 4.0 / 3.0) < 1e-15);
  EXPECT(rec.global_err == 0.0);
  EXPECT(rec.delta == 0.5);
  EXPECT(!rec.loss.has_value());
  EXPECT(rec.duplicates == 0);
  EXPECT(rec.union_count == 3);
  EXPECT((rec.k_rank == std::vector<int64_t>{2, 1}));
  EXPECT(rec.adjust_moves == 0 && rec.adjust_skips == 0 && rec.idle_workers == 0);

  const auto x0 = engine.vector<double>(0, EXD_VEC_X);
  EXPECT(x0[0] == -(0.6 + -0.4) / 2);
  EXPECT(x0[2] == -(-0.7 + 0.1) / 2);
  EXPECT(x0[7] == -(-0.05 + 0.8) / 2);
  for (int j : {1, 3, 4, 5, 6}) EXPECT(x0[j] == 0.0);
  EXPECT((engine.vector<double>(0, EXD_VEC_E) ==
          std::vector<double>{0, 0.1, 0, 0.2, 0.05, -0.3, 0.9, 0}));
  EXPECT((engine.vector<double>(1, EXD_VEC_E) ==
          std::vector<double>{0, 0.55, 0, -0.6, 0.45, 0.2, -0.1, 0}));
  const auto st = engine.state(0);
  EXPECT(std::fabs(st.delta - 0.5 * 1.0025) < 1e-15);
  EXPECT(st.k_t[0] == 2 && st.k_t[1] == 1);

  // the invalid-config path throws std::invalid_argument with the reference text
  bool threw = false;
  try {
    exdyna::SparsifierConfig bad = cfg;
    bad.n_b = 128;
    exdyna::Engine e2(bad);
  } catch (const std::invalid_argument& e) {
    threw = std::string(e.what()) == "n_b > n_g";
  }
  EXPECT(threw);
  cudaFree(d0);
  cudaFree(d1);
  std::printf("engine_facade_golden: PASS\n");
  // baselines through the facade: test_baselines.cpp:27-37, 66-71 known answers
  {
    const std::vector<double> a{0.1, -0.5, 0.3}, b{0.5, 0.5, 0.1}, c{0.1, 0.4};
    double* dv;
    int32_t* di;
    cudaMalloc(&dv, 3 * sizeof(double));
    cudaMalloc(&di, 3 * sizeof(int32_t));
    const auto F64 = exdyna::Precision::F64;
    cudaMemcpy(dv, a.data(), 3 * sizeof(double), cudaMemcpyHostToDevice);
    EXPECT((exdyna::topk_select(dv, 3, F64, 2, di) == std::vector<int64_t>{1, 2}));
    EXPECT((exdyna::topk_select(dv, 3, F64, 3, di) == std::vector<int64_t>{0, 1, 2}));
    cudaMemcpy(dv, b.data(), 3 * sizeof(double), cudaMemcpyHostToDevice);
    EXPECT((exdyna::topk_select(dv, 3, F64, 1, di) == std::vector<int64_t>{0}));
    EXPECT((exdyna::topk_select(dv, 3, F64, 2, di) == std::vector<int64_t>{0, 1}));
    bool threw = false;
    try {
      exdyna::topk_select(dv, 3, F64, 4, di);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    EXPECT(threw);
    cudaMemcpy(dv, c.data(), 2 * sizeof(double), cudaMemcpyHostToDevice);
    EXPECT((exdyna::hard_threshold_select(dv, 2, F64, 0.3, di) == std::vector<int64_t>{1}));
    EXPECT((exdyna::hard_threshold_select(dv, 2, F64, 0.05, di) == std::vector<int64_t>{0, 1}));
    EXPECT(exdyna::hard_threshold_select(dv, 2, F64, 9.0, di).empty());
    cudaFree(dv);
    cudaFree(di);
  }
  std::printf("PASS baselines\n");
  return 0;
}
