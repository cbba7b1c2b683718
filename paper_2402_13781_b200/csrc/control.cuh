// control.cuh — ExDyna's O(n) control plane, compiled for host AND device.
//
// The same functions serve the C ABI's pure host entry points
// (exd_rotate_to_partition_order, exd_adjust_topology, ...) and the
// single-thread control epilogue that runs on the GPU each step, so the
// replicated control state never has to visit the host.
//
// Bit-exactness rules (SURVEY.md §7 hard part 2): every fp64 operation that
// the reference writes as a separate multiply and add is issued with explicit
// round-to-nearest intrinsics on the device (no FMA contraction); the host
// side is compiled with -ffp-contract=off.
#pragma once

#include <stdint.h>

#include "exdyna.h"

#ifdef __CUDACC__
#define EXD_HD __host__ __device__ __forceinline__
#else
#define EXD_HD inline
#endif

namespace exd {

EXD_HD double dmul(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}
EXD_HD double dadd(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}
EXD_HD double ddiv(double a, double b) {
#ifdef __CUDA_ARCH__
  return __ddiv_rn(a, b);
#else
  return a / b;
#endif
}
EXD_HD int64_t llround_d(double v) {
#ifdef __CUDA_ARCH__
  return (int64_t)llround(v);
#else
  return (int64_t)__builtin_llround(v);
#endif
}

// types.hpp:30-32
EXD_HD int64_t mod_floor(int64_t a, int64_t n) { return ((a % n) + n) % n; }

// partition_range, partition.cpp:60-68
EXD_HD void partition_range(const exd_topology& t, int p, int64_t n_g, int64_t* st,
                            int64_t* end) {
  *st = t.blk_pos[p] * t.sz_blk;
  *end = p == t.n - 1 ? n_g : (t.blk_pos[p] + t.blk_part[p]) * t.sz_blk;
}

// rotate_to_partition_order, allocator.cpp:23-38 (Alg. 3 l.3-6)
EXD_HD void rotate(const int64_t* k_rank, int64_t t, int n, int64_t* k_part) {
  const int64_t shift = mod_floor(t - 1, n);
  for (int i = 0; i < n; ++i) k_part[(shift + i) % n] = k_rank[i];
}

// rotate with t-1 already reduced mod n (the device keeps t mod n): the same
// mapping with 32-bit arithmetic and no division
EXD_HD void rotate_m(const int64_t* k_rank, int shift, int n, int64_t* k_part) {
  for (int i = 0; i < n; ++i) {
    int j = shift + i;
    if (j >= n) j -= n;
    k_part[j] = k_rank[i];
  }
}

// adjust_topology, allocator.cpp:40-90 (Alg. 3): one left-to-right sweep of
// adjacent-pair block migrations; later pairs see updated counts. `inv_alpha`
// is 1.0 / alpha, precomputed (the same IEEE quotient on host and device).
EXD_HD void adjust_r(exd_topology& topo, int64_t* k, double alpha, double inv_alpha,
                     int64_t blk_move, int64_t min_blk, int64_t n_g, int32_t* moves,
                     int32_t* skips);

EXD_HD void adjust(exd_topology& topo, int64_t* k, double alpha, int64_t blk_move,
                   int64_t min_blk, int64_t n_g, int32_t* moves, int32_t* skips) {
  adjust_r(topo, k, alpha, ddiv(1.0, alpha), blk_move, min_blk, n_g, moves, skips);
}

EXD_HD void adjust_r(exd_topology& topo, int64_t* k, double alpha, double inv_alpha,
                     int64_t blk_move, int64_t min_blk, int64_t n_g, int32_t* moves,
                     int32_t* skips) {
  const int n = topo.n;
  *moves = 0;
  *skips = 0;
  int64_t total = 0;
  for (int i = 0; i < n; ++i) total += k[i];
  if (total <= 0) return;
  const double pk_prev = ddiv((double)total, (double)n);
  const double den_prev = ddiv((double)total, (double)n_g);
  const int64_t k_move = llround_d(dmul((double)(blk_move * topo.sz_blk), den_prev));
  for (int i = 0; i + 1 < n; ++i) {
    const double det = ddiv((double)k[i], pk_prev);
    const double det2 = ddiv((double)k[i + 1], pk_prev);
    if (det > alpha && det2 < inv_alpha) {
      if (topo.blk_part[i] - blk_move < min_blk) {
        ++*skips;
        continue;
      }
      topo.blk_part[i] -= blk_move;
      topo.blk_part[i + 1] += blk_move;
      topo.blk_pos[i + 1] -= blk_move;
      const int64_t moved = k_move < k[i] ? k_move : k[i];
      k[i] -= moved;
      k[i + 1] += moved;
      ++*moves;
    } else if (det < inv_alpha && det2 > alpha) {
      if (topo.blk_part[i + 1] - blk_move < min_blk) {
        ++*skips;
        continue;
      }
      topo.blk_part[i] += blk_move;
      topo.blk_part[i + 1] -= blk_move;
      topo.blk_pos[i + 1] += blk_move;
      const int64_t moved = k_move < k[i + 1] ? k_move : k[i + 1];
      k[i] += moved;
      k[i + 1] -= moved;
      ++*moves;
    }
  }
}

// allocate_partition, allocator.cpp:92-99: cyclic (t % n + rank) % n
EXD_HD int allocate(const exd_topology& t, int64_t it, int rank, int64_t n_g, int64_t* st,
                    int64_t* end) {
  const int p = (int)mod_floor(mod_floor(it, t.n) + rank, t.n);
  partition_range(t, p, n_g, st, end);
  return p;
}

// allocate with t reduced mod n (device): (t % n + rank) % n without division
EXD_HD int allocate_m(const exd_topology& t, int tmod, int rank, int64_t n_g, int64_t* st,
                      int64_t* end) {
  int p = tmod + rank;
  if (p >= t.n) p -= t.n;
  partition_range(t, p, n_g, st, end);
  return p;
}

// scale_threshold, threshold.cpp:23-35 (Alg. 5). `1.0 + 0.25*gamma` must not
// be contracted into an FMA. `inv_beta` is 1.0 / beta, precomputed.
EXD_HD double scale_threshold_r(int64_t k, int64_t k_prime, double delta, double beta,
                                double inv_beta, double gamma) {
  const double exam = ddiv((double)k_prime, (double)k);
  double sf;
  if (exam > beta) {
    sf = dadd(1.0, gamma);
  } else if (exam > inv_beta) {
    sf = dadd(1.0, dmul(0.25, gamma));
  } else {
    sf = dadd(1.0, -gamma);
  }
  return dmul(delta, sf);
}

EXD_HD double scale_threshold(int64_t k, int64_t k_prime, double delta, double beta,
                              double gamma) {
  return scale_threshold_r(k, k_prime, delta, beta, ddiv(1.0, beta), gamma);
}

// all_gather accounting, collectives.cpp:29-45 (Eqs. 2-5)
EXD_HD void gather_stats(const int64_t* k_rank, int n, exd_gather_stats* s) {
  int64_t total = 0, m = 0, pad = 0;
  for (int i = 0; i < n; ++i) {
    total += k_rank[i];
    if (k_rank[i] > m) m = k_rank[i];
  }
  for (int i = 0; i < n; ++i) pad += m - k_rank[i];
  s->k_prime = total;
  s->m_t = m;
  s->c_t = (int64_t)n * pad;
  s->f_t = total > 0 ? ddiv(dmul((double)n, (double)m), (double)total) : 1.0;
}

}  // namespace exd
