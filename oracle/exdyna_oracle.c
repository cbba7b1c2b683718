/*
 * oracle/exdyna_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's ExDyna sparsify+sync step
 * (sparsim, /root/reference/proj) used as the checker for the CUDA path.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it; the product library never links or calls it.
 *
 * The engine is instantiated twice from oracle_step.inc:
 *   T = double  -> must reproduce the unmodified reference bit for bit
 *                  (pinned by tests/test_oracle_vs_ref.py against oracle/_ref);
 *   T = float   -> the fp32 restatement the GPU's fp32 mode is checked against:
 *                  the same step with float vectors and fp64 control, i.e.
 *                  every vector element is computed in double exactly as the
 *                  reference does and rounded once to float on store.
 * Pure functions cite the reference lines they restate. Build with
 * -ffp-contract=off and no -march (SURVEY.md §7 hard part 2).
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../include/exdyna.h"

static __thread char g_err[256];

static int fail(int code, const char* what) {
  snprintf(g_err, sizeof g_err, "%s", what);
  return code;
}

const char* orc_last_error(void) { return g_err; }

static int64_t mod_floor(int64_t a, int64_t n) { return ((a % n) + n) % n; } /* types.hpp:30-32 */

/* config.cpp:28-51 */
int orc_validate(const exd_config* in, exd_config* out) {
  const exd_config c = *in;
  if (c.n < 1) return fail(EXD_EINVAL, "worker count out of range");
  if (c.n_g < 1) return fail(EXD_EINVAL, "gradient count out of range");
  if (c.n_b < 1) return fail(EXD_EINVAL, "block count out of range");
  if (!(c.d > 0.0) || c.d > 1.0) return fail(EXD_EINVAL, "density out of range");
  if (c.has_delta0 && !(c.delta0 > 0.0)) return fail(EXD_EINVAL, "delta0 out of range");
  if (!(c.alpha > 1.0)) return fail(EXD_EINVAL, "alpha out of range");
  if (!(c.beta > 1.0)) return fail(EXD_EINVAL, "beta out of range");
  if (!(c.gamma > 0.0) || !(c.gamma < 1.0)) return fail(EXD_EINVAL, "gamma out of range");
  if (c.blk_move < 1) return fail(EXD_EINVAL, "blk_move out of range");
  if (c.min_blk < 1) return fail(EXD_EINVAL, "min_blk out of range");
  if (!(c.eta > 0.0)) return fail(EXD_EINVAL, "eta out of range");
  if (c.has_max_density_cap && (!(c.max_density_cap > 0.0) || c.max_density_cap > 1.0))
    return fail(EXD_EINVAL, "max_density_cap out of range");
  *out = c;
  out->k = (int64_t)llround(c.d * (double)c.n_g);
  if (c.n_b < (int64_t)c.n * c.min_blk) return fail(EXD_EINVAL, "n_b < n*min_blk");
  if (c.n_b > c.n_g) return fail(EXD_EINVAL, "n_b > n_g");
  if (out->k < c.n) return fail(EXD_EINVAL, "k < n");
  return 0;
}

/* partition.cpp:22-58 */
int orc_build_topology(int64_t n_g, int64_t n_b, int32_t n, int64_t min_blk,
                       exd_topology* out, char* warning, size_t wlen) {
  if (n < 1) return fail(EXD_EINVAL, "worker count out of range");
  if (n_b < 1 || n_b > n_g) return fail(EXD_EINVAL, "n_b out of range");
  if (n > EXD_MAX_WORKERS) return fail(EXD_EINVAL, "worker count out of range");
  const int64_t q = n_g / n_b;
  int64_t sz;
  if (q >= 32) {
    sz = q - q % 32;
    if (warning && wlen) warning[0] = 0;
  } else {
    sz = q > 1 ? q : 1;
    if (warning && wlen)
      snprintf(warning, wlen, "block size %lld below 32-element alignment; using unaligned blocks",
               (long long)sz);
  }
  const int64_t quo = n_b / n, rem = n_b % n;
  if (quo < min_blk) return fail(EXD_EINVAL, "partition would hold fewer than min_blk blocks");
  memset(out, 0, sizeof *out);
  out->n = n;
  out->sz_blk = sz;
  for (int i = 0; i < n; ++i) out->blk_part[i] = quo + (i < rem ? 1 : 0);
  for (int i = 1; i < n; ++i) out->blk_pos[i] = out->blk_pos[i - 1] + out->blk_part[i - 1];
  return 0;
}

/* partition.cpp:60-68 */
void orc_partition_range(const exd_topology* t, int32_t p, int64_t n_g, int64_t* st, int64_t* end) {
  *st = t->blk_pos[p] * t->sz_blk;
  *end = p == t->n - 1 ? n_g : (t->blk_pos[p] + t->blk_part[p]) * t->sz_blk;
}

/* allocator.cpp:23-38 */
void orc_rotate(const int64_t* k_rank, int64_t t, int32_t n, int64_t* k_part) {
  const int64_t shift = mod_floor(t - 1, n);
  for (int i = 0; i < n; ++i) k_part[(shift + i) % n] = k_rank[i];
}

/* allocator.cpp:40-90 */
void orc_adjust(exd_topology* topo, int64_t* k, double alpha, int64_t blk_move,
                int64_t min_blk, int64_t n_g, int32_t* moves, int32_t* skips) {
  const int n = topo->n;
  *moves = 0;
  *skips = 0;
  int64_t total = 0;
  for (int i = 0; i < n; ++i) total += k[i];
  if (total <= 0) return;
  const double pk_prev = (double)total / n;
  const double den_prev = (double)total / (double)n_g;
  const int64_t k_move = (int64_t)llround((double)(blk_move * topo->sz_blk) * den_prev);
  for (int i = 0; i + 1 < n; ++i) {
    const double det = (double)k[i] / pk_prev;
    const double det2 = (double)k[i + 1] / pk_prev;
    if (det > alpha && det2 < 1.0 / alpha) {
      if (topo->blk_part[i] - blk_move < min_blk) { ++*skips; continue; }
      topo->blk_part[i] -= blk_move;
      topo->blk_part[i + 1] += blk_move;
      topo->blk_pos[i + 1] -= blk_move;
      const int64_t moved = k_move < k[i] ? k_move : k[i];
      k[i] -= moved;
      k[i + 1] += moved;
      ++*moves;
    } else if (det < 1.0 / alpha && det2 > alpha) {
      if (topo->blk_part[i + 1] - blk_move < min_blk) { ++*skips; continue; }
      topo->blk_part[i] += blk_move;
      topo->blk_part[i + 1] -= blk_move;
      topo->blk_pos[i + 1] += blk_move;
      const int64_t moved = k_move < k[i + 1] ? k_move : k[i + 1];
      k[i] += moved;
      k[i + 1] -= moved;
      ++*moves;
    }
  }
}

/* allocator.cpp:92-99 */
void orc_allocate(const exd_topology* t, int64_t it, int32_t rank, int64_t n_g,
                  int32_t* partition, int64_t* st, int64_t* end) {
  *partition = (int32_t)mod_floor(mod_floor(it, t->n) + rank, t->n);
  orc_partition_range(t, *partition, n_g, st, end);
}

/* threshold.cpp:23-35 */
double orc_scale_threshold(int64_t k, int64_t kp, double delta, double beta, double gamma) {
  const double exam = (double)kp / (double)k;
  double sf;
  if (exam > beta) sf = 1.0 + gamma;
  else if (exam > 1.0 / beta) sf = 1.0 + 0.25 * gamma;
  else sf = 1.0 - gamma;
  return delta * sf;
}

/* order statistic: the value std::nth_element places at `pos` (unique as a value) */
static double select_kth(double* a, int64_t m, int64_t pos) {
  int64_t lo = 0, hi = m - 1;
  while (hi > lo) {
    const double pivot = a[lo + (hi - lo) / 2];
    int64_t i = lo, j = hi;
    while (i <= j) {
      while (a[i] < pivot) ++i;
      while (a[j] > pivot) --j;
      if (i <= j) { double tmp = a[i]; a[i] = a[j]; a[j] = tmp; ++i; --j; }
    }
    if (pos <= j) hi = j;
    else if (pos >= i) lo = i;
    else return a[pos];
  }
  return a[pos];
}

/* threshold.cpp:37-47; mags is clobbered */
int orc_initial_threshold(double* mags, int64_t m, double d, double* out) {
  if (m < 1) return fail(EXD_EINVAL, "initial_threshold: empty sample");
  int64_t pos = (int64_t)floor((1.0 - d) * (double)m);
  if (pos > m - 1) pos = m - 1;
  *out = select_kth(mags, m, pos);
  return 0;
}

/* collectives.cpp:29-45 accounting */
void orc_gather_stats(const int64_t* k_rank, int32_t n, exd_gather_stats* s) {
  int64_t total = 0, m = 0, pad = 0;
  for (int i = 0; i < n; ++i) { total += k_rank[i]; if (k_rank[i] > m) m = k_rank[i]; }
  for (int i = 0; i < n; ++i) pad += m - k_rank[i];
  s->k_prime = total;
  s->m_t = m;
  s->c_t = (int64_t)n * pad;
  s->f_t = total > 0 ? (double)n * (double)m / (double)total : 1.0;
}

/* ---- synthetic stream: rng.hpp:28-59 + workloads.cpp:42-85 ---- */
static uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

uint64_t orc_derive_key(const uint64_t* words, int nw) {
  uint64_t h = 0x6a09e667f3bcc909ULL;
  for (int i = 0; i < nw; ++i) h = mix64(h ^ words[i]);
  return h;
}

static double unit_of(uint64_t u) { return ((double)(u >> 11) + 0.5) * 0x1.0p-53; }

int orc_synthetic_gradient(const exd_stream_spec* s, int64_t t, int32_t rank, double* out) {
  int64_t pos = 0;
  for (int si = 0; si < s->nseg; ++si) {
    double scale = s->seg_scale[si] * pow(s->decay, (double)t);
    if (s->has_decay_step && t >= s->decay_step) scale *= s->decay_step_factor;
    const uint64_t words[5] = {s->seed, 0x53545245414dULL, (uint64_t)t, (uint64_t)rank,
                               (uint64_t)si};
    uint64_t state = orc_derive_key(words, 5);
    for (int64_t j = 0; j < s->seg_length[si]; ++j) {
      if (s->distribution == 0) {
        state += 0x9e3779b97f4a7c15ULL;
        const double u = unit_of(mix64(state)) - 0.5;
        const double mag = -scale * log1p(-2.0 * fabs(u));
        out[pos++] = u < 0.0 ? -mag : mag;
      } else {
        state += 0x9e3779b97f4a7c15ULL;
        const double u1 = unit_of(mix64(state));
        state += 0x9e3779b97f4a7c15ULL;
        const double u2 = unit_of(mix64(state));
        const double z = sqrt(-2.0 * log(u1)) * cos(6.283185307179586477 * u2);
        const double mag = scale * exp(z);
        state += 0x9e3779b97f4a7c15ULL;
        out[pos++] = (mix64(state) & 1ULL) ? mag : -mag;
      }
    }
  }
  return 0;
}

/* ---- the engine, once per element type ---- */
static int cmp_i64(const void* a, const void* b) {
  const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return (x > y) - (x < y);
}

#define T double
#define SUF f64
#include "oracle_step.inc"
#undef T
#undef SUF

#define T float
#define SUF f32
#include "oracle_step.inc"
#undef T
#undef SUF
