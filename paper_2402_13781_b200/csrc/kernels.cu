// kernels.cu — the sm_100a kernels of the ExDyna sparsify+sync path.
//
//   stream_kernel   (K1) accumulate e <- e + eta*g over the full vector,
//                   |acc| >= delta over the worker's exclusive partition,
//                   own selected residuals zeroed, the selection staged in
//                   order per warp chunk as (index, value) pairs, per-block
//                   counts. PUSH variant (one rank per GPU): the staged
//                   indices (packed per tile) and counts also go to every
//                   peer's inbox.
//   finish_kernel   (K2) per-chunk counts -> global offsets, dense ascending
//                   idx/val lists; for n == 1 also x -= g/n and the control
//                   epilogue, so a step is two launches chained by PDL.
//   exchange_kernel (K2 + sync, one rank per GPU, push-reduce) union in
//                   partition order, contributions out and in as {value,
//                   epoch} words, rank-order sum, x -= g/n, epilogue.
//   p2p_sync        (pull-reduce peer sync) and union / allreduce_local /
//                   finalize (in-process workers, NCCL path): K4-K9.
//   cap_kernel      density cap (selector.cpp:44-61).
//   quantile        (K8) radix select of the (1-d)-quantile of |acc| at t = 0.
//   synthetic       device GradientSource (workloads.cpp:62-85).
//   verify / hash / conservation kernels: the reference's debug invariants.
//
// Reference lines are cited at each kernel. Everything here is HBM- or
// latency-bound integer/byte work: there is no GEMM to put on tcgen05, so the
// design levers are 128-bit coalesced loads, enough bytes in flight, one pass
// over HBM, and grids sized to the 148 SMs.
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>
#include <atomic>

#include "internal.cuh"

namespace exd {

#ifdef EXD_PROBE
// experiment build only: globaltimer stamps of the finish kernel's phases
__device__ unsigned long long g_probe[64];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define PROBE(i) \
  do { if (threadIdx.x == 0) g_probe[i] = gtimer(); } while (0)
#define PROBE_ANY(i) do { g_probe[i] = gtimer(); } while (0)
#define PROBE_MAX(i) do { if (threadIdx.x == 0) atomicMax(&g_probe[i], gtimer()); } while (0)
__device__ unsigned long long g_cta[4][2048];
#define CPROBE(i, c) do { if (threadIdx.x == 0 && (c) < 2048) g_cta[i][c] = gtimer(); } while (0)
#define CPROBE_V(i, c, v) do { if (threadIdx.x == 0 && (c) < 2048) g_cta[i][c] = (v); } while (0)
#else
#define CPROBE(i, c) do {} while (0)
#define CPROBE_V(i, c, v) do {} while (0)
#define PROBE_MAX(i) do {} while (0)
#define PROBE(i) do {} while (0)
#define PROBE_ANY(i) do {} while (0)
#endif

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
#ifndef EXD_K1_UNROLL
#define EXD_K1_UNROLL 4
#endif
#ifndef EXD_K1_MINB
#define EXD_K1_MINB 4
#endif
constexpr int kUnroll = EXD_K1_UNROLL;  // 16 B vectors per lane per stream in the stream kernel


template <typename T> struct Vec;
template <> struct Vec<float> {
  using V = float4;
  static constexpr int N = 4;
};
template <> struct Vec<double> {
  using V = double2;
  static constexpr int N = 2;
};

template <typename T> __host__ __device__ constexpr int tile_of() { return kThreads * Vec<T>::N * kUnroll; }

template <typename T> __device__ __forceinline__ void vload(const T* p, T (&r)[Vec<T>::N]);
template <> __device__ __forceinline__ void vload<float>(const float* p, float (&r)[4]) {
  const float4 v = __ldcs(reinterpret_cast<const float4*>(p));
  r[0] = v.x; r[1] = v.y; r[2] = v.z; r[3] = v.w;
}
template <> __device__ __forceinline__ void vload<double>(const double* p, double (&r)[2]) {
  const double2 v = __ldcs(reinterpret_cast<const double2*>(p));
  r[0] = v.x; r[1] = v.y;
}
template <typename T> __device__ __forceinline__ void vstore(T* p, const T (&r)[Vec<T>::N]);
template <> __device__ __forceinline__ void vstore<float>(float* p, const float (&r)[4]) {
  __stcs(reinterpret_cast<float4*>(p), make_float4(r[0], r[1], r[2], r[3]));
}
template <> __device__ __forceinline__ void vstore<double>(double* p, const double (&r)[2]) {
  __stcs(reinterpret_cast<double2*>(p), make_double2(r[0], r[1]));
}

// e + eta * g with the reference's rounding (engine.cpp:139): one fp64 mul,
// one fp64 add, one rounding to T. For T = float and eta == 1 the float add is
// the same correctly rounded result (double rounding of a float sum through
// double is innocuous), so the fast path is exact.
template <typename T> __device__ __forceinline__ T accumulate(T prev, T g, double eta, bool unit);
template <> __device__ __forceinline__ float accumulate<float>(float prev, float g, double eta,
                                                               bool unit) {
  if (unit) return __fadd_rn(prev, g);
  return __double2float_rn(__dadd_rn((double)prev, __dmul_rn(eta, (double)g)));
}
template <> __device__ __forceinline__ double accumulate<double>(double prev, double g, double eta,
                                                                 bool) {
  return __dadd_rn(prev, __dmul_rn(eta, g));  // eta == 1: the multiply is exact
}

// x -= g / n (engine.cpp:215) evaluated in fp64, rounded once to T
template <typename T> __device__ __forceinline__ T apply_update(T x, T g, int n) {
  // g / n is exact as g * (1/n) when n is a power of two
  const double q = (n & (n - 1)) == 0 ? __dmul_rn((double)g, 1.0 / (double)n)
                                      : __ddiv_rn((double)g, (double)n);
  return (T)__dadd_rn((double)x, -q);
}

__device__ __forceinline__ float thr_of(double delta) { return __double2float_ru(delta); }

// |acc| >= delta (selector.cpp:39) with delta in fp64: for float acc,
// (double)|acc| >= delta  <=>  |acc| >= round_up_to_float(delta); for double
// acc the key is delta itself.
template <typename T> __device__ __forceinline__ T thr_key(const Ctrl* c);
template <> __device__ __forceinline__ float thr_key<float>(const Ctrl* c) { return c->thr_f; }
template <> __device__ __forceinline__ double thr_key<double>(const Ctrl* c) { return c->delta; }
__device__ __forceinline__ float fabs_t(float v) { return fabsf(v); }
__device__ __forceinline__ double fabs_t(double v) { return fabs(v); }

// ---- control epilogue ----------------------------------------------------
// The end of step t, once the gathered counts are known:
//   delta   threshold rescale, k_t update, topology commit (engine.cpp:206-213)
//   plan    step t+1's rotate -> adjust -> allocate (engine.cpp:125-131)
//   record  the raw ledger row; the host derives the reference's
//           IterationRecord from it at sync (engine.cpp:327-349)
// It is sequential O(n) fp64 work with long dependency chains, so one CTA
// stages the control block in shared memory (prefetched while the CTA's
// totals are still loading) and runs delta and plan on two warps
// concurrently; step t+1's plan goes to the other plan slot, so nothing else
// has to wait.
__device__ __forceinline__ void copy_topo(exd_topology* dst, const exd_topology* src, int n) {
  dst->n = src->n;
  dst->sz_blk = src->sz_blk;
  for (int i = 0; i < n; ++i) {
    dst->blk_part[i] = src->blk_part[i];
    dst->blk_pos[i] = src->blk_pos[i];
  }
}

// plan of step t_next from the topology committed by step t_next-1 and the
// counts gathered at step t_next-1 (rank order)
// (`kp` is shared-memory scratch: a local array would live in local memory,
// where every first touch of the dependent chain is an L2 round trip)
// inlined into the epilogue: one straight code path to fetch cold after the
// stream has evicted it (measured: 34.5 -> 34.0 us per R18 step vs __noinline__)
#ifdef EXD_XP_NOINLINE_EPI
#define EXD_EPI_INLINE __noinline__
#else
#define EXD_EPI_INLINE __forceinline__
#endif
__device__ EXD_EPI_INLINE void make_plan(Plan* p, const exd_topology* base, const int64_t* k_rank,
                                       int tm_next, const RunConst& rc, int64_t* kp) {
  // tm_next = t_next mod n; rotate's shift is (t_next - 1) mod n
  const int n = rc.n;
  copy_topo(&p->topo, base, n);
  int32_t mv = 0, sk = 0;
  if (!rc.static_partitions && n > 1) {  // one partition: no pairs to adjust
    rotate_m(k_rank, tm_next == 0 ? n - 1 : tm_next - 1, n, kp);
    adjust_r(p->topo, kp, rc.alpha, rc.inv_alpha, rc.blk_move, rc.min_blk, rc.n_g, &mv, &sk);
  }
  p->moves = mv;
  p->skips = sk;
  int64_t st, end;
  p->partition = allocate_m(p->topo, tm_next, rc.rank, rc.n_g, &st, &end);
  p->st = st;
  p->end = end;
}

__device__ EXD_EPI_INLINE void advance_delta(Ctrl* c, const int64_t* k_rank, const RunConst& rc) {
  const int n = rc.n;
  int64_t kp = 0;
  for (int r = 0; r < n; ++r) {
    kp += k_rank[r];
    c->k_t[r] = k_rank[r];
  }
  c->delta = scale_threshold_r(rc.k, kp, c->delta, rc.beta, rc.inv_beta, rc.gamma);
  c->thr_f = thr_of(c->delta);
  const Plan* cur = &c->plan[c->t & 1];
  copy_topo(&c->topo, &cur->topo, n);
  copy_topo(&c->last.topo, &cur->topo, n);
  c->last.st = cur->st;
  c->last.end = cur->end;
  c->last.partition = cur->partition;
  c->last.moves = cur->moves;
  c->last.skips = cur->skips;
  c->t += 1;
  c->tmod = c->tmod + 1 == n ? 0 : c->tmod + 1;
}

// Shared-memory staging of the control block for one CTA.
struct EpiShared {
  Ctrl c;
  int64_t k_rank[EXD_MAX_WORKERS];
  double norm2[EXD_MAX_WORKERS];
  int64_t capped[EXD_MAX_WORKERS];
  int64_t scratch[EXD_MAX_WORKERS];  // make_plan's partition-order counts
};

__device__ __forceinline__ void epi_load(EpiShared& sh, const Ctrl* cg) {
  static_assert(sizeof(Ctrl) % 8 == 0, "word copies");
  unsigned long long* sw = reinterpret_cast<unsigned long long*>(&sh.c);
  const unsigned long long* gw = reinterpret_cast<const unsigned long long*>(cg);
  constexpr int W = (int)(sizeof(Ctrl) / 8);
#pragma unroll 4
  for (int i = threadIdx.x; i < W; i += blockDim.x) sw[i] = __ldcg(&gw[i]);
}

// Run the epilogue on the staged copy (sh.c, sh.k_rank, sh.norm2 filled;
// caller synced), then write the control block and the record back. Whole CTA.
__device__ __forceinline__ void epi_run_store(EpiShared& sh, Ctrl* cg, const RunConst& rc,
                                              RawRecord* rec_out) {
  const int tid = threadIdx.x;
  const int64_t t = sh.c.t;
  const int tm_next = sh.c.tmod + 1 == rc.n ? 0 : sh.c.tmod + 1;
  const double delta_used = sh.c.delta;
  __syncthreads();  // everyone read t / tmod / delta before warp 0 changes them
  if (tid == 0) {
    advance_delta(&sh.c, sh.k_rank, rc);
    sh.c.done = 0;
    PROBE_ANY(26);
  } else if (tid == 32) {
    make_plan(&sh.c.plan[(t + 1) & 1], &sh.c.plan[t & 1].topo, sh.k_rank, tm_next, rc, sh.scratch);
    PROBE_ANY(27);
  } else if (tid == 64 && rec_out) {
    const Plan& cur = sh.c.plan[t & 1];
    rec_out->t = t;
    rec_out->delta = delta_used;
    rec_out->moves = cur.moves;
    rec_out->skips = cur.skips;
    rec_out->n = rc.n;
    rec_out->reserved = 0;
  }
  if (rec_out)
    for (int r = tid; r < rc.n; r += blockDim.x) {
      rec_out->k_rank[r] = sh.k_rank[r];
      rec_out->norm2[r] = sh.norm2[r];
      rec_out->capped[r] = sh.capped[r];
    }
  __syncthreads();
  unsigned long long* sw = reinterpret_cast<unsigned long long*>(&sh.c);
  unsigned long long* gw = reinterpret_cast<unsigned long long*>(cg);
  for (int i = tid; i < (int)(sizeof(Ctrl) / 8); i += blockDim.x) gw[i] = sw[i];
}

// Standalone form: load, run, store (finalize kernel, block 0).
__device__ __forceinline__ void control_epilogue_cta(Ctrl* cg, const CountRec* counts,
                                                     const RunConst& rc, RawRecord* rec_out) {
  __shared__ EpiShared sh;
  epi_load(sh, cg);
  for (int r = threadIdx.x; r < rc.n; r += blockDim.x) {
    sh.k_rank[r] = __ldcg(&counts[r].k);
    sh.norm2[r] = __ldcg(&counts[r].norm2);
    sh.capped[r] = __ldcg(&counts[r].capped);
  }
  __syncthreads();
  PROBE(4);
  epi_run_store(sh, cg, rc, rec_out);
  PROBE(5);
}

// ---- K1: the streaming kernel (accumulate / select / stage) -----------------
// engine.cpp:135-141 (accumulate), selector.cpp:35-42 (select), engine.cpp:199-202
// (values), selector.cpp:63-65 (clear, own partition).
//
// One tile per CTA, one contiguous warp chunk of 32 * VN * kUnroll elements per
// warp; lane `l` owns elements chunk + u*32*VN + l*VN + c, so every u is one
// fully coalesced 512 B warp access and the ascending order of a chunk's
// selection is (u, lane, c). Each warp compacts its own chunk with ballots into
// a staging run of its own (no block barriers, no inter-CTA waiting); the
// finish kernel turns the per-chunk counts into global offsets. This keeps K1
// a pure stream: it runs at the measured copy bandwidth.
template <typename T> __host__ __device__ constexpr int chunk_of() { return 32 * Vec<T>::N * kUnroll; }

// staged (index, value) pairs: one 8 B (fp32) / 16 B (fp64) store per selected
// element instead of two scattered ones
template <typename T> struct Pair;
template <> struct Pair<float> {
  using P = uint2;
  __device__ static P make(uint32_t j, float v) { return make_uint2(j, __float_as_uint(v)); }
  __device__ static uint32_t idx(const P& p) { return p.x; }
  __device__ static float val(const P& p) { return __uint_as_float(p.y); }
  __device__ static void store_keep(P* q, const P& p, uint64_t pol) {  // L2 policy `pol`
    asm volatile("st.global.L2::cache_hint.v2.u32 [%0], {%1, %2}, %3;" ::"l"(q), "r"(p.x), "r"(p.y),
                 "l"(pol) : "memory");
  }
};
template <> struct Pair<double> {
  using P = ulonglong2;
  __device__ static P make(uint32_t j, double v) {
    return make_ulonglong2((unsigned long long)j, (unsigned long long)__double_as_longlong(v));
  }
  __device__ static uint32_t idx(const P& p) { return (uint32_t)p.x; }
  __device__ static double val(const P& p) { return __longlong_as_double((long long)p.y); }
  __device__ static void store_keep(P* q, const P& p, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.u64 [%0], {%1, %2}, %3;" ::"l"(q), "l"(p.x), "l"(p.y),
                 "l"(pol) : "memory");
  }
};

template <typename V>
__device__ __forceinline__ V warp_sum(V v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ExDyna block of element j: min(j / sz_blk, n_b - 1) (the last block absorbs
// the tail, partition.cpp:60-68), by multiply-shift with the run's magic
// numbers (exact for j < 2^31; see blk_magic in engine.cu)
__device__ __forceinline__ uint32_t block_of(uint32_t j, const RunConst& rc) {
  const uint32_t b = (uint32_t)(((unsigned long long)j * rc.blk_magic) >> rc.blk_shift);
  return b < (uint32_t)(rc.n_b - 1) ? b : (uint32_t)(rc.n_b - 1);
}

// {payload, epoch} words (the low-latency protocol of the push-reduce sync):
// each aligned 8-byte word is single-copy atomic, so it is its own flag
__device__ __forceinline__ void st_relaxed_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys_v2u64(unsigned long long* p, unsigned long long a,
                                                     unsigned long long b) {
  asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// PUSH (one rank per GPU, push-reduce sync): the staged indices and the
// per-chunk / per-tile counts of the partition also go to every peer's inbox.
template <typename T, int MODE, bool UNIT, bool PUSH>
__global__ void __launch_bounds__(kThreads, EXD_K1_MINB) stream_kernel(SelectArgs a, RunConst rc) {
  constexpr int VN = Vec<T>::N;
  constexpr int CH = chunk_of<T>();
  constexpr bool ACCUM = MODE != kSelectOnly;
  constexpr bool SELECT = MODE != kAccumulate;
  static_assert(CH * kWarps == tile_of<T>(), "tile = kWarps chunks");
  __shared__ double s_norm[kWarps];
  __shared__ int s_cnt[kWarps];
  // PUSH: each warp's run of staged indices, packed per tile for the peers
  __shared__ int32_t s_run[PUSH ? kWarps * CH : 1];

  const Ctrl* ctrl = a.ctrl;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tile = a.tile_base + (int)blockIdx.x;
#ifdef EXD_PROBE
  // the previous step's last stamps, before this step overwrites them
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    g_probe[50] = g_probe[44];
    g_probe[51] = g_probe[16];
    g_probe[52] = g_probe[30];  // the finish kernel's last stamp (n == 1)
  }
#endif
  if (blockIdx.x == 0) PROBE(16);
  if (blockIdx.x == gridDim.x - 1) PROBE(17);
  // programmatic dependent launch: once every CTA of this grid has started,
  // the finish kernel may be scheduled (it waits for our completion before
  // reading anything we write)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // n_g < 2^31 (checked at engine creation): 32-bit element indices throughout
  const uint32_t n_g = (uint32_t)rc.n_g;
  const uint32_t cbeg = (uint32_t)(tile * kWarps + warp) * CH;
  const uint32_t lbeg = cbeg + lane * VN;  // this lane's first element
  T* e = static_cast<T*>(a.e);
  const T* g = static_cast<const T*>(a.g);

  // issue every load of the chunk before any use: 2 * kUnroll 16 B loads in
  // flight per lane
  T ev[kUnroll][VN], gv[kUnroll][VN];
  const bool full = cbeg + CH <= n_g;
  if (full) {
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      vload<T>(e + lbeg + u * 32 * VN, ev[u]);
      if (ACCUM) vload<T>(g + lbeg + u * 32 * VN, gv[u]);
    }
  } else {
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
#pragma unroll
      for (int c = 0; c < VN; ++c) {
        const uint32_t j = lbeg + u * 32 * VN + c;
        ev[u][c] = j < n_g ? e[j] : T(0);
        gv[u][c] = (ACCUM && j < n_g) ? g[j] : T(0);
      }
  }
  const Plan& plan = ctrl->plan[a.t & 1];
  const uint32_t st = (uint32_t)plan.st, end = (uint32_t)plan.end;

  T v[kUnroll][VN];
  double nrm = 0.0;
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) {
    if (ACCUM) {
      // squares of VN elements in T, then one fp64 add (global_err is checked
      // to 1e-6 relative; the reference sums sequentially in fp64)
      T sq = T(0);
#pragma unroll
      for (int c = 0; c < VN; ++c) {
        sq = fma(ev[u][c], ev[u][c], sq);
        v[u][c] = accumulate<T>(ev[u][c], gv[u][c], rc.eta, UNIT);
      }
#ifndef EXD_XP_NO_NORM
      nrm += (double)sq;
#endif
    } else {
#pragma unroll
      for (int c = 0; c < VN; ++c) v[u][c] = ev[u][c];
    }
  }

#ifdef EXD_XP_NO_SELECT
  const bool sel_chunk = false;
#else
  const bool sel_chunk = SELECT && cbeg < end && cbeg + CH > st;
#endif
  uint32_t flags = 0;
  if (sel_chunk) {
    const T thr = thr_key<T>(ctrl);
    if (cbeg >= st && cbeg + CH <= end) {
#pragma unroll
      for (int u = 0; u < kUnroll; ++u)
#pragma unroll
        for (int c = 0; c < VN; ++c)
          flags |= (uint32_t)(fabs_t(v[u][c]) >= thr) << (u * VN + c);
    } else {
#pragma unroll
      for (int u = 0; u < kUnroll; ++u)
#pragma unroll
        for (int c = 0; c < VN; ++c) {
          const uint32_t j = lbeg + u * 32 * VN + c;
          flags |= (uint32_t)(j >= st && j < end && fabs_t(v[u][c]) >= thr) << (u * VN + c);
        }
    }
  }

  // residual write-back: acc, or 0 where selected (own partition cleared here)
  if (ACCUM) {
    if (full) {
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        T w[VN];
#pragma unroll
        for (int c = 0; c < VN; ++c) w[c] = (flags >> (u * VN + c)) & 1u ? T(0) : v[u][c];
        vstore<T>(e + lbeg + u * 32 * VN, w);
      }
    } else {
#pragma unroll
      for (int u = 0; u < kUnroll; ++u)
#pragma unroll
        for (int c = 0; c < VN; ++c) {
          const uint32_t j = lbeg + u * 32 * VN + c;
          if (j < n_g) e[j] = (flags >> (u * VN + c)) & 1u ? T(0) : v[u][c];
        }
    }
  } else if (flags) {
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
#pragma unroll
      for (int c = 0; c < VN; ++c)
        if ((flags >> (u * VN + c)) & 1u) e[lbeg + u * 32 * VN + c] = T(0);
  }

  // warp-level ordered compaction of the chunk into its staging run
  int running = 0;
  if (sel_chunk) {
    const uint32_t lt = (1u << lane) - 1u;
    const uint32_t lo = cbeg > st ? cbeg : st;
    // the run's place in the staging buffer: the global index of the chunk's
    // first element of this partition, so the runs of the two holders of a
    // chunk that straddles a partition boundary never overlap (the peers'
    // inboxes keep one staging slot for all sources)
    const uint32_t sbase = lo;
    uint64_t keep;
    if (a.stage_keep)
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
    else
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(keep));
    typename Pair<T>::P* sp = static_cast<typename Pair<T>::P*>(a.stage);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint32_t nib = (flags >> (u * VN)) & ((1u << VN) - 1u);
      const uint32_t cnt = __popc(nib);
      const uint32_t b0 = __ballot_sync(0xffffffffu, cnt & 1u);
      const uint32_t b1 = __ballot_sync(0xffffffffu, cnt & 2u);
      const uint32_t b2 = __ballot_sync(0xffffffffu, cnt & 4u);
      if (nib) {
        uint32_t pos = running + __popc(b0 & lt) + 2u * __popc(b1 & lt) + 4u * __popc(b2 & lt);
#pragma unroll
        for (int c = 0; c < VN; ++c) {
          if ((nib >> c) & 1u) {
            const uint32_t j = lbeg + u * 32 * VN + c;
            // straight to the staging buffer (measured faster than compacting
            // through shared memory first: 24.0 vs 27.6 us at R18)
            Pair<T>::store_keep(&sp[sbase + pos], Pair<T>::make(j, v[u][c]), keep);
            if (PUSH) s_run[warp * CH + pos] = (int32_t)j;
            ++pos;
          }
        }
      }
      running += (int)(__popc(b0) + 2u * __popc(b1) + 4u * __popc(b2));
    }
    if (PUSH && !a.tile_pack && running) {
      // the run sbase + [0, running) in every peer's staging slot as
      // {index, epoch} words, each word its own flag: 16 B stores of two words
      // (a leading word when sbase is odd)
      __syncwarp();
      const unsigned long long eph = (unsigned long long)(uint32_t)(a.t + 1) << 32;
      const int32_t* run = s_run + warp * CH;
      const int h0 = (int)(sbase & 1u);
      for (int q = 0; q < a.k1_npush; ++q) {
        unsigned long long* dst = a.push_stage[q] + sbase;
        if (h0 && lane == 0) st_relaxed_sys_u64(dst, eph | (uint32_t)run[0]);
        for (int i = h0 + 2 * lane; i < running; i += 64) {
          if (i + 1 < running)
            st_relaxed_sys_v2u64(dst + i, eph | (uint32_t)run[i], eph | (uint32_t)run[i + 1]);
          else
            st_relaxed_sys_u64(dst + i, eph | (uint32_t)run[i]);
        }
      }
    }
  }
  constexpr int TILE = tile_of<T>();
  const bool push_tile = PUSH && (uint32_t)tile >= st / TILE && (uint32_t)tile <= (end - 1) / TILE;
  if (SELECT && lane == 0) a.chunk_count[tile * kWarps + warp] = running;
#ifdef EXD_XP_NO_TILE
  return;
#endif

  if (ACCUM) nrm = warp_sum(nrm);
  if (lane == 0) {
    s_norm[warp] = nrm;
    s_cnt[warp] = running;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (ACCUM) {
      double sn = 0.0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) sn += s_norm[w];
      a.tile_norm[tile] = sn;
    }
    if (SELECT) {
      int sc = 0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) sc += s_cnt[w];
      a.tile_count[tile] = sc;
    }
  }
  if (PUSH && a.tile_pack && s_cnt[0] + s_cnt[1] + s_cnt[2] + s_cnt[3] + s_cnt[4] + s_cnt[5] + s_cnt[6] +
                   s_cnt[7] > 0) {
    // the tile's staged indices, packed in chunk order, into every peer's inbox
    // at max(tile start, partition start) as {index, epoch} words (each word
    // its own flag): one contiguous burst per tile and destination. Per-warp
    // runs of a few words each were bound by the NVLink request rate
    // (tools/nvl_word_bench.cu: ~5 G short runs/s per GPU), not by bytes.
    static_assert(kWarps == 8, "the packed offsets below sum 8 chunk counts");
    int woff[kWarps], sc = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      woff[w] = sc;
      sc += s_cnt[w];
    }
    const uint32_t t0 = (uint32_t)tile * TILE;
    const uint32_t tb = t0 > st ? t0 : st;
    const int h0 = (int)(tb & 1u);  // a leading single word when tb is odd
    const unsigned long long eph = (unsigned long long)(uint32_t)(a.t + 1) << 32;
    auto word = [&](int i) {
      int w = 0;
#pragma unroll
      for (int k = 1; k < kWarps; ++k) w += woff[k] <= i;
      return eph | (uint32_t)s_run[w * CH + (i - woff[w])];
    };
    for (int q = 0; q < a.k1_npush; ++q) {
      unsigned long long* dst = a.push_stage[q] + tb;
      for (int i = 2 * (int)threadIdx.x - h0; i < sc; i += 2 * kThreads) {
        if (i < 0)
          st_relaxed_sys_u64(dst, word(0));
        else if (i + 1 < sc)
          st_relaxed_sys_v2u64(dst + i, word(i), word(i + 1));
        else
          st_relaxed_sys_u64(dst + i, word(i));
      }
    }
  }
  if (push_tile && warp == 0) {
    // the tile's kWarps chunk counts and its count as {count, epoch} words into
    // every inbox: one store per lane (4 chunk-count pairs + the tile count per
    // destination), not a serial loop on one thread
    static_assert(kWarps == 8, "4 chunk-count pairs per tile");
    int sc = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) sc += s_cnt[w];
    const unsigned long long eph = (unsigned long long)(uint32_t)(a.t + 1) << 32;
    for (int l = lane; l < a.k1_npush * 5; l += 32) {
      const int q = l / 5, i = l - 5 * q;
      if (i < 4)
        st_relaxed_sys_v2u64(a.push_chunk[q] + tile * kWarps + 2 * i, eph | (uint32_t)s_cnt[2 * i],
                             eph | (uint32_t)s_cnt[2 * i + 1]);
      else
        st_relaxed_sys_u64(a.push_tile[q] + tile, eph | (uint32_t)sc);
    }
  }
  PROBE_MAX(31);
}

// ---- K2: the finish kernel ----------------------------------------------------
// Turns per-tile / per-chunk counts into global offsets and moves the staged
// runs to the ascending (index, value) lists; applies x -= g/n (engine.cpp:215)
// when n == 1 (the all-reduce is the identity). One extra CTA (the last block)
// reduces the per-tile counts and norm partials in a fixed order, publishes
// {k_i, ||e||^2} and, for n == 1, runs the control epilogue; it never waits for
// the copy CTAs because step t+1's plan goes to the other plan slot.
// Everything is latency-bound here, so every phase issues its loads wide and
// independent before using them.
constexpr int kSumUnroll = 12;
static_assert(kSumUnroll * kThreads == kBaseRoundTiles, "engine.cu sizes the range words by this");

// sum of cnt[lo, hi) (int32) by the whole CTA: kSumUnroll independent loads per
// thread per round (one round covers 3072 tiles)
__device__ __forceinline__ int64_t cta_sum_counts(const int32_t* __restrict__ cnt, int lo, int hi,
                                                  int64_t* red) {
  int64_t s = 0;
  for (int i = lo + (int)threadIdx.x; i < hi; i += kSumUnroll * kThreads) {
    int v[kSumUnroll];
#pragma unroll
    for (int k = 0; k < kSumUnroll; ++k) {
      const int ik = i + k * kThreads;
      v[k] = ik < hi ? __ldcg(&cnt[ik]) : 0;
    }
#pragma unroll
    for (int k = 0; k < kSumUnroll; ++k) s += v[k];
  }
  s = warp_sum(s);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  int64_t t = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) t += red[w];
  return t;
}

// Large vectors (more tiles than one round of cta_sum_counts covers): every
// copy CTA publishes, as {payload, epoch} words (no fences: an aligned 8-byte
// word is single-copy atomic), the selection count of its tile range and the
// two halves of an ||e||^2 partial over an equal slice of ALL tiles; a CTA's
// base is then the sum of the earlier CTAs' range words and the epilogue CTA
// totals G words, instead of rounds over every tile count before it. All
// finish CTAs are resident (<= 4 per SM by registers, the grid is 3 per SM + 1),
// so the polls cannot deadlock; the words are read only within this launch.
struct RangeWords {
  unsigned long long* sum;   // [G] selected in the CTA's tile range
  unsigned long long* nlo;   // [G] low / high 32 bits of the ||e||^2 partial
  unsigned long long* nhi;
};

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
  return *(volatile const unsigned long long*)p;
}

// sum of words w[0, m) carrying epoch ep (polled), by the whole CTA
__device__ int64_t cta_sum_words(const unsigned long long* w, int m, uint32_t ep, int64_t* red) {
  int64_t s = 0;
  for (int i = threadIdx.x; i < m; i += kThreads) {
    unsigned long long v;
    while ((uint32_t)((v = ld_volatile_u64(&w[i])) >> 32) != ep) __nanosleep(32);
    s += (uint32_t)v;
  }
  s = warp_sum(s);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  int64_t t = 0;
#pragma unroll
  for (int q = 0; q < kWarps; ++q) t += red[q];
  return t;
}

#ifndef EXD_COPY_UNROLL
#define EXD_COPY_UNROLL 8
#endif
#ifndef EXD_COPY_PER_SM
#define EXD_COPY_PER_SM 3  // measured: 2 -> 36.3 us, 3 -> 34.4 us, 4 -> 36.1 us per R18 step
#endif
constexpr int kCopyUnroll = EXD_COPY_UNROLL;  // staged entries in flight per thread

template <typename T, bool FUSED, bool BIG>
__global__ void __launch_bounds__(kThreads) finish_kernel(SelectArgs a, RunConst rc) {
  constexpr int CH = chunk_of<T>();
  constexpr int TILE = tile_of<T>();
  __shared__ int64_t s_red[kWarps];
  __shared__ double s_dred[kWarps];
  __shared__ int s_off[kThreads + 1];
  __shared__ int s_wtot[kWarps];

  Ctrl* ctrl = a.ctrl;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // P2P: let the union kernel launch early (it waits for our completion)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // block 0 is the epilogue CTA (dispatched first, so its control-block
  // prefetch overlaps the stream kernel's tail); blocks 1..G copy
  const int G = gridDim.x - 1, r = (int)blockIdx.x - 1;
  const int64_t n_g = rc.n_g;
  const Plan& plan = ctrl->plan[a.t & 1];
  const int64_t st = plan.st, end = plan.end;
  const int ft = (int)(st / TILE), lt = (int)((end - 1) / TILE);

  if (r < 0) {
    PROBE(0);
    // ---- epilogue CTA: prefetch the control block (n == 1), then the totals
    // in a fixed order, then the control epilogue
    __shared__ EpiShared esh;
    if (FUSED) epi_load(esh, ctrl);  // the stream kernel never writes the control block
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // one round of wide independent loads for both totals
    const int nt = (int)((n_g + TILE - 1) / TILE);
    double pn = 0.0;
    int64_t pk = 0;
    if (BIG) {  // large vector: the copy CTAs' published partials
      const RangeWords rw{a.range_words, a.range_words + kMaxCtas, a.range_words + 2 * kMaxCtas};
      const uint32_t ep = (uint32_t)(a.t + 1);
      // fixed order: thread i takes CTAs i, i + 256, ... in turn
      for (int q = tid; q < G; q += kThreads) {
        unsigned long long s_, lo, hi;
        while ((uint32_t)((s_ = ld_volatile_u64(&rw.sum[q])) >> 32) != ep) __nanosleep(32);
        while ((uint32_t)((lo = ld_volatile_u64(&rw.nlo[q])) >> 32) != ep) __nanosleep(32);
        while ((uint32_t)((hi = ld_volatile_u64(&rw.nhi[q])) >> 32) != ep) __nanosleep(32);
        pk += (uint32_t)s_;
        pn += __longlong_as_double((long long)((hi << 32) | (lo & 0xffffffffull)));
      }
    }
    for (int i = tid; i < (BIG ? 0 : nt); i += kSumUnroll * kThreads) {
      double v[kSumUnroll];
      int c[kSumUnroll];
#pragma unroll
      for (int k = 0; k < kSumUnroll; ++k) {
        const int ik = i + k * kThreads;
        v[k] = ik < nt ? __ldcg(&a.tile_norm[ik]) : 0.0;
        c[k] = (ik < nt && ik >= ft && ik <= lt) ? __ldcg(&a.tile_count[ik]) : 0;
      }
#pragma unroll
      for (int k = 0; k < kSumUnroll; ++k) {
        pn += v[k];
        pk += c[k];
      }
    }
    PROBE(1);
    pn = warp_sum(pn);
    pk = warp_sum(pk);
    if (lane == 0) {
      s_dred[warp] = pn;
      s_red[warp] = pk;
    }
    __syncthreads();
    if (tid == 0) {
      double n2 = 0.0;
      int64_t kt = 0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        n2 += s_dred[w];
        kt += s_red[w];
      }
      a.cnt_out->k = kt;
      a.cnt_out->norm2 = n2;
      a.cnt_out->capped = 0;
      if (FUSED) {
        esh.c.k_local = kt;
        esh.c.norm2 = n2;
        esh.k_rank[0] = kt;
        esh.norm2[0] = n2;
        esh.capped[0] = 0;
      } else {
        ctrl->k_local = kt;
        ctrl->norm2 = n2;
      }
    }
    if (FUSED) {
      __syncthreads();
      PROBE(2);
      epi_run_store(esh, ctrl, rc, a.rec);
    }
    PROBE(3);
    PROBE_MAX(30);
    return;
  }

  // ---- copy CTAs: a static contiguous range of the partition's tiles
  if (r == 0) PROBE(8);
  CPROBE(0, r);
  const int ntp = lt - ft + 1;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the stream kernel's counts and runs
  const int t0 = ft + (int)(((int64_t)ntp * r) / G);
  const int t1 = ft + (int)(((int64_t)ntp * (r + 1)) / G);
  const int nch = (t1 - t0) * kWarps;
  T* __restrict__ val = static_cast<T*>(a.val);
  T* __restrict__ x = static_cast<T*>(a.x);
  int32_t* __restrict__ idx = a.idx;
  using P = typename Pair<T>::P;
  const P* __restrict__ sp = static_cast<const P*>(a.stage);
  // the chunk counts do not depend on the base: load them in the same round trip
  int cnt = tid < nch ? __ldcg(&a.chunk_count[t0 * kWarps + tid]) : 0;
  int64_t base;
  if (BIG) {
    // own range count and the ||e||^2 partial of an equal slice of all tiles,
    // published; the base from the earlier CTAs' words
    const int nt = (int)((n_g + TILE - 1) / TILE);
    const int n0 = (int)(((int64_t)nt * r) / G), n1 = (int)(((int64_t)nt * (r + 1)) / G);
    double pn = 0.0;
    for (int i = n0 + tid; i < n1; i += kThreads) pn += __ldcg(&a.tile_norm[i]);
    const int64_t mine = cta_sum_counts(a.tile_count, t0, t1, s_red);
    pn = warp_sum(pn);
    if (lane == 0) s_dred[warp] = pn;
    __syncthreads();
    const uint32_t ep = (uint32_t)(a.t + 1);
    if (tid == 0) {
      double n2 = 0.0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) n2 += s_dred[w];
      const unsigned long long eph = (unsigned long long)ep << 32;
      const unsigned long long nb = (unsigned long long)__double_as_longlong(n2);
      st_relaxed_sys_u64(&a.range_words[r], eph | (uint32_t)mine);
      st_relaxed_sys_u64(&a.range_words[kMaxCtas + r], eph | (nb & 0xffffffffull));
      st_relaxed_sys_u64(&a.range_words[2 * kMaxCtas + r], eph | (nb >> 32));
    }
    base = cta_sum_words(a.range_words, r, ep, s_red);
  } else {
    base = cta_sum_counts(a.tile_count, ft, t0, s_red);
  }
  if (r == 0) PROBE(9);
  if (r == G - 1) PROBE(10);
  CPROBE(1, r);

  int64_t running = base;
  for (int cb = 0; cb < nch; cb += kThreads) {
    const int nb = nch - cb < kThreads ? nch - cb : kThreads;
    // large vectors: the next batch's counts, in flight during this batch's copy
    const int cn = cb + kThreads + tid;
    const int cnt_next = BIG && cn < nch ? __ldcg(&a.chunk_count[t0 * kWarps + cn]) : 0;
    if (!BIG && cb) cnt = tid < nb ? __ldcg(&a.chunk_count[t0 * kWarps + cb + tid]) : 0;
    // block exclusive scan of the chunk counts
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_wtot[warp] = incl;
    __syncthreads();
    int wpre = 0, btot = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      wpre += w < warp ? s_wtot[w] : 0;
      btot += s_wtot[w];
    }
    s_off[tid] = wpre + incl - cnt;
    __syncthreads();
    // flattened copy, kCopyUnroll entries per thread in flight: entry i of the
    // batch lives in chunk k with s_off[k] <= i < s_off[k + 1]
    const int64_t cbase = (int64_t)(t0 * kWarps + cb);  // global chunk of s_off[0]
    for (int i0 = tid; i0 < btot; i0 += kCopyUnroll * kThreads) {
      int32_t jj[kCopyUnroll];
      T vv[kCopyUnroll];
      T xx[kCopyUnroll];
#pragma unroll
      for (int q = 0; q < kCopyUnroll; ++q) {
        const int i = i0 + q * kThreads;
        if (i < btot) {
          int lo = 0, hi = nb;  // last k with s_off[k] <= i
          while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (s_off[mid] <= i) lo = mid; else hi = mid;
          }
          const int64_t cst = (cbase + lo) * CH;  // the run starts at max(chunk, partition start)
          const int64_t src = (cst > st ? cst : st) + (i - s_off[lo]);
          const typename Pair<T>::P pr = __ldcg(&sp[src]);
          jj[q] = (int32_t)Pair<T>::idx(pr);
          vv[q] = Pair<T>::val(pr);
        }
      }
      if (FUSED) {
#pragma unroll
        for (int q = 0; q < kCopyUnroll; ++q)
          if (i0 + q * kThreads < btot) xx[q] = x[jj[q]];
      }
#pragma unroll
      for (int q = 0; q < kCopyUnroll; ++q) {
        const int i = i0 + q * kThreads;
        if (i < btot) {
          idx[running + i] = jj[q];
          val[running + i] = vv[q];
          // P2P: push the list into every peer's inbox (posted NVLink stores)
          for (int pr = 0; pr < a.npush; ++pr) a.push_idx[pr][running + i] = jj[q];
          if (FUSED) x[jj[q]] = apply_update<T>(xx[q], vv[q], rc.n);
        }
      }
    }
    running += btot;
    if (BIG) cnt = cnt_next;
    __syncthreads();
  }
  if (r == 0) PROBE(11);
  if (r == G - 1) PROBE(12);
  CPROBE(2, r);
  CPROBE_V(3, r, (unsigned long long)(running - base));
  PROBE_MAX(30);
}

template <typename T, bool UNIT, bool PUSH>
void launch_stream_p(int mode, const SelectArgs& a, const RunConst& rc, cudaStream_t s) {
  const dim3 grid(a.num_tiles), block(kThreads);
  if (mode == kFused) stream_kernel<T, kFused, UNIT, PUSH><<<grid, block, 0, s>>>(a, rc);
  else if (mode == kAccumulate) stream_kernel<T, kAccumulate, UNIT, false><<<grid, block, 0, s>>>(a, rc);
  else stream_kernel<T, kSelectOnly, UNIT, PUSH><<<grid, block, 0, s>>>(a, rc);
}

template <typename T, bool UNIT>
void launch_stream_u(int mode, const SelectArgs& a, const RunConst& rc, cudaStream_t s) {
  if (a.k1_npush > 0) launch_stream_p<T, UNIT, true>(mode, a, rc, s);
  else launch_stream_p<T, UNIT, false>(mode, a, rc, s);
}

template <typename T>
cudaError_t launch_stream_t(int mode, const SelectArgs& a, const RunConst& rc, cudaStream_t s) {
  // eta == 1 (the reference default) takes the plain-add path; for double
  // eta * g with eta == 1 is exact so one instantiation serves both
  if (rc.eta == 1.0 || sizeof(T) == 8) launch_stream_u<T, true>(mode, a, rc, s);
  else launch_stream_u<T, false>(mode, a, rc, s);
  return cudaGetLastError();
}

constexpr int kMaxDevices = 64;

template <typename T>
cudaError_t launch_finish_t(const SelectArgs& a, const RunConst& rc, cudaStream_t s) {
  // copy-CTA cap per device (engines of one process may sit on different GPUs)
  static std::atomic<int> caps[kMaxDevices];
  int dev = 0;
  cudaGetDevice(&dev);
  int cap = dev < kMaxDevices ? caps[dev].load(std::memory_order_relaxed) : 0;
  if (cap == 0) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cap = sms * EXD_COPY_PER_SM > kMaxCtas ? kMaxCtas : sms * EXD_COPY_PER_SM;
    if (dev < kMaxDevices) caps[dev].store(cap, std::memory_order_relaxed);
  }
  // the partition's tile count is device-resident; size for the whole vector,
  // plus one epilogue CTA
  const int64_t nt = num_tiles(rc.n_g, rc.dtype);
  int grid = nt < cap ? (int)nt : cap;
  if (grid < 1) grid = 1;
  // programmatic stream serialization: overlaps this launch with the tail of
  // the stream kernel (see griddepcontrol in both kernels)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid + 1);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const bool big = a.range_words != nullptr;
  if (rc.fused)
    return big ? cudaLaunchKernelEx(&cfg, finish_kernel<T, true, true>, a, rc)
               : cudaLaunchKernelEx(&cfg, finish_kernel<T, true, false>, a, rc);
  return big ? cudaLaunchKernelEx(&cfg, finish_kernel<T, false, true>, a, rc)
             : cudaLaunchKernelEx(&cfg, finish_kernel<T, false, false>, a, rc);
}

// ---- K4+K5: union + contributions + clear -----------------------------------
// collectives.cpp:47-55 (union; here a concatenation in partition order since
// partitions are disjoint and each list ascends), engine.cpp:310-317
// (c_r[pos] = acc_r[idx_global[pos]]) and selector.cpp:63-65 (clear, moved
// before the sum; equivalent because contributions are already taken).
template <typename T>
__global__ void __launch_bounds__(256) union_kernel(UnionArgs a, RunConst rc) {
  __shared__ int64_t s_off[EXD_MAX_WORKERS + 1];
  __shared__ int32_t s_rank[EXD_MAX_WORKERS];
  __shared__ int64_t s_mt;
  const int n = rc.n;
  if (threadIdx.x == 0) {
    const int64_t t = a.ctrl->t;  // step still running: finalize has not advanced t
    const int64_t tm = mod_floor(t, n);
    int64_t off = 0, mt = 0;
    for (int p = 0; p < n; ++p) {
      const int r = (int)mod_floor(p - tm, n);
      s_rank[p] = r;
      s_off[p] = off;
      off += a.counts[r].k;
    }
    for (int r = 0; r < n; ++r) mt = a.counts[r].k > mt ? a.counts[r].k : mt;
    s_off[n] = off;
    s_mt = mt;
  }
  __syncthreads();
  const int64_t kp = s_off[n];
  T* e = static_cast<T*>(a.e);
  T* c = static_cast<T*>(a.contrib);
  const T* own = static_cast<const T*>(a.own_val);
  for (int64_t pos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pos < kp;
       pos += (int64_t)gridDim.x * blockDim.x) {
    int p = 0;
    while (p + 1 < n && s_off[p + 1] <= pos) ++p;
    const int r = s_rank[p];
    const int64_t local = pos - s_off[p];
    const int32_t j = a.lists ? a.lists[r][local] : a.padded[(int64_t)r * s_mt + local];
    a.idx_global[pos] = j;
    if (r == rc.rank) {
      c[pos] = own[local];  // own residual was cleared by the fused kernel
    } else {
      c[pos] = e[j];
      e[j] = T(0);
    }
  }
}

// ---- K6 (in-process): rank-order sum, collectives.cpp:59-70 ----------------
template <typename T>
__global__ void __launch_bounds__(256) allreduce_local_kernel(const void* const* contribs, void* sum,
                                                              const CountRec* counts, RunConst rc) {
  int64_t kp = 0;
  for (int r = 0; r < rc.n; ++r) kp += counts[r].k;
  T* out = static_cast<T*>(sum);
  for (int64_t pos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pos < kp;
       pos += (int64_t)gridDim.x * blockDim.x) {
    T s = static_cast<const T*>(contribs[0])[pos];
    for (int r = 1; r < rc.n; ++r) s += static_cast<const T*>(contribs[r])[pos];
    out[pos] = s;
  }
}

// ---- K7+K9: x scatter + control epilogue, engine.cpp:206-219 -----------------
template <typename T>
__global__ void __launch_bounds__(256) finalize_kernel(FinalizeArgs a, RunConst rc) {
  int64_t kp = 0;
  for (int r = 0; r < rc.n; ++r) kp += a.counts[r].k;
  T* x = static_cast<T*>(a.x);
  const T* g = static_cast<const T*>(a.sum);
  for (int64_t pos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pos < kp;
       pos += (int64_t)gridDim.x * blockDim.x) {
    const int32_t j = a.idx_global[pos];
    x[j] = apply_update<T>(x[j], g[pos], rc.n);
  }
  if (blockIdx.x == 0) {
    __syncthreads();
    control_epilogue_cta(a.ctrl, a.counts, rc, a.rec);
  }
}

// ---- f1: NVLink peer-memory sync -------------------------
// Replaces the NCCL chain (count all-gather -> host wait -> padded index
// all-gather -> all-reduce) with kernels that talk over NVLink directly, with
// no host in the loop and no padding:
//   finish      (already running) also PUSHES this rank's ascending index list
//               into its slot of every peer's inbox (posted NVLink stores).
//   p2p_sync    publishes {k_i, ||e||^2} + an epoch into every peer's inbox,
//               waits on its OWN inbox (local polling), builds the union in
//               partition order from the (now local) lists, gathers this rank's
//               contributions, clears e at the union; then (in-kernel arrive
//               counter instead of a kernel boundary) publishes "contributions
//               ready", waits, sums the contributions in RANK ORDER straight
//               from the peers' buffers (bit-identical to all_reduce_sum,
//               collectives.cpp:59-70, for every n), x -= g/n, and runs the
//               control epilogue on a spare block.
// Buffer reuse is safe without extra handshakes: a rank overwrites its list
// slot / count in a peer's inbox only in step t+1, after its own p2p_sync(t)
// saw that peer's contrib epoch t+1 (published when the peer had finished
// phase A of p2p_sync(t)); contributions are double buffered by step parity.
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long gtime_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void st_relaxed_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys_i64(int64_t* p, int64_t v) {
  asm volatile("st.relaxed.sys.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys_f64(double* p, double v) {
  asm volatile("st.relaxed.sys.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Block 0 polls its LOCAL inbox (the senders pushed their epochs there), one
// system-scope acquire fence once everyone is in, then opens a local gate word
// for the other blocks. Gives up after 20 s (sets `err`) so a dead peer cannot
// hang the GPU. Call from thread 0; returns false on timeout.
__device__ bool poll_inbox_open_gate(const PeerFlags* inbox, int n, bool contrib,
                                     unsigned long long epoch, unsigned long long* gate,
                                     unsigned int* err) {
  const unsigned long long t0 = gtime_ns();
  for (int r = 0; r < n; ++r) {
    const unsigned long long* w = contrib ? &inbox[r].contrib_epoch : &inbox[r].count_epoch;
    unsigned spins = 0;
    while (ld_relaxed_sys(w) < epoch) {
      if ((++spins & 255u) == 0 && gtime_ns() - t0 > 20000000000ull) {
        atomicExch(err, 1u);
        st_release_gpu(gate, ~0ull);  // release the other blocks, they see err
        return false;
      }
      __nanosleep(20);
    }
  }
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  st_release_gpu(gate, epoch);
  return true;
}

__device__ bool wait_gate(const unsigned long long* gate, unsigned long long epoch,
                          unsigned int* err) {
  const unsigned long long t0 = gtime_ns();
  unsigned spins = 0;
  unsigned long long gv;
  while ((gv = ld_acquire_gpu(gate)) < epoch) {
    if ((++spins & 255u) == 0 && gtime_ns() - t0 > 21000000000ull) {
      atomicExch(err, 1u);
      return false;
    }
    __nanosleep(20);
  }
  return gv != ~0ull && *(volatile unsigned int*)err == 0;
}

__device__ bool wait_inbox(const PeerFlags* inbox, int n, bool contrib, unsigned long long epoch,
                           unsigned long long* gate, unsigned int* err) {
  if (blockIdx.x == 0) return poll_inbox_open_gate(inbox, n, contrib, epoch, gate, err);
  return wait_gate(gate, epoch, err);
}

// One kernel for both exchange rounds: phase A builds the union and this
// rank's contributions, an in-kernel arrive counter replaces the kernel
// boundary, phase B sums the peers' contributions. Every CTA is resident (the
// grid is 2 per SM + 1 and the previous kernel retires), so the counter cannot
// deadlock. The last block runs the control epilogue as soon as the counts are
// in (it needs nothing else).
template <typename T>
__global__ void __launch_bounds__(256) p2p_sync_kernel(P2PArgs a, RunConst rc) {
  __shared__ int64_t s_off[EXD_MAX_WORKERS + 1];
  __shared__ int32_t s_rank[EXD_MAX_WORKERS];
  __shared__ bool s_ok;
  const int n = rc.n, tid = threadIdx.x;
  const int G = gridDim.x - 1;  // work blocks; block G: control epilogue
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the finish/cap kernel's list pushes
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (blockIdx.x == 0) PROBE(20);
  if (blockIdx.x == 0 && tid < n) {
    // announce {k_i, ||e||^2}: the pushed list is complete (previous kernel);
    // one system fence orders the payload before the epoch (a release store
    // would add a second one: profiles/p2p_latency_r01.txt)
    PeerFlags* slot = a.peer_slot[tid];
    st_relaxed_sys_i64(&slot->k, a.own_cnt->k);
    st_relaxed_sys_f64(&slot->norm2, a.own_cnt->norm2);
    st_relaxed_sys_i64(&slot->capped, a.own_cnt->capped);
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    st_relaxed_sys(&slot->count_epoch, a.epoch);
  }
  if (tid == 0) s_ok = wait_inbox(a.inbox, n, false, a.epoch, &a.gate[0], a.err);
  __syncthreads();
  if (blockIdx.x == 0) PROBE(21);
  if (!s_ok) return;
  if ((int)blockIdx.x == G) {
    // the counts of every rank are in the inbox (block 0 copies them to
    // counts_all concurrently, so read the inbox itself)
    __shared__ EpiShared esh;
    epi_load(esh, a.ctrl);
    for (int r = tid; r < n; r += blockDim.x) {
      esh.k_rank[r] = __ldcg(&a.inbox[r].k);
      esh.norm2[r] = __ldcg(&a.inbox[r].norm2);
      esh.capped[r] = __ldcg(&a.inbox[r].capped);
    }
    __syncthreads();
    // the counts are read: join the arrive counter, so block 0 publishes
    // "contributions ready" (which lets the peers overwrite these inbox words
    // in step t+1) only after this block is done with them
    if (tid == 0) {
      __threadfence();
      atomicAdd(&a.gate[2], 1ull);
    }
    epi_run_store(esh, a.ctrl, rc, a.rec);
    PROBE(24);
    return;
  }
  if (tid == 0) {
    // the step from the launch argument, not a.ctrl->t: block G's epilogue
    // rewrites the control block (t + 1) concurrently
    const int64_t tm = mod_floor((int64_t)a.epoch - 1, n);
    int64_t off = 0;
    for (int p = 0; p < n; ++p) {
      const int r = (int)mod_floor(p - tm, n);
      s_rank[p] = r;
      s_off[p] = off;
      off += __ldcg(&a.inbox[r].k);
    }
    s_off[n] = off;
  }
  if (blockIdx.x == 0 && tid < n) {
    a.counts_all[tid].k = __ldcg(&a.inbox[tid].k);
    a.counts_all[tid].norm2 = __ldcg(&a.inbox[tid].norm2);
    a.counts_all[tid].capped = __ldcg(&a.inbox[tid].capped);
  }
  __syncthreads();
  const int64_t kp = s_off[n];
  {
    // ---- phase A: union in partition order, own contributions, clear e
    T* e = static_cast<T*>(a.e);
    T* c = static_cast<T*>(a.contrib[a.me]);
    const T* own = static_cast<const T*>(a.own_val);
    const T* xx = static_cast<const T*>(a.x);
    const int64_t stride = (int64_t)G * blockDim.x;
    // 4 entries per thread in flight: list reads, then residual reads, then writes
    for (int64_t p0 = (int64_t)blockIdx.x * blockDim.x + tid; p0 < kp; p0 += 4 * stride) {
      int32_t j[4];
      int r4[4];
      int64_t loc[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t pos = p0 + q * stride;
        r4[q] = -1;
        if (pos < kp) {
          int p = 0;
          while (p + 1 < n && s_off[p + 1] <= pos) ++p;
          r4[q] = s_rank[p];
          loc[q] = pos - s_off[p];
          j[q] = __ldcg(&a.lists[r4[q]][loc[q]]);  // local: own list or pushed inbox slot
        }
      }
      T v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (r4[q] < 0) continue;
        v[q] = r4[q] == a.me ? own[loc[q]] : e[j[q]];  // own residual already cleared
        // phase B read-modify-writes x[j]: pull the line into L2 now
        asm volatile("prefetch.global.L2 [%0];" ::"l"(xx + j[q]));
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (r4[q] < 0) continue;
        const int64_t pos = p0 + q * stride;
        a.idx_global[pos] = j[q];
        c[pos] = v[q];
        if (r4[q] != a.me) e[j[q]] = T(0);
      }
    }
  }
  // ---- every work block's contributions are written: block 0 announces
  // "contributions ready" (one system fence), waits for the peers', opens gate 1
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    atomicAdd(&a.gate[2], 1ull);
  }
  if (blockIdx.x == 0) {
    if (tid == 0) {
      // G work blocks + the epilogue block arrive once per step
      const unsigned long long want = a.epoch * (unsigned long long)(G + 1);
      const unsigned long long t0 = gtime_ns();
      unsigned spins = 0;
      while (*(volatile unsigned long long*)&a.gate[2] < want) {
        if ((++spins & 255u) == 0 &&
            (gtime_ns() - t0 > 20000000000ull || *(volatile unsigned int*)a.err)) {
          atomicExch(a.err, 1u);  // the engine is unusable after this (sync reports it)
          break;
        }
        __nanosleep(32);
      }
      __threadfence();
    }
    __syncthreads();
    PROBE(22);
    if (tid < n) {
      asm volatile("fence.acq_rel.sys;" ::: "memory");
      st_relaxed_sys(&a.peer_slot[tid]->contrib_epoch, a.epoch);
    }
  }
  if (tid == 0) s_ok = wait_inbox(a.inbox, n, true, a.epoch, &a.gate[1], a.err);
  __syncthreads();
  if (blockIdx.x == 0) PROBE(23);
  if (!s_ok) return;
  {
    // ---- phase B: rank-order sum straight from the peers' buffers, x -= g/n
    T* x = static_cast<T*>(a.x);
    T* g = static_cast<T*>(a.sum);
    const int64_t stride = (int64_t)G * blockDim.x;
    const int nn = n < 8 ? n : 8;
    // 2 entries per thread in flight: every peer's contribution for both, then x
    for (int64_t p0 = (int64_t)blockIdx.x * blockDim.x + tid; p0 < kp; p0 += 2 * stride) {
      T v[2][8];
      int32_t j[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int64_t pos = p0 + q * stride;
        if (pos < kp) {
#pragma unroll
          for (int r = 0; r < 8; ++r)
            if (r < nn) v[q][r] = __ldcg(&static_cast<const T*>(a.contrib[r])[pos]);
          j[q] = a.idx_global[pos];
        }
      }
      T xv[2];
#pragma unroll
      for (int q = 0; q < 2; ++q)
        if (p0 + q * stride < kp) xv[q] = x[j[q]];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int64_t pos = p0 + q * stride;
        if (pos >= kp) continue;
        T sv = v[q][0];  // rank order, as all_reduce_sum (collectives.cpp:62-68)
#pragma unroll
        for (int r = 1; r < 8; ++r)
          if (r < nn) sv += v[q][r];
        for (int r = 8; r < n; ++r) sv += __ldcg(&static_cast<const T*>(a.contrib[r])[pos]);
        g[pos] = sv;
        x[j[q]] = apply_update<T>(xv[q], sv, n);
      }
    }
  }
  if (blockIdx.x == 0) PROBE(25);
}

// ---- f1, push-reduce: the whole sync in the kernel after the stream ---------
// One rank per GPU, no density cap. Replaces finish + p2p_sync with ONE kernel.
// Everything crosses NVLink as posted stores of {payload, epoch} words (the
// low-latency protocol: an aligned 8-byte word is single-copy atomic, so the
// word is its own flag): no remote reads, no fences and no handshake on the
// critical path.
//   K1  (stream_kernel<..., PUSH>) besides staging its (index, value) pairs
//       locally, stores each warp's run of staged indices and its tile's chunk
//       and tile counts into its slots of every peer's inbox as words tagged
//       with the step.
//   A+B every work block owns a contiguous tile range of ONE partition (the
//       partition table is the replicated plan; allocator.cpp:92-99). Its union
//       positions (collectives.cpp:47-55: the union is the concatenation of the
//       ascending lists in partition order) come from the tile counts of every
//       tile before its range and from its chunk counts, polled as words. Per
//       entry, one thread: takes the index from the holder's pushed run (own
//       staged pairs for its own partition), gathers its own contribution
//       acc[j] (engine.cpp:310-317), stores it as a word into every peer's
//       inbox, clears e[j] (selector.cpp:63-65), then polls the peers' words
//       for the same position, sums the n contributions in rank order
//       (all_reduce_sum, collectives.cpp:62-68: bit-identical for every n) and
//       applies x -= g/n (engine.cpp:215).
//   block 0 totals this rank's {k_i, ||e||^2}, exchanges them with a flag (off
//       the critical path: only the control epilogue needs every rank's
//       counts) and runs the epilogue.
// Reuse, by construction: every inbox slot (pushed runs and counts, flags,
// contribution words) is double-buffered by step parity. Rank q rewrites
// parity slot (t & 1) of r's inbox only in step t+2, after its step t+1 polled
// every contribution word of r for step t+1, which r's blocks store only
// after r's kernels of step t completed. A stale word carries an older epoch
// and is polled again.

// {payload, epoch} words of one contribution: 1 for fp32, 2 for fp64
template <typename T> struct LL;
template <> struct LL<float> {
  static constexpr int W = 1;
  __device__ static void put(unsigned long long* p, float v, uint32_t ep) {
    st_relaxed_sys_u64(p, ((unsigned long long)ep << 32) | __float_as_uint(v));
  }
  __device__ static bool get(const unsigned long long* p, uint32_t ep, float& v) {
    const unsigned long long w = ld_relaxed_sys_u64(p);
    v = __uint_as_float((uint32_t)w);
    return (uint32_t)(w >> 32) == ep;
  }
};
template <> struct LL<double> {
  static constexpr int W = 2;
  __device__ static void put(unsigned long long* p, double v, uint32_t ep) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    st_relaxed_sys_v2u64(p, ((unsigned long long)ep << 32) | (b & 0xffffffffull),
                         ((unsigned long long)ep << 32) | (b >> 32));
  }
  __device__ static bool get(const unsigned long long* p, uint32_t ep, double& v) {
    const unsigned long long lo = ld_relaxed_sys_u64(p), hi = ld_relaxed_sys_u64(p + 1);
    v = __longlong_as_double((long long)(((hi & 0xffffffffull) << 32) | (lo & 0xffffffffull)));
    return (uint32_t)(lo >> 32) == ep && (uint32_t)(hi >> 32) == ep;
  }
};

// Poll one {count, epoch} word until it carries `ep`; gives up after 20 s
// (sets *err, returns 0) so a dead peer cannot hang the GPU.
__device__ __noinline__ uint32_t poll_word(const unsigned long long* p, uint32_t ep, unsigned int* err) {
  const unsigned long long t0 = gtime_ns();
  unsigned spins = 0;
  unsigned long long w;
  while ((uint32_t)((w = ld_relaxed_sys_u64(p)) >> 32) != ep) {
    if ((++spins & 255u) == 0 &&
        (gtime_ns() - t0 > 20000000000ull || *(volatile unsigned int*)err)) {
      atomicExch(err, 1u);
      return 0;
    }
    __nanosleep(20);
  }
  return (uint32_t)w;
}

// relaxed system-scope load of one value (peer memory, after an acquire fence)
template <typename T> __device__ __forceinline__ T ld_relaxed_sys_t(const T* p);
template <> __device__ __forceinline__ float ld_relaxed_sys_t<float>(const float* p) {
  float v;
  asm volatile("ld.relaxed.sys.global.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
  return v;
}
template <> __device__ __forceinline__ double ld_relaxed_sys_t<double>(const double* p) {
  double v;
  asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}

// Poll one {value, epoch} contribution / sum until it carries `ep`; gives up
// after 20 s (sets *err) so a dead peer cannot hang the GPU.
template <typename T>
__device__ __forceinline__ T poll_ll(const unsigned long long* w, uint32_t ep, unsigned int* err) {
  T v;
  if (LL<T>::get(w, ep, v)) return v;
  const unsigned long long t0 = gtime_ns();
  unsigned spins = 0;
  while (!LL<T>::get(w, ep, v)) {
    if ((++spins & 255u) == 0 &&
        (gtime_ns() - t0 > 20000000000ull || *(volatile unsigned int*)err)) {
      atomicExch(err, 1u);
      break;
    }
    __nanosleep(20);
  }
  return v;
}

constexpr int kXUnroll = 4;   // union entries per thread in flight
constexpr int kX2Unroll = 8;  // pass-2 positions per thread in flight (TWO)
constexpr int kXPeers = 4;    // peer words per entry polled together

// TWO (large k'): the work loop runs in two passes per block, so no NVLink
// round trip sits inside an iteration. Pass 1 streams the block's entries:
// index words, own contribution (also into this rank's own inbox slot), the
// contributions out, union entry, residual clear. Pass 2 streams the block's
// contiguous union positions: the n contribution words (they were posted
// during the peers' pass 1, so the polls rarely wait) or the holder's sum,
// the rank-order sum and x -= g/n. Small k' keeps the one-pass loop, which
// needs one iteration per block and overlaps the lookups with the stream
// kernel's drain.
template <typename T, bool BIG, bool TWO>
// 3 blocks per SM by registers: the 2-per-SM grid + block 0 is always resident
__global__ void __launch_bounds__(kThreads, 3) exchange_kernel(ExchangeArgs a, RunConst rc) {
  using P = typename Pair<T>::P;
  constexpr int CH = chunk_of<T>();
  constexpr int TILE = tile_of<T>();
  constexpr int W = LL<T>::W;
  __shared__ int64_t s_red[kWarps];
  __shared__ double s_dred[kWarps];
  __shared__ int s_off[kThreads + 1];
  __shared__ int s_wtot[kWarps];
  __shared__ int32_t s_prank[EXD_MAX_WORKERS];      // rank holding partition p
  __shared__ int32_t s_ft[EXD_MAX_WORKERS];         // first tile of partition p
  __shared__ int32_t s_tcum[EXD_MAX_WORKERS + 1];   // tiles of partitions < p
  __shared__ int64_t s_pst[EXD_MAX_WORKERS];        // first element of partition p
  __shared__ int32_t s_bcum[EXD_MAX_WORKERS + 1];   // work blocks of partitions < p
  __shared__ bool s_ok;
  const SelectArgs& sa = a.s;
  Ctrl* ctrl = sa.ctrl;
  const int n = rc.n, me = a.me;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x - 1, r = (int)blockIdx.x - 1;
  const int par = (int)(sa.t & 1);
  const uint32_t ep = (uint32_t)a.epoch;
  const Plan& plan = ctrl->plan[par];  // the epilogue writes only the other slot

  if (tid == 0) {
    // partition table from the replicated plan (allocate_partition,
    // allocator.cpp:92-99: partition p is held by rank (p - t) mod n; the last
    // one ends at n_g)
    const int tm = (int)mod_floor(sa.t, n);
    const exd_topology& tp = plan.topo;
    int32_t tc = 0;
    for (int p = 0; p < n; ++p) {
      const int rk = p - tm < 0 ? p - tm + n : p - tm;
      const int64_t pst = tp.blk_pos[p] * tp.sz_blk;
      const int64_t pend = p == n - 1 ? rc.n_g : (tp.blk_pos[p] + tp.blk_part[p]) * tp.sz_blk;
      s_prank[p] = rk;
      s_ft[p] = (int32_t)(pst / TILE);
      s_pst[p] = pst;
      s_tcum[p] = tc;
      tc += pend > pst ? (int32_t)((pend - 1) / TILE - pst / TILE + 1) : 0;
    }
    s_tcum[n] = tc;
    // work blocks per partition, by tiles, at least one each (G >= n)
    for (int p = 0; p <= n; ++p)
      s_bcum[p] = p + (int32_t)(((int64_t)(G - n) * s_tcum[p]) / (tc > 0 ? tc : 1));
  }
  __syncthreads();  // the table is read by every block (block 0: BIG totals)
  if (r < 0) {
    // ---- block 0: totals, count exchange, control epilogue
    __shared__ EpiShared esh;
    __shared__ int64_t s_k;
    __shared__ double s_n2;
    const PeerFlags* inbox = a.inbox + par * n;
    const int64_t st = plan.st, end = plan.end;
    const int ft = (int)(st / TILE), lt = (int)((end - 1) / TILE);
    epi_load(esh, ctrl);  // the stream kernel never writes the control block
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (tid == 0) PROBE(0);
    const int nt = (int)((rc.n_g + TILE - 1) / TILE);
    double pn = 0.0;
    int64_t pk = 0;
    if (BIG) {
      // large vectors: own k_i from the range words of the blocks working on
      // this rank's partition; ||e||^2 from the norm partials every work block
      // publishes at its end (fixed order: thread i takes blocks i, i + 256, ...)
      const int po = (int)mod_floor(sa.t + me, n);  // allocate_partition: (t % n + rank) % n
      for (int q = s_bcum[po] + tid; q < s_bcum[po + 1]; q += kThreads)
        pk += poll_word(&a.xrange_words[q], ep, a.err);
      for (int q = tid; q < G; q += kThreads) {
        const unsigned long long lo = poll_word(&a.xrange_words[kMaxCtas + q], ep, a.err);
        const unsigned long long hi = poll_word(&a.xrange_words[2 * kMaxCtas + q], ep, a.err);
        pn += __longlong_as_double((long long)((hi << 32) | lo));
      }
    }
    for (int i = tid; i < (BIG ? 0 : nt); i += kSumUnroll * kThreads) {
      double v[kSumUnroll];
      int c[kSumUnroll];
#pragma unroll
      for (int k = 0; k < kSumUnroll; ++k) {
        const int ik = i + k * kThreads;
        v[k] = ik < nt ? __ldcg(&sa.tile_norm[ik]) : 0.0;
        c[k] = (ik < nt && ik >= ft && ik <= lt) ? __ldcg(&sa.tile_count[ik]) : 0;
      }
#pragma unroll
      for (int k = 0; k < kSumUnroll; ++k) {
        pn += v[k];
        pk += c[k];
      }
    }
    pn = warp_sum(pn);
    pk = warp_sum(pk);
    if (lane == 0) {
      s_dred[warp] = pn;
      s_red[warp] = pk;
    }
    __syncthreads();
    if (tid == 0) {
      double n2 = 0.0;
      int64_t kt = 0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        n2 += s_dred[w];
        kt += s_red[w];
      }
      s_k = kt;
      s_n2 = n2;
      sa.cnt_out->k = kt;
      sa.cnt_out->norm2 = n2;
      sa.cnt_out->capped = 0;
    }
    __syncthreads();
    if (tid < n) {  // {k, epoch} and the two halves of ||e||^2 as words: no fence
      PeerFlags* slot = a.peer_slot[tid] + par * n;
      const unsigned long long eph = (unsigned long long)ep << 32;
      const unsigned long long nb = (unsigned long long)__double_as_longlong(s_n2);
      st_relaxed_sys_u64(&slot->ll[0], eph | (uint32_t)s_k);
      st_relaxed_sys_v2u64(&slot->ll[1], eph | (nb & 0xffffffffull), eph | (nb >> 32));
    }
    if (tid == 0) PROBE(1);
    for (int q = tid; q < n; q += kThreads) {
      const int64_t k = poll_word(&inbox[q].ll[0], ep, a.err);
      const unsigned long long lo = poll_word(&inbox[q].ll[1], ep, a.err);
      const unsigned long long hi = poll_word(&inbox[q].ll[2], ep, a.err);
      const double n2 = __longlong_as_double((long long)((hi << 32) | lo));
      esh.k_rank[q] = k;
      esh.norm2[q] = n2;
      esh.capped[q] = 0;
      a.counts_all[q].k = k;
      a.counts_all[q].norm2 = n2;
      a.counts_all[q].capped = 0;
    }
    __syncthreads();
    if (tid == 0) PROBE(2);
    epi_run_store(esh, ctrl, rc, a.rec);
    if (tid == 0) PROBE(4);
    return;
  }

  // ---- work blocks
  // No griddepcontrol.wait yet: the partition's runs and counts arrive as words
  // (this rank's own too), so the lookups below overlap this rank's stream
  // kernel draining its remote stores. The wait comes before the first access
  // to what the stream kernel writes locally (e, the staged values).
  __syncthreads();
  if (r == 0) PROBE(8);

  {
    T* __restrict__ e = static_cast<T*>(sa.e);
    T* __restrict__ x = static_cast<T*>(sa.x);
    T* __restrict__ gsum = static_cast<T*>(a.sum);
    int p = 0;
    while (p + 1 < n && s_bcum[p + 1] <= r) ++p;
    const int rl = r - s_bcum[p], nbl = s_bcum[p + 1] - s_bcum[p];
    const int ntp = s_tcum[p + 1] - s_tcum[p];
    const int rk = s_prank[p];
    const bool own = rk == me;
    const bool hs = a.holder_sum != 0;
    const int ftp = s_ft[p];
    const int t0 = ftp + (int)(((int64_t)ntp * rl) / nbl);
    const int t1 = ftp + (int)(((int64_t)ntp * (rl + 1)) / nbl);
    const unsigned long long* ccnt_ll = a.chunk_in[par][rk];
    const unsigned long long* sidx = a.stage_in[par][rk];
    const P* sp = static_cast<const P*>(sa.stage);
    const int nch = (t1 - t0) * kWarps;
    // chunk counts of the first batch, issued before the base
    int cnt = 0;
    unsigned long long cw = (unsigned long long)ep << 32;
    if (tid < nch) cw = ld_relaxed_sys_u64(&ccnt_ll[t0 * kWarps + tid]);
    // base: the counts of every tile before t0 in partition order (tiles of
    // partitions < p, then [ftp, t0) of p), as words
    int64_t base = 0, poff = 0;  // union position of t0's first entry / of partition p
    if (BIG) {
      // large vectors: this block's range count from the holder's tile words,
      // published as a word; base / poff from the earlier blocks' words (the
      // blocks run in partition order, then tile order)
      int64_t mine = 0;
      const unsigned long long* tw = a.tile_in[par][rk];
      for (int f = t0 + tid; f < t1; f += kThreads) {
        const unsigned long long w = ld_relaxed_sys_u64(&tw[f]);
        mine += (uint32_t)(w >> 32) == ep ? (uint32_t)w : poll_word(&tw[f], ep, a.err);
      }
      mine = warp_sum(mine);
      if (lane == 0) s_red[warp] = mine;
      __syncthreads();
      if (tid == 0) {
        int64_t m = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) m += s_red[w];
        st_relaxed_sys_u64(&a.xrange_words[r], ((unsigned long long)ep << 32) | (uint32_t)m);
      }
      int64_t sb = 0, sp_ = 0;
      for (int q = tid; q < r; q += kThreads) {
        const uint32_t c = poll_word(&a.xrange_words[q], ep, a.err);
        sb += c;
        if (q < s_bcum[p]) sp_ += c;
      }
      sb = warp_sum(sb);
      sp_ = warp_sum(sp_);
      __shared__ int64_t s_redb[kWarps];
      __syncthreads();
      if (lane == 0) {
        s_red[warp] = sb;
        s_redb[warp] = sp_;
      }
      __syncthreads();
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        base += s_red[w];
        poff += s_redb[w];
      }
      __syncthreads();
    } else {
      const int F = s_tcum[p] + (t0 - ftp), Fp = s_tcum[p];
      int64_t sum = 0, sum_before = 0;
      for (int f0 = tid; f0 < F; f0 += kSumUnroll * kThreads) {
        unsigned long long wv[kSumUnroll];
        const unsigned long long* wp[kSumUnroll];
#pragma unroll
        for (int k = 0; k < kSumUnroll; ++k) {
          const int f = f0 + k * kThreads;
          wv[k] = (unsigned long long)ep << 32;  // count 0, current epoch
          wp[k] = nullptr;
          if (f < F) {
            int q = 0;
            while (q + 1 < n && s_tcum[q + 1] <= f) ++q;
            const int tile = s_ft[q] + (f - s_tcum[q]);
            wp[k] = a.tile_in[par][s_prank[q]] + tile;
            wv[k] = ld_relaxed_sys_u64(wp[k]);
          }
        }
#pragma unroll
        for (int k = 0; k < kSumUnroll; ++k) {
          uint32_t c = (uint32_t)wv[k];
          if ((uint32_t)(wv[k] >> 32) != ep) c = poll_word(wp[k], ep, a.err);
          sum += c;
          if (f0 + k * kThreads < Fp) sum_before += c;
        }
      }
      sum = warp_sum(sum);
      sum_before = warp_sum(sum_before);
      __shared__ int64_t s_red2[kWarps];
      if (lane == 0) {
        s_red[warp] = sum;
        s_red2[warp] = sum_before;
      }
      __syncthreads();
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        base += s_red[w];
        poff += s_red2[w];
      }
      __syncthreads();
    }
    if (tid < nch && (uint32_t)(cw >> 32) != ep)
      cw = poll_word(&ccnt_ll[t0 * kWarps + tid], ep, a.err) | ((unsigned long long)ep << 32);
    cnt = (int)(uint32_t)cw;
    PROBE_MAX(41);
    int64_t running = base;  // union position of tile t0's first entry
    unsigned long long cw_next = (unsigned long long)ep << 32;  // BIG: next batch's count word
    for (int cb = 0; cb < nch; cb += kThreads) {
      const int nb = nch - cb < kThreads ? nch - cb : kThreads;
      if (cb) {
        cnt = 0;
        if (tid < nb) {
          const unsigned long long* wp = &ccnt_ll[t0 * kWarps + cb + tid];
          cnt = BIG && (uint32_t)(cw_next >> 32) == ep ? (int)(uint32_t)cw_next
                                                         : (int)poll_word(wp, ep, a.err);
        }
      }
      if (BIG) {  // issue the next batch's count words now: in flight during this batch
        const int cn = cb + kThreads + tid;
        cw_next = cn < nch ? ld_relaxed_sys_u64(&ccnt_ll[t0 * kWarps + cn])
                           : (unsigned long long)ep << 32;
      }
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) s_wtot[warp] = incl;
      __syncthreads();
      int wpre = 0, btot = 0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        wpre += w < warp ? s_wtot[w] : 0;
        btot += s_wtot[w];
      }
      s_off[tid] = wpre + incl - cnt;
      __syncthreads();
      const int64_t cbase = (int64_t)(t0 * kWarps + cb);  // global chunk of s_off[0]
      const int64_t pst = s_pst[p];
      for (int i0 = tid; i0 < btot; i0 += kXUnroll * kThreads) {
        int32_t jj[kXUnroll];
        T vv[kXUnroll];
        unsigned long long jw[kXUnroll];
        int64_t src[kXUnroll], wsrc[kXUnroll];
#pragma unroll
        for (int q = 0; q < kXUnroll; ++q) {
          const int i = i0 + q * kThreads;
          jj[q] = 0;
          vv[q] = T(0);
          jw[q] = (unsigned long long)ep << 32;
          src[q] = wsrc[q] = 0;
          if (i < btot) {
            int lo = 0, hi = nb;  // last chunk k with s_off[k] <= i
            while (hi - lo > 1) {
              const int mid = (lo + hi) >> 1;
              if (s_off[mid] <= i) lo = mid; else hi = mid;
            }
            const int64_t cst = (cbase + lo) * CH;  // runs start at max(chunk, partition start)
            src[q] = (cst > pst ? cst : pst) + (i - s_off[lo]);
            // the pushed words are packed per tile from max(tile start,
            // partition start); batches start on tile boundaries (cbase % 8 == 0)
            const int64_t tst = (cbase + lo) / kWarps * TILE;
            wsrc[q] = sa.tile_pack ? (tst > pst ? tst : pst) + (i - s_off[lo & ~(kWarps - 1)])
                                   : src[q];
            jw[q] = ld_relaxed_sys_u64(&sidx[wsrc[q]]);
          }
        }
#pragma unroll
        for (int q = 0; q < kXUnroll; ++q) {
          if ((uint32_t)(jw[q] >> 32) != ep) jw[q] = poll_word(&sidx[wsrc[q]], ep, a.err);
          jj[q] = (int32_t)(uint32_t)jw[q];
        }
        // x is not written by the stream kernel (the previous step's kernels
        // completed before it started): gather it before the wait
        T xv[kXUnroll];
        if (!TWO) {
#pragma unroll
          for (int q = 0; q < kXUnroll; ++q)
            if (i0 + q * kThreads < btot) xv[q] = x[jj[q]];
        }
        // from here on: what this rank's stream kernel wrote (e, staged values)
        asm volatile("griddepcontrol.wait;" ::: "memory");
#ifdef EXD_PROBE
        if (jj[0] == 0x7fffffff) g_probe[63] = 1;  // force the loads before the stamp
        PROBE_MAX(42);
#endif
#pragma unroll
        for (int q = 0; q < kXUnroll; ++q)
          if (i0 + q * kThreads < btot) vv[q] = own ? Pair<T>::val(__ldcg(&sp[src[q]])) : e[jj[q]];
        // own contribution out (every peer's inbox), union entry, residual clear
#pragma unroll
        for (int q = 0; q < kXUnroll; ++q) {
          const int i = i0 + q * kThreads;
          if (i >= btot) continue;
          const int64_t pos = running + i;
          if (TWO && pos >= a.xcap) {
            // past the contribution slots: the peers pull it (pass 2)
            static_cast<T*>(a.spill_peer[par][me])[pos] = vv[q];
          } else if (!hs) {  // to every peer: each rank sums all n itself
            for (int rr = 0; rr < n; ++rr)
              if (rr != me)
                LL<T>::put(static_cast<unsigned long long*>(a.contrib_out[par][rr]) + pos * W, vv[q], ep);
          } else if (!own) {  // to the partition's holder, which sums and sends the sum back
            LL<T>::put(static_cast<unsigned long long*>(a.contrib_out[par][rk]) + pos * W, vv[q], ep);
          }
          if (TWO && pos < a.xcap && (!hs || own))  // pass 2 sums every source's word, own included
            LL<T>::put(static_cast<unsigned long long*>(a.contrib_out[par][me]) + pos * W, vv[q], ep);
          a.idx_global[pos] = jj[q];
          if (own) {  // this rank's ascending selection (partition-local index)
            sa.idx[pos - poff] = jj[q];
            static_cast<T*>(sa.val)[pos - poff] = vv[q];
          } else {
            e[jj[q]] = T(0);  // own partition was cleared by the stream kernel
          }
        }
#ifdef EXD_PROBE
        PROBE_MAX(43);
#endif
        if (TWO) continue;  // pass 2 below
        // the peers' contributions for the same positions; rank-order sum (the
        // holder only, under the holder sum; the others poll the holder's sum)
        T sv[kXUnroll];
        for (int r0 = 0; r0 < ((!hs || own) ? n : 0); r0 += kXPeers) {
          T pv[kXUnroll][kXPeers];
          bool ok[kXUnroll][kXPeers];
#pragma unroll
          for (int q = 0; q < kXUnroll; ++q)
#pragma unroll
            for (int b = 0; b < kXPeers; ++b) {
              const int rr = r0 + b;
              pv[q][b] = vv[q];
              ok[q][b] = true;
              if (rr < n && rr != me && i0 + q * kThreads < btot)
                ok[q][b] = LL<T>::get(static_cast<const unsigned long long*>(a.contrib_in[par][rr]) +
                                          (running + i0 + q * kThreads) * W, ep, pv[q][b]);
            }
#pragma unroll
          for (int q = 0; q < kXUnroll; ++q)
#pragma unroll
            for (int b = 0; b < kXPeers; ++b) {
              if (ok[q][b]) continue;
              const unsigned long long* w = static_cast<const unsigned long long*>(
                  a.contrib_in[par][r0 + b]) + (running + i0 + q * kThreads) * W;
              const unsigned long long tw = gtime_ns();
              unsigned spins = 0;
              while (!LL<T>::get(w, ep, pv[q][b])) {
                if ((++spins & 255u) == 0 &&
                    (gtime_ns() - tw > 20000000000ull || *(volatile unsigned int*)a.err)) {
                  atomicExch(a.err, 1u);  // a dead peer: the step reports EXD_ENCCL
                  break;
                }
                __nanosleep(20);
              }
            }
#pragma unroll
          for (int q = 0; q < kXUnroll; ++q)
#pragma unroll
            for (int b = 0; b < kXPeers; ++b)
              if (r0 + b < n) sv[q] = r0 + b == 0 ? pv[q][b] : sv[q] + pv[q][b];
        }
        if (hs && own) {  // the holder sends the sums to every peer
#pragma unroll
          for (int q = 0; q < kXUnroll; ++q) {
            if (i0 + q * kThreads >= btot) continue;
            const int64_t pos = running + i0 + q * kThreads;
            for (int rr = 0; rr < n; ++rr)
              if (rr != me)
                LL<T>::put(static_cast<unsigned long long*>(a.sum_out[par][rr]) + pos * W, sv[q], ep);
          }
        } else if (hs) {  // everyone else polls the holder's sum
#pragma unroll
          for (int q = 0; q < kXUnroll; ++q) {
            if (i0 + q * kThreads >= btot) continue;
            const unsigned long long* w = static_cast<const unsigned long long*>(a.sum_in[par]) +
                                          (running + i0 + q * kThreads) * W;
            const unsigned long long tw = gtime_ns();
            unsigned spins = 0;
            while (!LL<T>::get(w, ep, sv[q])) {
              if ((++spins & 255u) == 0 &&
                  (gtime_ns() - tw > 20000000000ull || *(volatile unsigned int*)a.err)) {
                atomicExch(a.err, 1u);
                break;
              }
              __nanosleep(20);
            }
          }
        }
#pragma unroll
        for (int q = 0; q < kXUnroll; ++q) {
          const int i = i0 + q * kThreads;
          if (i >= btot) continue;
          gsum[running + i] = sv[q];
          x[jj[q]] = apply_update<T>(xv[q], sv[q], n);
        }
      }
      running += btot;
      __syncthreads();
    }
    if (TWO) {
      PROBE_MAX(45);  // pass 1 done (probe builds)
      // spilled positions (past the contribution slots): publish this block's
      // spill writes to the peers, then wait for theirs (one flag per source
      // and block; every rank splits the union the same way)
      const bool spills = running > a.xcap;
      if (spills) {
        __syncthreads();  // the block's spill stores, before the fence
        if (tid == 0) {
          asm volatile("fence.acq_rel.sys;" ::: "memory");
          for (int rr = 0; rr < n; ++rr)  // {0, epoch}: poll_word matches the high half
            if (rr != me) st_relaxed_sys_u64(a.spill_flag_out[par][rr] + r, (unsigned long long)ep << 32);
          for (int rr = 0; rr < n; ++rr)
            if (rr != me) poll_word(a.spill_flag_in[par] + (size_t)rr * kMaxCtas + r, ep, a.err);
          asm volatile("fence.acq_rel.sys;" ::: "memory");
        }
        __syncthreads();
      }
      // pass 2 over this block's union positions [base, running)
      const bool sums = !hs || own;  // this rank sums the n words (else: the holder's sum)
      for (int64_t p0 = base + tid; p0 < running; p0 += kX2Unroll * kThreads) {
        int32_t jj[kX2Unroll];
        T xv[kX2Unroll], sv[kX2Unroll];
#pragma unroll
        for (int q = 0; q < kX2Unroll; ++q) {
          const int64_t pos = p0 + (int64_t)q * kThreads;
          if (pos < running) jj[q] = a.idx_global[pos];
        }
#pragma unroll
        for (int q = 0; q < kX2Unroll; ++q)
          if (p0 + (int64_t)q * kThreads < running) xv[q] = x[jj[q]];
#pragma unroll
        for (int q = 0; q < kX2Unroll; ++q) {
          const int64_t pos = p0 + (int64_t)q * kThreads;
          if (pos >= running) continue;
          if (pos >= a.xcap) {  // spilled: pull every source's value, rank order
            for (int rr = 0; rr < n; ++rr) {
              const T v = ld_relaxed_sys_t<T>(static_cast<const T*>(a.spill_peer[par][rr]) + pos);
              sv[q] = rr == 0 ? v : sv[q] + v;
            }
          } else if (sums) {  // rank order, as all_reduce_sum (collectives.cpp:62-68)
            for (int rr = 0; rr < n; ++rr) {
              const T v = poll_ll<T>(static_cast<const unsigned long long*>(a.contrib_in[par][rr]) +
                                         pos * W, ep, a.err);
              sv[q] = rr == 0 ? v : sv[q] + v;
            }
            if (hs)  // the holder sends the sum to every peer
              for (int rr = 0; rr < n; ++rr)
                if (rr != me)
                  LL<T>::put(static_cast<unsigned long long*>(a.sum_out[par][rr]) + pos * W, sv[q], ep);
          } else {
            sv[q] = poll_ll<T>(static_cast<const unsigned long long*>(a.sum_in[par]) + pos * W, ep,
                               a.err);
          }
          gsum[pos] = sv[q];
          x[jj[q]] = apply_update<T>(xv[q], sv[q], n);
        }
      }
    }
  }
  if (BIG) {
    // the ||e||^2 partial of an equal slice of all tiles, for block 0's totals
    asm volatile("griddepcontrol.wait;" ::: "memory");  // returns at once if passed
    const int nt = (int)((rc.n_g + TILE - 1) / TILE);
    const int n0 = (int)(((int64_t)nt * r) / G), n1 = (int)(((int64_t)nt * (r + 1)) / G);
    double pn = 0.0;
    for (int i = n0 + tid; i < n1; i += kThreads) pn += __ldcg(&sa.tile_norm[i]);
    pn = warp_sum(pn);
    __syncthreads();
    if (lane == 0) s_dred[warp] = pn;
    __syncthreads();
    if (tid == 0) {
      double n2 = 0.0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) n2 += s_dred[w];
      const unsigned long long eph = (unsigned long long)ep << 32;
      const unsigned long long nb = (unsigned long long)__double_as_longlong(n2);
      st_relaxed_sys_u64(&a.xrange_words[kMaxCtas + r], eph | (nb & 0xffffffffull));
      st_relaxed_sys_u64(&a.xrange_words[2 * kMaxCtas + r], eph | (nb >> 32));
    }
  }
  if (r == 0) PROBE(9);
  PROBE_MAX(44);
}

template <typename T> struct Bits;
template <> struct Bits<float> {
  using U = uint32_t;
  static constexpr int W = 32;
  __device__ static U abs_bits(float v) { return __float_as_uint(v) & 0x7fffffffu; }
};
template <> struct Bits<double> {
  using U = unsigned long long;
  static constexpr int W = 64;
  __device__ static U abs_bits(double v) {
    return (unsigned long long)__double_as_longlong(v) & 0x7fffffffffffffffULL;
  }
};

// ---- density cap (selector.cpp:44-61, engine.cpp:164-186) --------------------
// When a rank selected more than cap = max(1, llround(cap_frac * n_g / n))
// elements, keep the cap largest |acc| (ties: lower index first), in ascending
// index order. One CTA works on the compacted list (k_i entries): an 8-bit
// radix select finds V, the (k_i - cap)-th smallest |acc| (nth_element's
// partition point); everything above V is kept, and of the elements equal to V
// the first (cap - #above) in index order. Dropped elements get their residual
// back (they are not in the union) and leave the per-block counts.
constexpr int kCapThreads = 1024;

template <typename T>
__global__ void __launch_bounds__(kCapThreads) cap_kernel(CapArgs a, RunConst rc) {
  using U = typename Bits<T>::U;
  __shared__ unsigned int hist[256];
  __shared__ unsigned long long s_prefix, s_mask;
  __shared__ long long s_rank;
  __shared__ int s_wsum[kCapThreads / 32];
  __shared__ int s_wsum2[kCapThreads / 32];
  __shared__ long long s_gt;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t ki = a.cnt->k;
  const int64_t cap = rc.cap;
  T* val = static_cast<T*>(a.val);
  T* e = static_cast<T*>(a.e);
  if (ki <= cap) {
    if (tid == 0) a.cnt->capped = 0;
    for (int64_t i = tid; i < ki; i += kCapThreads)
      for (int p = 0; p < a.npush; ++p) a.push[p][i] = a.idx[i];
    return;
  }
  // radix select of the pos-th smallest |val|, pos = k_i - cap
  if (tid == 0) {
    s_prefix = 0;
    s_mask = 0;
    s_rank = ki - cap;
  }
  for (int shift = Bits<T>::W - 8; shift >= 0; shift -= 8) {
    if (tid < 256) hist[tid] = 0;
    __syncthreads();
    const unsigned long long prefix = s_prefix, mask = s_mask;
    for (int64_t i = tid; i < ki; i += kCapThreads) {
      const unsigned long long b = Bits<T>::abs_bits(val[i]);
      if ((b & mask) == prefix) atomicAdd(&hist[(b >> shift) & 0xffu], 1u);
    }
    __syncthreads();
    if (tid == 0) {
      long long r = s_rank;
      int d = 0;
      for (; d < 256; ++d) {
        if (r < (long long)hist[d]) break;
        r -= hist[d];
      }
      s_rank = r;
      s_prefix |= (unsigned long long)d << shift;
      s_mask |= 0xffULL << shift;
    }
    __syncthreads();
  }
  const unsigned long long V = s_prefix;
  // #elements strictly above V
  int gt = 0;
  for (int64_t i = tid; i < ki; i += kCapThreads) gt += Bits<T>::abs_bits(val[i]) > V;
  gt = warp_sum(gt);
  if (lane == 0) s_wsum[warp] = gt;
  __syncthreads();
  if (tid == 0) {
    long long sgt = 0;
    for (int w = 0; w < kCapThreads / 32; ++w) sgt += s_wsum[w];
    s_gt = sgt;
  }
  __syncthreads();
  const long long keep_ties = cap - s_gt;
  // order-preserving in-place compaction, one chunk of kCapThreads at a time
  long long ties_before = 0, out = 0;
  for (int64_t base = 0; base < ki; base += kCapThreads) {
    const int64_t i = base + tid;
    int32_t j = 0;
    T v = T(0);
    int is_tie = 0, above = 0;
    if (i < ki) {
      j = a.idx[i];
      v = val[i];
      const unsigned long long b = Bits<T>::abs_bits(v);
      above = b > V;
      is_tie = b == V;
    }
    // exclusive scan of is_tie over the chunk (tie rank), then of keep
    int tincl = is_tie;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, tincl, o);
      if (lane >= o) tincl += y;
    }
    if (lane == 31) s_wsum[warp] = tincl;
    __syncthreads();
    int wpre = 0, ttot = 0;
    for (int w = 0; w < kCapThreads / 32; ++w) {
      wpre += w < warp ? s_wsum[w] : 0;
      ttot += s_wsum[w];
    }
    const long long tie_rank = ties_before + wpre + tincl - is_tie;
    const int keep = (i < ki) && (above || (is_tie && tie_rank < keep_ties));
    int kincl = keep;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, kincl, o);
      if (lane >= o) kincl += y;
    }
    if (lane == 31) s_wsum2[warp] = kincl;
    __syncthreads();  // every read of this chunk is done before anyone writes
    int kpre = 0, ktot = 0;
    for (int w = 0; w < kCapThreads / 32; ++w) {
      kpre += w < warp ? s_wsum2[w] : 0;
      ktot += s_wsum2[w];
    }
    if (keep) {
      const int64_t o = out + kpre + kincl - 1;
      a.idx[o] = j;
      val[o] = v;
      for (int p = 0; p < a.npush; ++p) a.push[p][o] = j;
    } else if (i < ki) {
      e[j] = v;  // not in the union: the residual keeps acc (selector.cpp:63-65)
    }
    ties_before += ttot;
    out += ktot;
    __syncthreads();
  }
  if (tid == 0) {
    a.cnt->k = cap;
    a.cnt->capped = 1;
    a.ctrl->k_local = cap;
  }
}

// ---- delta0 broadcast into every worker's control block ---------------------
template <typename T>
__global__ void set_delta_kernel(Ctrl* const* ctrls, int nctrl, const void* bits) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  // engine.cpp:157: max(quantile, 1e-300)
  double d = (double)*static_cast<const T*>(bits);
  if (!(d >= 1e-300)) d = 1e-300;
  for (int i = 0; i < nctrl; ++i) {
    ctrls[i]->delta = d;
    ctrls[i]->thr_f = thr_of(d);
    ctrls[i]->has_delta = 1;
  }
}

// ---- K8: radix select of the pos-th smallest |v| (threshold.cpp:37-47) ------
// The |v| bit patterns order like unsigned integers; 11-bit digits MSB first
// (3 passes over an fp32 vector, 6 over fp64; the last digit may be narrower).
constexpr int kQBits = 11;
constexpr int kQBins = 1 << kQBits;

struct QState {
  unsigned long long prefix, mask;
  long long rank;
  unsigned int hist[kQBins];
};

template <typename T>
__global__ void __launch_bounds__(256) quantile_hist_kernel(const T* v, int64_t m, QState* q,
                                                            int shift, unsigned int dmask,
                                                            bool vec) {
  __shared__ unsigned int h[kQBins];
  for (int i = threadIdx.x; i < kQBins; i += 256) h[i] = 0;
  __syncthreads();
  const unsigned long long prefix = q->prefix, mask = q->mask;
  // 128-bit loads, two per thread in flight (when v is 16-byte aligned); scalar tail
  constexpr int V = 16 / (int)sizeof(T);
  const int64_t n16 = vec ? m / V : 0;
  const int4* v16 = reinterpret_cast<const int4*>(v);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += 2 * stride) {
    T r[2 * V];
    reinterpret_cast<int4*>(r)[0] = __ldg(v16 + i);
    const bool two = i + stride < n16;
    if (two) reinterpret_cast<int4*>(r)[1] = __ldg(v16 + i + stride);
#pragma unroll
    for (int j = 0; j < 2 * V; ++j) {
      if (j >= V && !two) break;
      const unsigned long long b = Bits<T>::abs_bits(r[j]);
      if ((b & mask) == prefix) atomicAdd(&h[(unsigned)(b >> shift) & dmask], 1u);
    }
  }
  for (int64_t i = n16 * V + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    const unsigned long long b = Bits<T>::abs_bits(v[i]);
    if ((b & mask) == prefix) atomicAdd(&h[(unsigned)(b >> shift) & dmask], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kQBins; i += 256)
    if (h[i]) atomicAdd(&q->hist[i], h[i]);
}

// 256 threads, 8 consecutive bins each: block scan of the thread sums, then
// the thread whose range holds rank walks its bins to the next digit. Every
// thread clears the bins it has read.
__global__ void __launch_bounds__(256) quantile_pick_kernel(QState* q, int shift,
                                                            unsigned int dmask) {
  constexpr int P = kQBins / 256;
  __shared__ long long inc[256];
  const int i = threadIdx.x;
  const long long r = q->rank;
  unsigned int v[P];
  long long mine = 0;
#pragma unroll
  for (int j = 0; j < P; ++j) {
    v[j] = q->hist[i * P + j];
    q->hist[i * P + j] = 0;
    mine += v[j];
  }
  inc[i] = mine;
  __syncthreads();
  for (int o = 1; o < 256; o <<= 1) {
    const long long add = i >= o ? inc[i - o] : 0;
    __syncthreads();
    inc[i] += add;
    __syncthreads();
  }
  long long excl = inc[i] - mine;
  if (mine > 0 && r >= excl && r < inc[i]) {
    int d = 0;
    for (; d < P - 1; ++d) {
      if (r < excl + (long long)v[d]) break;
      excl += v[d];
    }
    q->rank = r - excl;
    q->prefix |= (unsigned long long)(i * P + d) << shift;
    q->mask |= (unsigned long long)dmask << shift;
  }
}

template <typename T>
__global__ void __launch_bounds__(256) quantile_init_kernel(QState* q, int64_t pos) {
  if (threadIdx.x == 0) {
    q->prefix = 0;
    q->mask = 0;
    q->rank = pos;
  }
  for (int i = threadIdx.x; i < kQBins; i += 256) q->hist[i] = 0;
}

template <typename T>
__global__ void quantile_out_kernel(const QState* q, T* out) {
  if (threadIdx.x != 0) return;
  if (sizeof(T) == 4) {
    const uint32_t b = (uint32_t)q->prefix;
    *reinterpret_cast<uint32_t*>(out) = b;
  } else {
    *reinterpret_cast<unsigned long long*>(out) = q->prefix;
  }
}

template <typename T>
cudaError_t quantile_t(const T* v, int64_t m, int64_t pos, QState* q, T* out, cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const bool vec = (reinterpret_cast<uintptr_t>(v) & 15u) == 0;
  quantile_init_kernel<T><<<1, 256, 0, s>>>(q, pos);
  int64_t blocks = (m + 256 * 16 / (int64_t)sizeof(T) - 1) / (256 * 16 / (int64_t)sizeof(T));
  const int64_t per_sm = sizeof(T) == 8 ? 8 : 4;  // measured: f32 4 CTAs/SM, f64 8
  if (blocks > (int64_t)sms * per_sm) blocks = (int64_t)sms * per_sm;
  if (blocks < 1) blocks = 1;
  for (int hi = Bits<T>::W; hi > 0; hi -= kQBits) {
    const int shift = hi > kQBits ? hi - kQBits : 0;
    const unsigned int dmask = (1u << (hi - shift)) - 1u;
    quantile_hist_kernel<T><<<(unsigned)blocks, 256, 0, s>>>(v, m, q, shift, dmask, vec);
    quantile_pick_kernel<<<1, 256, 0, s>>>(q, shift, dmask);
  }
  quantile_out_kernel<T><<<1, 32, 0, s>>>(q, out);
  return cudaGetLastError();
}

// ---- replica check (engine.cpp:251-272), debug option -----------------------
template <typename T>
__global__ void verify_kernel(const Ctrl* c0, const Ctrl* cw, const T* x0, const T* xw,
                              int64_t n_g, int32_t w, uint32_t* flag) {
  // flag bits: 1 delta, 2 k_t, 4 topology, 8 x; value (w << 8) | bits
  uint32_t bits = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (__double_as_longlong(c0->delta) != __double_as_longlong(cw->delta)) bits |= 1;
    for (int i = 0; i < EXD_MAX_WORKERS; ++i)
      if (c0->k_t[i] != cw->k_t[i]) bits |= 2;
    const int64_t* a = reinterpret_cast<const int64_t*>(&c0->topo);
    const int64_t* b = reinterpret_cast<const int64_t*>(&cw->topo);
    for (size_t i = 0; i < sizeof(exd_topology) / 8; ++i)
      if (a[i] != b[i]) bits |= 4;
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_g;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (Bits<T>::abs_bits(x0[i]) != Bits<T>::abs_bits(xw[i]) || signbit(x0[i]) != signbit(xw[i])) {
      bits |= 8;
      break;
    }
  }
  if (bits) atomicCAS(flag, 0u, ((uint32_t)w << 8) | bits);
}

__host__ __device__ inline unsigned long long mix64(unsigned long long z);

// ---- verify_replication across ranks (engine.cpp:251-272) --------------------
// Replicas live on different GPUs: each rank hashes its replicated state per
// field (delta bits, k_t, topology, x) into 4 words; the words are all-gathered
// and compared against rank 0's. XOR of per-element mixes is order-free, so the
// hash is deterministic whatever the reduction order.
__device__ __forceinline__ unsigned long long mix_word(unsigned long long v, unsigned long long i) {
  return mix64(v ^ (i * 0x9e3779b97f4a7c15ULL));
}

template <typename T>
__global__ void __launch_bounds__(256) replica_hash_kernel(const Ctrl* c, const T* x, int64_t n_g,
                                                           int n, unsigned long long* out4) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long hd = mix_word((unsigned long long)__double_as_longlong(c->delta), 0);
    unsigned long long hk = 0, ht = mix_word((unsigned long long)c->topo.sz_blk, 1);
    for (int r = 0; r < n; ++r) {
      hk ^= mix_word((unsigned long long)c->k_t[r], 2 + r);
      ht ^= mix_word((unsigned long long)c->topo.blk_part[r], 100 + r);
      ht ^= mix_word((unsigned long long)c->topo.blk_pos[r], 200 + r);
    }
    atomicXor(&out4[0], hd);
    atomicXor(&out4[1], hk);
    atomicXor(&out4[2], ht);
  }
  unsigned long long hx = 0;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_g;
       j += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long b = sizeof(T) == 4 ? (unsigned long long)__float_as_uint((float)x[j])
                                                : (unsigned long long)__double_as_longlong((double)x[j]);
    hx ^= mix_word(b, (unsigned long long)j + 1000);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) hx ^= __shfl_xor_sync(0xffffffffu, hx, o);
  if ((threadIdx.x & 31) == 0 && hx) atomicXor(&out4[3], hx);
}

__global__ void replica_compare_kernel(const unsigned long long* all4, int n, uint32_t* flag) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (int r = 1; r < n; ++r)
    for (int f = 0; f < 4; ++f)  // reference order: delta, k_t, topology, x
      if (all4[4 * r + f] != all4[f]) {
        atomicCAS(flag, 0u, ((uint32_t)r << 8) | (1u << f));
        return;
      }
}

// ---- verify_conservation (engine.cpp:221-249), debug option -----------------
// snapshot: acc = e + eta*g with the stream kernel's exact arithmetic, taken
// before the step; after it: every contribution equals the snapshot at its
// union index, the residual is cleared there, and untouched everywhere else.
// Violations are reported through `flag` as 0x10000 * code | rank << 8.
template <typename T>
__global__ void __launch_bounds__(256) snapshot_kernel(const T* e, const T* g, T* snap, int64_t n_g,
                                                       double eta) {
  const bool unit = eta == 1.0;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_g;
       j += (int64_t)gridDim.x * blockDim.x)
    snap[j] = accumulate<T>(e[j], g[j], eta, unit);
}

template <typename T> __device__ __forceinline__ bool same_bits(T a, T b);
template <> __device__ __forceinline__ bool same_bits<float>(float a, float b) {
  return __float_as_uint(a) == __float_as_uint(b);
}
template <> __device__ __forceinline__ bool same_bits<double>(double a, double b) {
  return __double_as_longlong(a) == __double_as_longlong(b);
}

template <typename T>
__global__ void __launch_bounds__(256) conserve_union_kernel(const int32_t* uni, const CountRec* counts,
                                                             int n, const T* contrib, const T* e,
                                                             const T* snap, uint32_t* bitmap,
                                                             uint32_t* flag, uint32_t rank) {
  int64_t kp = 0;
  for (int r = 0; r < n; ++r) kp += counts[r].k;
  for (int64_t pos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pos < kp;
       pos += (int64_t)gridDim.x * blockDim.x) {
    const int32_t j = uni[pos];
    if (!same_bits<T>(contrib[pos], snap[j])) atomicCAS(flag, 0u, 0x10000u | (rank << 8));
    if (e[j] != T(0)) atomicCAS(flag, 0u, 0x20000u | (rank << 8));
    atomicOr(&bitmap[j >> 5], 1u << (j & 31));
  }
}

template <typename T>
__global__ void __launch_bounds__(256) conserve_rest_kernel(const T* e, const T* snap,
                                                            const uint32_t* bitmap, int64_t n_g,
                                                            uint32_t* flag, uint32_t rank) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_g;
       j += (int64_t)gridDim.x * blockDim.x) {
    if ((bitmap[j >> 5] >> (j & 31)) & 1u) continue;
    if (!same_bits<T>(e[j], snap[j])) {
      atomicCAS(flag, 0u, 0x30000u | (rank << 8));
      return;
    }
  }
}

// ---- device GradientSource: workloads.cpp:62-85 + rng.hpp:28-59 ----------
struct SegTable {
  int32_t nseg;
  int32_t dist;
  int64_t start[EXD_MAX_SEGMENTS + 1];
  unsigned long long key[EXD_MAX_SEGMENTS];
  double scale[EXD_MAX_SEGMENTS];
};

__host__ __device__ inline unsigned long long mix64(unsigned long long z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

template <typename T>
__global__ void __launch_bounds__(256) synthetic_kernel(SegTable tab, int64_t n_g, T* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_g;
       i += (int64_t)gridDim.x * blockDim.x) {
    int s = 0;
    while (s + 1 < tab.nseg && tab.start[s + 1] <= i) ++s;
    const unsigned long long j = (unsigned long long)(i - tab.start[s]);
    const double scale = tab.scale[s];
    double v;
    if (tab.dist == 0) {
      // Stream::next_laplace: state advances once per draw (counter-based)
      const unsigned long long u64 = mix64(tab.key[s] + (j + 1) * 0x9e3779b97f4a7c15ULL);
      const double u = ((double)(u64 >> 11) + 0.5) * 0x1.0p-53 - 0.5;
      const double mag = -scale * log1p(-2.0 * fabs(u));
      v = u < 0.0 ? -mag : mag;
    } else {
      const unsigned long long b = tab.key[s] + 3 * j * 0x9e3779b97f4a7c15ULL;
      const double u1 = ((double)(mix64(b + 0x9e3779b97f4a7c15ULL) >> 11) + 0.5) * 0x1.0p-53;
      const double u2 = ((double)(mix64(b + 2 * 0x9e3779b97f4a7c15ULL) >> 11) + 0.5) * 0x1.0p-53;
      const double z = sqrt(-2.0 * log(u1)) * cos(6.283185307179586477 * u2);
      const double mag = scale * exp(z);
      v = (mix64(b + 3 * 0x9e3779b97f4a7c15ULL) & 1ULL) ? mag : -mag;
    }
    out[i] = (T)v;
  }
}

int grid_for(int64_t work, int per_block) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t b = (work + per_block - 1) / per_block;
  const int64_t cap = (int64_t)sms * 8;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

}  // namespace

// L2 flush for timing hygiene: write a buffer larger than L2, then read it
// back so the lines left in L2 are clean (no write-back lands on the next
// kernel's timeline).
static __global__ void l2_read_kernel(const float4* __restrict__ p, int64_t n4, int* sink) {
  float s = 0.f;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x)
    s += __ldcg(&p[i]).x;
  if (s == 1234.5f) atomicAdd(sink, 1);
}

#ifdef EXD_PROBE
extern "C" int exd_debug_probe(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_probe, sizeof(g_probe));
}
extern "C" int exd_debug_ctas(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_cta, sizeof(g_cta));
}
#endif

cudaError_t launch_l2_flush(void* buf, size_t bytes, cudaStream_t s) {
  cudaError_t err = cudaMemsetAsync(buf, 1, bytes, s);
  if (err != cudaSuccess) return err;
  const int blocks = grid_for((int64_t)(bytes / 16), 256 * 4);
  l2_read_kernel<<<blocks, 256, 0, s>>>(static_cast<const float4*>(buf), (int64_t)((bytes - 64) / 16),
                                        reinterpret_cast<int*>(static_cast<char*>(buf) + bytes - 64));
  return cudaGetLastError();
}

int tile_elems(int dtype) { return dtype == EXD_F64 ? tile_of<double>() : tile_of<float>(); }

int64_t num_tiles(int64_t n_g, int dtype) {
  const int t = tile_elems(dtype);
  return (n_g + t - 1) / t;
}

cudaError_t launch_stream(int mode, SelectArgs a, RunConst rc, cudaStream_t s) {
  return rc.dtype == EXD_F64 ? launch_stream_t<double>(mode, a, rc, s)
                             : launch_stream_t<float>(mode, a, rc, s);
}

cudaError_t launch_finish(SelectArgs a, RunConst rc, cudaStream_t s) {
  return rc.dtype == EXD_F64 ? launch_finish_t<double>(a, rc, s) : launch_finish_t<float>(a, rc, s);
}

cudaError_t launch_union(UnionArgs a, RunConst rc, cudaStream_t s) {
  // k' is device-resident; size for the worst case the grid-stride loop covers
  const int blocks = grid_for(rc.n_g, 256 * 4);
  if (rc.dtype == EXD_F64) union_kernel<double><<<blocks, 256, 0, s>>>(a, rc);
  else union_kernel<float><<<blocks, 256, 0, s>>>(a, rc);
  return cudaGetLastError();
}

cudaError_t launch_allreduce_local(const void* const* contribs, void* sum, const Ctrl*,
                                   const CountRec* counts, RunConst rc, cudaStream_t s) {
  const int blocks = grid_for(rc.n_g, 256 * 4);
  if (rc.dtype == EXD_F64)
    allreduce_local_kernel<double><<<blocks, 256, 0, s>>>(contribs, sum, counts, rc);
  else
    allreduce_local_kernel<float><<<blocks, 256, 0, s>>>(contribs, sum, counts, rc);
  return cudaGetLastError();
}

cudaError_t launch_finalize(FinalizeArgs a, RunConst rc, cudaStream_t s) {
  const int blocks = grid_for(rc.n_g, 256 * 4);
  if (rc.dtype == EXD_F64) finalize_kernel<double><<<blocks, 256, 0, s>>>(a, rc);
  else finalize_kernel<float><<<blocks, 256, 0, s>>>(a, rc);
  return cudaGetLastError();
}

// every block's thread 0 polls the peers' flags: keep the grid at two CTAs
// per SM (k' <= n_g entries are covered by the grid-stride loops)
static int p2p_blocks() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return 2 * sms;
}

// programmatic launch: overlap each launch with the previous kernel's tail;
// the kernels start with griddepcontrol.wait
template <typename K>
static cudaError_t launch_pdl(K kernel, int blocks, cudaStream_t s, const P2PArgs& a,
                              const RunConst& rc) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, a, rc);
}

cudaError_t launch_p2p_sync(const P2PArgs& a, RunConst rc, cudaStream_t s) {
  const int blocks = p2p_blocks() + 1;
  if (rc.dtype == EXD_F64) return launch_pdl(p2p_sync_kernel<double>, blocks, s, a, rc);
  return launch_pdl(p2p_sync_kernel<float>, blocks, s, a, rc);
}

cudaError_t launch_exchange(const ExchangeArgs& a, RunConst rc, cudaStream_t s) {
  // 3 per SM, all resident (__launch_bounds__(kThreads, 3)): block 0 + 3*SMs - 1
  // work blocks, so a dense tile range is split finely enough for one pass
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p2p_blocks() / 2 * 3);
  cfg.blockDim = dim3(kThreads);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const bool big = a.xrange_words != nullptr;
  const bool two = a.two_pass != 0;
#define EXD_XK(T_, B_, P_) cudaLaunchKernelEx(&cfg, exchange_kernel<T_, B_, P_>, a, rc)
  if (rc.dtype == EXD_F64)
    return big ? (two ? EXD_XK(double, true, true) : EXD_XK(double, true, false))
               : (two ? EXD_XK(double, false, true) : EXD_XK(double, false, false));
  return big ? (two ? EXD_XK(float, true, true) : EXD_XK(float, true, false))
             : (two ? EXD_XK(float, false, true) : EXD_XK(float, false, false));
#undef EXD_XK
}

cudaError_t launch_cap(const CapArgs& a, RunConst rc, cudaStream_t s) {
  if (rc.dtype == EXD_F64) cap_kernel<double><<<1, kCapThreads, 0, s>>>(a, rc);
  else cap_kernel<float><<<1, kCapThreads, 0, s>>>(a, rc);
  return cudaGetLastError();
}

cudaError_t launch_snapshot(const void* e, const void* g, void* snap, RunConst rc, cudaStream_t s) {
  const int blocks = grid_for(rc.n_g, 256 * 8);
  if (rc.dtype == EXD_F64)
    snapshot_kernel<double><<<blocks, 256, 0, s>>>(static_cast<const double*>(e),
                                                   static_cast<const double*>(g),
                                                   static_cast<double*>(snap), rc.n_g, rc.eta);
  else
    snapshot_kernel<float><<<blocks, 256, 0, s>>>(static_cast<const float*>(e),
                                                  static_cast<const float*>(g),
                                                  static_cast<float*>(snap), rc.n_g, rc.eta);
  return cudaGetLastError();
}

cudaError_t launch_conservation(const int32_t* uni, const CountRec* counts, int ncounts,
                                const void* contrib, const void* e, const void* snap,
                                uint32_t* bitmap, uint32_t* flag, RunConst rc, cudaStream_t s) {
  cudaError_t err = cudaMemsetAsync(bitmap, 0, 4 * (size_t)((rc.n_g + 31) / 32), s);
  if (err != cudaSuccess) return err;
  const int blocks = grid_for(rc.n_g, 256 * 8);
  const uint32_t rank = (uint32_t)rc.rank;
  if (rc.dtype == EXD_F64) {
    conserve_union_kernel<double><<<blocks, 256, 0, s>>>(
        uni, counts, ncounts, static_cast<const double*>(contrib), static_cast<const double*>(e),
        static_cast<const double*>(snap), bitmap, flag, rank);
    conserve_rest_kernel<double><<<blocks, 256, 0, s>>>(static_cast<const double*>(e),
                                                        static_cast<const double*>(snap), bitmap,
                                                        rc.n_g, flag, rank);
  } else {
    conserve_union_kernel<float><<<blocks, 256, 0, s>>>(
        uni, counts, ncounts, static_cast<const float*>(contrib), static_cast<const float*>(e),
        static_cast<const float*>(snap), bitmap, flag, rank);
    conserve_rest_kernel<float><<<blocks, 256, 0, s>>>(static_cast<const float*>(e),
                                                       static_cast<const float*>(snap), bitmap,
                                                       rc.n_g, flag, rank);
  }
  return cudaGetLastError();
}

cudaError_t launch_replica_hash(const Ctrl* c, const void* x, unsigned long long* out4, RunConst rc,
                                cudaStream_t s) {
  cudaError_t err = cudaMemsetAsync(out4, 0, 4 * sizeof(unsigned long long), s);
  if (err != cudaSuccess) return err;
  const int blocks = grid_for(rc.n_g, 256 * 8);
  if (rc.dtype == EXD_F64)
    replica_hash_kernel<double><<<blocks, 256, 0, s>>>(c, static_cast<const double*>(x), rc.n_g, rc.n,
                                                       out4);
  else
    replica_hash_kernel<float><<<blocks, 256, 0, s>>>(c, static_cast<const float*>(x), rc.n_g, rc.n,
                                                      out4);
  return cudaGetLastError();
}

cudaError_t launch_replica_compare(const unsigned long long* all4, int n, uint32_t* flag,
                                   cudaStream_t s) {
  replica_compare_kernel<<<1, 32, 0, s>>>(all4, n, flag);
  return cudaGetLastError();
}

cudaError_t launch_set_delta(Ctrl* const* ctrls, int nctrl, const void* bits, int dtype,
                             cudaStream_t s) {
  if (dtype == EXD_F64) set_delta_kernel<double><<<1, 32, 0, s>>>(ctrls, nctrl, bits);
  else set_delta_kernel<float><<<1, 32, 0, s>>>(ctrls, nctrl, bits);
  return cudaGetLastError();
}

size_t quantile_scratch_bytes() { return sizeof(QState); }

int quantile_launches(int dtype) {
  const int w = dtype == EXD_F64 ? 64 : 32;
  return 2 + 2 * ((w + kQBits - 1) / kQBits);  // init, (hist + pick) per digit, out
}

cudaError_t launch_quantile(const void* v, int64_t m, int64_t pos, int dtype, void* scratch,
                            void* out_bits, cudaStream_t s) {
  QState* q = static_cast<QState*>(scratch);
  if (dtype == EXD_F64)
    return quantile_t<double>(static_cast<const double*>(v), m, pos, q,
                              static_cast<double*>(out_bits), s);
  return quantile_t<float>(static_cast<const float*>(v), m, pos, q, static_cast<float*>(out_bits), s);
}

// Per-ExDyna-block selection counts of the last step (a diagnostic: the
// reference keeps only per-partition counts, Appendix A of SURVEY.md), from the
// worker's own ascending selection on demand. Counting them in the stream
// kernel cost 40-55 us per step at n_g = 1e8: every warp of a wave added into
// the same few block counters.
__global__ void __launch_bounds__(256) block_counts_kernel(const int32_t* idx, const CountRec* cnt,
                                                           int32_t* out, RunConst rc) {
  extern __shared__ int32_t s_h[];
  const bool smem = rc.n_b <= 8192;
  if (smem)
    for (int b = threadIdx.x; b < rc.n_b; b += blockDim.x) s_h[b] = 0;
  __syncthreads();
  const int64_t k = cnt->k;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t b = block_of((uint32_t)idx[i], rc);
    if (smem) atomicAdd(&s_h[b], 1);
    else atomicAdd(&out[b], 1);
  }
  __syncthreads();
  if (smem)
    for (int b = threadIdx.x; b < rc.n_b; b += blockDim.x)
      if (s_h[b]) atomicAdd(&out[b], s_h[b]);
}

cudaError_t launch_block_counts(const int32_t* idx, const CountRec* cnt, int64_t cap, int32_t* out,
                                RunConst rc, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(int32_t) * (size_t)rc.n_b, s);
  if (e != cudaSuccess) return e;
  const int blocks = grid_for(cap > 0 ? cap : 1, 256 * 4);
  const size_t sm = rc.n_b <= 8192 ? sizeof(int32_t) * (size_t)rc.n_b : 0;
  block_counts_kernel<<<blocks, 256, sm, s>>>(idx, cnt, out, rc);
  return cudaGetLastError();
}

cudaError_t launch_verify_replication(const Ctrl* c0, const Ctrl* cw, const void* x0,
                                      const void* xw, int64_t n_g, int dtype, int32_t w,
                                      uint32_t* flag, cudaStream_t s) {
  const int blocks = grid_for(n_g, 256 * 8);
  if (dtype == EXD_F64)
    verify_kernel<double><<<blocks, 256, 0, s>>>(c0, cw, static_cast<const double*>(x0),
                                                 static_cast<const double*>(xw), n_g, w, flag);
  else
    verify_kernel<float><<<blocks, 256, 0, s>>>(c0, cw, static_cast<const float*>(x0),
                                                static_cast<const float*>(xw), n_g, w, flag);
  return cudaGetLastError();
}

cudaError_t launch_synthetic(const exd_stream_spec* spec, int64_t t, int32_t rank, int dtype,
                             void* out, cudaStream_t s) {
  SegTable tab{};
  tab.nseg = spec->nseg;
  tab.dist = spec->distribution;
  int64_t pos = 0;
  for (int si = 0; si < spec->nseg; ++si) {
    tab.start[si] = pos;
    pos += spec->seg_length[si];
    // effective_scale, workloads.cpp:42-46 (host pow, as the reference)
    double sc = spec->seg_scale[si] * pow(spec->decay, (double)t);
    if (spec->has_decay_step && t >= spec->decay_step) sc *= spec->decay_step_factor;
    tab.scale[si] = sc;
    // derive_key({seed, kTagStream, t, rank, si}), rng.hpp:37-41
    const unsigned long long words[5] = {spec->seed, 0x53545245414dULL, (unsigned long long)t,
                                         (unsigned long long)rank, (unsigned long long)si};
    unsigned long long h = 0x6a09e667f3bcc909ULL;
    for (int w = 0; w < 5; ++w) h = mix64(h ^ words[w]);
    tab.key[si] = h;
  }
  tab.start[spec->nseg] = pos;
  const int blocks = grid_for(spec->n_g, 256 * 4);
  if (dtype == EXD_F64)
    synthetic_kernel<double><<<blocks, 256, 0, s>>>(tab, spec->n_g, static_cast<double*>(out));
  else
    synthetic_kernel<float><<<blocks, 256, 0, s>>>(tab, spec->n_g, static_cast<float*>(out));
  return cudaGetLastError();
}

}  // namespace exd
