// kernels.cu — the sm_100a kernels of the ExDyna sparsify+sync path.
//
//   select_kernel   (K1+K2) fused accumulate e <- e + eta*g over the full
//                   vector, |acc| >= delta test over the worker's exclusive
//                   partition, per-block counts, and ordered single-pass
//                   compaction to (int32 index, value) pairs by decoupled
//                   look-back; own selected residuals are zeroed in the same
//                   pass. For n == 1 it also applies x -= g/n and runs the
//                   control epilogue, so a whole step is one launch.
//   union_kernel    (K4+K5) union in partition order + contribution gather +
//                   residual clear at the union.
//   allreduce_local rank-order sum of n in-process contributions (K6, sim mode).
//   finalize_kernel (K7+K9) x scatter, threshold scaling, record, next plan.
//   quantile        (K8) radix select of the (1-d)-quantile of |acc| at t = 0.
//   synthetic       device GradientSource (workloads.cpp:62-85).
//
// Reference lines are cited at each kernel. Everything here is HBM- or
// latency-bound integer/byte work: there is no GEMM to put on tcgen05, so the
// design levers are 128-bit coalesced loads, enough bytes in flight, one pass
// over HBM, and grids sized to the 148 SMs.
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.cuh"

namespace exd {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kUnroll = 4;
static_assert(kUnroll * kWarps == 32, "the block scan assumes one warp of partials");

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

__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// look-back status word: epoch:30 | flag:2 | value:32
constexpr unsigned kAgg = 1, kIncl = 2;
__device__ __forceinline__ unsigned long long pack_status(uint32_t epoch, unsigned flag,
                                                          uint32_t v) {
  return ((unsigned long long)((epoch << 2) | flag) << 32) | v;
}

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
  return __dadd_rn(prev, __dmul_rn(eta, g));
}

// |acc| >= delta (selector.cpp:39) with delta in fp64. For float acc,
// (double)|acc| >= delta  <=>  |acc| >= round_up_to_float(delta).
template <typename T> __device__ __forceinline__ bool selected(T a, const Ctrl* c);
template <> __device__ __forceinline__ bool selected<float>(float a, const Ctrl* c) {
  return fabsf(a) >= c->thr_f;
}
template <> __device__ __forceinline__ bool selected<double>(double a, const Ctrl* c) {
  return fabs(a) >= c->delta;
}

// x -= g / n (engine.cpp:215) evaluated in fp64, rounded once to T
template <typename T> __device__ __forceinline__ T apply_update(T x, T g, int n) {
  return (T)__dadd_rn((double)x, -__ddiv_rn((double)g, (double)n));
}

__device__ __forceinline__ float thr_of(double delta) { return __double2float_ru(delta); }

// ---- control epilogue ----------------------------------------------------
// Runs on ONE thread at the end of step t: the all-gather accounting
// (collectives.cpp:29-45), the ledger row (engine.cpp:327-349), the threshold
// rescale and k_t update (engine.cpp:206-213) and the plan of step t+1
// (engine.cpp:125-131: rotate -> adjust -> allocate).
// The epilogue works in place on the global control block with loops bounded
// by n (no whole-struct copies), and is kept out of line so it does not
// inflate the register allocation of the streaming kernels that call it.
__device__ __forceinline__ void copy_topo(exd_topology* dst, const exd_topology* src, int n) {
  dst->n = src->n;
  dst->sz_blk = src->sz_blk;
  for (int i = 0; i < n; ++i) {
    dst->blk_part[i] = src->blk_part[i];
    dst->blk_pos[i] = src->blk_pos[i];
  }
}

__device__ __noinline__ void make_plan(Ctrl* c, const RunConst& rc) {
  Plan* p = &c->plan;
  const int n = rc.n;
  copy_topo(&p->topo, &c->topo, n);
  int32_t mv = 0, sk = 0;
  if (!rc.static_partitions) {
    int64_t kp[EXD_MAX_WORKERS];
    rotate(c->k_t, c->t, n, kp);
    adjust(p->topo, kp, rc.alpha, rc.blk_move, rc.min_blk, rc.n_g, &mv, &sk);
  }
  p->moves = mv;
  p->skips = sk;
  int64_t st, end;
  p->partition = allocate(p->topo, c->t, rc.rank, rc.n_g, &st, &end);
  p->st = st;
  p->end = end;
}

__device__ __noinline__ void control_epilogue(Ctrl* c, const CountRec* counts, const RunConst& rc,
                                              exd_record* rec) {
  const int n = rc.n;
  int64_t k_rank[EXD_MAX_WORKERS];
  double norm_sum = 0.0;
  for (int r = 0; r < n; ++r) {
    k_rank[r] = counts[r].k;
    norm_sum = __dadd_rn(norm_sum, sqrt(counts[r].norm2));
  }
  exd_gather_stats gs;
  gather_stats(k_rank, n, &gs);
  const double delta_used = c->delta;
  if (rec) {
    rec->t = c->t;
    rec->k_prime = gs.k_prime;
    rec->density = __ddiv_rn((double)gs.k_prime, (double)rc.n_g);
    const int64_t diff = rc.k - gs.k_prime;
    rec->eps = __ddiv_rn((double)(diff < 0 ? -diff : diff), (double)rc.n_g);
    rec->m_t = gs.m_t;
    rec->c_t = gs.c_t;
    rec->f_t = gs.f_t;
    rec->global_err = __ddiv_rn(norm_sum, (double)n);
    rec->delta = delta_used;
    rec->has_loss = 0;
    rec->loss = 0.0;
    rec->duplicates = 0;  // disjoint partitions + ascending lists: no duplicates by construction
    rec->union_count = gs.k_prime;
    rec->n = n;
    rec->adjust_moves = c->plan.moves;
    rec->adjust_skips = c->plan.skips;
    rec->cap_hits = 0;
    rec->idle_workers = 0;
    for (int r = 0; r < n; ++r) rec->k_rank[r] = k_rank[r];
  }
  // apply_phase control (engine.cpp:211-213)
  c->delta = scale_threshold(rc.k, gs.k_prime, c->delta, rc.beta, rc.gamma);
  c->thr_f = thr_of(c->delta);
  for (int r = 0; r < n; ++r) c->k_t[r] = k_rank[r];
  copy_topo(&c->topo, &c->plan.topo, n);
  copy_topo(&c->last.topo, &c->plan.topo, n);
  c->last.st = c->plan.st;
  c->last.end = c->plan.end;
  c->last.partition = c->plan.partition;
  c->last.moves = c->plan.moves;
  c->last.skips = c->plan.skips;
  c->t += 1;
  make_plan(c, rc);
}

// ---- K1+K2: fused accumulate / select / compact ----------------------------
// engine.cpp:135-141 (accumulate), selector.cpp:35-42 (select), engine.cpp:199-202
// (values), selector.cpp:63-65 (clear, own partition). One tile per CTA, tile
// ids handed out by an atomic ticket so look-back only ever waits on CTAs that
// are already resident.
template <typename T, int MODE, bool FUSED>
__global__ void __launch_bounds__(kThreads) select_kernel(SelectArgs a, RunConst rc) {
  constexpr int VN = Vec<T>::N;
  constexpr int TILE = tile_of<T>();
  constexpr bool ACCUM = MODE != kSelectOnly;
  constexpr bool SELECT = MODE != kAccumulate;

  __shared__ int s_tile;
  __shared__ int s_off[32];
  __shared__ uint32_t s_prefix;
  __shared__ double s_norm[kWarps];
  __shared__ bool s_last;
  __shared__ bool s_split;

  Ctrl* ctrl = a.ctrl;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = a.tile_base + (int)atomicAdd(&ctrl->ticket, 1u);
  __syncthreads();
  const int tile = s_tile;
  const int64_t n_g = rc.n_g;
  const int64_t st = ctrl->plan.st, end = ctrl->plan.end;
  const int64_t tbeg = (int64_t)tile * TILE;
  const int64_t tend = tbeg + TILE < n_g ? tbeg + TILE : n_g;
  const bool sel_tile = SELECT && tbeg < end && tend > st;
  const bool full_in = tbeg >= st && tend <= end;
  const bool unit = rc.eta == 1.0;

  T* e = static_cast<T*>(a.e);
  const T* g = static_cast<const T*>(a.g);

  T v[kUnroll][VN];
  double nrm = 0.0;
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) {
    const int64_t base = tbeg + ((int64_t)u * kThreads + tid) * VN;
    T ev[VN], gv[VN];
    if (base + VN <= n_g) {
      vload<T>(e + base, ev);
      if (ACCUM) vload<T>(g + base, gv);
    } else {
#pragma unroll
      for (int c = 0; c < VN; ++c) {
        ev[c] = base + c < n_g ? e[base + c] : T(0);
        gv[c] = (ACCUM && base + c < n_g) ? g[base + c] : T(0);
      }
    }
#pragma unroll
    for (int c = 0; c < VN; ++c) {
      if (ACCUM) {
        const double prev = (double)ev[c];
        nrm = fma(prev, prev, nrm);
        v[u][c] = accumulate<T>(ev[c], gv[c], rc.eta, unit);
      } else {
        v[u][c] = ev[c];
      }
    }
  }

  // selection flags, bit (u*VN + c)
  uint32_t flags = 0;
  if (sel_tile) {
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t base = tbeg + ((int64_t)u * kThreads + tid) * VN;
#pragma unroll
      for (int c = 0; c < VN; ++c) {
        const int64_t j = base + c;
        const bool in = full_in ? (j < n_g) : (j >= st && j < end);
        if (in && selected<T>(v[u][c], ctrl)) flags |= 1u << (u * VN + c);
      }
    }
  }

  // residual write-back: acc, or 0 where selected (own partition cleared here)
  if (ACCUM) {
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t base = tbeg + ((int64_t)u * kThreads + tid) * VN;
      T w[VN];
#pragma unroll
      for (int c = 0; c < VN; ++c) w[c] = (flags >> (u * VN + c)) & 1u ? T(0) : v[u][c];
      if (base + VN <= n_g) {
        vstore<T>(e + base, w);
      } else {
#pragma unroll
        for (int c = 0; c < VN; ++c)
          if (base + c < n_g) e[base + c] = w[c];
      }
    }
  } else if (flags) {
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t base = tbeg + ((int64_t)u * kThreads + tid) * VN;
#pragma unroll
      for (int c = 0; c < VN; ++c)
        if ((flags >> (u * VN + c)) & 1u) e[base + c] = T(0);
    }
  }

  if (ACCUM) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
    if (lane == 0) s_norm[warp] = nrm;
  }

  if (sel_tile) {
    // per (u, warp) counts and intra-warp exclusive prefixes
    const uint32_t lt = (1u << lane) - 1u;
    uint32_t lane_pre[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint32_t cnt = __popc((flags >> (u * VN)) & ((1u << VN) - 1u));
      const uint32_t b0 = __ballot_sync(0xffffffffu, cnt & 1u);
      const uint32_t b1 = __ballot_sync(0xffffffffu, cnt & 2u);
      const uint32_t b2 = __ballot_sync(0xffffffffu, cnt & 4u);
      lane_pre[u] = __popc(b0 & lt) + 2u * __popc(b1 & lt) + 4u * __popc(b2 & lt);
      if (lane == 0) s_off[u * kWarps + warp] = __popc(b0) + 2 * __popc(b1) + 4 * __popc(b2);
    }
    __syncthreads();
    if (warp == 0) {
      // exclusive scan of the 32 (u, warp) partials in (u, warp) order
      const int x = s_off[lane];
      int incl = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      s_off[lane] = incl - x;
      const uint32_t total = (uint32_t)__shfl_sync(0xffffffffu, incl, 31);
      // decoupled look-back over the partition's tiles
      const int first = (int)(st / TILE);
      const int sidx = tile - first;
      const uint32_t epoch = ctrl->epoch;
      unsigned long long* status = a.status;
      uint32_t prefix = 0;
      if (sidx == 0) {
        if (lane == 0) st_relaxed(&status[0], pack_status(epoch, kIncl, total));
      } else {
        if (lane == 0) st_relaxed(&status[sidx], pack_status(epoch, kAgg, total));
        int look = sidx - 1;
        while (true) {
          const int idx = look - lane;
          unsigned long long w = idx >= 0 ? ld_relaxed(&status[idx]) : pack_status(epoch, kIncl, 0);
          auto ok = [&](unsigned long long s) {
            return (uint32_t)(s >> 34) == (epoch & 0x3fffffffu) && ((s >> 32) & 3u) != 0u;
          };
          while (!__all_sync(0xffffffffu, ok(w))) {
            if (!ok(w)) w = ld_relaxed(&status[idx]);
          }
          const uint32_t incl_mask = __ballot_sync(0xffffffffu, ((w >> 32) & 3u) == kIncl);
          const uint32_t val = (uint32_t)w;
          if (incl_mask) {
            const int stop = __ffs(incl_mask) - 1;
            uint32_t s = lane <= stop ? val : 0u;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            prefix += s;
            break;
          }
          uint32_t s = val;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
          prefix += s;
          look -= 32;
        }
        if (lane == 0) st_relaxed(&status[sidx], pack_status(epoch, kIncl, prefix + total));
      }
      if (lane == 0) {
        s_prefix = prefix;
        if (tend >= end) ctrl->k_local = (int64_t)prefix + total;  // last tile of the partition
        // per-block counts (build diagnostic): one atomic when the tile's
        // slice of the partition lies inside one ExDyna block
        const int64_t sz_blk = ctrl->plan.topo.sz_blk;
        const int64_t lo = tbeg > st ? tbeg : st;
        const int64_t hi = (tend < end ? tend : end) - 1;
        int64_t b_lo = lo / sz_blk, b_hi = hi / sz_blk;
        if (b_lo > rc.n_b - 1) b_lo = rc.n_b - 1;
        if (b_hi > rc.n_b - 1) b_hi = rc.n_b - 1;
        if (b_lo == b_hi && total) atomicAdd(&a.blk_counts[b_lo], (int)total);
        s_split = b_lo != b_hi;
      }
      __syncwarp();
    }
    __syncthreads();
    const bool split_blocks = s_split;

    if (flags) {
      const uint32_t prefix = s_prefix;
      T* val = static_cast<T*>(a.val);
      T* x = static_cast<T*>(a.x);
      const int64_t sz_blk = ctrl->plan.topo.sz_blk;
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        uint32_t pos = prefix + (uint32_t)s_off[u * kWarps + warp] + lane_pre[u];
        const int64_t base = tbeg + ((int64_t)u * kThreads + tid) * VN;
#pragma unroll
        for (int c = 0; c < VN; ++c) {
          if ((flags >> (u * VN + c)) & 1u) {
            const int64_t j = base + c;
            a.idx[pos] = (int32_t)j;
            val[pos] = v[u][c];
            if (FUSED) x[j] = apply_update<T>(x[j], v[u][c], rc.n);
            if (split_blocks) {
              int64_t b = j / sz_blk;
              if (b > rc.n_b - 1) b = rc.n_b - 1;
              atomicAdd(&a.blk_counts[b], 1);
            }
            ++pos;
          }
        }
      }
    }
  } else if (ACCUM) {
    __syncthreads();
  }

  if (ACCUM && tid == 0) {
    double s = 0.0;
    for (int w = 0; w < kWarps; ++w) s += s_norm[w];
    a.tile_norm[tile] = s;
  }

  // completion: the last CTA reduces the norm partials in a fixed order and
  // runs the epilogue, then re-arms the ticket for the next launch
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(&ctrl->done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (ACCUM) {
    // fixed-order reduction: thread i sums tiles i, i+256, ... then a fixed tree
    __shared__ double s_red[kThreads];
    const int nt = (int)((n_g + TILE - 1) / TILE);
    double s = 0.0;
    for (int i = tid; i < nt; i += kThreads) s += a.tile_norm[i];
    s_red[tid] = s;
    __syncthreads();
    for (int o = kThreads / 2; o > 0; o >>= 1) {
      if (tid < o) s_red[tid] += s_red[tid + o];
      __syncthreads();
    }
    if (tid == 0) ctrl->norm2 = s_red[0];
  }
  if (tid == 0) {
    if (SELECT) {
      if (end <= st) ctrl->k_local = 0;
      a.cnt_out->k = ctrl->k_local;
      a.cnt_out->norm2 = ctrl->norm2;
      ctrl->epoch = ctrl->epoch + 1 == 0x40000000u ? 1u : ctrl->epoch + 1;
    }
    if (FUSED) control_epilogue(ctrl, a.cnt_out, rc, a.rec);
    ctrl->ticket = 0;
    ctrl->done = 0;
    __threadfence();
  }
}

template <typename T>
cudaError_t launch_select_t(int mode, SelectArgs a, RunConst rc, cudaStream_t s) {
  const dim3 grid(a.num_tiles), block(kThreads);
  const bool fused = rc.n == 1;
  switch (mode) {
    case kFused:
      if (fused) select_kernel<T, kFused, true><<<grid, block, 0, s>>>(a, rc);
      else select_kernel<T, kFused, false><<<grid, block, 0, s>>>(a, rc);
      break;
    case kAccumulate:
      select_kernel<T, kAccumulate, false><<<grid, block, 0, s>>>(a, rc);
      break;
    default:
      if (fused) select_kernel<T, kSelectOnly, true><<<grid, block, 0, s>>>(a, rc);
      else select_kernel<T, kSelectOnly, false><<<grid, block, 0, s>>>(a, rc);
  }
  return cudaGetLastError();
}

// ---- initial plan (t = 0) ---------------------------------------------------
__global__ void plan_kernel(Ctrl* c, RunConst rc) {
  if (threadIdx.x == 0 && blockIdx.x == 0) make_plan(c, rc);
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
  if (blockIdx.x == 0 && threadIdx.x == 0) control_epilogue(a.ctrl, a.counts, rc, a.rec);
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
// The |v| bit patterns order like unsigned integers; 8-bit digits MSB first.
struct QState {
  unsigned long long prefix, mask;
  long long rank;
  unsigned int hist[256];
};

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

template <typename T>
__global__ void __launch_bounds__(256) quantile_hist_kernel(const T* v, int64_t m, QState* q,
                                                            int shift) {
  __shared__ unsigned int h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const unsigned long long prefix = q->prefix, mask = q->mask;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long b = Bits<T>::abs_bits(v[i]);
    if ((b & mask) == prefix) atomicAdd(&h[(b >> shift) & 0xffu], 1u);
  }
  __syncthreads();
  if (h[threadIdx.x]) atomicAdd(&q->hist[threadIdx.x], h[threadIdx.x]);
}

__global__ void quantile_pick_kernel(QState* q, int shift) {
  if (threadIdx.x != 0) return;
  long long r = q->rank;
  int d = 0;
  for (; d < 256; ++d) {
    if (r < (long long)q->hist[d]) break;
    r -= q->hist[d];
  }
  q->rank = r;
  q->prefix |= (unsigned long long)d << shift;
  q->mask |= 0xffULL << shift;
  for (int i = 0; i < 256; ++i) q->hist[i] = 0;
}

template <typename T>
__global__ void quantile_init_kernel(QState* q, int64_t pos) {
  if (threadIdx.x != 0) return;
  q->prefix = 0;
  q->mask = 0;
  q->rank = pos;
  for (int i = 0; i < 256; ++i) q->hist[i] = 0;
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
  quantile_init_kernel<T><<<1, 32, 0, s>>>(q, pos);
  int64_t blocks = (m + 255) / 256;
  if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
  if (blocks < 1) blocks = 1;
  for (int shift = Bits<T>::W - 8; shift >= 0; shift -= 8) {
    quantile_hist_kernel<T><<<(unsigned)blocks, 256, 0, s>>>(v, m, q, shift);
    quantile_pick_kernel<<<1, 32, 0, s>>>(q, shift);
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

int tile_elems(int dtype) { return dtype == EXD_F64 ? tile_of<double>() : tile_of<float>(); }

int64_t num_tiles(int64_t n_g, int dtype) {
  const int t = tile_elems(dtype);
  return (n_g + t - 1) / t;
}

cudaError_t launch_plan(Ctrl* ctrl, RunConst rc, cudaStream_t s) {
  plan_kernel<<<1, 32, 0, s>>>(ctrl, rc);
  return cudaGetLastError();
}

cudaError_t launch_select(int mode, SelectArgs a, RunConst rc, cudaStream_t s) {
  return rc.dtype == EXD_F64 ? launch_select_t<double>(mode, a, rc, s)
                             : launch_select_t<float>(mode, a, rc, s);
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

cudaError_t launch_set_delta(Ctrl* const* ctrls, int nctrl, const void* bits, int dtype,
                             cudaStream_t s) {
  if (dtype == EXD_F64) set_delta_kernel<double><<<1, 32, 0, s>>>(ctrls, nctrl, bits);
  else set_delta_kernel<float><<<1, 32, 0, s>>>(ctrls, nctrl, bits);
  return cudaGetLastError();
}

size_t quantile_scratch_bytes() { return sizeof(QState); }

cudaError_t launch_quantile(const void* v, int64_t m, int64_t pos, int dtype, void* scratch,
                            void* out_bits, cudaStream_t s) {
  QState* q = static_cast<QState*>(scratch);
  if (dtype == EXD_F64)
    return quantile_t<double>(static_cast<const double*>(v), m, pos, q,
                              static_cast<double*>(out_bits), s);
  return quantile_t<float>(static_cast<const float*>(v), m, pos, q, static_cast<float*>(out_bits), s);
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
