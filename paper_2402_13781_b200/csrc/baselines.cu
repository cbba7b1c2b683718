// Baseline sparsifiers of the reference on the device:
//   topk_select            baselines.cpp:26-41  (exact top-k by |acc|, ascending
//                                                indices, ties toward the lower index)
//   hard_threshold_select  baselines.cpp:43-46  (|acc| >= fixed_delta over [0, n_g))
//
// Both are one ordered stream compaction over the full vector, HBM-bound:
//   count  per tile (8192 f32 / 4096 f64 elements): #strict (|a| above the cut) and #tie (|a| at it)
//   scan   one CTA: exclusive tile offsets and the totals, need = k - #strict
//   emit   per tile: re-read, block scan of packed {strict, tie} thread counts,
//          element j is kept when strict, or tie with fewer than `need` ties
//          before it; it lands at (#strict before j) + min(#tie before j, need)
// Top-k first finds the cut, the k-th largest |acc|, with the K8 radix select
// (launch_quantile, ascending position n_g - k). Hard threshold has no tie
// class: strict = (double)|a| >= delta, the reference's comparison in fp64.
// Algorithmic bytes: 2 reads of acc (count + emit) + 4 B per kept index
// (+ 3 or 6 radix passes over acc for top-k).
#include <cuda_runtime.h>
#include <stdint.h>

#include "exdyna.h"
#include "internal.cuh"

namespace exd {
namespace {

constexpr int kBlThreads = 256;
constexpr int kBlSlots = 8;  // 128-bit slots per thread per tile (128 B in flight per thread)
constexpr int kBlTileMin = kBlThreads * kBlSlots * 2;  // elements per tile, f64 (f32: 2x)

template <typename T> struct AbsBits;
template <> struct AbsBits<float> {
  __device__ static unsigned long long of(float v) { return __float_as_uint(v) & 0x7fffffffu; }
};
template <> struct AbsBits<double> {
  __device__ static unsigned long long of(double v) {
    return (unsigned long long)__double_as_longlong(v) & 0x7fffffffffffffffULL;
  }
};

struct Cut {
  int topk;                  // 1: strict = bits > cut, tie = bits == cut; 0: |a| >= delta
  double delta;
  const void* cut_bits;      // device: |value| bits of the k-th largest (top-k)
  int vec;                   // acc is 16-byte aligned: 128-bit loads (else scalar)
};

// Layout of one tile: warp w owns the contiguous 32*PER elements (1024 f32 /
// 512 f64); inside it, 128-bit slot i of lane l holds elements
// i*(32*V) + l*V + [0, V) (V = 4 f32 / 2 f64), so every load instruction of a
// warp reads 512 contiguous bytes. Index order inside a warp chunk is
// (slot, lane, component).
template <typename T> struct Lay {
  static constexpr int V = 16 / (int)sizeof(T);   // elements per 128-bit slot
  static constexpr int S = kBlSlots;              // slots per thread
  static constexpr int PER = S * V;               // elements per thread
  static constexpr int TILE = kBlThreads * PER;   // 8192 f32 / 4096 f64
};

// per-slot packed {strict (low 16 bits), tie (high 16 bits)} counts; flags
// hold 2 bits per element (bit 0 strict, bit 1 tie) in (slot, component) order
template <typename T>
__device__ __forceinline__ void classify(const T* acc, int64_t n_g, int64_t wbase, const Cut& c,
                                         unsigned long long cut, uint32_t (&pc)[Lay<T>::S],
                                         unsigned long long* flags) {
  constexpr int V = Lay<T>::V, S = Lay<T>::S;
  const int lane = threadIdx.x & 31;
  T r[Lay<T>::PER];
  if (c.vec && wbase + 32 * Lay<T>::PER <= n_g) {
    const int4* p = reinterpret_cast<const int4*>(acc + wbase) + lane;
#pragma unroll
    for (int i = 0; i < S; ++i) reinterpret_cast<int4*>(r)[i] = __ldg(p + 32 * i);
  } else {
#pragma unroll
    for (int i = 0; i < S; ++i)
#pragma unroll
      for (int q = 0; q < V; ++q) {
        const int64_t j = wbase + i * 32 * V + lane * V + q;
        r[i * V + q] = j < n_g ? acc[j] : (T)0;
      }
  }
  unsigned long long f = 0;
#pragma unroll
  for (int i = 0; i < S; ++i) {
    uint32_t packed = 0;
#pragma unroll
    for (int q = 0; q < V; ++q) {
      const int64_t j = wbase + i * 32 * V + lane * V + q;
      if (j < n_g) {
        const T v = r[i * V + q];
        uint32_t st, ti;
        if (c.topk) {
          const unsigned long long b = AbsBits<T>::of(v);
          st = b > cut;
          ti = b == cut;
        } else {
          st = (double)(v < (T)0 ? -v : v) >= c.delta;
          ti = 0;
        }
        f |= (unsigned long long)(st | (ti << 1)) << (2 * (i * V + q));
        packed += st + (ti << 16);
      }
    }
    pc[i] = packed;
  }
  *flags = f;
}

template <typename T>
__device__ __forceinline__ unsigned long long load_cut(const Cut& c) {
  if (!c.topk) return 0;
  if (sizeof(T) == 4) return *static_cast<const uint32_t*>(c.cut_bits);
  return *static_cast<const unsigned long long*>(c.cut_bits);
}

// block-wide exclusive scan of one packed word per thread; *total gets the sum
__device__ __forceinline__ uint32_t block_exclusive(uint32_t v, uint32_t* total) {
  __shared__ uint32_t warp_sum[kBlThreads / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sum[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t s = lane < kBlThreads / 32 ? warp_sum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < kBlThreads / 32) warp_sum[lane] = s;
  }
  __syncthreads();
  const uint32_t before = (w ? warp_sum[w - 1] : 0) + x - v;
  *total = warp_sum[kBlThreads / 32 - 1];
  return before;
}

template <typename T>
__global__ void __launch_bounds__(kBlThreads) bl_count_kernel(const T* __restrict__ acc, int64_t n_g,
                                                             Cut c, uint32_t* tile_counts) {
  const unsigned long long cut = load_cut<T>(c);
  const int64_t wbase = (int64_t)blockIdx.x * Lay<T>::TILE + (int64_t)(threadIdx.x >> 5) * 32 * Lay<T>::PER;
  unsigned long long f;
  uint32_t pc[Lay<T>::S];
  classify<T>(acc, n_g, wbase, c, cut, pc, &f);
  uint32_t mine = 0;
#pragma unroll
  for (int i = 0; i < Lay<T>::S; ++i) mine += pc[i];
  uint32_t total;
  block_exclusive(mine, &total);
  if (threadIdx.x == 0) tile_counts[blockIdx.x] = total;
}

// totals[0] = #strict, totals[1] = #tie, totals[2] = need (ties kept)
__global__ void __launch_bounds__(1024) bl_scan_kernel(const uint32_t* tile_counts, int64_t tiles,
                                                       int64_t k, int topk, int64_t* offs_strict,
                                                       int64_t* offs_tie, int64_t* totals) {
  __shared__ long long ws[32], wt[32];
  __shared__ long long carry_s, carry_t;
  if (threadIdx.x == 0) carry_s = carry_t = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t b = 0; b < tiles; b += 1024) {
    const int64_t i = b + threadIdx.x;
    const uint32_t p = i < tiles ? tile_counts[i] : 0;
    long long s = p & 0xffffu, t = p >> 16, xs = s, xt = t;
    for (int o = 1; o < 32; o <<= 1) {
      const long long ys = __shfl_up_sync(0xffffffffu, xs, o);
      const long long yt = __shfl_up_sync(0xffffffffu, xt, o);
      if (lane >= o) { xs += ys; xt += yt; }
    }
    if (lane == 31) { ws[w] = xs; wt[w] = xt; }
    __syncthreads();
    if (w == 0) {
      long long a = ws[lane], bt = wt[lane];
      for (int o = 1; o < 32; o <<= 1) {
        const long long ya = __shfl_up_sync(0xffffffffu, a, o);
        const long long yb = __shfl_up_sync(0xffffffffu, bt, o);
        if (lane >= o) { a += ya; bt += yb; }
      }
      ws[lane] = a;
      wt[lane] = bt;
    }
    __syncthreads();
    const long long ps = carry_s + (w ? ws[w - 1] : 0) + xs - s;
    const long long pt = carry_t + (w ? wt[w - 1] : 0) + xt - t;
    if (i < tiles) {
      offs_strict[i] = ps;
      offs_tie[i] = pt;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      carry_s += ws[31];
      carry_t += wt[31];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    totals[0] = carry_s;
    totals[1] = carry_t;
    long long need = topk ? k - carry_s : 0;
    if (need < 0) need = 0;
    if (need > carry_t) need = carry_t;
    totals[2] = need;
  }
}

template <typename T>
__global__ void __launch_bounds__(kBlThreads) bl_emit_kernel(const T* __restrict__ acc, int64_t n_g,
                                                            Cut c, const int64_t* offs_strict,
                                                            const int64_t* offs_tie,
                                                            const int64_t* totals, int32_t* out,
                                                            int64_t cap) {
  constexpr int V = Lay<T>::V, S = Lay<T>::S;
  const unsigned long long cut = load_cut<T>(c);
  // the tile's offsets are loaded with the data, not after the scans
  const long long need = totals[2];
  const long long s0 = offs_strict[blockIdx.x], t0 = offs_tie[blockIdx.x];
  const int lane = threadIdx.x & 31;
  const int64_t wbase = (int64_t)blockIdx.x * Lay<T>::TILE + (int64_t)(threadIdx.x >> 5) * 32 * Lay<T>::PER;
  unsigned long long f;
  uint32_t pc[S];
  classify<T>(acc, n_g, wbase, c, cut, pc, &f);
  // per slot: lane-exclusive prefix inside the warp and the slot's warp total
  uint32_t excl[S], wsum = 0;
#pragma unroll
  for (int i = 0; i < S; ++i) {
    uint32_t x = pc[i];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    excl[i] = wsum + x - pc[i];
    wsum += __shfl_sync(0xffffffffu, x, 31);
  }
  // warps in order: lane 0 carries the warp's total into the block scan
  uint32_t total;
  const uint32_t wb = __shfl_sync(0xffffffffu, block_exclusive(lane == 0 ? wsum : 0u, &total), 0);
  if (f == 0) return;
  // walk only the set flag bits, in element order (bit 2q: strict, 2q+1: tie)
#pragma unroll
  for (int i = 0; i < S; ++i) {
    uint32_t sb = (uint32_t)(f >> (2 * i * V)) & ((1u << (2 * V)) - 1u);
    if (sb == 0) continue;
    const uint32_t before = wb + excl[i];
    long long s = s0 + (before & 0xffffu);
    long long t = t0 + (before >> 16);
    const int64_t jbase = wbase + i * 32 * V + lane * V;
    while (sb) {
      const int b = __ffs(sb) - 1;
      sb &= sb - 1;
      long long pos = -1;
      if (b & 1) {
        if (t < need) pos = s + t;
        ++t;
      } else {
        pos = s + (t < need ? t : need);
        ++s;
      }
      if (pos >= 0 && pos < cap) out[pos] = (int32_t)(jbase + (b >> 1));
    }
  }
}

template <typename T>
cudaError_t baseline_select_t(const T* acc, int64_t n_g, const Cut& c, int64_t k, int32_t* out,
                              int64_t cap, int64_t* totals_dev, void* scratch, cudaStream_t s) {
  const int64_t tiles = (n_g + Lay<T>::TILE - 1) / Lay<T>::TILE;
  uint32_t* tile_counts = static_cast<uint32_t*>(scratch);
  int64_t* offs_strict = reinterpret_cast<int64_t*>(
      static_cast<char*>(scratch) + ((tiles * 4 + 15) / 16) * 16);
  int64_t* offs_tie = offs_strict + tiles;
  bl_count_kernel<T><<<(unsigned)tiles, kBlThreads, 0, s>>>(acc, n_g, c, tile_counts);
  bl_scan_kernel<<<1, 1024, 0, s>>>(tile_counts, tiles, k, c.topk, offs_strict, offs_tie,
                                    totals_dev);
  bl_emit_kernel<T><<<(unsigned)tiles, kBlThreads, 0, s>>>(acc, n_g, c, offs_strict, offs_tie,
                                                          totals_dev, out, cap);
  return cudaGetLastError();
}

}  // namespace

size_t baseline_scratch_bytes(int64_t n_g) {
  const int64_t tiles = (n_g + kBlTileMin - 1) / kBlTileMin;  // the f64 tiling is the finer
  return (size_t)(((tiles * 4 + 15) / 16) * 16 + tiles * 16) + quantile_scratch_bytes() + 64;
}

// topk: cut = |acc| at ascending position n_g - k (the k-th largest);
// otherwise |acc| >= delta. scratch: baseline_scratch_bytes(n_g) device bytes;
// totals_dev: 3 int64 {#strict, #tie, ties kept}.
cudaError_t launch_baseline_select(const void* acc, int64_t n_g, int dtype, int topk, int64_t k,
                                   double delta, int32_t* out, int64_t cap, int64_t* totals_dev,
                                   void* scratch, cudaStream_t s) {
  Cut c{topk, delta, nullptr, (reinterpret_cast<uintptr_t>(acc) & 15u) == 0 ? 1 : 0};
  char* base = static_cast<char*>(scratch);
  char* qscratch = base + (baseline_scratch_bytes(n_g) - quantile_scratch_bytes() - 64);
  char* cut_bits = qscratch + quantile_scratch_bytes();
  if (topk) {
    cudaError_t e = launch_quantile(acc, n_g, n_g - k, dtype, qscratch, cut_bits, s);
    if (e != cudaSuccess) return e;
    c.cut_bits = cut_bits;
  }
  return dtype == EXD_F64
             ? baseline_select_t<double>(static_cast<const double*>(acc), n_g, c, k, out, cap,
                                         totals_dev, scratch, s)
             : baseline_select_t<float>(static_cast<const float*>(acc), n_g, c, k, out, cap,
                                        totals_dev, scratch, s);
}

}  // namespace exd
