// Engine runs of the reference's baseline sparsifiers:
// Top-k, CLT-k and hard threshold through Engine::step (engine.cpp:163-204,
// 274-350). Unlike ExDyna, their selections overlap across workers, so the
// union is deduplicated (collectives.cpp:47-55: sort + unique):
//
//   select   every worker (CLT-k: only the cyclic leader, baselines.hpp:37-39)
//            runs the device selector (baselines.cu) over its full |acc|
//   counts   {k_i, ||e_entering||^2} per worker from the selector totals
//   union    one bit per index over [0, n_g): every list sets its bits, then
//            an ordered compaction of the bitmap (count / one-CTA scan / emit)
//            gives the ascending, duplicate-free idx_global; the emit clears
//            the bitmap for the next step
//   gather   c_r[pos] = e_r[idx_global[pos]], e_r cleared at the union
//            (engine.cpp:310-317, selector.cpp:63-65)
//   sum      rank-order sum (collectives.cpp:59-70), x -= g / n (engine.cpp:215)
//   record   k_t = k_rank, t + 1; delta stays (no threshold scaling outside
//            ExDyna, engine.cpp:210-212); duplicates = k' - |union|
#include <cuda_runtime.h>
#include <stdint.h>

#include "exdyna.h"
#include "internal.cuh"

namespace exd {
namespace {

constexpr int kT = 256;
constexpr int kWordsPerThread = 32;
constexpr int kWordsPerBlock = kT * kWordsPerThread;  // 8192 words = 262144 indices

int grid_of(int64_t work, int per) {
  int64_t g = (work + per - 1) / per;
  if (g < 1) g = 1;
  if (g > 148 * 16) g = 148 * 16;
  return (int)g;
}

__global__ void __launch_bounds__(kT) bl_counts_kernel(const int64_t* totals, const double* tile_norm,
                                                      int ntiles, CountRec* cnt) {
  __shared__ double red[kT / 32];
  double s = 0.0;
  for (int i = threadIdx.x; i < ntiles; i += kT) s += tile_norm[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < kT / 32; ++w) t += red[w];
    cnt->k = totals ? totals[0] + totals[2] : 0;  // #strict + ties kept
    cnt->norm2 = t;
    cnt->capped = 0;
  }
}

__global__ void __launch_bounds__(kT) bl_bitmap_set_kernel(const int32_t* list, const CountRec* cnt,
                                                          uint32_t* bitmap) {
  const int64_t k = cnt->k;
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < k; i += (int64_t)gridDim.x * kT) {
    const uint32_t j = (uint32_t)list[i];
    atomicOr(&bitmap[j >> 5], 1u << (j & 31));
  }
}

// per block of kWordsPerBlock words: the number of set bits
__global__ void __launch_bounds__(kT) bl_union_count_kernel(const uint32_t* bitmap, int64_t nwords,
                                                           int64_t* blk_cnt) {
  __shared__ int red[kT / 32];
  const int64_t w0 = (int64_t)blockIdx.x * kWordsPerBlock;
  int c = 0;
  for (int i = threadIdx.x; i < kWordsPerBlock; i += kT) {  // coalesced
    const int64_t w = w0 + i;
    if (w < nwords) c += __popc(bitmap[w]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
#pragma unroll
    for (int w = 0; w < kT / 32; ++w) t += red[w];
    blk_cnt[blockIdx.x] = t;
  }
}

// one CTA: exclusive block offsets in place; ucnt->k = |union|
__global__ void __launch_bounds__(1024) bl_union_scan_kernel(int64_t* blk, int64_t nblk,
                                                            CountRec* ucnt) {
  __shared__ long long ws[32];
  __shared__ long long carry;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t b = 0; b < nblk; b += 1024) {
    const int64_t i = b + threadIdx.x;
    const long long v = i < nblk ? blk[i] : 0;
    long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) ws[w] = x;
    __syncthreads();
    if (w == 0) {
      long long s = ws[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += y;
      }
      ws[lane] = s;
    }
    __syncthreads();
    const long long excl = carry + (w ? ws[w - 1] : 0) + x - v;
    if (i < nblk) blk[i] = excl;
    __syncthreads();
    if (threadIdx.x == 0) carry += ws[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    ucnt->k = carry;
    ucnt->norm2 = 0.0;
    ucnt->capped = 0;
  }
}

// ordered emit of the set bits; clears the bitmap behind it
__global__ void __launch_bounds__(kT) bl_union_emit_kernel(uint32_t* bitmap, int64_t nwords,
                                                          const int64_t* blk_off, int32_t* out) {
  __shared__ int ws[kT / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t w0 = (int64_t)blockIdx.x * kWordsPerBlock + (int64_t)threadIdx.x * kWordsPerThread;
  uint32_t bits[kWordsPerThread];
  int mine = 0;
#pragma unroll
  for (int i = 0; i < kWordsPerThread; ++i) {
    bits[i] = w0 + i < nwords ? bitmap[w0 + i] : 0u;
    mine += __popc(bits[i]);
  }
  int x = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[w] = x;
  __syncthreads();
  int wpre = 0;
#pragma unroll
  for (int q = 0; q < kT / 32; ++q) wpre += q < w ? ws[q] : 0;
  int64_t pos = blk_off[blockIdx.x] + wpre + x - mine;
#pragma unroll
  for (int i = 0; i < kWordsPerThread; ++i) {
    uint32_t b = bits[i];
    while (b) {
      const int k = __ffs(b) - 1;
      b &= b - 1;
      out[pos++] = (int32_t)((w0 + i) * 32 + k);
    }
    if (bits[i]) bitmap[w0 + i] = 0u;
  }
}

template <typename T>
__global__ void __launch_bounds__(kT) bl_gather_clear_kernel(const int32_t* uni, const CountRec* ucnt,
                                                            T* e, T* contrib) {
  const int64_t kp = ucnt->k;
  for (int64_t pos = (int64_t)blockIdx.x * kT + threadIdx.x; pos < kp;
       pos += (int64_t)gridDim.x * kT) {
    const int32_t j = uni[pos];
    contrib[pos] = e[j];
    e[j] = T(0);
  }
}

// rank-order sum (collectives.cpp:62-68)
template <typename T>
__global__ void __launch_bounds__(kT) bl_sum_kernel(const void* const* contribs, int n,
                                                   const CountRec* ucnt, T* sum) {
  const int64_t kp = ucnt->k;
  for (int64_t pos = (int64_t)blockIdx.x * kT + threadIdx.x; pos < kp;
       pos += (int64_t)gridDim.x * kT) {
    T s = static_cast<const T*>(contribs[0])[pos];
    for (int r = 1; r < n; ++r) s += static_cast<const T*>(contribs[r])[pos];
    sum[pos] = s;
  }
}

// x -= g / n (engine.cpp:215), fp64 arithmetic rounded once, as apply_update
template <typename T>
__global__ void __launch_bounds__(kT) bl_apply_kernel(const int32_t* uni, const CountRec* ucnt,
                                                     const T* sum, T* x, int n) {
  const int64_t kp = ucnt->k;
  const bool pow2 = (n & (n - 1)) == 0;
  for (int64_t pos = (int64_t)blockIdx.x * kT + threadIdx.x; pos < kp;
       pos += (int64_t)gridDim.x * kT) {
    const int32_t j = uni[pos];
    const double g = (double)sum[pos];
    const double q = pow2 ? __dmul_rn(g, 1.0 / (double)n) : __ddiv_rn(g, (double)n);
    x[j] = (T)__dadd_rn((double)x[j], -q);
  }
}

// the control state and the raw ledger row of one worker
__global__ void bl_epilogue_kernel(Ctrl* c, const CountRec* counts, const CountRec* ucnt,
                                   RawRecord* rec, int n, double delta_used) {
  if (threadIdx.x != 0) return;
  rec->t = c->t;
  rec->delta = delta_used;
  rec->moves = rec->skips = 0;
  rec->n = n;
  rec->reserved = 0;
  for (int r = 0; r < n; ++r) {
    c->k_t[r] = counts[r].k;
    rec->k_rank[r] = counts[r].k;
    rec->norm2[r] = counts[r].norm2;
    rec->capped[r] = 0;
  }
  rec->union_count = ucnt->k;
  c->t += 1;
  c->tmod = c->tmod + 1 == n ? 0 : c->tmod + 1;
}

}  // namespace

size_t baseline_union_scratch_bytes(int64_t n_g) {
  const int64_t nwords = (n_g + 31) / 32;
  const int64_t nblk = (nwords + kWordsPerBlock - 1) / kWordsPerBlock;
  return (size_t)nwords * 4 + (size_t)nblk * 8 + 256;
}

cudaError_t launch_baseline_counts(const int64_t* totals, const double* tile_norm, int ntiles,
                                   CountRec* cnt, cudaStream_t s) {
  bl_counts_kernel<<<1, kT, 0, s>>>(totals, tile_norm, ntiles, cnt);
  return cudaGetLastError();
}

cudaError_t launch_baseline_union(const int32_t* const* lists_host, const CountRec* counts, int n,
                                  int64_t cap, int64_t n_g, void* scratch, int32_t* uni,
                                  CountRec* ucnt, cudaStream_t s) {
  const int64_t nwords = (n_g + 31) / 32;
  const int64_t nblk = (nwords + kWordsPerBlock - 1) / kWordsPerBlock;
  uint32_t* bitmap = static_cast<uint32_t*>(scratch);  // zero between steps (the emit clears it)
  int64_t* blk = reinterpret_cast<int64_t*>(static_cast<char*>(scratch) + ((nwords * 4 + 15) / 16) * 16);
  for (int r = 0; r < n; ++r)
    bl_bitmap_set_kernel<<<grid_of(cap, kT * 4), kT, 0, s>>>(lists_host[r], counts + r, bitmap);
  bl_union_count_kernel<<<(unsigned)nblk, kT, 0, s>>>(bitmap, nwords, blk);
  bl_union_scan_kernel<<<1, 1024, 0, s>>>(blk, nblk, ucnt);
  bl_union_emit_kernel<<<(unsigned)nblk, kT, 0, s>>>(bitmap, nwords, blk, uni);
  return cudaGetLastError();
}

int baseline_union_launches(int n) { return n + 3; }

cudaError_t launch_baseline_gather_clear(const int32_t* uni, const CountRec* ucnt, void* e,
                                         void* contrib, int64_t cap, int dtype, cudaStream_t s) {
  const int g = grid_of(cap, kT * 4);
  if (dtype == EXD_F64)
    bl_gather_clear_kernel<double><<<g, kT, 0, s>>>(uni, ucnt, static_cast<double*>(e),
                                                    static_cast<double*>(contrib));
  else
    bl_gather_clear_kernel<float><<<g, kT, 0, s>>>(uni, ucnt, static_cast<float*>(e),
                                                   static_cast<float*>(contrib));
  return cudaGetLastError();
}

cudaError_t launch_baseline_sum(const void* const* contribs_dev, int n, const CountRec* ucnt,
                                void* sum, int64_t cap, int dtype, cudaStream_t s) {
  const int g = grid_of(cap, kT * 4);
  if (dtype == EXD_F64)
    bl_sum_kernel<double><<<g, kT, 0, s>>>(contribs_dev, n, ucnt, static_cast<double*>(sum));
  else
    bl_sum_kernel<float><<<g, kT, 0, s>>>(contribs_dev, n, ucnt, static_cast<float*>(sum));
  return cudaGetLastError();
}

cudaError_t launch_baseline_apply(const int32_t* uni, const CountRec* ucnt, const void* sum,
                                  void* x, int n, int64_t cap, int dtype, cudaStream_t s) {
  const int g = grid_of(cap, kT * 4);
  if (dtype == EXD_F64)
    bl_apply_kernel<double><<<g, kT, 0, s>>>(uni, ucnt, static_cast<const double*>(sum),
                                             static_cast<double*>(x), n);
  else
    bl_apply_kernel<float><<<g, kT, 0, s>>>(uni, ucnt, static_cast<const float*>(sum),
                                            static_cast<float*>(x), n);
  return cudaGetLastError();
}

cudaError_t launch_baseline_epilogue(Ctrl* ctrl, const CountRec* counts, const CountRec* ucnt,
                                     RawRecord* rec, int n, double delta_used, cudaStream_t s) {
  bl_epilogue_kernel<<<1, 32, 0, s>>>(ctrl, counts, ucnt, rec, n, delta_used);
  return cudaGetLastError();
}

}  // namespace exd
