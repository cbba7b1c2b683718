// tools/stream_bench.cu — microbenchmark of the access pattern of the fused
// select kernel (read g, read e, write e; 12 B/element fp32) on sm_100a, to
// establish the achievable HBM roofline for this mix and compare load paths.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/stream_bench tools/stream_bench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); exit(1);} } while (0)

// (a) grid-stride, float4, U independent vectors in flight per thread
template <int U>
__global__ void __launch_bounds__(256) k_gs(const float4* __restrict__ g, float4* __restrict__ e, long n4, float thr, int* cnt) {
  int c = 0;
  for (long i = (long)blockIdx.x * 256 * U + threadIdx.x; i < n4; i += (long)gridDim.x * 256 * U) {
    float4 a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      long j = i + u * 256;
      if (j < n4) { a[u] = __ldcs(&e[j]); b[u] = __ldcs(&g[j]); }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      long j = i + u * 256;
      if (j < n4) {
        float4 r = make_float4(a[u].x + b[u].x, a[u].y + b[u].y, a[u].z + b[u].z, a[u].w + b[u].w);
        c += (fabsf(r.x) >= thr) + (fabsf(r.y) >= thr) + (fabsf(r.z) >= thr) + (fabsf(r.w) >= thr);
        __stcs(&e[j], r);
      }
    }
  }
  if (c) atomicAdd(cnt, c);
}

// (b) one tile per CTA (4096 floats), like the one-tile select kernel
__global__ void __launch_bounds__(256) k_tile(const float4* __restrict__ g, float4* __restrict__ e, long n4, float thr, int* cnt) {
  long base = (long)blockIdx.x * 1024;
  int c = 0;
  float4 a[4], b[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    long j = base + u * 256 + threadIdx.x;
    if (j < n4) { a[u] = __ldcs(&e[j]); b[u] = __ldcs(&g[j]); }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    long j = base + u * 256 + threadIdx.x;
    if (j < n4) {
      float4 r = make_float4(a[u].x + b[u].x, a[u].y + b[u].y, a[u].z + b[u].z, a[u].w + b[u].w);
      c += (fabsf(r.x) >= thr) + (fabsf(r.y) >= thr) + (fabsf(r.z) >= thr) + (fabsf(r.w) >= thr);
      __stcs(&e[j], r);
    }
  }
  if (c) atomicAdd(cnt, c);
}

// (c) default-cached loads/stores variant of (a)
template <int U>
__global__ void __launch_bounds__(256) k_gs_def(const float4* __restrict__ g, float4* __restrict__ e, long n4, float thr, int* cnt) {
  int c = 0;
  for (long i = (long)blockIdx.x * 256 * U + threadIdx.x; i < n4; i += (long)gridDim.x * 256 * U) {
    float4 a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      long j = i + u * 256;
      if (j < n4) { a[u] = e[j]; b[u] = __ldg(&g[j]); }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      long j = i + u * 256;
      if (j < n4) {
        float4 r = make_float4(a[u].x + b[u].x, a[u].y + b[u].y, a[u].z + b[u].z, a[u].w + b[u].w);
        c += (fabsf(r.x) >= thr) + (fabsf(r.y) >= thr) + (fabsf(r.z) >= thr) + (fabsf(r.w) >= thr);
        e[j] = r;
      }
    }
  }
  if (c) atomicAdd(cnt, c);
}

// (d) persistent, static contiguous ranges, TMA bulk loads into a 3-stage smem ring
__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
template <int STAGES>
__global__ void __launch_bounds__(256, 2) k_tma(const float* __restrict__ g, float* __restrict__ e, long n, int ntiles, float thr, int* cnt) {
  extern __shared__ __align__(128) float sb[];
  __shared__ unsigned long long bar[STAGES];
  const int TILE = 4096;
  int t0 = (int)((long)ntiles * blockIdx.x / gridDim.x), t1 = (int)((long)ntiles * (blockIdx.x + 1) / gridDim.x);
  auto issue = [&](int tile, int s) {
    long tb = (long)tile * TILE; long len = tb + TILE < n ? TILE : n - tb; unsigned bytes = (unsigned)(len * 4) & ~15u;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(sa(&bar[s])), "r"(2 * bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(sa(sb + s * 2 * TILE)), "l"(g + tb), "r"(bytes), "r"(sa(&bar[s])) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(sa(sb + s * 2 * TILE + TILE)), "l"(e + tb), "r"(bytes), "r"(sa(&bar[s])) : "memory");
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < STAGES && t0 + s < t1; ++s) issue(t0 + s, s);
  }
  __syncthreads();
  int c = 0;
  for (int tile = t0, it = 0; tile < t1; ++tile, ++it) {
    int s = it % STAGES; unsigned ph = (it / STAGES) & 1;
    unsigned ok = 0;
    do { asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(ok) : "r"(sa(&bar[s])), "r"(ph) : "memory"); } while (!ok);
    float4 r[4];
    const float4* sg = (const float4*)(sb + s * 2 * TILE); const float4* se = (const float4*)(sb + s * 2 * TILE + TILE);
#pragma unroll
    for (int u = 0; u < 4; ++u) { float4 a = se[u * 256 + threadIdx.x], b = sg[u * 256 + threadIdx.x];
      r[u] = make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w); }
    __syncthreads();
    if (threadIdx.x == 0 && tile + STAGES < t1) issue(tile + STAGES, s);
    float4* eo = (float4*)(e + (long)tile * TILE);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      c += (fabsf(r[u].x) >= thr) + (fabsf(r[u].y) >= thr) + (fabsf(r[u].z) >= thr) + (fabsf(r[u].w) >= thr);
      __stcs(&eo[u * 256 + threadIdx.x], r[u]);
    }
  }
  if (c) atomicAdd(cnt, c);
}

__global__ void k_read(const float4* __restrict__ a, long n4, int* out) {
  float s = 0.f;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) s += a[i].x;
  if (s == 12345.f) atomicAdd(out, 1);
}

__global__ void k_copy(const float4* __restrict__ a, float4* __restrict__ b, long n4) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) b[i] = a[i];
}

int main(int argc, char** argv) {
  long n = argc > 1 ? atol(argv[1]) : 11200000;
  long n4 = n / 4;
  float *g, *e, *fl, *c1, *c2;
  int* cnt;
  size_t fbytes = 512ull << 20;
  CK(cudaMalloc(&g, n * 4)); CK(cudaMalloc(&e, n * 4)); CK(cudaMalloc(&fl, fbytes)); CK(cudaMalloc(&cnt, 4));
  CK(cudaMalloc(&c1, 1ull << 30)); CK(cudaMalloc(&c2, 1ull << 30));
  CK(cudaMemset(g, 0, n * 4)); CK(cudaMemset(e, 0, n * 4));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* name, auto launch, double bytes, bool flush) {
    float best = 1e9, sum = 0; int reps = 20;
    for (int r = 0; r < reps + 3; ++r) {
      if (flush) { CK(cudaMemsetAsync(fl, r, fbytes)); k_copy<<<sms * 8, 256>>>((float4*)fl, (float4*)fl, 0); k_read<<<sms * 8, 256>>>((const float4*)fl, (long)(fbytes / 16), cnt); }
      cudaEventRecord(a); launch(); cudaEventRecord(b); CK(cudaEventSynchronize(b));
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (r >= 3) { best = ms < best ? ms : best; sum += ms; }
    }
    printf("%-28s flush=%d best %8.2f us (%7.0f GB/s)  mean %8.2f us (%7.0f GB/s)\n", name, (int)flush, best * 1e3,
           bytes / best / 1e6, sum / reps * 1e3, bytes / (sum / reps) / 1e6);
  };
  double B = 12.0 * n;
  for (int flush = 0; flush < 2; ++flush) {
    for (int bpsm : {2, 4, 8, 16}) {
      char nm[64];
      snprintf(nm, 64, "gs U=4 grid=%dx148", bpsm);
      run(nm, [&] { k_gs<4><<<sms * bpsm, 256>>>((float4*)g, (float4*)e, n4, 1.f, cnt); }, B, flush);
    }
    run("gs U=8 grid=4x148", [&] { k_gs<8><<<sms * 4, 256>>>((float4*)g, (float4*)e, n4, 1.f, cnt); }, B, flush);
    run("gs U=2 grid=8x148", [&] { k_gs<2><<<sms * 8, 256>>>((float4*)g, (float4*)e, n4, 1.f, cnt); }, B, flush);
    run("gs_def U=4 grid=4x148", [&] { k_gs_def<4><<<sms * 4, 256>>>((float4*)g, (float4*)e, n4, 1.f, cnt); }, B, flush);
    {
      int ntiles = (int)((n + 4095) / 4096);
      size_t sm3 = 3 * 2 * 4096 * 4, sm2 = 2 * 2 * 4096 * 4;
      cudaFuncSetAttribute(k_tma<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm3);
      cudaFuncSetAttribute(k_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
      int occ3 = 0, occ2 = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ3, k_tma<3>, 256, sm3);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, k_tma<2>, 256, sm2);
      char nm[64];
      snprintf(nm, 64, "tma S=3 occ=%d", occ3);
      run(nm, [&] { k_tma<3><<<sms * occ3, 256, sm3>>>(g, e, n, ntiles, 1.f, cnt); }, B, flush);
      snprintf(nm, 64, "tma S=2 occ=%d", occ2);
      run(nm, [&] { k_tma<2><<<sms * occ2, 256, sm2>>>(g, e, n, ntiles, 1.f, cnt); }, B, flush);
    }
    run("tile (1 tile/CTA)", [&] { k_tile<<<(n4 + 1023) / 1024, 256>>>((float4*)g, (float4*)e, n4, 1.f, cnt); }, B, flush);
  }
  long c4 = (1ull << 30) / 16;
  run("copy 1 GiB (read+write)", [&] { k_copy<<<sms * 8, 256>>>((float4*)c1, (float4*)c2, c4); }, 2.0 * (1ull << 30), false);
  return 0;
}
