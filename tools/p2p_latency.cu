// tools/p2p_latency.cu — NVLink flag round-trip latency between two GPUs with
// the primitives the peer-memory sync uses (one process, peer access on).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/p2p_latency tools/p2p_latency.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); exit(1);} } while (0)

__device__ __forceinline__ unsigned long long ld_relaxed_sys(const unsigned long long* p) {
  unsigned long long v; asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v; asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }

// mode 0: remote st.release.sys, local ld.relaxed.sys polling
// mode 1: remote st.relaxed.sys, local ld.relaxed.sys polling
// mode 2: __threadfence_system + remote st.relaxed.sys
// mode 3: remote volatile store, local volatile poll
// mode 4: local store, REMOTE polling (pull model)
__global__ void pingpong(unsigned long long* my_flag, unsigned long long* peer_flag, int iters, int first, int mode,
                         unsigned long long* out) {
  if (threadIdx.x != 0) return;
  unsigned long long t0 = gt();
  for (int i = 1; i <= iters; ++i) {
    if (first) {
      if (mode == 0) st_release_sys(peer_flag, i);
      else if (mode == 1) st_relaxed_sys(peer_flag, i);
      else if (mode == 2) { __threadfence_system(); st_relaxed_sys(peer_flag, i); }
      else if (mode == 3) *(volatile unsigned long long*)peer_flag = i;
      else st_relaxed_sys(my_flag, i);
      if (mode == 4) { while (ld_relaxed_sys(peer_flag) < (unsigned long long)i) {} }
      else if (mode == 3) { while (*(volatile unsigned long long*)my_flag < (unsigned long long)i) {} }
      else { while (ld_relaxed_sys(my_flag) < (unsigned long long)i) {} }
    } else {
      if (mode == 4) { while (ld_relaxed_sys(peer_flag) < (unsigned long long)i) {} }
      else if (mode == 3) { while (*(volatile unsigned long long*)my_flag < (unsigned long long)i) {} }
      else { while (ld_relaxed_sys(my_flag) < (unsigned long long)i) {} }
      if (mode == 0) st_release_sys(peer_flag, i);
      else if (mode == 1) st_relaxed_sys(peer_flag, i);
      else if (mode == 2) { __threadfence_system(); st_relaxed_sys(peer_flag, i); }
      else if (mode == 3) *(volatile unsigned long long*)peer_flag = i;
      else st_relaxed_sys(my_flag, i);
    }
  }
  *out = gt() - t0;
}

// cost of fences alone
__global__ void fences(int iters, int kind, unsigned long long* out, unsigned long long* scratch) {
  if (threadIdx.x != 0) return;
  unsigned long long t0 = gt();
  for (int i = 0; i < iters; ++i) {
    scratch[i & 63] = i;
    if (kind == 0) __threadfence();
    else if (kind == 1) __threadfence_system();
    else asm volatile("fence.acq_rel.sys;" ::: "memory");
  }
  *out = gt() - t0;
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) { printf("need 2 GPUs\n"); return 0; }
  unsigned long long *f0, *f1, *o0, *o1;
  CK(cudaSetDevice(0)); CK(cudaDeviceEnablePeerAccess(1, 0)); CK(cudaMalloc(&f0, 4096)); CK(cudaMalloc(&o0, 64));
  CK(cudaSetDevice(1)); CK(cudaDeviceEnablePeerAccess(0, 0)); CK(cudaMalloc(&f1, 4096)); CK(cudaMalloc(&o1, 64));
  const int iters = 2000;
  const char* names[] = {"release.sys store / relaxed poll", "relaxed.sys store / relaxed poll",
                         "threadfence_system + relaxed store", "volatile store / volatile poll",
                         "local store / REMOTE poll"};
  for (int mode = 0; mode < 5; ++mode) {
    CK(cudaSetDevice(0)); CK(cudaMemset(f0, 0, 4096));
    CK(cudaSetDevice(1)); CK(cudaMemset(f1, 0, 4096));
    CK(cudaDeviceSynchronize()); CK(cudaSetDevice(0)); CK(cudaDeviceSynchronize());
    CK(cudaSetDevice(1));
    pingpong<<<1, 32>>>(f1, f0, iters, 0, mode, o1);
    CK(cudaSetDevice(0));
    pingpong<<<1, 32>>>(f0, f1, iters, 1, mode, o0);
    CK(cudaDeviceSynchronize()); CK(cudaSetDevice(1)); CK(cudaDeviceSynchronize());
    unsigned long long t;
    CK(cudaSetDevice(0)); CK(cudaMemcpy(&t, o0, 8, cudaMemcpyDeviceToHost));
    printf("%-40s round trip %.2f us\n", names[mode], t / 1e3 / iters);
  }
  CK(cudaSetDevice(0));
  const char* fn[] = {"__threadfence (gpu)", "__threadfence_system", "fence.acq_rel.sys"};
  for (int k = 0; k < 3; ++k) {
    fences<<<1, 32>>>(10000, k, o0, f0 + 64);
    CK(cudaDeviceSynchronize());
    unsigned long long t;
    CK(cudaMemcpy(&t, o0, 8, cudaMemcpyDeviceToHost));
    printf("%-40s %.3f us each\n", fn[k], t / 1e3 / 10000);
  }
  return 0;
}
