// tools/nvl_word_bench.cu — NVLink ceiling of the push-reduce protocol's
// posted stores: one kernel on GPU 0 stores {payload, epoch} words into a
// buffer on GPU 1 (peer access on, one process), as the exchange kernel does
// with contributions, and the time gives the link rate for that store shape.
// Run alone for the rate; run under ncu with nvltx__bytes.sum for the link
// bytes per launch (the peer-memory sync kernels themselves wait on other
// processes and could not be captured here).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/nvl_word_bench tools/nvl_word_bench.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e_ = (x);                                                  \
    if (e_ != cudaSuccess) {                                               \
      std::printf("%s: %s\n", #x, cudaGetErrorString(e_));                 \
      std::exit(1);                                                        \
    }                                                                      \
  } while (0)

// mode 0: one 8 B word per thread per iteration (st.relaxed.sys.u64)
// mode 1: two words per thread per iteration as one 16 B store (st.relaxed.sys.v2.u64)
// mode 2: short runs like the stream kernel's pushes: each warp writes `run`
//         consecutive words at the start of every 512-word chunk it owns
__global__ void push_words(unsigned long long* dst, long long nwords, unsigned ep, int mode,
                           int run) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  const unsigned long long tag = (unsigned long long)ep << 32;
  if (mode == 2) {
    const int lane = threadIdx.x & 31;
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = stride >> 5;
    for (long long c = warp; c * 512 < nwords; c += nwarps)
      if (lane < run)
        asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(dst + c * 512 + lane),
                     "l"(tag | (unsigned)lane) : "memory");
    return;
  }
  if (mode == 0) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nwords; i += stride)
      asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(dst + i), "l"(tag | (unsigned)i)
                   : "memory");
  } else {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; 2 * i + 1 < nwords;
         i += stride)
      asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1, %2};" ::"l"(dst + 2 * i),
                   "l"(tag | (unsigned)(2 * i)), "l"(tag | (unsigned)(2 * i + 1))
                   : "memory");
  }
}

int main(int argc, char** argv) {
  const long long mb = argc > 1 ? atoll(argv[1]) : 512;
  const long long nwords = mb * (1 << 20) / 8;
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) {
    std::printf("needs 2 GPUs\n");
    return 1;
  }
  int can = 0;
  CK(cudaDeviceCanAccessPeer(&can, 0, 1));
  if (!can) {
    std::printf("no peer access 0 -> 1\n");
    return 1;
  }
  unsigned long long* remote = nullptr;
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&remote, nwords * 8));
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  int sms = 148;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  for (int mode = 0; mode < 2; ++mode) {
    for (int per_sm : {2, 4, 8}) {
      float best = 1e30f;
      for (int rep = 0; rep < 6; ++rep) {
        CK(cudaEventRecord(a));
        push_words<<<sms * per_sm, 256>>>(remote, nwords, rep + 1, mode, 0);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, a, b));
        if (rep > 0 && ms < best) best = ms;
      }
      std::printf("mode=%s blocks/SM=%d: %lld MB of words in %.3f ms = %.1f GB/s (%.1f%% of 770)\n",
                  mode ? "v2.u64 (16 B)" : "u64 (8 B)", per_sm, mb, best,
                  nwords * 8 / (best * 1e-3) / 1e9, nwords * 8 / (best * 1e-3) / 770e9 * 100);
    }
  }
  // short runs: the same chunk grid, `run` words written per 512-word chunk
  for (int run : {1, 5, 16, 32}) {
    for (int local = 0; local < 2; ++local) {
      unsigned long long* dst = remote;
      unsigned long long* loc = nullptr;
      if (local) {
        CK(cudaMalloc(&loc, nwords * 8));
        dst = loc;
      }
      float best = 1e30f;
      for (int rep = 0; rep < 6; ++rep) {
        CK(cudaEventRecord(a));
        push_words<<<sms * 4, 256>>>(dst, nwords, rep + 1, 2, run);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, a, b));
        if (rep > 0 && ms < best) best = ms;
      }
      const double nruns = (double)(nwords / 512);
      std::printf("runs of %2d words per 512-word chunk to %s: %.0f runs in %.3f ms = %.1f M runs/s, %.1f GB/s of words\n",
                  run, local ? "LOCAL memory" : "the peer", nruns, best, nruns / (best * 1e-3) / 1e6,
                  nruns * run * 8 / (best * 1e-3) / 1e9);
      if (loc) cudaFree(loc);
    }
  }
  return 0;
}
