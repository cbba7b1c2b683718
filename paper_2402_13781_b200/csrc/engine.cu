// engine.cu — host side of the B200 ExDyna path: the sparsim::Engine
// replacement (engine.hpp:61-105) and the C ABI of include/exdyna.h.
//
// Two deployment shapes share every kernel:
//   * in-process workers (exd_engine_create): all n workers of the reference's
//     simulator on one GPU, one stream; collectives are device kernels over
//     the workers' buffers. No host synchronisation inside a step.
//   * one rank per GPU (exd_engine_create_rank): the data-parallel job the
//     paper runs. Collectives are NCCL over NVLink 5 / NVSwitch; the only host
//     wait per step is the 16 B x n count all-gather that sizes the padded
//     index all-gather (SURVEY.md §7 hard part 3).
// Control state (topology, delta, k_t, plan) lives on the device and is
// advanced by the kernels' single-thread epilogue.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <chrono>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include "control.cuh"
#include "exdyna.h"
#include "internal.cuh"

using namespace exd;

namespace {

thread_local std::string g_err;

int set_err(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CU(expr)                                                                   \
  do {                                                                             \
    cudaError_t _e = (expr);                                                       \
    if (_e != cudaSuccess)                                                         \
      return set_err(EXD_ECUDA, std::string(#expr " failed: ") + cudaGetErrorString(_e)); \
  } while (0)

double nccl_timeout_s() {
  static double v = [] {
    const char* e = std::getenv("EXD_NCCL_TIMEOUT_S");
    const double d = e ? std::atof(e) : 0.0;
    return d > 0.0 ? d : 60.0;
  }();
  return v;
}

// ---- validate(), config.cpp:28-51 -----------------------------------------
int validate_cfg(const exd_config* in, exd_config* out) {
  const exd_config c = *in;
  auto bad = [](const char* m) { return set_err(EXD_EINVAL, m); };
  if (c.n < 1) return bad("worker count out of range");
  if (c.n_g < 1) return bad("gradient count out of range");
  if (c.n_b < 1) return bad("block count out of range");
  if (!(c.d > 0.0) || c.d > 1.0) return bad("density out of range");
  if (c.has_delta0 && !(c.delta0 > 0.0)) return bad("delta0 out of range");
  if (!(c.alpha > 1.0)) return bad("alpha out of range");
  if (!(c.beta > 1.0)) return bad("beta out of range");
  if (!(c.gamma > 0.0) || !(c.gamma < 1.0)) return bad("gamma out of range");
  if (c.blk_move < 1) return bad("blk_move out of range");
  if (c.min_blk < 1) return bad("min_blk out of range");
  if (!(c.eta > 0.0)) return bad("eta out of range");
  if (c.has_max_density_cap && (!(c.max_density_cap > 0.0) || c.max_density_cap > 1.0))
    return bad("max_density_cap out of range");
  *out = c;
  out->k = (int64_t)std::llround(c.d * (double)c.n_g);
  if (c.n_b < (int64_t)c.n * c.min_blk) return bad("n_b < n*min_blk");
  if (c.n_b > c.n_g) return bad("n_b > n_g");
  if (out->k < c.n) return bad("k < n");
  return EXD_OK;
}

// ---- build_topology, partition.cpp:22-58 ------------------------------------
int build_topo(int64_t n_g, int64_t n_b, int n, int64_t min_blk, exd_topology* out,
               std::string* warning) {
  if (n < 1 || n > EXD_MAX_WORKERS) return set_err(EXD_EINVAL, "worker count out of range");
  if (n_b < 1 || n_b > n_g) return set_err(EXD_EINVAL, "n_b out of range");
  const int64_t q = n_g / n_b;
  int64_t sz;
  if (q >= 32) {
    sz = q - q % 32;
  } else {
    sz = q > 1 ? q : 1;
    if (warning)
      *warning = "block size " + std::to_string(sz) +
                 " below 32-element alignment; using unaligned blocks";
  }
  const int64_t quo = n_b / n, rem = n_b % n;
  if (quo < min_blk) return set_err(EXD_EINVAL, "partition would hold fewer than min_blk blocks");
  std::memset(out, 0, sizeof(*out));
  out->n = n;
  out->sz_blk = sz;
  for (int i = 0; i < n; ++i) out->blk_part[i] = quo + (i < rem ? 1 : 0);
  for (int i = 1; i < n; ++i) out->blk_pos[i] = out->blk_pos[i - 1] + out->blk_part[i - 1];
  return EXD_OK;
}

// ---- NCCL, loaded on first use so the library has no link-time NCCL -------
struct Nccl {
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclAllGather) AllGather = nullptr;
  decltype(&ncclAllReduce) AllReduce = nullptr;
  decltype(&ncclBroadcast) Broadcast = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
  decltype(&ncclCommGetAsyncError) CommGetAsyncError = nullptr;
  decltype(&ncclCommAbort) CommAbort = nullptr;
  bool ok = false;
  std::string why;
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      n.why = std::string("dlopen libnccl.so.2: ") + dlerror();
      return;
    }
#define SYM(name) n.name = reinterpret_cast<decltype(n.name)>(dlsym(h, "nccl" #name))
    SYM(GetUniqueId);
    SYM(CommInitRank);
    SYM(CommDestroy);
    SYM(AllGather);
    SYM(AllReduce);
    SYM(Broadcast);
    SYM(GetErrorString);
    SYM(CommGetAsyncError);
    SYM(CommAbort);
#undef SYM
    n.ok = n.GetUniqueId && n.CommInitRank && n.CommDestroy && n.AllGather && n.AllReduce &&
           n.Broadcast && n.GetErrorString && n.CommGetAsyncError && n.CommAbort;
    if (!n.ok) n.why = "libnccl.so.2 lacks a required symbol";
  });
  return n;
}

#define NC(expr)                                                                        \
  do {                                                                                  \
    ncclResult_t _r = (expr);                                                           \
    if (_r != ncclSuccess)                                                              \
      return set_err(EXD_ENCCL, std::string(#expr " failed: ") + nccl().GetErrorString(_r)); \
  } while (0)

// IEEE round-toward-+inf of a positive double to float (the host twin of
// __double2float_ru): (double)|acc| >= delta  <=>  |acc| >= round_up(delta).
float round_up_float(double d) {
  float f = (float)d;
  if ((double)f < d) f = std::nextafter(f, INFINITY);
  return f;
}

size_t elem_size(int dtype) { return dtype == EXD_F64 ? 8 : 4; }

// Granlund-Montgomery magic numbers for n / d with 31-bit n: with
// l = ceil(log2 d), s = 31 + l and M = ceil(2^s / d) (<= 2^32),
// floor(n * M / 2^s) == n / d for every n < 2^31, and n * M fits in 64 bits.
void blk_magic(int64_t d, unsigned long long* magic, int32_t* shift) {
  int l = 0;
  while ((1LL << l) < d) ++l;
  const int s = 31 + l;
  const unsigned __int128 p = (unsigned __int128)1 << s;
  *magic = (unsigned long long)((p + (unsigned __int128)(d - 1)) / (unsigned __int128)d);
  *shift = s;
}

// per-step records stay on the device; the host copies the latest at sync
constexpr int64_t kRecRing = EXD_RECORD_RING;

}  // namespace

// ---------------------------------------------------------------------------
struct Worker {
  int rank = 0;
  RunConst rc{};
  void* x = nullptr;
  void* e = nullptr;
  int32_t* idx = nullptr;
  void* val = nullptr;
  int32_t* blk = nullptr;             // n_b: per-block counts, computed on demand
  void* stage = nullptr;              // warp-chunk staging of the compaction ((idx, val) pairs)
  int32_t* chunk_count = nullptr;
  int32_t* tile_count = nullptr;
  double* tile_norm = nullptr;
  Ctrl* ctrl = nullptr;
  CountRec* cnt = nullptr;            // this worker's count slot
  int32_t* idx_global = nullptr;
  void* contrib = nullptr;
  void* grad_stage = nullptr;         // exd_engine_step_host staging
  void* snapshot = nullptr;           // verify_conservation: acc of the running step
  uint32_t* bitmap = nullptr;         // verify_conservation: union membership
  exd_record* rec_host = nullptr;     // pinned: last record copied back at sync
  RawRecord* rec_dev = nullptr;       // device ring of kRecRing raw records (slot t % kRecRing)
  RawRecord* raw_host = nullptr;      // pinned: last raw record copied back at sync
  unsigned long long* range_words = nullptr;  // finish kernel, large vectors ([3][kMaxCtas])
  Plan plan0{};                       // host copy of the t = 0 plan
};

struct exd_engine {
  exd_config cfg{};
  exd_options opt{};
  bool dist = false;
  int device = 0;
  int n = 1;
  cudaStream_t stream = nullptr;
  std::vector<Worker> w;
  size_t esz = 4;
  int64_t tiles = 0;
  int tile = 0;
  int64_t cap_part = 0;
  long long t = 0;                    // steps enqueued
  int64_t cap = 0;                    // per-rank density cap (0: none)
  bool union_flow = false;            // union / reduce / finalize kernels run (n > 1 or cap)
  // shared device buffers
  CountRec* counts_all = nullptr;     // [n]
  CountRec* counts_host = nullptr;    // pinned (dist)
  void* sum = nullptr;                // all-reduced values [n_g]
  const int32_t** d_lists = nullptr;  // [n] (sim)
  const void** d_contribs = nullptr;  // [n] (sim)
  Ctrl** d_ctrls = nullptr;           // [n local]
  void* qscratch = nullptr;
  void* qbits = nullptr;              // quantile result (T)
  uint32_t* verify_flag = nullptr;    // mapped pinned
  uint32_t* verify_flag_dev = nullptr;
  int64_t verify_t = -1;
  // dist
  ncclComm_t comm = nullptr;
  // NVLink peer-memory sync (f1)
  bool p2p = false;
  void* region = nullptr;             // exported inbox: flags[n] | lists[n] | contrib[2]
  std::vector<void*> peer_regions;    // opened IPC mappings (nullptr for self)
  PeerFlags* inbox = nullptr;         // own inbox flag slots (local)
  PeerFlags** d_slot = nullptr;       // [n] my slot in every rank's inbox
  const int32_t** d_p2p_lists = nullptr;  // [n] lists to read (own idx / inbox slots)
  int32_t** d_push = nullptr;         // [n-1] my list slot in every peer's inbox
  void** d_contrib = nullptr;         // [2][n]
  unsigned int* p2p_err = nullptr;    // pinned host copy
  unsigned int* p2p_err_dev = nullptr;  // device word: peer timeout
  unsigned long long* p2p_gate = nullptr;  // [3] local gate words + arrive counter
  unsigned long long* xrange_words = nullptr;  // push-reduce, large vectors: [3][kMaxCtas]
  int64_t xcap = 0;                   // push-reduce contribution capacity (union positions)
  std::vector<void*> spill_peer[2];   // [n] every rank's exported spill buffer (own: local)
  std::vector<unsigned long long*> spill_flag_out[2];  // [n] my flag row in every inbox
  unsigned long long* spill_flag_in[2] = {nullptr, nullptr};  // own flag area [n][kMaxCtas]
  int two_pass = -1;                  // exchange work loop: -1 by size, 0/1 forced (EXD_TWO_PASS)
  int tile_pack = -1;                 // K1 pushes its indices packed per tile: -1 by size, 0/1
                                      // forced (EXD_TILE_PACK)
  int xchg_blocks = 444;              // exchange work blocks (3 per SM - 1)
  void* p2p_own_contrib[2] = {nullptr, nullptr};  // own contribution buffers (parity)
  // push-reduce (EXD_SYNC_P2P without a cap): inbox = flags[2][n] | staged idx[2][n][stage_cap]
  //   | chunk counts[2][n] | tile counts[2][n] | contrib[2][n][n_g]   ([2]: step parity;
  //   everything but the flags as {payload, epoch} words)
  bool xchg = false;
  // ({payload, epoch} words; [2]: step parity)
  std::vector<unsigned long long*> push_stage[2], push_chunk[2], push_tile[2];  // [n-1] my slots in every peer's inbox
  std::vector<PeerFlags*> slot_host;                   // [n] my parity-0 flag slot in every rank's inbox
  std::vector<const unsigned long long*> stage_in[2], chunk_in[2], tile_in[2];  // [n] inbox slots by source
  std::vector<void*> contrib_out[2];                   // [n] my contribution slot in every inbox
  std::vector<void*> sum_out[2];                       // [n] the holder-sum slot of every inbox
  const void* sum_in[2] = {nullptr, nullptr};          // own holder-sum slots
  bool holder_sum = false;                             // n >= 4 (EXD_HOLDER_SUM=0/1 overrides)
  std::vector<const void*> contrib_in[2];              // [n] contribution slots by source (local)
  unsigned long long* rep_hash = nullptr;  // [4 * (n + 1)]: own words, then all ranks' words
  int32_t* recv = nullptr;
  int64_t recv_cap = 0;
  // profiling
  struct Pending {
    cudaEvent_t a, b, c;
    bool finish;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> free_ev;
  exd_kernel_stats stats{};
  bool has_record = false;
  bool broken = false;                // a peer timed out: further steps are refused
  // baseline sparsifiers (Top-k / CLT-k / hard threshold, baseline_engine.cu)
  bool baseline = false;
  void* bl_scratch = nullptr;         // selector scratch (baselines.cu)
  int64_t* bl_totals = nullptr;       // [n_local][4] selector totals
  void* bl_union = nullptr;           // union bitmap + block offsets
  CountRec* bl_ucnt = nullptr;        // |idx_global|
};

namespace {

// Host wait for the engine's stream. With a communicator, poll instead of
// blocking: ncclCommGetAsyncError reports a failed collective, and a
// collective stuck on a dead peer gives up after EXD_NCCL_TIMEOUT_S (60 s).
// Either way the communicator is aborted, the engine refuses further steps
// and the call returns EXD_ENCCL (the reference's analogue is an EngineError
// out of step(), engine.cpp:251-272).
int wait_stream(exd_engine* h) {
  if (!h->comm) {
    CU(cudaStreamSynchronize(h->stream));
    return EXD_OK;
  }
  const auto t0 = std::chrono::steady_clock::now();
  for (unsigned spin = 0;; ++spin) {
    const cudaError_t e = cudaStreamQuery(h->stream);
    if (e == cudaSuccess) return EXD_OK;
    if (e != cudaErrorNotReady)
      return set_err(EXD_ECUDA, std::string("engine stream: ") + cudaGetErrorString(e));
    // spin for the first ~50 ms (a sleeping host wakes late and every peer's
    // kernel then waits for this rank's next step); check the communicator
    // every 1024 polls, then poll at 50 us
    const double el =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (el < 0.05 && (spin & 1023u) != 1023u) continue;
    ncclResult_t ar = ncclSuccess;
    nccl().CommGetAsyncError(h->comm, &ar);
    if ((ar != ncclSuccess && ar != ncclInProgress) || el > nccl_timeout_s()) {
      const std::string why =
          ar != ncclSuccess && ar != ncclInProgress
              ? std::string("NCCL asynchronous error: ") + nccl().GetErrorString(ar)
              : "NCCL collective did not complete within " + std::to_string((int)nccl_timeout_s()) +
                    " s (a peer is gone?)";
      nccl().CommAbort(h->comm);
      h->comm = nullptr;
      h->broken = true;
      return set_err(EXD_ENCCL, why);
    }
    if (el >= 0.05) std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

int alloc_zero(void** p, size_t bytes) {
  if (bytes == 0) bytes = 16;
  CU(cudaMalloc(p, bytes));
  CU(cudaMemset(*p, 0, bytes));
  return EXD_OK;
}

// The plan of step t = 0 on the host (identical to make_plan on the device):
// the t = 0 select-only launch needs its tile range before the kernel runs.
Plan host_plan(const exd_topology& topo0, const int64_t* k_t, const exd_config& c,
               int static_partitions, int rank) {
  Plan p{};
  p.topo = topo0;
  if (!static_partitions) {
    int64_t kp[EXD_MAX_WORKERS];
    rotate(k_t, 0, c.n, kp);
    adjust(p.topo, kp, c.alpha, c.blk_move, c.min_blk, c.n_g, &p.moves, &p.skips);
  }
  p.partition = allocate(p.topo, 0, rank, c.n_g, &p.st, &p.end);
  return p;
}

int setup(exd_engine* h, const exd_config* raw, const exd_options* opt, int first_rank,
          int n_local) {
  exd_config cfg;
  if (int rc = validate_cfg(raw, &cfg)) return rc;
  if (cfg.n > EXD_MAX_WORKERS) return set_err(EXD_EINVAL, "worker count out of range");
  if (cfg.n_g > 0x7fffffffLL) return set_err(EXD_EINVAL, "gradient count exceeds int32 index range");
  if (opt->sparsifier < EXD_SPARSIFIER_EXDYNA || opt->sparsifier > EXD_SPARSIFIER_HARD_THRESHOLD)
    return set_err(EXD_EINVAL, "sparsifier out of range");
  // engine.cpp:58-61
  if (opt->sparsifier == EXD_SPARSIFIER_HARD_THRESHOLD && !(opt->fixed_delta > 0.0))
    return set_err(EXD_EINVAL, "fixed_delta out of range");

  if (opt->dtype != EXD_F32 && opt->dtype != EXD_F64) return set_err(EXD_EINVAL, "dtype out of range");
  h->cfg = cfg;
  h->opt = *opt;
  h->n = cfg.n;
  h->baseline = opt->sparsifier != EXD_SPARSIFIER_EXDYNA;
  // engine.cpp:166-171: cap = max(1, llround(max_density_cap * n_g / n)), ExDyna only
  if (cfg.has_max_density_cap && !h->baseline) {
    const int64_t c = (int64_t)std::llround(cfg.max_density_cap * (double)cfg.n_g / cfg.n);
    h->cap = c > 1 ? c : 1;
  }
  h->union_flow = cfg.n > 1 || h->cap > 0 || h->baseline;
  h->esz = elem_size(opt->dtype);
  h->tiles = num_tiles(cfg.n_g, opt->dtype);
  h->tile = tile_elems(opt->dtype);
  CU(cudaSetDevice(h->device));
  CU(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));

  exd_topology topo0;
  std::string warn;
  if (int rc = build_topo(cfg.n_g, cfg.n_b, cfg.n, cfg.min_blk, &topo0, &warn)) return rc;
  // Largest partition any plan can produce: every other partition keeps at
  // least min_blk blocks of sz_blk elements.
  h->cap_part = cfg.n_g - (int64_t)(cfg.n - 1) * cfg.min_blk * topo0.sz_blk;
  if (h->cap_part < 1 || h->baseline) h->cap_part = cfg.n_g;  // baselines select over [0, n_g)

  const int n = cfg.n;
  const size_t ng = (size_t)cfg.n_g;
  h->w.resize(n_local);
  if (int rc = alloc_zero((void**)&h->counts_all, sizeof(CountRec) * n)) return rc;
  CU(cudaHostAlloc((void**)&h->counts_host, sizeof(CountRec) * n, cudaHostAllocDefault));
  if (h->union_flow) {
    if (int rc = alloc_zero(&h->sum, h->esz * ng)) return rc;
  }
  if (int rc = alloc_zero(&h->qscratch, quantile_scratch_bytes())) return rc;
  if (h->baseline) {
    if (int rc = alloc_zero(&h->bl_scratch, baseline_scratch_bytes(cfg.n_g))) return rc;
    if (int rc = alloc_zero((void**)&h->bl_totals, sizeof(int64_t) * 4 * n_local)) return rc;
    if (int rc = alloc_zero(&h->bl_union, baseline_union_scratch_bytes(cfg.n_g))) return rc;
    if (int rc = alloc_zero((void**)&h->bl_ucnt, sizeof(CountRec))) return rc;
  }
  if (int rc = alloc_zero(&h->qbits, 16)) return rc;
  CU(cudaHostAlloc((void**)&h->verify_flag, sizeof(uint32_t), cudaHostAllocMapped));
  *h->verify_flag = 0;
  CU(cudaHostGetDevicePointer((void**)&h->verify_flag_dev, h->verify_flag, 0));

  std::vector<Ctrl*> ctrls;
  for (int i = 0; i < n_local; ++i) {
    Worker& wk = h->w[i];
    wk.rank = first_rank + i;
    RunConst& rc = wk.rc;
    rc.n_g = cfg.n_g;
    rc.n_b = cfg.n_b;
    rc.k = cfg.k;
    rc.n = n;
    rc.rank = wk.rank;
    rc.eta = cfg.eta;
    rc.alpha = cfg.alpha;
    rc.beta = cfg.beta;
    rc.gamma = cfg.gamma;
    rc.blk_move = cfg.blk_move;
    rc.min_blk = cfg.min_blk;
    rc.static_partitions = opt->static_partitions;
    rc.dtype = opt->dtype;
    rc.cap = h->cap;
    rc.inv_alpha = 1.0 / cfg.alpha;
    rc.inv_beta = 1.0 / cfg.beta;
    rc.fused = (n == 1 && h->cap == 0) ? 1 : 0;
    blk_magic(topo0.sz_blk, &rc.blk_magic, &rc.blk_shift);
    if (int r = alloc_zero(&wk.x, h->esz * ng)) return r;
    if (int r = alloc_zero(&wk.e, h->esz * ng)) return r;
    if (int r = alloc_zero((void**)&wk.idx, 4 * (size_t)h->cap_part)) return r;
    if (int r = alloc_zero(&wk.val, h->esz * (size_t)h->cap_part)) return r;
    if (int r = alloc_zero((void**)&wk.blk, 4 * (size_t)cfg.n_b)) return r;
    // runs are placed at their first element's global index (stream kernel)
    const size_t stage_cap = ng + 2 * (size_t)h->tile;
    if (int r = alloc_zero(&wk.stage, 2 * h->esz * stage_cap)) return r;
    if (int r = alloc_zero((void**)&wk.chunk_count, 4 * (size_t)(h->tiles + 1) * kChunksPerTile)) return r;
    if (int r = alloc_zero((void**)&wk.tile_count, 4 * (size_t)(h->tiles + 8))) return r;
    if (int r = alloc_zero((void**)&wk.tile_norm, 8 * (size_t)(h->tiles + 1))) return r;
    if (int r = alloc_zero((void**)&wk.ctrl, sizeof(Ctrl))) return r;
    // more tiles than one round of the finish kernel's base sum: published range words
    if (h->tiles > kBaseRoundTiles)
      if (int r = alloc_zero((void**)&wk.range_words, sizeof(unsigned long long) * 3 * kMaxCtas))
        return r;
    if (opt->verify_conservation) {
      if (int r = alloc_zero(&wk.snapshot, h->esz * ng)) return r;
      if (int r = alloc_zero((void**)&wk.bitmap, 4 * ((ng + 31) / 32))) return r;
    }
    if (h->union_flow) {
      if (int r = alloc_zero((void**)&wk.idx_global, 4 * ng)) return r;
      if (int r = alloc_zero(&wk.contrib, h->esz * ng)) return r;
    }
    if (h->dist && n > 1) {
      if (int r = alloc_zero((void**)&wk.cnt, sizeof(CountRec))) return r;  // all-gather source
    } else {
      wk.cnt = h->counts_all + (h->dist ? 0 : wk.rank);
    }
    CU(cudaHostAlloc((void**)&wk.rec_host, sizeof(exd_record), cudaHostAllocDefault));
    std::memset(wk.rec_host, 0, sizeof(exd_record));
    if (int r = alloc_zero((void**)&wk.rec_dev, sizeof(RawRecord) * kRecRing)) return r;
    CU(cudaHostAlloc((void**)&wk.raw_host, sizeof(RawRecord), cudaHostAllocDefault));

    // engine.cpp:68-87: x = 0, e = 0, topology, k_t = k/n, delta = delta0
    Ctrl c;
    std::memset(&c, 0, sizeof(c));
    c.t = 0;
    c.tmod = 0;
    // engine.cpp:76-86
    c.delta = h->baseline ? (opt->sparsifier == EXD_SPARSIFIER_HARD_THRESHOLD ? opt->fixed_delta : 0.0)
                          : cfg.has_delta0 ? cfg.delta0 : 0.0;
    c.has_delta = cfg.has_delta0;
    c.thr_f = cfg.has_delta0 ? round_up_float(cfg.delta0) : 0.0f;
    for (int r = 0; r < n; ++r) c.k_t[r] = cfg.k / n;
    c.topo = topo0;
    c.epoch = 1;
    wk.plan0 = host_plan(topo0, c.k_t, cfg, opt->static_partitions, wk.rank);
    c.plan[0] = wk.plan0;
    c.plan[1] = wk.plan0;
    c.last = wk.plan0;
    CU(cudaMemcpy(wk.ctrl, &c, sizeof(c), cudaMemcpyHostToDevice));
    ctrls.push_back(wk.ctrl);
  }
  CU(cudaMalloc((void**)&h->d_ctrls, sizeof(Ctrl*) * n_local));
  CU(cudaMemcpy(h->d_ctrls, ctrls.data(), sizeof(Ctrl*) * n_local, cudaMemcpyHostToDevice));
  if (!(h->dist && n > 1) && h->union_flow) {
    std::vector<const int32_t*> lists(n);
    std::vector<const void*> contribs(n);
    for (int i = 0; i < n; ++i) {
      lists[i] = h->w[i].idx;
      contribs[i] = h->w[i].contrib;
    }
    CU(cudaMalloc((void**)&h->d_lists, sizeof(void*) * n));
    CU(cudaMemcpy(h->d_lists, lists.data(), sizeof(void*) * n, cudaMemcpyHostToDevice));
    CU(cudaMalloc((void**)&h->d_contribs, sizeof(void*) * n));
    CU(cudaMemcpy(h->d_contribs, contribs.data(), sizeof(void*) * n, cudaMemcpyHostToDevice));
  }
  CU(cudaDeviceSynchronize());
  return EXD_OK;
}

void teardown(exd_engine* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->broken && h->comm) {  // a peer is gone: no teardown barrier with it
    nccl().CommAbort(h->comm);
    h->comm = nullptr;
  }
  if (h->stream) cudaStreamSynchronize(h->stream);
  if (h->p2p && h->comm) {
    // barrier: no peer may still be reading our region when it is freed
    float* one = nullptr;
    if (cudaMalloc((void**)&one, sizeof(float)) == cudaSuccess) {
      cudaMemset(one, 0, sizeof(float));
      nccl().AllReduce(one, one, 1, ncclFloat32, ncclSum, h->comm, h->stream);
      cudaStreamSynchronize(h->stream);
      cudaFree(one);
    }
  }
  for (void* p : h->peer_regions)
    if (p) cudaIpcCloseMemHandle(p);
  if (h->p2p) cudaFree(h->region);
  cudaFree(h->rep_hash);
  cudaFree(h->d_slot);
  cudaFree(h->d_p2p_lists);
  cudaFree(h->d_push);
  cudaFree(h->d_contrib);
  cudaFreeHost(h->p2p_err);
  cudaFree(h->p2p_err_dev);
  cudaFree(h->p2p_gate);
  cudaFree(h->xrange_words);
  for (auto& wk : h->w) {
    cudaFree(wk.x);
    cudaFree(wk.e);
    cudaFree(wk.idx);
    cudaFree(wk.val);
    cudaFree(wk.blk);
    cudaFree(wk.stage);
    cudaFree(wk.chunk_count);
    cudaFree(wk.tile_count);
    cudaFree(wk.tile_norm);
    cudaFree(wk.ctrl);
    cudaFree(wk.range_words);
    cudaFree(wk.idx_global);
    cudaFree(wk.contrib);
    cudaFree(wk.grad_stage);
    cudaFree(wk.snapshot);
    cudaFree(wk.bitmap);
    if (h->dist && h->n > 1) cudaFree(wk.cnt);
    cudaFreeHost(wk.rec_host);
    cudaFree(wk.rec_dev);
    cudaFreeHost(wk.raw_host);
  }
  cudaFree(h->counts_all);
  cudaFreeHost(h->counts_host);
  cudaFree(h->sum);
  cudaFree(h->d_lists);
  cudaFree(h->d_contribs);
  cudaFree(h->d_ctrls);
  cudaFree(h->qscratch);
  cudaFree(h->bl_scratch);
  cudaFree(h->bl_totals);
  cudaFree(h->bl_union);
  cudaFree(h->bl_ucnt);
  cudaFree(h->qbits);
  cudaFree(h->recv);
  cudaFreeHost(h->verify_flag);
  for (auto& p : h->pending) { cudaEventDestroy(p.a); cudaEventDestroy(p.b); cudaEventDestroy(p.c); }
  for (auto& ev : h->free_ev) cudaEventDestroy(ev);
  if (h->comm) nccl().CommDestroy(h->comm);
  if (h->stream) cudaStreamDestroy(h->stream);
}

// f1: export one IPC region per rank (flags | selection list | two contribution
// buffers), exchange the handles with one NCCL all-gather, map every peer.
// Returns EXD_OK with h->p2p == false when the peers are not P2P-reachable
// and the caller asked for EXD_SYNC_AUTO.
int setup_p2p(exd_engine* h) {
  const int n = h->n, me = h->w[0].rank;
  // can this device reach every other device directly? (decided collectively:
  // every rank must take the same path)
  int ndev = 0;
  CU(cudaGetDeviceCount(&ndev));
  int ok_local = 1;
  for (int d = 0; d < ndev; ++d) {
    if (d == h->device) continue;
    int can = 0;
    CU(cudaDeviceCanAccessPeer(&can, h->device, d));
    ok_local &= can;
  }
  int* d_ok = nullptr;
  CU(cudaMalloc((void**)&d_ok, sizeof(int)));
  CU(cudaMemcpy(d_ok, &ok_local, sizeof(int), cudaMemcpyHostToDevice));
  NC(nccl().AllReduce(d_ok, d_ok, 1, ncclInt32, ncclMin, h->comm, h->stream));
  int ok_all = 0;
  CU(cudaMemcpyAsync(&ok_all, d_ok, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  cudaFree(d_ok);
  if (!ok_all) {
    if (h->opt.sync_mode == EXD_SYNC_P2P || h->opt.sync_mode == EXD_SYNC_P2P_PULL)
      return set_err(EXD_EUNSUPPORTED, "EXD_SYNC_P2P: some peers are not P2P-reachable");
    return EXD_OK;
  }
  // push-reduce unless the caller asked for pull-reduce, or a density cap /
  // verify_conservation needs the trimmed lists and contribution buffers first
  h->xchg = h->opt.sync_mode != EXD_SYNC_P2P_PULL && h->cap == 0 && !h->opt.verify_conservation;
  // protocol switches: the peers' kernels read each other's inbox layout, so
  // every rank must run the same ones (the environment is per process)
  h->holder_sum = n >= 4;
  if (const char* hs = std::getenv("EXD_HOLDER_SUM")) h->holder_sum = hs[0] == '1';
  if (const char* tp = std::getenv("EXD_TWO_PASS")) h->two_pass = tp[0] == '1' ? 1 : 0;
  if (const char* tk = std::getenv("EXD_TILE_PACK")) h->tile_pack = tk[0] == '1' ? 1 : 0;
  {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device);
    h->xchg_blocks = 3 * sms - 1;  // the spill flags are indexed by work block
  }
  const char* push_cap_env = std::getenv("EXD_PUSH_CAP");
  {
    static const char* const kNames[] = {"sync mode / density cap / verify_conservation",
                                         "EXD_HOLDER_SUM", "EXD_TWO_PASS", "EXD_TILE_PACK",
                                         "EXD_PUSH_CAP", "SM count"};
    constexpr int kN = 6;
    int64_t v[2 * kN] = {h->xchg ? 1 : 0,
                         h->holder_sum ? 1 : 0,
                         h->two_pass,
                         h->tile_pack,
                         push_cap_env ? std::atoll(push_cap_env) : -1,
                         h->xchg_blocks};
    for (int i = 0; i < kN; ++i) v[kN + i] = -v[i];  // one min-reduce gives min and -max
    int64_t* d_v = nullptr;
    CU(cudaMalloc((void**)&d_v, sizeof(v)));
    CU(cudaMemcpy(d_v, v, sizeof(v), cudaMemcpyHostToDevice));
    NC(nccl().AllReduce(d_v, d_v, 2 * kN, ncclInt64, ncclMin, h->comm, h->stream));
    int64_t r[2 * kN];
    CU(cudaMemcpyAsync(r, d_v, sizeof(r), cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    cudaFree(d_v);
    for (int i = 0; i < kN; ++i)
      if (r[i] != -r[kN + i])
        return set_err(EXD_EINVAL, std::string("peer-memory sync: ") + kNames[i] +
                                       " differs across ranks; every rank must use the same");
  }
  auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
  size_t flags_b = 0, list_b = 0, con_b = 0, off_lists = 0, off_c0 = 0, off_c1 = 0, total = 0;
  size_t stage_b = 0, chunk_b = 0, tile_b = 0, xcon_b = 0, off_st = 0, off_ch = 0, off_ti = 0, off_xc = 0;
  // push-reduce contribution capacity in union positions: n_g (every position
  // a word slot per source) unless that does not fit or EXD_PUSH_CAP says
  // otherwise; positions past it spill to a pull from the sources' exported
  // buffers (exchange kernel). Halved per failed attempt down to a floor.
  const int64_t k_floor = std::max<int64_t>(1 << 20, 2 * h->cfg.k);
  int64_t xcap = h->cfg.n_g;
  if (push_cap_env) xcap = std::max<int64_t>(1, std::atoll(push_cap_env));
  xcap = std::min<int64_t>(xcap, h->cfg.n_g);
  size_t spill_b = 0, sflag_b = 0, off_sp = 0, off_sf = 0;
  for (int attempt = 0; attempt < 64; ++attempt) {
    if (h->xchg) {
      // push-reduce: flags[2][n] | stage[2] | chunk counts[2][n] | tile counts[2][n]
      //              | contributions[2][n]; words: 8 B per index / count / fp32 value, 16 B per fp64.
      // One staging slot per parity serves every source: a holder pushes its
      // runs at their global element index, and partitions are disjoint.
      flags_b = al(sizeof(PeerFlags) * (size_t)n * 2);
      stage_b = al(8 * ((size_t)h->cfg.n_g + 2 * (size_t)h->tile));
      chunk_b = al(8 * (size_t)(h->tiles + 1) * kChunksPerTile);
      tile_b = al(8 * (size_t)(h->tiles + 8));
      xcon_b = al(2 * h->esz * (size_t)xcap);
      const bool spill = xcap < h->cfg.n_g;
      spill_b = spill ? al(h->esz * (size_t)h->cfg.n_g) : 0;  // [2] own contributions to pull
      sflag_b = spill ? al(8 * (size_t)n * kMaxCtas) : 0;     // [2][source][work block]
      off_st = flags_b;
      off_ch = off_st + stage_b * 2;
      off_ti = off_ch + chunk_b * 2 * n;
      off_xc = off_ti + tile_b * 2 * n;
      off_sp = off_xc + xcon_b * 2 * n + xcon_b * 2;  // after the holder-sum slots [2]
      off_sf = off_sp + spill_b * 2;
      total = off_sf + sflag_b * 2;
    } else {
      // pull-reduce: flags[n] | lists[n][cap_part] | contrib[2][n_g]
      flags_b = al(sizeof(PeerFlags) * (size_t)n);
      list_b = al(4 * (size_t)h->cap_part);
      con_b = al(h->esz * (size_t)h->cfg.n_g);
      off_lists = flags_b;
      off_c0 = off_lists + list_b * (size_t)n;
      off_c1 = off_c0 + con_b;
      total = off_c1 + con_b;
    }
    // every rank must take the same path: agree on whether the region fits
    int ok = cudaMalloc(&h->region, total) == cudaSuccess ? 1 : 0;
    if (!ok) {
      cudaGetLastError();
      h->region = nullptr;
    }
    int* d_ok2 = nullptr;
    CU(cudaMalloc((void**)&d_ok2, sizeof(int)));
    CU(cudaMemcpy(d_ok2, &ok, sizeof(int), cudaMemcpyHostToDevice));
    NC(nccl().AllReduce(d_ok2, d_ok2, 1, ncclInt32, ncclMin, h->comm, h->stream));
    CU(cudaMemcpyAsync(&ok, d_ok2, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    cudaFree(d_ok2);
    if (ok) break;
    if (h->region) cudaFree(h->region);
    h->region = nullptr;
    if (!h->xchg) return set_err(EXD_ECUDA, "peer-memory inbox does not fit in device memory");
    if (xcap > k_floor) {  // a smaller contribution capacity, spilling past it
      xcap = std::max<int64_t>(k_floor, xcap / 2);
      continue;
    }
    h->xchg = false;  // even the floor does not fit: pull-reduce
  }
  h->xcap = h->xchg ? xcap : 0;
  CU(cudaMemset(h->region, 0, flags_b));
  // words start with epoch 0 (never a live epoch)
  if (h->xchg) CU(cudaMemset(static_cast<char*>(h->region) + off_st, 0, total - off_st));
  h->inbox = static_cast<PeerFlags*>(h->region);
  Worker& wk = h->w[0];
  cudaIpcMemHandle_t mine;
  CU(cudaIpcGetMemHandle(&mine, h->region));
  char* d_handles = nullptr;
  CU(cudaMalloc((void**)&d_handles, sizeof(cudaIpcMemHandle_t) * n));
  CU(cudaMemcpy(d_handles + sizeof(cudaIpcMemHandle_t) * me, &mine, sizeof(mine),
                cudaMemcpyHostToDevice));
  NC(nccl().AllGather(d_handles + sizeof(cudaIpcMemHandle_t) * me, d_handles,
                      sizeof(cudaIpcMemHandle_t), ncclUint8, h->comm, h->stream));
  std::vector<cudaIpcMemHandle_t> all(n);
  CU(cudaMemcpyAsync(all.data(), d_handles, sizeof(cudaIpcMemHandle_t) * n,
                     cudaMemcpyDeviceToHost, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  cudaFree(d_handles);
  h->peer_regions.assign(n, nullptr);
  std::vector<char*> base(n);
  for (int r = 0; r < n; ++r) {
    if (r == me) {
      base[r] = static_cast<char*>(h->region);
      continue;
    }
    void* p = nullptr;
    CU(cudaIpcOpenMemHandle(&p, all[r], cudaIpcMemLazyEnablePeerAccess));
    h->peer_regions[r] = p;
    base[r] = static_cast<char*>(p);
  }
  if (h->xchg) {
    char* own = static_cast<char*>(h->region);
    h->slot_host.assign(n, nullptr);
    for (int par = 0; par < 2; ++par) {
      h->stage_in[par].assign(n, nullptr);
      h->chunk_in[par].assign(n, nullptr);
      h->tile_in[par].assign(n, nullptr);
      // my slots in every rank's inbox, the peers first and my own last (the
      // exchange kernel reads its own partition's runs and counts as words
      // too, so it need not wait for the stream kernel to look them up)
      for (int q = 1; q <= n; ++q) {
        const int r = (me + q) % n;
        const size_t sm = (size_t)(par * n + me), sr = (size_t)(par * n + r);
        using W = unsigned long long;
        h->push_stage[par].push_back(reinterpret_cast<W*>(base[r] + off_st + stage_b * par));
        h->push_chunk[par].push_back(reinterpret_cast<W*>(base[r] + off_ch + chunk_b * sm));
        h->push_tile[par].push_back(reinterpret_cast<W*>(base[r] + off_ti + tile_b * sm));
        h->stage_in[par][r] = reinterpret_cast<const W*>(own + off_st + stage_b * par);
        h->chunk_in[par][r] = reinterpret_cast<const W*>(own + off_ch + chunk_b * sr);
        h->tile_in[par][r] = reinterpret_cast<const W*>(own + off_ti + tile_b * sr);
      }
      h->contrib_out[par].assign(n, nullptr);
      h->contrib_in[par].assign(n, nullptr);
      h->sum_out[par].assign(n, nullptr);
      h->sum_in[par] = own + off_xc + xcon_b * (size_t)(2 * n + par);
      for (int r = 0; r < n; ++r) {
        h->contrib_out[par][r] = base[r] + off_xc + xcon_b * (size_t)(par * n + me);
        h->contrib_in[par][r] = own + off_xc + xcon_b * (size_t)(par * n + r);
        h->sum_out[par][r] = base[r] + off_xc + xcon_b * (size_t)(2 * n + par);
      }
    }
    for (int r = 0; r < n; ++r) h->slot_host[r] = reinterpret_cast<PeerFlags*>(base[r]) + me;
    if (h->xcap < h->cfg.n_g) {
      for (int par = 0; par < 2; ++par) {
        h->spill_peer[par].assign(n, nullptr);
        h->spill_flag_out[par].assign(n, nullptr);
        for (int r = 0; r < n; ++r) {
          h->spill_peer[par][r] = base[r] + off_sp + spill_b * par;
          // my row of r's flag area [par][source = me][work block]
          h->spill_flag_out[par][r] = reinterpret_cast<unsigned long long*>(
              base[r] + off_sf + sflag_b * par) + (size_t)me * kMaxCtas;
        }
        h->spill_flag_in[par] = reinterpret_cast<unsigned long long*>(own + off_sf + sflag_b * par);
      }
    }
  }
  std::vector<PeerFlags*> slot(n);
  std::vector<const int32_t*> lists(n);
  std::vector<int32_t*> push;
  std::vector<void*> con(2 * n);
  char* own = static_cast<char*>(h->region);
  for (int r = 0; r < n; ++r) {
    slot[r] = reinterpret_cast<PeerFlags*>(base[r]) + me;
    lists[r] = r == me ? wk.idx : reinterpret_cast<const int32_t*>(own + off_lists + list_b * r);
    if (r != me) push.push_back(reinterpret_cast<int32_t*>(base[r] + off_lists + list_b * me));
    con[r] = h->xchg ? nullptr : base[r] + off_c0;
    con[n + r] = h->xchg ? nullptr : base[r] + off_c1;
  }
  h->p2p_own_contrib[0] = h->xchg ? nullptr : own + off_c0;
  h->p2p_own_contrib[1] = h->xchg ? nullptr : own + off_c1;
  CU(cudaMalloc((void**)&h->d_slot, sizeof(void*) * n));
  CU(cudaMalloc((void**)&h->d_p2p_lists, sizeof(void*) * n));
  CU(cudaMalloc((void**)&h->d_push, sizeof(void*) * (n > 1 ? n - 1 : 1)));
  CU(cudaMalloc((void**)&h->d_contrib, sizeof(void*) * 2 * n));
  CU(cudaMemcpy(h->d_slot, slot.data(), sizeof(void*) * n, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(h->d_p2p_lists, lists.data(), sizeof(void*) * n, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(h->d_push, push.data(), sizeof(void*) * push.size(), cudaMemcpyHostToDevice));
  CU(cudaMemcpy(h->d_contrib, con.data(), sizeof(void*) * 2 * n, cudaMemcpyHostToDevice));
  CU(cudaHostAlloc((void**)&h->p2p_err, sizeof(unsigned int), cudaHostAllocDefault));
  *h->p2p_err = 0;
  if (int r2 = alloc_zero((void**)&h->p2p_err_dev, sizeof(unsigned int))) return r2;
  if (int r2 = alloc_zero((void**)&h->p2p_gate, 3 * sizeof(unsigned long long))) return r2;
  if (h->xchg && h->tiles > kBaseRoundTiles)
    if (int r2 = alloc_zero((void**)&h->xrange_words, sizeof(unsigned long long) * 3 * kMaxCtas))
      return r2;
  // barrier: every rank has mapped every peer before anyone steps
  int* d_b = nullptr;
  CU(cudaMalloc((void**)&d_b, sizeof(int)));
  CU(cudaMemset(d_b, 0, sizeof(int)));
  NC(nccl().AllReduce(d_b, d_b, 1, ncclInt32, ncclSum, h->comm, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  cudaFree(d_b);
  h->p2p = true;
  return EXD_OK;
}

// K1 (stream) and, unless accumulate-only, K2 (finish); CUDA events around
// each when profiling so the bench can report the stream kernel's own time.
int select_phase(exd_engine* h, int mode, const SelectArgs& a, const RunConst& rc,
                 const ExchangeArgs* xa = nullptr) {
  cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
  const bool prof = h->opt.profile_kernels != 0;
  if (prof) {
    for (auto& x : ev) {
      if (h->free_ev.empty()) {
        CU(cudaEventCreate(&x));
      } else {
        x = h->free_ev.back();
        h->free_ev.pop_back();
      }
    }
    CU(cudaEventRecord(ev[0], h->stream));
  }
  CU(launch_stream(mode, a, rc, h->stream));
  h->stats.kernel_launches += 1;
  if (prof) CU(cudaEventRecord(ev[1], h->stream));
  if (mode != kAccumulate) {
    // push-reduce: the finish work and the whole sync are one kernel
    if (xa) CU(launch_exchange(*xa, rc, h->stream));
    else CU(launch_finish(a, rc, h->stream));
    h->stats.kernel_launches += 1;
  }
  if (prof) {
    CU(cudaEventRecord(ev[2], h->stream));
    h->pending.push_back({ev[0], ev[1], ev[2], mode != kAccumulate});
  }
  return EXD_OK;
}

SelectArgs select_args(exd_engine* h, Worker& wk, const void* grad) {
  SelectArgs a{};
  a.g = grad;
  a.e = wk.e;
  a.x = wk.x;
  a.idx = wk.idx;
  a.val = wk.val;
  a.stage = wk.stage;
  a.chunk_count = wk.chunk_count;
  a.tile_count = wk.tile_count;
  a.tile_norm = wk.tile_norm;
  a.ctrl = wk.ctrl;
  a.cnt_out = wk.cnt;
  a.rec = wk.rec_dev + (h->t % kRecRing);
  a.tile_base = 0;
  a.num_tiles = (int32_t)h->tiles;
  a.t = h->t;
  // with a cap the list is pushed only after it is trimmed (cap kernel)
  a.push_idx = (h->p2p && !h->xchg && h->cap == 0) ? h->d_push : nullptr;
  a.npush = (h->p2p && !h->xchg && h->cap == 0) ? h->n - 1 : 0;
  a.k1_npush = h->xchg ? h->n : 0;  // every peer, then this rank's own inbox
  // pairs of ~2k/n selections (16 B fp64, 8 B fp32) against a 32 MB share of L2
  a.stage_keep = 2 * (double)h->cfg.k / h->n * (h->esz == 8 ? 16 : 8) < 32e6 ? 1 : 0;
  // packed per tile on large vectors (fewer, longer NVLink bursts: 1e9 d = 0.001
  // at N = 4 2.86 vs 3.00 ms); per-warp runs on small ones, where the step is
  // latency-bound and a run leaves before its tile's barrier (R18 N = 4: 49.1 vs
  // 49.6 us)
  a.tile_pack = h->tile_pack >= 0 ? h->tile_pack : (h->tiles > kBaseRoundTiles ? 1 : 0);
  a.range_words = wk.range_words;
  const int par = (int)(h->t & 1);  // this step's parity slots
  for (int q = 0; q < a.k1_npush; ++q) {
    a.push_stage[q] = h->push_stage[par][q];
    a.push_chunk[q] = h->push_chunk[par][q];
    a.push_tile[q] = h->push_tile[par][q];
  }
  return a;
}

ExchangeArgs exchange_args(exd_engine* h, const SelectArgs& sa) {
  Worker& wk = h->w[0];
  ExchangeArgs o{};
  o.s = sa;
  o.holder_sum = h->holder_sum ? 1 : 0;
  o.sum_in[0] = h->sum_in[0];
  o.sum_in[1] = h->sum_in[1];
  o.inbox = h->inbox;
  for (int r = 0; r < h->n; ++r) {
    o.peer_slot[r] = h->slot_host[r];
    for (int par = 0; par < 2; ++par) {
      o.stage_in[par][r] = h->stage_in[par][r];
      o.chunk_in[par][r] = h->chunk_in[par][r];
      o.tile_in[par][r] = h->tile_in[par][r];
    }
    for (int par = 0; par < 2; ++par) {
      o.contrib_out[par][r] = h->contrib_out[par][r];
      o.contrib_in[par][r] = h->contrib_in[par][r];
      o.sum_out[par][r] = h->sum_out[par][r];
    }
  }
  o.idx_global = wk.idx_global;
  o.sum = h->sum;
  o.counts_all = h->counts_all;
  o.rec = wk.rec_dev + (h->t % kRecRing);
  o.epoch = (unsigned long long)h->t + 1;
  o.err = h->p2p_err_dev;
  o.me = wk.rank;
  o.xrange_words = h->xrange_words;
  // more than one iteration of the one-pass loop per work block expected
  // (k entries over ~3 blocks per SM, 4 per thread in flight): two passes
  o.two_pass = h->two_pass >= 0 ? h->two_pass : (h->cfg.k > (int64_t)h->xchg_blocks * 4 * 256 ? 1 : 0);
  o.xcap = h->xcap;
  if (h->xcap < h->cfg.n_g) {
    o.two_pass = 1;  // the spill pull lives in pass 2
    for (int par = 0; par < 2; ++par) {
      for (int r = 0; r < h->n; ++r) {
        o.spill_peer[par][r] = h->spill_peer[par][r];
        o.spill_flag_out[par][r] = h->spill_flag_out[par][r];
      }
      o.spill_flag_in[par] = h->spill_flag_in[par];
    }
  }
  return o;
}

// verify_conservation / verify_replication after a step (engine.cpp:221-272)
int enqueue_verify(exd_engine* h, const int32_t* uni_override, const CountRec* ucnt);

// Engine::step for Top-k / CLT-k / hard threshold (engine.cpp:119-144,
// 163-204, 274-350) with in-process workers: accumulate, each worker's device
// selector over its full |acc| (CLT-k: only the cyclic leader,
// baselines.hpp:37-39), a deduplicated union (collectives.cpp:47-55),
// rank-order sum, x update, clear; no threshold scaling, no topology.
int enqueue_baseline_step(exd_engine* h, const void* const* grads) {
  const exd_config& c = h->cfg;
  const int n = h->n, nl = (int)h->w.size();
  const int sp = h->opt.sparsifier;
  const bool topk = sp == EXD_SPARSIFIER_TOPK || sp == EXD_SPARSIFIER_CLTK;
  const int leader = (int)mod_floor(h->t, n);
  for (int i = 0; i < nl; ++i) {
    SelectArgs a = select_args(h, h->w[i], grads[i]);
    if (int r = select_phase(h, kAccumulate, a, h->w[i].rc)) return r;
  }
  for (int i = 0; i < nl; ++i) {
    Worker& wk = h->w[i];
    const bool sel = sp != EXD_SPARSIFIER_CLTK || wk.rank == leader;
    int64_t* tot = h->bl_totals + 4 * i;
    if (sel) {
      CU(launch_baseline_select(wk.e, c.n_g, h->opt.dtype, topk ? 1 : 0, c.k, h->opt.fixed_delta,
                                wk.idx, h->cap_part, tot, h->bl_scratch, h->stream));
      h->stats.kernel_launches += 3 + (topk ? quantile_launches(h->opt.dtype) : 0);
    }
    CU(launch_baseline_counts(sel ? tot : nullptr, wk.tile_norm, (int)h->tiles, wk.cnt, h->stream));
    h->stats.kernel_launches += 1;
  }
  std::vector<const int32_t*> lists(n);
  int32_t* uni = h->w[0].idx_global;
  int64_t list_cap = h->cap_part, kp_host = 0;
  if (h->dist && n > 1) {
    // one rank per GPU (NCCL): the counts all-gather, one host wait for the
    // padded list size (all_gather, collectives.cpp:22-57), the padded lists
    Worker& wk = h->w[0];
    NC(nccl().AllGather(wk.cnt, h->counts_all, sizeof(CountRec), ncclUint8, h->comm, h->stream));
    CU(cudaMemcpyAsync(h->counts_host, h->counts_all, sizeof(CountRec) * n, cudaMemcpyDeviceToHost,
                       h->stream));
    if (int rc = wait_stream(h)) return rc;
    int64_t m_t = 0;
    for (int r = 0; r < n; ++r) {
      m_t = std::max<int64_t>(m_t, h->counts_host[r].k);
      kp_host += h->counts_host[r].k;
    }
    if (m_t * n > h->recv_cap) {
      cudaFree(h->recv);
      h->recv_cap = m_t * n + (m_t * n) / 4 + 1024;
      CU(cudaMalloc((void**)&h->recv, 4 * (size_t)h->recv_cap));
    }
    if (m_t > 0)
      NC(nccl().AllGather(wk.idx, h->recv, (size_t)m_t, ncclInt32, h->comm, h->stream));
    for (int r = 0; r < n; ++r) lists[r] = h->recv + (size_t)r * m_t;
    list_cap = m_t > 0 ? m_t : 1;
  } else {
    for (int i = 0; i < nl; ++i) lists[i] = h->w[i].idx;
  }
  CU(launch_baseline_union(lists.data(), h->counts_all, n, list_cap, c.n_g, h->bl_union, uni,
                           h->bl_ucnt, h->stream));
  h->stats.kernel_launches += baseline_union_launches(n);
  if (h->dist && n > 1) {
    // own contributions at the union, NCCL sum over the k' (>= |union|)
    // entries the host knows (zero past the union: the NCCL order differs
    // from rank order, as on the ExDyna NCCL path)
    Worker& wk = h->w[0];
    if (kp_host > 0) {
      CU(cudaMemsetAsync(wk.contrib, 0, h->esz * (size_t)kp_host, h->stream));
      CU(launch_baseline_gather_clear(uni, h->bl_ucnt, wk.e, wk.contrib, kp_host, h->opt.dtype,
                                      h->stream));
      NC(nccl().AllReduce(wk.contrib, h->sum, (size_t)kp_host,
                          h->opt.dtype == EXD_F64 ? ncclFloat64 : ncclFloat32, ncclSum, h->comm,
                          h->stream));
    }
  } else {
    for (int i = 0; i < nl; ++i) {
      CU(launch_baseline_gather_clear(uni, h->bl_ucnt, h->w[i].e, h->w[i].contrib, c.n_g,
                                      h->opt.dtype, h->stream));
    }
    CU(launch_baseline_sum(h->d_contribs, n, h->bl_ucnt, h->sum, c.n_g, h->opt.dtype, h->stream));
  }
  const double delta_used = sp == EXD_SPARSIFIER_HARD_THRESHOLD ? h->opt.fixed_delta : 0.0;
  for (int i = 0; i < nl; ++i) {
    Worker& wk = h->w[i];
    CU(launch_baseline_apply(uni, h->bl_ucnt, h->sum, wk.x, n, c.n_g, h->opt.dtype, h->stream));
    CU(launch_baseline_epilogue(wk.ctrl, h->counts_all, h->bl_ucnt, wk.rec_dev + (h->t % kRecRing),
                                n, delta_used, h->stream));
  }
  h->stats.kernel_launches += 3 * nl + 1;
  if (int r = enqueue_verify(h, uni, h->bl_ucnt)) return r;
  h->t += 1;
  h->stats.steps += 1;
  h->has_record = true;
  return EXD_OK;
}

// Engine::step, engine.cpp:274-350, enqueued on the engine's stream.
int enqueue_step(exd_engine* h, const void* const* grads) {
  const exd_config& c = h->cfg;
  const int n = h->n;
  const int nl = (int)h->w.size();
  if (h->broken) return set_err(EXD_ENCCL, "engine unusable after a failed collective (peer timeout or NCCL error)");
  for (int i = 0; i < nl; ++i) {
    if (!grads || !grads[i]) return set_err(EXD_EINVAL, "null gradient pointer");
    // the stream kernel reads g with 16-byte vector loads
    if (reinterpret_cast<uintptr_t>(grads[i]) % 16 != 0)
      return set_err(EXD_EINVAL, "gradient pointer must be 16-byte aligned");
  }
  CU(cudaSetDevice(h->device));

  // verify_conservation (engine.cpp:142): acc snapshot of every worker
  if (h->opt.verify_conservation) {
    for (int i = 0; i < nl; ++i) {
      CU(launch_snapshot(h->w[i].e, grads[i], h->w[i].snapshot, h->w[i].rc, h->stream));
      h->stats.kernel_launches += 1;
    }
  }

  if (h->baseline) return enqueue_baseline_step(h, grads);

  if (h->t == 0 && !c.has_delta0) {
    // accumulate_phase, then initialize_threshold (engine.cpp:146-161) on
    // rank 0's accumulated vector, broadcast, then the selection
    for (int i = 0; i < nl; ++i) {
      SelectArgs a = select_args(h, h->w[i], grads[i]);
      if (int r = select_phase(h, kAccumulate, a, h->w[i].rc)) return r;
    }
    const int64_t m = c.n_g;
    int64_t pos = (int64_t)std::floor((1.0 - c.d) * (double)m);
    if (pos > m - 1) pos = m - 1;
    if (!h->dist || h->w[0].rank == 0)
    {
      CU(launch_quantile(h->w[0].e, m, pos, h->opt.dtype, h->qscratch, h->qbits, h->stream));
      h->stats.kernel_launches += quantile_launches(h->opt.dtype);
    }
    if (h->dist && n > 1)
      NC(nccl().Broadcast(h->qbits, h->qbits, h->esz, ncclUint8, 0, h->comm, h->stream));
    CU(launch_set_delta(h->d_ctrls, nl, h->qbits, h->opt.dtype, h->stream));
    h->stats.kernel_launches += 1;
    for (int i = 0; i < nl; ++i) {
      Worker& wk = h->w[i];
      SelectArgs a = select_args(h, wk, grads[i]);
      const int64_t first = wk.plan0.st / h->tile;
      const int64_t last = (wk.plan0.end - 1) / h->tile;
      a.tile_base = (int32_t)first;
      a.num_tiles = (int32_t)(last - first + 1);
      const ExchangeArgs xa = h->xchg ? exchange_args(h, a) : ExchangeArgs{};
      if (int r = select_phase(h, kSelectOnly, a, wk.rc, h->xchg ? &xa : nullptr)) return r;
    }
  } else {
    for (int i = 0; i < nl; ++i) {
      SelectArgs a = select_args(h, h->w[i], grads[i]);
      const ExchangeArgs xa = h->xchg ? exchange_args(h, a) : ExchangeArgs{};
      if (int r = select_phase(h, kFused, a, h->w[i].rc, h->xchg ? &xa : nullptr)) return r;
    }
  }

  // density cap on each worker's compacted selection (selector.cpp:44-61)
  if (h->cap > 0) {
    for (int i = 0; i < nl; ++i) {
      Worker& wk = h->w[i];
      CapArgs ca{};
      ca.idx = wk.idx;
      ca.val = wk.val;
      ca.e = wk.e;
      ca.cnt = wk.cnt;
      ca.ctrl = wk.ctrl;
      ca.push = h->p2p ? h->d_push : nullptr;
      ca.npush = h->p2p ? n - 1 : 0;
      CU(launch_cap(ca, wk.rc, h->stream));
      h->stats.kernel_launches += 1;
    }
  }

  if (h->union_flow && !h->xchg) {
    if (h->dist && n > 1 && h->p2p) {
      // f1: peer-memory sync, no host wait, no NCCL
      Worker& wk = h->w[0];
      P2PArgs pa{};
      pa.inbox = h->inbox;
      pa.peer_slot = h->d_slot;
      pa.lists = h->d_p2p_lists;
      pa.contrib = h->d_contrib + (h->t & 1) * n;
      pa.own_val = wk.val;
      pa.e = wk.e;
      pa.x = wk.x;
      pa.idx_global = wk.idx_global;
      pa.sum = h->sum;
      pa.counts_all = h->counts_all;
      pa.own_cnt = wk.cnt;
      pa.ctrl = wk.ctrl;
      pa.rec = wk.rec_dev + (h->t % kRecRing);
      pa.epoch = (unsigned long long)h->t + 1;
      pa.err = h->p2p_err_dev;
      pa.gate = h->p2p_gate;
      pa.me = wk.rank;
      CU(launch_p2p_sync(pa, wk.rc, h->stream));
      h->stats.kernel_launches += 1;
    } else if (h->dist && n > 1) {
      Worker& wk = h->w[0];
      NC(nccl().AllGather(wk.cnt, h->counts_all, sizeof(CountRec), ncclUint8, h->comm, h->stream));
      CU(cudaMemcpyAsync(h->counts_host, h->counts_all, sizeof(CountRec) * n,
                         cudaMemcpyDeviceToHost, h->stream));
      if (int rc = wait_stream(h)) return rc;
      int64_t m_t = 0, kp = 0;
      for (int r = 0; r < n; ++r) {
        m_t = h->counts_host[r].k > m_t ? h->counts_host[r].k : m_t;
        kp += h->counts_host[r].k;
      }
      if (m_t * n > h->recv_cap) {
        cudaFree(h->recv);
        h->recv_cap = m_t * n + (m_t * n) / 4 + 1024;
        CU(cudaMalloc((void**)&h->recv, 4 * (size_t)h->recv_cap));
      }
      if (m_t > 0)
        NC(nccl().AllGather(wk.idx, h->recv, (size_t)m_t, ncclInt32, h->comm, h->stream));
      UnionArgs u{};
      u.lists = nullptr;
      u.padded = h->recv;
      u.counts = h->counts_all;
      u.own_val = wk.val;
      u.e = wk.e;
      u.idx_global = wk.idx_global;
      u.contrib = wk.contrib;
      u.ctrl = wk.ctrl;
      CU(launch_union(u, wk.rc, h->stream));
      h->stats.kernel_launches += 1;
      if (kp > 0)
        NC(nccl().AllReduce(wk.contrib, h->sum, (size_t)kp,
                            h->opt.dtype == EXD_F64 ? ncclFloat64 : ncclFloat32, ncclSum,
                            h->comm, h->stream));
      FinalizeArgs f{};
      f.idx_global = wk.idx_global;
      f.sum = h->sum;
      f.x = wk.x;
      f.ctrl = wk.ctrl;
      f.counts = h->counts_all;
      f.rec = wk.rec_dev + (h->t % kRecRing);
      CU(launch_finalize(f, wk.rc, h->stream));
      h->stats.kernel_launches += 1;
    } else {
      for (int i = 0; i < nl; ++i) {
        Worker& wk = h->w[i];
        UnionArgs u{};
        u.lists = h->d_lists;
        u.padded = nullptr;
        u.counts = h->counts_all;
        u.own_val = wk.val;
        u.e = wk.e;
        u.idx_global = wk.idx_global;
        u.contrib = wk.contrib;
        u.ctrl = wk.ctrl;
        CU(launch_union(u, wk.rc, h->stream));
        h->stats.kernel_launches += 1;
      }
      CU(launch_allreduce_local(h->d_contribs, h->sum, h->w[0].ctrl, h->counts_all, h->w[0].rc,
                                h->stream));
      h->stats.kernel_launches += 1;
      for (int i = 0; i < nl; ++i) {
        Worker& wk = h->w[i];
        FinalizeArgs f{};
        f.idx_global = wk.idx_global;
        f.sum = h->sum;
        f.x = wk.x;
        f.ctrl = wk.ctrl;
        f.counts = h->counts_all;
        f.rec = wk.rec_dev + (h->t % kRecRing);
        CU(launch_finalize(f, wk.rc, h->stream));
        h->stats.kernel_launches += 1;
      }
    }
  }
  if (int r = enqueue_verify(h, nullptr, nullptr)) return r;
  h->t += 1;
  h->stats.steps += 1;
  h->has_record = true;
  return EXD_OK;
}

// uni_override / ucnt: the baselines' shared union and its size (nullptr:
// ExDyna's per-worker union of sum(counts) entries)
int enqueue_verify(exd_engine* h, const int32_t* uni_override, const CountRec* ucnt) {
  const int n = h->n;
  const int nl = (int)h->w.size();
  const exd_config& c = h->cfg;
  // verify_conservation, engine.cpp:221-249 (each worker against its snapshot)
  if (h->opt.verify_conservation) {
    for (int i = 0; i < nl; ++i) {
      Worker& wk = h->w[i];
      const int32_t* uni = uni_override ? uni_override : h->union_flow ? wk.idx_global : wk.idx;
      const void* contrib = !h->union_flow ? wk.val
                            : (h->dist && n > 1 && h->p2p) ? h->p2p_own_contrib[h->t & 1]
                                                           : wk.contrib;
      const CountRec* cnts = ucnt ? ucnt : h->union_flow ? h->counts_all : wk.cnt;
      const int ncnt = ucnt ? 1 : h->union_flow ? n : 1;
      CU(launch_conservation(uni, cnts, ncnt, contrib, wk.e, wk.snapshot, wk.bitmap,
                             h->verify_flag_dev, wk.rc, h->stream));
      h->stats.kernel_launches += 2;
    }
    h->verify_t = h->t;
  }
  // verify_replication, engine.cpp:251-272 (in-process replicas)
  if (h->opt.verify_replication && !h->dist && nl > 1) {
    for (int i = 1; i < nl; ++i)
      CU(launch_verify_replication(h->w[0].ctrl, h->w[i].ctrl, h->w[0].x, h->w[i].x, c.n_g,
                                   h->opt.dtype, h->w[i].rank, h->verify_flag_dev, h->stream));
    h->stats.kernel_launches += nl - 1;
    h->verify_t = h->t;
  }
  // verify_replication across ranks: hash, all-gather, compare with rank 0
  if (h->opt.verify_replication && h->dist && n > 1) {
    if (!h->rep_hash) CU(cudaMalloc((void**)&h->rep_hash, sizeof(unsigned long long) * 4 * (n + 1)));
    Worker& wk = h->w[0];
    CU(launch_replica_hash(wk.ctrl, wk.x, h->rep_hash, wk.rc, h->stream));
    NC(nccl().AllGather(h->rep_hash, h->rep_hash + 4, 4, ncclUint64, h->comm, h->stream));
    CU(launch_replica_compare(h->rep_hash + 4, n, h->verify_flag_dev, h->stream));
    h->stats.kernel_launches += 2;
    h->verify_t = h->t;
  }
  return EXD_OK;
}

// IterationRecord of one step (collectives.cpp:29-45, engine.cpp:327-349) from
// the device's raw record, with the reference's formulas (host side of
// control.cuh, compiled without FMA contraction).
void finalize_record(const RawRecord& r, const exd_config& cfg, int sparsifier, exd_record* rec) {
  const int n = r.n;
  double norm_sum = 0.0;
  for (int i = 0; i < n; ++i) norm_sum += std::sqrt(r.norm2[i]);
  exd_gather_stats gs;
  gather_stats(r.k_rank, n, &gs);
  std::memset(rec, 0, sizeof(*rec));
  rec->t = r.t;
  rec->k_prime = gs.k_prime;
  rec->density = (double)gs.k_prime / (double)cfg.n_g;
  const int64_t diff = cfg.k - gs.k_prime;
  rec->eps = (double)(diff < 0 ? -diff : diff) / (double)cfg.n_g;
  rec->m_t = gs.m_t;
  rec->c_t = gs.c_t;
  rec->f_t = gs.f_t;
  rec->global_err = norm_sum / (double)n;
  rec->delta = r.delta;
  if (sparsifier == EXD_SPARSIFIER_EXDYNA) {
    rec->duplicates = 0;  // disjoint partitions + ascending lists: no duplicates by construction
    rec->union_count = gs.k_prime;
  } else {  // collectives.cpp:52-55: total - |sorted unique union|
    rec->duplicates = gs.k_prime - r.union_count;
    rec->union_count = r.union_count;
  }
  rec->idle_workers = sparsifier == EXD_SPARSIFIER_CLTK ? n - 1 : 0;  // engine.cpp:346
  rec->n = n;
  rec->adjust_moves = r.moves;
  rec->adjust_skips = r.skips;
  int cap_hits = 0;  // engine.cpp:345
  for (int i = 0; i < n; ++i) cap_hits += r.capped[i] ? 1 : 0;
  rec->cap_hits = cap_hits;
  for (int i = 0; i < n; ++i) rec->k_rank[i] = r.k_rank[i];
}

int sync_engine(exd_engine* h, exd_record* out) {
  CU(cudaSetDevice(h->device));
  if (int rc = wait_stream(h)) return rc;
  for (auto& p : h->pending) {
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, p.a, p.b));
    h->stats.select_ms += ms;
    h->stats.select_launches += 1;
    if (p.finish) {
      CU(cudaEventElapsedTime(&ms, p.b, p.c));
      h->stats.finish_ms += ms;
      h->stats.finish_launches += 1;
    }
    h->free_ev.push_back(p.a);
    h->free_ev.push_back(p.b);
    h->free_ev.push_back(p.c);
  }
  h->pending.clear();
  if (h->p2p) {
    CU(cudaMemcpy(h->p2p_err, h->p2p_err_dev, sizeof(unsigned int), cudaMemcpyDeviceToHost));
    if (*h->p2p_err) {
      // the in-kernel counters and epochs no longer line up across ranks
      h->broken = true;
      return set_err(EXD_ENCCL, "peer-memory sync: a peer did not arrive within 20 s");
    }
  }
  if (*h->verify_flag) {
    const uint32_t f = *h->verify_flag;
    char msg[160];
    if (f >= 0x10000u) {  // engine.cpp:229-245
      const uint32_t code = f >> 16;
      const char* what = code == 1 ? "contribution != acc" : code == 2 ? "residual not cleared"
                                                                      : "unselected residual changed";
      std::snprintf(msg, sizeof msg, "conservation violated: %s at t=%lld", what,
                    (long long)h->verify_t);
    } else {
      const char* field = (f & 1) ? "delta" : (f & 2) ? "k_t" : (f & 4) ? "topology" : "x";
      std::snprintf(msg, sizeof msg, "replicated state diverged at iteration %lld: rank %u field %s",
                    (long long)h->verify_t, (f >> 8) & 0xffu, field);
    }
    *h->verify_flag = 0;
    return set_err(EXD_EINVARIANT, msg);
  }
  if (h->has_record) {
    for (auto& wk : h->w) {
      CU(cudaMemcpy(wk.raw_host, wk.rec_dev + ((h->t - 1) % kRecRing), sizeof(RawRecord),
                    cudaMemcpyDeviceToHost));
      finalize_record(*wk.raw_host, h->cfg, h->opt.sparsifier, wk.rec_host);
    }
  }
  if (out) {
    if (!h->has_record) std::memset(out, 0, sizeof(*out));
    else std::memcpy(out, h->w[0].rec_host, sizeof(*out));
  }
  return EXD_OK;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

const char* exd_last_error(void) { return g_err.c_str(); }
int32_t exd_version(void) { return 1; }

int exd_validate(const exd_config* in, exd_config* out) {
  if (!in || !out) return set_err(EXD_EINVAL, "null argument");
  return validate_cfg(in, out);
}

int64_t exd_default_block_count(int32_t n) { return 64 * (int64_t)n; }

int exd_build_topology(int64_t n_g, int64_t n_b, int32_t n, int64_t min_blk, exd_topology* out,
                       char* warning, size_t warning_len) {
  std::string w;
  const int rc = build_topo(n_g, n_b, n, min_blk, out, &w);
  if (warning && warning_len) {
    std::strncpy(warning, w.c_str(), warning_len - 1);
    warning[warning_len - 1] = 0;
  }
  return rc;
}

int exd_partition_range(const exd_topology* topo, int32_t p, int64_t n_g, int64_t* st,
                        int64_t* end) {
  if (p < 0 || p >= topo->n) return set_err(EXD_EINVAL, "partition out of range");
  partition_range(*topo, p, n_g, st, end);
  return EXD_OK;
}

int exd_rotate_to_partition_order(const int64_t* k_rank, int64_t t, int32_t n, int64_t* k_part) {
  if (n < 1 || n > EXD_MAX_WORKERS) return set_err(EXD_EINVAL, "partial-k length mismatch");
  rotate(k_rank, t, n, k_part);
  return EXD_OK;
}

int exd_adjust_topology(exd_topology* topo, int64_t* k_part, double alpha, int64_t blk_move,
                        int64_t min_blk, int64_t n_g, int32_t* moves, int32_t* skips) {
  int32_t mv = 0, sk = 0;
  adjust(*topo, k_part, alpha, blk_move, min_blk, n_g, &mv, &sk);
  if (moves) *moves = mv;
  if (skips) *skips = sk;
  return EXD_OK;
}

int exd_allocate_partition(const exd_topology* topo, int64_t t, int32_t rank, int64_t n_g,
                           int32_t* partition, int64_t* st, int64_t* end) {
  const int p = allocate(*topo, t, rank, n_g, st, end);
  if (partition) *partition = p;
  return EXD_OK;
}

double exd_scale_threshold(int64_t k, int64_t k_prime, double delta, double beta, double gamma) {
  return scale_threshold(k, k_prime, delta, beta, gamma);
}

int exd_gather_stats_of(const int64_t* k_rank, int32_t n, exd_gather_stats* out) {
  if (n < 1 || n > EXD_MAX_WORKERS) return set_err(EXD_EINVAL, "worker count out of range");
  gather_stats(k_rank, n, out);
  return EXD_OK;
}

int exd_initial_threshold_device(const void* mags_dev, int64_t m, int32_t dtype, double d,
                                 double* out) {
  if (m < 1) return set_err(EXD_EINVAL, "initial_threshold: empty sample");
  int64_t pos = (int64_t)std::floor((1.0 - d) * (double)m);
  if (pos > m - 1) pos = m - 1;
  void* scratch = nullptr;
  void* bits = nullptr;
  CU(cudaMalloc(&scratch, quantile_scratch_bytes()));
  CU(cudaMalloc(&bits, 16));
  CU(launch_quantile(mags_dev, m, pos, dtype, scratch, bits, 0));
  if (dtype == EXD_F64) {
    CU(cudaMemcpy(out, bits, 8, cudaMemcpyDeviceToHost));
  } else {
    float f;
    CU(cudaMemcpy(&f, bits, 4, cudaMemcpyDeviceToHost));
    *out = (double)f;
  }
  cudaFree(scratch);
  cudaFree(bits);
  return EXD_OK;
}

}  // extern "C"

namespace {
// topk_select / hard_threshold_select (baselines.cpp:26-46) on the device
int baseline_select(const void* acc, int64_t n_g, int32_t dtype, int topk, int64_t k,
                    double delta, int32_t* idx, int64_t cap, int64_t* count, void* stream) {
  if (dtype != EXD_F32 && dtype != EXD_F64) return set_err(EXD_EINVAL, "dtype out of range");
  if (n_g < 0 || n_g > 0x7fffffffLL) return set_err(EXD_EINVAL, "n_g out of range");
  if (topk && (k < 1 || k > n_g)) return set_err(EXD_EINVAL, "topk_select: k out of range");
  if (n_g == 0) {
    if (count) *count = 0;
    return EXD_OK;
  }
  if (!acc || (!idx && cap > 0)) return set_err(EXD_EINVAL, "null argument");
  // run on the device that owns acc (the caller's current device may differ)
  int prev = 0, dev = 0;
  CU(cudaGetDevice(&prev));
  dev = prev;
  {
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, acc) == cudaSuccess && pa.type == cudaMemoryTypeDevice)
      dev = pa.device;
    cudaGetLastError();
  }
  if (dev != prev) CU(cudaSetDevice(dev));
  struct Restore {
    int d, p;
    ~Restore() { if (d != p) cudaSetDevice(p); }
  } restore{dev, prev};
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // Grow-only scratch per device, plus a pinned read-back slot; the call is
  // synchronous, so one caller at a time holds them.
  struct Scratch {
    void* dev = nullptr;
    size_t bytes = 0;
    int64_t* host = nullptr;
  };
  static std::mutex mu;
  static Scratch cache[64];
  if (dev < 0 || dev >= 64) return set_err(EXD_EINVAL, "device ordinal out of range");
  std::lock_guard<std::mutex> lock(mu);
  Scratch& sc = cache[dev];
  const size_t sb = baseline_scratch_bytes(n_g) + 3 * sizeof(int64_t);
  if (sc.bytes < sb) {
    if (sc.dev) {
      CU(cudaStreamSynchronize(s));
      CU(cudaFree(sc.dev));
      sc.dev = nullptr;
      sc.bytes = 0;
    }
    CU(cudaMalloc(&sc.dev, sb));
    sc.bytes = sb;
  }
  if (!sc.host) CU(cudaMallocHost(&sc.host, 3 * sizeof(int64_t)));
  void* scratch = sc.dev;
  int64_t* totals = reinterpret_cast<int64_t*>(static_cast<char*>(scratch) + sb - 3 * sizeof(int64_t));
  cudaError_t e = launch_baseline_select(acc, n_g, dtype, topk, k, delta, idx, cap, totals,
                                         scratch, s);
  int64_t* host = sc.host;
  if (e == cudaSuccess) e = cudaMemcpyAsync(host, totals, 3 * sizeof(int64_t), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return set_err(EXD_ECUDA, std::string("baseline select: ") + cudaGetErrorString(e));
  const int64_t n_sel = host[0] + host[2];
  if (topk && n_sel != k) return set_err(EXD_EINVARIANT, "topk_select: selected count != k");
  if (count) *count = n_sel;
  return EXD_OK;
}
}  // namespace

extern "C" {

int exd_topk_select_device(const void* acc_dev, int64_t n_g, int32_t dtype, int64_t k,
                           int32_t* idx_dev, int64_t cap, void* cuda_stream) {
  if (cap < k) return set_err(EXD_EINVAL, "topk_select: output capacity below k");
  return baseline_select(acc_dev, n_g, dtype, 1, k, 0.0, idx_dev, cap, nullptr, cuda_stream);
}

int exd_hard_threshold_select_device(const void* acc_dev, int64_t n_g, int32_t dtype,
                                     double fixed_delta, int32_t* idx_dev, int64_t cap,
                                     int64_t* count, void* cuda_stream) {
  return baseline_select(acc_dev, n_g, dtype, 0, 0, fixed_delta, idx_dev, cap, count, cuda_stream);
}

int exd_synthetic_gradient(const exd_stream_spec* spec, int64_t t, int32_t rank, int32_t dtype,
                           void* out_dev, void* cuda_stream) {
  if (!spec || spec->nseg < 1 || spec->nseg > EXD_MAX_SEGMENTS)
    return set_err(EXD_EINVAL, "stream has no segments");
  int64_t total = 0;
  for (int i = 0; i < spec->nseg; ++i) {
    if (spec->seg_length[i] < 1) return set_err(EXD_EINVAL, "segment length out of range");
    if (!(spec->seg_scale[i] > 0.0)) return set_err(EXD_EINVAL, "segment scale out of range");
    total += spec->seg_length[i];
  }
  if (total != spec->n_g) return set_err(EXD_EINVAL, "segment lengths do not sum to n_g");
  CU(launch_synthetic(spec, t, rank, dtype, out_dev, (cudaStream_t)cuda_stream));
  return EXD_OK;
}

int exd_engine_create(const exd_config* cfg, const exd_options* opt, const int32_t* devices,
                      int32_t ndev, exd_engine** out) {
  if (!cfg || !opt || !out) return set_err(EXD_EINVAL, "null argument");
  if (ndev > 1 && cfg->n > 1)
    return set_err(EXD_EUNSUPPORTED,
                   "in-process workers share one device; use exd_engine_create_rank per GPU");
  auto* h = new exd_engine;
  h->dist = false;
  h->device = (devices && ndev > 0) ? devices[0] : 0;
  const int rc = setup(h, cfg, opt, 0, cfg->n > 0 ? cfg->n : 1);
  if (rc) {
    const std::string msg = g_err;
    teardown(h);
    delete h;
    g_err = msg;
    return rc;
  }
  *out = h;
  return EXD_OK;
}

int exd_nccl_unique_id(uint8_t* out) {
  Nccl& nc = nccl();
  if (!nc.ok) return set_err(EXD_ENCCL, nc.why);
  ncclUniqueId id;
  NC(nc.GetUniqueId(&id));
  std::memcpy(out, &id, EXD_NCCL_ID_BYTES);
  return EXD_OK;
}

int exd_engine_create_rank(const exd_config* cfg, const exd_options* opt, int32_t rank,
                           int32_t device, const uint8_t* nccl_id, exd_engine** out) {
  if (!cfg || !opt || !out) return set_err(EXD_EINVAL, "null argument");
  if (rank < 0 || rank >= cfg->n) return set_err(EXD_EINVAL, "rank out of range");
  auto* h = new exd_engine;
  h->dist = true;
  h->device = device;
  int rc = setup(h, cfg, opt, rank, 1);
  if (!rc && cfg->n > 1) {
    Nccl& nc = nccl();
    if (!nc.ok) {
      rc = set_err(EXD_ENCCL, nc.why);
    } else {
      ncclUniqueId id;
      std::memcpy(&id, nccl_id, EXD_NCCL_ID_BYTES);
      cudaSetDevice(device);
      ncclResult_t r = nc.CommInitRank(&h->comm, cfg->n, id, rank);
      if (r != ncclSuccess) rc = set_err(EXD_ENCCL, std::string("ncclCommInitRank: ") + nc.GetErrorString(r));
      // the baseline sparsifiers' overlapping lists go through NCCL (all-gather +
      // deduplicating union on every rank); ExDyna uses the peer-memory sync
      if (!rc && opt->sync_mode != EXD_SYNC_NCCL && opt->sparsifier == EXD_SPARSIFIER_EXDYNA)
        rc = setup_p2p(h);
    }
  }
  if (rc) {
    const std::string msg = g_err;
    teardown(h);
    delete h;
    g_err = msg;
    return rc;
  }
  *out = h;
  return EXD_OK;
}

void exd_engine_destroy(exd_engine* h) {
  teardown(h);
  delete h;
}

int32_t exd_engine_local_workers(const exd_engine* h) { return (int32_t)h->w.size(); }
int32_t exd_engine_first_rank(const exd_engine* h) { return h->w.empty() ? 0 : h->w[0].rank; }
int64_t exd_engine_iteration(const exd_engine* h) { return h->t; }
int32_t exd_engine_sync_mode(const exd_engine* h) {
  return !h->dist ? -1 : !h->p2p ? EXD_SYNC_NCCL : h->xchg ? EXD_SYNC_P2P : EXD_SYNC_P2P_PULL;
}
void* exd_engine_stream(const exd_engine* h, int32_t) { return (void*)h->stream; }

int exd_engine_step_async(exd_engine* h, const void* const* grads_dev) {
  return enqueue_step(h, grads_dev);
}

int exd_engine_sync(exd_engine* h, exd_record* out) { return sync_engine(h, out); }

int exd_engine_records(exd_engine* h, int64_t first, int64_t count, exd_record* out) {
  if (int rc = sync_engine(h, nullptr)) return rc;
  if (count == 0) return EXD_OK;
  if (!out || count < 0 || first < 0 || first + count > h->t)
    return set_err(EXD_EINVAL, "record range out of range");
  if (h->t - first > kRecRing) return set_err(EXD_EINVAL, "records no longer on the device");
  std::vector<RawRecord> raw((size_t)count);
  const Worker& wk = h->w[0];
  int64_t done = 0;
  while (done < count) {  // the ring may wrap
    const int64_t slot = (first + done) % kRecRing;
    const int64_t run = std::min<int64_t>(count - done, kRecRing - slot);
    CU(cudaMemcpy(raw.data() + done, wk.rec_dev + slot, sizeof(RawRecord) * (size_t)run,
                  cudaMemcpyDeviceToHost));
    done += run;
  }
  for (int64_t i = 0; i < count; ++i) finalize_record(raw[(size_t)i], h->cfg, h->opt.sparsifier, out + i);
  return EXD_OK;
}

int exd_engine_step(exd_engine* h, const void* const* grads_dev, exd_record* out) {
  if (int rc = enqueue_step(h, grads_dev)) return rc;
  return sync_engine(h, out);
}

int exd_engine_step_host(exd_engine* h, const void* const* grads_host, exd_record* out) {
  const size_t bytes = h->esz * (size_t)h->cfg.n_g;
  std::vector<const void*> dev(h->w.size());
  CU(cudaSetDevice(h->device));
  for (size_t i = 0; i < h->w.size(); ++i) {
    Worker& wk = h->w[i];
    if (!wk.grad_stage) CU(cudaMalloc(&wk.grad_stage, bytes));
    CU(cudaMemcpyAsync(wk.grad_stage, grads_host[i], bytes, cudaMemcpyHostToDevice, h->stream));
    dev[i] = wk.grad_stage;
  }
  return exd_engine_step(h, dev.data(), out);
}

int exd_engine_get_state(exd_engine* h, int32_t w, exd_worker_state* out) {
  if (w < 0 || w >= (int)h->w.size()) return set_err(EXD_EINVAL, "worker out of range");
  CU(cudaSetDevice(h->device));
  CU(cudaStreamSynchronize(h->stream));
  Ctrl c;
  CU(cudaMemcpy(&c, h->w[w].ctrl, sizeof(c), cudaMemcpyDeviceToHost));
  std::memset(out, 0, sizeof(*out));
  out->t = c.t;
  out->rank = h->w[w].rank;
  out->delta = c.delta;
  out->partition = c.last.partition;
  out->st = c.last.st;
  out->end = c.last.end;
  for (int i = 0; i < h->n; ++i) out->k_t[i] = c.k_t[i];
  out->topology = c.topo;
  return EXD_OK;
}

}  // extern "C"

namespace {
// (pointer, length, element size) of one EXD_VEC_* vector of worker w
int vector_of(exd_engine* h, int32_t w, int32_t which, const void** src, int64_t* n_el,
              size_t* es_out) {
  if (w < 0 || w >= (int)h->w.size()) return set_err(EXD_EINVAL, "worker out of range");
  if (int rc = sync_engine(h, nullptr)) return rc;
  Worker& wk = h->w[w];
  const exd_record& rec = *wk.rec_host;
  size_t es = h->esz;
  switch (which) {
    case EXD_VEC_X: *n_el = h->cfg.n_g; *src = wk.x; break;
    case EXD_VEC_E: *n_el = h->cfg.n_g; *src = wk.e; break;
    case EXD_VEC_IDX_GLOBAL:
      *n_el = h->has_record ? rec.union_count : 0;
      *src = h->baseline     ? (const void*)h->w[0].idx_global  // one shared union
             : h->union_flow ? (const void*)wk.idx_global
                             : (const void*)wk.idx;
      es = 4;
      break;
    case EXD_VEC_LOCAL_IDX:
    case EXD_VEC_LOCAL_VAL: {
      CountRec cr;
      CU(cudaMemcpy(&cr, wk.cnt, sizeof(cr), cudaMemcpyDeviceToHost));
      *n_el = h->has_record ? cr.k : 0;
      *src = which == EXD_VEC_LOCAL_IDX ? (const void*)wk.idx : wk.val;
      if (which == EXD_VEC_LOCAL_IDX) es = 4;
      break;
    }
    case EXD_VEC_BLOCK_COUNTS:
      *n_el = h->cfg.n_b;
      // counted on demand from the worker's own selection of the last step
      if (h->has_record && !h->baseline)
        CU(launch_block_counts(wk.idx, wk.cnt, h->cap_part, wk.blk, wk.rc, h->stream));
      else
        CU(cudaMemsetAsync(wk.blk, 0, 4 * (size_t)h->cfg.n_b, h->stream));
      CU(cudaStreamSynchronize(h->stream));
      *src = wk.blk;
      es = 4;
      break;
    case EXD_VEC_SUM:
      *n_el = h->has_record ? rec.union_count : 0;
      *src = h->union_flow ? h->sum : wk.val;
      break;
    default:
      return set_err(EXD_EINVAL, "unknown vector");
  }
  *es_out = es;
  return EXD_OK;
}
}  // namespace

extern "C" {

int exd_engine_copy_out(exd_engine* h, int32_t w, int32_t which, void* host, int64_t cap,
                        int64_t* len) {
  const void* src = nullptr;
  int64_t n_el = 0;
  size_t es = 0;
  if (int rc = vector_of(h, w, which, &src, &n_el, &es)) return rc;
  if (len) *len = n_el;
  if (!host) return EXD_OK;
  if (n_el > cap) return set_err(EXD_EINVAL, "host buffer too small");
  if (n_el) CU(cudaMemcpy(host, src, es * (size_t)n_el, cudaMemcpyDeviceToHost));
  return EXD_OK;
}

int exd_engine_device_vector(exd_engine* h, int32_t w, int32_t which, void** ptr, int64_t* len) {
  const void* src = nullptr;
  int64_t n_el = 0;
  size_t es = 0;
  if (int rc = vector_of(h, w, which, &src, &n_el, &es)) return rc;
  if (ptr) *ptr = const_cast<void*>(src);
  if (len) *len = n_el;
  return EXD_OK;
}

int exd_engine_copy_in(exd_engine* h, int32_t w, int32_t which, const void* host, int64_t n_el) {
  if (w < 0 || w >= (int)h->w.size()) return set_err(EXD_EINVAL, "worker out of range");
  if (which != EXD_VEC_X && which != EXD_VEC_E) return set_err(EXD_EINVAL, "only x and e are writable");
  if (n_el != h->cfg.n_g) return set_err(EXD_EINVAL, "length != n_g");
  CU(cudaSetDevice(h->device));
  CU(cudaStreamSynchronize(h->stream));
  CU(cudaMemcpy(which == EXD_VEC_X ? h->w[w].x : h->w[w].e, host, h->esz * (size_t)n_el,
                cudaMemcpyHostToDevice));
  return EXD_OK;
}

int exd_engine_kernel_stats(exd_engine* h, exd_kernel_stats* out) {
  if (int rc = sync_engine(h, nullptr)) return rc;
  *out = h->stats;
  return EXD_OK;
}

int exd_engine_set_profile(exd_engine* h, int32_t on) {
  if (int rc = sync_engine(h, nullptr)) return rc;
  h->opt.profile_kernels = on ? 1 : 0;
  return EXD_OK;
}

int exd_engine_reset_kernel_stats(exd_engine* h) {
  if (int rc = sync_engine(h, nullptr)) return rc;
  std::memset(&h->stats, 0, sizeof(h->stats));
  return EXD_OK;
}

int exd_flush_l2(int32_t device, void* cuda_stream) {
  static void* buf[16] = {nullptr};
  static size_t bytes = 0;
  if (device < 0 || device >= 16) return set_err(EXD_EINVAL, "device out of range");
  CU(cudaSetDevice(device));
  if (!buf[device]) {
    int l2 = 0;
    CU(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device));
    bytes = (size_t)l2 * 2 + (64u << 20);
    CU(cudaMalloc(&buf[device], bytes));
  }
  CU(launch_l2_flush(buf[device], bytes, (cudaStream_t)cuda_stream));
  return EXD_OK;
}

}  // extern "C"
