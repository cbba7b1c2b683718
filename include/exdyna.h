/*
 * exdyna.h — C ABI of the B200-native ExDyna sparsify+sync path.
 *
 * This is the drop-in boundary for the reference's C++ sparsifier API
 * (`sparsim`, /root/reference/proj). Every entry point below names the
 * reference interface it replaces (file:line, relative to proj/). Types are
 * plain C: fixed-size PODs, int64 counts, raw pointers and sizes; no C++ or
 * torch types cross this boundary.
 *
 * Error model (mirrors the reference's exception classes):
 *   EXD_EINVAL      <-> std::invalid_argument   (config.cpp:29-49, engine.cpp:55-61)
 *   EXD_EINVARIANT  <-> sparsim::EngineError    (engine.hpp:47-50, engine.cpp:229-306)
 *   EXD_ECUDA / EXD_ENCCL / EXD_ENOMEM / EXD_EUNSUPPORTED: device-side failures.
 * Every non-zero status sets a thread-local message readable with
 * exd_last_error(); for EXD_EINVAL the text equals the reference's what().
 *
 * Threading contract: one host thread drives one engine handle; each local
 * worker owns one CUDA stream. exd_engine_step() returns after the record is
 * on the host (like sparsim::Engine::step); exd_engine_step_async() only
 * enqueues and the record is collected with exd_engine_sync().
 */
#ifndef EXDYNA_H
#define EXDYNA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EXD_MAX_WORKERS 64
#define EXD_MAX_SEGMENTS 64
#define EXD_NCCL_ID_BYTES 128

enum {
  EXD_OK = 0,
  EXD_EINVAL = 1,
  EXD_EINVARIANT = 2,
  EXD_ECUDA = 3,
  EXD_ENCCL = 4,
  EXD_ENOMEM = 5,
  EXD_EUNSUPPORTED = 6
};

/* element type of the gradient / residual / model vectors */
enum { EXD_F32 = 0, EXD_F64 = 1 };

/* engine.hpp:35 SparsifierKind (only ExDyna is on the hot path) */
enum { EXD_SPARSIFIER_EXDYNA = 0, EXD_SPARSIFIER_TOPK = 1,
       EXD_SPARSIFIER_CLTK = 2, EXD_SPARSIFIER_HARD_THRESHOLD = 3 };

/* SparsifierConfig, config.hpp:28-45. std::optional fields carry a has_ flag. */
typedef struct exd_config {
  int32_t n;                 /* worker count */
  int32_t has_delta0;
  int64_t n_g;               /* gradients in the model */
  int64_t n_b;               /* blocks in the gradient vector */
  double d;                  /* target density in (0, 1] */
  int64_t k;                 /* llround(d * n_g); filled by exd_validate */
  double delta0;             /* initial threshold when has_delta0 */
  double alpha;              /* imbalance trigger ratio (> 1) */
  double beta;               /* density band ratio (> 1) */
  double gamma;              /* threshold scaling step in (0, 1) */
  int64_t blk_move;          /* blocks moved per adjustment */
  int64_t min_blk;           /* minimum blocks a partition may keep */
  double eta;                /* learning rate */
  uint64_t seed;
  int32_t has_max_density_cap;
  int32_t reserved0;
  double max_density_cap;
} exd_config;

/* EngineOptions, engine.hpp:37-45, plus the device-side knobs of this build. */
typedef struct exd_options {
  int32_t sparsifier;            /* EXD_SPARSIFIER_*; only EXDYNA is supported */
  int32_t static_partitions;     /* freeze topology after the initial build */
  double fixed_delta;            /* hard-threshold only (unsupported here) */
  int32_t parallel_workers;      /* accepted for API parity; workers are streams */
  int32_t verify_replication;    /* bit-compare replicated state every step */
  int32_t verify_conservation;   /* deep error-feedback mass check (debug) */
  int32_t record_loss;           /* accepted; synthetic streams have no loss */
  int32_t dtype;                 /* EXD_F32 (default) or EXD_F64 (strict oracle mode) */
  int32_t profile_kernels;       /* time the fused select kernel with CUDA events */
  int32_t sync_mode;             /* one-rank-per-GPU sync: EXD_SYNC_* */
} exd_options;

/* exd_options.sync_mode (exd_engine_create_rank only) */
enum {
  EXD_SYNC_AUTO = 0,   /* NVLink peer memory when every peer is P2P-reachable, else NCCL */
  EXD_SYNC_NCCL = 1,   /* count all-gather, host wait, padded index all-gather, all-reduce */
  EXD_SYNC_P2P = 2,    /* peer-memory kernels, no host in the loop (fails if unavailable):
                          push-reduce (the stream kernel pushes its selection runs to the
                          peers; every rank pushes its contributions as {value, epoch}
                          words and sums them in rank order), or pull-reduce under a
                          density cap or verify_conservation */
  EXD_SYNC_P2P_PULL = 3  /* peer-memory kernels, pull-reduce always (index lists pushed
                            first, every rank sums the whole union from the peers'
                            contribution buffers) */
};

/* PartitionTopology, types.hpp:36-46 */
typedef struct exd_topology {
  int32_t n;
  int32_t reserved0;
  int64_t sz_blk;
  int64_t blk_part[EXD_MAX_WORKERS];
  int64_t blk_pos[EXD_MAX_WORKERS];
} exd_topology;

/* IterationRecord, types.hpp:84-103 */
typedef struct exd_record {
  int64_t t;
  int64_t k_prime;
  double density;
  double eps;
  int64_t m_t;
  int64_t c_t;
  double f_t;
  double global_err;
  double delta;
  int32_t has_loss;
  int32_t reserved0;
  double loss;
  int64_t duplicates;
  int64_t union_count;
  int32_t n;
  int32_t adjust_moves;
  int32_t adjust_skips;
  int32_t cap_hits;
  int32_t idle_workers;
  int32_t reserved1;
  int64_t k_rank[EXD_MAX_WORKERS];
} exd_record;

/* GatherResult accounting, collectives.hpp:30-39 (idx_global excluded) */
typedef struct exd_gather_stats {
  int64_t k_prime;
  int64_t m_t;
  int64_t c_t;
  double f_t;
} exd_gather_stats;

/* Replicated per-worker control state, WorkerState types.hpp:73-80 */
typedef struct exd_worker_state {
  int64_t t;                 /* next iteration to run */
  int32_t rank;
  int32_t partition;         /* partition searched in the last step */
  double delta;
  int64_t st, end;           /* last search range */
  int64_t k_t[EXD_MAX_WORKERS];
  exd_topology topology;
} exd_worker_state;

/* StreamSpec, workloads.hpp:121-129 */
typedef struct exd_stream_spec {
  int64_t n_g;
  int32_t nseg;
  int32_t distribution;      /* 0 Laplace, 1 LogNormal */
  int64_t seg_length[EXD_MAX_SEGMENTS];
  double seg_scale[EXD_MAX_SEGMENTS];
  double decay;
  int32_t has_decay_step;
  int32_t reserved0;
  int64_t decay_step;
  double decay_step_factor;
  uint64_t seed;
} exd_stream_spec;

/* vectors that exd_engine_copy_out / copy_in can address */
enum {
  EXD_VEC_X = 0,             /* model x (T, n_g) */
  EXD_VEC_E = 1,             /* residual e (T, n_g) */
  EXD_VEC_IDX_GLOBAL = 2,    /* union of the last step (int32, k') */
  EXD_VEC_LOCAL_IDX = 3,     /* own selection of the last step (int32, k_i) */
  EXD_VEC_LOCAL_VAL = 4,     /* own selected values (T, k_i) */
  EXD_VEC_BLOCK_COUNTS = 5,  /* per-block selection counts of the last step (int32, n_b) */
  EXD_VEC_SUM = 6            /* all-reduced values of the last step (T, k') */
};

typedef struct exd_kernel_stats {
  int64_t select_launches;   /* stream-kernel launches timed (accumulate+select+stage) */
  double select_ms;          /* summed CUDA-event time of those launches */
  int64_t steps;
  int64_t kernel_launches;   /* every kernel this library launched (all steps) */
  int64_t finish_launches;   /* finish-kernel launches timed (offsets, lists, epilogue) */
  double finish_ms;          /* summed CUDA-event time of those launches */
} exd_kernel_stats;

/* ---- status ---------------------------------------------------------- */
const char* exd_last_error(void);
int32_t exd_version(void);

/* ---- pure host functions (identical semantics to the reference) ------ */
/* validate(), config.cpp:28-51. Copies *in to *out and fills out->k. */
int exd_validate(const exd_config* in, exd_config* out);
/* default_block_count, config.hpp:49 */
int64_t exd_default_block_count(int32_t n);
/* build_topology, partition.cpp:22-58; warning may be NULL */
int exd_build_topology(int64_t n_g, int64_t n_b, int32_t n, int64_t min_blk,
                       exd_topology* out, char* warning, size_t warning_len);
/* partition_range, partition.cpp:60-68 */
int exd_partition_range(const exd_topology* topo, int32_t p, int64_t n_g,
                        int64_t* st, int64_t* end);
/* rotate_to_partition_order, allocator.cpp:23-38 (rank order in, partition order out) */
int exd_rotate_to_partition_order(const int64_t* k_rank, int64_t t, int32_t n,
                                  int64_t* k_part);
/* adjust_topology, allocator.cpp:40-90 (k_part in partition order, in place) */
int exd_adjust_topology(exd_topology* topo, int64_t* k_part, double alpha,
                        int64_t blk_move, int64_t min_blk, int64_t n_g,
                        int32_t* moves, int32_t* skips);
/* allocate_partition, allocator.cpp:92-99 */
int exd_allocate_partition(const exd_topology* topo, int64_t t, int32_t rank,
                           int64_t n_g, int32_t* partition, int64_t* st,
                           int64_t* end);
/* scale_threshold, threshold.cpp:23-35 */
double exd_scale_threshold(int64_t k, int64_t k_prime, double delta,
                           double beta, double gamma);
/* all_gather accounting, collectives.cpp:22-45 */
int exd_gather_stats_of(const int64_t* k_rank, int32_t n, exd_gather_stats* out);

/* ---- device functions ----------------------------------------------- */
/* initial_threshold, threshold.cpp:37-47, as a device radix select over
 * |mags| (dtype elements, device pointer); result written to *out (host). */
int exd_initial_threshold_device(const void* mags_dev, int64_t m, int32_t dtype,
                                 double d, double* out);
/* Baseline sparsifiers, baselines.hpp:25-34 / baselines.cpp:26-46 (SURVEY
 * §8f row f4), over a device vector acc (dtype elements, n_g long). Indices
 * are ascending int32 written to idx_dev (device, capacity cap); enqueued on
 * cuda_stream, which the call synchronises, on the device that owns acc_dev.
 * Any element alignment is accepted (16-byte aligned vectors take 128-bit
 * loads, others a scalar path).
 * topk_select: exactly k indices, largest |acc| first, ties toward the lower
 * index; EXD_EINVAL "topk_select: k out of range" unless 1 <= k <= n_g. */
int exd_topk_select_device(const void* acc_dev, int64_t n_g, int32_t dtype, int64_t k,
                           int32_t* idx_dev, int64_t cap, void* cuda_stream);
/* hard_threshold_select: {j : |acc[j]| >= fixed_delta} compared in fp64;
 * *count (host) gets the full count, at most cap indices are written. */
int exd_hard_threshold_select_device(const void* acc_dev, int64_t n_g, int32_t dtype,
                                     double fixed_delta, int32_t* idx_dev, int64_t cap,
                                     int64_t* count, void* cuda_stream);
/* synthetic_gradient, workloads.cpp:62-85, generated on device (dtype). */
int exd_synthetic_gradient(const exd_stream_spec* spec, int64_t t, int32_t rank,
                           int32_t dtype, void* out_dev, void* cuda_stream);

/* ---- engine: sparsim::Engine, engine.hpp:61-105 ---------------------- */
typedef struct exd_engine exd_engine;

/* Engine::Engine, engine.cpp:51-88. All cfg->n workers live in this process,
 * worker w on devices[w % ndev] (ndev == 1: every worker shares one GPU, the
 * reference's simulated-worker mode). Collectives are device kernels. */
int exd_engine_create(const exd_config* cfg, const exd_options* opt,
                      const int32_t* devices, int32_t ndev, exd_engine** out);
/* One rank of a cfg->n-process data-parallel job (one worker per GPU);
 * collectives are NCCL over NVLink. nccl_id from exd_nccl_unique_id on rank 0. */
int exd_nccl_unique_id(uint8_t* out /* EXD_NCCL_ID_BYTES */);
int exd_engine_create_rank(const exd_config* cfg, const exd_options* opt,
                           int32_t rank, int32_t device, const uint8_t* nccl_id,
                           exd_engine** out);
void exd_engine_destroy(exd_engine* h);
int32_t exd_engine_local_workers(const exd_engine* h);
int32_t exd_engine_first_rank(const exd_engine* h);
int64_t exd_engine_iteration(const exd_engine* h);
/* collective path in use: EXD_SYNC_P2P (push-reduce), EXD_SYNC_P2P_PULL or EXD_SYNC_NCCL
   (-1: in-process workers) */
int32_t exd_engine_sync_mode(const exd_engine* h);
/* CUDA stream of local worker w (cudaStream_t as void*) */
void* exd_engine_stream(const exd_engine* h, int32_t w);

/* Engine::step, engine.cpp:274-350. grads[w] is the device gradient of local
 * worker w (dtype elements, n_g long, 16-byte aligned: the stream kernel reads
 * it with 128-bit loads; EXD_EINVAL "gradient pointer must be 16-byte aligned"
 * otherwise), produced on or before that worker's stream. Blocks until the
 * record is on the host. After a peer-memory sync timeout (EXD_ENCCL) the
 * engine refuses further steps. */
int exd_engine_step(exd_engine* h, const void* const* grads_dev, exd_record* out);
/* Enqueue one step without waiting for its record. */
int exd_engine_step_async(exd_engine* h, const void* const* grads_dev);
/* Wait for all enqueued steps; *out (may be NULL) gets the last record. */
int exd_engine_sync(exd_engine* h, exd_record* out);
/* Records of steps [first, first + count) after waiting for all enqueued steps
 * (Engine::run's record vector, engine.cpp:352-358). The device keeps the
 * last EXD_RECORD_RING steps; older ones give EXD_EINVAL. */
#define EXD_RECORD_RING 256
int exd_engine_records(exd_engine* h, int64_t first, int64_t count, exd_record* out);
/* Host-buffer step (GradientSource::gradient fills host memory,
 * workloads.hpp:77-87): copies grads_host[w] to the device on worker w's
 * stream, steps, and returns the record. */
int exd_engine_step_host(exd_engine* h, const void* const* grads_host, exd_record* out);

/* Engine::workers() / mutable_workers(), engine.hpp:72-74 */
int exd_engine_get_state(exd_engine* h, int32_t w, exd_worker_state* out);
int exd_engine_copy_out(exd_engine* h, int32_t w, int32_t which, void* host,
                        int64_t cap_elems, int64_t* len);
int exd_engine_copy_in(exd_engine* h, int32_t w, int32_t which, const void* host,
                       int64_t n_elems);
/* Device address and current length of one of the EXD_VEC_* vectors (valid
 * until exd_engine_destroy; contents valid after exd_engine_sync). The
 * zero-copy form of Engine::workers() for device-side consumers. */
int exd_engine_device_vector(exd_engine* h, int32_t w, int32_t which, void** ptr,
                             int64_t* len);
int exd_engine_kernel_stats(exd_engine* h, exd_kernel_stats* out);
/* Turn per-kernel CUDA-event timing on/off (exd_options.profile_kernels).
 * With it on, an event sits between the stream and finish kernels, which
 * also serialises their otherwise overlapped (programmatic) launch. */
int exd_engine_set_profile(exd_engine* h, int32_t on);
int exd_engine_reset_kernel_stats(exd_engine* h);

/* ---- ledger ------------------------------------- */
/* RunStats, runner.hpp:27-40 */
typedef struct exd_run_stats {
  int64_t iterations;
  double mean_density, mean_f, mean_eps;
  int64_t duplicates;
  int64_t adjust_moves, adjust_skips, cap_hits;
  double mean_idle_workers;
  double final_delta, final_global_err;
  int32_t has_final_loss;
  int32_t reserved0;
  double final_loss;
} exd_run_stats;

/* format_csv, runner.cpp:55-80: the same bytes (shortest round-trip doubles).
 * Writes at most cap bytes (NUL-terminated when room); *len gets the full length. */
int exd_format_csv(const exd_record* recs, int64_t count, char* out, size_t cap, size_t* len);
/* summarize, runner.cpp:89-113 */
int exd_summarize(const exd_record* recs, int64_t count, exd_run_stats* out);

/* Writes a buffer larger than L2 on worker w's device (timing hygiene). */
int exd_flush_l2(int32_t device, void* cuda_stream);

#ifdef __cplusplus
}
#endif

#endif /* EXDYNA_H */
