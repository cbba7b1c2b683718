// internal.cuh — device-resident state and kernel launch interfaces shared by
// kernels.cu and engine.cu. Not part of the C ABI.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "control.cuh"
#include "exdyna.h"

namespace exd {

// Per-step plan of one worker: the reference's accumulate-phase control
// (rotate -> adjust -> allocate, engine.cpp:125-131), computed on the device
// at the end of the previous step so the fused kernel never waits on the host.
struct Plan {
  exd_topology topo;        // topology after this step's adjust
  int64_t st, end;          // exclusive search range [st, end)
  int32_t partition;
  int32_t moves, skips;     // AdjustStats
  int32_t reserved;
};

// Replicated control state of one worker (WorkerState minus the vectors,
// types.hpp:73-80) plus the device-side bookkeeping of the fused kernel.
struct Ctrl {
  int64_t t;                // iteration the next step runs
  double delta;             // selection threshold (fp64, as the reference)
  float thr_f;              // __double2float_ru(delta): fp32 compare key
  int32_t has_delta;        // delta known (delta0 given or estimated)
  int32_t tmod;             // t mod n (keeps the epilogue free of 64-bit division)
  int32_t reserved_tm;
  int64_t k_t[EXD_MAX_WORKERS];  // last gathered counts, rank order
  exd_topology topo;        // committed topology (reference's WorkerState::topology)
  Plan plan[2];             // plan of step t lives in plan[t & 1]: the epilogue
                            // writes step t+1's plan while step t's is still read
  Plan last;                // plan the last completed step ran with
  // fused-kernel bookkeeping (self-resetting)
  uint32_t ticket;          // dynamic tile ticket
  uint32_t done;            // completed CTAs
  uint32_t epoch;           // look-back status epoch (never 0)
  uint32_t error;           // device-detected invariant violation (bitmask)
  int64_t k_local;          // own selection count of the running step
  double norm2;             // ||e_entering||^2 of the running step
};

// The device half of one ledger row (IterationRecord, engine.cpp:327-349): what
// the step produced. The host turns it into the exd_record at sync
// (finalize_record, engine.cu) with the reference's formulas, so the device
// epilogue only does the control work the next step needs.
struct RawRecord {
  int64_t t;
  double delta;                       // threshold the step selected with
  int32_t moves, skips;               // AdjustStats of the step's plan
  int32_t n, reserved;
  int64_t k_rank[EXD_MAX_WORKERS];    // gathered counts, rank order
  double norm2[EXD_MAX_WORKERS];      // ||e_entering||^2 per rank
  int64_t capped[EXD_MAX_WORKERS];    // the density cap trimmed that rank
  int64_t union_count;                // baseline sparsifiers: |idx_global| (deduplicated)
};

// What each rank contributes to the count all-gather (32 bytes).
struct CountRec {
  int64_t k;
  double norm2;
  int64_t capped;          // the density cap trimmed this rank's selection
  int64_t reserved;
};

// Everything a kernel needs to know about the run (by value).
struct RunConst {
  int64_t n_g, n_b, k;
  int32_t n, rank;
  double eta, alpha, beta, gamma;
  int64_t blk_move, min_blk;
  int32_t static_partitions;
  int32_t dtype;
  unsigned long long blk_magic;  // j / sz_blk == (j * blk_magic) >> blk_shift for j < 2^31
  int32_t blk_shift;
  int32_t fused;                 // n == 1 without a cap: x update + epilogue in the finish kernel
  int64_t cap;                   // per-rank density cap (engine.cpp:166-171); 0 = none
  double inv_alpha, inv_beta;    // 1/alpha, 1/beta (host IEEE quotients, identical on device)
};

struct SelectArgs {
  const void* g;            // T[n_g]   gradient (ACCUM)
  void* e;                  // T[n_g]   residual, in place
  void* x;                  // T[n_g]   model (fused n == 1 only)
  int32_t* idx;             // [cap]    own selection, ascending
  void* val;                // T[cap]   own selected values
  void* stage;              // [cap + 2 tiles] (index, value) pairs: warp-chunk staging runs
  int32_t* chunk_count;     // [tiles * kChunksPerTile] selected per warp chunk
  int32_t* tile_count;      // [tiles + 4] selected per tile (<= tile size)
  double* tile_norm;        // [tiles] ||e_entering||^2 partial per tile
  Ctrl* ctrl;
  CountRec* cnt_out;        // this rank's slot of the count all-gather
  RawRecord* rec;           // fused n == 1: this step's raw record
  int32_t tile_base;        // first tile covered by the stream launch
  int32_t num_tiles;        // tiles covered by the stream launch
  int64_t t;                // the step these kernels run (selects plan[t & 1])
  int32_t* const* push_idx;  // P2P pull: [n] my list slot in every peer's inbox (nullptr: none)
  int32_t npush;
  // P2P push-reduce: the stream kernel's pushes into every peer's inbox (by
  // value: kernel parameters are constant-bank reads, no pointer round trip)
  // ({payload, epoch} words, this step's parity)
  unsigned long long* push_stage[EXD_MAX_WORKERS];  // [k1_npush] my staged-index slot (peers, then own)
  unsigned long long* push_chunk[EXD_MAX_WORKERS];  // [k1_npush] my per-chunk count slot
  unsigned long long* push_tile[EXD_MAX_WORKERS];   // [k1_npush] my per-tile count slot
  int32_t k1_npush;             // 0: no pushes
  unsigned long long* range_words;  // finish kernel, large vectors: [3][kMaxCtas] published
                                    // range counts / ||e||^2 halves (nullptr: small vector)
  int32_t tile_pack;            // PUSH: staged indices packed per tile (1) or pushed as
                                // per-warp runs at the chunk's position (0)
  int32_t stage_keep;           // staged pairs small enough to keep in L2 (evict_last);
                                // else streamed (evict_first) so they do not crowd the
                                // 126 MB L2 at large k
};

constexpr int kMaxCtas = 2048;
constexpr int kBaseRoundTiles = 3072;  // tiles one round of the finish kernel's base sum covers
constexpr int kChunksPerTile = 8;  // one warp chunk per warp of the stream kernel

// union build + contribution gather + residual clear (K4 + K5)
struct UnionArgs {
  const int32_t* const* lists;  // [n] per-rank index lists (device); NULL -> padded
  const int32_t* padded;        // dist mode: all-gather recv buffer, stride m_t
  const CountRec* counts;       // [n] gathered counts
  const void* own_val;          // own selected values (T)
  void* e;                      // T residual, cleared at the union
  int32_t* idx_global;          // [k'] out
  void* contrib;                // T [k'] out
  const Ctrl* ctrl;
};

struct FinalizeArgs {
  const int32_t* idx_global;
  const void* sum;              // T [k'] all-reduced values
  void* x;
  Ctrl* ctrl;
  const CountRec* counts;       // [n]
  RawRecord* rec;               // this step's raw record
};

// ---- NVLink peer-memory sync (one rank per GPU, no host in the loop) --------
// Each rank exports one IPC region = its INBOX: one flag slot per source rank,
// one index-list slot per source rank, and its own contributions (two step-
// parity buffers). Senders PUSH into the receiver's inbox (posted NVLink
// stores); receivers poll their own local memory. Epochs are t + 1.
struct PeerFlags {                   // inbox[src] on the receiver
  unsigned long long count_epoch;    // src's {k, norm2} and index list of step epoch-1 arrived
  int64_t k;
  double norm2;
  unsigned long long contrib_epoch;  // src's contributions of step epoch-1 are readable
  int64_t capped;
  unsigned long long pad0[2];
  unsigned long long ll[3];          // push-reduce: {k, epoch}, {norm2 lo, epoch}, {norm2 hi, epoch}
  unsigned long long pad[6];         // 128 B: one slot per line
};
static_assert(sizeof(PeerFlags) == 128, "one flag slot per 128 B line");
static_assert(offsetof(PeerFlags, ll) % 16 == 8, "ll[1..2] is one 16 B vector store");

struct P2PArgs {
  PeerFlags* inbox;                  // [n] own inbox flag slots (local)
  PeerFlags* const* peer_slot;       // [n] my slot in every rank's inbox (remote; own = local)
  const int32_t* const* lists;       // [n] index lists: own `idx` or inbox list slot (local)
  void* const* contrib;              // [n] contribution buffers of this step's parity (remote; own local)
  const void* own_val;               // own selected values (T)
  void* e;
  void* x;
  int32_t* idx_global;               // [k'] union
  void* sum;                         // [k'] all-reduced values (T)
  CountRec* counts_all;              // [n] local copy of the gathered counts
  const CountRec* own_cnt;           // the finish kernel's {k_i, ||e||^2}
  Ctrl* ctrl;
  RawRecord* rec;
  unsigned long long epoch;          // t + 1
  unsigned int* err;                 // set on a peer timeout (device memory)
  unsigned long long* gate;          // [3] local gates: count / contrib epoch seen by block 0, arrive counter
  int32_t me;
};

// Push-reduce step (one rank per GPU, no density cap): replaces the finish
// kernel + p2p_sync. The stream kernel pushes its staged indices and counts
// into the peers' inboxes; the exchange kernel builds the union from them,
// pushes this rank's contributions into every inbox (coalesced posted stores)
// and sums the n local contribution slots in rank order.
struct ExchangeArgs {
  SelectArgs s;                      // the stream kernel's outputs, own idx/val, x, e, ctrl
  PeerFlags* inbox;                  // [2][n] own inbox flag slots by step parity (local)
  // pointer tables by value (constant bank)
  PeerFlags* peer_slot[EXD_MAX_WORKERS];        // my parity-0 flag slot in every rank's inbox
  // [step parity][source rank]: pushed staged-index runs / per-chunk / per-tile counts (local)
  // ({payload, epoch} words)
  const unsigned long long* stage_in[2][EXD_MAX_WORKERS];
  const unsigned long long* chunk_in[2][EXD_MAX_WORKERS];
  const unsigned long long* tile_in[2][EXD_MAX_WORKERS];
  void* contrib_out[2][EXD_MAX_WORKERS];        // [parity] my {value, epoch} slot in every inbox
  const void* contrib_in[2][EXD_MAX_WORKERS];   // [parity] {value, epoch} slots by source (local)
  // holder sum (n >= 4): contributions go to the partition's holder only, which
  // sums them and sends the sums to everyone: 2(n-1)/n instead of n-1 words
  // per union entry leave each GPU, for one more NVLink flight
  int32_t holder_sum;
  void* sum_out[2][EXD_MAX_WORKERS];            // [parity] the sum slot of every rank's inbox
  const void* sum_in[2];                        // [parity] own sum slot (local)
  int32_t* idx_global;               // [k'] union, partition order
  void* sum;                         // [k'] aggregated values (T)
  CountRec* counts_all;              // [n] local copy of the gathered counts
  RawRecord* rec;
  unsigned long long epoch;          // t + 1
  unsigned int* err;                 // set on a peer timeout (device memory)
  int32_t me;
  int32_t two_pass;                  // large k': the work loop in two passes (exchange_kernel)
  // bounded contribution slots: union positions >= xcap are not pushed; each
  // source writes them to its exported spill buffer, raises a per-block flag
  // in every peer's inbox, and the peers pull them (pass 2)
  int64_t xcap;
  void* spill_peer[2][EXD_MAX_WORKERS];                 // [parity][source] spill buffers
  unsigned long long* spill_flag_out[2][EXD_MAX_WORKERS];  // [parity][dest] my flag row
  unsigned long long* spill_flag_in[2];                  // [parity] own flags [source][block]
  unsigned long long* xrange_words;  // large vectors: [3][kMaxCtas] work blocks' range counts
                                     // and ||e||^2 halves as {payload, epoch} words
                                     // (nullptr: small vector)
};

// kernel launchers (kernels.cu)
int tile_elems(int dtype);
int64_t num_tiles(int64_t n_g, int dtype);
cudaError_t launch_stream(int mode, SelectArgs a, RunConst rc, cudaStream_t s);
cudaError_t launch_finish(SelectArgs a, RunConst rc, cudaStream_t s);
cudaError_t launch_union(UnionArgs a, RunConst rc, cudaStream_t s);
cudaError_t launch_allreduce_local(const void* const* contribs, void* sum, const Ctrl* ctrl,
                                   const CountRec* counts, RunConst rc, cudaStream_t s);
cudaError_t launch_finalize(FinalizeArgs a, RunConst rc, cudaStream_t s);
cudaError_t launch_set_delta(Ctrl* const* ctrls, int nctrl, const void* src_bits, int dtype,
                             cudaStream_t s);
cudaError_t launch_quantile(const void* v, int64_t m, int64_t pos, int dtype, void* scratch,
                            void* out_bits, cudaStream_t s);
size_t quantile_scratch_bytes();
int quantile_launches(int dtype);  // kernels one launch_quantile enqueues
cudaError_t launch_verify_replication(const Ctrl* c0, const Ctrl* cw, const void* x0,
                                      const void* xw, int64_t n_g, int dtype, int32_t w,
                                      uint32_t* flag, cudaStream_t s);
cudaError_t launch_l2_flush(void* buf, size_t bytes, cudaStream_t s);
// per-block counts of a worker's own selection (EXD_VEC_BLOCK_COUNTS), on demand
cudaError_t launch_block_counts(const int32_t* idx, const CountRec* cnt, int64_t cap, int32_t* out,
                                RunConst rc, cudaStream_t s);
// density cap (selector.cpp:44-61) on the compacted own selection
struct CapArgs {
  int32_t* idx;                  // [k_i] own selection, ascending (compacted in place)
  void* val;                     // [k_i] own values (T)
  void* e;                       // residual: dropped elements get their acc back
  CountRec* cnt;                 // own {k_i, norm2, capped}
  Ctrl* ctrl;
  int32_t* const* push;          // P2P: [npush] my list slot in every peer's inbox
  int32_t npush;
};
cudaError_t launch_cap(const CapArgs& a, RunConst rc, cudaStream_t s);
cudaError_t launch_replica_hash(const Ctrl* c, const void* x, unsigned long long* out4, RunConst rc,
                                cudaStream_t s);
cudaError_t launch_replica_compare(const unsigned long long* all4, int n, uint32_t* flag,
                                   cudaStream_t s);
cudaError_t launch_snapshot(const void* e, const void* g, void* snap, RunConst rc, cudaStream_t s);
cudaError_t launch_conservation(const int32_t* uni, const CountRec* counts, int ncounts,
                                const void* contrib, const void* e, const void* snap,
                                uint32_t* bitmap, uint32_t* flag, RunConst rc, cudaStream_t s);
cudaError_t launch_p2p_sync(const P2PArgs& a, RunConst rc, cudaStream_t s);
cudaError_t launch_exchange(const ExchangeArgs& a, RunConst rc, cudaStream_t s);
// baseline sparsifiers (baselines.cpp:26-46), baselines.cu
size_t baseline_scratch_bytes(int64_t n_g);
cudaError_t launch_baseline_select(const void* acc, int64_t n_g, int dtype, int topk, int64_t k,
                                   double delta, int32_t* out, int64_t cap, int64_t* totals_dev,
                                   void* scratch, cudaStream_t s);
cudaError_t launch_synthetic(const exd_stream_spec* spec, int64_t t, int32_t rank, int dtype,
                             void* out, cudaStream_t s);
// Engine runs of the baseline sparsifiers (baseline_engine.cu)
size_t baseline_union_scratch_bytes(int64_t n_g);
int baseline_union_launches(int n);
cudaError_t launch_baseline_counts(const int64_t* totals, const double* tile_norm, int ntiles,
                                   CountRec* cnt, cudaStream_t s);
cudaError_t launch_baseline_union(const int32_t* const* lists_host, const CountRec* counts, int n,
                                  int64_t cap, int64_t n_g, void* scratch, int32_t* uni,
                                  CountRec* ucnt, cudaStream_t s);
cudaError_t launch_baseline_gather_clear(const int32_t* uni, const CountRec* ucnt, void* e,
                                         void* contrib, int64_t cap, int dtype, cudaStream_t s);
cudaError_t launch_baseline_sum(const void* const* contribs_dev, int n, const CountRec* ucnt,
                                void* sum, int64_t cap, int dtype, cudaStream_t s);
cudaError_t launch_baseline_apply(const int32_t* uni, const CountRec* ucnt, const void* sum,
                                  void* x, int n, int64_t cap, int dtype, cudaStream_t s);
cudaError_t launch_baseline_epilogue(Ctrl* ctrl, const CountRec* counts, const CountRec* ucnt,
                                     RawRecord* rec, int n, double delta_used, cudaStream_t s);

// modes of the stream kernel
enum SelectMode {
  kFused = 0,        // accumulate + select + stage (steady state)
  kAccumulate = 1,   // t = 0 without delta0: accumulate only
  kSelectOnly = 2,   // t = 0 without delta0: select over the partition only
};

}  // namespace exd
