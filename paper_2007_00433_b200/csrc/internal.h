// internal.h -- libsesgd internals shared by the C ABI (sesgd_capi.cu), the host
// scheduler (schedule.cpp) and the kernels (resident.cu, p2p.cu).  Not installed.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/sesgd.h"

namespace sesgd {

// ---------------------------------------------------------------- host scheduler
// A1 (Alg.1 lines 1, 9-10), readings R1-R6 of DESIGN.md.
// canon[n]: canonical partition, group_of[n]: group index per worker.
void shuffle_exchange_groups(uint64_t seed, int64_t t, int n, int m, int32_t *canon,
                             int32_t *group_of);
// NEXT-3: Stone's dimension-exchange schedule (n, m powers of two).
void dimension_exchange_groups(int64_t t, int n, int m, int32_t *canon, int32_t *group_of);
// Eq. 2 / Eq. 3 exact forms (A6/A7).
void latency_model(int n, int m, double bytes, double nu, double tau, sesgd_cost *out);

// ---------------------------------------------------------------- kernels
constexpr int kMaxLocal = SESGD_MAX_WORKERS;

// Device-resident iteration state (SESGD_OPT_DEVICE_ITER; iter.cu): the iteration t, its
// schedule and the call history of the multi-GPU kernels live in device memory, so one captured
// CUDA graph of [sesgd_begin_iter_device, sync launches] replays every iteration.  Every worker
// derives its groups on the device from the shared seed, with no message.
struct DevIter {
  int64_t t;              // current iteration (its schedule is below)
  int64_t seq;            // multi-GPU sync launches of this context so far
  uint64_t claim_base;    // K4W / K4W-M chunk-claim counter before the next launch
  unsigned int fin;       // CTAs of the running launch that finished (the last one advances)
  int32_t ring_pos;       // K5: position of local slot 0 in its group
  int8_t canon[SESGD_MAX_WORKERS], group_of[SESGD_MAX_WORKERS];
  int8_t member_slot[SESGD_MAX_WORKERS];  // K6: canon mapped to local slots (every worker local)
  int8_t my_pos[SESGD_MAX_WORKERS];       // per local slot: position in its group
  int8_t slot_kind[SESGD_MAX_WORKERS];    // per local slot: as P2PArgs::slot_kind
  int8_t ring_rank[SESGD_MAX_WORKERS];    // K5: rank of ring position q (local slot 0's group)
};
struct DevBucket {
  int64_t calls;    // sync launches that covered the bucket
  int64_t hist[2];  // launch sequence numbers of the last two calls, by call parity
};
// static inputs of the begin kernel (host-side attach / layout data)
struct IterBeginArgs {
  uint64_t seed;
  int64_t t;        // >= 0: set the iteration; < 0: advance the device's t by one
  int n, m, schedule, n_local, rank, direct;
  int8_t local_workers[SESGD_MAX_WORKERS];
  int8_t slot_of[SESGD_MAX_WORKERS];      // worker -> local slot (every worker local: K6)
  int8_t worker_rank[SESGD_MAX_WORKERS];  // -1 before the layout is frozen
};
cudaError_t launch_iter_begin(const IterBeginArgs &a, DevIter *d, cudaStream_t stream);

// K6: all n workers resident on this GPU (1-GPU "k simulated workers").
struct ResidentArgs {
  float *const *x;        // [n_local] device table, indexed by local slot
  float *const *v;        // [n_local]
  const float *const *g;  // [n_local]
  int64_t numel;
  float lr, mu;
  float wd;               // weight decay (sesgd_set_weight_decay)
  int m;                  // group size
  int k;                  // groups
  int nb;                 // 0: one bucket (x, v, g, numel); > 0: all buckets via the tables
  int n_local;
  float *const *bx;       // [nb * n_local] tables of the all-bucket launch
  float *const *bv;
  const float *const *bg;
  const int64_t *numels;  // [nb]
  int8_t member_slot[SESGD_MAX_WORKERS];  // canonical order, mapped to local slots
  const DevIter *dev;     // non-null: member_slot comes from the device iteration state
};
// mode: SESGD_MODE_*; vec: all pointers 16-byte aligned; grid_x: CTAs per group;
// unroll: 0 = default (SESGD_OPT_RESIDENT_UNROLL)
cudaError_t launch_resident(const ResidentArgs &a, int mode, bool vec, int grid_x, int unroll,
                            cudaStream_t stream);
int resident_block_threads();
// K8: global average (Alg.1 last line): outs[s][e] = fold_i rows[i][e] / nrows
struct AverageArgs {
  const float *rows[SESGD_MAX_WORKERS];  // the n workers' parameters, ascending worker id
  float *outs[SESGD_MAX_WORKERS];        // every local worker's parameters
  int nrows, nouts;
  int64_t numel;
};
cudaError_t launch_average(const AverageArgs &a, bool vec, int sm_count, cudaStream_t stream);
// K10: pair co-membership counts over iterations [t0, t0 + T): counts[min(i,j) * n + max(i,j)] +=
// number of iterations in which workers i and j share a group (schedule 0 random, 1 dimension exchange)
cudaError_t launch_pair_counts(uint64_t seed, int64_t t0, int64_t T, int n, int m, int schedule,
                               unsigned long long *counts, int sm_count, cudaStream_t stream);
// K9: consistency metric (rows only; outs unused): out[0] += sum (x - mean)^2, out[1] = max |x - mean|
cudaError_t launch_consensus(const AverageArgs &a, double *out, int sm_count, cudaStream_t stream);
int resident_occupancy(int mode, bool vec, int m, int unroll);

// K3: one-shot push over NVLink, SM-specialised (COMM CTAs + COMPUTE CTAs), see p2p.cu.
struct BucketMeta {
  int64_t numel;       // elements
  int64_t stage_off;   // float offset inside a stage / receive region
  int64_t chunk_base;  // first global chunk index
  int64_t nchunks;
};
struct P2PArgs {
  const BucketMeta *meta;           // [NB] device table
  float *const *bx;                 // [NB * r] device tables: bucket b, local slot s -> b*r + s
  float *const *bv;
  const float *const *bg;
  char *ws[SESGD_MAX_RANKS];        // every rank's workspace, mapped here
  char *mc_ws;                      // NVLS: multicast mapping of the workspaces (nullptr: none)
  int payload_bf16;                 // two-shot reduce-scatter values as bf16 (SESGD_OPT_PAYLOAD_BF16)
  int64_t g0, g1;                   // global chunk range of this launch
  int64_t total_chunks;             // chunks of all buckets (flag array stride)
  int64_t region_floats;            // floats of one stage / receive region (all buckets)
  int64_t ready_off, sent_off, staged_off, consumed_off, stage_off, recv_off;  // byte offsets
  uint64_t seq_epoch0;              // S(seq, g) = seq_epoch0 + g / Gc for this launch
  uint64_t prev2_epoch0;            // the same for the launch that made call - 2 (guard)
  int64_t seq, prev2_seq;           // launch sequence numbers of this launch / of call - 2's (K4W)
  uint64_t claim_base;              // K4W: value of the chunk-claim counter when this launch starts
  int64_t call;                     // call index of the bucket(s) (identical on every rank)
  uint64_t timeout_ns;
  uint64_t hop_delay_ns;
  unsigned long long *err_host;     // mapped host block: [code, kind, cta, seen, target, worker, pos, rank]
  unsigned int *abort_dev;          // device word: set on timeout, skips further waits
  uint64_t *prof;                   // optional per-CTA phase timers [grid][8] (SESGD_OPT_PROFILE)
  float lr, mu, wd;
  int n, m, r, grid;
  int comm_ctas, comm_batch;        // COMM CTAs (blockIdx < comm_ctas) and chunks per release
  int lag;                          // COMPUTE folds chunk step k - lag after staging step k
  int release_delay;                // two-shot: steps between a push and its flag release
  int release_every;                // two-shot: chunk steps between flag-release batches
  int release_stagger;              // offset each CTA's release steps by its index
  int parity;                       // call & 1: receive slots / ready flags double buffer
  int my_rank;
  int bucket, nbuckets;             // bucket of a single-bucket launch, -1 for all buckets
  int discard;                      // drop dead stage / receive lines from L2 (no write-back)
  int experiment;                   // SESGD_OPT_EXPERIMENT (measurement only)
  int protocol;                     // SESGD_OPT_PROTOCOL: 0 epoch flags, 1 value-carried (sentinel)
  int cooperative;                  // SESGD_OPT_COOPERATIVE: cooperative launch (co-residency)
  unsigned long long *counters;     // device handshake counters [kCnt*] (sesgd_get_stats), or null
  int8_t my_workers[SESGD_MAX_WORKERS];      // global ids of local slots
  int8_t my_pos[SESGD_MAX_WORKERS];          // position of each local slot in its group
  int8_t slot_kind[SESGD_MAX_WORKERS];       // 0: group has remote members; 1: all-local group,
                                             // first member; 2: all-local group, other member
  int8_t worker_rank[SESGD_MAX_WORKERS];
  int8_t worker_slot[SESGD_MAX_WORKERS];
  int8_t canon[SESGD_MAX_WORKERS];           // canonical groups of the iteration
  int8_t group_of[SESGD_MAX_WORKERS];
  // device iteration state (null: the fields above are this launch's): the kernel patches call,
  // parity, seq, prev2_seq, epochs, claim_base and the schedule fields from it, and its last CTA
  // to finish advances it (dev_claim_inc: claims this launch makes)
  DevIter *dev;
  DevBucket *dev_buckets;
  uint64_t dev_claim_inc;
  int64_t kmax;             // epochs per launch (seq_epoch0 = seq * kmax + 1)
  int ws_split;             // K4W-M: S warps (8, 12, 16; SESGD_OPT_WS_SPLIT)
  int wsm_spanning_only;    // K4W-M: skip the all-local groups (a K6 launch updates them)
};
// device-side handshake counters (one block per context, cumulative; fire-and-forget atomics)
enum DevCounter : int {
  kCntFlagStores = 0,  // cross-GPU handshake stores: ready flags (K3, K4 protocol 0), ring step flags (K5)
  kCntFlagSpins = 1,   // flag waits that found the peer's flag not yet there
  kCntValueSpins = 2,  // value-carried polls that found a sentinel (protocols 1, 2)
  kCntLaunches = 3,    // multi-GPU kernel launches (CTA 0 of every grid)
  kCntHopNs = 4,       // elapsed ns of the last sesgd_measure_hop ping-pong (written, not added)
  kNumCounters = 8
};
#ifdef __CUDACC__
__device__ __forceinline__ void count(unsigned long long *c, int which, unsigned long long v = 1) {
  if (c && v) atomicAdd(c + which, v);
}
#endif

// K5: paper-faithful Ring-AllReduce inside each group (one worker per GPU), see ring.cu.
struct RingArgs {
  float *x, *v;                     // this bucket's buffers of the (single) local worker
  const float *g;
  char *ws[SESGD_MAX_RANKS];
  int64_t numel;
  int64_t rbuf_off;                 // byte offset of this bucket's receive buffers
  int64_t slice_cap;                // floats per (parity, step) receive buffer
  int64_t rflag_off, rcons_off;     // byte offsets: flags [2][NB][steps][grid], consumed [NB][grid]
  int64_t call;
  uint64_t timeout_ns, hop_delay_ns;
  unsigned long long *err_host;
  unsigned int *abort_dev;
  float lr, mu, wd;
  int parity, steps, m, pos, grid, my_rank, bucket, nbuckets;
  int cooperative;
  unsigned long long *counters;
  int8_t ring_rank[SESGD_MAX_WORKERS];  // rank of ring position 0..m-1 (ascending worker id)
  DevIter *dev;                         // device iteration state (as P2PArgs::dev)
  DevBucket *dev_buckets;
  int64_t seq;                          // launch sequence number (patched in device mode)
};
cudaError_t launch_ring(const RingArgs &a, int mode, cudaStream_t stream);
cudaError_t launch_pingpong(uint64_t *mine, uint64_t *peer, int iters, int initiator, uint64_t base,
                            uint64_t *out_ns, cudaStream_t stream);
int ring_block_threads();
int ring_occupancy(int mode);

// variant = COMM CTAs per launch (1..148); smem = guard cache bytes
cudaError_t launch_p2p_oneshot(const P2PArgs &a, int variant, int mode, bool vec, size_t smem,
                               cudaStream_t stream);
bool p2p_variant_valid(int variant);
int p2p_block_threads(int variant);
int p2p_chunk_elems(int variant);
int p2p_guard_pairs_max();
size_t p2p_smem_bytes(int variant, int guard_pairs, int grid);  // COMM ring + mbarriers + guard cache
int p2p_occupancy(int variant, int r, int mode, bool vec, size_t smem);
// K4: two-shot (reduce-scatter + all-gather pushes), one worker per GPU, DIRECT grid (no COMM CTAs)
// tma: pushes staged in shared memory and sent with cp.async.bulk (SESGD_OPT_PUSH_TMA)
cudaError_t launch_p2p_twoshot(const P2PArgs &a, int mode, bool vec, bool tma, cudaStream_t stream);
int p2p_twoshot_occupancy(int mode, bool vec, bool tma, bool multi);
// K4W (SESGD_OPT_PROTOCOL = 2): warp-specialised two-shot, one worker per GPU, one CTA per SM
cudaError_t launch_p2p_ws(const P2PArgs &a, int mode, bool vec, cudaStream_t stream);
cudaError_t launch_p2p_ws_pair(const P2PArgs &a0, const P2PArgs &a1, int mode, bool vec, cudaStream_t stream);
int p2p_ws_occupancy(int m);
int p2p_ws_threads();
// K4W-M (SESGD_OPT_PROTOCOL = 2 with several workers per GPU), p2p_wsm.cu
cudaError_t launch_p2p_wsm(const P2PArgs &a, int mode, bool vec, cudaStream_t stream);
cudaError_t launch_p2p_wsm_pair(const P2PArgs &a0, const P2PArgs &a1, int mode, bool vec, cudaStream_t stream);
bool p2p_wsm_supported(int r, int m);
int p2p_wsm_occupancy(int r);
int64_t p2p_wsm_units(int r, int m, int64_t chunks);  // claimable units of `chunks` chunks

}  // namespace sesgd

// ---------------------------------------------------------------- the context
struct sesgd_bucket {
  bool registered = false;
  int64_t numel = 0;
  bool vec = false;
  float **d_x = nullptr, **d_v = nullptr;
  const float **d_g = nullptr;
  std::vector<float *> hx, hv;
  std::vector<const float *> hg;
  sesgd_stats stats{};
  int64_t stage_bucket_off = 0;  // multi-GPU layout
  int64_t nchunks = 0, chunk_base = 0;
  int64_t calls = 0;             // sync_step calls on this bucket (flag epochs, parity)
  int64_t seq_hist[2] = {0, 0};  // launch sequence numbers of the last two calls (by call parity)
  int64_t ring_off = 0, ring_cap = 0;  // K5 receive buffers (bytes offset, floats per buffer)
};

struct sesgd_ctx {
  int32_t n = 0, m = 0;
  uint64_t seed = 0;
  int mode = SESGD_MODE_PARAM_AVG;
  int path = SESGD_PATH_AUTO;
  int64_t timeout_ms = 20000;
  int64_t grid_opt = 0;
  int64_t hop_delay_ns = 0;
  int p2p_variant = 0;   // SESGD_OPT_P2P_VARIANT: 0 = DIRECT push, n = n COMM CTAs
  int comm_batch = 16;   // chunks per COMM release (SESGD_OPT_COMM_BATCH)
  int fold_lag = 4;      // SESGD_OPT_FOLD_LAG
  int discard = 1;      // SESGD_OPT_DISCARD
  int resident_unroll = 0;  // SESGD_OPT_RESIDENT_UNROLL
  int push_tma = 0;         // SESGD_OPT_PUSH_TMA (two-shot kernel)
  int release_delay = 1;    // SESGD_OPT_RELEASE_DELAY (two-shot kernel)
  int release_every = 3;    // SESGD_OPT_RELEASE_EVERY (two-shot kernel)
  int release_stagger = 1;  // SESGD_OPT_RELEASE_STAGGER
  int64_t local_period = 1; // SESGD_OPT_LOCAL_PERIOD (Local-SESGD)
  char *mc_ws = nullptr;    // sesgd_attach_multicast (SESGD_PATH_NVLS)
  int payload_bf16 = 0;     // SESGD_OPT_PAYLOAD_BF16
  int experiment = 0;       // SESGD_OPT_EXPERIMENT
  int protocol = -1;        // SESGD_OPT_PROTOCOL (two-shot kernel; -1 auto, resolved at layout freeze)
  int cooperative = 0;      // SESGD_OPT_COOPERATIVE
  int ws_split = 8;         // SESGD_OPT_WS_SPLIT (K4W-M S warps)
  int wsm_hybrid = 0;       // SESGD_OPT_WSM_HYBRID: all-local groups through K6, the rest K4W-M
  int schedule = 0;         // SESGD_OPT_SCHEDULE: 0 uniform random (R1), 1 dimension exchange
  float weight_decay = 0.f; // sesgd_set_weight_decay
  // sesgd_sync_all_host: copy streams and per-bucket events (created on first use)
  cudaStream_t copy_in = nullptr, copy_out = nullptr;
  std::vector<cudaEvent_t> ev_in, ev_k, ev_out;
  cudaEvent_t ev_start = nullptr;
  int64_t *d_numels = nullptr;  // resident all-bucket launch: numel table [NB]
  bool resident_tables_ok = false;
  // attach
  bool attached = false;
  int device = -1;
  int sm_count = 0;       // SMs the persistent grids are sized for (SESGD_OPT_SM_BUDGET)
  int dev_sm_count = 0;   // SMs of the device
  int sm_budget = 0;      // SESGD_OPT_SM_BUDGET (0: the whole device)
  int n_local = 0;
  std::vector<int32_t> local_workers;
  int8_t slot_of[SESGD_MAX_WORKERS];
  std::vector<sesgd_bucket> buckets;
  // multi-GPU
  bool layout_frozen = false;
  bool peers = false;
  int n_ranks = 1, rank = 0;
  char *ws[SESGD_MAX_RANKS] = {};
  int8_t worker_rank[SESGD_MAX_WORKERS];
  int8_t worker_slot[SESGD_MAX_WORKERS];
  int grid = 0;
  int64_t chunk = 0, kmax = 0;
  int64_t ws_bytes = 0, ready_off = 0, sent_off = 0, staged_off = 0, consumed_off = 0,
          stage_off = 0, recv_off = 0, stage_slot_floats = 0, total_chunks = 0;
  int64_t seq = 0;  // one-shot launches so far (staged / consumed epochs)
  size_t guard_smem = 0;
  int ring_grid = 0;                      // K5 (0: ring path unavailable for this layout)
  int64_t rflag_off = 0, rcons_off = 0;
  sesgd::BucketMeta *d_meta = nullptr;  // device bucket tables (multi-GPU path)
  float **d_bx = nullptr, **d_bv = nullptr;
  const float **d_bg = nullptr;
  uint64_t layout_hash = 0;
  // iteration
  bool iter_set = false;
  int64_t t = 0;
  int32_t canon[SESGD_MAX_WORKERS], group_of[SESGD_MAX_WORKERS];
  // errors
  unsigned long long *h_err = nullptr;  // pinned mapped error block (8 words)
  unsigned long long *d_err = nullptr;  // device alias of h_err
  unsigned int *d_abort = nullptr;
  uint64_t *d_prof = nullptr;     // SESGD_OPT_PROFILE timers
  unsigned long long *d_counters = nullptr;  // device handshake counters [kNumCounters] (+ hop ns)
  cudaEvent_t ev_l0 = nullptr, ev_l1 = nullptr;  // around the most recent sync launch
  bool ev_l_valid = false;
  uint64_t hop_base[SESGD_MAX_RANKS] = {};
  uint64_t claim_base = 0;        // K4W dynamic chunk claims so far (chunks + one failed claim per CTA)
  int hop_iters = 0;
  int profile = 0;
  // SESGD_OPT_DEVICE_ITER: iteration state in device memory (iter.cu, dev_iter.cuh); the host
  // fields (t, seq, claim_base, bucket calls / seq_hist) keep shadowing what was ENQUEUED
  int device_iter = 0;
  sesgd::DevIter *d_iter = nullptr;
  sesgd::DevBucket *d_bstate = nullptr;
  std::string last_error;
};
