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
// Eq. 2 / Eq. 3 exact forms (A6/A7).
void latency_model(int n, int m, double bytes, double nu, double tau, sesgd_cost *out);

// ---------------------------------------------------------------- kernels
constexpr int kMaxLocal = SESGD_MAX_WORKERS;

// K6: all n workers resident on this GPU (1-GPU "k simulated workers").
struct ResidentArgs {
  float *const *x;        // [n_local] device table, indexed by local slot
  float *const *v;        // [n_local]
  const float *const *g;  // [n_local]
  int64_t numel;
  float lr, mu;
  int m;                  // group size
  int k;                  // groups
  int8_t member_slot[SESGD_MAX_WORKERS];  // canonical order, mapped to local slots
};
// mode: SESGD_MODE_*; vec: all pointers 16-byte aligned; grid_x: CTAs per group.
cudaError_t launch_resident(const ResidentArgs &a, int mode, bool vec, int grid_x,
                            cudaStream_t stream);
int resident_block_threads();
int resident_occupancy(int mode, bool vec, int m);

// K3: one-shot NVLink P2P group exchange (worker(s) on several GPUs).
struct P2PArgs {
  float *const *x;        // [r] local workers' buffers
  float *const *v;
  const float *const *g;
  char *ws[SESGD_MAX_RANKS];        // every rank's workspace, mapped here
  int64_t numel;                    // bucket elements
  int64_t chunk;                    // elements per chunk (multiple of 4 * threads)
  int64_t nchunks;
  int64_t stage_off;                // byte offset of the stage area in a workspace
  int64_t stage_slot_floats;        // floats of one (parity, slot) stage region
  int64_t stage_bucket_off;         // float offset of this bucket inside a region
  int64_t ready_off, done_off;      // byte offsets of the flag arrays
  uint64_t epoch0;                  // epoch of (t, bucket, k=0)
  uint64_t epoch_prev0;             // epoch of (t-2, bucket, k=0), 0 if t < 2
  uint64_t timeout_ns;
  uint64_t hop_delay_ns;
  unsigned int *err_host;           // mapped host word (latched error)
  unsigned int *abort_dev;          // device word: set on timeout, skips further waits
  float lr, mu;
  int n, m, r, grid;
  int parity;
  int my_rank;
  int8_t my_workers[SESGD_MAX_WORKERS];      // global ids of local slots
  int8_t worker_rank[SESGD_MAX_WORKERS];
  int8_t worker_slot[SESGD_MAX_WORKERS];
  int8_t canon[SESGD_MAX_WORKERS];           // iteration t
  int8_t group_of[SESGD_MAX_WORKERS];
  int8_t canon_prev[SESGD_MAX_WORKERS];      // iteration t-2 (valid if epoch_prev0)
  int8_t group_of_prev[SESGD_MAX_WORKERS];
};
cudaError_t launch_p2p_oneshot(const P2PArgs &a, int mode, bool vec, cudaStream_t stream);
int p2p_block_threads();
int p2p_chunk_elems();
int p2p_occupancy(int mode, bool vec);

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
  int64_t nchunks = 0;
};

struct sesgd_ctx {
  int32_t n = 0, m = 0;
  uint64_t seed = 0;
  int mode = SESGD_MODE_PARAM_AVG;
  int path = SESGD_PATH_AUTO;
  int64_t timeout_ms = 20000;
  int64_t grid_opt = 0;
  int64_t hop_delay_ns = 0;
  // attach
  bool attached = false;
  int device = -1;
  int sm_count = 0;
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
  int64_t ws_bytes = 0, ready_off = 0, done_off = 0, stage_off = 0, stage_slot_floats = 0;
  uint64_t layout_hash = 0;
  // iteration
  bool iter_set = false;
  int64_t t = 0;
  int32_t canon[SESGD_MAX_WORKERS], group_of[SESGD_MAX_WORKERS];
  int32_t canon_prev[SESGD_MAX_WORKERS], group_of_prev[SESGD_MAX_WORKERS];
  // errors
  unsigned int *h_err = nullptr;  // pinned mapped
  unsigned int *d_err = nullptr;  // device alias of h_err
  unsigned int *d_abort = nullptr;
  std::string last_error;
};
