// sesgd_capi.cu -- the C ABI of libsesgd.so (declared and documented in include/sesgd.h).
//
// Host-side control only: argument validation, the per-iteration schedule
// (schedule.cpp), device tables, workspace layout, and kernel selection.  Every
// step of the hot path runs in the kernels of resident.cu (1 GPU) and p2p.cu
// (NVLink P2P); there is no CPU fallback.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "internal.h"

using sesgd::P2PArgs;
using sesgd::ResidentArgs;

namespace {

constexpr int kMaxBuckets = 4096;
constexpr uint64_t kMagic = 0x5345534744423230ULL;  // "SESGDB20"

int fail(sesgd_ctx *ctx, int code, const std::string &why) {
  if (ctx) ctx->last_error = why;
  return code;
}

int cuda_fail(sesgd_ctx *ctx, cudaError_t e, const char *what) {
  std::string s = std::string(what) + ": " + cudaGetErrorString(e);
  return fail(ctx, SESGD_ECUDA, s);
}

bool valid_nm(int32_t n, int32_t m) { return n >= 1 && n <= SESGD_MAX_WORKERS && m >= 1 && m <= n; }

uint64_t fnv(uint64_t h, uint64_t v) {
  for (int i = 0; i < 8; ++i) {
    h ^= (v >> (8 * i)) & 0xff;
    h *= 0x100000001b3ULL;
  }
  return h;
}

int64_t round_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int check_latched(sesgd_ctx *ctx) {
  volatile unsigned long long *e = ctx->h_err;
  if (!e || e[0] == 0) return SESGD_OK;
  static const char *kinds[] = {"?", "consumed", "ready", "staged", "sent", "TMA-load"};
  char buf[256];
  std::snprintf(buf, sizeof buf,
                "a group peer did not signal before the timeout: rank %llu CTA %llu waited for "
                "%s flag of worker %llu (position %lld): saw epoch %llu, needed %llu",
                e[7], e[2], kinds[e[1] < 6 ? e[1] : 0], e[5], (long long)e[6], e[3], e[4]);
  return fail(ctx, SESGD_ETIMEOUT, buf);
}

// CUDA events around every sync launch: sesgd_stats.last_launch_us is the device time of the most
// recent one (an event record is not a kernel and costs ~1 us of host time)
void mark_start(sesgd_ctx *ctx, cudaStream_t st) {
  if (ctx->ev_l0) cudaEventRecord(ctx->ev_l0, st);
}
void mark_end(sesgd_ctx *ctx, cudaStream_t st) {
  if (ctx->ev_l1 && cudaEventRecord(ctx->ev_l1, st) == cudaSuccess) ctx->ev_l_valid = true;
}

void free_bucket(sesgd_bucket &b) {
  if (b.d_x) cudaFree(b.d_x);
  if (b.d_v) cudaFree(b.d_v);
  if (b.d_g) cudaFree(const_cast<float **>(b.d_g));
  b.d_x = b.d_v = nullptr;
  b.d_g = nullptr;
}

// ---- multi-GPU workspace layout (identical on every rank) ----
//   [0, 256)            header: magic, layout hash
//   [ready_off, ..)     u64 ready   [2 parity][r slot][total_chunks][m position] (written by peers)
//   [sent_off, ..)      u64 sent    [r slot][total_chunks]        (local: COMM -> COMPUTE)
//   [staged_off, ..)    u64 staged  [r slot][Gc]                  (local: COMPUTE -> COMM)
//   [consumed_off, ..)  u64 consumed[r slot][Gc]                  (read by peers' COMM: guard)
//   [stage_off, ..)     f32 stage   [r slot][region]              (own x_hat, L2-resident)
//   [recv_off, ..)      f32 recv    [2 parity][r slot][m position][region]
// region = stage_slot_floats = sum over buckets of round_up(numel, 64).
int resolve_path(const sesgd_ctx *ctx);

void freeze_layout(sesgd_ctx *ctx) {
  if (ctx->path == SESGD_PATH_TWOSHOT || ctx->path == SESGD_PATH_NVLS)
    ctx->p2p_variant = 0;  // K4 runs on the DIRECT grid
  // SESGD_OPT_PROTOCOL auto (-1): value-carried validity wherever the two-shot kernel supports it
  // (fp32 LSU pushes), in the warp-specialised K4W when one worker lives on each GPU (K4W-M with
  // 2..8); else flags
  // (measured, profiles/r02_k4_experiments.json: n = m = 2 kernel 0.188 ms K4W, 0.190 K4 value-
  // carried, 0.185-0.228 K4 flags)
  if (ctx->protocol < 0) {
    const bool value = resolve_path(ctx) == SESGD_PATH_TWOSHOT && ctx->m >= 2 && !ctx->push_tma &&
                       !ctx->payload_bf16;
    // K4W-M for 2..8 workers per GPU (same box, kernel p50: cfg 2 on 2 GPUs r = 4 0.567 ms vs K4
    // 0.610; n = 4, r = 2 0.393 vs 0.41, profiles/r02_k4wm_ab/)
    const bool wsm = sesgd::p2p_wsm_supported(ctx->n_local, ctx->m);
    ctx->protocol = !value ? 0 : (ctx->n_local == 1 || wsm) ? 2 : 1;
  }
  const int var = ctx->p2p_variant;
  const int chunk = sesgd::p2p_chunk_elems(var);
  const int r = ctx->n_local;
  const int pairs = std::min(sesgd::p2p_guard_pairs_max(), r * (ctx->m - 1));
  auto occupancy = [&](size_t smem) {
    int occ = sesgd::p2p_occupancy(var, r, SESGD_MODE_PARAM_AVG, true, smem);
    occ = std::min(occ, sesgd::p2p_occupancy(var, r, SESGD_MODE_GRAD_AVG, true, smem));
    occ = std::min(occ, sesgd::p2p_occupancy(var, r, SESGD_MODE_PARAM_AVG, false, smem));
    occ = std::min(occ, sesgd::p2p_occupancy(var, r, SESGD_MODE_GRAD_AVG, false, smem));
    if (var == 0)  // K4 (two-shot) shares the grid and the flag layout
      for (int mode = 0; mode < 2; ++mode)
        for (int vec = 0; vec < 2; ++vec)
          for (int tma = 0; tma < 2; ++tma)
            occ = std::min(occ, sesgd::p2p_twoshot_occupancy(mode, vec, tma, r > 1));
    return occ;
  };
  // every CTA must be co-resident (COMM and COMPUTE wait on each other): grid = SMs x
  // occupancy, with the COMM guard cache (pairs x Gc u64) in dynamic shared memory
  int grid = ctx->sm_count * occupancy(sesgd::p2p_smem_bytes(var, 0, 0));
  if (ctx->protocol == 2)  // K4W / K4W-M: one CTA per SM
    grid = ctx->sm_count * (r == 1 ? sesgd::p2p_ws_occupancy(ctx->m) : sesgd::p2p_wsm_occupancy(r));
  if (ctx->grid_opt > 0 && ctx->grid_opt < grid) grid = int(ctx->grid_opt);
  size_t smem = sesgd::p2p_smem_bytes(var, pairs, grid);
  const int grid2 = ctx->sm_count * occupancy(smem);
  if (grid2 < grid) {
    grid = grid2;
    smem = sesgd::p2p_smem_bytes(var, pairs, grid);
  }
  const int comm = std::min(var, std::max(1, grid / 2));  // 0 = DIRECT push (no COMM CTAs)
  const int gc = grid - comm;
  ctx->grid = grid;
  ctx->chunk = chunk;
  ctx->guard_smem = smem;
  int64_t off = 0, chunks = 0;
  uint64_t h = 0xcbf29ce484222325ULL;
  h = fnv(h, uint64_t(ctx->n));
  h = fnv(h, uint64_t(ctx->m));
  h = fnv(h, uint64_t(ctx->n_local));
  h = fnv(h, uint64_t(grid));
  h = fnv(h, uint64_t(chunk));
  h = fnv(h, uint64_t(comm));
  h = fnv(h, uint64_t(ctx->comm_batch));
  h = fnv(h, uint64_t(ctx->protocol));
  for (size_t b = 0; b < ctx->buckets.size(); ++b) {
    sesgd_bucket &bk = ctx->buckets[b];
    bk.stage_bucket_off = off;
    bk.nchunks = (bk.numel + chunk - 1) / chunk;
    bk.chunk_base = chunks;
    chunks += bk.nchunks;
    off += round_up(bk.numel, 64);  // 256-byte aligned buckets
    h = fnv(h, uint64_t(b));
    h = fnv(h, uint64_t(bk.registered ? bk.numel : -1));
  }
  ctx->p2p_variant = comm;
  ctx->total_chunks = std::max<int64_t>(chunks, 1);
  ctx->kmax = (ctx->total_chunks + gc - 1) / gc + 1;  // > any floor(g / Gc)
  ctx->stage_slot_floats = std::max<int64_t>(off, 64);
  ctx->ready_off = 256;
  ctx->sent_off = round_up(ctx->ready_off + 2 * int64_t(r) * ctx->total_chunks * ctx->m * 8, 256);
  ctx->staged_off = round_up(ctx->sent_off + int64_t(r) * ctx->total_chunks * 8, 256);
  ctx->consumed_off = round_up(ctx->staged_off + int64_t(r) * gc * 8, 256);
  ctx->stage_off = round_up(ctx->consumed_off + int64_t(r) * gc * 8, 4096);
  ctx->recv_off = ctx->stage_off + int64_t(r) * ctx->stage_slot_floats * 4;
  ctx->ws_bytes = ctx->recv_off + 2 * int64_t(r) * ctx->m * ctx->stage_slot_floats * 4;
  // K5 ring (one worker per GPU only): per bucket 2 parities x 2(m-1) step buffers of one
  // slice, flags [2][NB][steps][ring grid], consumed [NB][ring grid]
  ctx->ring_grid = 0;
  if (r == 1 && ctx->m >= 2) {
    const int steps = 2 * (ctx->m - 1);
    const int rgrid = ctx->sm_count * std::min(sesgd::ring_occupancy(SESGD_MODE_PARAM_AVG),
                                               sesgd::ring_occupancy(SESGD_MODE_GRAD_AVG));
    const int64_t nb = int64_t(ctx->buckets.size());
    int64_t off = round_up(ctx->ws_bytes, 4096);
    ctx->rflag_off = off;
    off = round_up(off + 2 * nb * steps * rgrid * 8, 256);
    ctx->rcons_off = off;
    off = round_up(off + nb * rgrid * 8, 4096);
    for (auto &bk : ctx->buckets) {
      bk.ring_cap = round_up((bk.numel + ctx->m - 1) / ctx->m, 64);
      bk.ring_off = off;
      off += 2 * int64_t(steps) * bk.ring_cap * 4;
    }
    ctx->ws_bytes = off;
    ctx->ring_grid = rgrid;
    h = fnv(h, uint64_t(rgrid));
  }
  ctx->layout_hash = h;
  ctx->layout_frozen = true;
}

// Local-SESGD: an iteration whose (t + 1) is not a multiple of the local period only
// takes the local step on every local worker -- K6 with singleton groups (m = 1, k = n_local),
// no flags, no exchange; the exchange paths' call counters do not move (every rank skips the
// same iterations).  bucket < 0: every bucket in one launch.
int upload_resident_tables(sesgd_ctx *ctx);

// the canonical partition of iteration t under the context's schedule (SESGD_OPT_SCHEDULE)
void make_groups(const sesgd_ctx *ctx, int64_t t, int32_t *canon, int32_t *group_of) {
  if (ctx->schedule == 1)
    sesgd::dimension_exchange_groups(t, ctx->n, ctx->m, canon, group_of);
  else
    sesgd::shuffle_exchange_groups(ctx->seed, t, ctx->n, ctx->m, canon, group_of);
}

bool local_only_iteration(const sesgd_ctx *ctx) {
  return ctx->local_period > 1 && (ctx->t + 1) % ctx->local_period != 0;
}

// ---- device-resident iteration state (SESGD_OPT_DEVICE_ITER) ----
sesgd::IterBeginArgs iter_begin_args(const sesgd_ctx *ctx, int64_t t) {
  sesgd::IterBeginArgs a{};
  a.seed = ctx->seed;
  a.t = t;
  a.n = ctx->n;
  a.m = ctx->m;
  a.schedule = ctx->schedule;
  a.n_local = ctx->n_local;
  a.rank = ctx->peers ? ctx->rank : 0;
  a.direct = ctx->p2p_variant == 0 ? 1 : 0;
  for (int s = 0; s < ctx->n_local; ++s) a.local_workers[s] = int8_t(ctx->local_workers[s]);
  for (int w = 0; w < ctx->n; ++w) {
    a.slot_of[w] = ctx->slot_of[w];
    a.worker_rank[w] = ctx->peers ? ctx->worker_rank[w] : int8_t(ctx->slot_of[w] >= 0 ? 0 : -1);
  }
  return a;
}

int device_iter_enable(sesgd_ctx *ctx) {
  if (!ctx->attached || ctx->buckets.empty()) return fail(ctx, SESGD_ESTATE, "attach and register buckets first");
  for (auto &b : ctx->buckets)
    if (!b.registered) return fail(ctx, SESGD_ESTATE, "bucket ids must be dense from 0");
  if (ctx->local_period > 1) return fail(ctx, SESGD_ENOTSUP, "device iteration state with Local-SESGD");
  if (ctx->n_local == ctx->n && !ctx->resident_tables_ok) {  // no allocation may happen inside a capture
    const int rc = upload_resident_tables(ctx);
    if (rc != SESGD_OK) return rc;
  }
  const size_t nb = ctx->buckets.size();
  cudaError_t e = cudaSuccess;
  if (!ctx->d_iter) e = cudaMalloc(reinterpret_cast<void **>(&ctx->d_iter), sizeof(sesgd::DevIter));
  if (e == cudaSuccess && ctx->d_bstate) e = cudaFree(ctx->d_bstate);
  ctx->d_bstate = nullptr;
  if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void **>(&ctx->d_bstate), nb * sizeof(sesgd::DevBucket));
  if (e != cudaSuccess) return cuda_fail(ctx, e, "device iteration state");
  sesgd::DevIter h{};
  h.t = ctx->iter_set ? ctx->t : -1;
  h.seq = ctx->seq;
  h.claim_base = ctx->claim_base;
  std::vector<sesgd::DevBucket> hb(nb);
  for (size_t b = 0; b < nb; ++b) {
    hb[b].calls = ctx->buckets[b].calls;
    hb[b].hist[0] = ctx->buckets[b].seq_hist[0];
    hb[b].hist[1] = ctx->buckets[b].seq_hist[1];
  }
  e = cudaDeviceSynchronize();  // no launch of this context may still read the old state
  if (e == cudaSuccess) e = cudaMemcpy(ctx->d_iter, &h, sizeof(h), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(ctx->d_bstate, hb.data(), nb * sizeof(sesgd::DevBucket), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && ctx->iter_set) e = sesgd::launch_iter_begin(iter_begin_args(ctx, ctx->t), ctx->d_iter, 0);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cuda_fail(ctx, e, "device iteration state upload");
  ctx->device_iter = 1;
  return SESGD_OK;
}

int device_iter_disable(sesgd_ctx *ctx) {
  if (!ctx->device_iter) return SESGD_OK;
  sesgd::DevIter h{};
  std::vector<sesgd::DevBucket> hb(ctx->buckets.size());
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpy(&h, ctx->d_iter, sizeof(h), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess)
    e = cudaMemcpy(hb.data(), ctx->d_bstate, hb.size() * sizeof(sesgd::DevBucket), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "device iteration state download");
  ctx->seq = h.seq;
  ctx->claim_base = h.claim_base;
  for (size_t b = 0; b < hb.size(); ++b) {
    ctx->buckets[b].calls = hb[b].calls;
    ctx->buckets[b].seq_hist[0] = hb[b].hist[0];
    ctx->buckets[b].seq_hist[1] = hb[b].hist[1];
  }
  ctx->iter_set = h.t >= 0;
  if (ctx->iter_set) {
    ctx->t = h.t;
    make_groups(ctx, ctx->t, ctx->canon, ctx->group_of);
  }
  ctx->device_iter = 0;
  return SESGD_OK;
}

int local_step(sesgd_ctx *ctx, int bucket, float lr, float momentum, cudaStream_t st) {
  ResidentArgs a{};
  a.lr = lr;
  a.mu = momentum;
  a.wd = ctx->weight_decay;
  a.m = 1;
  a.k = ctx->n_local;
  a.n_local = ctx->n_local;
  for (int s = 0; s < ctx->n_local; ++s) a.member_slot[s] = int8_t(s);
  bool vec = true;
  int64_t biggest = 0;
  if (bucket >= 0) {
    const sesgd_bucket &b = ctx->buckets[bucket];
    a.x = b.d_x;
    a.v = b.d_v;
    a.g = b.d_g;
    a.numel = b.numel;
    vec = b.vec;
    biggest = b.numel;
  } else {
    if (!ctx->resident_tables_ok) {
      const int rc = upload_resident_tables(ctx);
      if (rc != SESGD_OK) return rc;
    }
    for (auto &b : ctx->buckets) {
      vec = vec && b.vec;
      biggest = std::max(biggest, b.numel);
    }
    a.nb = int(ctx->buckets.size());
    a.bx = ctx->d_bx;
    a.bv = ctx->d_bv;
    a.bg = ctx->d_bg;
    a.numels = ctx->d_numels;
  }
  const int threads = sesgd::resident_block_threads();
  const int target = ctx->sm_count * sesgd::resident_occupancy(ctx->mode, vec, 1, 0);
  int gx = (target + a.k - 1) / a.k;
  const int64_t need = ((vec ? biggest / 4 : biggest) + threads - 1) / threads;
  if (need < gx) gx = int(need > 0 ? need : 1);
  mark_start(ctx, st);
  cudaError_t e = sesgd::launch_resident(a, ctx->mode, vec, gx, 0, st);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "launch local step");
  mark_end(ctx, st);
  for (size_t b = 0; b < ctx->buckets.size(); ++b) {
    if (bucket >= 0 && int(b) != bucket) continue;
    ctx->buckets[b].stats.hbm_algo_bytes += 20 * ctx->buckets[b].numel * ctx->n_local;
    if (bucket >= 0 || b == 0) ctx->buckets[b].stats.kernel_launches++;
  }
  return SESGD_OK;
}

// SESGD_PATH_AUTO: every worker on this GPU -> K6; else K4 two-shot (a remote member receives
// 2(m-1)/m of a bucket per member pair instead of one-shot's full copy: measured faster at
// m = 2 and 2x at m = 4); a COMM-CTA layout (P2P variant >= 1) -> K3 one-shot
int resolve_path(const sesgd_ctx *ctx) {
  if (ctx->path != SESGD_PATH_AUTO) return ctx->path;
  if (ctx->n_local == ctx->n) return SESGD_PATH_RESIDENT;
  if (ctx->m >= 2 && ctx->p2p_variant == 0) return SESGD_PATH_TWOSHOT;
  return SESGD_PATH_ONESHOT;
}

// CTAs per group row of a resident launch covering `numel` elements (per bucket, or the
// largest bucket of an all-bucket launch): SMs x occupancy spread over the k group rows
int resident_grid_x(const sesgd_ctx *ctx, bool vec, int64_t numel) {
  const int k = ctx->n / ctx->m;
  const int threads = sesgd::resident_block_threads();
  int target = ctx->sm_count * sesgd::resident_occupancy(ctx->mode, vec, ctx->m, ctx->resident_unroll);
  if (ctx->grid_opt > 0) target = int(ctx->grid_opt);
  int gx = (target + k - 1) / k;
  const int64_t items = vec ? numel / 4 : numel;
  const int64_t need = (items + threads - 1) / threads;
  if (need < gx) gx = int(need > 0 ? need : 1);
  return gx;
}

// device tables of the resident all-bucket launch: x/v/g pointers [NB * n_local], numel [NB]
int upload_resident_tables(sesgd_ctx *ctx) {
  const size_t nb = ctx->buckets.size();
  const int r = ctx->n_local;
  std::vector<float *> bx(nb * r), bv(nb * r);
  std::vector<const float *> bg(nb * r);
  std::vector<int64_t> numels(nb);
  for (size_t b = 0; b < nb; ++b) {
    const sesgd_bucket &bk = ctx->buckets[b];
    numels[b] = bk.numel;
    for (int s = 0; s < r; ++s) {
      bx[b * r + s] = bk.hx[s];
      bv[b * r + s] = bk.hv[s];
      bg[b * r + s] = bk.hg[s];
    }
  }
  if (ctx->d_bx) {
    cudaFree(ctx->d_bx);
    cudaFree(ctx->d_bv);
    cudaFree(const_cast<float **>(ctx->d_bg));
    ctx->d_bx = ctx->d_bv = nullptr;
    ctx->d_bg = nullptr;
  }
  if (ctx->d_numels) cudaFree(ctx->d_numels);
  ctx->d_numels = nullptr;
  cudaError_t e = cudaMalloc(reinterpret_cast<void **>(&ctx->d_bx), std::max<size_t>(nb * r, 1) * 8);
  if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void **>(&ctx->d_bv), std::max<size_t>(nb * r, 1) * 8);
  if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void **>(&ctx->d_bg), std::max<size_t>(nb * r, 1) * 8);
  if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void **>(&ctx->d_numels), std::max<size_t>(nb, 1) * 8);
  if (e == cudaSuccess) e = cudaMemcpy(ctx->d_bx, bx.data(), nb * r * 8, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(ctx->d_bv, bv.data(), nb * r * 8, cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = cudaMemcpy(const_cast<float **>(ctx->d_bg), bg.data(), nb * r * 8, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(ctx->d_numels, numels.data(), nb * 8, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "resident bucket tables");
  ctx->resident_tables_ok = true;
  return SESGD_OK;
}

// device bucket tables of the one-shot kernel: meta[NB], x/v/g pointers [NB * r]
int upload_tables(sesgd_ctx *ctx) {
  const size_t nb = ctx->buckets.size();
  const int r = ctx->n_local;
  std::vector<sesgd::BucketMeta> meta(nb);
  std::vector<float *> bx(nb * r), bv(nb * r);
  std::vector<const float *> bg(nb * r);
  for (size_t b = 0; b < nb; ++b) {
    const sesgd_bucket &bk = ctx->buckets[b];
    meta[b] = {bk.numel, bk.stage_bucket_off, bk.chunk_base, bk.nchunks};
    for (int s = 0; s < r; ++s) {
      bx[b * r + s] = bk.hx[s];
      bv[b * r + s] = bk.hv[s];
      bg[b * r + s] = bk.hg[s];
    }
  }
  cudaError_t e = cudaSuccess;
  if (!ctx->d_meta) {
    e = cudaMalloc(reinterpret_cast<void **>(&ctx->d_meta), std::max<size_t>(nb, 1) * sizeof(sesgd::BucketMeta));
    if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void **>(&ctx->d_bx), std::max<size_t>(nb * r, 1) * 8);
    if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void **>(&ctx->d_bv), std::max<size_t>(nb * r, 1) * 8);
    if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void **>(&ctx->d_bg), std::max<size_t>(nb * r, 1) * 8);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMalloc(bucket tables)");
  }
  e = cudaMemcpy(ctx->d_meta, meta.data(), nb * sizeof(sesgd::BucketMeta), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(ctx->d_bx, bx.data(), nb * r * 8, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(ctx->d_bv, bv.data(), nb * r * 8, cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = cudaMemcpy(const_cast<float **>(ctx->d_bg), bg.data(), nb * r * 8, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMemcpy(bucket tables)");
  return SESGD_OK;
}

// Hybrid K4W-M launch (SESGD_OPT_WSM_HYBRID, several workers per GPU, host iterations): the groups
// whose members are all on this GPU are updated by K6 first -- plain 128-bit streaming at ~0.96
// of HBM, where K4W-M's TMA ring drained by its S warps reaches ~4 TB/s -- and the
// K4W-M launch that follows streams only the workers whose group spans GPUs.  Same arithmetic
// and fold order in both kernels, so the same bits.
int launch_local_groups(sesgd_ctx *ctx, int bucket, float lr, float momentum, cudaStream_t st) {
  sesgd::ResidentArgs a{};
  int rows = 0;
  for (int s = 0; s < ctx->n_local; ++s) {
    const int me = ctx->local_workers[s];
    const int *G = ctx->canon + ctx->group_of[me] * ctx->m;
    bool all_local = true;
    for (int p = 0; p < ctx->m; ++p) all_local = all_local && ctx->worker_rank[G[p]] == ctx->rank;
    if (!all_local || G[0] != me) continue;
    for (int p = 0; p < ctx->m; ++p) a.member_slot[rows * ctx->m + p] = int8_t(ctx->worker_slot[G[p]]);
    ++rows;
  }
  if (rows == 0) return SESGD_OK;
  a.lr = lr;
  a.mu = momentum;
  a.wd = ctx->weight_decay;
  a.m = ctx->m;
  a.k = rows;
  a.n_local = ctx->n_local;
  bool vec = true;
  int64_t biggest = 0;
  if (bucket >= 0) {
    const sesgd_bucket &b = ctx->buckets[bucket];
    a.x = b.d_x;
    a.v = b.d_v;
    a.g = b.d_g;
    a.numel = b.numel;
    vec = b.vec;
    biggest = b.numel;
  } else {
    if (!ctx->d_numels) {
      std::vector<int64_t> numels(ctx->buckets.size());
      for (size_t b = 0; b < numels.size(); ++b) numels[b] = ctx->buckets[b].numel;
      cudaError_t e = cudaMalloc(reinterpret_cast<void **>(&ctx->d_numels), std::max<size_t>(numels.size(), 1) * 8);
      if (e == cudaSuccess) e = cudaMemcpy(ctx->d_numels, numels.data(), numels.size() * 8, cudaMemcpyHostToDevice);
      if (e != cudaSuccess) return cuda_fail(ctx, e, "bucket sizes table");
    }
    for (auto &b : ctx->buckets) {
      vec = vec && b.vec;
      biggest = std::max(biggest, b.numel);
    }
    a.nb = int(ctx->buckets.size());
    a.bx = ctx->d_bx;  // the multi-GPU [NB * r] pointer tables (upload_tables)
    a.bv = ctx->d_bv;
    a.bg = ctx->d_bg;
    a.numels = ctx->d_numels;
  }
  const int threads = sesgd::resident_block_threads();
  const int target = ctx->sm_count * sesgd::resident_occupancy(ctx->mode, vec, ctx->m, ctx->resident_unroll);
  int gx = (target + rows - 1) / rows;
  const int64_t need = ((vec ? biggest / 4 : biggest) + threads - 1) / threads;
  if (need < gx) gx = int(need > 0 ? need : 1);
  cudaError_t e = sesgd::launch_resident(a, ctx->mode, vec, gx, ctx->resident_unroll, st);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "launch resident kernel (all-local groups)");
  return SESGD_OK;
}

// One one-shot launch over bucket `bucket` (>= 0) or over every bucket (-1, all buckets
// share the same call history).  Host bookkeeping of calls / launch sequence follows.
// dry != nullptr: build the arguments into *dry and do the bookkeeping without launching (the
// two-rank pair harness launches both ranks' arguments as one grid)
int launch_oneshot(sesgd_ctx *ctx, int bucket, float lr, float momentum, cudaStream_t st,
                   bool twoshot = false, bool nvls = false, P2PArgs *dry = nullptr) {
  const sesgd_bucket &ref = ctx->buckets[bucket >= 0 ? bucket : 0];
  P2PArgs a{};
  a.meta = ctx->d_meta;
  a.bx = ctx->d_bx;
  a.bv = ctx->d_bv;
  a.bg = ctx->d_bg;
  for (int r = 0; r < ctx->n_ranks; ++r) a.ws[r] = ctx->ws[r];
  a.mc_ws = nvls ? ctx->mc_ws : nullptr;
  a.payload_bf16 = (twoshot && !nvls) ? ctx->payload_bf16 : 0;
  if (bucket >= 0) {
    a.g0 = ref.chunk_base;
    a.g1 = ref.chunk_base + ref.nchunks;
  } else {
    a.g0 = 0;
    a.g1 = ctx->total_chunks;
  }
  a.total_chunks = ctx->total_chunks;
  a.region_floats = ctx->stage_slot_floats;
  a.ready_off = ctx->ready_off;
  a.sent_off = ctx->sent_off;
  a.staged_off = ctx->staged_off;
  a.consumed_off = ctx->consumed_off;
  a.stage_off = ctx->stage_off;
  a.recv_off = ctx->recv_off;
  const int64_t call = ref.calls;
  a.call = call;
  a.seq_epoch0 = uint64_t(ctx->seq) * uint64_t(ctx->kmax) + 1;
  a.prev2_epoch0 = call >= 2 ? uint64_t(ref.seq_hist[call & 1]) * uint64_t(ctx->kmax) + 1 : 0;
  a.seq = ctx->seq;
  a.prev2_seq = call >= 2 ? ref.seq_hist[call & 1] : -1;
  a.claim_base = ctx->claim_base;
  a.timeout_ns = uint64_t(ctx->timeout_ms) * 1000000ULL;
  a.hop_delay_ns = uint64_t(ctx->hop_delay_ns);
  a.err_host = ctx->d_err;
  a.abort_dev = ctx->d_abort;
  if (ctx->profile && !ctx->d_prof) {
    cudaError_t pe = cudaMalloc(reinterpret_cast<void **>(&ctx->d_prof), size_t(ctx->grid) * 64);
    if (pe == cudaSuccess) pe = cudaMemset(ctx->d_prof, 0, size_t(ctx->grid) * 64);
    if (pe != cudaSuccess) return cuda_fail(ctx, pe, "profile buffer");
  }
  a.prof = ctx->profile ? ctx->d_prof : nullptr;
  a.lr = lr;
  a.mu = momentum;
  a.wd = ctx->weight_decay;
  a.n = ctx->n;
  a.m = ctx->m;
  a.r = ctx->n_local;
  a.grid = ctx->grid;
  a.comm_ctas = twoshot ? 0 : ctx->p2p_variant;
  a.comm_batch = ctx->comm_batch;
  a.lag = twoshot ? (ctx->fold_lag + 1) / 2 : ctx->fold_lag;  // two-shot: per round
  a.release_delay = ctx->release_delay;
  a.release_every = ctx->release_every;
  a.release_stagger = ctx->release_stagger;
  a.parity = int(call & 1);
  a.my_rank = ctx->rank;
  a.bucket = bucket;
  a.nbuckets = int(ctx->buckets.size());
  a.discard = ctx->discard;
  a.experiment = ctx->experiment;
  a.protocol = ctx->protocol;
  a.cooperative = ctx->cooperative;
  a.counters = ctx->d_counters;
  a.ws_split = ctx->ws_split;
  const bool hybrid = twoshot && !nvls && ctx->protocol == 2 && ctx->n_local > 1 && ctx->wsm_hybrid &&
                      !ctx->device_iter && !dry;
  a.wsm_spanning_only = hybrid ? 1 : 0;
  for (int s = 0; s < ctx->n_local; ++s) {
    const int me = ctx->local_workers[s];
    a.my_workers[s] = int8_t(me);
    const int *G = ctx->canon + ctx->group_of[me] * ctx->m;
    bool all_local = true;
    for (int p = 0; p < ctx->m; ++p) {
      if (G[p] == me) a.my_pos[s] = int8_t(p);
      all_local = all_local && ctx->worker_rank[G[p]] == ctx->rank;
    }
    // the DIRECT kernel updates an all-local group in registers, once, by its first member
    const bool direct = (ctx->p2p_variant == 0);
    a.slot_kind[s] = int8_t(!direct || !all_local ? 0 : (G[0] == me ? 1 : 2));
  }
  for (int i = 0; i < ctx->n; ++i) {
    a.worker_rank[i] = ctx->worker_rank[i];
    a.worker_slot[i] = ctx->worker_slot[i];
    a.canon[i] = int8_t(ctx->canon[i]);
    a.group_of[i] = int8_t(ctx->group_of[i]);
  }
  bool vec = true;
  for (size_t b = 0; b < ctx->buckets.size(); ++b)
    if (bucket < 0 || int(b) == bucket) vec = vec && ctx->buckets[b].vec;
  const bool ws_kernel = twoshot && ctx->protocol == 2 && !nvls;
  const uint64_t claim_inc =
      (ws_kernel && ctx->m >= 2)  // every claimed unit + one failed claim per CTA
          ? uint64_t(ctx->n_local == 1 ? a.g1 - a.g0 : sesgd::p2p_wsm_units(ctx->n_local, ctx->m, a.g1 - a.g0)) +
                uint64_t(ctx->grid)
          : 0;
  if (ctx->device_iter) {
    if (!ws_kernel || dry)
      return fail(ctx, SESGD_ENOTSUP, "device iteration state: the exchange needs protocol 2 (K4W / K4W-M)");
    a.dev = ctx->d_iter;
    a.dev_buckets = ctx->d_bstate;
    a.dev_claim_inc = claim_inc;
    a.kmax = ctx->kmax;
  }
  if (dry) {
    *dry = a;
  } else {
    mark_start(ctx, st);
    if (hybrid) {
      const int rc = launch_local_groups(ctx, bucket, lr, momentum, st);
      if (rc != SESGD_OK) return rc;
    }
    cudaError_t e = (twoshot && ctx->protocol == 2 && !nvls)
                        ? (ctx->n_local == 1 ? sesgd::launch_p2p_ws(a, ctx->mode, vec, st)
                                             : sesgd::launch_p2p_wsm(a, ctx->mode, vec, st))
                    : twoshot ? sesgd::launch_p2p_twoshot(a, ctx->mode, vec, ctx->push_tma != 0, st)
                              : sesgd::launch_p2p_oneshot(a, ctx->p2p_variant, ctx->mode, vec,
                                                          ctx->guard_smem, st);
    if (e != cudaSuccess) return cuda_fail(ctx, e, twoshot ? "launch two-shot kernel" : "launch one-shot kernel");
    mark_end(ctx, st);
  }
  ctx->claim_base += claim_inc;
  // bookkeeping
  int remote_peers = 0;
  for (int s = 0; s < ctx->n_local; ++s) {
    const int me = ctx->local_workers[s];
    const int *G = ctx->canon + ctx->group_of[me] * ctx->m;
    for (int r = 0; r < ctx->m; ++r)
      if (G[r] != me && ctx->worker_rank[G[r]] != ctx->rank) remote_peers++;
  }
  for (size_t b = 0; b < ctx->buckets.size(); ++b) {
    if (bucket >= 0 && int(b) != bucket) continue;
    sesgd_bucket &bk = ctx->buckets[b];
    bk.seq_hist[bk.calls & 1] = ctx->seq;
    bk.calls++;
    bk.stats.kernel_launches += (bucket >= 0 || b == 0) ? 1 : 0;
    bk.stats.hbm_algo_bytes += 20 * bk.numel * ctx->n_local;
    if (ctx->m > 1 && twoshot) {  // RS + AG flag per (chunk, peer); 2 (m-1)/m of the bucket in
      bk.stats.handshake_rounds = 2;
      if (ctx->protocol == 0 || nvls)  // the value-carried protocols store no flag
        bk.stats.flag_messages += 2 * int64_t(remote_peers) * bk.nchunks;
      bk.stats.payload_bytes_in += 2 * int64_t(remote_peers) * bk.numel * 4 / ctx->m;
    } else if (ctx->m > 1) {
      bk.stats.handshake_rounds = 1;
      bk.stats.flag_messages += int64_t(remote_peers) * bk.nchunks;  // one ready flag per chunk
      bk.stats.payload_bytes_in += int64_t(remote_peers) * bk.numel * 4;
    }
  }
  ctx->seq++;
  return SESGD_OK;
}

}  // namespace

extern "C" {

const char *sesgd_strerror(int code) {
  switch (code) {
    case SESGD_OK: return "ok";
    case SESGD_EINVAL: return "invalid argument";
    case SESGD_ENOTDIV: return "group_size does not divide n";
    case SESGD_ESTATE: return "invalid state for this call";
    case SESGD_ECUDA: return "CUDA error";
    case SESGD_ETIMEOUT: return "group peer timed out";
    case SESGD_ENOMEM: return "out of memory";
    case SESGD_ENOTSUP: return "not supported";
    default: return "unknown status";
  }
}

const char *sesgd_last_error(const sesgd_ctx *ctx) {
  return ctx ? ctx->last_error.c_str() : "null context";
}

int sesgd_init(int32_t n, int32_t group_size, uint64_t seed, sesgd_ctx **out) {
  if (!out) return SESGD_EINVAL;
  *out = nullptr;
  if (!valid_nm(n, group_size)) return SESGD_EINVAL;
  if (n % group_size != 0) return SESGD_ENOTDIV;
  sesgd_ctx *ctx = new (std::nothrow) sesgd_ctx();
  if (!ctx) return SESGD_ENOMEM;
  ctx->n = n;
  ctx->m = group_size;
  ctx->seed = seed;
  std::memset(ctx->slot_of, -1, sizeof(ctx->slot_of));
  *out = ctx;
  return SESGD_OK;
}

void sesgd_destroy(sesgd_ctx *ctx) {
  if (!ctx) return;
  for (auto &b : ctx->buckets) free_bucket(b);
  if (ctx->h_err) cudaFreeHost(ctx->h_err);
  if (ctx->d_abort) cudaFree(ctx->d_abort);
  if (ctx->d_prof) cudaFree(ctx->d_prof);
  if (ctx->d_meta) cudaFree(ctx->d_meta);
  if (ctx->d_bx) cudaFree(ctx->d_bx);
  if (ctx->d_bv) cudaFree(ctx->d_bv);
  if (ctx->d_bg) cudaFree(const_cast<float **>(ctx->d_bg));
  if (ctx->d_numels) cudaFree(ctx->d_numels);
  if (ctx->d_counters) cudaFree(ctx->d_counters);
  if (ctx->d_iter) cudaFree(ctx->d_iter);
  if (ctx->d_bstate) cudaFree(ctx->d_bstate);
  if (ctx->ev_l0) cudaEventDestroy(ctx->ev_l0);
  if (ctx->ev_l1) cudaEventDestroy(ctx->ev_l1);
  for (auto *v : {&ctx->ev_in, &ctx->ev_k, &ctx->ev_out})
    for (cudaEvent_t e : *v) cudaEventDestroy(e);
  if (ctx->ev_start) cudaEventDestroy(ctx->ev_start);
  if (ctx->copy_in) cudaStreamDestroy(ctx->copy_in);
  if (ctx->copy_out) cudaStreamDestroy(ctx->copy_out);
  delete ctx;
}

int sesgd_groups(const sesgd_ctx *ctx, int64_t iter, int32_t *perm_out, int32_t *group_of_out) {
  if (!ctx || !perm_out || iter < 0) return SESGD_EINVAL;
  make_groups(ctx, iter, perm_out, group_of_out);
  return SESGD_OK;
}

int sesgd_latency_model(int32_t n, int32_t group_size, double bytes, double nu_Bps, double tau_s,
                        sesgd_cost *out) {
  if (!out || n < 1 || group_size < 1 || group_size > n) return SESGD_EINVAL;
  if (n % group_size != 0) return SESGD_ENOTDIV;
  if (!(nu_Bps > 0.0) || !(tau_s >= 0.0) || !(bytes >= 0.0)) return SESGD_EINVAL;
  sesgd::latency_model(n, group_size, bytes, nu_Bps, tau_s, out);
  return SESGD_OK;
}

int sesgd_set_option(sesgd_ctx *ctx, int32_t option, int64_t value) {
  if (!ctx) return SESGD_EINVAL;
  switch (option) {
    case SESGD_OPT_MODE:
      if (value != SESGD_MODE_PARAM_AVG && value != SESGD_MODE_GRAD_AVG)
        return fail(ctx, SESGD_EINVAL, "mode must be SESGD_MODE_PARAM_AVG or SESGD_MODE_GRAD_AVG");
      ctx->mode = int(value);
      return SESGD_OK;
    case SESGD_OPT_PATH:
      if (value < SESGD_PATH_AUTO || value > SESGD_PATH_NVLS)
        return fail(ctx, SESGD_EINVAL, "unknown path");
      if (ctx->peers && value != ctx->path)  // the consumption guards are per path
        return fail(ctx, SESGD_ESTATE, "the path is fixed once peers attach");
      if (value == SESGD_PATH_TWOSHOT && ctx->layout_frozen && ctx->p2p_variant != 0)
        return fail(ctx, SESGD_ESTATE, "the two-shot path needs the DIRECT layout (P2P variant 0)");
      ctx->path = int(value);
      return SESGD_OK;
    case SESGD_OPT_TIMEOUT_MS:
      if (value < 1) return fail(ctx, SESGD_EINVAL, "timeout must be >= 1 ms");
      ctx->timeout_ms = value;
      return SESGD_OK;
    case SESGD_OPT_GRID:
      if (value < 0) return fail(ctx, SESGD_EINVAL, "grid must be >= 0");
      if (ctx->layout_frozen) return fail(ctx, SESGD_ESTATE, "grid is fixed once peers attach");
      ctx->grid_opt = value;
      return SESGD_OK;
    case SESGD_OPT_P2P_VARIANT:
      if (!sesgd::p2p_variant_valid(int(value))) return fail(ctx, SESGD_EINVAL, "unknown P2P variant");
      if (ctx->layout_frozen) return fail(ctx, SESGD_ESTATE, "variant is fixed once peers attach");
      ctx->p2p_variant = int(value);
      return SESGD_OK;
    case SESGD_OPT_COMM_BATCH:
      if (value < 1 || value > 1024) return fail(ctx, SESGD_EINVAL, "comm batch must be in [1, 1024]");
      if (ctx->layout_frozen) return fail(ctx, SESGD_ESTATE, "comm batch is fixed once peers attach");
      ctx->comm_batch = int(value);
      return SESGD_OK;
    case SESGD_OPT_FOLD_LAG:
      if (value < 1 || value > 64) return fail(ctx, SESGD_EINVAL, "fold lag must be in [1, 64]");
      ctx->fold_lag = int(value);
      return SESGD_OK;
    case SESGD_OPT_RESIDENT_UNROLL:
      if (value != 0 && value != 1 && value != 2 && value != 4 && value != 8)
        return fail(ctx, SESGD_EINVAL, "resident unroll must be 0, 1, 2, 4 or 8");
      ctx->resident_unroll = int(value);
      return SESGD_OK;
    case SESGD_OPT_PUSH_TMA:
      if (value != 0 && value != 1) return fail(ctx, SESGD_EINVAL, "push TMA must be 0 or 1");
      ctx->push_tma = int(value);
      return SESGD_OK;
    case SESGD_OPT_RELEASE_DELAY:
      if (value < 1 || value > 8) return fail(ctx, SESGD_EINVAL, "release delay must be in [1, 8]");
      ctx->release_delay = int(value);
      return SESGD_OK;
    case SESGD_OPT_RELEASE_EVERY:
      if (value < 1 || value > 16) return fail(ctx, SESGD_EINVAL, "release interval must be in [1, 16]");
      ctx->release_every = int(value);
      return SESGD_OK;
    case SESGD_OPT_SCHEDULE: {
      auto pow2 = [](int v) { return v > 0 && (v & (v - 1)) == 0; };
      if (value != 0 && value != 1) return fail(ctx, SESGD_EINVAL, "schedule must be 0 or 1");
      if (value == 1 && (!pow2(ctx->n) || !pow2(ctx->m)))
        return fail(ctx, SESGD_EINVAL, "the dimension-exchange schedule needs n and group_size powers of two");
      ctx->schedule = int(value);
      return SESGD_OK;
    }
    case SESGD_OPT_WSM_HYBRID:
      if (value != 0 && value != 1) return fail(ctx, SESGD_EINVAL, "WSM hybrid must be 0 or 1");
      ctx->wsm_hybrid = int(value);
      return SESGD_OK;
    case SESGD_OPT_WS_SPLIT:
      if (value != 8 && value != 12 && value != 16) return fail(ctx, SESGD_EINVAL, "WS split must be 8, 12 or 16");
      ctx->ws_split = int(value);
      return SESGD_OK;
    case SESGD_OPT_DEVICE_ITER:
      if (value != 0 && value != 1) return fail(ctx, SESGD_EINVAL, "device iteration must be 0 or 1");
      if (value == ctx->device_iter) return SESGD_OK;
      return value ? device_iter_enable(ctx) : device_iter_disable(ctx);
    case SESGD_OPT_LOCAL_PERIOD:
      if (value < 1) return fail(ctx, SESGD_EINVAL, "local period must be >= 1");
      if (value > 1 && ctx->device_iter) return fail(ctx, SESGD_ENOTSUP, "Local-SESGD with the device iteration state");
      ctx->local_period = value;
      return SESGD_OK;
    case SESGD_OPT_RELEASE_STAGGER:
      if (value != 0 && value != 1) return fail(ctx, SESGD_EINVAL, "release stagger must be 0 or 1");
      ctx->release_stagger = int(value);
      return SESGD_OK;
    case SESGD_OPT_PAYLOAD_BF16:
      if (value != 0 && value != 1) return fail(ctx, SESGD_EINVAL, "bf16 payload must be 0 or 1");
      ctx->payload_bf16 = int(value);
      return SESGD_OK;
    case SESGD_OPT_SM_BUDGET:
      if (value < 0) return fail(ctx, SESGD_EINVAL, "SM budget must be >= 0");
      if (ctx->layout_frozen) return fail(ctx, SESGD_ESTATE, "the SM budget is fixed once the layout freezes");
      ctx->sm_budget = int(value);
      if (ctx->attached)
        ctx->sm_count = ctx->sm_budget > 0 ? std::min(ctx->sm_budget, ctx->dev_sm_count) : ctx->dev_sm_count;
      return SESGD_OK;
    case SESGD_OPT_PROFILE:
      if (value != 0 && value != 1) return fail(ctx, SESGD_EINVAL, "profile must be 0 or 1");
      ctx->profile = int(value);
      return SESGD_OK;
    case SESGD_OPT_DISCARD:
      if (value != 0 && value != 1) return fail(ctx, SESGD_EINVAL, "discard must be 0 or 1");
      ctx->discard = int(value);
      return SESGD_OK;
    case SESGD_OPT_PROTOCOL:
      if (value < -1 || value > 2) return fail(ctx, SESGD_EINVAL, "protocol must be -1 (auto), 0, 1 or 2");
      if (ctx->layout_frozen) return fail(ctx, SESGD_ESTATE, "the protocol is fixed once the layout freezes");
      ctx->protocol = int(value);
      return SESGD_OK;
    case SESGD_OPT_COOPERATIVE:
      if (value != 0 && value != 1) return fail(ctx, SESGD_EINVAL, "cooperative must be 0 or 1");
      ctx->cooperative = int(value);
      return SESGD_OK;
    case SESGD_OPT_EXPERIMENT:
      if (value < 0 || value > 3) return fail(ctx, SESGD_EINVAL, "experiment bits must be in [0, 3]");
      ctx->experiment = int(value);
      return SESGD_OK;
    case SESGD_OPT_HOP_DELAY_NS:
      if (value < 0) return fail(ctx, SESGD_EINVAL, "delay must be >= 0");
      ctx->hop_delay_ns = value;
      return SESGD_OK;
    default:
      return fail(ctx, SESGD_EINVAL, "unknown option");
  }
}

int sesgd_set_weight_decay(sesgd_ctx *ctx, float weight_decay) {
  if (!ctx) return SESGD_EINVAL;
  if (!std::isfinite(weight_decay) || weight_decay < 0.f)
    return fail(ctx, SESGD_EINVAL, "weight decay must be finite and >= 0");
  ctx->weight_decay = weight_decay;
  return SESGD_OK;
}

int sesgd_attach(sesgd_ctx *ctx, int32_t device, int32_t n_local, const int32_t *local_workers) {
  if (!ctx) return SESGD_EINVAL;
  if (ctx->attached) return fail(ctx, SESGD_ESTATE, "already attached");
  if (n_local < 1 || n_local > ctx->n || !local_workers)
    return fail(ctx, SESGD_EINVAL, "n_local must be in [1, n] with a worker list");
  int8_t slot_of[SESGD_MAX_WORKERS];
  std::memset(slot_of, -1, sizeof(slot_of));
  for (int s = 0; s < n_local; ++s) {
    const int w = local_workers[s];
    if (w < 0 || w >= ctx->n) return fail(ctx, SESGD_EINVAL, "worker id out of range");
    if (slot_of[w] >= 0) return fail(ctx, SESGD_EINVAL, "duplicate worker id");
    slot_of[w] = int8_t(s);
  }
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaSetDevice");
  int sms = 0;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaDeviceGetAttribute");
  unsigned long long *h = nullptr;
  e = cudaHostAlloc(reinterpret_cast<void **>(&h), 8 * sizeof(unsigned long long), cudaHostAllocMapped);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaHostAlloc(error block)");
  std::memset(h, 0, 8 * sizeof(unsigned long long));
  unsigned long long *d = nullptr;
  e = cudaHostGetDevicePointer(reinterpret_cast<void **>(&d), h, 0);
  if (e != cudaSuccess) {
    cudaFreeHost(h);
    return cuda_fail(ctx, e, "cudaHostGetDevicePointer");
  }
  unsigned int *ab = nullptr;
  e = cudaMalloc(reinterpret_cast<void **>(&ab), sizeof(unsigned int));
  if (e == cudaSuccess) e = cudaMemset(ab, 0, sizeof(unsigned int));
  if (e != cudaSuccess) {
    cudaFreeHost(h);
    return cuda_fail(ctx, e, "cudaMalloc(abort word)");
  }
  unsigned long long *cnt = nullptr;
  e = cudaMalloc(reinterpret_cast<void **>(&cnt), sesgd::kNumCounters * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemset(cnt, 0, sesgd::kNumCounters * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaEventCreate(&ctx->ev_l0);
  if (e == cudaSuccess) e = cudaEventCreate(&ctx->ev_l1);
  if (e != cudaSuccess) {
    cudaFreeHost(h);
    cudaFree(ab);
    if (cnt) cudaFree(cnt);
    return cuda_fail(ctx, e, "device counters");
  }
  ctx->d_counters = cnt;
  ctx->h_err = h;
  ctx->d_err = d;
  ctx->d_abort = ab;
  ctx->device = device;
  ctx->dev_sm_count = sms;
  ctx->sm_count = ctx->sm_budget > 0 ? std::min(ctx->sm_budget, sms) : sms;
  ctx->n_local = n_local;
  ctx->local_workers.assign(local_workers, local_workers + n_local);
  std::memcpy(ctx->slot_of, slot_of, sizeof(slot_of));
  ctx->attached = true;
  return SESGD_OK;
}

int sesgd_register_bucket(sesgd_ctx *ctx, int32_t bucket, int64_t numel, float *const *x,
                          float *const *v, const float *const *g) {
  if (!ctx) return SESGD_EINVAL;
  if (!ctx->attached) return fail(ctx, SESGD_ESTATE, "sesgd_attach first");
  if (bucket < 0 || bucket >= kMaxBuckets) return fail(ctx, SESGD_EINVAL, "bucket id out of range");
  if (numel < 0 || !x || !v || !g) return fail(ctx, SESGD_EINVAL, "null pointer table or numel < 0");
  if (ctx->device_iter) return fail(ctx, SESGD_ESTATE, "buckets are fixed while the device iteration state is on");
  if (ctx->layout_frozen && (size_t(bucket) >= ctx->buckets.size() ||
                             ctx->buckets[bucket].numel != numel))
    return fail(ctx, SESGD_ESTATE, "bucket layout is fixed once peers attach");
  bool vec = true;
  for (int s = 0; s < ctx->n_local; ++s) {
    if (numel > 0 && (!x[s] || !v[s] || !g[s]))
      return fail(ctx, SESGD_EINVAL, "null device pointer");
    vec = vec && aligned16(x[s]) && aligned16(v[s]) && aligned16(g[s]);
  }
  if (size_t(bucket) >= ctx->buckets.size()) ctx->buckets.resize(size_t(bucket) + 1);
  sesgd_bucket &b = ctx->buckets[bucket];
  const size_t bytes = sizeof(float *) * size_t(ctx->n_local);
  if (!b.d_x) {
    cudaError_t e = cudaMalloc(reinterpret_cast<void **>(&b.d_x), bytes);
    if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void **>(&b.d_v), bytes);
    if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void **>(&b.d_g), bytes);
    if (e != cudaSuccess) {
      free_bucket(b);
      return cuda_fail(ctx, e, "cudaMalloc(pointer tables)");
    }
  }
  b.hx.assign(x, x + ctx->n_local);
  b.hv.assign(v, v + ctx->n_local);
  b.hg.assign(g, g + ctx->n_local);
  cudaError_t e = cudaMemcpy(b.d_x, b.hx.data(), bytes, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(b.d_v, b.hv.data(), bytes, cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = cudaMemcpy(const_cast<float **>(b.d_g), b.hg.data(), bytes, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMemcpy(pointer tables)");
  b.numel = numel;
  b.vec = vec;
  b.registered = true;
  ctx->resident_tables_ok = false;  // the all-bucket resident launch re-uploads its tables
  if (ctx->layout_frozen) return upload_tables(ctx);  // re-registration after the layout froze
  return SESGD_OK;
}

int sesgd_workspace_bytes(const sesgd_ctx *cctx, int64_t *bytes_out) {
  sesgd_ctx *ctx = const_cast<sesgd_ctx *>(cctx);
  if (!ctx || !bytes_out) return SESGD_EINVAL;
  if (!ctx->attached || ctx->buckets.empty())
    return fail(ctx, SESGD_ESTATE, "attach and register buckets first");
  for (auto &b : ctx->buckets)
    if (!b.registered) return fail(ctx, SESGD_ESTATE, "bucket ids must be dense from 0");
  if (!ctx->layout_frozen) freeze_layout(ctx);
  *bytes_out = ctx->ws_bytes;
  return SESGD_OK;
}

int sesgd_workspace_prepare(sesgd_ctx *ctx, void *local_ws) {
  if (!ctx || !local_ws) return SESGD_EINVAL;
  int64_t bytes = 0;
  int rc = sesgd_workspace_bytes(ctx, &bytes);
  if (rc != SESGD_OK) return rc;
  // zero flags (stage contents are don't-care), then the header; the value-carried protocol
  // arms every receive float with the sentinel (0xFFFFFFFF)
  cudaError_t e = cudaMemset(local_ws, 0, size_t(ctx->stage_off));
  if (e == cudaSuccess && ctx->protocol >= 1)
    e = cudaMemset(static_cast<char *>(local_ws) + ctx->recv_off, 0xFF,
                   size_t(2 * int64_t(ctx->n_local) * ctx->m * ctx->stage_slot_floats * 4));
  uint64_t hdr[2] = {kMagic, ctx->layout_hash};
  if (e == cudaSuccess) e = cudaMemcpy(local_ws, hdr, sizeof(hdr), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cuda_fail(ctx, e, "workspace prepare");
  return SESGD_OK;
}

int sesgd_attach_peers(sesgd_ctx *ctx, int32_t n_ranks, int32_t rank, void *const *rank_ws,
                       const int32_t *worker_rank) {
  if (!ctx || !rank_ws || !worker_rank) return SESGD_EINVAL;
  if (n_ranks < 1 || n_ranks > SESGD_MAX_RANKS || rank < 0 || rank >= n_ranks)
    return fail(ctx, SESGD_EINVAL, "rank / n_ranks out of range");
  if (!ctx->layout_frozen) return fail(ctx, SESGD_ESTATE, "sesgd_workspace_prepare first");
  // worker -> (rank, slot): slot = position among the rank's workers in ascending id
  int count[SESGD_MAX_RANKS] = {0};
  for (int w = 0; w < ctx->n; ++w) {
    const int r = worker_rank[w];
    if (r < 0 || r >= n_ranks) return fail(ctx, SESGD_EINVAL, "worker_rank out of range");
    ctx->worker_rank[w] = int8_t(r);
    ctx->worker_slot[w] = int8_t(count[r]++);
  }
  for (int r = 0; r < n_ranks; ++r)
    if (count[r] != ctx->n_local)
      return fail(ctx, SESGD_EINVAL, "every rank must host the same number of workers");
  for (int s = 0; s < ctx->n_local; ++s) {
    const int w = ctx->local_workers[s];
    if (ctx->worker_rank[w] != rank || ctx->worker_slot[w] != s)
      return fail(ctx, SESGD_EINVAL, "local workers must be this rank's workers in ascending order");
  }
  for (int r = 0; r < n_ranks; ++r) {
    if (!rank_ws[r]) return fail(ctx, SESGD_EINVAL, "null workspace pointer");
    uint64_t hdr[2] = {0, 0};
    cudaError_t e = cudaMemcpy(hdr, rank_ws[r], sizeof(hdr), cudaMemcpyDefault);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "reading a peer workspace header");
    if (hdr[0] != kMagic || hdr[1] != ctx->layout_hash) {
      char buf[160];
      std::snprintf(buf, sizeof buf, "rank %d workspace layout differs (magic %llx hash %llx vs %llx)",
                    r, (unsigned long long)hdr[0], (unsigned long long)hdr[1],
                    (unsigned long long)ctx->layout_hash);
      return fail(ctx, SESGD_ESTATE, buf);
    }
    ctx->ws[r] = static_cast<char *>(rank_ws[r]);
    // a peer workspace on another device of this process (e.g. mapped through CUDA IPC) needs
    // peer access from this device; symmetric-memory mappings already have it
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, rank_ws[r]) == cudaSuccess && pa.type == cudaMemoryTypeDevice &&
        pa.device != ctx->device) {
      int cur = 0;
      cudaGetDevice(&cur);
      cudaSetDevice(ctx->device);
      const cudaError_t pe = cudaDeviceEnablePeerAccess(pa.device, 0);
      cudaSetDevice(cur);
      if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled)
        return cuda_fail(ctx, pe, "enabling peer access to a peer workspace");
      cudaGetLastError();  // clear a sticky "already enabled"
    }
  }
  ctx->n_ranks = n_ranks;
  ctx->rank = rank;
  int rc = upload_tables(ctx);
  if (rc != SESGD_OK) return rc;
  ctx->peers = true;
  return SESGD_OK;
}

int sesgd_pair_counts(sesgd_ctx *ctx, int64_t t0, int64_t T, unsigned long long *counts_dev,
                      void *stream) {
  if (!ctx || !counts_dev || t0 < 0 || T < 0) return SESGD_EINVAL;
  if (!ctx->attached) return fail(ctx, SESGD_ESTATE, "sesgd_attach first");
  if (T == 0) return SESGD_OK;
  cudaError_t e = sesgd::launch_pair_counts(ctx->seed, t0, T, ctx->n, ctx->m, ctx->schedule, counts_dev,
                                            ctx->sm_count, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(ctx, e, "launch pair counts");
  return SESGD_OK;
}

int sesgd_attach_multicast(sesgd_ctx *ctx, void *mc_ws) {
  if (!ctx || !mc_ws) return SESGD_EINVAL;
  if (!ctx->peers) return fail(ctx, SESGD_ESTATE, "sesgd_attach_peers first");
  ctx->mc_ws = static_cast<char *>(mc_ws);
  return SESGD_OK;
}

int sesgd_begin_iter(sesgd_ctx *ctx, int64_t iter) {
  if (!ctx) return SESGD_EINVAL;
  if (iter < 0) return fail(ctx, SESGD_EINVAL, "iteration must be >= 0");
  if (!ctx->attached) return fail(ctx, SESGD_ESTATE, "sesgd_attach first");
  if (ctx->device_iter)
    return fail(ctx, SESGD_ESTATE, "the iteration lives on the device: sesgd_begin_iter_device");
  make_groups(ctx, iter, ctx->canon, ctx->group_of);
  ctx->t = iter;
  ctx->iter_set = true;
  return SESGD_OK;
}

int sesgd_begin_iter_device(sesgd_ctx *ctx, int64_t iter, void *stream) {
  if (!ctx) return SESGD_EINVAL;
  if (iter < -1) return fail(ctx, SESGD_EINVAL, "iteration must be >= 0 or SESGD_ITER_NEXT");
  if (!ctx->device_iter) return fail(ctx, SESGD_ESTATE, "SESGD_OPT_DEVICE_ITER is off");
  cudaError_t e = sesgd::launch_iter_begin(iter_begin_args(ctx, iter), ctx->d_iter, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(ctx, e, "launch begin_iter_device");
  ctx->t = iter >= 0 ? iter : (ctx->iter_set ? ctx->t + 1 : 0);  // the host shadow (per enqueue)
  make_groups(ctx, ctx->t, ctx->canon, ctx->group_of);
  ctx->iter_set = true;
  return SESGD_OK;
}

int sesgd_device_iter_ptr(const sesgd_ctx *ctx, const int64_t **t_dev_out) {
  if (!ctx || !t_dev_out) return SESGD_EINVAL;
  if (!ctx->device_iter) return SESGD_ESTATE;
  *t_dev_out = &ctx->d_iter->t;
  return SESGD_OK;
}

int sesgd_device_iter_read(const sesgd_ctx *ctx, sesgd_device_iter_state *out, int64_t *bucket_calls,
                           int32_t nbuckets) {
  if (!ctx || !out || nbuckets < 0 || (nbuckets > 0 && !bucket_calls)) return SESGD_EINVAL;
  if (!ctx->device_iter) return SESGD_ESTATE;
  sesgd::DevIter h{};
  std::vector<sesgd::DevBucket> hb(ctx->buckets.size());
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpy(&h, ctx->d_iter, sizeof(h), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(hb.data(), ctx->d_bstate, hb.size() * sizeof(sesgd::DevBucket), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return SESGD_ECUDA;
  out->t = h.t;
  out->seq = h.seq;
  out->claim_base = int64_t(h.claim_base);
  for (int i = 0; i < SESGD_MAX_WORKERS; ++i) {
    out->canon[i] = i < ctx->n ? h.canon[i] : -1;
    out->ring_rank[i] = i < ctx->m ? h.ring_rank[i] : -1;
  }
  out->ring_pos = h.ring_pos;
  for (int b = 0; b < nbuckets && size_t(b) < hb.size(); ++b) bucket_calls[b] = hb[b].calls;
  return SESGD_OK;
}

int sesgd_sync_step(sesgd_ctx *ctx, int32_t bucket, float lr, float momentum, void *stream) {
  if (!ctx) return SESGD_EINVAL;
  int rc = check_latched(ctx);
  if (rc != SESGD_OK) return rc;
  if (!ctx->attached || !ctx->iter_set) return fail(ctx, SESGD_ESTATE, "attach and begin_iter first");
  if (bucket < 0 || size_t(bucket) >= ctx->buckets.size() || !ctx->buckets[bucket].registered)
    return fail(ctx, SESGD_EINVAL, "bucket not registered");
  if (!std::isfinite(lr) || !std::isfinite(momentum))
    return fail(ctx, SESGD_EINVAL, "lr and momentum must be finite");
  sesgd_bucket &b = ctx->buckets[bucket];
  b.stats.sync_calls++;
  if (b.numel == 0) return SESGD_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (local_only_iteration(ctx)) return local_step(ctx, bucket, lr, momentum, st);
  const bool all_local = (ctx->n_local == ctx->n);
  const int path = resolve_path(ctx);

  if (path == SESGD_PATH_RESIDENT) {
    if (!all_local) return fail(ctx, SESGD_ESTATE, "resident path needs all n workers on this GPU");
    if (ctx->payload_bf16)  // R21 rounds what crosses NVLink; K6 keeps every contribution in fp32
      return fail(ctx, SESGD_ENOTSUP, "the bf16 payload needs a multi-GPU two-shot path (K4), not K6");
    ResidentArgs a{};
    a.x = b.d_x;
    a.v = b.d_v;
    a.g = b.d_g;
    a.numel = b.numel;
    a.lr = lr;
    a.mu = momentum;
    a.wd = ctx->weight_decay;
    a.m = ctx->m;
    a.k = ctx->n / ctx->m;
    for (int i = 0; i < ctx->n; ++i) a.member_slot[i] = ctx->slot_of[ctx->canon[i]];
    a.dev = ctx->device_iter ? ctx->d_iter : nullptr;
    const int gx = resident_grid_x(ctx, b.vec, b.numel);
    mark_start(ctx, st);
    cudaError_t e = sesgd::launch_resident(a, ctx->mode, b.vec, gx, ctx->resident_unroll, st);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "launch resident kernel");
    mark_end(ctx, st);
    b.stats.kernel_launches++;
    b.stats.hbm_algo_bytes += 20 * b.numel * ctx->n;
    return SESGD_OK;
  }

  if (path == SESGD_PATH_RING) {  // K5: paper-faithful ring inside each group
    if (!ctx->peers) return fail(ctx, SESGD_ESTATE, "sesgd_attach_peers first (multi-GPU path)");
    if (ctx->n_local != 1 || ctx->ring_grid == 0)
      return fail(ctx, SESGD_ENOTSUP, "the ring path needs one worker per GPU and group_size >= 2");
    sesgd::RingArgs ra{};
    ra.x = b.hx[0];
    ra.v = b.hv[0];
    ra.g = b.hg[0];
    for (int r = 0; r < ctx->n_ranks; ++r) ra.ws[r] = ctx->ws[r];
    ra.numel = b.numel;
    ra.rbuf_off = b.ring_off;
    ra.slice_cap = b.ring_cap;
    ra.rflag_off = ctx->rflag_off;
    ra.rcons_off = ctx->rcons_off;
    ra.call = b.calls;
    ra.timeout_ns = uint64_t(ctx->timeout_ms) * 1000000ULL;
    ra.hop_delay_ns = uint64_t(ctx->hop_delay_ns);
    ra.err_host = ctx->d_err;
    ra.abort_dev = ctx->d_abort;
    ra.lr = lr;
    ra.mu = momentum;
    ra.wd = ctx->weight_decay;
    ra.parity = int(b.calls & 1);
    ra.steps = 2 * (ctx->m - 1);
    ra.m = ctx->m;
    ra.grid = ctx->ring_grid;
    ra.my_rank = ctx->rank;
    ra.bucket = bucket;
    ra.nbuckets = int(ctx->buckets.size());
    ra.cooperative = ctx->cooperative;
    ra.counters = ctx->d_counters;
    const int me = ctx->local_workers[0];
    const int *G = ctx->canon + ctx->group_of[me] * ctx->m;
    for (int q = 0; q < ctx->m; ++q) {
      ra.ring_rank[q] = ctx->worker_rank[G[q]];
      if (G[q] == me) ra.pos = q;
    }
    ra.seq = ctx->seq;
    if (ctx->device_iter) {
      ra.dev = ctx->d_iter;
      ra.dev_buckets = ctx->d_bstate;
    }
    mark_start(ctx, st);
    cudaError_t e = sesgd::launch_ring(ra, ctx->mode, st);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "launch ring kernel");
    mark_end(ctx, st);
    b.seq_hist[b.calls & 1] = ctx->seq;  // keep the one-shot guard history consistent
    b.calls++;
    ctx->seq++;
    b.stats.kernel_launches++;
    b.stats.hbm_algo_bytes += 20 * b.numel;
    if (ctx->m > 1) {
      b.stats.handshake_rounds = 2 * (ctx->m - 1);  // Eq. 2 / Eq. 3: 2(m-1) per call
      b.stats.flag_messages += 2 * int64_t(ctx->m - 1) * ctx->ring_grid;
      b.stats.payload_bytes_in += 2 * int64_t(ctx->m - 1) * ((b.numel + ctx->m - 1) / ctx->m) * 4;
    }
    return SESGD_OK;
  }

  // one-shot (K3) or two-shot (K4) push over NVLink P2P
  if (!ctx->peers) return fail(ctx, SESGD_ESTATE, "sesgd_attach_peers first (multi-GPU path)");
  if (path == SESGD_PATH_TWOSHOT && (ctx->p2p_variant != 0 || (ctx->push_tma && ctx->n_local != 1)))
    return fail(ctx, SESGD_ENOTSUP, "two-shot needs the DIRECT layout; its TMA pushes one worker per GPU");
  if (ctx->payload_bf16 && (path != SESGD_PATH_TWOSHOT || ctx->push_tma))
    return fail(ctx, SESGD_ENOTSUP, "the bf16 payload needs the two-shot path with LSU pushes");
  if (ctx->protocol >= 1 && (path != SESGD_PATH_TWOSHOT || ctx->push_tma || ctx->payload_bf16))
    return fail(ctx, SESGD_ENOTSUP, "the value-carried protocol needs the fp32 two-shot path with LSU pushes");
  if (ctx->protocol == 2 && ctx->n_local != 1 && !sesgd::p2p_wsm_supported(ctx->n_local, ctx->m))
    return fail(ctx, SESGD_ENOTSUP, "protocol 2 (K4W-M) supports 2..8 workers per GPU");
  if (path == SESGD_PATH_NVLS && (ctx->p2p_variant != 0 || ctx->n_local != 1 || ctx->m != ctx->n || !ctx->mc_ws))
    return fail(ctx, SESGD_ENOTSUP,
                "the NVLS path needs one worker per GPU, group_size = n and sesgd_attach_multicast");
  return launch_oneshot(ctx, bucket, lr, momentum, st,
                        path == SESGD_PATH_TWOSHOT || path == SESGD_PATH_NVLS, path == SESGD_PATH_NVLS);
}

int sesgd_sync_all(sesgd_ctx *ctx, float lr, float momentum, void *stream) {
  if (!ctx) return SESGD_EINVAL;
  int rc = check_latched(ctx);
  if (rc != SESGD_OK) return rc;
  if (!ctx->attached || !ctx->iter_set) return fail(ctx, SESGD_ESTATE, "attach and begin_iter first");
  if (ctx->buckets.empty()) return fail(ctx, SESGD_ESTATE, "no bucket registered");
  for (auto &b : ctx->buckets)
    if (!b.registered) return fail(ctx, SESGD_ESTATE, "bucket ids must be dense from 0");
  if (!std::isfinite(lr) || !std::isfinite(momentum))
    return fail(ctx, SESGD_EINVAL, "lr and momentum must be finite");
  if (local_only_iteration(ctx)) {  // Local-SESGD: local step only, every bucket in one launch
    for (auto &b : ctx->buckets) b.stats.sync_calls++;
    return local_step(ctx, -1, lr, momentum, static_cast<cudaStream_t>(stream));
  }
  const bool all_local = (ctx->n_local == ctx->n);
  const int path = resolve_path(ctx);
  if (path == SESGD_PATH_RESIDENT && all_local) {  // K6 over every bucket in one launch
    if (ctx->payload_bf16)
      return fail(ctx, SESGD_ENOTSUP, "the bf16 payload needs a multi-GPU two-shot path (K4), not K6");
    if (!ctx->resident_tables_ok) {
      rc = upload_resident_tables(ctx);
      if (rc != SESGD_OK) return rc;
    }
    ResidentArgs a{};
    bool vec = true;
    int64_t biggest = 0;
    for (auto &b : ctx->buckets) {
      vec = vec && b.vec;
      biggest = std::max(biggest, b.numel);
    }
    a.lr = lr;
    a.mu = momentum;
    a.wd = ctx->weight_decay;
    a.m = ctx->m;
    a.k = ctx->n / ctx->m;
    a.nb = int(ctx->buckets.size());
    a.n_local = ctx->n_local;
    a.bx = ctx->d_bx;
    a.bv = ctx->d_bv;
    a.bg = ctx->d_bg;
    a.numels = ctx->d_numels;
    for (int i = 0; i < ctx->n; ++i) a.member_slot[i] = ctx->slot_of[ctx->canon[i]];
    a.dev = ctx->device_iter ? ctx->d_iter : nullptr;
    mark_start(ctx, static_cast<cudaStream_t>(stream));
    cudaError_t e = sesgd::launch_resident(a, ctx->mode, vec, resident_grid_x(ctx, vec, biggest),
                                           ctx->resident_unroll, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(ctx, e, "launch resident kernel (all buckets)");
    mark_end(ctx, static_cast<cudaStream_t>(stream));
    for (auto &b : ctx->buckets) {
      b.stats.sync_calls++;
      b.stats.hbm_algo_bytes += 20 * b.numel * ctx->n;
    }
    ctx->buckets[0].stats.kernel_launches++;
    return SESGD_OK;
  }
  const bool nvls = (path == SESGD_PATH_NVLS);
  const bool twoshot = (path == SESGD_PATH_TWOSHOT) || nvls;
  bool fuse = (path == SESGD_PATH_ONESHOT ||
               (twoshot && ctx->p2p_variant == 0 && (!ctx->push_tma || ctx->n_local == 1)) ||
               (nvls && ctx->n_local == 1 && ctx->m == ctx->n && ctx->mc_ws)) &&
              ctx->peers;
  for (auto &b : ctx->buckets)  // one launch needs one shared call history
    fuse = fuse && b.calls == ctx->buckets[0].calls && b.seq_hist[0] == ctx->buckets[0].seq_hist[0] &&
           b.seq_hist[1] == ctx->buckets[0].seq_hist[1];
  if (!fuse) {
    for (size_t b = 0; b < ctx->buckets.size(); ++b) {
      rc = sesgd_sync_step(ctx, int32_t(b), lr, momentum, stream);
      if (rc != SESGD_OK) return rc;
    }
    return SESGD_OK;
  }
  if (ctx->payload_bf16 && (path != SESGD_PATH_TWOSHOT || ctx->push_tma))
    return fail(ctx, SESGD_ENOTSUP, "the bf16 payload needs the two-shot path with LSU pushes");
  if (ctx->protocol >= 1 && (path != SESGD_PATH_TWOSHOT || ctx->push_tma || ctx->payload_bf16))
    return fail(ctx, SESGD_ENOTSUP, "the value-carried protocol needs the fp32 two-shot path with LSU pushes");
  if (ctx->protocol == 2 && ctx->n_local != 1 && !sesgd::p2p_wsm_supported(ctx->n_local, ctx->m))
    return fail(ctx, SESGD_ENOTSUP, "protocol 2 (K4W-M) supports 2..8 workers per GPU");
  for (auto &b : ctx->buckets) b.stats.sync_calls++;
  return launch_oneshot(ctx, -1, lr, momentum, static_cast<cudaStream_t>(stream), twoshot, nvls);
}

int sesgd_sync_all_pair(sesgd_ctx *c0, sesgd_ctx *c1, float lr, float momentum, void *stream) {
  if (!c0 || !c1 || c0 == c1) return SESGD_EINVAL;
  for (sesgd_ctx *c : {c0, c1}) {
    int rc = check_latched(c);
    if (rc != SESGD_OK) return rc;
    if (!c->peers || !c->iter_set) return fail(c, SESGD_ESTATE, "attach peers and begin_iter first");
    if (c->n_ranks != 2 || c->protocol != 2 || resolve_path(c) != SESGD_PATH_TWOSHOT || c->m < 2 ||
        local_only_iteration(c) || c->device_iter)
      return fail(c, SESGD_ENOTSUP, "the pair harness runs K4W / K4W-M (protocol 2) on a two-rank loopback layout");
    for (auto &b : c->buckets)
      if (b.calls != c->buckets[0].calls) return fail(c, SESGD_ESTATE, "buckets must share one call history");
  }
  if (c0->rank != 0 || c1->rank != 1 || c0->ws[0] != c1->ws[0] || c0->ws[1] != c1->ws[1] ||
      c0->grid != c1->grid || c0->mode != c1->mode)
    return fail(c0, SESGD_EINVAL, "c0, c1 must be ranks 0 and 1 of the same two-rank layout");
  bool vec = true;
  for (sesgd_ctx *c : {c0, c1})
    for (auto &b : c->buckets) vec = vec && b.vec;
  P2PArgs a0{}, a1{};
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  for (auto &b : c0->buckets) b.stats.sync_calls++;
  for (auto &b : c1->buckets) b.stats.sync_calls++;
  int rc = launch_oneshot(c0, -1, lr, momentum, st, true, false, &a0);
  if (rc == SESGD_OK) rc = launch_oneshot(c1, -1, lr, momentum, st, true, false, &a1);
  if (rc != SESGD_OK) return rc;
  const cudaError_t e = c0->n_local == 1 ? sesgd::launch_p2p_ws_pair(a0, a1, c0->mode, vec, st)
                                         : sesgd::launch_p2p_wsm_pair(a0, a1, c0->mode, vec, st);
  if (e != cudaSuccess) return cuda_fail(c0, e, "launch the K4W pair");
  return SESGD_OK;
}

int sesgd_global_average(sesgd_ctx *ctx, int32_t bucket, const float *const *rows, int32_t nrows,
                         void *stream) {
  if (!ctx) return SESGD_EINVAL;
  int rc = check_latched(ctx);
  if (rc != SESGD_OK) return rc;
  if (!ctx->attached) return fail(ctx, SESGD_ESTATE, "sesgd_attach first");
  if (bucket < 0 || size_t(bucket) >= ctx->buckets.size() || !ctx->buckets[bucket].registered)
    return fail(ctx, SESGD_EINVAL, "bucket not registered");
  if (nrows != ctx->n) return fail(ctx, SESGD_EINVAL, "nrows must equal n (every worker's parameters)");
  sesgd_bucket &b = ctx->buckets[bucket];
  if (b.numel == 0) return SESGD_OK;
  sesgd::AverageArgs a{};
  bool vec = b.vec;
  for (int i = 0; i < ctx->n; ++i) {
    if (rows) {
      if (!rows[i]) return fail(ctx, SESGD_EINVAL, "null row pointer");
      a.rows[i] = rows[i];
      vec = vec && aligned16(rows[i]);
    } else {
      if (ctx->n_local != ctx->n)
        return fail(ctx, SESGD_EINVAL, "rows may be NULL only when every worker is local");
      a.rows[i] = b.hx[ctx->slot_of[i]];
    }
  }
  for (int s = 0; s < ctx->n_local; ++s) a.outs[s] = b.hx[s];
  a.nrows = ctx->n;
  a.nouts = ctx->n_local;
  a.numel = b.numel;
  cudaError_t e = sesgd::launch_average(a, vec, ctx->sm_count, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(ctx, e, "launch global average");
  b.stats.kernel_launches++;
  return SESGD_OK;
}

int sesgd_consensus(sesgd_ctx *ctx, int32_t bucket, const float *const *rows, int32_t nrows,
                    double *out_dev, void *stream) {
  if (!ctx || !out_dev) return SESGD_EINVAL;
  if (!ctx->attached) return fail(ctx, SESGD_ESTATE, "sesgd_attach first");
  if (bucket < 0 || size_t(bucket) >= ctx->buckets.size() || !ctx->buckets[bucket].registered)
    return fail(ctx, SESGD_EINVAL, "bucket not registered");
  if (nrows != ctx->n) return fail(ctx, SESGD_EINVAL, "nrows must equal n (every worker's parameters)");
  sesgd_bucket &b = ctx->buckets[bucket];
  if (b.numel == 0) return SESGD_OK;
  sesgd::AverageArgs a{};
  for (int i = 0; i < ctx->n; ++i) {
    if (rows) {
      if (!rows[i]) return fail(ctx, SESGD_EINVAL, "null row pointer");
      a.rows[i] = rows[i];
    } else {
      if (ctx->n_local != ctx->n)
        return fail(ctx, SESGD_EINVAL, "rows may be NULL only when every worker is local");
      a.rows[i] = b.hx[ctx->slot_of[i]];
    }
  }
  a.nrows = ctx->n;
  a.numel = b.numel;
  cudaError_t e = sesgd::launch_consensus(a, out_dev, ctx->sm_count, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(ctx, e, "launch consensus");
  return SESGD_OK;
}

int sesgd_sync_step_host(sesgd_ctx *ctx, int32_t bucket, float lr, float momentum,
                         const float *const *g_host, float *const *x_host_out, void *stream) {
  if (!ctx) return SESGD_EINVAL;
  if (!g_host || !x_host_out) return fail(ctx, SESGD_EINVAL, "null host buffer table");
  if (bucket < 0 || size_t(bucket) >= ctx->buckets.size() || !ctx->buckets[bucket].registered)
    return fail(ctx, SESGD_EINVAL, "bucket not registered");
  sesgd_bucket &b = ctx->buckets[bucket];
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t bytes = size_t(b.numel) * sizeof(float);
  for (int s = 0; s < ctx->n_local; ++s) {
    if (!g_host[s] || !x_host_out[s]) return fail(ctx, SESGD_EINVAL, "null host buffer");
    cudaError_t e = cudaMemcpyAsync(const_cast<float *>(b.hg[s]), g_host[s], bytes,
                                    cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "H2D gradient copy");
  }
  int rc = sesgd_sync_step(ctx, bucket, lr, momentum, stream);
  if (rc != SESGD_OK) return rc;
  for (int s = 0; s < ctx->n_local; ++s) {
    cudaError_t e = cudaMemcpyAsync(x_host_out[s], b.hx[s], bytes, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "D2H parameter copy");
  }
  return SESGD_OK;
}

int sesgd_sync_all_host(sesgd_ctx *ctx, float lr, float momentum, const float *const *g_host,
                        float *const *x_host_out, void *stream) {
  if (!ctx) return SESGD_EINVAL;
  if (!g_host || !x_host_out) return fail(ctx, SESGD_EINVAL, "null host buffer table");
  if (!ctx->attached || !ctx->iter_set) return fail(ctx, SESGD_ESTATE, "attach and begin_iter first");
  const size_t nb = ctx->buckets.size();
  if (nb == 0) return fail(ctx, SESGD_ESTATE, "no bucket registered");
  const int r = ctx->n_local;
  for (size_t i = 0; i < nb * size_t(r); ++i)
    if (!g_host[i] || !x_host_out[i]) return fail(ctx, SESGD_EINVAL, "null host buffer");
  cudaError_t e = cudaSuccess;
  if (!ctx->copy_in) {
    e = cudaStreamCreateWithFlags(&ctx->copy_in, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->copy_out, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_start, cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "copy streams");
  }
  for (auto *v : {&ctx->ev_in, &ctx->ev_k, &ctx->ev_out})
    while (v->size() < nb) {
      cudaEvent_t ev;
      e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
      if (e != cudaSuccess) return cuda_fail(ctx, e, "copy events");
      v->push_back(ev);
    }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // H2D of every bucket on copy_in, after the work already queued on `stream`
  e = cudaEventRecord(ctx->ev_start, st);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(ctx->copy_in, ctx->ev_start, 0);
  for (size_t b = 0; b < nb && e == cudaSuccess; ++b) {
    const sesgd_bucket &bk = ctx->buckets[b];
    for (int s = 0; s < r && e == cudaSuccess; ++s)
      e = cudaMemcpyAsync(const_cast<float *>(bk.hg[s]), g_host[b * r + s], size_t(bk.numel) * 4,
                          cudaMemcpyHostToDevice, ctx->copy_in);
    if (e == cudaSuccess) e = cudaEventRecord(ctx->ev_in[b], ctx->copy_in);
  }
  if (e != cudaSuccess) return cuda_fail(ctx, e, "H2D gradient copies");
  // bucket b's kernel as soon as its gradients landed; its D2H on copy_out right after it
  for (size_t b = 0; b < nb; ++b) {
    e = cudaStreamWaitEvent(st, ctx->ev_in[b], 0);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "wait H2D");
    const int rc = sesgd_sync_step(ctx, int32_t(b), lr, momentum, stream);
    if (rc != SESGD_OK) return rc;
    e = cudaEventRecord(ctx->ev_k[b], st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(ctx->copy_out, ctx->ev_k[b], 0);
    const sesgd_bucket &bk = ctx->buckets[b];
    for (int s = 0; s < r && e == cudaSuccess; ++s)
      e = cudaMemcpyAsync(x_host_out[b * r + s], bk.hx[s], size_t(bk.numel) * 4, cudaMemcpyDeviceToHost,
                          ctx->copy_out);
    if (e == cudaSuccess) e = cudaEventRecord(ctx->ev_out[b], ctx->copy_out);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "D2H parameter copies");
  }
  e = cudaStreamWaitEvent(st, ctx->ev_out[nb - 1], 0);  // copy_out is in order: every D2H done
  if (e != cudaSuccess) return cuda_fail(ctx, e, "wait D2H");
  return SESGD_OK;
}

int sesgd_poll(sesgd_ctx *ctx) {
  if (!ctx) return SESGD_EINVAL;
  return check_latched(ctx);
}

int sesgd_get_stats(const sesgd_ctx *ctx, int32_t bucket, sesgd_stats *out) {
  if (!ctx || !out || bucket < 0 || size_t(bucket) >= ctx->buckets.size()) return SESGD_EINVAL;
  *out = ctx->buckets[bucket].stats;
  if (ctx->d_counters) {
    unsigned long long c[sesgd::kNumCounters] = {};
    if (cudaMemcpy(c, ctx->d_counters, sizeof c, cudaMemcpyDeviceToHost) != cudaSuccess)
      return fail(const_cast<sesgd_ctx *>(ctx), SESGD_ECUDA, "reading the device counters");
    out->dev_flag_stores = int64_t(c[sesgd::kCntFlagStores]);
    out->dev_flag_spins = int64_t(c[sesgd::kCntFlagSpins]);
    out->dev_value_spins = int64_t(c[sesgd::kCntValueSpins]);
    out->dev_launches = int64_t(c[sesgd::kCntLaunches]);
    out->hop_ns = ctx->hop_iters > 0 ? double(c[sesgd::kCntHopNs]) / ctx->hop_iters / 2.0 : 0.0;
  }
  out->last_launch_us = 0.0;
  if (ctx->ev_l_valid && cudaEventQuery(ctx->ev_l1) == cudaSuccess) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, ctx->ev_l0, ctx->ev_l1) == cudaSuccess) out->last_launch_us = 1e3 * ms;
  }
  cudaGetLastError();  // a not-ready query is not an error of this call
  return SESGD_OK;
}

int sesgd_measure_hop(sesgd_ctx *ctx, int32_t peer_rank, int32_t iters, int32_t initiator, void *stream) {
  if (!ctx) return SESGD_EINVAL;
  if (!ctx->peers) return fail(ctx, SESGD_ESTATE, "sesgd_attach_peers first");
  if (peer_rank < 0 || peer_rank >= ctx->n_ranks || peer_rank == ctx->rank || iters < 1)
    return fail(ctx, SESGD_EINVAL, "peer_rank must be another attached rank, iters >= 1");
  // flag words in the workspace header, [128 + 8 * rank], one per peer rank, monotonic epochs
  auto flag = [&](int owner, int other) {
    return reinterpret_cast<uint64_t *>(ctx->ws[owner] + 128) + other;
  };
  const cudaError_t e = sesgd::launch_pingpong(
      flag(ctx->rank, peer_rank), flag(peer_rank, ctx->rank), iters, initiator ? 1 : 0,
      ctx->hop_base[peer_rank], reinterpret_cast<uint64_t *>(ctx->d_counters + sesgd::kCntHopNs),
      static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(ctx, e, "launch ping-pong");
  ctx->hop_base[peer_rank] += 2 * uint64_t(iters) + 2;
  ctx->hop_iters = iters;
  return SESGD_OK;
}

int sesgd_profile_read(sesgd_ctx *ctx, uint64_t *out, int64_t words, int32_t *comm_ctas_out) {
  if (!ctx || !out || words < 0) return SESGD_EINVAL;
  if (!ctx->d_prof) return fail(ctx, SESGD_ESTATE, "no profile recorded (SESGD_OPT_PROFILE, multi-GPU path)");
  const int64_t n = std::min<int64_t>(words, int64_t(ctx->grid) * 8);
  cudaError_t e = cudaMemcpy(out, ctx->d_prof, size_t(n) * 8, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemset(ctx->d_prof, 0, size_t(ctx->grid) * 64);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "profile read");
  if (comm_ctas_out) *comm_ctas_out = ctx->p2p_variant;
  return SESGD_OK;
}

int sesgd_launch_grid(const sesgd_ctx *ctx, int32_t *ctas_out) {
  if (!ctx || !ctas_out) return SESGD_EINVAL;
  *ctas_out = ctx->peers ? ctx->grid : ctx->sm_count;
  return SESGD_OK;
}

}  // extern "C"
