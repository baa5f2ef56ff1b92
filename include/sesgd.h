/*
 * sesgd.h -- C ABI of libsesgd.so, the B200-native hot path of Shuffle-Exchange
 * SGD (SESGD, arXiv 2007.00433).
 *
 * Citations: P:n = the paper's PAPER.md line n, S:n = SPEC.md line n; R1..R21 are
 * the readings of the paper listed in DESIGN.md ("Readings").
 *
 * What one iteration computes (Algorithm 1; Eq. 6):
 *   for every worker i (R8: local momentum, never communicated, v <- mu v + g):
 *     v_i   <- mu (x) v_i (+) g_i
 *     xh_i  <- x_i (-) lr (x) v_i                               (Alg.1 lines 3-8)
 *   G_t = shuffle-exchange partition of the n workers into n/m groups  (lines 9-10)
 *   x_i  <- (xh_{a0} (+) xh_{a1} (+) ... (+) xh_{a(m-1)}) (/) m  (line 11, R7, R10)
 * with (x)(+)(-)(/) single binary32 round-to-nearest operations (no FMA
 * contraction), a0 < a1 < ... the members of i's group.  SESGD_MODE_GRAD_AVG is
 * the Eq. 5 variant: gbar = fold(g)/m ; v <- mu v + gbar ; x <- x - lr v.
 *
 * Memory: every parameter / momentum / gradient buffer is CALLER-OWNED device
 * memory (fp32, contiguous); the library never frees it.  Multi-GPU peer
 * workspaces are caller-owned peer-mapped device memory (e.g. from
 * torch.distributed._symmetric_memory).  The library owns only the context and
 * small device tables it allocates itself (freed by sesgd_destroy).
 *
 * Threading: a context is not thread-safe; use one per process (per device).
 * Errors: every int-returning call returns SESGD_OK (0) or a negative code;
 * sesgd_last_error(ctx) gives a human-readable reason for the last failure.
 */
#ifndef SESGD_H
#define SESGD_H

#include <stdint.h>

#if defined(__GNUC__)
#define SESGD_API __attribute__((visibility("default")))
#else
#define SESGD_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ---- */
#define SESGD_OK 0
#define SESGD_EINVAL (-1)   /* bad argument (range, NULL, size mismatch) */
#define SESGD_ENOTDIV (-2)  /* group_size does not divide n (R13) */
#define SESGD_ESTATE (-3)   /* call out of order / layout mismatch across ranks */
#define SESGD_ECUDA (-4)    /* CUDA runtime error; see sesgd_last_error */
#define SESGD_ETIMEOUT (-5) /* a group peer did not signal within the timeout */
#define SESGD_ENOMEM (-6)   /* host or device allocation failed */
#define SESGD_ENOTSUP (-7)  /* configuration not supported by this build */

/* ---- compile-time limits ---- */
#define SESGD_MAX_WORKERS 64 /* n */
#define SESGD_MAX_RANKS 8    /* GPUs in one job (one NVLink/NVSwitch domain) */

/* ---- modes (R9) ---- */
#define SESGD_MODE_PARAM_AVG 0 /* Eq. 6: average locally-stepped parameters (default) */
#define SESGD_MODE_GRAD_AVG 1  /* Eq. 5 variant: average gradients, then local update */

/* ---- data paths for the intra-group exchange ---- */
#define SESGD_PATH_AUTO 0     /* resident if all workers are local; else two-shot (P2P variant 0),
                                 one-shot with COMM CTAs (variant >= 1) */
#define SESGD_PATH_RESIDENT 1 /* all n workers on this GPU (1-GPU "k resident replicas") */
#define SESGD_PATH_ONESHOT 2  /* NVLink P2P: one handshake round, members push to each other */
#define SESGD_PATH_RING 3     /* NVLink P2P, the paper's Ring-AllReduce inside each group: 2(m-1)
                                 handshake steps (Eq. 2/3); one worker per GPU; for the
                                 handshake / injected-latency comparison (config 4) */
#define SESGD_PATH_TWOSHOT 4  /* NVLink P2P, two handshake rounds: every member owns a slice of
                                 each chunk; reduce-scatter pushes to remote slice owners, all-gather
                                 pushes of the slice means (co-resident members are read / updated
                                 in place); a remote member pair exchanges 2/m of a bucket instead of
                                 one-shot's full copy; needs P2P variant 0 (else SESGD_ENOTSUP) */
#define SESGD_PATH_NVLS 5     /* NVLink SHARP, for group_size = n (Ring-SGD's single group) with one
                                 worker per GPU: chunk g's owner (member g mod n) reduces every GPU's
                                 stage of it inside the NVSwitch (multimem.ld_reduce) and multicasts the mean
                                 (multimem.st); needs sesgd_attach_multicast.  The switch's
                                 summation order is unspecified: parity within the north-star
                                 tolerance, bit-exact only for n = 2 (a + b = b + a) */

/* ---- options for sesgd_set_option ---- */
#define SESGD_OPT_MODE 1       /* SESGD_MODE_*                                   (default 0) */
#define SESGD_OPT_PATH 2       /* SESGD_PATH_*                                   (default 0) */
#define SESGD_OPT_TIMEOUT_MS 3 /* flag-wait timeout before SESGD_ETIMEOUT        (default 20000) */
#define SESGD_OPT_GRID 4       /* CTAs per launch, 0 = auto (SM count x occupancy) */
#define SESGD_OPT_HOP_DELAY_NS 5 /* injected delay before every flag store (latency sweep) */
#define SESGD_OPT_P2P_VARIANT 6  /* one-shot kernel shape: 0 (default) = every CTA pushes its own
                                    x_hat to remote members from registers; 1..148 = that many
                                    CTAs dedicated to NVLink pushes out of an L2 stage while the
                                    others stream HBM; fixed once peers attach (sets the layout) */
#define SESGD_OPT_DISCARD 7      /* 1 (default): drop consumed receive lines from L2 without
                                    write-back (discard.global.L2); 0: leave them to be evicted */
#define SESGD_OPT_PROFILE 8      /* 1: the one-shot kernel accumulates per-CTA phase times
                                    (%globaltimer ns) readable with sesgd_profile_read; 0 (default) */
#define SESGD_OPT_COMM_BATCH 9   /* chunks (16 KiB each) a COMM CTA pushes per flag release:
                                    amortises the system-scope release (default 16); fixed once
                                    peers attach */
#define SESGD_OPT_FOLD_LAG 10    /* chunk steps a COMPUTE CTA stages ahead of its fold (1..64,
                                    default 4): covers the push + release latency; the two-shot
                                    path uses ceil(lag / 2) per round (stage -> reduce -> finish) */
#define SESGD_OPT_RESIDENT_UNROLL 11 /* 1-GPU kernel, group size 2: independent items per
                                    thread per trip (1, 2, 4, 8; 0 = default 1) */
#define SESGD_OPT_PUSH_TMA 12    /* two-shot kernel: 1 = NVLink pushes assembled in shared memory
                                    and sent with cp.async.bulk (TMA) by one thread per CTA;
                                    0 (default) = 128-bit stores from every thread */
#define SESGD_OPT_RELEASE_DELAY 13 /* two-shot kernel: chunk steps between a push and the
                                    system-scope release of its flag (1..8, default 1; TMA >= 2) */
#define SESGD_OPT_RELEASE_EVERY 14 /* two-shot and DIRECT one-shot kernels: chunk steps between
                                    flag-release batches (1..16, default 3); each batch is ONE
                                    system-scope fence (~8 us under load) followed by relaxed
                                    flag stores; the lag is raised to cover it */
#define SESGD_OPT_LOCAL_PERIOD 15  /* Local-SESGD (paper Sec. 4.1, period 2 at
                                    P:328): the group exchange of iteration t (sesgd_begin_iter)
                                    fires only when (t + 1) mod H == 0; other iterations run the
                                    local step alone (x <- x_hat).  H >= 1, default 1 = SESGD;
                                    group_size = n gives Local-SGD */
#define SESGD_OPT_SCHEDULE 16      /* 0 (default): seeded uniform random partition (R1);
                                    1: Stone's shuffle-exchange network -- iteration t exchanges
                                    index dimensions (t p + q) mod d, q < p, for n = 2^d,
                                    group_size = 2^p (else SESGD_EINVAL); n = 4, m = 2 gives the
                                    paper's example {0,1},{2,3} -> {0,2},{1,3}; set it
                                    identically on every rank, before sesgd_begin_iter */
#define SESGD_OPT_RELEASE_STAGGER 17 /* 1 (default): CTA i takes its flag-release steps at
                                    (k + i) mod R = 0, so the CTAs sharing an SM fence in turn;
                                    0: all at k mod R = 0 */
#define SESGD_OPT_PAYLOAD_BF16 18  /* 1: the two-shot reduce-scatter carries bf16 (round to nearest
                                    even) instead of fp32 -- every member's contribution, its own
                                    included, is rounded before the fold; the fold and the mean stay
                                    fp32 (R21; a lossy variant, compare with the oracle's
                                    payload_bf16 mode; all-local groups of K4 round too); one
                                    or several workers per GPU, LSU pushes.  The resident K6 path
                                    (every worker on one GPU) returns SESGD_ENOTSUP with it set */
#define SESGD_OPT_SM_BUDGET 19     /* SMs this context sizes its grids for (0, default: every SM of
                                    the device).  Loopback ("virtual ranks"): R contexts on ONE GPU,
                                    each with its own workspace and sesgd_attach_peers given the R
                                    local workspace pointers, each with budget SMs / R, so that all
                                    R persistent grids are co-resident and the NVLink-path kernels
                                    (K3, K4, K5) run against each other through local memory.  Set
                                    before sesgd_workspace_bytes (the grid fixes the layout) */
#define SESGD_OPT_PROTOCOL 21      /* two-shot handshake (set before sesgd_workspace_bytes, identical
                                    on every rank): -1 (default, auto) = 2 with one worker per
                                    GPU (K4W) or with 2..8 (K4W-M), 1 with more than 8, where
                                    supported (the two-shot path with fp32 LSU pushes), else 0.
                                    0 = epoch flags released with a system-scope fence per batch.
                                    1 = value-carried validity: every receive-slot float holds a
                                    sentinel NaN (0xFFFFFFFF) until the peer's value lands; the
                                    receiver polls the values themselves and re-arms them (no
                                    sender fence, no flag).  A payload equal to the sentinel
                                    travels as the canonical NaN 0x7FFFFFFF.
                                    2 = 1 in K4W / K4W-M, the warp-specialised kernels (one CTA
                                    per SM; K4W-M: 2..8 workers per GPU).  1 and 2: fp32 LSU pushes only (else
                                    SESGD_ENOTSUP) */
#define SESGD_OPT_COOPERATIVE 22   /* 1: the persistent multi-GPU grids (K4, K4W, K3, K5) are launched
                                    cooperatively -- the runtime rejects a grid that cannot be
                                    co-resident (SESGD_ECUDA) and starts it only when all its CTAs
                                    fit at once.  0 (default): plain launch; safe because a K4 /
                                    K4W / K3-direct / K5 CTA waits only on data or flags of the
                                    SAME CTA index on peer GPUs (never on another CTA of its own
                                    grid), so a CTA that is not yet resident delays, never
                                    deadlocks, its peers.  The SM-specialised K3 (P2P variant
                                    >= 1, COMM and COMPUTE CTAs wait on each other) is always
                                    launched cooperatively.  (A cooperative launch cannot start
                                    while the previous kernel drains: measured +10..30 us per
                                    step, profiles/r02_proto_*.json) */
#define SESGD_OPT_DEVICE_ITER 23   /* 1: the iteration state lives in DEVICE memory -- the iteration t,
                                    its groups (evaluated on the GPU from the shared seed)
                                    and the call history of the exchange kernels -- so that
                                    sesgd_begin_iter_device + the sync calls of one iteration can be
                                    captured ONCE into a CUDA graph and the graph replayed for every
                                    iteration.  Setting it uploads the host's state (synchronous);
                                    setting 0 synchronises the device and copies the state back.
                                    Needs sesgd_attach and every bucket registered (none after);
                                    supported paths: resident (K6), two-shot with protocol 2
                                    (K4W, K4W-M) and ring (K5); others return SESGD_ENOTSUP from
                                    the sync call.  Not with SESGD_OPT_LOCAL_PERIOD > 1.  The
                                    host-side counters of sesgd_get_stats count enqueued calls,
                                    not graph replays (the dev_* counters count launches) */
#define SESGD_OPT_WS_SPLIT 24       /* K4W-M (protocol 2, several workers per GPU): warps of the
                                    streaming role S out of 24 (8 -- default, measured best --, 12 or 16); the
                                    fold (R) and gather (F) roles share the rest equally */
#define SESGD_OPT_WSM_HYBRID 25     /* K4W-M with host iterations: 1 = the groups whose members all
                                    live on this GPU are updated by the 1-GPU kernel K6 first,
                                    then K4W-M streams only the workers whose group spans GPUs;
                                    0 (default) = K4W-M does both.  Same bits either way.
                                    Measured slower (cfg 2, 2 GPUs: 0.71 vs 0.66 ms; the two
                                    kernels serialise and ranks with more all-local groups start
                                    the exchange later), kept for the record.  Device-resident
                                    iterations always use 0 */
#define SESGD_OPT_EXPERIMENT 20    /* MEASUREMENT ONLY -- results are wrong when set: bit 0 drops
                                    the system-scope fence before the two-shot flag releases,
                                    bit 1 sends the two-shot pushes to this rank's own receive
                                    slots instead of the peers' (no NVLink payload).  Bounds what
                                    the flag protocol and the NVLink traffic cost */

/* Latency model, Eq. 2 and Eq. 3 exact forms (R16). */
typedef struct sesgd_cost {
  double ring_handshakes;  /* 2(n-1)                       per tensor, Ring-AllReduce over n */
  double sesgd_handshakes; /* 2(m-1)                       per tensor, ring inside a group  */
  double ring_s;           /* 2(n-1) (G/(n nu) + tau)       seconds                          */
  double sesgd_s;          /* 2(m-1) (G/(m nu) + tau)       seconds                          */
  double ratio;            /* ring_s / sesgd_s (1 if both 0, +inf if only sesgd_s is 0)      */
} sesgd_cost;

/* Counters.  The first six are per bucket and host-side (exact: the schedule is deterministic);
 * the dev_* ones are counted ON THE DEVICE by the multi-GPU kernels of this context (all buckets,
 * cumulative since sesgd_attach; a snapshot -- synchronise the stream first for exact totals);
 * last_launch_us is the device time (CUDA events recorded by the library) of the context's most
 * recent completed sync launch, hop_ns the one-way handshake latency last measured by
 * sesgd_measure_hop (0 if never). */
typedef struct sesgd_stats {
  int64_t sync_calls;        /* sesgd_sync_step calls on this bucket                        */
  int64_t kernel_launches;   /* kernels this library launched for the bucket                */
  int64_t handshake_rounds;  /* flag rounds per call on the critical path (0 resident, 1 one-shot) */
  int64_t flag_messages;     /* cross-GPU flag stores issued by this process, cumulative    */
  int64_t payload_bytes_in;  /* bytes this process pulled from other GPUs, cumulative       */
  int64_t hbm_algo_bytes;    /* algorithmic HBM bytes (20 B per worker-element), cumulative */
  int64_t dev_flag_stores;   /* device: cross-GPU handshake flag stores (K3, K4 protocol 0, K5) */
  int64_t dev_flag_spins;    /* device: flag waits that had to spin (peer not ready yet)    */
  int64_t dev_value_spins;   /* device: value-carried polls that found a sentinel (protocols 1, 2) */
  int64_t dev_launches;      /* device: multi-GPU kernel launches that started               */
  double last_launch_us;     /* device time of the most recent completed sync launch (events) */
  double hop_ns;             /* one-way flag hop, sesgd_measure_hop (K7 ping-pong)           */
} sesgd_stats;

typedef struct sesgd_ctx sesgd_ctx;

/* Create a context for n workers in groups of m = group_size (k = n/m groups).
 * Host only: no GPU work, no communication.
 * Errors: SESGD_EINVAL (n < 1, n > SESGD_MAX_WORKERS, group_size < 1, group_size > n,
 *         out == NULL); SESGD_ENOTDIV (n % group_size != 0); SESGD_ENOMEM. */
SESGD_API int sesgd_init(int32_t n, int32_t group_size, uint64_t seed, sesgd_ctx **out);

/* Free the context and the library-owned device tables. NULL is a no-op. */
SESGD_API void sesgd_destroy(sesgd_ctx *ctx);

/* The shuffle-exchange partition of iteration `iter` (A1; Alg.1 lines 1, 9-10;
 * readings R1-R6).  Pure function of (seed, iter, n, m): random access in iter.
 * perm_out[n] (required): canonical order -- group j is perm_out[j*m .. j*m+m-1],
 *   members ascending, groups ordered by smallest member.
 * group_of_out[n] (may be NULL): group index of each worker in that order.
 * Caller owns both buffers.  Errors: SESGD_EINVAL (ctx/perm_out NULL, iter < 0). */
SESGD_API int sesgd_groups(const sesgd_ctx *ctx, int64_t iter, int32_t *perm_out, int32_t *group_of_out);

/* Latency-model query (A6/A7).  Pure, host only.
 * bytes = G (message bytes per tensor), nu_Bps = bandwidth (B/s), tau_s = per-hop latency.
 * Errors: SESGD_EINVAL (n < 1, group_size < 1 or > n, nu_Bps <= 0, tau_s < 0, bytes < 0,
 *         out NULL); SESGD_ENOTDIV (n % group_size != 0). */
SESGD_API int sesgd_latency_model(int32_t n, int32_t group_size, double bytes, double nu_Bps, double tau_s,
                        sesgd_cost *out);

/* Set an option (SESGD_OPT_*).  Errors: SESGD_EINVAL (unknown option / bad value). */
SESGD_API int sesgd_set_option(sesgd_ctx *ctx, int32_t option, int64_t value);

/* Bind this process to CUDA `device` and the global worker ids it hosts
 * (local_workers[n_local], distinct, in [0, n)).  1 GPU: n_local = n (all resident).
 * Must precede sesgd_register_bucket.  Errors: SESGD_EINVAL (duplicates, out of range,
 * n_local < 1), SESGD_ESTATE (already attached), SESGD_ECUDA. */
SESGD_API int sesgd_attach(sesgd_ctx *ctx, int32_t device, int32_t n_local, const int32_t *local_workers);

/* Register bucket `bucket` (0 <= bucket < 4096, ids dense from 0) of `numel` fp32 elements.
 * x[n_local], v[n_local], g[n_local]: device pointers of each local worker (in the order given
 * to sesgd_attach), each to numel contiguous floats; 16-byte aligned pointers take the
 * 128-bit vector path, others a scalar path.  Every worker must register the same
 * (bucket, numel) list (checked at sesgd_attach_peers on multi-GPU).
 * Re-registering an id replaces its pointers (numel must not change after attach_peers).
 * Errors: SESGD_EINVAL (NULL pointers, numel < 0, bad id), SESGD_ESTATE (not attached),
 *         SESGD_ECUDA / SESGD_ENOMEM (device table allocation). */
SESGD_API int sesgd_register_bucket(sesgd_ctx *ctx, int32_t bucket, int64_t numel, float *const *x,
                          float *const *v, const float *const *g);

/* Multi-GPU only.  Bytes of peer-visible workspace each rank must provide for the
 * registered buckets (stage double buffer + flag words).  Errors: SESGD_ESTATE. */
SESGD_API int sesgd_workspace_bytes(const sesgd_ctx *ctx, int64_t *bytes_out);

/* Multi-GPU only.  Zero this rank's workspace `local_ws` (device pointer of
 * sesgd_workspace_bytes bytes) and write its layout header.  Synchronous.
 * Call on every rank, then barrier, then sesgd_attach_peers. */
SESGD_API int sesgd_workspace_prepare(sesgd_ctx *ctx, void *local_ws);

/* Multi-GPU only.  rank_ws[n_ranks]: every rank's workspace, mapped into this process
 * (rank_ws[rank] == local_ws).  worker_rank[n]: the rank hosting each worker.  Reads the
 * peers' headers (P2P) and returns SESGD_ESTATE if any rank registered different buckets.
 * Errors: SESGD_EINVAL, SESGD_ESTATE, SESGD_ECUDA. */
SESGD_API int sesgd_attach_peers(sesgd_ctx *ctx, int32_t n_ranks, int32_t rank, void *const *rank_ws,
                       const int32_t *worker_rank);

/* Set the current iteration t (any t >= 0: random access / resume).  Computes the
 * schedule of t (and of t-2, for the stage-reuse guard) on the host.
 * Errors: SESGD_EINVAL (iter < 0), SESGD_ESTATE (not attached, or SESGD_OPT_DEVICE_ITER on:
 * the iteration then lives on the device, sesgd_begin_iter_device). */
SESGD_API int sesgd_begin_iter(sesgd_ctx *ctx, int64_t iter);

/* The hot path: one SESGD sync+update of bucket `bucket` at the current iteration for all
 * local workers.  ASYNCHRONOUS: validates, enqueues the fused kernel on `stream`
 * (a cudaStream_t; NULL = legacy default stream) and returns.  On multi-GPU every rank must
 * issue the same (iteration, bucket) sequence.  Device-side failures (peer timeout) are
 * latched and returned by the next call or by sesgd_poll as SESGD_ETIMEOUT.
 * Errors: SESGD_EINVAL (unregistered bucket, lr/momentum not finite), SESGD_ESTATE
 *         (begin_iter not called, peers not attached on multi-GPU), SESGD_ECUDA, SESGD_ETIMEOUT. */
SESGD_API int sesgd_sync_step(sesgd_ctx *ctx, int32_t bucket, float lr, float momentum, void *stream);

/* sesgd_sync_step for EVERY registered bucket of the current iteration.  On the multi-GPU
 * one-shot path, when all buckets share their call history (always the case if they are only
 * ever synced together), this is ONE fused launch over all buckets' chunks: the NVLink / HBM
 * pipeline fills and drains once per iteration instead of once per bucket.  Otherwise (and on
 * the resident path) it enqueues one launch per bucket in id order.  Asynchronous on `stream`.
 * Errors: as sesgd_sync_step; SESGD_ESTATE if no bucket is registered. */
SESGD_API int sesgd_sync_all(sesgd_ctx *ctx, float lr, float momentum, void *stream);

/* End-to-end variant through HOST buffers: for each local worker, copies g_host[w] (numel
 * floats, pinned for overlap) to the registered device gradient, runs sesgd_sync_step, and
 * copies the updated device parameters back into x_host_out[w].  Asynchronous on `stream`
 * like sesgd_sync_step; host buffers must stay valid until the stream is synchronised. */
SESGD_API int sesgd_sync_step_host(sesgd_ctx *ctx, int32_t bucket, float lr, float momentum,
                         const float *const *g_host, float *const *x_host_out, void *stream);

/* Every bucket through host buffers, pipelined: g_host[b * n_local + s] (bucket b, local slot s;
 * numel_b floats each, pinned) -> device gradients on an internal copy stream, bucket b's
 * sesgd_sync_step on `stream` as soon as its gradients landed, its parameters -> x_host_out[b *
 * n_local + s] on a second internal copy stream, so H2D, kernels and D2H of different buckets
 * overlap (PCIe is full duplex).  When `stream` completes, every copy has completed.  The
 * device gradients are overwritten only after the work already queued on `stream`.
 * Errors: as sesgd_sync_step, SESGD_EINVAL (null buffer). */
SESGD_API int sesgd_sync_all_host(sesgd_ctx *ctx, float lr, float momentum, const float *const *g_host,
                                  float *const *x_host_out, void *stream);

/* Algorithm 1's last line, xbar <- Ring-AllReduce(x_i; Global), for bucket `bucket`:
 * every LOCAL worker's parameters become (rows[0] (+) rows[1] (+) ... (+) rows[n-1]) (/) n,
 * a left fold in ascending worker id (R7, R10).  rows: host array of n device pointers to the n
 * workers' parameters of this bucket (numel fp32 each, caller-owned; e.g. an all-gather of every
 * rank's x), or NULL when all n workers are local (their registered x is used, in place).
 * Momentum buffers are not touched.  Asynchronous on `stream` (K8).  Errors: SESGD_EINVAL (nrows
 * != n, null row, NULL rows with remote workers), SESGD_ESTATE, SESGD_ECUDA. */
SESGD_API int sesgd_global_average(sesgd_ctx *ctx, int32_t bucket, const float *const *rows,
                                   int32_t nrows, void *stream);

/* Consistency of the workers' parameters (the question of Fig. 7b), bucket
 * `bucket`: with xbar the binary64 mean of the n workers' parameters,
 *   out_dev[0] += sum_i sum_e (x_i[e] - xbar[e])^2      (n x the consensus distance)
 *   out_dev[1]  = max(out_dev[1], max_i,e |x_i[e] - xbar[e]|)
 * out_dev: 2 doubles of caller-owned device memory (zero them before the first bucket; calls
 * accumulate across buckets).  rows as in sesgd_global_average (NULL: all workers local).
 * Asynchronous on `stream` (K9, binary64 accumulation).  Errors: as sesgd_global_average. */
SESGD_API int sesgd_consensus(sesgd_ctx *ctx, int32_t bucket, const float *const *rows, int32_t nrows,
                              double *out_dev, void *stream);

/* Pair-split statistics on the device (the appendix's Monte Carlo: Pr[i, j in different
 * groups] = n (k - 1) / (k (n - 1))): for every iteration t in [t0, t0 + T) the context's
 * schedule (seed, n, group_size, SESGD_OPT_SCHEDULE) is evaluated on the GPU (K10, one thread per
 * t) and counts_dev[min(i,j) * n + max(i,j)] is incremented when workers i and j share a group.
 * counts_dev: n*n unsigned 64-bit device counters, caller-owned, accumulated (zero them first).
 * Needs sesgd_attach (device).  Errors: SESGD_EINVAL, SESGD_ESTATE, SESGD_ECUDA. */
SESGD_API int sesgd_pair_counts(sesgd_ctx *ctx, int64_t t0, int64_t T, unsigned long long *counts_dev,
                                void *stream);

/* NVLS: the multicast mapping of the symmetric workspaces (e.g. torch symmetric memory's
 * multicast_ptr of the same allocation whose per-rank pointers went to sesgd_attach_peers), for
 * SESGD_PATH_NVLS.  Errors: SESGD_EINVAL (NULL), SESGD_ESTATE (peers not attached). */
SESGD_API int sesgd_attach_multicast(sesgd_ctx *ctx, void *mc_ws);

/* Weight decay folded into every update (the paper trains with 5e-4 / 1e-4; R20): the
 * gradient term of the momentum step becomes d = g (+) wd (x) x, as torch.optim.SGD's
 * weight_decay -- PARAM: v <- mu v + (g + wd x) before the local step; GRAD: v <- mu v +
 * (gbar + wd x) with the worker's own x after the group mean.  Default 0 (bit-identical to no
 * decay).  Applies to the following sesgd_sync_step / sync_all calls.  Errors: SESGD_EINVAL
 * (negative or not finite). */
SESGD_API int sesgd_set_weight_decay(sesgd_ctx *ctx, float weight_decay);

/* Non-blocking check of the latched device error word: SESGD_OK or SESGD_ETIMEOUT. */
SESGD_API int sesgd_poll(sesgd_ctx *ctx);

/* Counters of bucket `bucket`.  Errors: SESGD_EINVAL. */
SESGD_API int sesgd_get_stats(const sesgd_ctx *ctx, int32_t bucket, sesgd_stats *out);

/* Measurement harness, not part of an iteration's normal API: sesgd_sync_all for BOTH ranks of a
 * two-rank loopback layout (contexts c0 = rank 0 and c1 = rank 1 on the same GPU, attached to
 * each other, protocol 2: one worker each = K4W, or 2..8 workers each = K4W-M) as ONE kernel
 * launch whose first half of CTAs runs rank 0 and second half rank 1 -- same kernel body, same bits as two sesgd_sync_all calls
 * -- so a profiler that serialises launches (ncu, which would deadlock two concurrent grids that
 * wait on each other) can capture the whole exchange.  Both contexts' call histories advance.
 * Errors: SESGD_EINVAL, SESGD_ESTATE, SESGD_ENOTSUP (not that layout), SESGD_ECUDA. */
SESGD_API int sesgd_sync_all_pair(sesgd_ctx *c0, sesgd_ctx *c1, float lr, float momentum, void *stream);

/* Per-hop handshake latency t_tau (Eq. 2) between this rank and `peer_rank` through the
 * two ranks' workspaces (K7 flag ping-pong, one thread, system-scope release / acquire): both ranks
 * call it concurrently with the same `iters`, exactly one with initiator = 1.  Enqueued on
 * `stream`; the result (round trip / 2) appears in sesgd_stats.hop_ns once the stream completes.
 * Errors: SESGD_EINVAL (peer_rank out of range or == rank, iters < 1), SESGD_ESTATE (peers not
 * attached), SESGD_ECUDA. */
SESGD_API int sesgd_measure_hop(sesgd_ctx *ctx, int32_t peer_rank, int32_t iters, int32_t initiator,
                                void *stream);

/* Device-side begin_iter (SESGD_OPT_DEVICE_ITER = 1): enqueues on `stream` one single-thread
 * kernel that sets the device iteration to `iter` (>= 0) or, with iter = SESGD_ITER_NEXT (-1), to
 * the device's current iteration + 1 (0 if none was set), and evaluates that iteration's canonical
 * groups on the GPU -- the same partition sesgd_groups returns (A1; Alg.1 line 9,
 * P:236).  Graph-capturable: captured once with SESGD_ITER_NEXT, every replay moves to the next
 * iteration.  The host's iteration (shadow) advances the same way per ENQUEUE.
 * Errors: SESGD_EINVAL (iter < -1), SESGD_ESTATE (device iteration off), SESGD_ECUDA. */
#define SESGD_ITER_NEXT (-1)
SESGD_API int sesgd_begin_iter_device(sesgd_ctx *ctx, int64_t iter, void *stream);

/* Device address of the device iteration counter (int64, SESGD_OPT_DEVICE_ITER = 1): kernels of
 * the caller's own that depend on t (a data loader, an LR schedule, the synthetic gradients of
 * the tests) read it inside the same graph.  Owned by the context, valid until the option is
 * cleared or the context destroyed.  Errors: SESGD_EINVAL, SESGD_ESTATE (device iteration off). */
SESGD_API int sesgd_device_iter_ptr(const sesgd_ctx *ctx, const int64_t **t_dev_out);

/* Snapshot of the device iteration state (SESGD_OPT_DEVICE_ITER = 1), for tests and debugging:
 * synchronises the device, then copies t, the launch sequence number, the chunk-claim base, the
 * canonical groups of t (canon[n], -1 beyond n) and K5's ring of local worker 0, and the call
 * count of the first nbuckets buckets into bucket_calls (may be NULL when nbuckets = 0).
 * Errors: SESGD_EINVAL, SESGD_ESTATE (device iteration off), SESGD_ECUDA. */
typedef struct sesgd_device_iter_state {
  int64_t t, seq, claim_base;
  int32_t ring_pos;
  int8_t canon[SESGD_MAX_WORKERS];
  int8_t ring_rank[SESGD_MAX_WORKERS];
} sesgd_device_iter_state;
SESGD_API int sesgd_device_iter_read(const sesgd_ctx *ctx, sesgd_device_iter_state *out, int64_t *bucket_calls,
                                     int32_t nbuckets);

/* Number of SMs and CTAs per launch the library uses on the attached device (0 before attach). */
SESGD_API int sesgd_launch_grid(const sesgd_ctx *ctx, int32_t *ctas_out);

/* Copy and reset the one-shot kernel's per-CTA phase timers (SESGD_OPT_PROFILE = 1).
 * out[words] receives up to grid*8 u64: for CTA j, words [8j, 8j+8).  COMM CTAs (j <
 * *comm_ctas_out): 0 waiting for staged chunks, 1 pushing, 2 releasing flags, 3 total,
 * 7 launches.  COMPUTE CTAs: 0 staging, 1 folding (incl. waits), 2 total, 7 launches.
 * Errors: SESGD_EINVAL, SESGD_ESTATE (nothing recorded), SESGD_ECUDA. */
SESGD_API int sesgd_profile_read(sesgd_ctx *ctx, uint64_t *out, int64_t words, int32_t *comm_ctas_out);

/* ---- K7 probes (diagnostics; not part of an iteration) ---- */

/* Streaming 128-bit copy of `bytes` (multiple of 16, 16-byte aligned pointers) from `src` to
 * `dst`, any device-visible addresses: local->local (HBM), peer->local (NVLink pull) or
 * local->peer (NVLink push).  `ctas` CTAs (low 16 bits) of 512 threads (or, if bits 16..21
 * are non-zero, that many warps per CTA), enqueued on `stream`; the caller
 * times it (bandwidth bound of the exchange, row a5).  Errors: SESGD_EINVAL, SESGD_ECUDA. */
SESGD_API int sesgd_probe_copy(void *dst, const void *src, int64_t bytes, int32_t ctas, void *stream);

/* Flag ping-pong between two GPUs (per-hop handshake latency t_tau of Eq. 2).
 * Both ranks launch it concurrently on peer-mapped u64 flags: my_flag (local), peer_flag
 * (the other rank's my_flag).  The initiator stores base+2i+1 and waits for base+2i+2; the
 * responder mirrors it.  Writes the elapsed ns of `iters` round trips (or ~0 on a 10 s
 * timeout) to the device word out_ns_device.  `base` must exceed every earlier value written
 * to the flags.  Errors: SESGD_EINVAL, SESGD_ECUDA. */
SESGD_API int sesgd_probe_pingpong(uint64_t *my_flag, uint64_t *peer_flag, int32_t iters,
                                   int32_t initiator, uint64_t base, uint64_t *out_ns_device,
                                   void *stream);

SESGD_API const char *sesgd_strerror(int code);
SESGD_API const char *sesgd_last_error(const sesgd_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* SESGD_H */
