/*
 * sesgd_oracle.h -- TEST INFRASTRUCTURE.  Plain, slow, single-threaded CPU oracle
 * for the Shuffle-Exchange SGD hot path (arXiv 2007.00433).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this.  It shares no code with the CUDA product
 * (paper_2007_00433_b200/); the only shared include is synth/synth_gen.h, the
 * seeded input generator, which holds none of the method's arithmetic.
 *
 * Citations: P:n = PAPER.md line n, S:n = SPEC.md line n (both under the
 * read-only reference tree); R1..R21 = readings listed in DESIGN.md.
 */
#ifndef SESGD_ORACLE_H
#define SESGD_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (mirror of the product's meanings, defined independently) */
#define ORC_OK 0
#define ORC_EINVAL (-1)
#define ORC_ENOTDIV (-2)

#define ORC_MODE_PARAM 0 /* Eq. 6: average locally-stepped params */
#define ORC_MODE_GRAD 1  /* Eq. 5 variant: average gradients in group */

/* splitmix64 step (R2): state += gamma; return finaliser(state). */
uint64_t orc_splitmix64_next(uint64_t *state);
/* splitmix64 finaliser only (R3): the "mix" of s_t = mix(seed ^ t). */
uint64_t orc_mix(uint64_t z);
/* unbiased integer in [0, bound) by rejection (R5). bound==0 -> returns 0, *err=1. */
uint64_t orc_bounded(uint64_t *state, uint64_t bound, int *err);

/* Group schedule g(i,t) (A1; Alg.1 lines 1,9-10 P:226,236-237; R1-R6).
 * raw[n]     : Fisher-Yates permutation slots (may be NULL)
 * canon[n]   : canonical form: groups of m ascending members, groups ordered by
 *              smallest member; group j = canon[j*m .. j*m+m-1]       (may be NULL)
 * group_of[n]: index of worker i's group in canonical order           (may be NULL) */
int orc_groups(uint64_t seed, int64_t t, int32_t n, int32_t m, int32_t *raw, int32_t *canon,
               int32_t *group_of);

/* Latency model, Eq. 2 / Eq. 3 exact forms (R16).
 * out[0]=ring handshakes 2(n-1), out[1]=SESGD handshakes 2(m-1),
 * out[2]=ring seconds 2(n-1)(G/(n nu)+tau), out[3]=SESGD seconds 2(m-1)(G/(m nu)+tau),
 * out[4]=ring/SESGD ratio (1 if both are 0, +inf if only SESGD is 0). */
int orc_latency(int32_t n, int32_t m, double bytes, double nu, double tau, double out[5]);

/* One iteration over explicit arrays (worker-major, x[i*L + e]).
 * canon: canonical groups of this iteration (as orc_groups writes them).
 * PARAM (Eq. 6 + R8): v_i = mu v_i + g_i ; xh_i = x_i - lr v_i ; x_i = (sum_{j in G} xh_j) / m
 * GRAD  (Eq. 5 + R8): gb = (sum_{j in G} g_j) / m ; v_i = mu v_i + gb ; x_i = x_i - lr v_i
 * f32: every operation a single binary32 round-to-nearest op (compiled -ffp-contract=off). */
int orc_step_f32(int32_t n, int32_t m, const int32_t *canon, int64_t L, float *x, float *v,
                 const float *g, float lr, float mu, int32_t mode);
int orc_step_f64(int32_t n, int32_t m, const int32_t *canon, int64_t L, double *x, double *v,
                 const double *g, double lr, double mu, int32_t mode);
/* The same binary32 iteration with torch.optim.SGD's weight decay (R20): the momentum
 * step's gradient term is d = g + wd * x (not applied when wd == 0); GRAD mode: d = gbar + wd * x
 * with the worker's own x. */
int orc_step_wd_f32(int32_t n, int32_t m, const int32_t *canon, int64_t L, float *x, float *v,
                    const float *g, float lr, float mu, float wd, int32_t mode);
/* ... and the bf16-payload reading (R21): with payload_bf16 = 1 and m > 1 every contribution to
 * a group fold (xh in PARAM, g in GRAD) is first rounded to bfloat16 (round to nearest even);
 * the fold, the mean and the update stay binary32. */
int orc_step_ext_f32(int32_t n, int32_t m, const int32_t *canon, int64_t L, float *x, float *v,
                     const float *g, float lr, float mu, float wd, int32_t payload_bf16, int32_t mode);
float orc_round_bf16(float f);

/* The same iteration with the group mean computed by the paper's Ring-AllReduce (Sec. 2.2,
 * P:99-104) in ring order: members in ascending id form the ring; element e lies in slice
 * s = the slice of SPEC slice_bounds ([floor(sL/m), floor((s+1)L/m))) containing
 * it, and its sum is accumulated starting at ring position s: ((xh_s + xh_{s+1}) + ...) +
 * xh_{s+m-1} (positions mod m), then divided once by m.  Equals orc_step_f32 for m <= 2. */
int orc_step_ring_f32(int32_t n, int32_t m, const int32_t *canon, int64_t L, float *x, float *v,
                      const float *g, float lr, float mu, int32_t mode);
/* slice of element e in [0, L) split into m slices */
int32_t orc_slice_of(int64_t L, int32_t m, int64_t e);
/* T ring-order iterations over ONE bucket of L elements at global coordinates e0..e0+L-1 */
int orc_run_ring_f32(int32_t n, int32_t m, uint64_t seed, int64_t t0, int64_t T, int64_t L,
                     int64_t e0, uint64_t s_g, float lr, float mu, int32_t mode, float *x, float *v);

/* T iterations t0..t0+T-1 with synthetic gradients (synth_gen.h) at S global
 * coordinates coords[0..S-1] (coordinates are independent, so any subset of the
 * full problem replays exactly).  x, v: [n*S] in/out.  coords==NULL -> 0..S-1. */
int orc_run_f32(int32_t n, int32_t m, uint64_t seed, int64_t t0, int64_t T, int64_t S,
                const int64_t *coords, uint64_t s_g, float lr, float mu, int32_t mode, float *x,
                float *v);
int orc_run_f64(int32_t n, int32_t m, uint64_t seed, int64_t t0, int64_t T, int64_t S,
                const int64_t *coords, uint64_t s_g, double lr, double mu, int32_t mode, double *x,
                double *v);

/* Local-SESGD (paper Sec. 4.1 "Baseline" P:315-317): as orc_run_f32, but the
 * group exchange of iteration t fires only when (t + 1) mod H == 0 (groups of that t); on the
 * other iterations the locally updated parameters are kept (the iteration with m = 1:
 * PARAM x = xh, GRAD v = mu v + g, x = x - lr v).  H = 1 is SESGD; m = n is Local-SGD
 * (the paper's baseline with period 2).  schedule: 0 = orc_groups (R1),
 * 1 = orc_groups_stone (NEXT-3).  wd: weight decay as orc_step_wd_f32. */
int orc_run_local_f32(int32_t n, int32_t m, uint64_t seed, int64_t t0, int64_t T, int64_t S,
                      const int64_t *coords, uint64_t s_g, float lr, float mu, int32_t mode,
                      int64_t H, int32_t schedule, float wd, float *x, float *v);

int orc_run_ext_f32(int32_t n, int32_t m, uint64_t seed, int64_t t0, int64_t T, int64_t S,
                    const int64_t *coords, uint64_t s_g, float lr, float mu, int32_t mode, int64_t H,
                    int32_t schedule, float wd, int32_t payload_bf16, float *x, float *v);

/* NEXT-3, alternative reading of R1 (Stone's perfect shuffle): n = 2^d, m = 2^p; at
 * iteration t worker i's group is every worker equal to i outside index dimensions
 * (t*p + q) mod d, q < p (canonical form as orc_groups).  schedule 1 of orc_run_local_f32. */
int orc_groups_stone(int64_t t, int32_t n, int32_t m, int32_t *canon, int32_t *group_of);

/* Algorithm 1's last line: xbar = Ring-AllReduce(x_i; Global), the mean of the n
 * workers' parameters, left fold in ascending worker id then one division by n
 * (R7, R10); written back to every worker's row of x [n*L]. */
int orc_global_average_f32(int32_t n, int64_t L, float *x);
int orc_global_average_f64(int32_t n, int64_t L, double *x);

/* Consistency of the n workers' parameters x [n*L]: out[0] = sum over workers and
 * elements of (x_i - xbar)^2, out[1] = max |x_i - xbar|, in binary64 (xbar = worker mean). */
int orc_consensus(int32_t n, int64_t L, const float *x, double out[2]);

#ifdef __cplusplus
}
#endif
#endif
