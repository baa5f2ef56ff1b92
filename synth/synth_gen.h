/*
 * synth_gen.h -- seeded synthetic INPUT generators (test/bench infrastructure).
 *
 * This module holds none of the method's arithmetic.  It only manufactures the
 * inputs the SESGD hot path consumes: the initial parameters x_0 (shared by all
 * workers, "Note all workers start with the same x_0", Sec. 3.2)
 * and one synthetic gradient per (worker, iteration, element), standing in for
 * the backward pass of Algorithm 1 lines 4-8.
 *
 * It is the ONE piece of code both sides may share:
 * the CPU oracle (oracle/) includes it for host generation, and synth/synth.cu
 * wraps it in device fill kernels for the GPU benches and parity tests.  The
 * product library (paper_2007_00433_b200/csrc) never includes it.
 *
 * Counter-based, stateless, integer-only (no libm), so every value is
 * reproducible bit-for-bit on host and device:
 *   h(z)            = murmur3 fmix64 finaliser (deliberately NOT splitmix64, so
 *                     the generator shares no constant with the schedule PRNG)
 *   key(s_g, i, t)  = h(h(h(s_g ^ C_G) + i) + t)
 *   g_i,t[e]        = (int32(h(key ^ e) >> 40) - 2^23) * 2^-29   in [-2^-6, 2^-6)
 *   x_0[e]          = (int32(h(h(s_x ^ C_X) ^ e) >> 40) - 2^23) * 2^-26   in [-1/8, 1/8)
 * Each value is an integer of at most 24 bits times a power of two, hence exact
 * in binary32 (and binary64).
 */
#ifndef SYNTH_GEN_H
#define SYNTH_GEN_H

#include <stdint.h>

#if defined(__CUDACC__)
#define SYNTH_HD __host__ __device__ __forceinline__
#else
#define SYNTH_HD static inline
#endif

#define SYNTH_C_GRAD 0x6772616469656e74ULL /* "gradient" */
#define SYNTH_C_X0 0x706172616d733030ULL   /* "params00" */

SYNTH_HD uint64_t synth_h(uint64_t z) {
  z ^= z >> 33;
  z *= 0xff51afd7ed558ccdULL;
  z ^= z >> 33;
  z *= 0xc4ceb9fe1a85ec53ULL;
  z ^= z >> 33;
  return z;
}

/* 24 random bits -> centred integer in [-2^23, 2^23) */
SYNTH_HD int32_t synth_i24(uint64_t z) { return (int32_t)(z >> 40) - (1 << 23); }

SYNTH_HD uint64_t synth_grad_key(uint64_t s_g, int32_t worker, int64_t t) {
  return synth_h(synth_h(synth_h(s_g ^ SYNTH_C_GRAD) + (uint64_t)(int64_t)worker) +
                 (uint64_t)t);
}

/* gradient element e of worker i at iteration t, given key = synth_grad_key(s_g,i,t) */
SYNTH_HD float synth_grad(uint64_t key, int64_t e) {
  return (float)synth_i24(synth_h(key ^ (uint64_t)e)) * 1.862645149230957e-09f; /* 2^-29 */
}

SYNTH_HD uint64_t synth_x0_key(uint64_t s_x) { return synth_h(s_x ^ SYNTH_C_X0); }

SYNTH_HD float synth_x0(uint64_t xkey, int64_t e) {
  return (float)synth_i24(synth_h(xkey ^ (uint64_t)e)) * 1.4901161193847656e-08f; /* 2^-26 */
}

#endif /* SYNTH_GEN_H */
