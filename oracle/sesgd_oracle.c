/*
 * sesgd_oracle.c -- TEST INFRASTRUCTURE: the plain, slow CPU oracle for the
 * Shuffle-Exchange SGD hot path.  See sesgd_oracle.h for the contract.
 *
 * Built with gcc -O2 -ffp-contract=off (no -ffast-math), so every float
 * expression below is a sequence of single IEEE-754 binary32 (or binary64)
 * round-to-nearest operations in exactly the order written (R10).
 *
 * Follows Algorithm 1 in its own order, per iteration t:
 *   lines 3-8   local step     xh_i = x_i - eta * (momentum-smoothed gradient)  (R8, R11)
 *   lines 9-10  new groups     G_t = generate_groups(sigma, t)                  (R1-R6)
 *   line 11     x_{i,t+1} = Ring-AllReduce(xh_i; G_{i,t}) = group mean          (Eq. 6, R7)
 * The Eq. 5 ("gradient") variant is ORC_MODE_GRAD (R9).
 *
 * Parity status of every function: pinned by tests/test_oracle_pins.py (see
 * DESIGN.md "Oracle pins"); nothing here is "parity unpinned" except agreement
 * with the paper's own (unpublished) PRNG and runs, which no test can reach.
 */
#include "sesgd_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "../synth/synth_gen.h"

/* ---- R2: splitmix64, exactly as S:61 (SPEC core.rng_next) ---- */
uint64_t orc_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

uint64_t orc_splitmix64_next(uint64_t *state) {
  *state += 0x9E3779B97F4A7C15ULL;
  return orc_mix(*state);
}

/* ---- R5: rejection-bounded draw (S:71 with the 2^64 overflow resolved) ---- */
uint64_t orc_bounded(uint64_t *state, uint64_t bound, int *err) {
  if (bound == 0) {
    if (err) *err = 1;
    return 0;
  }
  if (err) *err = 0;
  /* floor(2^64/bound)*bound = 2^64 - (2^64 mod bound); 2^64 mod bound = (0 - bound) % bound */
  uint64_t rem = (0 - bound) % bound;
  for (;;) {
    uint64_t w = orc_splitmix64_next(state);
    if (rem == 0 || w < (uint64_t)0 - rem) return w % bound;
  }
}

/* ---- A1: shuffle-exchange groups (R1, R3, R4, R6) ---- */
static int cmp_i32(const void *a, const void *b) {
  int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
  return (x > y) - (x < y);
}

int orc_groups(uint64_t seed, int64_t t, int32_t n, int32_t m, int32_t *raw, int32_t *canon,
               int32_t *group_of) {
  if (n < 1 || m < 1 || m > n || t < 0) return ORC_EINVAL;
  if (n % m != 0) return ORC_ENOTDIV;
  int32_t k = n / m;
  int32_t *p = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
  int32_t *groups = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
  int32_t *order = (int32_t *)malloc(sizeof(int32_t) * (size_t)k);
  /* "Initialize the pseudo-random algorithm with sigma" (Alg.1 line 1); per-iteration
   * seed s_t = mix(sigma XOR t) gives random access in t (R3). */
  uint64_t state = orc_mix(seed ^ (uint64_t)t);
  for (int32_t i = 0; i < n; ++i) p[i] = i;
  /* R4: Durstenfeld Fisher-Yates, descending i */
  for (int32_t i = n - 1; i >= 1; --i) {
    int32_t j = (int32_t)orc_bounded(&state, (uint64_t)(i + 1), NULL);
    int32_t tmp = p[i];
    p[i] = p[j];
    p[j] = tmp;
  }
  if (raw) memcpy(raw, p, sizeof(int32_t) * (size_t)n);
  /* R6: group j = slots [j*m, (j+1)*m), sorted ascending; groups ordered by smallest member */
  memcpy(groups, p, sizeof(int32_t) * (size_t)n);
  for (int32_t j = 0; j < k; ++j) qsort(groups + (size_t)j * m, (size_t)m, sizeof(int32_t), cmp_i32);
  for (int32_t j = 0; j < k; ++j) order[j] = j;
  for (int32_t a = 1; a < k; ++a) { /* insertion sort of group indices by first member */
    int32_t cur = order[a], b = a - 1;
    while (b >= 0 && groups[(size_t)order[b] * m] > groups[(size_t)cur * m]) {
      order[b + 1] = order[b];
      --b;
    }
    order[b + 1] = cur;
  }
  for (int32_t j = 0; j < k; ++j) {
    const int32_t *src = groups + (size_t)order[j] * m;
    for (int32_t r = 0; r < m; ++r) {
      if (canon) canon[(size_t)j * m + r] = src[r];
      if (group_of) group_of[src[r]] = j;
    }
  }
  free(p);
  free(groups);
  free(order);
  return ORC_OK;
}

/* ---- NEXT-3: Stone's shuffle-exchange as a deterministic schedule (alternative reading of
 * R1).  n = 2^d workers, m = 2^p: at iteration t the group of worker i is every worker that
 * agrees with i on all index bits except dimensions (t*p + q) mod d, q = 0..p-1 (shuffling the
 * index bits t*p times, then exchanging the low p bits).  n = 4, m = 2 gives {0,1},{2,3} then
 * {0,2},{1,3}: the example of P:176-177. ---- */
static int is_pow2(int32_t v) { return v > 0 && (v & (v - 1)) == 0; }

int orc_groups_stone(int64_t t, int32_t n, int32_t m, int32_t *canon, int32_t *group_of) {
  if (n < 1 || m < 1 || m > n || t < 0 || !is_pow2(n) || !is_pow2(m)) return ORC_EINVAL;
  int32_t d = 0, p = 0;
  while ((1 << d) < n) ++d;
  while ((1 << p) < m) ++p;
  int32_t mask = 0; /* the p exchanged dimensions of iteration t */
  for (int32_t q = 0; q < p; ++q) mask |= 1 << (int32_t)(((int64_t)t * p + q) % d);
  int32_t j = 0;
  for (int32_t i = 0; i < n; ++i) {
    if ((i & mask) != 0) continue; /* i is the smallest member of its group */
    int32_t r = 0;
    for (int32_t w = 0; w < n; ++w) { /* ascending: every w that differs from i only in mask */
      if ((w & ~mask) != i) continue;
      if (canon) canon[(size_t)j * m + r] = w;
      if (group_of) group_of[w] = j;
      ++r;
    }
    ++j;
  }
  return ORC_OK;
}

/* ---- A6/A7: Eq. 2 and Eq. 3 exact forms ---- */
int orc_latency(int32_t n, int32_t m, double bytes, double nu, double tau, double out[5]) {
  if (n < 1 || m < 1 || m > n) return ORC_EINVAL;
  if (n % m != 0) return ORC_ENOTDIV;
  if (!(nu > 0.0) || !(tau >= 0.0) || !(bytes >= 0.0) || !out) return ORC_EINVAL;
  /* T = 2(n-1) * (G/(n nu) + t_tau)   -- Eq. 2 with the ring over n workers */
  double ring_hs = 2.0 * (double)(n - 1);
  double ring_s = ring_hs * (bytes / ((double)n * nu) + tau);
  /* SESGD: the same ring inside a group of m = n/k workers (Eq. 3 before the approximation) */
  double se_hs = 2.0 * (double)(m - 1);
  double se_s = se_hs * (bytes / ((double)m * nu) + tau);
  out[0] = ring_hs;
  out[1] = se_hs;
  out[2] = ring_s;
  out[3] = se_s;
  if (se_s == 0.0)
    out[4] = (ring_s == 0.0) ? 1.0 : INFINITY;
  else
    out[4] = ring_s / se_s;
  return ORC_OK;
}

/* ---- A2/A5 (Eq. 6) and Eq. 5 variant: one iteration, binary32 ---- */
int orc_step_f32(int32_t n, int32_t m, const int32_t *canon, int64_t L, float *x, float *v,
                 const float *g, float lr, float mu, int32_t mode) {
  return orc_step_wd_f32(n, m, canon, L, x, v, g, lr, mu, 0.0f, mode);
}

/* as orc_step_f32, with torch.optim.SGD's weight decay on the gradient term (R20):
 * d = g + wd * x (skipped when wd == 0), then v = mu v + d; GRAD mode decays the group mean
 * with the worker's own x */
int orc_step_wd_f32(int32_t n, int32_t m, const int32_t *canon, int64_t L, float *x, float *v,
                    const float *g, float lr, float mu, float wd, int32_t mode) {
  return orc_step_ext_f32(n, m, canon, L, x, v, g, lr, mu, wd, 0, mode);
}

/* bfloat16 round to nearest even (the payload reading R21): keep the top 16 bits of the
 * binary32 pattern after adding half an ulp of bf16 plus the tie-breaking bit */
float orc_round_bf16(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return f; /* inf / nan unchanged */
  u += 0x7fffu + ((u >> 16) & 1u);
  u &= 0xffff0000u;
  memcpy(&f, &u, 4);
  return f;
}

int orc_step_ext_f32(int32_t n, int32_t m, const int32_t *canon, int64_t L, float *x, float *v,
                     const float *g, float lr, float mu, float wd, int32_t payload_bf16, int32_t mode) {
  if (n < 1 || m < 1 || m > n || L < 0 || !canon) return ORC_EINVAL;
  const int rnd = payload_bf16 && m > 1; /* only exchanged values are rounded */
  if (n % m != 0) return ORC_ENOTDIV;
  int32_t k = n / m;
  const float fm = (float)m;
  if (mode == ORC_MODE_PARAM) {
    float *xh = (float *)malloc(sizeof(float) * (size_t)n * (size_t)(L > 0 ? L : 1));
    /* Alg.1 lines 3-8 on every worker: v_i <- mu v_i + g_i ; xh_i <- x_i - eta v_i (R8) */
    for (int32_t i = 0; i < n; ++i) {
      for (int64_t e = 0; e < L; ++e) {
        size_t at = (size_t)i * (size_t)L + (size_t)e;
        float d = g[at];
        if (wd != 0.0f) d = d + wd * x[at];
        float mv = mu * v[at];
        float vn = mv + d;
        float step = lr * vn;
        v[at] = vn;
        xh[at] = x[at] - step;
      }
    }
    /* Alg.1 line 11 / Eq. 6: x_i <- (k/n) sum_{j in g(i,t)} xh_j = group mean (R7);
     * left fold in ascending member id, one division by m (R10) */
    for (int32_t j = 0; j < k; ++j) {
      const int32_t *G = canon + (size_t)j * m;
      for (int64_t e = 0; e < L; ++e) {
        float s = xh[(size_t)G[0] * (size_t)L + (size_t)e];
        if (rnd) s = orc_round_bf16(s);
        for (int32_t r = 1; r < m; ++r) {
          float h = xh[(size_t)G[r] * (size_t)L + (size_t)e];
          if (rnd) h = orc_round_bf16(h);
          s = s + h;
        }
        float mean = s / fm;
        for (int32_t r = 0; r < m; ++r) x[(size_t)G[r] * (size_t)L + (size_t)e] = mean;
      }
    }
    free(xh);
  } else if (mode == ORC_MODE_GRAD) {
    /* Eq. 5 variant: gb_G = group mean of g ; v_i <- mu v_i + gb ; x_i <- x_i - eta v_i */
    for (int32_t j = 0; j < k; ++j) {
      const int32_t *G = canon + (size_t)j * m;
      for (int64_t e = 0; e < L; ++e) {
        float s = g[(size_t)G[0] * (size_t)L + (size_t)e];
        if (rnd) s = orc_round_bf16(s);
        for (int32_t r = 1; r < m; ++r) {
          float h = g[(size_t)G[r] * (size_t)L + (size_t)e];
          if (rnd) h = orc_round_bf16(h);
          s = s + h;
        }
        float gb = s / fm;
        for (int32_t r = 0; r < m; ++r) {
          size_t at = (size_t)G[r] * (size_t)L + (size_t)e;
          float d = gb;
          if (wd != 0.0f) d = d + wd * x[at];
          float mv = mu * v[at];
          float vn = mv + d;
          float step = lr * vn;
          v[at] = vn;
          x[at] = x[at] - step;
        }
      }
    }
  } else {
    return ORC_EINVAL;
  }
  return ORC_OK;
}

/* ---- the same, binary64 (for invariants / closed forms; not the GPU gate) ---- */
int orc_step_f64(int32_t n, int32_t m, const int32_t *canon, int64_t L, double *x, double *v,
                 const double *g, double lr, double mu, int32_t mode) {
  if (n < 1 || m < 1 || m > n || L < 0 || !canon) return ORC_EINVAL;
  if (n % m != 0) return ORC_ENOTDIV;
  int32_t k = n / m;
  const double dm = (double)m;
  if (mode == ORC_MODE_PARAM) {
    double *xh = (double *)malloc(sizeof(double) * (size_t)n * (size_t)(L > 0 ? L : 1));
    for (int32_t i = 0; i < n; ++i) {
      for (int64_t e = 0; e < L; ++e) {
        size_t at = (size_t)i * (size_t)L + (size_t)e;
        double mv = mu * v[at];
        double vn = mv + g[at];
        double step = lr * vn;
        v[at] = vn;
        xh[at] = x[at] - step;
      }
    }
    for (int32_t j = 0; j < k; ++j) {
      const int32_t *G = canon + (size_t)j * m;
      for (int64_t e = 0; e < L; ++e) {
        double s = xh[(size_t)G[0] * (size_t)L + (size_t)e];
        for (int32_t r = 1; r < m; ++r) s = s + xh[(size_t)G[r] * (size_t)L + (size_t)e];
        double mean = s / dm;
        for (int32_t r = 0; r < m; ++r) x[(size_t)G[r] * (size_t)L + (size_t)e] = mean;
      }
    }
    free(xh);
  } else if (mode == ORC_MODE_GRAD) {
    for (int32_t j = 0; j < k; ++j) {
      const int32_t *G = canon + (size_t)j * m;
      for (int64_t e = 0; e < L; ++e) {
        double s = g[(size_t)G[0] * (size_t)L + (size_t)e];
        for (int32_t r = 1; r < m; ++r) s = s + g[(size_t)G[r] * (size_t)L + (size_t)e];
        double gb = s / dm;
        for (int32_t r = 0; r < m; ++r) {
          size_t at = (size_t)G[r] * (size_t)L + (size_t)e;
          double mv = mu * v[at];
          double vn = mv + gb;
          double step = lr * vn;
          v[at] = vn;
          x[at] = x[at] - step;
        }
      }
    }
  } else {
    return ORC_EINVAL;
  }
  return ORC_OK;
}

/* ---- the group mean by Ring-AllReduce in ring order (Sec. 2.2) ---- */
int32_t orc_slice_of(int64_t L, int32_t m, int64_t e) {
  /* slice s = [floor(s L / m), floor((s+1) L / m)): the largest s with floor(s L / m) <= e */
  int32_t s = 0;
  while (s + 1 < m && ((s + 1) * L) / m <= e) ++s;
  return s;
}

int orc_step_ring_f32(int32_t n, int32_t m, const int32_t *canon, int64_t L, float *x, float *v,
                      const float *g, float lr, float mu, int32_t mode) {
  if (n < 1 || m < 1 || m > n || L < 0 || !canon) return ORC_EINVAL;
  if (n % m != 0) return ORC_ENOTDIV;
  int32_t k = n / m;
  const float fm = (float)m;
  float *pay = (float *)malloc(sizeof(float) * (size_t)n * (size_t)(L > 0 ? L : 1));
  if (mode == ORC_MODE_PARAM) {
    /* Alg.1 lines 3-8: the payload is xh_i = x_i - eta (mu v_i + g_i) */
    for (int32_t i = 0; i < n; ++i)
      for (int64_t e = 0; e < L; ++e) {
        size_t at = (size_t)i * (size_t)L + (size_t)e;
        float mv = mu * v[at];
        float vn = mv + g[at];
        float step = lr * vn;
        v[at] = vn;
        pay[at] = x[at] - step;
      }
  } else if (mode == ORC_MODE_GRAD) {
    memcpy(pay, g, sizeof(float) * (size_t)n * (size_t)L);
  } else {
    free(pay);
    return ORC_EINVAL;
  }
  for (int32_t j = 0; j < k; ++j) {
    const int32_t *G = canon + (size_t)j * m;
    for (int64_t e = 0; e < L; ++e) {
      /* Scatter-Reduce: "slice s accumulated in ring order starting from member (s+1) mod m"
       * (S:263): it starts at ring position s+1 and travels the ring, each member adding its
       * own value to what it received, so member s adds last and holds the full sum */
      int32_t s = orc_slice_of(L, m, e);
      float acc = pay[(size_t)G[(s + 1) % m] * (size_t)L + (size_t)e];
      for (int32_t t = 2; t <= m; ++t) acc = acc + pay[(size_t)G[(s + t) % m] * (size_t)L + (size_t)e];
      float mean = acc / fm; /* "division by m applied once after full accumulation" */
      /* All-Gather: every member receives the same mean */
      for (int32_t r = 0; r < m; ++r) {
        size_t at = (size_t)G[r] * (size_t)L + (size_t)e;
        if (mode == ORC_MODE_PARAM) {
          x[at] = mean;
        } else {
          float mv = mu * v[at];
          float vn = mv + mean;
          float step = lr * vn;
          v[at] = vn;
          x[at] = x[at] - step;
        }
      }
    }
  }
  free(pay);
  return ORC_OK;
}

int orc_run_ring_f32(int32_t n, int32_t m, uint64_t seed, int64_t t0, int64_t T, int64_t L,
                     int64_t e0, uint64_t s_g, float lr, float mu, int32_t mode, float *x, float *v) {
  if (n < 1 || m < 1 || m > n || t0 < 0 || T < 0 || L < 0) return ORC_EINVAL;
  if (n % m != 0) return ORC_ENOTDIV;
  float *g = (float *)malloc(sizeof(float) * (size_t)n * (size_t)(L > 0 ? L : 1));
  int32_t *canon = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
  int rc = ORC_OK;
  for (int64_t t = t0; t < t0 + T && rc == ORC_OK; ++t) {
    for (int32_t i = 0; i < n; ++i) {
      uint64_t key = synth_grad_key(s_g, i, t);
      for (int64_t e = 0; e < L; ++e) g[(size_t)i * (size_t)L + (size_t)e] = synth_grad(key, e0 + e);
    }
    rc = orc_groups(seed, t, n, m, NULL, canon, NULL);
    if (rc == ORC_OK) rc = orc_step_ring_f32(n, m, canon, L, x, v, g, lr, mu, mode);
  }
  free(g);
  free(canon);
  return rc;
}

/* ---- T iterations with synthetic gradients at chosen coordinates ---- */
int orc_run_f32(int32_t n, int32_t m, uint64_t seed, int64_t t0, int64_t T, int64_t S,
                const int64_t *coords, uint64_t s_g, float lr, float mu, int32_t mode, float *x,
                float *v) {
  if (n < 1 || m < 1 || m > n || t0 < 0 || T < 0 || S < 0) return ORC_EINVAL;
  if (n % m != 0) return ORC_ENOTDIV;
  float *g = (float *)malloc(sizeof(float) * (size_t)n * (size_t)(S > 0 ? S : 1));
  int32_t *canon = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
  int rc = ORC_OK;
  for (int64_t t = t0; t < t0 + T && rc == ORC_OK; ++t) {
    for (int32_t i = 0; i < n; ++i) { /* Alg.1 lines 4-6: worker i's gradient (synthetic) */
      uint64_t key = synth_grad_key(s_g, i, t);
      for (int64_t e = 0; e < S; ++e)
        g[(size_t)i * (size_t)S + (size_t)e] = synth_grad(key, coords ? coords[e] : e);
    }
    rc = orc_groups(seed, t, n, m, NULL, canon, NULL); /* Alg.1 lines 9-10 */
    if (rc == ORC_OK) rc = orc_step_f32(n, m, canon, S, x, v, g, lr, mu, mode);
  }
  free(g);
  free(canon);
  return rc;
}

int orc_run_f64(int32_t n, int32_t m, uint64_t seed, int64_t t0, int64_t T, int64_t S,
                const int64_t *coords, uint64_t s_g, double lr, double mu, int32_t mode, double *x,
                double *v) {
  if (n < 1 || m < 1 || m > n || t0 < 0 || T < 0 || S < 0) return ORC_EINVAL;
  if (n % m != 0) return ORC_ENOTDIV;
  double *g = (double *)malloc(sizeof(double) * (size_t)n * (size_t)(S > 0 ? S : 1));
  int32_t *canon = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
  int rc = ORC_OK;
  for (int64_t t = t0; t < t0 + T && rc == ORC_OK; ++t) {
    for (int32_t i = 0; i < n; ++i) {
      uint64_t key = synth_grad_key(s_g, i, t);
      for (int64_t e = 0; e < S; ++e)
        g[(size_t)i * (size_t)S + (size_t)e] = (double)synth_grad(key, coords ? coords[e] : e);
    }
    rc = orc_groups(seed, t, n, m, NULL, canon, NULL);
    if (rc == ORC_OK) rc = orc_step_f64(n, m, canon, S, x, v, g, lr, mu, mode);
  }
  free(g);
  free(canon);
  return rc;
}

/* ---- Local-SESGD: exchange only when (t + 1) mod H == 0 ---- */
int orc_run_local_f32(int32_t n, int32_t m, uint64_t seed, int64_t t0, int64_t T, int64_t S,
                      const int64_t *coords, uint64_t s_g, float lr, float mu, int32_t mode,
                      int64_t H, int32_t schedule, float wd, float *x, float *v) {
  return orc_run_ext_f32(n, m, seed, t0, T, S, coords, s_g, lr, mu, mode, H, schedule, wd, 0, x, v);
}

int orc_run_ext_f32(int32_t n, int32_t m, uint64_t seed, int64_t t0, int64_t T, int64_t S,
                    const int64_t *coords, uint64_t s_g, float lr, float mu, int32_t mode, int64_t H,
                    int32_t schedule, float wd, int32_t payload_bf16, float *x, float *v) {
  if (n < 1 || m < 1 || m > n || t0 < 0 || T < 0 || S < 0 || H < 1) return ORC_EINVAL;
  if (schedule != 0 && schedule != 1) return ORC_EINVAL;
  if (n % m != 0) return ORC_ENOTDIV;
  float *g = (float *)malloc(sizeof(float) * (size_t)n * (size_t)(S > 0 ? S : 1));
  int32_t *canon = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
  int rc = ORC_OK;
  for (int64_t t = t0; t < t0 + T && rc == ORC_OK; ++t) {
    for (int32_t i = 0; i < n; ++i) {
      uint64_t key = synth_grad_key(s_g, i, t);
      for (int64_t e = 0; e < S; ++e)
        g[(size_t)i * (size_t)S + (size_t)e] = synth_grad(key, coords ? coords[e] : e);
    }
    if ((t + 1) % H == 0) { /* synchronisation iteration: SESGD step with the groups of t */
      rc = schedule == 1 ? orc_groups_stone(t, n, m, canon, NULL)
                         : orc_groups(seed, t, n, m, NULL, canon, NULL);
      if (rc == ORC_OK) rc = orc_step_ext_f32(n, m, canon, S, x, v, g, lr, mu, wd, payload_bf16, mode);
    } else { /* local iteration: every worker its own singleton group */
      for (int32_t i = 0; i < n; ++i) canon[i] = i;
      rc = orc_step_ext_f32(n, 1, canon, S, x, v, g, lr, mu, wd, payload_bf16, mode);
    }
  }
  free(g);
  free(canon);
  return rc;
}

/* ---- final global average (Alg.1 last line) ---- */
int orc_global_average_f32(int32_t n, int64_t L, float *x) {
  if (n < 1 || L < 0 || (L > 0 && !x)) return ORC_EINVAL;
  for (int64_t e = 0; e < L; ++e) {
    float s = x[e];
    for (int32_t i = 1; i < n; ++i) s = s + x[(size_t)i * (size_t)L + (size_t)e];
    s = s / (float)n;
    for (int32_t i = 0; i < n; ++i) x[(size_t)i * (size_t)L + (size_t)e] = s;
  }
  return ORC_OK;
}

int orc_global_average_f64(int32_t n, int64_t L, double *x) {
  if (n < 1 || L < 0 || (L > 0 && !x)) return ORC_EINVAL;
  for (int64_t e = 0; e < L; ++e) {
    double s = x[e];
    for (int32_t i = 1; i < n; ++i) s = s + x[(size_t)i * (size_t)L + (size_t)e];
    s = s / (double)n;
    for (int32_t i = 0; i < n; ++i) x[(size_t)i * (size_t)L + (size_t)e] = s;
  }
  return ORC_OK;
}

/* ---- NEXT-4: consistency of the workers' parameters (Fig. 7b's question) ----
 * out[0] = sum_i sum_e (x_i[e] - xbar[e])^2   (xbar = mean over the n workers, binary64)
 * out[1] = max_i max_e |x_i[e] - xbar[e]|
 * the consensus distance of decentralised SGD is out[0] / n. */
int orc_consensus(int32_t n, int64_t L, const float *x, double out[2]) {
  if (n < 1 || L < 0 || !out || (L > 0 && !x)) return ORC_EINVAL;
  double ss = 0.0, mx = 0.0;
  for (int64_t e = 0; e < L; ++e) {
    double mean = 0.0;
    for (int32_t i = 0; i < n; ++i) mean += (double)x[(size_t)i * (size_t)L + (size_t)e];
    mean /= (double)n;
    for (int32_t i = 0; i < n; ++i) {
      double d = (double)x[(size_t)i * (size_t)L + (size_t)e] - mean;
      ss += d * d;
      if (fabs(d) > mx) mx = fabs(d);
    }
  }
  out[0] = ss;
  out[1] = mx;
  return ORC_OK;
}
