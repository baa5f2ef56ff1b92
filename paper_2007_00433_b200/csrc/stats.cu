// stats.cu -- K10: the group schedule evaluated on the device for many iterations at once, to
// count how often every pair of workers shares a group (the pair-split Monte Carlo of the
// paper's appendix: Pr[i, j in different groups] = n (k - 1) / (k (n - 1))).
//
// One thread per iteration t: the same schedule the host scheduler (schedule.cpp) emits --
// s_t = F(sigma XOR t) (R3), a splitmix64 stream (R2), descending Fisher-Yates with rejection-
// bounded draws (R4, R5), group j = slots [j m, (j + 1) m) -- or Stone's dimension exchange
// (SESGD_OPT_SCHEDULE = 1).  Pair counts go to a per-CTA shared-memory histogram first.
#include "common.cuh"
#include "internal.h"

namespace sesgd {
namespace {

constexpr int kStatsThreads = 256;

__device__ __forceinline__ uint64_t fin(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t draw_below(uint64_t &state, uint64_t bound) {
  const uint64_t tail = (0ULL - bound) % bound;  // 2^64 mod bound
  for (;;) {
    state += 0x9E3779B97F4A7C15ULL;
    const uint64_t w = fin(state);
    if (tail == 0 || w < 0ULL - tail) return w % bound;
  }
}

__global__ void __launch_bounds__(kStatsThreads) k10_pair_counts(uint64_t seed, int64_t t0, int64_t T,
                                                                 int n, int m, int schedule,
                                                                 unsigned long long *counts) {
  extern __shared__ unsigned int hist[];  // [n * n]
  for (int i = threadIdx.x; i < n * n; i += kStatsThreads) hist[i] = 0;
  __syncthreads();
  for (int64_t it = int64_t(blockIdx.x) * kStatsThreads + threadIdx.x; it < T;
       it += int64_t(gridDim.x) * kStatsThreads) {
    const int64_t t = t0 + it;
    int8_t slot[SESGD_MAX_WORKERS];  // worker in each slot
    if (schedule == 1) {  // dimension exchange: slots ordered by (bits outside the mask, mask bits)
      const int d = __ffs(n) - 1, p = __ffs(m) - 1;
      unsigned mask = 0;
      for (int q = 0; q < p; ++q) mask |= 1u << int((t * p + q) % d);
      int s = 0;
      for (unsigned base = 0; base < unsigned(n); ++base) {
        if (base & mask) continue;
        unsigned sub = 0;
        do {
          slot[s++] = int8_t(base | sub);
          sub = (sub - mask) & mask;
        } while (sub != 0);
      }
    } else {
      uint64_t state = fin(seed ^ uint64_t(t));
      for (int i = 0; i < n; ++i) slot[i] = int8_t(i);
      for (int i = n - 1; i > 0; --i) {
        const int j = int(draw_below(state, uint64_t(i) + 1));
        const int8_t tmp = slot[i];
        slot[i] = slot[j];
        slot[j] = tmp;
      }
    }
    for (int g = 0; g < n; g += m)
      for (int a = 0; a < m; ++a)
        for (int b = a + 1; b < m; ++b) {
          const int u = slot[g + a], v = slot[g + b];
          atomicAdd(&hist[(u < v ? u : v) * n + (u < v ? v : u)], 1u);
        }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n * n; i += kStatsThreads)
    if (hist[i]) atomicAdd(&counts[i], (unsigned long long)hist[i]);
}

}  // namespace

cudaError_t launch_pair_counts(uint64_t seed, int64_t t0, int64_t T, int n, int m, int schedule,
                               unsigned long long *counts, int sm_count, cudaStream_t stream) {
  int64_t blocks = (T + kStatsThreads - 1) / kStatsThreads;
  blocks = blocks < 1 ? 1 : (blocks > int64_t(sm_count) * 8 ? int64_t(sm_count) * 8 : blocks);
  k10_pair_counts<<<unsigned(blocks), kStatsThreads, size_t(n) * n * 4, stream>>>(seed, t0, T, n, m,
                                                                                 schedule, counts);
  return cudaGetLastError();
}

}  // namespace sesgd
