// stats.cu -- K10: the group schedule evaluated on the device for many iterations at once, to
// count how often every pair of workers shares a group (the pair-split Monte Carlo of the
// paper's appendix: Pr[i, j in different groups] = n (k - 1) / (k (n - 1))).
//
// One thread per iteration t: the same schedule the host scheduler (schedule.cpp) emits --
// s_t = F(sigma XOR t) (R3), a splitmix64 stream (R2), descending Fisher-Yates with rejection-
// bounded draws (R4, R5), group j = slots [j m, (j + 1) m) -- or Stone's dimension exchange
// (SESGD_OPT_SCHEDULE = 1), sched_dev.cuh.  Pair counts go to a per-CTA shared-memory histogram first.
#include "common.cuh"
#include "internal.h"
#include "sched_dev.cuh"

namespace sesgd {
namespace {

constexpr int kStatsThreads = 256;

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
    sched::slots(seed, t, n, m, schedule, slot);
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
