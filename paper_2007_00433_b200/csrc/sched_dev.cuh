// sched_dev.cuh -- the group schedule (A1) evaluated on the device: the same slots the host
// scheduler (schedule.cpp) emits, for K10 (pair counts over many iterations) and for the
// device-resident iteration state (iter.cu, SESGD_OPT_DEVICE_ITER).
//
// "use the pseudo-random algorithm to generate the grouping information and set the same random
// seed on every worker to avoid extra message exchange" (Sec. 3.1); Alg.1 line 9
// (P:236).  Readings R2-R6: s_t = F(sigma XOR t) with F the splitmix64 output finaliser, a
// splitmix64 stream seeded with s_t, descending Fisher-Yates whose bounded draws redraw the top
// 2^64 mod b words; group j = slots [j m, (j + 1) m).  Or Stone's dimension exchange (R19).
#pragma once
#include <stdint.h>

namespace sesgd {
namespace sched {

__host__ __device__ __forceinline__ uint64_t fin(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint64_t draw_below(uint64_t &state, uint64_t bound) {
  const uint64_t tail = (0ULL - bound) % bound;  // 2^64 mod bound
  for (;;) {
    state += 0x9E3779B97F4A7C15ULL;
    const uint64_t w = fin(state);
    if (tail == 0 || w < 0ULL - tail) return w % bound;
  }
}

// slot[s] = worker in slot s of iteration t (group j = slots [j m, (j + 1) m), not canonical)
__host__ __device__ __forceinline__ void slots(uint64_t seed, int64_t t, int n, int m, int schedule, int8_t *slot) {
  if (schedule == 1) {  // dimension exchange: slots ordered by (bits outside the mask, mask bits)
#ifdef __CUDA_ARCH__
    const int d = __ffs(n) - 1, p = __ffs(m) - 1;
#else
    const int d = __builtin_ffs(n) - 1, p = __builtin_ffs(m) - 1;
#endif
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
    return;
  }
  uint64_t state = fin(seed ^ uint64_t(t));
  for (int i = 0; i < n; ++i) slot[i] = int8_t(i);
  for (int i = n - 1; i > 0; --i) {
    const int j = int(draw_below(state, uint64_t(i) + 1));
    const int8_t tmp = slot[i];
    slot[i] = slot[j];
    slot[j] = tmp;
  }
}

// R6: canonical form in place -- every group sorted ascending, groups ordered by first member;
// group_of[w] = index of w's group.  Insertion sorts: n <= 64.
__host__ __device__ __forceinline__ void canonical(int8_t *slot, int n, int m, int8_t *group_of) {
  const int k = n / m;
  for (int j = 0; j < k; ++j) {
    int8_t *g = slot + j * m;
    for (int a = 1; a < m; ++a) {
      const int8_t v = g[a];
      int b = a - 1;
      while (b >= 0 && g[b] > v) {
        g[b + 1] = g[b];
        --b;
      }
      g[b + 1] = v;
    }
  }
  for (int a = 1; a < k; ++a) {  // groups by first member (first members are distinct)
    int b = a;
    while (b > 0 && slot[(b - 1) * m] > slot[b * m]) {
      for (int r = 0; r < m; ++r) {
        const int8_t tmp = slot[(b - 1) * m + r];
        slot[(b - 1) * m + r] = slot[b * m + r];
        slot[b * m + r] = tmp;
      }
      --b;
    }
  }
  for (int j = 0; j < k; ++j)
    for (int r = 0; r < m; ++r) group_of[slot[j * m + r]] = int8_t(j);
}

}  // namespace sched
}  // namespace sesgd
