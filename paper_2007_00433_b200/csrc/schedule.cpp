// schedule.cpp -- host-side group scheduler and latency model of libsesgd.
//
// Independent of the oracle (written from DESIGN.md's readings, not from its code).
//
// Group schedule (A1): "randomly shuffle these workers into different groups"
// (Sec. 3.1); "use the pseudo-random algorithm to generate the grouping
// information and set the same random seed on every worker to avoid extra
// message exchange"; Alg.1 line 9 "Randomly generate new groups
// depending on sigma".  Concretely (R1-R6):
//   s_t = F(sigma XOR t) with F the splitmix64 output finaliser (R3);
//   a splitmix64 stream seeded with s_t drives a descending Fisher-Yates shuffle
//   of 0..n-1 (R2, R4) whose bounded draws reject the top 2^64 mod b words (R5);
//   group j = slots [j*m, (j+1)*m), each sorted, groups ordered by first member (R6).
#include <algorithm>
#include <array>
#include <cmath>
#include <limits>
#include <numeric>
#include <vector>

#include "internal.h"

namespace sesgd {
namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;

inline uint64_t finalize(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}

class SplitMix64 {
 public:
  explicit SplitMix64(uint64_t s) : s_(s) {}
  uint64_t operator()() { return finalize(s_ += kGolden); }
  // uniform in [0, bound): words in the incomplete top block [2^64 - (2^64 mod bound), 2^64)
  // are redrawn (R5).
  uint64_t below(uint64_t bound) {
    const uint64_t tail = (uint64_t{0} - bound) % bound;  // 2^64 mod bound
    uint64_t w = (*this)();
    if (tail != 0) {
      const uint64_t first_rejected = uint64_t{0} - tail;  // 2^64 - tail
      while (w >= first_rejected) w = (*this)();
    }
    return w % bound;
  }

 private:
  uint64_t s_;
};

}  // namespace

void shuffle_exchange_groups(uint64_t seed, int64_t t, int n, int m, int32_t *canon,
                             int32_t *group_of) {
  SplitMix64 rng(finalize(seed ^ static_cast<uint64_t>(t)));
  std::vector<int32_t> slots(n);
  std::iota(slots.begin(), slots.end(), 0);
  for (int i = n - 1; i > 0; --i) std::swap(slots[i], slots[rng.below(uint64_t(i) + 1)]);

  const int k = n / m;
  std::vector<std::vector<int32_t>> groups(k);
  for (int j = 0; j < k; ++j) {
    groups[j].assign(slots.begin() + j * m, slots.begin() + (j + 1) * m);
    std::sort(groups[j].begin(), groups[j].end());
  }
  std::sort(groups.begin(), groups.end(),
            [](const std::vector<int32_t> &a, const std::vector<int32_t> &b) { return a[0] < b[0]; });
  for (int j = 0; j < k; ++j)
    for (int r = 0; r < m; ++r) {
      canon[j * m + r] = groups[j][r];
      if (group_of) group_of[groups[j][r]] = j;
    }
}

// NEXT-3 (SESGD_OPT_SCHEDULE = 1): Stone's shuffle-exchange network as the schedule, the
// deterministic reading of "shuffle-exchange" whose first two iterations for n = 4, m = 2 are
// the paper's example {0,1},{2,3} -> {0,2},{1,3}.  n = 2^d, m = 2^p: iteration t
// exchanges index dimensions (t p + q) mod d, q < p; a group is a base worker (zero in those
// bits) OR-ed with every subset of them.  After d/p iterations of pure averaging every worker
// holds the exact global mean (hypercube all-reduce).
void dimension_exchange_groups(int64_t t, int n, int m, int32_t *canon, int32_t *group_of) {
  const int d = __builtin_ctz(unsigned(n)), p = __builtin_ctz(unsigned(m));
  unsigned mask = 0;
  for (int q = 0; q < p; ++q) mask |= 1u << int((t * p + q) % d);
  int j = 0;
  for (unsigned base = 0; base < unsigned(n); ++base) {
    if (base & mask) continue;
    int r = 0;
    unsigned sub = 0;
    do {  // subsets of mask in increasing order
      const int w = int(base | sub);
      canon[j * m + r++] = w;
      if (group_of) group_of[w] = j;
      sub = (sub - mask) & mask;
    } while (sub != 0);
    ++j;
  }
}

// Eq. 2: T = 2(n-1)(G/(n nu) + t_tau); Eq. 3 before its approximation
// (P:179-181): the same ring inside a group of m = n/k members.
void latency_model(int n, int m, double bytes, double nu, double tau, sesgd_cost *out) {
  auto ring = [&](int p, double *hs, double *sec) {
    *hs = 2.0 * double(p - 1);
    *sec = (p <= 1) ? 0.0 : *hs * (bytes / (double(p) * nu) + tau);
  };
  ring(n, &out->ring_handshakes, &out->ring_s);
  ring(m, &out->sesgd_handshakes, &out->sesgd_s);
  if (out->sesgd_s > 0.0)
    out->ratio = out->ring_s / out->sesgd_s;
  else
    out->ratio = out->ring_s > 0.0 ? std::numeric_limits<double>::infinity() : 1.0;
}

}  // namespace sesgd
