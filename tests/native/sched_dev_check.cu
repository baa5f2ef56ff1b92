// Host-compiled check (tests/test_sched_dev.py): the device schedule of sched_dev.cuh (K10 and
// sesgd_begin_iter_device's K11) equals the host scheduler of schedule.cpp (pinned against the
// oracle by tests/test_boundary.py) for every n <= 64, every m | n, both schedules, 300 t each.
#include <cstdio>

#include "../../paper_2007_00433_b200/csrc/internal.h"
#include "../../paper_2007_00433_b200/csrc/sched_dev.cuh"

int main() {
  long cases = 0, bad = 0;
  for (int n = 1; n <= 64; ++n)
    for (int m = 1; m <= n; ++m) {
      if (n % m) continue;
      for (int sch = 0; sch < 2; ++sch) {
        if (sch == 1 && ((n & (n - 1)) || (m & (m - 1)))) continue;
        for (long t = 0; t < 300; ++t) {
          const uint64_t seed = 42ull ^ (uint64_t(t) * 0x9E3779B97F4A7C15ull);
          const int64_t tt = t * 7919 + (t & 1) * (int64_t(1) << 40);
          int8_t sl[64], gof[64];
          int32_t c[64], g[64];
          sesgd::sched::slots(seed, tt, n, m, sch, sl);
          sesgd::sched::canonical(sl, n, m, gof);
          if (sch)
            sesgd::dimension_exchange_groups(tt, n, m, c, g);
          else
            sesgd::shuffle_exchange_groups(seed, tt, n, m, c, g);
          ++cases;
          for (int i = 0; i < n; ++i)
            if (sl[i] != c[i] || gof[i] != g[i]) {
              ++bad;
              break;
            }
        }
      }
    }
  std::printf("cases=%ld bad=%ld\n", cases, bad);
  return bad != 0;
}
