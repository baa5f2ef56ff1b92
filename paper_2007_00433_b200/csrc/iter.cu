// iter.cu -- sesgd_begin_iter_device: one thread evaluates iteration t's groups on the device (the
// same schedule as the host scheduler and K10, sched_dev.cuh) into the context's device iteration
// state, with the per-local-slot tables the sync kernels take from it.  "set the same random seed
// on every worker to avoid extra message exchange": every rank runs this on its own
// GPU and derives the same partition.  Enqueued once per iteration, so a CUDA graph of
// [this, sync launches] replays every iteration with the device's t (SESGD_OPT_DEVICE_ITER).
#include "common.cuh"
#include "internal.h"
#include "sched_dev.cuh"

namespace sesgd {
namespace {

__global__ void k_iter_begin(const __grid_constant__ IterBeginArgs a, DevIter *d) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int64_t t = a.t >= 0 ? a.t : d->t + 1;
  const int n = a.n, m = a.m;
  int8_t canon[SESGD_MAX_WORKERS], group_of[SESGD_MAX_WORKERS];
  sched::slots(a.seed, t, n, m, a.schedule, canon);
  sched::canonical(canon, n, m, group_of);
  d->t = t;
  for (int i = 0; i < n; ++i) {
    d->canon[i] = canon[i];
    d->group_of[i] = group_of[i];
    d->member_slot[i] = a.slot_of[canon[i]];
  }
  for (int s = 0; s < a.n_local; ++s) {
    const int me = a.local_workers[s];
    const int8_t *G = canon + group_of[me] * m;
    bool all_local = true;
    int pos = 0;
    for (int p = 0; p < m; ++p) {
      if (G[p] == me) pos = p;
      all_local = all_local && a.worker_rank[G[p]] == a.rank;
    }
    d->my_pos[s] = int8_t(pos);
    // as launch_oneshot: the DIRECT kernels update an all-local group once, by its first member
    d->slot_kind[s] = int8_t(!a.direct || !all_local ? 0 : (G[0] == me ? 1 : 2));
    if (s == 0) {
      d->ring_pos = pos;
      for (int q = 0; q < m; ++q) d->ring_rank[q] = a.worker_rank[G[q]];
    }
  }
}

}  // namespace

cudaError_t launch_iter_begin(const IterBeginArgs &a, DevIter *d, cudaStream_t stream) {
  k_iter_begin<<<1, 32, 0, stream>>>(a, d);
  return cudaGetLastError();
}

}  // namespace sesgd
