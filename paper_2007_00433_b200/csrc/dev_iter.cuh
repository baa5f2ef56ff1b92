// dev_iter.cuh -- the kernels' side of the device-resident iteration state (SESGD_OPT_DEVICE_ITER,
// iter.cu).  A launch in that mode carries only its static arguments; thread 0 of every CTA copies
// them to shared memory and patches the per-launch fields (call history, parity, sequence number,
// chunk-claim base) and the iteration's schedule from the device state, so a captured CUDA graph
// replays correctly for every iteration.  The LAST CTA of the launch to finish advances the state
// (every CTA read it before finishing), and stream order hands it to the next launch.
#pragma once
#include "internal.h"

namespace sesgd {
namespace devit {

// the launch's arguments in shared memory with the per-call fields from the state: every thread of
// the CTA copies a part (8-byte words: the parameter block is only 8-byte aligned), then patches a part (scalars: thread 0; the schedule
// tables: one thread per entry); the caller's __syncthreads() publishes the result
__device__ __forceinline__ void load_patched(const P2PArgs &a, P2PArgs &s) {
  static_assert(sizeof(P2PArgs) % 8 == 0 && alignof(P2PArgs) == 8, "8-byte copy of the arguments");
  const int2 *src = reinterpret_cast<const int2 *>(&a);
  int2 *dst = reinterpret_cast<int2 *>(&s);
  for (int i = threadIdx.x; i < int(sizeof(P2PArgs) / 8); i += blockDim.x) dst[i] = src[i];
  __syncthreads();
  const DevIter *d = a.dev;
  const int i = threadIdx.x;
  if (i == 0) {
    const DevBucket B = a.dev_buckets[a.bucket >= 0 ? a.bucket : 0];  // an all-bucket launch: one history
    s.call = B.calls;
    s.parity = int(B.calls & 1);
    s.seq = d->seq;
    s.prev2_seq = B.calls >= 2 ? B.hist[B.calls & 1] : -1;
    s.seq_epoch0 = uint64_t(s.seq) * uint64_t(a.kmax) + 1;
    s.prev2_epoch0 = B.calls >= 2 ? uint64_t(s.prev2_seq) * uint64_t(a.kmax) + 1 : 0;
    s.claim_base = d->claim_base;
  }
  if (i < a.n) {
    s.canon[i] = d->canon[i];
    s.group_of[i] = d->group_of[i];
  }
  if (i < a.r) {
    s.my_pos[i] = d->my_pos[i];
    s.slot_kind[i] = d->slot_kind[i];
  }
}

// thread 0 of every CTA, after the CTA's last access to its arguments: the last CTA advances the
// call history of the launch's buckets, the launch sequence and the chunk-claim base
__device__ __forceinline__ bool last_cta(DevIter *d) {
  __threadfence();
  return atomicAdd(&d->fin, 1u) + 1u == gridDim.x;
}
__device__ __forceinline__ void advance(DevIter *d, DevBucket *bk, int bucket, int nbuckets, int64_t seq,
                                        uint64_t claim_next) {
  for (int b = (bucket >= 0 ? bucket : 0); b < (bucket >= 0 ? bucket + 1 : nbuckets); ++b) {
    DevBucket &B = bk[b];
    B.hist[B.calls & 1] = seq;
    B.calls += 1;
  }
  d->seq = seq + 1;
  d->claim_base = claim_next;
  d->fin = 0u;
  __threadfence();
}
__device__ __forceinline__ void finish(const P2PArgs &s) {
  if (last_cta(s.dev)) advance(s.dev, s.dev_buckets, s.bucket, s.nbuckets, s.seq, s.claim_base + s.dev_claim_inc);
}
__device__ __forceinline__ void finish(const RingArgs &s, int64_t seq) {
  if (last_cta(s.dev)) advance(s.dev, s.dev_buckets, s.bucket, s.nbuckets, seq, s.dev->claim_base);
}

}  // namespace devit
}  // namespace sesgd
