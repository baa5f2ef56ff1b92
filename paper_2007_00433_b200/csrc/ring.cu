// ring.cu -- K5: paper-faithful Ring-AllReduce inside each SESGD group over NVLink, with a
// handshake per step and an optional injected per-hop delay (BASELINE config 4).
//
// The paper's collective (Sec. 2.2; Alg.1 line 11 "Ring-AllReduce(x_hat; G_i,t)"):
// the m members of a group form a logical ring in ascending worker id; each splits the
// payload into m slices; m-1 Scatter-Reduce steps then m-1 All-Gather steps, "in one
// handshake, each worker sends one slice to its right neighbor while receives slice from its
// left", so a group allreduce costs 2(m-1) handshakes (Eq. 2 over n workers for Ring-SGD,
// Eq. 3 over m = n/k for SESGD).  This kernel executes exactly that schedule with one
// flag handshake per step, so measured time ~ 2(m-1) (G/(m nu) + t_tau): the SESGD-vs-ring
// latency sweep of config 4 runs it with group_size m and with m = n.
//
// One worker per GPU.  Slices follow SPEC collectives.slice_bounds:
// slice s = [floor(sL/m), floor((s+1)L/m)).  CTA j of every member owns the same strip of
// every slice, so CTA j only waits on CTA j of its ring neighbour (all CTAs co-resident).
// Scatter-Reduce step t: member p sends slice (p - 1 - t) mod m: its own x_hat at t = 0, else
// (received (+) own x_hat); so slice s is "accumulated in ring order starting from member
// (s+1) mod m" and member p, adding last, holds the full sum of its own slice p after
// step m-2 and divides by m.  The ascending-fold oracle agrees bit-for-bit only for m <= 2;
// the ring-order oracle (orc_step_ring_f32) follows the same S:263 order.
// Receive buffers: one per (call parity, step), no reuse inside a launch; reuse two calls
// later is guarded by the receiver's consumed counter.  Every spin has a timeout.
#include "common.cuh"
#include "internal.h"
#include "dev_iter.cuh"

namespace sesgd {
namespace {

constexpr int kRingThreads = 256;

__device__ bool ring_wait(const RingArgs &a, const uint64_t *p, uint64_t target, int kind) {
  if (dev::ld_acquire_sys(p) >= target) return true;
  count(a.counters, kCntFlagSpins);
  const uint64_t t0 = dev::globaltimer();
  for (;;) {
    const uint64_t v = dev::ld_acquire_sys(p);
    if (v >= target) return true;
    if (*reinterpret_cast<volatile unsigned int *>(a.abort_dev)) return false;
    if (dev::globaltimer() - t0 > a.timeout_ns) {
      if (atomicExch(a.abort_dev, 1u) == 0u) {
        a.err_host[1] = (unsigned long long)kind;
        a.err_host[2] = blockIdx.x;
        a.err_host[3] = v;
        a.err_host[4] = target;
        a.err_host[7] = (unsigned long long)a.my_rank;
        __threadfence_system();
        atomicExch(a.err_host, (unsigned long long)(-SESGD_ETIMEOUT));
      }
      return false;
    }
  }
}

// the per-call fields (call history, this member's ring) -- the launch's arguments, or (device
// iteration state) the context's device memory: read by every thread, no shared-memory copy, so
// the kernel keeps the resource footprint of the plain one (a loopback virtual rank's grid must fit
// next to its peers' exactly; a different footprint broke that co-residency)
struct RingCall {
  int64_t call, seq;
  int parity, pos;
  const int8_t *ring;  // rank of ring position q
};

template <bool GRAD>
struct Ring {
  const RingArgs &a;
  const int64_t call;
  const int parity, pos;
  const int8_t *ring;
  __device__ Ring(const RingArgs &args, const RingCall &c)
      : a(args), call(c.call), parity(c.parity), pos(c.pos), ring(c.ring) {}

  __device__ __forceinline__ int rank_at(int q) const { return ring[(q % a.m + a.m) % a.m]; }
  __device__ __forceinline__ int64_t slice_lo(int s) const { return int64_t(s) * a.numel / a.m; }
  // this CTA's strip [lo, hi) of slice s (vector-aligned strips; the last CTA takes the rest)
  __device__ __forceinline__ void strip(int s, int64_t &lo, int64_t &hi) const {
    const int64_t s0 = slice_lo(s), s1 = slice_lo(s + 1);
    const int64_t per = ((s1 - s0 + a.grid - 1) / a.grid + 3) & ~int64_t(3);
    lo = min(s0 + int64_t(blockIdx.x) * per, s1);
    hi = min(lo + per, s1);
  }
  __device__ __forceinline__ float *rbuf(int rank, int step) const {  // rank's receive buffer
    return reinterpret_cast<float *>(a.ws[rank] + a.rbuf_off) +
           (int64_t(parity) * a.steps + step) * a.slice_cap;
  }
  __device__ __forceinline__ uint64_t *flag(int rank, int step) const {
    return reinterpret_cast<uint64_t *>(a.ws[rank] + a.rflag_off) +
           ((int64_t(parity) * a.nbuckets + a.bucket) * a.steps + step) * a.grid + blockIdx.x;
  }
  __device__ __forceinline__ uint64_t *consumed(int rank) const {
    return reinterpret_cast<uint64_t *>(a.ws[rank] + a.rcons_off) + int64_t(a.bucket) * a.grid + blockIdx.x;
  }

  // local step on [lo, hi): returns the payload value (x_hat, or g in GRAD mode) via f(e, val)
  template <typename F>
  __device__ __forceinline__ void local(int64_t lo, int64_t hi, F &&f) const {
    for (int64_t e = lo + threadIdx.x; e < hi; e += kRingThreads) {
      const float g = __ldcs(a.g + e);
      if constexpr (!GRAD) {
        const float v = dev::momentum(a.mu, a.v[e], dev::decay(g, a.wd, a.x[e]));
        a.v[e] = v;
        f(e, dev::sgd(a.x[e], a.lr, v));
      } else {
        f(e, g);
      }
    }
  }
  // write the group mean of slice range [lo, hi) held in `src` (offset by the slice start)
  __device__ __forceinline__ void apply_mean(int64_t lo, int64_t hi, const float *src, int64_t base) const {
    for (int64_t e = lo + threadIdx.x; e < hi; e += kRingThreads) {
      const float mean = src[e - base];
      if constexpr (!GRAD) {
        a.x[e] = mean;
      } else {
        const float v = dev::momentum(a.mu, a.v[e], dev::decay(mean, a.wd, a.x[e]));
        a.v[e] = v;
        a.x[e] = dev::sgd(a.x[e], a.lr, v);
      }
    }
  }
  __device__ __forceinline__ void signal(int step) const {
    __syncthreads();  // every push of this step precedes the flag (cumulativity)
    if (threadIdx.x == 0) {
      if (a.hop_delay_ns) {  // injected per-hop latency t_tau (config 4)
        const uint64_t t0 = dev::globaltimer();
        while (dev::globaltimer() - t0 < a.hop_delay_ns) {
        }
      }
      dev::st_release_sys(flag(rank_at(pos + 1), step), uint64_t(call) + 1);
      count(a.counters, kCntFlagStores);
    }
  }
  __device__ __forceinline__ void await(int step) const {
    if (threadIdx.x == 0) ring_wait(a, flag(a.my_rank, step), uint64_t(call) + 1, 2);
    __syncthreads();
  }

  __device__ void run() const {
    const int m = a.m, p = pos;
    const int next = rank_at(p + 1);
    if (call >= 2 && threadIdx.x == 0)  // next member consumed its call-2 buffers
      ring_wait(a, consumed(next), uint64_t(call) - 1, 1);
    __syncthreads();
    // ---- Scatter-Reduce: m - 1 steps
    for (int t = 0; t < m - 1; ++t) {
      const int s = ((p - 1 - t) % m + m) % m;
      int64_t lo, hi;
      strip(s, lo, hi);
      const int64_t base = slice_lo(s);
      float *out = rbuf(next, t);  // next member's receive buffer of step t
      if (t == 0) {
        local(lo, hi, [&](int64_t e, float xh) { out[e - base] = xh; });
      } else {
        await(t - 1);
        const float *in = rbuf(a.my_rank, t - 1);
        local(lo, hi, [&](int64_t e, float xh) { out[e - base] = __fadd_rn(in[e - base], xh); });
      }
      signal(t);
    }
    // the full sum of my own slice p arrives at the last scatter step
    const int sf = p;
    int64_t lo, hi;
    strip(sf, lo, hi);
    int64_t base = slice_lo(sf);
    await(m - 2);
    {
      const float *in = rbuf(a.my_rank, m - 2);
      float *out = rbuf(next, m - 1);  // All-Gather step 0 sends the mean of slice sf
      for (int64_t e = lo + threadIdx.x; e < hi; e += kRingThreads) {
        const float g = __ldcs(a.g + e);
        if constexpr (!GRAD) {
          const float v = dev::momentum(a.mu, a.v[e], dev::decay(g, a.wd, a.x[e]));
          a.v[e] = v;
          const float mean = __fdiv_rn(__fadd_rn(in[e - base], dev::sgd(a.x[e], a.lr, v)), float(m));
          out[e - base] = mean;
          a.x[e] = mean;  // my own copy of the mean of slice sf
        } else {
          const float mean = __fdiv_rn(__fadd_rn(in[e - base], g), float(m));
          out[e - base] = mean;
          const float v = dev::momentum(a.mu, a.v[e], dev::decay(mean, a.wd, a.x[e]));
          a.v[e] = v;
          a.x[e] = dev::sgd(a.x[e], a.lr, v);
        }
      }
    }
    signal(m - 1);
    // ---- All-Gather: m - 1 steps (step index m - 1 + u)
    for (int u = 0; u < m - 1; ++u) {
      const int s = ((p - 1 - u) % m + m) % m;  // slice received at this step
      strip(s, lo, hi);
      base = slice_lo(s);
      await(m - 1 + u);
      const float *in = rbuf(a.my_rank, m - 1 + u);
      if (u < m - 2) {  // forward it
        float *out = rbuf(next, m + u);
        for (int64_t e = lo + threadIdx.x; e < hi; e += kRingThreads) out[e - base] = in[e - base];
        signal(m + u);
      }
      apply_mean(lo, hi, in, base);
    }
    __syncthreads();  // every read of my receive buffers is done
    if (threadIdx.x == 0) dev::st_release_sys(consumed(a.my_rank), uint64_t(call) + 1);
  }

  __device__ void local_only() const {
    for (int64_t e = int64_t(blockIdx.x) * kRingThreads + threadIdx.x; e < a.numel;
         e += int64_t(a.grid) * kRingThreads) {
      const float v = dev::momentum(a.mu, a.v[e], dev::decay(a.g[e], a.wd, a.x[e]));
      a.v[e] = v;
      a.x[e] = dev::sgd(a.x[e], a.lr, v);
    }
  }
};

template <bool GRAD>
__global__ void __launch_bounds__(kRingThreads) k5_ring(const __grid_constant__ RingArgs a) {
  const Ring<GRAD> r(a, RingCall{a.call, a.seq, a.parity, a.pos, a.ring_rank});
  if (blockIdx.x == 0 && threadIdx.x == 0) count(a.counters, kCntLaunches);
  if (a.m == 1)
    r.local_only();
  else
    r.run();
}

// device-resident iteration state (SESGD_OPT_DEVICE_ITER, dev_iter.cuh)
__device__ __forceinline__ RingCall ring_call_dev(const RingArgs &a) {
  const DevIter *d = a.dev;
  const DevBucket B = a.dev_buckets[a.bucket];
  return RingCall{B.calls, d->seq, int(B.calls & 1), d->ring_pos, d->ring_rank};
}

template <bool GRAD>
__global__ void __launch_bounds__(kRingThreads, 5) k5_ring_dev(const __grid_constant__ RingArgs a) {
  const RingCall c = ring_call_dev(a);
  const Ring<GRAD> r(a, c);
  if (blockIdx.x == 0 && threadIdx.x == 0) count(a.counters, kCntLaunches);
  if (a.m == 1)
    r.local_only();
  else
    r.run();
  __syncthreads();
  if (threadIdx.x == 0) devit::finish(a, c.seq);
}

const void *pick(int mode, bool devi = false) {
  if (devi)
    return mode == SESGD_MODE_GRAD_AVG ? reinterpret_cast<const void *>(&k5_ring_dev<true>)
                                       : reinterpret_cast<const void *>(&k5_ring_dev<false>);
  return mode == SESGD_MODE_GRAD_AVG ? reinterpret_cast<const void *>(&k5_ring<true>)
                                     : reinterpret_cast<const void *>(&k5_ring<false>);
}

}  // namespace

int ring_block_threads() { return kRingThreads; }

int ring_occupancy(int mode) {
  int blocks = 0, bd = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, pick(mode), kRingThreads, 0) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bd, pick(mode, true), kRingThreads, 0) != cudaSuccess)
    return 1;
  blocks = bd < blocks ? bd : blocks;
  return blocks > 0 ? blocks : 1;
}

cudaError_t launch_ring(const RingArgs &a, int mode, cudaStream_t stream) {
  void *args[] = {const_cast<RingArgs *>(&a)};
  return launch_persistent(pick(mode, a.dev != nullptr), unsigned(a.grid), kRingThreads, args, 0, stream, a.cooperative != 0);
}

}  // namespace sesgd
