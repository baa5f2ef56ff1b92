// p2p.cu -- the multi-GPU kernels: fused local update + intra-group exchange over NVLink,
// one persistent kernel over a range of chunks (one bucket, or every bucket of the
// iteration at once with sesgd_sync_all):
//   K4 k4_twoshot (default, "K4 TWO-SHOT" below): reduce-scatter + all-gather pushes, every
//      member owns a slice of each chunk; variants with TMA bulk pushes, several workers per
//      GPU (MULTI) and NVLink SHARP (NV: multimem.ld_reduce / multimem.st);
//   K3 k3_direct: one-shot push from every CTA (DIRECT, below);
//   K3 k3_split: SM-specialised one-shot, a few COMM CTAs move data over NVLink while the
//      COMPUTE CTAs stream HBM (described in this header).
//
// Each iteration every group G = {a_0 < ... < a_{m-1}} of the shuffle-exchange
// partition (A1) averages its members' locally-stepped parameters (Eq. 6,
// P:204-207; Alg.1 line 11 "Ring-AllReduce(x_hat; G)").  The paper's ring over
// Ethernet is prior art: on NVSwitch every peer is one hop at full bandwidth, so one
// handshake round suffices (instead of the ring's 2(m-1)).
//
// Why this shape (measured on B200; profiles/r01_nvlink_probe_2gpu*.json,
// profiles/r01_k3_phases*.json):
//  * remote loads hold an SM's request slots for ~2.5 us and starve a local HBM
//    stream; remote STORES do not, and both-direction push keeps 705 GB/s/dir;
//  * 32 CTAs of pushes reach 698 GB/s/dir and leave the other SMs free to stream
//    HBM concurrently; pushing from >= 64 CTAs starves the local stream;
//  * a system-scope release stalls until the CTA's remote stores drain, so flags
//    are released once per COMM batch of chunks;
//  * every launch pays a pipeline fill and drain, so one launch covers as many
//    chunks as possible (all buckets of the iteration with sesgd_sync_all).
//
// Chunks (4096 floats) are numbered globally over the concatenated buckets; a launch
// covers [g0, g1).  Roles (blockIdx < Q: COMM, else COMPUTE; all CTAs co-resident):
//  COMPUTE CTA i (i = g mod Gc for its chunks g):
//    stage(g):  load g, v, x ; v <- mu v + g ; x_hat <- x - lr v ; store v ;
//               x_hat -> own stage (L2) ; staged[s][i] = S(seq, g)
//               (GRAD: g -> stage; v and x are updated at fold time)
//    fold(g)  `lag` chunk steps later: wait sent[s][g] (own COMM pushed it) and the
//               ready flags of remote members ; fold the m contributions in ascending
//               position (= ascending worker id): own / co-resident members from
//               their stages, remote members from the receive slots ; (/) m ; store x ;
//               discard the dead lines from L2
//    end:       consumed[s][i] = S(seq, last g)  (one system-scope release per launch)
//  COMM CTA q, batches of B chunks (batch j = q, q+Q, ...):
//    guard: every remote member consumed its receive slot of the call two back
//               (consumed counters bulk-read once per launch into shared memory)
//    wait staged ; copy own stage -> remote members' receive slots (NVLink stores) ;
//    one st.release.sys per (chunk, remote member) ready flag ; sent flags
// S(seq, g) = seq * KMAX + floor(g / Gc) + 1 is strictly increasing in every compute
// CTA's processing order across launches; ready / sent flags hold the bucket's call
// index + 1, with ready and receive slots double-buffered by call parity.  All waits
// point to a strictly smaller chunk (or an earlier step of the same chunk), so the
// smallest unfinished step can always progress: no deadlock.  Flags are never reset.
// Every spin has a %globaltimer timeout that latches SESGD_ETIMEOUT.
#include <cuda_bf16.h>

#include "common.cuh"
#include "internal.h"

namespace sesgd {
namespace {

constexpr int kThreads = 256;
constexpr int kVec = 4;                                   // float4 items per thread per chunk
constexpr int64_t kChunk = int64_t(kThreads) * 4 * kVec;  // 4096 floats = 16 KiB
constexpr int kMaxGuardPairs = 8;                         // (slot, remote member) pairs cached in smem
constexpr int kRing = 3;                                  // COMM TMA ring: chunks in flight
constexpr int kRingBytes = kRing * int(kChunk) * 4;       // 48 KiB

// ---- element access with a per-component mask on the ragged last vector ----
template <int W>
__device__ __forceinline__ void load_m(const float *p, float (&r)[W], int nvalid) {
  if constexpr (W == 4) {
    if (nvalid >= 4) {
      float4 t = dev::ld4(p);
      r[0] = t.x; r[1] = t.y; r[2] = t.z; r[3] = t.w;
    } else {
#pragma unroll
      for (int w = 0; w < 4; ++w) r[w] = (w < nvalid) ? p[w] : 0.f;
    }
  } else {
    r[0] = __ldcs(p);
  }
}
template <int W>
__device__ __forceinline__ void store_m(float *p, const float (&r)[W], int nvalid) {
  if constexpr (W == 4) {
    if (nvalid >= 4) {
      dev::st4(p, make_float4(r[0], r[1], r[2], r[3]));
    } else {
#pragma unroll
      for (int w = 0; w < 4; ++w)
        if (w < nvalid) p[w] = r[w];
    }
  } else {
    __stcs(p, r[0]);
  }
}
// stage / receive slots: default (L2-allocating) policy, they are read back soon
template <int W>
__device__ __forceinline__ void st_slot(float *p, const float (&r)[W], int nvalid) {
  if constexpr (W == 4) {
    if (nvalid >= 4) {
      *reinterpret_cast<float4 *>(p) = make_float4(r[0], r[1], r[2], r[3]);
    } else {
#pragma unroll
      for (int w = 0; w < 4; ++w)
        if (w < nvalid) p[w] = r[w];
    }
  } else {
    *p = r[0];
  }
}
template <int W>
__device__ __forceinline__ void ld_slot(const float *p, float (&r)[W], int nvalid) {
  if constexpr (W == 4) {
    if (nvalid >= 4) {
      float4 t = __ldcg(reinterpret_cast<const float4 *>(p));
      r[0] = t.x; r[1] = t.y; r[2] = t.z; r[3] = t.w;
    } else {
#pragma unroll
      for (int w = 0; w < 4; ++w) r[w] = (w < nvalid) ? __ldcg(p + w) : 0.f;
    }
  } else {
    r[0] = __ldcg(p);
  }
}

// invalidate a 128-byte L2 line without writing it back (its contents are dead)
__device__ __forceinline__ void discard_l2(const void *p) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}
__device__ __forceinline__ void st_release_gpu(uint64_t *p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// NVLS (NVLink SHARP): loads that the NVSwitch reduces over every GPU's copy of a multicast
// address, and stores it replicates to every GPU (sm_90+ multimem)
__device__ __forceinline__ void mm_ld_reduce4(const float *mc, float (&r)[4]) {
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3])
               : "l"(mc)
               : "memory");
}
__device__ __forceinline__ float mm_ld_reduce1(const float *mc) {
  float r;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(r) : "l"(mc) : "memory");
  return r;
}
__device__ __forceinline__ void mm_st4(float *mc, const float (&r)[4]) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc), "f"(r[0]),
               "f"(r[1]), "f"(r[2]), "f"(r[3])
               : "memory");
}
__device__ __forceinline__ void mm_st1(float *mc, float r) {
  asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(mc), "f"(r) : "memory");
}
// the same memory is accessed through the multicast and the unicast mappings
__device__ __forceinline__ void fence_proxy_alias() { asm volatile("fence.proxy.alias;" ::: "memory"); }

// bf16 payload (SESGD_OPT_PAYLOAD_BF16): a slice's reduce-scatter values travel as bf16, packed in
// the first half of that slice's own float range, so they never overlap the fp32 all-gather data
// that other slices receive in the same slot.  Round to nearest even, as __float2bfloat16_rn.
template <int W>
__device__ __forceinline__ void st_bf(__nv_bfloat16 *p, const float (&r)[W], int nvalid) {
  if constexpr (W == 4) {
    if (nvalid == 4) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(r[0], r[1]), hi = __floats2bfloat162_rn(r[2], r[3]);
      uint2 u;
      u.x = *reinterpret_cast<unsigned int *>(&lo);
      u.y = *reinterpret_cast<unsigned int *>(&hi);
      *reinterpret_cast<uint2 *>(p) = u;
      return;
    }
  }
  for (int q = 0; q < W; ++q)
    if (q < nvalid) p[q] = __float2bfloat16_rn(r[q]);
}
template <int W>
__device__ __forceinline__ void ld_bf(const __nv_bfloat16 *p, float (&r)[W], int nvalid) {
  if constexpr (W == 4) {
    if (nvalid == 4) {
      const uint2 u = __ldcg(reinterpret_cast<const uint2 *>(p));
      const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&u.x));
      const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&u.y));
      r[0] = a.x; r[1] = a.y; r[2] = b.x; r[3] = b.y;
      return;
    }
  }
  for (int q = 0; q < W; ++q) r[q] = (q < nvalid) ? __bfloat162float(p[q]) : 0.f;
}

__device__ __forceinline__ void st_relaxed_sys(uint64_t *p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// what a timed-out wait was waiting for (reported through sesgd_last_error)
enum WaitKind : int { kWaitConsumed = 1, kWaitReady = 2, kWaitStaged = 3, kWaitSent = 4, kWaitData = 6 };

// ---- value-carried validity (SESGD_OPT_PROTOCOL = 1): a receive slot float holds kSentinel until
// the peer's value lands.  A 32-bit aligned access is single-copy atomic (PTX memory model), so a
// float is either the sentinel or the whole new value: the receiver polls the data itself and the
// sender needs no fence and no flag.  kSentinel is a NaN bit pattern GPU arithmetic never produces
// (canonical NaN is 0x7FFFFFFF); a payload equal to it is sent as the canonical NaN.  After reading,
// the receiver re-arms the float with kSentinel; the per-launch `consumed` release orders those
// re-arms before the peer's next use of the slot (two calls later).
constexpr uint32_t kSentinel = 0xFFFFFFFFu;
__device__ __forceinline__ float unsentinel(float v) {
  return __float_as_uint(v) == kSentinel ? __uint_as_float(0x7FFFFFFFu) : v;
}
template <int W>
__device__ __forceinline__ void st_sent(float *p, const float (&r)[W], int nvalid) {
  if constexpr (W == 4) {
    if (nvalid >= 4) {
      asm volatile("st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(unsentinel(r[0])),
                   "f"(unsentinel(r[1])), "f"(unsentinel(r[2])), "f"(unsentinel(r[3]))
                   : "memory");
      return;
    }
  }
  for (int w = 0; w < W; ++w)
    if (w < nvalid) asm volatile("st.relaxed.sys.global.f32 [%0], %1;" ::"l"(p + w), "f"(unsentinel(r[w])) : "memory");
}
__device__ __forceinline__ float ld_relaxed1(const float *p) {
  float v;
  asm volatile("ld.relaxed.sys.global.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void ld_relaxed4(const float *p, float (&r)[4]) {
  asm volatile("ld.relaxed.sys.global.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3])
               : "l"(p)
               : "memory");
}
template <int W>
__device__ __forceinline__ void rearm(float *p, int nvalid) {
  const float s = __uint_as_float(kSentinel);
  if constexpr (W == 4) {
    if (nvalid >= 4) {
      *reinterpret_cast<float4 *>(p) = make_float4(s, s, s, s);
      return;
    }
  }
  for (int w = 0; w < W; ++w)
    if (w < nvalid) p[w] = s;
}

// spin until *p >= target (sys-scope acquire); on timeout the first CTA to give up
// latches SESGD_ETIMEOUT plus a description of the flag in the host-mapped block
__device__ uint64_t wait_geq(const P2PArgs &a, const uint64_t *p, uint64_t target, int kind,
                             int worker, int pos) {
  uint64_t v = dev::ld_acquire_sys(p);
  if (v >= target) return v;
  count(a.counters, kCntFlagSpins);
  const uint64_t t0 = dev::globaltimer();
  for (;;) {
    v = dev::ld_acquire_sys(p);
    if (v >= target) return v;
    if (*reinterpret_cast<volatile unsigned int *>(a.abort_dev)) return target;
    if (dev::globaltimer() - t0 > a.timeout_ns) {
      if (atomicExch(a.abort_dev, 1u) == 0u) {
        unsigned long long *e = a.err_host;
        e[1] = (unsigned long long)kind;
        e[2] = blockIdx.x;
        e[3] = v;
        e[4] = target;
        e[5] = (unsigned long long)worker;
        e[6] = (unsigned long long)pos;
        e[7] = (unsigned long long)a.my_rank;
        __threadfence_system();
        atomicExch(e, (unsigned long long)(-SESGD_ETIMEOUT));
        __threadfence_system();
      }
      return target;
    }
  }
}

// poll `nvalid` floats at p until none is the sentinel (timeout latches SESGD_ETIMEOUT), then re-arm
template <int W>
__device__ __forceinline__ void ld_poll(const P2PArgs &a, float *p, float (&r)[W], int nvalid, int worker,
                                        int pos) {
  auto pending = [&]() {
    bool any = false;
#pragma unroll
    for (int w = 0; w < W; ++w) any |= (w < nvalid) && __float_as_uint(r[w]) == kSentinel;
    return any;
  };
  auto load = [&]() {
    if constexpr (W == 4) {
      if (nvalid >= 4) {
        ld_relaxed4(p, r);
        return;
      }
    }
#pragma unroll
    for (int w = 0; w < W; ++w) r[w] = (w < nvalid) ? ld_relaxed1(p + w) : 0.f;
  };
  load();
  if (pending()) {
    count(a.counters, kCntValueSpins);
    const uint64_t t0 = dev::globaltimer();
    do {
      if (*reinterpret_cast<volatile unsigned int *>(a.abort_dev)) break;
      if (dev::globaltimer() - t0 > a.timeout_ns) {
        if (atomicExch(a.abort_dev, 1u) == 0u) {
          unsigned long long *e = a.err_host;
          e[1] = (unsigned long long)kWaitData;
          e[2] = blockIdx.x;
          e[3] = 0;
          e[4] = uint64_t(a.call) + 1;
          e[5] = (unsigned long long)worker;
          e[6] = (unsigned long long)pos;
          e[7] = (unsigned long long)a.my_rank;
          __threadfence_system();
          atomicExch(e, (unsigned long long)(-SESGD_ETIMEOUT));
          __threadfence_system();
        }
        break;
      }
      load();
    } while (pending());
  }
  rearm<W>(p, nvalid);
}

__device__ __forceinline__ void hop_delay(const P2PArgs &a) {
  if (a.hop_delay_ns == 0) return;
  const uint64_t t0 = dev::globaltimer();
  while (dev::globaltimer() - t0 < a.hop_delay_ns) {
  }
}

struct ChunkRef {
  int b;           // bucket
  int64_t e0, e1;  // element range inside the bucket
  int64_t soff;    // float offset of the bucket inside a stage / receive region
};

template <int W, bool GRAD>
struct Split {
  static constexpr int kItems = int(kChunk / W) / kThreads;  // W-wide items per thread per chunk

  const P2PArgs &a;
  int gc;  // compute CTAs
  __device__ explicit Split(const P2PArgs &args) : a(args) { gc = a.grid - a.comm_ctas; }

  // ---- chunk -> bucket ----
  __device__ __forceinline__ ChunkRef locate(int64_t g) const {
    int b = a.bucket;
    if (b < 0) {  // multi-bucket launch: last bucket whose chunk_base <= g
      int lo = 0, hi = a.nbuckets - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (a.meta[mid].chunk_base <= g) lo = mid; else hi = mid - 1;
      }
      b = lo;
    }
    SESGD_CHECK(b >= 0 && b < a.nbuckets && g >= a.g0 && g < a.g1);
    const BucketMeta &mb = a.meta[b];
    ChunkRef c;
    c.b = b;
    c.e0 = (g - mb.chunk_base) * kChunk;
    c.e1 = min(c.e0 + kChunk, mb.numel);
    c.soff = mb.stage_off;
    return c;
  }

  // ---- addressing (workspace layout: see sesgd_capi.cu freeze_layout) ----
  __device__ __forceinline__ const int8_t *group(int me) const {
    return a.canon + a.group_of[me] * a.m;
  }
  __device__ __forceinline__ bool remote(int w) const { return a.worker_rank[w] != a.my_rank; }
  __device__ __forceinline__ float *stage(int slot) const {  // my rank's stage of a local slot
    SESGD_CHECK(slot >= 0 && slot < a.r);
    return reinterpret_cast<float *>(a.ws[a.my_rank] + a.stage_off) + int64_t(slot) * a.region_floats;
  }
  __device__ __forceinline__ float *recv(int worker, int pos) const {  // worker's receive slot
    SESGD_CHECK(worker >= 0 && worker < a.n && pos >= 0 && pos < a.m);
    SESGD_CHECK(a.worker_slot[worker] >= 0 && a.worker_slot[worker] < a.r);
    char *base = a.ws[(a.experiment & 2) ? a.my_rank : a.worker_rank[worker]] + a.recv_off;
    const int64_t region = (int64_t(a.parity) * a.r + a.worker_slot[worker]) * a.m + pos;
    return reinterpret_cast<float *>(base) + region * a.region_floats;
  }
  __device__ __forceinline__ uint64_t *ready(int worker, int64_t g, int pos) const {
    uint64_t *f = reinterpret_cast<uint64_t *>(a.ws[a.worker_rank[worker]] + a.ready_off);
    return f + ((int64_t(a.parity) * a.r + a.worker_slot[worker]) * a.total_chunks + g) * a.m + pos;
  }
  __device__ __forceinline__ uint64_t *sent(int s, int64_t g) const {
    return reinterpret_cast<uint64_t *>(a.ws[a.my_rank] + a.sent_off) + int64_t(s) * a.total_chunks + g;
  }
  __device__ __forceinline__ uint64_t *staged(int s, int i) const {
    return reinterpret_cast<uint64_t *>(a.ws[a.my_rank] + a.staged_off) + int64_t(s) * gc + i;
  }
  __device__ __forceinline__ uint64_t *consumed(int worker, int i) const {
    return reinterpret_cast<uint64_t *>(a.ws[a.worker_rank[worker]] + a.consumed_off) +
           int64_t(a.worker_slot[worker]) * gc + i;
  }
  __device__ __forceinline__ uint64_t step_epoch(uint64_t base, int64_t g) const {
    return base + uint64_t(g / gc);
  }
  // the pi-th (slot, remote member) pair of this rank's groups
  __device__ __forceinline__ int remote_pair_member(int pi) const {
    int seen = -1;
    for (int p = 0; p < a.r * a.m; ++p) {
      const int s = p / a.m, rr = p % a.m;
      const int me = a.my_workers[s];
      const int w = group(me)[rr];
      if (w != me && remote(w) && ++seen == pi) return w;
    }
    return -1;
  }

  // ---------------------------------------------------------------- COMPUTE
  __device__ void stage_chunk(int i, int64_t g) const {
    const ChunkRef c = locate(g);
    for (int s = 0; s < a.r; ++s) {
      float *xs = a.bx[c.b * a.r + s], *vs = a.bv[c.b * a.r + s];
      const float *gs = a.bg[c.b * a.r + s];
      float *st = stage(s) + c.soff;
#pragma unroll
      for (int it = 0; it < kItems; ++it) {
        const int64_t e = c.e0 + (int64_t(it) * kThreads + threadIdx.x) * W;
        const int nv = (int)min(int64_t(W), c.e1 - e);
        if (nv <= 0) continue;
        float gr[W];
        load_m<W>(gs + e, gr, nv);
        if constexpr (!GRAD) {
          float v[W], x[W];
          load_m<W>(vs + e, v, nv);
          load_m<W>(xs + e, x, nv);
#pragma unroll
          for (int q = 0; q < W; ++q) {
            v[q] = dev::momentum(a.mu, v[q], dev::decay(gr[q], a.wd, x[q]));
            x[q] = dev::sgd(x[q], a.lr, v[q]);  // x_hat
          }
          store_m<W>(vs + e, v, nv);
          st_slot<W>(st + e, x, nv);
        } else {
          st_slot<W>(st + e, gr, nv);
        }
      }
    }
    __syncthreads();  // every stage store of chunk g precedes the release
    if (threadIdx.x < a.r) st_release_gpu(staged(threadIdx.x, i), step_epoch(a.seq_epoch0, g));
  }

  __device__ void fold_chunk(int i, int64_t g) const {
    const ChunkRef c = locate(g);
    const uint64_t call = uint64_t(a.call) + 1;
    // warp 0: my COMM pushed chunk g of every slot, and every remote member's chunk arrived
    if (threadIdx.x < 32) {
      const int pairs = a.r * a.m;
      for (int p = threadIdx.x; p < pairs; p += 32) {
        const int s = p / a.m, rr = p % a.m;
        const int me = a.my_workers[s];
        const int w = group(me)[rr];
        if (w == me)
          wait_geq(a, sent(s, g), call, kWaitSent, me, rr);
        else if (remote(w))
          wait_geq(a, ready(me, g, rr), call, kWaitReady, me, rr);
      }
    }
    __syncthreads();
    for (int s = 0; s < a.r; ++s) {
      const int me = a.my_workers[s];
      const int8_t *G = group(me);
      float *xs = a.bx[c.b * a.r + s], *vs = a.bv[c.b * a.r + s];
#pragma unroll
      for (int it = 0; it < kItems; ++it) {
        const int64_t e = c.e0 + (int64_t(it) * kThreads + threadIdx.x) * W;
        const int nv = (int)min(int64_t(W), c.e1 - e);
        if (nv <= 0) continue;
        float acc[W];
        for (int rr = 0; rr < a.m; ++rr) {  // ascending position = ascending worker id
          const int w = G[rr];
          const float *src = remote(w) ? recv(me, rr) : stage(a.worker_slot[w]);
          float y[W];
          ld_slot<W>(src + c.soff + e, y, nv);
#pragma unroll
          for (int q = 0; q < W; ++q) acc[q] = (rr == 0) ? y[q] : __fadd_rn(acc[q], y[q]);
        }
#pragma unroll
        for (int q = 0; q < W; ++q) acc[q] = __fdiv_rn(acc[q], (float)a.m);
        if constexpr (!GRAD) {
          store_m<W>(xs + e, acc, nv);
        } else {
          float v[W], x[W];
          load_m<W>(vs + e, v, nv);
          load_m<W>(xs + e, x, nv);
#pragma unroll
          for (int q = 0; q < W; ++q) {
            v[q] = dev::momentum(a.mu, v[q], dev::decay(acc[q], a.wd, x[q]));
            x[q] = dev::sgd(x[q], a.lr, v[q]);
          }
          store_m<W>(vs + e, v, nv);
          store_m<W>(xs + e, x, nv);
        }
      }
    }
    __syncthreads();  // every slot's fold has read the co-resident stages
    // The stage and receive lines of chunk g are dead: drop them from L2 without
    // write-back (a discard is a write, so it precedes the `consumed` release below).
    if constexpr (W == 4) {
      if (a.discard && (threadIdx.x & 7) == 0) {
        for (int s = 0; s < a.r; ++s) {
          const int me = a.my_workers[s];
          const int8_t *G = group(me);
#pragma unroll
          for (int it = 0; it < kItems; ++it) {
            const int64_t e = c.e0 + (int64_t(it) * kThreads + threadIdx.x) * W;
            if (e + 32 > c.e1) continue;
            discard_l2(stage(s) + c.soff + e);
            for (int rr = 0; rr < a.m; ++rr)
              if (remote(G[rr])) discard_l2(recv(me, rr) + c.soff + e);
          }
        }
      }
    }
    __syncthreads();  // this chunk's reads and discards precede the next stage / final release
  }

  __device__ void compute(int i) const {
    // my chunks: g = first, first + gc, ... in [g0, g1)
    const int64_t first = a.g0 + ((int64_t(i) - a.g0 % gc) % gc + gc) % gc;
    const int64_t nk = (a.g1 > first) ? (a.g1 - first + gc - 1) / gc : 0;
    uint64_t t_stage = 0, t_fold = 0, t0 = a.prof ? dev::globaltimer() : 0, tstart = t0;
    for (int64_t k = 0; k < nk + a.lag; ++k) {
      if (k < nk) stage_chunk(i, first + k * gc);
      if (a.prof) {
        const uint64_t t1 = dev::globaltimer();
        t_stage += t1 - t0;
        t0 = t1;
      }
      if (k >= a.lag) fold_chunk(i, first + (k - a.lag) * gc);
      if (a.prof) {
        const uint64_t t1 = dev::globaltimer();
        t_fold += t1 - t0;
        t0 = t1;
      }
    }
    // One system-scope release per launch (not per chunk: a sys fence per chunk stalls the
    // SM's pushes): my receive slots of every chunk of this launch may be overwritten by
    // senders two calls later.  Monotone, so it covers every chunk g of mine in [g0, g1).
    if (nk > 0 && threadIdx.x < a.r)
      dev::st_release_sys(consumed(a.my_workers[threadIdx.x], i),
                          step_epoch(a.seq_epoch0, first + (nk - 1) * gc));
    if (a.prof && threadIdx.x == 0) {
      uint64_t *pr = a.prof + int64_t(blockIdx.x) * 8;
      pr[0] += t_stage;
      pr[1] += t_fold;
      pr[2] += t0 - tstart;
      pr[7] += 1;
    }
  }

  // ---------------------------------------------------------------- COMM
  __device__ void comm(int q, unsigned char *smem) const {
    // dynamic smem: [TMA ring: kRing chunks][kRing mbarriers][guard cache: pairs x Gc u64]
    float *ring = reinterpret_cast<float *>(smem);
    uint64_t *mbar = reinterpret_cast<uint64_t *>(smem + kRingBytes);
    uint64_t *cache = mbar + kRing;
    if (threadIdx.x == 0) {
      for (int s = 0; s < kRing; ++s) dev::mbar_init(&mbar[s], 1);
      dev::fence_mbar_init();
    }
    // (slot, remote member) pairs of this rank; their consumed counters cached in smem
    int npairs = 0;
    for (int p = 0; p < a.r * a.m; ++p) {
      const int s = p / a.m, rr = p % a.m;
      const int me = a.my_workers[s];
      const int w = group(me)[rr];
      if (w != me && remote(w)) ++npairs;
    }
    const bool guard = a.call >= 2 && npairs > 0;
    const bool cached = guard && npairs <= kMaxGuardPairs;
    if (cached) {  // one bulk remote read of every counter (one round trip per CTA)
      for (int idx = threadIdx.x; idx < npairs * gc; idx += kThreads)
        cache[idx] = dev::ld_acquire_sys(consumed(remote_pair_member(idx / gc), idx % gc));
    }
    __syncthreads();
    // Per batch of B chunks: warp 0 waits (lane-parallel) for the guard and the staged flags;
    // then every (slot, chunk) item with remote members streams through a kRing-deep smem
    // ring: thread 0 prefetches the staged chunk with a TMA bulk load (stage in L2 -> smem,
    // mbarrier completion), and all threads copy it out with 128-bit stores into every remote
    // member's receive slot (NVLink; LSU stores keep ~22 GB/s per SM, a TMA bulk store to a
    // peer only ~6 GB/s per SM).  One system-scope release per (chunk, member) ends the batch.
    const int B = a.comm_batch;
    const int64_t nbatches = (a.g1 - a.g0 + B - 1) / B;
    const int ns = a.r;
    const uint64_t call1 = uint64_t(a.call) + 1;
    uint64_t t_wait = 0, t_push = 0, t_rel = 0, t0 = a.prof ? dev::globaltimer() : 0, tstart = t0;
    auto has_remote = [&](int s) {
      const int me = a.my_workers[s];
      for (int rr = 0; rr < a.m; ++rr) {
        const int w = group(me)[rr];
        if (w != me && remote(w)) return true;
      }
      return false;
    };
    uint32_t ring_uses = 0;  // items streamed so far (all threads agree): slot = uses % kRing
    for (int64_t j = q; j < nbatches; j += a.comm_ctas) {
      const int64_t c0 = a.g0 + j * B, c1 = min(c0 + B, a.g1);
      const int nb = int(c1 - c0);
      if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        if (guard) {  // receivers consumed their call-2 slots
          for (int idx = lane; idx < nb * npairs; idx += 32) {
            const int pi = idx % npairs;
            const int64_t g = c0 + idx / npairs;
            const int i = int(g % gc);
            const uint64_t need = step_epoch(a.prev2_epoch0, g);
            if (cached && cache[pi * gc + i] >= need) continue;
            const int w = remote_pair_member(pi);
            const uint64_t got = wait_geq(a, consumed(w, i), need, kWaitConsumed, w, pi);
            if (cached) cache[pi * gc + i] = got;
          }
        }
        for (int idx = lane; idx < nb * ns; idx += 32)  // my compute CTAs staged the batch
          wait_geq(a, staged(idx % ns, int((c0 + idx / ns) % gc)),
                   step_epoch(a.seq_epoch0, c0 + idx / ns), kWaitStaged, a.my_workers[idx % ns], -1);
      }
      __syncthreads();
      if (a.prof) {
        const uint64_t t1 = dev::globaltimer();
        t_wait += t1 - t0;
        t0 = t1;
      }
      // items of the batch that have a remote member: (s, g) in batch order
      const int total = nb * ns;
      auto item_live = [&](int idx) { return has_remote(idx % ns); };
      auto issue_load = [&](int idx, uint32_t use) {
        const int s = idx % ns;
        const ChunkRef c = locate(c0 + idx / ns);
        const uint32_t bytes = uint32_t(((c.e1 - c.e0) & ~int64_t(3)) * 4);
        const int slot = use % kRing;
        dev::mbar_arrive_expect_tx(&mbar[slot], bytes);
        if (bytes > 0) dev::bulk_g2s(ring + slot * kChunk, stage(s) + c.soff + c.e0, bytes, &mbar[slot]);
      };
      // prefetch the first kRing live items
      if (threadIdx.x == 0) {
        dev::fence_proxy_async_global();  // the stage was written by other CTAs (generic proxy)
        uint32_t u = ring_uses;
        for (int idx = 0, k = 0; idx < total && k < kRing; ++idx)
          if (item_live(idx)) issue_load(idx, u++), ++k;
      }
      int next_load = 0;  // thread 0: index of the next live item to prefetch (after the first kRing)
      if (threadIdx.x == 0) {
        int k = 0;
        for (; next_load < total && k < kRing; ++next_load)
          if (item_live(next_load)) ++k;
      }
      for (int idx = 0; idx < total; ++idx) {
        if (!item_live(idx)) continue;
        const int s = idx % ns;
        const int64_t g = c0 + idx / ns;
        const ChunkRef c = locate(g);
        const int slot = ring_uses % kRing;
        if (!dev::mbar_wait(&mbar[slot], (ring_uses / kRing) & 1, a.timeout_ns) && threadIdx.x == 0) {
          if (atomicExch(a.abort_dev, 1u) == 0u) {  // a TMA load never landed: latch, don't hang
            a.err_host[1] = 5;
            a.err_host[2] = blockIdx.x;
            a.err_host[7] = (unsigned long long)a.my_rank;
            __threadfence_system();
            atomicExch(a.err_host, (unsigned long long)(-SESGD_ETIMEOUT));
          }
        }
        const float *src = ring + slot * kChunk;
        const int me = a.my_workers[s];
        const int mypos = a.my_pos[s];
        const int64_t len = c.e1 - c.e0;
        float4 val[kVec];
#pragma unroll
        for (int it = 0; it < kVec; ++it) {
          const int64_t o = (int64_t(it) * kThreads + threadIdx.x) * 4;
          if (o + 4 <= len) val[it] = *reinterpret_cast<const float4 *>(src + o);
        }
        for (int rr = 0; rr < a.m; ++rr) {
          const int w = group(me)[rr];
          if (w == me || !remote(w)) continue;
          float *dst = recv(w, mypos) + c.soff + c.e0;
#pragma unroll
          for (int it = 0; it < kVec; ++it) {
            const int64_t o = (int64_t(it) * kThreads + threadIdx.x) * 4;
            if (o + 4 <= len) {
              *reinterpret_cast<float4 *>(dst + o) = val[it];
            } else if (o < len) {  // ragged 1..3-float tail (not covered by the bulk load)
              for (int64_t e = o; e < len; ++e) dst[e] = __ldcg(stage(s) + c.soff + c.e0 + e);
            }
          }
        }
        ++ring_uses;
        __syncthreads();  // every thread has read the slot: refill it
        if (threadIdx.x == 0) {
          while (next_load < total && !item_live(next_load)) ++next_load;
          if (next_load < total) issue_load(next_load++, ring_uses + kRing - 1);
        }
      }
      if (a.prof) {
        const uint64_t t1 = dev::globaltimer();
        t_push += t1 - t0;
        t0 = t1;
      }
      __syncthreads();  // every store of the batch precedes the releases (cumulativity)
      if (threadIdx.x < 32) {
        if (j == q) hop_delay(a);  // one handshake round per launch: delay once (config 4)
        const int n = nb * ns * a.m;
        for (int p = threadIdx.x; p < n; p += 32) {
          const int rr = p % a.m, s = (p / a.m) % ns;
          const int64_t g = c0 + p / (a.m * ns);
          const int me = a.my_workers[s];
          const int w = group(me)[rr];
          if (w == me) {
            st_release_gpu(sent(s, g), call1);
          } else if (remote(w)) {
            dev::st_release_sys(ready(w, g, a.my_pos[s]), call1);
            count(a.counters, kCntFlagStores);
          }
        }
      }
      if (a.prof) {
        const uint64_t t1 = dev::globaltimer();
        t_rel += t1 - t0;
        t0 = t1;
      }
    }
    if (a.prof && threadIdx.x == 0) {
      uint64_t *pr = a.prof + int64_t(blockIdx.x) * 8;
      pr[0] += t_wait;
      pr[1] += t_push;
      pr[2] += t_rel;
      pr[3] += t0 - tstart;
      pr[7] += 1;
    }
  }

  // ---------------------------------------------------------------- DIRECT (no COMM CTAs)
  // Every CTA is a compute CTA that pushes its own x_hat to the remote members straight from
  // registers (remote stores are fire-and-forget), so nothing is ever re-read from the stage
  // for sending.  Ready flags go out in batches every R = release_every chunk steps, at the
  // top of a step, covering every chunk staged before it: ONE system-scope fence per batch (a
  // fence waits for the SM's outstanding remote stores, ~8 us under load), then relaxed stores.

  // release the ready flags of my chunk ordinals [c0, c1) (chunk first + c * gc; warp 0,
  // lane-parallel); every thread's stores of those chunks precede this call through the
  // __syncthreads that ends stage_push
  __device__ __forceinline__ void release_ready(int64_t first, int64_t c0, int64_t c1) const {
    if (threadIdx.x >= 32 || c1 <= c0) return;
    // injected per-hop latency (config 4): the chunk flags of one launch are pipelined messages
    // of ONE handshake round, so the delay is paid once, before the first of them
    if (c0 == 0) hop_delay(a);
    const uint64_t call1 = uint64_t(a.call) + 1;
    const int pairs = a.r * a.m;
    dev::fence_acq_rel_sys();
    unsigned long long nst = 0;
    for (int64_t q = threadIdx.x; q < (c1 - c0) * pairs; q += 32) {
      const int64_t c = c0 + q / pairs;
      const int p = int(q % pairs), s = p / a.m, rr = p % a.m;
      const int me = a.my_workers[s];
      const int w = group(me)[rr];
      if (w != me && remote(w)) {
        st_relaxed_sys(ready(w, first + c * gc, a.my_pos[s]), call1);
        ++nst;
      }
    }
    count(a.counters, kCntFlagStores, nst);
  }

  // A group whose members all live on this GPU: the whole update in registers, like the
  // 1-GPU kernel (no stage, no flags, no fold); run once, by the group's first member.
  // BF (bf16 payload, R21): every contribution to the fold is rounded to bf16 first, as if it
  // had crossed NVLink, so all-local groups give the bits of the oracle's payload_bf16 reading.
  template <bool BF = false>
  __device__ void local_group_update(const ChunkRef &c, const int8_t *G) const {
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      const int64_t e = c.e0 + (int64_t(it) * kThreads + threadIdx.x) * W;
      const int nv = (int)min(int64_t(W), c.e1 - e);
      if (nv <= 0) continue;
      float acc[W];
      for (int rr = 0; rr < a.m; ++rr) {  // ascending member id
        const int sl = a.worker_slot[G[rr]];
        float gr[W];
        load_m<W>(a.bg[c.b * a.r + sl] + e, gr, nv);
        if constexpr (!GRAD) {
          float v[W], x[W];
          load_m<W>(a.bv[c.b * a.r + sl] + e, v, nv);
          load_m<W>(a.bx[c.b * a.r + sl] + e, x, nv);
#pragma unroll
          for (int q = 0; q < W; ++q) {
            v[q] = dev::momentum(a.mu, v[q], dev::decay(gr[q], a.wd, x[q]));
            float xh = dev::sgd(x[q], a.lr, v[q]);
            if constexpr (BF) xh = __bfloat162float(__float2bfloat16_rn(xh));
            acc[q] = (rr == 0) ? xh : __fadd_rn(acc[q], xh);
          }
          store_m<W>(a.bv[c.b * a.r + sl] + e, v, nv);
        } else {
#pragma unroll
          for (int q = 0; q < W; ++q) {
            if constexpr (BF) gr[q] = __bfloat162float(__float2bfloat16_rn(gr[q]));
            acc[q] = (rr == 0) ? gr[q] : __fadd_rn(acc[q], gr[q]);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < W; ++q) acc[q] = __fdiv_rn(acc[q], (float)a.m);
      for (int rr = 0; rr < a.m; ++rr) {
        const int sl = a.worker_slot[G[rr]];
        if constexpr (!GRAD) {
          store_m<W>(a.bx[c.b * a.r + sl] + e, acc, nv);
        } else {
          float v[W], x[W];
          load_m<W>(a.bv[c.b * a.r + sl] + e, v, nv);
          load_m<W>(a.bx[c.b * a.r + sl] + e, x, nv);
#pragma unroll
          for (int q = 0; q < W; ++q) {
            v[q] = dev::momentum(a.mu, v[q], dev::decay(acc[q], a.wd, x[q]));
            x[q] = dev::sgd(x[q], a.lr, v[q]);
          }
          store_m<W>(a.bv[c.b * a.r + sl] + e, v, nv);
          store_m<W>(a.bx[c.b * a.r + sl] + e, x, nv);
        }
      }
    }
  }

  __device__ void stage_push(int64_t g) const {
    const ChunkRef c = locate(g);
    for (int s = 0; s < a.r; ++s) {
      if (a.slot_kind[s] == 2) continue;  // done by its group's first member
      if (a.slot_kind[s] == 1) {
        local_group_update(c, group(a.my_workers[s]));
        continue;
      }
      float *xs = a.bx[c.b * a.r + s], *vs = a.bv[c.b * a.r + s];
      const float *gs = a.bg[c.b * a.r + s];
      const int me = a.my_workers[s];
      const int8_t *G = group(me);
      const int mypos = a.my_pos[s];
      float *st = stage(s) + c.soff;
#pragma unroll
      for (int it = 0; it < kItems; ++it) {
        const int64_t e = c.e0 + (int64_t(it) * kThreads + threadIdx.x) * W;
        const int nv = (int)min(int64_t(W), c.e1 - e);
        if (nv <= 0) continue;
        float gr[W], val[W];
        load_m<W>(gs + e, gr, nv);
        if constexpr (!GRAD) {
          float v[W], x[W];
          load_m<W>(vs + e, v, nv);
          load_m<W>(xs + e, x, nv);
#pragma unroll
          for (int q = 0; q < W; ++q) {
            v[q] = dev::momentum(a.mu, v[q], dev::decay(gr[q], a.wd, x[q]));
            val[q] = dev::sgd(x[q], a.lr, v[q]);  // x_hat
          }
          store_m<W>(vs + e, v, nv);
        } else {
#pragma unroll
          for (int q = 0; q < W; ++q) val[q] = gr[q];
        }
        st_slot<W>(st + e, val, nv);  // own copy, read by my fold (and co-resident members')
        for (int rr = 0; rr < a.m; ++rr) {
          const int w = G[rr];
          if (w != me && remote(w)) st_slot<W>(recv(w, mypos) + c.soff + e, val, nv);  // NVLink
        }
      }
    }
    __syncthreads();  // every store of chunk g precedes its (deferred) flag release
  }

  __device__ void fold_direct(int64_t g) const {
    const ChunkRef c = locate(g);
    const uint64_t call1 = uint64_t(a.call) + 1;
    if (threadIdx.x < 32) {  // every remote member's chunk g arrived
      for (int p = threadIdx.x; p < a.r * a.m; p += 32) {
        const int s = p / a.m, rr = p % a.m;
        const int me = a.my_workers[s];
        const int w = group(me)[rr];
        if (w != me && remote(w)) wait_geq(a, ready(me, g, rr), call1, kWaitReady, me, rr);
      }
    }
    __syncthreads();
    for (int s = 0; s < a.r; ++s) {
      if (a.slot_kind[s] != 0) continue;  // all-local group: already updated at stage time
      const int me = a.my_workers[s];
      const int8_t *G = group(me);
      float *xs = a.bx[c.b * a.r + s], *vs = a.bv[c.b * a.r + s];
#pragma unroll
      for (int it = 0; it < kItems; ++it) {
        const int64_t e = c.e0 + (int64_t(it) * kThreads + threadIdx.x) * W;
        const int nv = (int)min(int64_t(W), c.e1 - e);
        if (nv <= 0) continue;
        float acc[W];
        for (int rr = 0; rr < a.m; ++rr) {  // ascending position = ascending worker id
          const int w = G[rr];
          const float *src = remote(w) ? recv(me, rr) : stage(a.worker_slot[w]);
          float y[W];
          ld_slot<W>(src + c.soff + e, y, nv);
#pragma unroll
          for (int q = 0; q < W; ++q) acc[q] = (rr == 0) ? y[q] : __fadd_rn(acc[q], y[q]);
        }
#pragma unroll
        for (int q = 0; q < W; ++q) acc[q] = __fdiv_rn(acc[q], (float)a.m);
        if constexpr (!GRAD) {
          store_m<W>(xs + e, acc, nv);
        } else {
          float v[W], x[W];
          load_m<W>(vs + e, v, nv);
          load_m<W>(xs + e, x, nv);
#pragma unroll
          for (int q = 0; q < W; ++q) {
            v[q] = dev::momentum(a.mu, v[q], dev::decay(acc[q], a.wd, x[q]));
            x[q] = dev::sgd(x[q], a.lr, v[q]);
          }
          store_m<W>(vs + e, v, nv);
          store_m<W>(xs + e, x, nv);
        }
      }
    }
    __syncthreads();  // all slots folded (co-resident stages read)
    if constexpr (W == 4) {
      if (a.discard && (threadIdx.x & 7) == 0) {
        for (int s = 0; s < a.r; ++s) {
          if (a.slot_kind[s] != 0) continue;  // nothing staged for all-local groups
          const int me = a.my_workers[s];
          const int8_t *G = group(me);
#pragma unroll
          for (int it = 0; it < kItems; ++it) {
            const int64_t e = c.e0 + (int64_t(it) * kThreads + threadIdx.x) * W;
            if (e + 32 > c.e1) continue;
            discard_l2(stage(s) + c.soff + e);
            for (int rr = 0; rr < a.m; ++rr)
              if (remote(G[rr])) discard_l2(recv(me, rr) + c.soff + e);
          }
        }
      }
    }
    __syncthreads();
  }

  __device__ void compute_direct(int i) const {
    const int64_t first = a.g0 + ((int64_t(i) - a.g0 % gc) % gc + gc) % gc;
    const int64_t nk = (a.g1 > first) ? (a.g1 - first + gc - 1) / gc : 0;
    if (nk == 0) return;
    // guard, once: every remote member consumed its receive slots of call-2 for my chunks
    // (its CTA i folds exactly my chunks, so one remote counter per member)
    if (a.call >= 2 && threadIdx.x < 32) {
      const uint64_t need = step_epoch(a.prev2_epoch0, first + (nk - 1) * gc);
      for (int p = threadIdx.x; p < a.r * a.m; p += 32) {
        const int s = p / a.m, rr = p % a.m;
        const int me = a.my_workers[s];
        const int w = group(me)[rr];
        if (w != me && remote(w)) wait_geq(a, consumed(w, i), need, kWaitConsumed, w, rr);
      }
    }
    __syncthreads();
    // chunk c is staged at step c and released by step c + R (the first multiple of R above c),
    // so the fold of chunk k - L at step k finds its flags out when L >= R
    const int R = max(a.release_every, 1);
    const int L = max(a.lag, R);
    int64_t out = 0;  // chunk ordinals whose ready flags are released
    uint64_t t_stage = 0, t_fold = 0, t0 = a.prof ? dev::globaltimer() : 0, tstart = t0;
    for (int64_t k = 0; k < nk + L; ++k) {
      if ((k + (a.release_stagger ? i : 0)) % R == 0 || k == nk) {
        const int64_t c1 = k < nk ? k : nk;
        release_ready(first, out, c1);
        out = c1;
      }
      if (k < nk) stage_push(first + k * gc);
      if (a.prof) {
        const uint64_t t1 = dev::globaltimer();
        t_stage += t1 - t0;
        t0 = t1;
      }
      if (k >= L) fold_direct(first + (k - L) * gc);
      if (a.prof) {
        const uint64_t t1 = dev::globaltimer();
        t_fold += t1 - t0;
        t0 = t1;
      }
    }
    if (threadIdx.x < a.r)
      dev::st_release_sys(consumed(a.my_workers[threadIdx.x], i),
                          step_epoch(a.seq_epoch0, first + (nk - 1) * gc));
    if (a.prof && threadIdx.x == 0) {
      uint64_t *pr = a.prof + int64_t(blockIdx.x) * 8;
      pr[0] += t_stage;
      pr[1] += t_fold;
      pr[2] += t0 - tstart;
      pr[7] += 1;
    }
  }

  // ---------------------------------------------------------------- K4 TWO-SHOT
  // Reduce-scatter + all-gather inside the group, both as NVLink pushes: the member at
  // position j OWNS slice j of every chunk.  Per chunk g (epochs e1 = 2 call + 1, e2 = e1 + 1):
  //  rs_stage(g): local step in registers; own slice -> own stage, slice j -> member a_j's
  //               receive slot [my position] (NVLink); flag ready(a_j, g, my pos) = e1
  //  reduce(g):   wait e1 from every peer; fold my slice over positions in ascending order
  //               (= ascending worker id, the oracle's order) ; (/) m ; apply it to my x
  //               (PARAM: x = mean; GRAD: momentum update with the mean gradient) and push the
  //               mean to every peer's receive slot [my position] at my slice; ready = e2
  //  finish(g):   wait e2 from every peer; apply the peers' slices (PARAM: x = mean slice;
  //               GRAD: momentum update)
  // A sender's RS data (the receiver's slice) and AG data (the sender's slice) share the
  // receiver's slot [sender position] without overlap.  Bytes pushed per GPU per element:
  // 2 (m-1)/m x 4 (one-shot: (m-1) x 4).  Flags are released at the top of the next chunk
  // step (a system-scope release waits for the CTA's remote stores to drain; by then they
  // have), reduce runs `lag` chunk steps after rs_stage and finish `lag` after reduce; every
  // wait targets a flag released at the top of an earlier step or of this one: no deadlock.
  __device__ __forceinline__ int ts_slice() const { return (int(kChunk) / a.m) & ~31; }
  __device__ __forceinline__ int64_t ts_lo(int j, int64_t len) const {
    return min(int64_t(j) * ts_slice(), len);
  }
  __device__ __forceinline__ int64_t ts_hi(int j, int64_t len) const {
    return j == a.m - 1 ? len : min(int64_t(j + 1) * ts_slice(), len);
  }

  // TMA variant (SESGD_OPT_PUSH_TMA): the remote part of a push is assembled in a shared-memory
  // ring entry (one 16 KiB chunk image) and sent with one cp.async.bulk shared -> peer global per
  // peer, issued by thread 0, so remote stores never occupy the LSU request slots the HBM
  // stream needs.  Group q of the CTA's bulk groups uses entry q mod kPushRing; flags of a
  // step's pushes are released two steps later, after cp.async.bulk.wait_group.
  static constexpr int kPushRing = 3;

  // bulk-copyable prefix of slice j (whole float4s; the ragged tail goes by plain stores)
  __device__ __forceinline__ int64_t ts_bulk_hi(int j, int64_t len) const {
    const int64_t lo = ts_lo(j, len);
    return lo + ((ts_hi(j, len) - lo) & ~int64_t(3));
  }

  // issue (thread 0) the bulk copies of ring entry `ent` for slice range owner `j` (or every
  // slice but mine when j < 0) to the peers' receive slots, and commit one group
  __device__ __forceinline__ void ts_bulk_push(const ChunkRef &c, const float *ent, int j) const {
    const int me = a.my_workers[0];
    const int8_t *G = group(me);
    const int p = a.my_pos[0];
    const int64_t len = c.e1 - c.e0;
    dev::fence_proxy_async_shared();
    for (int q = 0; q < a.m; ++q) {
      if (q == p) continue;
      const int s = (j < 0) ? q : j;  // RS: peer q's slice; AG: my slice to every peer
      const int64_t lo = ts_lo(s, len), bh = ts_bulk_hi(s, len);
      if (bh > lo)
        dev::bulk_s2g(recv(G[q], p) + c.soff + c.e0 + lo, ent + lo, uint32_t((bh - lo) * 4));
    }
    dev::bulk_commit();
  }

  // is worker w on another GPU?  (one worker per GPU: every other member is)
  template <bool MULTI>
  __device__ __forceinline__ bool rem(int w) const {
    return MULTI ? remote(w) : w != a.my_workers[0];
  }

  // ---- K4 with r >= 1 workers per GPU.  Slot s (worker me_s at position p_s of its group G_s)
  // owns slice p_s of every chunk.  A member's x_hat for a slice owned by a co-resident worker
  // (or itself) stays in its own stage, read in place by the owner; for a remote owner it is
  // pushed to the owner's receive slot [p_s].  The owner applies the mean to co-resident members
  // directly (their x, v are on this GPU) and pushes it to remote members.  Groups whose members
  // all live here are updated in registers (slot_kind 1 / 2, as in K3).
  // ---- NVLS (one worker per GPU, group_size = n): chunk g is OWNED by position g mod m.  The
  // owner waits until every member staged chunk g (RS flags), then reduces the whole chunk in the
  // NVSwitch with multimem.ld_reduce on the multicast mapping of the stages (kItems 16-byte loads
  // in flight per thread), divides by m, stores its own x and multicasts the mean into every
  // member's receive slot [owner] with multimem.st (AG flag).  The other members take the mean
  // from that slot in nv_finish.  A member's stage of chunk g is read only by the owner, which
  // releases its AG flag after the read, so the next call's stage cannot overtake it.
  __device__ void nv_reduce(int64_t g) const {
    const ChunkRef c = locate(g);
    const int me = a.my_workers[0];
    const int p = a.my_pos[0];
    const int own = int(g % a.m);
    if (own != p) return;
    if (threadIdx.x < 32) {
      for (int j = threadIdx.x; j < a.m; j += 32)
        if (j != p) wait_geq(a, ready(me, g, j), 2 * uint64_t(a.call) + 1, kWaitReady, me, j);
    }
    __syncthreads();
    fence_proxy_alias();  // peers' stages are read through the multicast mapping
    const float *mcs = reinterpret_cast<const float *>(a.mc_ws + a.stage_off) + c.soff;
    float *mcr = reinterpret_cast<float *>(a.mc_ws + a.recv_off) +
                 (int64_t(a.parity) * a.m + p) * a.region_floats + c.soff;
    float *xs = a.bx[c.b * a.r], *vs = a.bv[c.b * a.r];
    float acc[kItems][W];
#pragma unroll
    for (int it = 0; it < kItems; ++it) {  // every load in flight before the first use
      const int64_t e = c.e0 + (int64_t(it) * kThreads + threadIdx.x) * W;
      const int nv = (int)min(int64_t(W), c.e1 - e);
      if (W == 4 && nv == 4) {
        mm_ld_reduce4(mcs + e, reinterpret_cast<float(&)[4]>(acc[it]));
      } else {
#pragma unroll
        for (int q = 0; q < W; ++q) acc[it][q] = (q < nv) ? mm_ld_reduce1(mcs + e + q) : 0.f;
      }
    }
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      const int64_t e = c.e0 + (int64_t(it) * kThreads + threadIdx.x) * W;
      const int nv = (int)min(int64_t(W), c.e1 - e);
      if (nv <= 0) continue;
      float m4[W];
#pragma unroll
      for (int q = 0; q < W; ++q) m4[q] = __fdiv_rn(acc[it][q], (float)a.m);
      if (W == 4 && nv == 4)
        mm_st4(mcr + e, reinterpret_cast<float(&)[4]>(m4));
      else
        for (int q = 0; q < nv; ++q) mm_st1(mcr + e + q, m4[q]);
      if constexpr (!GRAD) {
        store_m<W>(xs + e, m4, nv);
      } else {
        float v[W], x[W];
        load_m<W>(vs + e, v, nv);
        load_m<W>(xs + e, x, nv);
#pragma unroll
        for (int q = 0; q < W; ++q) {
          v[q] = dev::momentum(a.mu, v[q], dev::decay(m4[q], a.wd, x[q]));
          x[q] = dev::sgd(x[q], a.lr, v[q]);
        }
        store_m<W>(vs + e, v, nv);
        store_m<W>(xs + e, x, nv);
      }
    }
    __syncthreads();  // the multicast stores precede the (deferred) AG flag release
  }

  __device__ void nv_finish(int64_t g) const {
    const ChunkRef c = locate(g);
    const int me = a.my_workers[0];
    const int p = a.my_pos[0];
    const int own = int(g % a.m);
    if (own == p) return;  // applied in nv_reduce
    if (threadIdx.x == 0) wait_geq(a, ready(me, g, own), 2 * uint64_t(a.call) + 2, kWaitReady, me, own);
    __syncthreads();
    fence_proxy_alias();  // the mean arrived through the multicast mapping
    const float *src = recv(me, own) + c.soff;
    float *xs = a.bx[c.b * a.r], *vs = a.bv[c.b * a.r];
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      const int64_t e = c.e0 + (int64_t(it) * kThreads + threadIdx.x) * W;
      const int nv = (int)min(int64_t(W), c.e1 - e);
      if (nv <= 0) continue;
      float y[W];
      ld_slot<W>(src + e, y, nv);
      if constexpr (!GRAD) {
        store_m<W>(xs + e, y, nv);
      } else {
        float v[W], x[W];
        load_m<W>(vs + e, v, nv);
        load_m<W>(xs + e, x, nv);
#pragma unroll
        for (int q = 0; q < W; ++q) {
          v[q] = dev::momentum(a.mu, v[q], dev::decay(y[q], a.wd, x[q]));
          x[q] = dev::sgd(x[q], a.lr, v[q]);
        }
        store_m<W>(vs + e, v, nv);
        store_m<W>(xs + e, x, nv);
      }
    }
    __syncthreads();
  }

  template <bool TMA, bool MULTI, bool NV = false, bool BF = false, bool SENT = false>
  __device__ void ts_rs_stage(int64_t g, float *ent) const {
    const ChunkRef c = locate(g);
    const int S = ts_slice();
    const int64_t len = c.e1 - c.e0;
    if constexpr (TMA) {  // the entry's previous bulk group has finished reading it (r == 1)
      if (threadIdx.x == 0) dev::bulk_wait_read<kPushRing - 1>();
      __syncthreads();
    }
    for (int s = 0; s < (MULTI ? a.r : 1); ++s) {
      if (MULTI && a.slot_kind[s] == 2) continue;  // done by its group's first member
      const int8_t *G = group(a.my_workers[s]);
      if (MULTI && a.slot_kind[s] == 1) {
        local_group_update<BF>(c, G);
        continue;
      }
      const int p = a.my_pos[s];
      float *xs = a.bx[c.b * a.r + s], *vs = a.bv[c.b * a.r + s];
      const float *gs = a.bg[c.b * a.r + s];
      // items in batches of kB: every load of a batch is in flight before its first store (the
      // compiler cannot hoist loads above stores it cannot prove disjoint, so an unbatched loop
      // pays one HBM latency per item)
      // (several workers per GPU: 4 CTAs per SM without batching measured faster than 3 with it,
      // profiles/r02_k4_experiments.json)
      constexpr int kB = MULTI ? 1 : (W == 4) ? 2 : 8;
#pragma unroll
      for (int b0 = 0; b0 < kItems; b0 += kB) {
        float gr[kB][W], v[GRAD ? 1 : kB][W], x[GRAD ? 1 : kB][W];
#pragma unroll
        for (int ib = 0; ib < kB; ++ib) {
          const int64_t o = (int64_t(b0 + ib) * kThreads + threadIdx.x) * W;
          const int64_t e = c.e0 + o;
          const int nv = (int)min(int64_t(W), c.e1 - e);
          if (nv <= 0) continue;
          load_m<W>(gs + e, gr[ib], nv);
          if constexpr (!GRAD) {
            load_m<W>(vs + e, v[ib], nv);
            load_m<W>(xs + e, x[ib], nv);
          }
        }
#pragma unroll
        for (int ib = 0; ib < kB; ++ib) {
        const int it = b0 + ib;
        const int64_t o = (int64_t(it) * kThreads + threadIdx.x) * W;  // offset inside the chunk
        const int64_t e = c.e0 + o;
        const int nv = (int)min(int64_t(W), c.e1 - e);
        if (nv <= 0) continue;
        float val[W];
        if constexpr (!GRAD) {
#pragma unroll
          for (int q = 0; q < W; ++q) {
            v[ib][q] = dev::momentum(a.mu, v[ib][q], dev::decay(gr[ib][q], a.wd, x[ib][q]));
            val[q] = dev::sgd(x[ib][q], a.lr, v[ib][q]);  // x_hat
          }
          store_m<W>(vs + e, v[ib], nv);
        } else {
#pragma unroll
          for (int q = 0; q < W; ++q) val[q] = gr[ib][q];
        }
        const int j = min(int(o / S), a.m - 1);  // owner position (a W-vector never straddles)
        const int w = G[j];
        if constexpr (BF) {  // packed at the owner's slice: local owner -> my stage, remote -> its slot
          const int64_t lo = ts_lo(j, len);
          float *base = (rem<MULTI>(w) ? recv(w, p) : stage(s)) + c.soff + c.e0 + lo;
          st_bf<W>(reinterpret_cast<__nv_bfloat16 *>(base) + (o - lo), val, nv);
          continue;
        }
        if (NV || !rem<MULTI>(w)) {  // NVLS: every owner reduces my stage through the switch
          st_slot<W>(stage(s) + c.soff + e, val, nv);  // read in place by the local owner
        } else if (TMA && o + nv <= ts_bulk_hi(j, len)) {
          st_slot<W>(ent + o, val, nv);  // shared memory image of the chunk
        } else if constexpr (SENT) {
          st_sent<W>(recv(w, p) + c.soff + e, val, nv);  // NVLink store, validity in the value
        } else {
          st_slot<W>(recv(w, p) + c.soff + e, val, nv);  // NVLink store
        }
        }
      }
    }
    __syncthreads();  // every store of chunk g precedes its bulk push / (deferred) flag release
    if constexpr (TMA) {
      if (threadIdx.x == 0) ts_bulk_push(c, ent, -1);
    }
  }

  // Flags of earlier pushes, one batch: RS of my chunk ordinals [rs0, rs1), AG of [ag0, ag1)
  // (ordinal c = chunk first + c * gc), for every (slot, remote member) pair.  ONE system-scope
  // fence per batch (a fence waits for the SM's outstanding remote stores: measured ~8 us per
  // chunk step under load), then relaxed flag stores spread over warp 0's lanes.  TMA (r == 1):
  // the `newer` most recent bulk groups may still be in flight, every older one must have landed.
  template <bool TMA, bool MULTI, bool NV = false>
  __device__ __forceinline__ void ts_release(int64_t first, int64_t rs0, int64_t rs1, int64_t ag0,
                                             int64_t ag1, int newer) const {
    if (threadIdx.x >= 32 || (rs1 <= rs0 && ag1 <= ag0)) return;
    if ((rs0 == 0 && rs1 > 0) || (ag0 == 0 && ag1 > 0)) hop_delay(a);  // once per round (config 4)
    const int pairs = (MULTI ? a.r : 1) * a.m;
    const uint64_t e1 = 2 * uint64_t(a.call) + 1;
    if constexpr (TMA) {
      if (threadIdx.x == 0) {
        dev::bulk_wait_upto(newer);  // those bulk writes are complete ...
        dev::fence_proxy_async_global();
      }
      __syncwarp();
    }
    if constexpr (NV) fence_proxy_alias();  // NVLS: multicast stores before the unicast flags
    if (!(a.experiment & 1))    // (SESGD_OPT_EXPERIMENT bit 0: measurement only)
      dev::fence_acq_rel_sys();  // ... before the flags (release pattern: fence + relaxed stores)
    const int64_t nrs = (rs1 - rs0) * pairs, nall = nrs + (ag1 - ag0) * pairs;
    unsigned long long nst = 0;
    for (int64_t q = threadIdx.x; q < nall; q += 32) {
      const int kind = q < nrs ? 0 : 1;
      const int64_t qq = kind == 0 ? q : q - nrs;
      const int64_t c = (kind == 0 ? rs0 : ag0) + qq / pairs;
      const int pr = int(qq % pairs), s = pr / a.m, j = pr % a.m;
      if ((MULTI && a.slot_kind[s] != 0) || j == a.my_pos[s]) continue;
      if constexpr (NV) {  // NVLS: staged -> the chunk's owner only; AG flags only from the owner
        const int own = int((first + c * gc) % a.m);
        if (kind == 0 ? (j != own) : (a.my_pos[s] != own)) continue;
      }
      const int w = group(a.my_workers[s])[j];
      if (rem<MULTI>(w)) {
        st_relaxed_sys(ready(w, first + c * gc, a.my_pos[s]), e1 + kind);
        ++nst;
      }
    }
    count(a.counters, kCntFlagStores, nst);
  }

  // every remote member's flag of chunk g (for every slot) reached `epoch`
  template <bool MULTI>
  __device__ __forceinline__ void ts_wait(int64_t g, uint64_t epoch) const {
    if (threadIdx.x < 32) {
      for (int pr = threadIdx.x; pr < (MULTI ? a.r : 1) * a.m; pr += 32) {
        const int s = pr / a.m, j = pr % a.m;
        if ((MULTI && a.slot_kind[s] != 0) || j == a.my_pos[s]) continue;
        const int me = a.my_workers[s];
        if (rem<MULTI>(group(me)[j])) wait_geq(a, ready(me, g, j), epoch, kWaitReady, me, j);
      }
    }
    __syncthreads();
  }

  template <bool TMA, bool MULTI, bool NV = false, bool BF = false, bool SENT = false>
  __device__ void ts_reduce(int64_t g, float *ent) const {
    const ChunkRef c = locate(g);
    if (TMA && threadIdx.x == 0) dev::bulk_wait_read<kPushRing - 1>();  // entry free (+ sync below)
    if constexpr (NV) {
      nv_reduce(g);
      return;
    }
    if constexpr (!SENT) ts_wait<MULTI>(g, 2 * uint64_t(a.call) + 1);  // SENT: polled per value below
    const int64_t len = c.e1 - c.e0;
    for (int s = 0; s < (MULTI ? a.r : 1); ++s) {
      if (MULTI && a.slot_kind[s] != 0) continue;
      const int me = a.my_workers[s];
      const int8_t *G = group(me);
      const int p = a.my_pos[s];
      const int64_t lo = ts_lo(p, len), hi = ts_hi(p, len), bh = ts_bulk_hi(p, len);
      for (int64_t o = lo + int64_t(threadIdx.x) * W; o < hi; o += int64_t(kThreads) * W) {
        const int64_t e = c.e0 + o;
        const int nv = (int)min(int64_t(W), hi - o);
        float acc[W];
        for (int rr = 0; rr < a.m; ++rr) {  // ascending position = ascending worker id
          const int w = G[rr];
          float *src = rem<MULTI>(w) ? recv(me, rr) : stage(a.worker_slot[w]);
          float y[W];
          if constexpr (BF)
            ld_bf<W>(reinterpret_cast<const __nv_bfloat16 *>(src + c.soff + c.e0 + lo) + (o - lo), y, nv);
          else if (SENT && rem<MULTI>(w))
            ld_poll<W>(a, src + c.soff + e, y, nv, me, rr);
          else
            ld_slot<W>(src + c.soff + e, y, nv);
#pragma unroll
          for (int q = 0; q < W; ++q) acc[q] = (rr == 0) ? y[q] : __fadd_rn(acc[q], y[q]);
        }
#pragma unroll
        for (int q = 0; q < W; ++q) acc[q] = __fdiv_rn(acc[q], (float)a.m);
        const bool bulk = TMA && o + nv <= bh;
        if (bulk) st_slot<W>(ent + o, acc, nv);  // all-gather image, bulk-pushed below (r == 1)
        for (int rr = 0; rr < a.m; ++rr) {  // apply to every member: here directly, else push
          const int w = G[rr];
          if (rem<MULTI>(w)) {
            if constexpr (SENT)
              st_sent<W>(recv(w, p) + c.soff + e, acc, nv);
            else if (!bulk)
              st_slot<W>(recv(w, p) + c.soff + e, acc, nv);
            continue;
          }
          const int sl = a.worker_slot[w];
          float *xw = a.bx[c.b * a.r + sl] + e, *vw = a.bv[c.b * a.r + sl] + e;
          if constexpr (!GRAD) {
            store_m<W>(xw, acc, nv);
          } else {
            float v[W], x[W];
            load_m<W>(vw, v, nv);
            load_m<W>(xw, x, nv);
#pragma unroll
            for (int q = 0; q < W; ++q) {
              v[q] = dev::momentum(a.mu, v[q], dev::decay(acc[q], a.wd, x[q]));
              x[q] = dev::sgd(x[q], a.lr, v[q]);
            }
            store_m<W>(vw, v, nv);
            store_m<W>(xw, x, nv);
          }
        }
      }
    }
    __syncthreads();  // my slices are folded: drop the dead lines (stages, RS data)
    if constexpr (TMA) {
      if (threadIdx.x == 0) ts_bulk_push(c, ent, a.my_pos[0]);
    }
    if constexpr (W == 4) {
      if (a.discard) {
        for (int s = 0; s < (MULTI ? a.r : 1); ++s) {
          if (MULTI && a.slot_kind[s] != 0) continue;
          const int me = a.my_workers[s];
          const int8_t *G = group(me);
          const int p = a.my_pos[s];
          const int64_t lo = ts_lo(p, len), hi = ts_hi(p, len);
          for (int64_t o = lo + int64_t(threadIdx.x) * 32; o + 32 <= hi; o += int64_t(kThreads) * 32)
            for (int rr = 0; rr < a.m; ++rr) {
              const int w = G[rr];
              if (SENT && rem<MULTI>(w)) continue;  // re-armed receive lines stay (not dead)
              discard_l2((rem<MULTI>(w) ? recv(me, rr) : stage(a.worker_slot[w])) + c.soff + c.e0 + o);
            }
        }
      }
    }
    __syncthreads();  // the AG stores precede the (deferred) flag release
  }

  // the slices owned by remote members: their means arrived in my receive slots
  template <bool MULTI, bool NV = false, bool SENT = false>
  __device__ void ts_finish(int64_t g) const {
    const ChunkRef c = locate(g);
    if constexpr (NV) {
      nv_finish(g);
      return;
    }
    if constexpr (!SENT) ts_wait<MULTI>(g, 2 * uint64_t(a.call) + 2);  // SENT: polled per value
    const int64_t len = c.e1 - c.e0;
    for (int s = 0; s < (MULTI ? a.r : 1); ++s) {
      if (MULTI && a.slot_kind[s] != 0) continue;
      const int me = a.my_workers[s];
      const int8_t *G = group(me);
      float *xs = a.bx[c.b * a.r + s], *vs = a.bv[c.b * a.r + s];
      for (int j = 0; j < a.m; ++j) {
        if (j == a.my_pos[s] || !rem<MULTI>(G[j])) continue;
        const int64_t lo = ts_lo(j, len), hi = ts_hi(j, len);
        float *src = recv(me, j) + c.soff;
        for (int64_t o = lo + int64_t(threadIdx.x) * W; o < hi; o += int64_t(kThreads) * W) {
          const int64_t e = c.e0 + o;
          const int nv = (int)min(int64_t(W), hi - o);
          float y[W];
          if constexpr (SENT)
            ld_poll<W>(a, src + e, y, nv, me, j);
          else
            ld_slot<W>(src + e, y, nv);
          if constexpr (!GRAD) {
            store_m<W>(xs + e, y, nv);
          } else {
            float v[W], x[W];
            load_m<W>(vs + e, v, nv);
            load_m<W>(xs + e, x, nv);
#pragma unroll
            for (int q = 0; q < W; ++q) {
              v[q] = dev::momentum(a.mu, v[q], dev::decay(y[q], a.wd, x[q]));
              x[q] = dev::sgd(x[q], a.lr, v[q]);
            }
            store_m<W>(vs + e, v, nv);
            store_m<W>(xs + e, x, nv);
          }
        }
      }
    }
    __syncthreads();
    if constexpr (W == 4 && !SENT) {  // SENT: the receive lines were re-armed, they stay
      if (a.discard) {
        for (int s = 0; s < (MULTI ? a.r : 1); ++s) {
          if (MULTI && a.slot_kind[s] != 0) continue;
          const int me = a.my_workers[s];
          const int8_t *G = group(me);
          for (int j = 0; j < a.m; ++j) {
            if (j == a.my_pos[s] || !rem<MULTI>(G[j])) continue;
            const int64_t lo = ts_lo(j, len), hi = ts_hi(j, len);
            for (int64_t o = lo + int64_t(threadIdx.x) * 32; o + 32 <= hi; o += int64_t(kThreads) * 32)
              discard_l2(recv(me, j) + c.soff + c.e0 + o);
          }
        }
      }
    }
    __syncthreads();
  }

  // Releases happen at the top of every R-th chunk step (R = release_every) and cover every push
  // made at least D steps earlier (D = 1 for LSU stores; 2 for TMA, whose bulk groups of the
  // last step may still be in flight).  A chunk pushed at step s is released by step
  // s + D + R - 1, so with reduce L >= D + R - 1 steps after rs_stage (and finish L after
  // reduce) every wait targets a flag released at the top of this step or an earlier one.
  template <bool TMA, bool MULTI, bool NV = false, bool BF = false, bool SENT = false>
  __device__ void compute_twoshot(int i, float *ring) const {
    const int64_t first = a.g0 + ((int64_t(i) - a.g0 % gc) % gc + gc) % gc;
    const int64_t nk = (a.g1 > first) ? (a.g1 - first + gc - 1) / gc : 0;
    if (nk == 0) return;
    if (a.call >= 2 && threadIdx.x < 32) {  // guard: remote members consumed their call-2 slots
      const uint64_t need = step_epoch(a.prev2_epoch0, first + (nk - 1) * gc);
      for (int pr = threadIdx.x; pr < (MULTI ? a.r : 1) * a.m; pr += 32) {
        const int sl = pr / a.m, j = pr % a.m;
        if (MULTI && a.slot_kind[sl] != 0) continue;
        const int w = group(a.my_workers[sl])[j];
        if (rem<MULTI>(w)) wait_geq(a, consumed(w, i), need, kWaitConsumed, w, j);
      }
    }
    __syncthreads();
    const int D = TMA ? max(a.release_delay, 2) : max(a.release_delay, 1);
    const int R = max(a.release_every, 1);
    const int L = SENT ? max(a.lag, 1) : max(a.lag, D + R - 1);  // SENT: no release schedule
    auto groups_of = [&](int64_t k) {  // bulk groups committed in step k
      return int(k >= 0 && k < nk) + int(k >= L && k - L < nk);
    };
    auto clampk = [&](int64_t v) { return v < 0 ? int64_t(0) : (v > nk ? nk : v); };
    int64_t rs_out = 0, ag_out = 0;  // chunk ordinals whose RS / AG flags are released
    uint32_t q = 0;  // bulk groups committed so far (uniform across the CTA)
    uint64_t t_stage = 0, t_red = 0, t_fin = 0, t_rel = 0;
    uint64_t t0 = a.prof ? dev::globaltimer() : 0, tstart = t0;
    for (int64_t k = 0; k < nk + 2 * L; ++k) {
      // pushes of steps <= k - D: RS of ordinals < k-D+1, AG of < k-D-L+1; with stagger the CTAs
      // of an SM take their release steps in turn instead of all at once
      if (SENT && a.hop_delay_ns && (k == 0 || k == L)) {  // config 4: one delay per round
        if (threadIdx.x == 0) hop_delay(a);
        __syncthreads();
      }
      if (!SENT && (k + (a.release_stagger ? i : 0)) % R == 0) {
        const int64_t rs1 = clampk(k - D + 1), ag1 = clampk(k - D - L + 1);
        int newer = 0;
        if constexpr (TMA)
          for (int64_t s2 = k - D + 1; s2 < k; ++s2) newer += groups_of(s2);
        ts_release<TMA, MULTI, NV>(first, rs_out, rs1, ag_out, ag1, newer);
        rs_out = rs1;
        ag_out = ag1;
      }
      if (a.prof) {
        const uint64_t t1 = dev::globaltimer();
        t_rel += t1 - t0;
        t0 = t1;
      }
      if (k < nk) {
        ts_rs_stage<TMA, MULTI, NV, BF, SENT>(first + k * gc, ring + (q % kPushRing) * kChunk);
        q += TMA ? 1 : 0;
      }
      if (a.prof) {
        const uint64_t t1 = dev::globaltimer();
        t_stage += t1 - t0;
        t0 = t1;
      }
      if (k >= L && k - L < nk) {
        ts_reduce<TMA, MULTI, NV, BF, SENT>(first + (k - L) * gc, ring + (q % kPushRing) * kChunk);
        q += TMA ? 1 : 0;
      }
      if (a.prof) {
        const uint64_t t1 = dev::globaltimer();
        t_red += t1 - t0;
        t0 = t1;
      }
      if (k >= 2 * L && k - 2 * L < nk) ts_finish<MULTI, NV, SENT>(first + (k - 2 * L) * gc);
      if (a.prof) {
        const uint64_t t1 = dev::globaltimer();
        t_fin += t1 - t0;
        t0 = t1;
      }
    }
    if (TMA && threadIdx.x == 0) dev::bulk_wait_all();  // no bulk copy outlives the CTA
    if (threadIdx.x < (MULTI ? a.r : 1))  // every read of my receive slots is done (call + 2 guard)
      dev::st_release_sys(consumed(a.my_workers[threadIdx.x], i),
                          step_epoch(a.seq_epoch0, first + (nk - 1) * gc));
    if (a.prof && threadIdx.x == 0) {
      uint64_t *pr = a.prof + int64_t(blockIdx.x) * 8;
      pr[0] += t_stage;
      pr[1] += t_red;
      pr[2] += t0 - tstart;
      pr[3] += t_fin;
      pr[4] += t_rel;
      pr[7] += 1;
    }
  }

  // m == 1: no exchange, the local step is the whole update (x / 1 = x)
  __device__ void local_only() const {
    for (int64_t g = a.g0 + blockIdx.x; g < a.g1; g += a.grid) {
      const ChunkRef c = locate(g);
      for (int s = 0; s < a.r; ++s) {
        float *xs = a.bx[c.b * a.r + s], *vs = a.bv[c.b * a.r + s];
        const float *gs = a.bg[c.b * a.r + s];
#pragma unroll
        for (int it = 0; it < kItems; ++it) {
          const int64_t e = c.e0 + (int64_t(it) * kThreads + threadIdx.x) * W;
          const int nv = (int)min(int64_t(W), c.e1 - e);
          if (nv <= 0) continue;
          float gr[W], v[W], x[W];
          load_m<W>(gs + e, gr, nv);
          load_m<W>(vs + e, v, nv);
          load_m<W>(xs + e, x, nv);
#pragma unroll
          for (int q = 0; q < W; ++q) {
            v[q] = dev::momentum(a.mu, v[q], dev::decay(gr[q], a.wd, x[q]));
            x[q] = dev::sgd(x[q], a.lr, v[q]);
          }
          store_m<W>(vs + e, v, nv);
          store_m<W>(xs + e, x, nv);
        }
      }
    }
  }
};

template <int W, bool GRAD>
__global__ void __launch_bounds__(kThreads, 3) k3_split(const __grid_constant__ P2PArgs a) {
  extern __shared__ __align__(128) unsigned char dsmem[];
  const Split<W, GRAD> p(a);
  if (blockIdx.x == 0 && threadIdx.x == 0) count(a.counters, kCntLaunches);
  if (a.m == 1) {
    p.local_only();
  } else if (int(blockIdx.x) < a.comm_ctas) {
    p.comm(blockIdx.x, dsmem);
  } else {
    p.compute(blockIdx.x - a.comm_ctas);
  }
}

template <int W, bool GRAD>
__global__ void __launch_bounds__(kThreads, 4) k3_direct(const __grid_constant__ P2PArgs a) {
  const Split<W, GRAD> p(a);
  if (blockIdx.x == 0 && threadIdx.x == 0) count(a.counters, kCntLaunches);
  if (a.m == 1)
    p.local_only();
  else
    p.compute_direct(blockIdx.x);
}

template <int W, bool GRAD, bool TMA, bool MULTI, bool NV = false, bool BF = false, bool SENT = false>
__global__ void __launch_bounds__(kThreads, MULTI ? 4 : 3) k4_twoshot(const __grid_constant__ P2PArgs a) {
  extern __shared__ __align__(128) unsigned char dsmem[];  // TMA: kPushRing chunk images
  const Split<W, GRAD> p(a);
  if (blockIdx.x == 0 && threadIdx.x == 0) count(a.counters, kCntLaunches);
  if (a.m == 1)
    p.local_only();
  else
    p.template compute_twoshot<TMA, MULTI, NV, BF, SENT>(blockIdx.x, reinterpret_cast<float *>(dsmem));
}

constexpr size_t kTwoshotTmaSmem = size_t(Split<4, false>::kPushRing) * size_t(kChunk) * 4;  // 48 KiB

template <bool TMA, bool MULTI>
const void *pick_twoshot_t(int mode, bool vec) {
  const bool grad = (mode == SESGD_MODE_GRAD_AVG);
  if (vec)
    return grad ? reinterpret_cast<const void *>(&k4_twoshot<4, true, TMA, MULTI>)
                : reinterpret_cast<const void *>(&k4_twoshot<4, false, TMA, MULTI>);
  return grad ? reinterpret_cast<const void *>(&k4_twoshot<1, true, TMA, MULTI>)
              : reinterpret_cast<const void *>(&k4_twoshot<1, false, TMA, MULTI>);
}
// NVLS: the switch reduces and multicasts (one worker per GPU, one group of all workers)
const void *pick_nvls(int mode, bool vec) {
  const bool grad = (mode == SESGD_MODE_GRAD_AVG);
  if (vec)
    return grad ? reinterpret_cast<const void *>(&k4_twoshot<4, true, false, false, true>)
                : reinterpret_cast<const void *>(&k4_twoshot<4, false, false, false, true>);
  return grad ? reinterpret_cast<const void *>(&k4_twoshot<1, true, false, false, true>)
              : reinterpret_cast<const void *>(&k4_twoshot<1, false, false, false, true>);
}
// bf16 payload: LSU pushes, one or several workers per GPU
template <bool MULTI>
const void *pick_bf16_t(int mode, bool vec) {
  const bool grad = (mode == SESGD_MODE_GRAD_AVG);
  if (vec)
    return grad ? reinterpret_cast<const void *>(&k4_twoshot<4, true, false, MULTI, false, true>)
                : reinterpret_cast<const void *>(&k4_twoshot<4, false, false, MULTI, false, true>);
  return grad ? reinterpret_cast<const void *>(&k4_twoshot<1, true, false, MULTI, false, true>)
              : reinterpret_cast<const void *>(&k4_twoshot<1, false, false, MULTI, false, true>);
}
const void *pick_bf16(int mode, bool vec, bool multi) {
  return multi ? pick_bf16_t<true>(mode, vec) : pick_bf16_t<false>(mode, vec);
}
// value-carried validity (SESGD_OPT_PROTOCOL = 1): LSU pushes, fp32, one or several workers per GPU
template <bool MULTI>
const void *pick_sent_t(int mode, bool vec) {
  const bool grad = (mode == SESGD_MODE_GRAD_AVG);
  if (vec)
    return grad ? reinterpret_cast<const void *>(&k4_twoshot<4, true, false, MULTI, false, false, true>)
                : reinterpret_cast<const void *>(&k4_twoshot<4, false, false, MULTI, false, false, true>);
  return grad ? reinterpret_cast<const void *>(&k4_twoshot<1, true, false, MULTI, false, false, true>)
              : reinterpret_cast<const void *>(&k4_twoshot<1, false, false, MULTI, false, false, true>);
}
// TMA pushes: one worker per GPU only; several workers per GPU: the MULTI kernel
const void *pick_twoshot(int mode, bool vec, bool tma, bool multi) {
  if (tma) return pick_twoshot_t<true, false>(mode, vec);
  return multi ? pick_twoshot_t<false, true>(mode, vec) : pick_twoshot_t<false, false>(mode, vec);
}

// variant 0: DIRECT push from the compute CTAs; variant >= 1: that many COMM CTAs
const void *pick(int variant, int mode, bool vec) {
  const bool grad = (mode == SESGD_MODE_GRAD_AVG);
  if (variant == 0) {
    if (vec)
      return grad ? reinterpret_cast<const void *>(&k3_direct<4, true>)
                  : reinterpret_cast<const void *>(&k3_direct<4, false>);
    return grad ? reinterpret_cast<const void *>(&k3_direct<1, true>)
                : reinterpret_cast<const void *>(&k3_direct<1, false>);
  }
  if (vec)
    return grad ? reinterpret_cast<const void *>(&k3_split<4, true>)
                : reinterpret_cast<const void *>(&k3_split<4, false>);
  return grad ? reinterpret_cast<const void *>(&k3_split<1, true>)
              : reinterpret_cast<const void *>(&k3_split<1, false>);
}

}  // namespace

bool p2p_variant_valid(int variant) { return variant >= 0 && variant <= 148; }
int p2p_block_threads(int) { return kThreads; }
int p2p_chunk_elems(int) { return int(kChunk); }
int p2p_guard_pairs_max() { return kMaxGuardPairs; }
size_t p2p_smem_bytes(int variant, int pairs, int grid) {
  if (variant == 0) return 0;  // DIRECT: no COMM ring, no guard cache
  return size_t(kRingBytes) + size_t(kRing) * 8 + size_t(pairs > 0 ? pairs : 0) * size_t(grid) * 8;
}

int p2p_occupancy(int variant, int r, int mode, bool vec, size_t smem) {
  (void)r;
  const void *k = pick(variant, mode, vec);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  int blocks = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k, kThreads, smem) != cudaSuccess)
    return 1;
  return blocks > 0 ? blocks : 1;
}

cudaError_t launch_p2p_oneshot(const P2PArgs &a, int variant, int mode, bool vec, size_t smem,
                               cudaStream_t stream) {
  const void *k = pick(variant, mode, vec);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  void *args[] = {const_cast<P2PArgs *>(&a)};
  // the SM-specialised variant's COMM and COMPUTE CTAs wait on each other: always cooperative
  return launch_persistent(k, unsigned(a.grid), kThreads, args, smem, stream,
                           a.cooperative != 0 || (variant >= 1 && a.m > 1));
}

int p2p_twoshot_occupancy(int mode, bool vec, bool tma, bool multi) {
  int nv = 0;  // the NVLS kernels must fit the same grid
  if (!tma && !multi &&
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nv, pick_nvls(mode, vec), kThreads, 0) == cudaSuccess &&
      nv > 0) {
    int base = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&base, pick_twoshot(mode, vec, false, false), kThreads, 0) ==
            cudaSuccess && base > 0)
      return nv < base ? nv : base;
  }
  const void *k = pick_twoshot(mode, vec, tma, multi);
  const size_t smem = tma ? kTwoshotTmaSmem : 0;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  int blocks = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k, kThreads, smem) != cudaSuccess)
    return 1;
  if (!tma) {  // the value-carried protocol's kernels share the grid
    int sb = 0;
    const void *ks = multi ? pick_sent_t<true>(mode, vec) : pick_sent_t<false>(mode, vec);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&sb, ks, kThreads, 0) == cudaSuccess && sb > 0 && sb < blocks)
      blocks = sb;
  }
  return blocks > 0 ? blocks : 1;
}

cudaError_t launch_p2p_twoshot(const P2PArgs &a, int mode, bool vec, bool tma, cudaStream_t stream) {
  const void *k = a.mc_ws ? pick_nvls(mode, vec)
                 : a.payload_bf16 ? pick_bf16(mode, vec, a.r > 1)
                 : a.protocol == 1 ? (a.r > 1 ? pick_sent_t<true>(mode, vec) : pick_sent_t<false>(mode, vec))
                                   : pick_twoshot(mode, vec, tma, a.r > 1);
  const size_t smem = tma ? kTwoshotTmaSmem : 0;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  void *args[] = {const_cast<P2PArgs *>(&a)};
  return launch_persistent(k, unsigned(a.grid), kThreads, args, smem, stream, a.cooperative != 0);
}

}  // namespace sesgd
