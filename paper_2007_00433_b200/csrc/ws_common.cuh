// ws_common.cuh -- device helpers of the warp-specialised two-shot kernels (p2p_ws.cu: K4W, one
// worker per GPU; p2p_wsm.cu: K4W-M, several workers per GPU): value-carried validity (a receive
// float holds kSentinelWS until the peer's value lands, p2p.cu), 128-bit HBM accesses, mbarrier
// spins, and the per-rank chunk-claim / launch-done counters in the workspace header.
#pragma once
#include "common.cuh"
#include "internal.h"

namespace sesgd {
namespace wsx {

constexpr int64_t kClaimOff = 64, kDoneOff = 72;  // workspace header words: claim / done counters
constexpr uint32_t kSentinelWS = 0xFFFFFFFFu;    // as p2p.cu's kSentinel
constexpr int kWaitDataWS = 6;

__device__ __forceinline__ float unsent(float v) {
  return __float_as_uint(v) == kSentinelWS ? __uint_as_float(0x7FFFFFFFu) : v;
}
template <int W>
__device__ __forceinline__ void ldm(const float *p, float (&r)[W], int nv) {
  if constexpr (W == 4) {
    if (nv >= 4) {
      const float4 t = dev::ld4(p);
      r[0] = t.x; r[1] = t.y; r[2] = t.z; r[3] = t.w;
      return;
    }
  }
#pragma unroll
  for (int w = 0; w < W; ++w) r[w] = (w < nv) ? __ldcs(p + w) : 0.f;
}
template <int W>
__device__ __forceinline__ void stm(float *p, const float (&r)[W], int nv) {
  if constexpr (W == 4) {
    if (nv >= 4) {
      dev::st4(p, make_float4(r[0], r[1], r[2], r[3]));
      return;
    }
  }
#pragma unroll
  for (int w = 0; w < W; ++w)
    if (w < nv) __stcs(p + w, r[w]);
}
// NVLink push of a payload vector: relaxed system-scope stores (the receiver polls the values)
template <int W>
__device__ __forceinline__ void push(float *p, const float (&r)[W], int nv) {
  if constexpr (W == 4) {
    if (nv >= 4) {
      asm volatile("st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(unsent(r[0])),
                   "f"(unsent(r[1])), "f"(unsent(r[2])), "f"(unsent(r[3]))
                   : "memory");
      return;
    }
  }
#pragma unroll
  for (int w = 0; w < W; ++w)
    if (w < nv) asm volatile("st.relaxed.sys.global.f32 [%0], %1;" ::"l"(p + w), "f"(unsent(r[w])) : "memory");
}
template <int W>
__device__ __forceinline__ void ld_rel(const float *p, float (&r)[W], int nv) {
  if constexpr (W == 4) {
    if (nv >= 4) {
      asm volatile("ld.relaxed.sys.global.v4.f32 {%0, %1, %2, %3}, [%4];"
                   : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3])
                   : "l"(p)
                   : "memory");
      return;
    }
  }
#pragma unroll
  for (int w = 0; w < W; ++w) {
    if (w < nv)
      asm volatile("ld.relaxed.sys.global.f32 %0, [%1];" : "=f"(r[w]) : "l"(p + w) : "memory");
    else
      r[w] = 0.f;
  }
}
template <int W>
__device__ __forceinline__ bool pending(const float (&r)[W], int nv) {
  bool any = false;
#pragma unroll
  for (int w = 0; w < W; ++w) any |= (w < nv) && __float_as_uint(r[w]) == kSentinelWS;
  return any;
}
template <int W>
__device__ __forceinline__ void rearm(float *p, int nv) {
  const float s = __uint_as_float(kSentinelWS);
  if constexpr (W == 4) {
    if (nv >= 4) {
      *reinterpret_cast<float4 *>(p) = make_float4(s, s, s, s);
      return;
    }
  }
#pragma unroll
  for (int w = 0; w < W; ++w)
    if (w < nv) p[w] = s;
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(dev::smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_spin(uint64_t *bar, uint32_t parity) {
  while (!dev::mbar_try_wait_suspend(bar, parity)) {
  }
}

__device__ __forceinline__ unsigned long long *ws_counter(const P2PArgs &a, int rank, int64_t off) {
  return reinterpret_cast<unsigned long long *>(a.ws[rank] + off);
}

// latch a timed-out wait (first CTA to give up) into the host-mapped error block
__device__ __forceinline__ void latch_timeout(const P2PArgs &a, int kind, int cta, uint64_t seen,
                                              uint64_t need, int worker, int pos) {
  if (atomicExch(a.abort_dev, 1u) == 0u) {
    unsigned long long *e = a.err_host;
    e[1] = (unsigned long long)kind;
    e[2] = (unsigned long long)cta;
    e[3] = seen;
    e[4] = need;
    e[5] = (unsigned long long)worker;
    e[6] = (unsigned long long)pos;
    e[7] = (unsigned long long)a.my_rank;
    __threadfence_system();
    atomicExch(e, (unsigned long long)(-SESGD_ETIMEOUT));
    __threadfence_system();
  }
}

// poll a payload vector until it is no longer the sentinel (the caller re-arms it); spin time
// accumulates into *spin when non-null
template <int W>
__device__ __forceinline__ void wait_value(const P2PArgs &a, int cta, int me, const float *src, float (&y)[W],
                                           int nv, int pos, uint64_t *spin) {
  if (!pending<W>(y, nv) || (a.experiment & 2)) return;  // (experiment: nobody writes my slots)
  count(a.counters, kCntValueSpins);
  const uint64_t t0 = dev::globaltimer();
  unsigned nap = 32;  // back off between polls: a polling warp sleeps instead of taking issue slots
  for (;;) {
    __nanosleep(nap);
    nap = nap < 256 ? 2 * nap : 256;
    ld_rel<W>(src, y, nv);
    if (!pending<W>(y, nv)) break;
    if (*reinterpret_cast<volatile unsigned int *>(a.abort_dev)) break;
    if (dev::globaltimer() - t0 > a.timeout_ns) {
      latch_timeout(a, kWaitDataWS, cta, 0, uint64_t(a.call) + 1, me, pos);
      break;
    }
  }
  if (spin) *spin += dev::globaltimer() - t0;
}

// reuse guard: rank `rank` has finished its launch of call - 2 (every CTA of every launch bumps
// the rank's done counter once; launches run in stream order)
__device__ __forceinline__ void wait_done(const P2PArgs &a, int cta, int rank, int worker, int pos) {
  const uint64_t need = uint64_t(a.grid) * uint64_t(a.prev2_seq + 1);
  const uint64_t *f = reinterpret_cast<const uint64_t *>(ws_counter(a, rank, kDoneOff));
  if (dev::ld_acquire_sys(f) >= need) return;
  count(a.counters, kCntFlagSpins);
  const uint64_t t0 = dev::globaltimer();
  while (dev::ld_acquire_sys(f) < need) {
    if (*reinterpret_cast<volatile unsigned int *>(a.abort_dev)) break;
    if (dev::globaltimer() - t0 > a.timeout_ns) {
      latch_timeout(a, 1 /* consumed */, cta, dev::ld_acquire_sys(f), need, worker, pos);
      break;
    }
  }
}

// this CTA is done with the launch (every re-arm before it, cumulativity through the caller's
// __syncthreads)
__device__ __forceinline__ void signal_done(const P2PArgs &a) {
  dev::fence_acq_rel_sys();
  atomicAdd(ws_counter(a, a.my_rank, kDoneOff), 1ull);
}

}  // namespace wsx
}  // namespace sesgd
