// p2p_ws.cu -- K4W: the two-shot group exchange of K4 (same slices, same arithmetic, same
// ascending fold, so the same bits) as a WARP-SPECIALISED persistent kernel with value-carried
// validity (SESGD_OPT_PROTOCOL = 2), one worker per GPU -- the north star's 8-GPU layout and the
// n = m = 2 two-GPU shape.
//
// Why (measured, profiles/r02_k4_experiments.json): K4's CTAs run stage -> reduce -> finish of
// successive chunks in lock step, so every chunk step pays three latency-bound phases and a
// system-scope fence; with NO NVLink payload at all (pushes to local memory) K4 still takes
// 0.24 ms at n = 2 (ResNet-50), against an HBM floor of 0.078 ms.  Here the three phases are
// three warp groups of one CTA (one CTA per SM) that never wait for each other except through
// data:
//   S (16 warps)  streams g, v, x from HBM (Alg.1 lines 3-8: v <- mu v + g, x_hat <- x - lr v),
//                 stores v, keeps its own slice of x_hat in a shared-memory ring and pushes the
//                 other members' slices to their receive slots over NVLink (reduce-scatter);
//   R (4 warps)   per chunk: waits for the ring entry (mbarrier), folds the m contributions of
//                 its slice in ascending member order (own from shared memory, peers' polled in
//                 the receive slots), divides by m (Eq. 6; Alg.1 line 11), stores x and
//                 pushes the mean to every peer (all-gather); frees the ring entry;
//   F (4 warps)   per chunk: polls the peers' means of their slices and stores x.
// No flags and no fence on the data path: every receive float is armed with a sentinel NaN and
// polled until the peer's value replaces it (p2p.cu, "value-carried validity"), then re-armed.
// The only system-scope synchronisation is K4's per-launch `consumed` counter (a peer must have
// re-armed its slots of call - 2 before they are written again), one acquire at the start and
// one release at the end of every CTA.  GRAD mode (Eq. 5): the payload is g and R / F apply the
// momentum update with the group-mean gradient.
#include "common.cuh"
#include "internal.h"

namespace sesgd {
namespace {

// warp-group layouts (S, R, F warps; vectors in flight per R / F thread); 768 threads, 1 CTA/SM
template <int LAY>
struct Lay;
template <>
struct Lay<0> {
  static constexpr int S = 16, R = 4, F = 4, U = 4;
};
template <>
struct Lay<1> {
  static constexpr int S = 8, R = 8, F = 8, U = 2;
};
template <>
struct Lay<2> {  // 640 threads: up to 102 registers (S loads 4 items at once without spills)
  static constexpr int S = 8, R = 6, F = 6, U = 2;
};
template <int LAY>
constexpr int threads_of() { return 32 * (Lay<LAY>::S + Lay<LAY>::R + Lay<LAY>::F); }
constexpr int kChunkWS = 4096;                  // K4's chunking (p2p_chunk_elems): same slices
constexpr int kRing = 8;                        // ring entries (chunks S may run ahead of R)
constexpr uint32_t kSentinelWS = 0xFFFFFFFFu;   // as p2p.cu's kSentinel
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
__device__ __forceinline__ void push(float *p, const float (&r)[W], int nv, bool weak = false) {
  if constexpr (W == 4) {
    if (nv >= 4 && weak) {  // (SESGD_OPT_EXPERIMENT bit 2: measurement only)
      *reinterpret_cast<float4 *>(p) = make_float4(unsent(r[0]), unsent(r[1]), unsent(r[2]), unsent(r[3]));
      return;
    }
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
__device__ __forceinline__ void ld_rel(const float *p, float (&r)[W], int nv, bool weak = false) {
  if constexpr (W == 4) {
    if (nv >= 4 && weak) {  // (SESGD_OPT_EXPERIMENT bit 3: measurement only)
      const float4 t = __ldcg(reinterpret_cast<const float4 *>(p));
      r[0] = t.x; r[1] = t.y; r[2] = t.z; r[3] = t.w;
      return;
    }
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

template <int W, bool GRAD, int LAY>
struct WS {
  static constexpr int kThS = Lay<LAY>::S * 32, kThR = Lay<LAY>::R * 32, kThF = Lay<LAY>::F * 32;
  static constexpr int kU = Lay<LAY>::U;
  static constexpr int kItemsS = kChunkWS / W / kThS;  // W-vectors per S thread per chunk
  const P2PArgs &a;
  int me, p, m;
  const int8_t *G;
  int64_t first, nk;
  int gc;

  __device__ WS(const P2PArgs &args) : a(args) {
    me = a.my_workers[0];
    p = a.my_pos[0];
    m = a.m;
    G = a.canon + a.group_of[me] * a.m;
    gc = a.grid;
    const int i = blockIdx.x;
    first = a.g0 + ((int64_t(i) - a.g0 % gc) % gc + gc) % gc;
    nk = (a.g1 > first) ? (a.g1 - first + gc - 1) / gc : 0;
  }

  struct Ref {
    int b;
    int64_t e0, len, soff;
  };
  __device__ __forceinline__ Ref locate(int64_t g) const {
    int b = a.bucket;
    if (b < 0) {
      int lo = 0, hi = a.nbuckets - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (a.meta[mid].chunk_base <= g) lo = mid; else hi = mid - 1;
      }
      b = lo;
    }
    const BucketMeta &mb = a.meta[b];
    Ref c;
    c.b = b;
    c.e0 = (g - mb.chunk_base) * kChunkWS;
    c.len = min(int64_t(kChunkWS), mb.numel - c.e0);
    c.soff = mb.stage_off;
    return c;
  }
  // K4's slices: position j owns [lo, hi) of every chunk (ts_slice / ts_lo / ts_hi)
  __device__ __forceinline__ int slice() const { return (kChunkWS / m) & ~31; }
  __device__ __forceinline__ int64_t lo(int j, int64_t len) const { return min(int64_t(j) * slice(), len); }
  __device__ __forceinline__ int64_t hi(int j, int64_t len) const {
    return j == m - 1 ? len : min(int64_t(j + 1) * slice(), len);
  }
  // receive slot [pos] of worker w (one worker per rank: slot 0), parity of this call
  __device__ __forceinline__ float *recv(int w, int pos) const {
    char *base = a.ws[(a.experiment & 2) ? a.my_rank : a.worker_rank[w]] + a.recv_off;
    return reinterpret_cast<float *>(base) + (int64_t(a.parity) * m + pos) * a.region_floats;
  }
  __device__ __forceinline__ uint64_t *consumed(int w) const {
    return reinterpret_cast<uint64_t *>(a.ws[a.worker_rank[w]] + a.consumed_off) + blockIdx.x;
  }

  // poll a payload vector until it is no longer the sentinel, then re-arm it
  __device__ __forceinline__ void wait_value(float *src, float (&y)[W], int nv, int pos,
                                             uint64_t *spin = nullptr) const {
    if (!pending<W>(y, nv) || (a.experiment & 2)) return;  // (experiment: nobody writes my slots)
    count(a.counters, kCntValueSpins);
    const uint64_t t0 = dev::globaltimer();
    struct Acc {
      uint64_t *s;
      uint64_t t0;
      __device__ ~Acc() {
        if (s) *s += dev::globaltimer() - t0;
      }
    } acc{spin, t0};
    do {
      if (*reinterpret_cast<volatile unsigned int *>(a.abort_dev)) return;
      if (dev::globaltimer() - t0 > a.timeout_ns) {
        if (atomicExch(a.abort_dev, 1u) == 0u) {
          unsigned long long *e = a.err_host;
          e[1] = (unsigned long long)kWaitDataWS;
          e[2] = blockIdx.x;
          e[3] = 0;
          e[4] = uint64_t(a.call) + 1;
          e[5] = (unsigned long long)me;
          e[6] = (unsigned long long)pos;
          e[7] = (unsigned long long)a.my_rank;
          __threadfence_system();
          atomicExch(e, (unsigned long long)(-SESGD_ETIMEOUT));
          __threadfence_system();
        }
        return;
      }
      ld_rel<W>(src, y, nv, (a.experiment & 8) != 0);
    } while (pending<W>(y, nv));
  }

  // ---------------------------------------------------------------- S: stream + scatter
  __device__ void run_s(float *ring, int cap, uint64_t *full, uint64_t *empty) const {
    const int t = threadIdx.x;
    const bool lead = a.prof && t == 0;
    const uint64_t ts = lead ? dev::globaltimer() : 0;
    uint64_t t_wait = 0;
    for (int64_t k = 0; k < nk; ++k) {
      const Ref c = locate(first + k * gc);
      const int q = int(k % kRing);
      if (k >= kRing) {  // R has folded the entry's previous chunk
        const uint32_t par = uint32_t((k / kRing - 1) & 1);
        const uint64_t tw = lead ? dev::globaltimer() : 0;
        while (!dev::mbar_try_wait(&empty[q], par)) {
        }
        if (lead) t_wait += dev::globaltimer() - tw;
      }
      float *ent = ring + q * cap;
      const int64_t mlo = lo(p, c.len);
      const int S = slice();
      float *xs = a.bx[c.b], *vs = a.bv[c.b];
      const float *gs = a.bg[c.b];
      // every load of the chunk in flight before the first store (one HBM latency per chunk; the
      // compiler cannot hoist loads above stores it cannot prove disjoint)
      float val[kItemsS][W], v[GRAD ? 1 : kItemsS][W], x[GRAD ? 1 : kItemsS][W];
#pragma unroll
      for (int it = 0; it < kItemsS; ++it) {
        const int64_t o = (int64_t(it) * kThS + t) * W;
        const int nv = int(min(int64_t(W), c.len - o));
        if (nv <= 0) continue;
        const int64_t e = c.e0 + o;
        ldm<W>(gs + e, val[it], nv);
        if constexpr (!GRAD) {
          ldm<W>(vs + e, v[it], nv);
          ldm<W>(xs + e, x[it], nv);
        }
      }
#pragma unroll
      for (int it = 0; it < kItemsS; ++it) {
        const int64_t o = (int64_t(it) * kThS + t) * W;
        const int nv = int(min(int64_t(W), c.len - o));
        if (nv <= 0) continue;
        const int64_t e = c.e0 + o;
        if constexpr (!GRAD) {
#pragma unroll
          for (int w = 0; w < W; ++w) {
            v[it][w] = dev::momentum(a.mu, v[it][w], dev::decay(val[it][w], a.wd, x[it][w]));
            val[it][w] = dev::sgd(x[it][w], a.lr, v[it][w]);  // x_hat
          }
          stm<W>(vs + e, v[it], nv);
        }
        const int j = min(int(o / S), m - 1);  // owner position (a vector never straddles)
        if (j == p) {
          if (W == 4 && nv == 4) {
            *reinterpret_cast<float4 *>(ent + (o - mlo)) =
                make_float4(val[it][0], val[it][W > 1 ? 1 : 0], val[it][W > 2 ? 2 : 0], val[it][W > 3 ? 3 : 0]);
          } else {
#pragma unroll
            for (int w = 0; w < W; ++w)
              if (w < nv) ent[o - mlo + w] = val[it][w];
          }
        } else {
          push<W>(recv(G[j], p) + c.soff + e, val[it], nv, (a.experiment & 4) != 0);  // reduce-scatter
        }
      }
      __syncwarp();
      if ((t & 31) == 0) mbar_arrive(&full[q]);
    }
    if (lead) {
      uint64_t *pr = a.prof + int64_t(blockIdx.x) * 8;
      pr[0] += dev::globaltimer() - ts;
      pr[4] += t_wait;
    }
  }

  // ---------------------------------------------------------------- R: fold my slice + gather
  __device__ void run_r(const float *ring, int cap, uint64_t *full, uint64_t *empty) const {
    const int t = threadIdx.x - kThS;
    const bool lead = a.prof && t == 0;
    const uint64_t ts = lead ? dev::globaltimer() : 0;
    uint64_t t_wait = 0, t_spin = 0;
    uint64_t *spin = lead ? &t_spin : nullptr;
    for (int64_t k = 0; k < nk; ++k) {
      const Ref c = locate(first + k * gc);
      const int q = int(k % kRing);
      const uint32_t par = uint32_t((k / kRing) & 1);
      const uint64_t tw = lead ? dev::globaltimer() : 0;
      while (!dev::mbar_try_wait(&full[q], par)) {
      }
      if (lead) t_wait += dev::globaltimer() - tw;
      if (k == 0 && a.hop_delay_ns) {  // config 4: the all-gather round's injected hop
        const uint64_t t0 = dev::globaltimer();
        while (dev::globaltimer() - t0 < a.hop_delay_ns) {
        }
      }
      const float *ent = ring + q * cap;
      const int64_t mlo = lo(p, c.len), mhi = hi(p, c.len);
      float *xs = a.bx[c.b], *vs = a.bv[c.b];
      for (int64_t base = mlo; base < mhi; base += int64_t(kThR) * W * kU) {
        float acc[kU][W];
        for (int rr = 0; rr < m; ++rr) {  // ascending position = ascending worker id
          float y[kU][W];
          if (rr == p) {
#pragma unroll
            for (int u = 0; u < kU; ++u) {
              const int64_t o = base + (int64_t(u) * kThR + t) * W;
              const int nv = int(max(int64_t(0), min(int64_t(W), mhi - o)));
#pragma unroll
              for (int w = 0; w < W; ++w) y[u][w] = (w < nv) ? ent[o - mlo + w] : 0.f;
            }
          } else {
            float *src = recv(me, rr) + c.soff + c.e0;
#pragma unroll
            for (int u = 0; u < kU; ++u) {  // every vector's load in flight first
              const int64_t o = base + (int64_t(u) * kThR + t) * W;
              const int nv = int(max(int64_t(0), min(int64_t(W), mhi - o)));
              if (nv > 0) ld_rel<W>(src + o, y[u], nv, (a.experiment & 8) != 0);
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
              const int64_t o = base + (int64_t(u) * kThR + t) * W;
              const int nv = int(max(int64_t(0), min(int64_t(W), mhi - o)));
              if (nv <= 0) continue;
              wait_value(src + o, y[u], nv, rr, spin);
              rearm<W>(src + o, nv);
            }
          }
#pragma unroll
          for (int u = 0; u < kU; ++u)
#pragma unroll
            for (int w = 0; w < W; ++w) acc[u][w] = (rr == 0) ? y[u][w] : __fadd_rn(acc[u][w], y[u][w]);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int64_t o = base + (int64_t(u) * kThR + t) * W;
          const int nv = int(max(int64_t(0), min(int64_t(W), mhi - o)));
          if (nv <= 0) continue;
          const int64_t e = c.e0 + o;
#pragma unroll
          for (int w = 0; w < W; ++w) acc[u][w] = __fdiv_rn(acc[u][w], float(m));
          for (int rr = 0; rr < m; ++rr)  // all-gather: my slice's mean to every peer
            if (rr != p) push<W>(recv(G[rr], p) + c.soff + e, acc[u], nv, (a.experiment & 4) != 0);
          if constexpr (!GRAD) {
            stm<W>(xs + e, acc[u], nv);
          } else {
            float v[W], x[W];
            ldm<W>(vs + e, v, nv);
            ldm<W>(xs + e, x, nv);
#pragma unroll
            for (int w = 0; w < W; ++w) {
              v[w] = dev::momentum(a.mu, v[w], dev::decay(acc[u][w], a.wd, x[w]));
              x[w] = dev::sgd(x[w], a.lr, v[w]);
            }
            stm<W>(vs + e, v, nv);
            stm<W>(xs + e, x, nv);
          }
        }
      }
      __syncwarp();
      if ((t & 31) == 0) mbar_arrive(&empty[q]);
    }
    if (lead) {
      uint64_t *pr = a.prof + int64_t(blockIdx.x) * 8;
      pr[1] += dev::globaltimer() - ts;
      pr[5] += t_wait;
      pr[6] += t_spin;
    }
  }

  // ---------------------------------------------------------------- F: the peers' slices
  __device__ void run_f() const {
    const int t = threadIdx.x - kThS - kThR;
    const bool lead = a.prof && t == 0;
    const uint64_t ts = lead ? dev::globaltimer() : 0;
    uint64_t t_spin = 0;
    uint64_t *spin = lead ? &t_spin : nullptr;
    for (int64_t k = 0; k < nk; ++k) {
      const Ref c = locate(first + k * gc);
      float *xs = a.bx[c.b], *vs = a.bv[c.b];
      for (int j = 0; j < m; ++j) {
        if (j == p) continue;
        const int64_t jlo = lo(j, c.len), jhi = hi(j, c.len);
        float *src = recv(me, j) + c.soff + c.e0;
        for (int64_t base = jlo; base < jhi; base += int64_t(kThF) * W * kU) {
          float y[kU][W];
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const int64_t o = base + (int64_t(u) * kThF + t) * W;
            const int nv = int(max(int64_t(0), min(int64_t(W), jhi - o)));
            if (nv > 0) ld_rel<W>(src + o, y[u], nv, (a.experiment & 8) != 0);
          }
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const int64_t o = base + (int64_t(u) * kThF + t) * W;
            const int nv = int(max(int64_t(0), min(int64_t(W), jhi - o)));
            if (nv <= 0) continue;
            wait_value(src + o, y[u], nv, j, spin);
            rearm<W>(src + o, nv);
            const int64_t e = c.e0 + o;
            if constexpr (!GRAD) {
              stm<W>(xs + e, y[u], nv);
            } else {
              float v[W], x[W];
              ldm<W>(vs + e, v, nv);
              ldm<W>(xs + e, x, nv);
#pragma unroll
              for (int w = 0; w < W; ++w) {
                v[w] = dev::momentum(a.mu, v[w], dev::decay(y[u][w], a.wd, x[w]));
                x[w] = dev::sgd(x[w], a.lr, v[w]);
              }
              stm<W>(vs + e, v, nv);
              stm<W>(xs + e, x, nv);
            }
          }
        }
      }
    }
    if (lead) {
      uint64_t *pr = a.prof + int64_t(blockIdx.x) * 8;
      pr[3] += dev::globaltimer() - ts;
      pr[2] += t_spin;
      pr[7] += 1;
    }
  }

  // m == 1: no exchange, the local step is the whole update
  __device__ void local_only() const {
    for (int64_t g = a.g0 + blockIdx.x; g < a.g1; g += a.grid) {
      const Ref c = locate(g);
      float *xs = a.bx[c.b], *vs = a.bv[c.b];
      const float *gs = a.bg[c.b];
      for (int64_t o = int64_t(threadIdx.x) * W; o < c.len; o += int64_t(blockDim.x) * W) {
        const int nv = int(min(int64_t(W), c.len - o));
        const int64_t e = c.e0 + o;
        float gr[W], v[W], x[W];
        ldm<W>(gs + e, gr, nv);
        ldm<W>(vs + e, v, nv);
        ldm<W>(xs + e, x, nv);
#pragma unroll
        for (int w = 0; w < W; ++w) {
          v[w] = dev::momentum(a.mu, v[w], dev::decay(gr[w], a.wd, x[w]));
          x[w] = dev::sgd(x[w], a.lr, v[w]);
        }
        stm<W>(vs + e, v, nv);
        stm<W>(xs + e, x, nv);
      }
    }
  }
};

template <int W, bool GRAD, int LAY>
__global__ void __launch_bounds__(threads_of<LAY>(), 1) k4w_twoshot(const __grid_constant__ P2PArgs a) {
  extern __shared__ __align__(128) unsigned char dsmem[];
  using L = Lay<LAY>;
  const WS<W, GRAD, LAY> s(a);
  if (blockIdx.x == 0 && threadIdx.x == 0) count(a.counters, kCntLaunches);
  if (a.m == 1) {
    s.local_only();
    return;
  }
  if (s.nk == 0) return;
  const int cap = (kChunkWS - (a.m - 1) * s.slice() + 3) & ~3;  // largest slice (the last one)
  uint64_t *full = reinterpret_cast<uint64_t *>(dsmem);
  uint64_t *empty = full + kRing;
  float *ring = reinterpret_cast<float *>(dsmem + 2 * kRing * sizeof(uint64_t));
  if (threadIdx.x == 0) {
    for (int q = 0; q < kRing; ++q) {
      dev::mbar_init(&full[q], L::S);
      dev::mbar_init(&empty[q], L::R);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // guard: every peer re-armed its receive slots of call - 2 for my chunks (its CTA i polls
  // exactly my CTA i's chunks); one acquire per peer and launch
  if (a.call >= 2 && threadIdx.x < 32) {
    const uint64_t need = a.prev2_epoch0 + uint64_t((s.first + (s.nk - 1) * s.gc) / s.gc);
    for (int j = threadIdx.x; j < a.m; j += 32) {
      if (j == s.p) continue;
      const uint64_t *f = s.consumed(s.G[j]);
      if (dev::ld_acquire_sys(f) >= need) continue;
      const uint64_t t0 = dev::globaltimer();
      while (dev::ld_acquire_sys(f) < need) {
        if (*reinterpret_cast<volatile unsigned int *>(a.abort_dev)) break;
        if (dev::globaltimer() - t0 > a.timeout_ns) {
          if (atomicExch(a.abort_dev, 1u) == 0u) {
            unsigned long long *e = a.err_host;
            e[1] = 1;  // consumed
            e[2] = blockIdx.x;
            e[3] = dev::ld_acquire_sys(f);
            e[4] = need;
            e[5] = (unsigned long long)s.G[j];
            e[6] = (unsigned long long)j;
            e[7] = (unsigned long long)a.my_rank;
            __threadfence_system();
            atomicExch(e, (unsigned long long)(-SESGD_ETIMEOUT));
            __threadfence_system();
          }
          break;
        }
      }
    }
  }
  __syncthreads();
  if (a.hop_delay_ns) {  // injected per-hop latency (config 4): once per handshake round
    if (threadIdx.x == 0) {
      const uint64_t t0 = dev::globaltimer();
      while (dev::globaltimer() - t0 < a.hop_delay_ns) {
      }
    }
    __syncthreads();
  }
  const int warp = threadIdx.x >> 5;
  if (warp < L::S)
    s.run_s(ring, cap, full, empty);
  else if (warp < L::S + L::R)
    s.run_r(ring, cap, full, empty);
  else
    s.run_f();
  __syncthreads();  // every re-arm of this CTA precedes the release (cumulativity)
  if (threadIdx.x == 0)
    dev::st_release_sys(s.consumed(s.me), a.seq_epoch0 + uint64_t((s.first + (s.nk - 1) * s.gc) / s.gc));
}

template <int LAY>
const void *pick_ws_t(int mode, bool vec) {
  const bool grad = (mode == SESGD_MODE_GRAD_AVG);
  if (vec)
    return grad ? reinterpret_cast<const void *>(&k4w_twoshot<4, true, LAY>)
                : reinterpret_cast<const void *>(&k4w_twoshot<4, false, LAY>);
  return grad ? reinterpret_cast<const void *>(&k4w_twoshot<1, true, LAY>)
              : reinterpret_cast<const void *>(&k4w_twoshot<1, false, LAY>);
}
const void *pick_ws(int mode, bool vec, int lay) {
  return lay == 2 ? pick_ws_t<2>(mode, vec) : lay == 1 ? pick_ws_t<1>(mode, vec) : pick_ws_t<0>(mode, vec);
}
int ws_threads(int lay) {
  return lay == 2 ? threads_of<2>() : lay == 1 ? threads_of<1>() : threads_of<0>();
}
// layout of this launch (SESGD_OPT_EXPERIMENT bits 4/5 select 1/2: measurement only)
int ws_layout(const P2PArgs &a) { return (a.experiment & 32) ? 2 : (a.experiment & 16) ? 1 : 0; }

size_t ws_smem(int m) {
  const int slice = (kChunkWS / (m > 0 ? m : 1)) & ~31;
  const int cap = (kChunkWS - (m - 1) * slice + 3) & ~3;
  return 2 * kRing * sizeof(uint64_t) + size_t(kRing) * size_t(cap) * 4;
}

}  // namespace

int p2p_ws_threads() { return ws_threads(0); }

int p2p_ws_occupancy(int m) {
  const size_t smem = ws_smem(m);
  int occ = 1 << 30;
  for (int mode = 0; mode < 2; ++mode)
    for (int vec = 0; vec < 2; ++vec) {
      for (int lay = 0; lay < 3; ++lay) {
      const void *k = pick_ws(mode, vec != 0, lay);
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      int b = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k, ws_threads(lay), smem) != cudaSuccess) b = 1;
      occ = b < occ ? b : occ;
      }
    }
  return occ > 0 ? occ : 1;
}

cudaError_t launch_p2p_ws(const P2PArgs &a, int mode, bool vec, cudaStream_t stream) {
  const int lay = ws_layout(a);
  const void *k = pick_ws(mode, vec, lay);
  const size_t smem = ws_smem(a.m);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  void *args[] = {const_cast<P2PArgs *>(&a)};
  return launch_persistent(k, unsigned(a.grid), unsigned(ws_threads(lay)), args, smem, stream, a.cooperative != 0);
}

}  // namespace sesgd
