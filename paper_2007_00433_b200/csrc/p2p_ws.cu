// p2p_ws.cu -- K4W: the two-shot group exchange of K4 (same slices, same arithmetic, same
// ascending fold, so the same bits) as a WARP-SPECIALISED persistent kernel with value-carried
// validity (SESGD_OPT_PROTOCOL = 2), one worker per GPU -- the north star's 8-GPU layout and the
// n = m = 2 two-GPU shape.  One CTA per SM; its warps are five roles joined only by data:
//   P (1 warp)    claims chunks dynamically (one global atomic per chunk: a fast SM takes more
//                 chunks, so no CTA waits for a slow one at the end) and loads the chunk's g, v, x
//                 (16 KiB each) with cp.async.bulk into a 3-stage shared-memory ring (mbarrier
//                 complete_tx): every SM keeps two to three chunks of HBM reads in flight;
//   S (8 warps)   the local step from shared memory (Alg.1 lines 3-8: v <- mu v + g,
//                 x_hat <- x - lr v), v back to HBM, its own slice of x_hat into a second ring
//                 for R, the other members' slices pushed to their receive slots over NVLink
//                 (reduce-scatter);
//   R (2 x 4)     two groups, each folding every other chunk: the m contributions of my slice in
//                 ascending member order (own from the x_hat ring, the peers' polled in the
//                 receive slots), / m (Eq. 6; Alg.1 line 11), x to HBM and the mean pushed
//                 to every peer (all-gather);
//   F (2 x 4)     two groups, every other chunk: poll the peers' means of their slices, x to HBM.
// Measured on K4W v1 (profiles/r02_k4w_phases_*.json): with S loading through registers the
// stream was latency-bound (one HBM round trip per chunk, ~4.7 us per chunk per SM) and a single
// R / F group kept only one chunk in flight; the TMA ring and the interleaved groups remove both.
// No flags and no fence on the data path: every receive float is armed with a sentinel NaN and
// polled until the peer's value replaces it (p2p.cu, "value-carried validity"), then re-armed.
// The only system-scope synchronisation is one per-launch counter per rank, bumped (release) by
// every CTA when it is done: a peer must have finished -- re-armed every receive slot of -- its
// launch of call - 2 before this launch writes those slots again (one acquire per peer at start).
// Chunk ids travel from P to S and F through a shared-memory id ring; an id < 0 ends a role.  GRAD mode (Eq. 5): the payload is g, R / F apply the
// momentum update with the group-mean gradient (they load v, x themselves).
#include "common.cuh"
#include "internal.h"
#include "ws_common.cuh"
#include "dev_iter.cuh"

namespace sesgd {
namespace {
using namespace wsx;

constexpr int kWarpsP = 1, kWarpsS = 8, kGroupsR = 2, kWarpsR = 4, kGroupsF = 2, kWarpsF = 4;
constexpr int kThS = kWarpsS * 32, kThR = kWarpsR * 32, kThF = kWarpsF * 32;
constexpr int kWarpsAll = kWarpsP + kWarpsS + kGroupsR * kWarpsR + kGroupsF * kWarpsF;  // 25
constexpr int kThreadsWS = kWarpsAll * 32;                                             // 800
constexpr int kChunkWS = 4096;  // K4's chunking (p2p_chunk_elems): same slices
constexpr int kQL = 3;          // load ring stages (g, v, x of one chunk each)
constexpr int kQX = 4;          // x_hat ring entries (a multiple of kGroupsR)
constexpr int kU = 2;           // vectors in flight per R / F thread
constexpr int kQI = 8;          // chunk-id ring entries (P -> S, F; a multiple of kGroupsF)
static_assert(kQX % kGroupsR == 0, "an x_hat ring entry is always consumed by the same R group");
static_assert(kQI % kGroupsF == 0 && kQI > kQL, "id ring: same F group per entry, deeper than the load ring");

// shared memory: barriers, then the load ring (g, v, x per stage) and the x_hat ring
struct Smem {
  uint64_t full_ld[kQL], empty_ld[kQL], full_x[kQX], empty_x[kQX], full_id[kQI], empty_id[kQI];
  int64_t id[kQI];   // chunk of step k at [k % kQI] (written by P)
  int64_t xid[kQX];  // chunk of the x_hat ring entry (written by S)
};
constexpr size_t kSmemHead = 512;  // >= sizeof(Smem), keeps the rings 128-byte aligned
constexpr size_t kStageBytes = size_t(3) * kChunkWS * 4;

template <int W, bool GRAD>
struct WS {
  static constexpr bool kTma = (W == 4);  // bulk copies need 16-byte aligned buffers
  const P2PArgs &a;
  Smem *sm;
  float *ld_ring;  // [kQL][3][kChunkWS]
  float *x_ring;   // [kQX][cap]
  int cap;
  int me, p, m;
  float inv_m;  // dev::pow2_inverse(m)
  const int8_t *G;
  int64_t nk;  // chunks of this launch (claimed dynamically)
  int gc;
  int cta;     // CTA index within this rank's grid (the pair harness runs two ranks in one grid)

  __device__ WS(const P2PArgs &args, unsigned char *smem) : a(args) {
    me = a.my_workers[0];
    p = a.my_pos[0];
    m = a.m;
    inv_m = dev::pow2_inverse(m);
    G = a.canon + a.group_of[me] * a.m;
    gc = a.grid;
    cta = int(blockIdx.x) % a.grid;
    nk = a.g1 - a.g0;
    sm = reinterpret_cast<Smem *>(smem);
    ld_ring = reinterpret_cast<float *>(smem + kSmemHead);
    x_ring = reinterpret_cast<float *>(smem + kSmemHead + kQL * kStageBytes);
    cap = (kChunkWS - (m - 1) * slice() + 3) & ~3;  // largest slice (the last one)
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
    SESGD_CHECK(b >= 0 && b < a.nbuckets && g >= a.g0 && g < a.g1);
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
    SESGD_CHECK(w >= 0 && w < a.n && pos >= 0 && pos < m && a.worker_rank[w] >= 0);
    char *base = a.ws[(a.experiment & 2) ? a.my_rank : a.worker_rank[w]] + a.recv_off;
    return reinterpret_cast<float *>(base) + (int64_t(a.parity) * m + pos) * a.region_floats;
  }
  __device__ __forceinline__ unsigned long long *counter(int rank, int64_t off) const {
    return ws_counter(a, rank, off);
  }
  __device__ __forceinline__ void wait_value(const float *src, float (&y)[W], int nv, int pos,
                                             uint64_t *spin) const {
    wsx::wait_value<W>(a, cta, me, src, y, nv, pos, spin);
  }

  // ---------------------------------------------------------------- P: TMA loads
  // publish chunk id g for step k to F (and, through the load ring, to S)
  __device__ __forceinline__ void post_id(int64_t k, int64_t g) const {
    const int qi = int(k % kQI);
    if (k >= kQI) mbar_spin(&sm->empty_id[qi], uint32_t((k / kQI - 1) & 1));
    sm->id[qi] = g;
    mbar_arrive(&sm->full_id[qi]);
  }
  __device__ void run_p() const {
    if ((threadIdx.x & 31) != 0) return;
    unsigned long long *claim = counter(a.my_rank, kClaimOff);
    for (int64_t k = 0;; ++k) {
      const uint64_t idx = atomicAdd(claim, 1ull) - a.claim_base;
      const int64_t g = idx < uint64_t(nk) ? a.g0 + int64_t(idx) : -1;
      const int q = int(k % kQL);
      if (k >= kQL) mbar_spin(&sm->empty_ld[q], uint32_t((k / kQL - 1) & 1));
      post_id(k, g);
      if (g < 0) {  // end: S sees it through the load ring, each F group through its own id entry
        dev::mbar_arrive_expect_tx(&sm->full_ld[q], 0);
        post_id(k + 1, -1);
        return;
      }
      if (!kTma) {
        mbar_arrive(&sm->full_ld[q]);
        continue;
      }
      const Ref c = locate(g);
      const uint32_t bytes = uint32_t(c.len / 4) * 16;  // whole float4s; the tail is read by S
      float *st = ld_ring + size_t(q) * 3 * kChunkWS;
      dev::mbar_arrive_expect_tx(&sm->full_ld[q], (GRAD ? 1u : 3u) * bytes);
      if (bytes) {
        dev::bulk_g2s(st, a.bg[c.b] + c.e0, bytes, &sm->full_ld[q]);
        if constexpr (!GRAD) {
          dev::bulk_g2s(st + kChunkWS, a.bv[c.b] + c.e0, bytes, &sm->full_ld[q]);
          dev::bulk_g2s(st + 2 * kChunkWS, a.bx[c.b] + c.e0, bytes, &sm->full_ld[q]);
        }
      }
    }
  }

  // ---------------------------------------------------------------- S: local step + scatter
  __device__ void run_s() const {
    const int t = threadIdx.x - kWarpsP * 32;
    const bool lead = a.prof && t == 0;
    const uint64_t ts = lead ? dev::globaltimer() : 0;
    uint64_t t_wait = 0;
    constexpr int kItems = kChunkWS / W / kThS;
    for (int64_t k = 0;; ++k) {
      const int q = int(k % kQL), qx = int(k % kQX);
      const uint64_t tw = lead ? dev::globaltimer() : 0;
      mbar_spin(&sm->full_ld[q], uint32_t((k / kQL) & 1));
      const int64_t g = sm->id[k % kQI];
      if (g < 0) {  // end: one marker per R group
        for (int64_t kk = k; kk < k + kGroupsR; ++kk) {
          const int qq = int(kk % kQX);
          if (kk >= kQX) mbar_spin(&sm->empty_x[qq], uint32_t((kk / kQX - 1) & 1));
          if ((t & 31) == 0) {
            sm->xid[qq] = -1;
            mbar_arrive(&sm->full_x[qq]);
          }
        }
        break;
      }
      if (k >= kQX) mbar_spin(&sm->empty_x[qx], uint32_t((k / kQX - 1) & 1));
      if (lead) t_wait += dev::globaltimer() - tw;
      const Ref c = locate(g);
      const float *sg = ld_ring + size_t(q) * 3 * kChunkWS;
      float *ent = x_ring + size_t(qx) * cap;
      const int64_t mlo = lo(p, c.len);
      const int S = slice();
      const int64_t len4 = c.len & ~int64_t(3);
      float *xs = a.bx[c.b], *vs = a.bv[c.b];
      const float *gs = a.bg[c.b];
#pragma unroll
      for (int it = 0; it < kItems; ++it) {
        const int64_t o = (int64_t(it) * kThS + t) * W;
        const int nv = int(min(int64_t(W), c.len - o));
        if (nv <= 0) continue;
        const int64_t e = c.e0 + o;
        const bool from_smem = kTma && o + W <= len4;
        float val[W], v[W], x[W];
        if (from_smem) {
          const float4 t4 = *reinterpret_cast<const float4 *>(sg + o);
          val[0] = t4.x; val[W > 1 ? 1 : 0] = t4.y; val[W > 2 ? 2 : 0] = t4.z; val[W > 3 ? 3 : 0] = t4.w;
        } else {
          ldm<W>(gs + e, val, nv);
        }
        if constexpr (!GRAD) {
          if (from_smem) {
            const float4 v4 = *reinterpret_cast<const float4 *>(sg + kChunkWS + o);
            const float4 x4 = *reinterpret_cast<const float4 *>(sg + 2 * kChunkWS + o);
            v[0] = v4.x; v[W > 1 ? 1 : 0] = v4.y; v[W > 2 ? 2 : 0] = v4.z; v[W > 3 ? 3 : 0] = v4.w;
            x[0] = x4.x; x[W > 1 ? 1 : 0] = x4.y; x[W > 2 ? 2 : 0] = x4.z; x[W > 3 ? 3 : 0] = x4.w;
          } else {
            ldm<W>(vs + e, v, nv);
            ldm<W>(xs + e, x, nv);
          }
#pragma unroll
          for (int w = 0; w < W; ++w) {
            v[w] = dev::momentum(a.mu, v[w], dev::decay(val[w], a.wd, x[w]));
            val[w] = dev::sgd(x[w], a.lr, v[w]);  // x_hat
          }
          stm<W>(vs + e, v, nv);
        }
        const int j = min(int(o / S), m - 1);  // owner position (a vector never straddles)
        SESGD_CHECK(o + nv <= hi(j, c.len) && o >= lo(j, c.len));
        if (j == p) {
          SESGD_CHECK(o - mlo >= 0 && o - mlo + nv <= cap);
          if (W == 4 && nv == 4) {
            *reinterpret_cast<float4 *>(ent + (o - mlo)) =
                make_float4(val[0], val[W > 1 ? 1 : 0], val[W > 2 ? 2 : 0], val[W > 3 ? 3 : 0]);
          } else {
#pragma unroll
            for (int w = 0; w < W; ++w)
              if (w < nv) ent[o - mlo + w] = val[w];
          }
        } else {
          push<W>(recv(G[j], p) + c.soff + e, val, nv);  // reduce-scatter over NVLink
        }
      }
      __syncwarp();
      if ((t & 31) == 0) {
        mbar_arrive(&sm->empty_ld[q]);  // the load stage is free for the producer
        sm->xid[qx] = g;
        mbar_arrive(&sm->full_x[qx]);   // my slice's x_hat is ready for R
      }
    }
    if (lead) {
      uint64_t *pr = a.prof + int64_t(cta) * 8;
      pr[0] += dev::globaltimer() - ts;
      pr[4] += t_wait;
    }
  }

  // ---------------------------------------------------------------- R: fold my slice + gather
  __device__ void run_r(int grp, int t) const {
    const bool lead = a.prof && t == 0 && grp == 0;
    const uint64_t ts = lead ? dev::globaltimer() : 0;
    uint64_t t_wait = 0, t_spin = 0;
    uint64_t *spin = lead ? &t_spin : nullptr;
    for (int64_t k = grp;; k += kGroupsR) {
      const int qx = int(k % kQX);
      const uint64_t tw = lead ? dev::globaltimer() : 0;
      mbar_spin(&sm->full_x[qx], uint32_t((k / kQX) & 1));
      if (lead) t_wait += dev::globaltimer() - tw;
      const int64_t g = sm->xid[qx];
      if (g < 0) break;
      const Ref c = locate(g);
      if (k == grp && a.hop_delay_ns) {  // config 4: the all-gather round's injected hop
        const uint64_t t0 = dev::globaltimer();
        while (dev::globaltimer() - t0 < a.hop_delay_ns) {
        }
      }
      const float *ent = x_ring + size_t(qx) * cap;
      const int64_t mlo = lo(p, c.len), mhi = hi(p, c.len);
      SESGD_CHECK(mhi - mlo <= cap && c.soff + c.e0 + mhi <= a.region_floats);
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
              if (nv > 0) ld_rel<W>(src + o, y[u], nv);
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
          for (int w = 0; w < W; ++w) acc[u][w] = dev::mean_rt(acc[u][w], m, inv_m);
          for (int rr = 0; rr < m; ++rr)  // all-gather: my slice's mean to every peer
            if (rr != p) push<W>(recv(G[rr], p) + c.soff + e, acc[u], nv);
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
      if ((t & 31) == 0) mbar_arrive(&sm->empty_x[qx]);
    }
    if (lead) {
      uint64_t *pr = a.prof + int64_t(cta) * 8;
      pr[1] += dev::globaltimer() - ts;
      pr[5] += t_wait;
      pr[6] += t_spin;
    }
  }

  // ---------------------------------------------------------------- F: the peers' slices
  __device__ void run_f(int grp, int t) const {
    const bool lead = a.prof && t == 0 && grp == 0;
    const uint64_t ts = lead ? dev::globaltimer() : 0;
    uint64_t t_spin = 0;
    uint64_t *spin = lead ? &t_spin : nullptr;
    for (int64_t k = grp;; k += kGroupsF) {
      const int qi = int(k % kQI);
      mbar_spin(&sm->full_id[qi], uint32_t((k / kQI) & 1));
      const int64_t g = sm->id[qi];
      __syncwarp();
      if ((t & 31) == 0) mbar_arrive(&sm->empty_id[qi]);  // the id is read: P may reuse the entry
      if (g < 0) break;
      const Ref c = locate(g);
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
            if (nv > 0) ld_rel<W>(src + o, y[u], nv);
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
      uint64_t *pr = a.prof + int64_t(cta) * 8;
      pr[3] += dev::globaltimer() - ts;
      pr[2] += t_spin;
      pr[7] += 1;
    }
  }

  // m == 1: no exchange, the local step is the whole update
  __device__ void local_only() const {
    for (int64_t g = a.g0 + cta; g < a.g1; g += a.grid) {
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

template <int W, bool GRAD>
__device__ __forceinline__ void k4w_body(const P2PArgs &a, unsigned char *dsmem) {
  const WS<W, GRAD> s(a, dsmem);
  if (s.cta == 0 && threadIdx.x == 0) count(a.counters, kCntLaunches);
  if (a.m == 1) {
    s.local_only();
    return;
  }
  if (threadIdx.x == 0) {
    for (int q = 0; q < kQL; ++q) {
      dev::mbar_init(&s.sm->full_ld[q], 1);
      dev::mbar_init(&s.sm->empty_ld[q], kWarpsS);
    }
    for (int q = 0; q < kQX; ++q) {
      dev::mbar_init(&s.sm->full_x[q], kWarpsS);
      dev::mbar_init(&s.sm->empty_x[q], kWarpsR);
    }
    for (int q = 0; q < kQI; ++q) {
      dev::mbar_init(&s.sm->full_id[q], 1);
      dev::mbar_init(&s.sm->empty_id[q], kWarpsF);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // guard: every peer has finished (and so re-armed every receive slot of) its launch of call - 2
  if (a.prev2_seq >= 0 && threadIdx.x < 32)
    for (int j = threadIdx.x; j < a.m; j += 32)
      if (j != s.p) wait_done(a, s.cta, a.worker_rank[s.G[j]], s.G[j], j);
  __syncthreads();
  if (a.hop_delay_ns) {  // injected per-hop latency (config 4): the reduce-scatter round's hop
    if (threadIdx.x == 0) {
      const uint64_t t0 = dev::globaltimer();
      while (dev::globaltimer() - t0 < a.hop_delay_ns) {
      }
    }
    __syncthreads();
  }
  const int warp = threadIdx.x >> 5;
  constexpr int kR0 = kWarpsP + kWarpsS, kF0 = kR0 + kGroupsR * kWarpsR;
  if (warp < kWarpsP) {
    s.run_p();
  } else if (warp < kR0) {
    s.run_s();
  } else if (warp < kF0) {
    const int w = warp - kR0;
    s.run_r(w / kWarpsR, (w % kWarpsR) * 32 + (threadIdx.x & 31));
  } else {
    const int w = warp - kF0;
    s.run_f(w / kWarpsF, (w % kWarpsF) * 32 + (threadIdx.x & 31));
  }
  __syncthreads();  // every re-arm of this CTA precedes the release (cumulativity)
  if (threadIdx.x == 0) signal_done(a);
}

template <int W, bool GRAD>
__global__ void __launch_bounds__(kThreadsWS, 1) k4w_twoshot(const __grid_constant__ P2PArgs a) {
  extern __shared__ __align__(128) unsigned char dsmem[];
  k4w_body<W, GRAD>(a, dsmem);
}

// device-resident iteration state (SESGD_OPT_DEVICE_ITER): the per-call fields and the schedule
// come from device memory (dev_iter.cuh), so one captured graph replays every iteration
template <int W, bool GRAD>
__global__ void __launch_bounds__(kThreadsWS, 1) k4w_twoshot_dev(const __grid_constant__ P2PArgs a) {
  extern __shared__ __align__(128) unsigned char dsmem[];
  __shared__ P2PArgs sa;
  devit::load_patched(a, sa);
  __syncthreads();
  k4w_body<W, GRAD>(sa, dsmem);
  if (threadIdx.x == 0) devit::finish(sa);
}

// measurement harness (sesgd_sync_all_pair): two loopback virtual ranks of one GPU in ONE grid --
// CTAs [0, a0.grid) are rank a0's, the rest rank a1's -- so a profiler that serialises kernel
// launches (ncu) sees the whole exchange in one kernel.  Same body, same bits.
template <int W, bool GRAD>
__global__ void __launch_bounds__(kThreadsWS, 1) k4w_pair(const __grid_constant__ P2PArgs a0,
                                                          const __grid_constant__ P2PArgs a1) {
  extern __shared__ __align__(128) unsigned char dsmem[];
  if (int(blockIdx.x) < a0.grid)
    k4w_body<W, GRAD>(a0, dsmem);
  else
    k4w_body<W, GRAD>(a1, dsmem);
}

const void *pick_ws(int mode, bool vec, bool devi = false) {
  const bool grad = (mode == SESGD_MODE_GRAD_AVG);
  if (devi) {
    if (vec)
      return grad ? reinterpret_cast<const void *>(&k4w_twoshot_dev<4, true>)
                  : reinterpret_cast<const void *>(&k4w_twoshot_dev<4, false>);
    return grad ? reinterpret_cast<const void *>(&k4w_twoshot_dev<1, true>)
                : reinterpret_cast<const void *>(&k4w_twoshot_dev<1, false>);
  }
  if (vec)
    return grad ? reinterpret_cast<const void *>(&k4w_twoshot<4, true>)
                : reinterpret_cast<const void *>(&k4w_twoshot<4, false>);
  return grad ? reinterpret_cast<const void *>(&k4w_twoshot<1, true>)
              : reinterpret_cast<const void *>(&k4w_twoshot<1, false>);
}

size_t ws_smem(int m) {
  const int slice = (kChunkWS / (m > 0 ? m : 1)) & ~31;
  const int cap = (kChunkWS - (m - 1) * slice + 3) & ~3;
  return kSmemHead + size_t(kQL) * kStageBytes + size_t(kQX) * size_t(cap) * 4;
}

}  // namespace

int p2p_ws_threads() { return kThreadsWS; }

int p2p_ws_occupancy(int m) {
  static_assert(sizeof(Smem) <= kSmemHead, "barrier block");
  const size_t smem = ws_smem(m);
  int occ = 1 << 30;
  for (int mode = 0; mode < 2; ++mode)
    for (int vec = 0; vec < 4; ++vec) {  // bit 1: the device-iteration variant
      const void *k = pick_ws(mode, (vec & 1) != 0, (vec & 2) != 0);
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      int b = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k, kThreadsWS, smem) != cudaSuccess) b = 1;
      occ = b < occ ? b : occ;
    }
  return occ > 0 ? occ : 1;
}

cudaError_t launch_p2p_ws_pair(const P2PArgs &a0, const P2PArgs &a1, int mode, bool vec, cudaStream_t stream) {
  const bool grad = (mode == SESGD_MODE_GRAD_AVG);
  const void *k = vec ? (grad ? reinterpret_cast<const void *>(&k4w_pair<4, true>)
                              : reinterpret_cast<const void *>(&k4w_pair<4, false>))
                      : (grad ? reinterpret_cast<const void *>(&k4w_pair<1, true>)
                              : reinterpret_cast<const void *>(&k4w_pair<1, false>));
  const size_t smem = ws_smem(a0.m);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  void *args[] = {const_cast<P2PArgs *>(&a0), const_cast<P2PArgs *>(&a1)};
  return launch_persistent(k, unsigned(a0.grid + a1.grid), kThreadsWS, args, smem, stream, false);
}

cudaError_t launch_p2p_ws(const P2PArgs &a, int mode, bool vec, cudaStream_t stream) {
  const void *k = pick_ws(mode, vec, a.dev != nullptr);
  const size_t smem = ws_smem(a.m);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  void *args[] = {const_cast<P2PArgs *>(&a)};
  return launch_persistent(k, unsigned(a.grid), kThreadsWS, args, smem, stream, a.cooperative != 0);
}

}  // namespace sesgd
