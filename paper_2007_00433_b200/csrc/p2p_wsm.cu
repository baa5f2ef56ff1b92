// p2p_wsm.cu -- K4W-M: the warp-specialised two-shot exchange (K4W, p2p_ws.cu) for SEVERAL
// workers per GPU (r = 2..8; SESGD_OPT_PROTOCOL 2 with r > 1).  Same slices, arithmetic and
// ascending fold as K4 / K4W, so the same bits.  A unit of work is one piece (<= `sub` floats) of
// one member position's slice j of one chunk, for every local worker at once:
//   P (1 warp)   claims units dynamically and cp.async.bulk-loads g, v, x of the piece for all r
//                local workers into a 3-stage shared-memory ring;
//   S (8 warps)  per local worker s: an all-local group (every member on this GPU) is updated
//                entirely here (fold of the members' x_hat in registers, the 1-GPU kernel's
//                arithmetic); in a group with remote members, x_hat (or g in GRAD mode) is pushed to
//                the slice's owner when it is remote, or kept in the x_hat ring when the owner is a
//                local worker (itself or a co-resident member);
//   R (2 x 4)    per unit, for every local worker that OWNS slice j of its group: fold the m
//                contributions in ascending member order (local ones from the x_hat ring, remote
//                ones polled in the receive slots), / m, apply to the local members, push the mean
//                to the remote ones (all-gather);
//   F (2 x 4)    per unit, for every local worker whose slice-j owner is remote: poll the mean.
// Value-carried validity and the per-rank done counter as in K4W (ws_common.cuh).
#include "common.cuh"
#include "internal.h"
#include "ws_common.cuh"
#include "dev_iter.cuh"

namespace sesgd {
namespace {
using namespace wsx;

// 25 warps: P (1), S (ws_s), R (2 groups) and F (2 groups) sharing the other 24 - ws_s equally.
// S streams every local worker's data (r items per vector); R and F only touch the groups that
// span GPUs (SESGD_OPT_WS_SPLIT: ws_s = 8 -- the default, measured best -- 12 or 16)
constexpr int kWarpsP = 1, kGroupsR = 2, kGroupsF = 2, kWarpsRest = 24;
constexpr int kThreadsWSM = (kWarpsP + kWarpsRest) * 32;  // 800
constexpr int kChunkWSM = 4096;  // K4's chunking: same slices
constexpr int kQL = 3, kQX = 4, kQI = 8;
constexpr int kU = 2;            // vectors in flight per R / F thread
constexpr int kMaxR = 8;         // local workers supported (else K4)
static_assert(kQX % kGroupsR == 0 && kQI % kGroupsF == 0 && kQI > kQL, "ring depths");

// a decoded unit: bucket b, slice j, chunk start e0 (bucket element), stage offset of the bucket,
// piece [plo, phi) of the chunk.  P decodes each claimed unit ONCE and publishes it with the id
// (a 64-bit division and a bucket search per unit; every S / R / F thread used to redo them)
struct UnitM {
  int b, j;
  int64_t e0, soff, plo, phi;
};
struct SmemM {
  uint64_t full_ld[kQL], empty_ld[kQL], full_x[kQX], empty_x[kQX], full_id[kQI], empty_id[kQI];
  int64_t uid[kQI];   // unit of step k (P -> S, F); < 0 ends the role
  int64_t xuid[kQX];  // unit of the x_hat ring entry (S -> R)
  UnitM unit[kQI];    // decoded uid[]
  UnitM xunit[kQX];   // decoded xuid[]
};
constexpr size_t kHeadM = 1024;

__host__ __device__ inline int sub_of(int r) { return r <= 4 ? 1024 : 512; }

template <int W, bool GRAD>
struct WSM {
  static constexpr bool kTma = (W == 4);
  const P2PArgs &a;
  SmemM *sm;
  float *ld_ring;  // [kQL][r][3][sub]
  float *x_ring;   // [kQX][r][sub]
  int r, m, sub, upc, cta;
  int kWarpsS, kWarpsR, kWarpsF, kThS, kThR, kThF;  // the warp split (a.ws_split)
  float inv_m;  // dev::pow2_inverse(m)
  int64_t nunits;

  __device__ WSM(const P2PArgs &args, unsigned char *smem) : a(args) {
    r = a.r;
    m = a.m;
    kWarpsS = a.ws_split;
    kWarpsR = kWarpsF = (kWarpsRest - kWarpsS) / 4;
    kThS = kWarpsS * 32;
    kThR = kWarpsR * 32;
    kThF = kWarpsF * 32;
    inv_m = dev::pow2_inverse(m);
    sub = sub_of(r);
    cta = int(blockIdx.x) % a.grid;
    sm = reinterpret_cast<SmemM *>(smem);
    ld_ring = reinterpret_cast<float *>(smem + kHeadM);
    x_ring = ld_ring + size_t(kQL) * r * 3 * sub;
    upc = 0;
    for (int j = 0; j < m; ++j) upc += int((hi(j, kChunkWSM) - lo(j, kChunkWSM) + sub - 1) / sub);
    nunits = (a.g1 - a.g0) * upc;
  }

  __device__ __forceinline__ int slice() const { return (kChunkWSM / m) & ~31; }
  __device__ __forceinline__ int64_t lo(int j, int64_t len) const { return min(int64_t(j) * slice(), len); }
  __device__ __forceinline__ int64_t hi(int j, int64_t len) const {
    return j == m - 1 ? len : min(int64_t(j + 1) * slice(), len);
  }
  using Unit = UnitM;  // the piece is [plo, phi) of the chunk (may be empty)
  __device__ __forceinline__ Unit decode(int64_t u) const {
    const int64_t g = a.g0 + u / upc;
    int p = int(u % upc);
    int b = a.bucket;
    if (b < 0) {
      int l = 0, h = a.nbuckets - 1;
      while (l < h) {
        const int mid = (l + h + 1) >> 1;
        if (a.meta[mid].chunk_base <= g) l = mid; else h = mid - 1;
      }
      b = l;
    }
    SESGD_CHECK(b >= 0 && b < a.nbuckets && g >= a.g0 && g < a.g1);
    const BucketMeta &mb = a.meta[b];
    Unit x;
    x.b = b;
    x.e0 = (g - mb.chunk_base) * kChunkWSM;
    x.soff = mb.stage_off;
    const int64_t len = min(int64_t(kChunkWSM), mb.numel - x.e0);
    x.j = 0;
    for (int j = 0; j < m; ++j) {  // piece p of the full chunk's slice enumeration
      const int np = int((hi(j, kChunkWSM) - lo(j, kChunkWSM) + sub - 1) / sub);
      if (p < np) {
        x.j = j;
        const int64_t fl = lo(j, kChunkWSM) + int64_t(p) * sub;
        const int64_t fh = min(fl + sub, hi(j, kChunkWSM));
        // the same slice of a ragged chunk: K4's bounds, clipped to the chunk
        const int64_t sl = lo(j, len), sh = hi(j, len);
        x.plo = min(max(fl, sl), sh);
        x.phi = (j == m - 1 && p == np - 1) ? sh : min(max(fh, sl), sh);
        break;
      }
      p -= np;
    }
    return x;
  }
  __device__ __forceinline__ const int8_t *group(int w) const { return a.canon + a.group_of[w] * m; }
  __device__ __forceinline__ bool local(int w) const { return a.worker_rank[w] == a.my_rank; }
  __device__ __forceinline__ float *recv(int w, int pos) const {
    SESGD_CHECK(w >= 0 && w < a.n && pos >= 0 && pos < m);
    char *base = a.ws[(a.experiment & 2) ? a.my_rank : a.worker_rank[w]] + a.recv_off;
    const int64_t region = (int64_t(a.parity) * r + a.worker_slot[w]) * m + pos;
    return reinterpret_cast<float *>(base) + region * a.region_floats;
  }
  __device__ __forceinline__ float *stage(int q, int s, int arr) const {
    return ld_ring + ((size_t(q) * r + s) * 3 + arr) * sub;
  }
  __device__ __forceinline__ float *xent(int q, int s) const { return x_ring + (size_t(q) * r + s) * sub; }

  __device__ __forceinline__ void post_id(int64_t k, int64_t u, const Unit *x = nullptr) const {
    const int qi = int(k % kQI);
    if (k >= kQI) mbar_spin(&sm->empty_id[qi], uint32_t((k / kQI - 1) & 1));
    sm->uid[qi] = u;
    if (x) sm->unit[qi] = *x;
    mbar_arrive(&sm->full_id[qi]);
  }

  // spanning_only: the all-local groups are updated by a K6 launch before this one (the hybrid
  // launch of sesgd_capi.cu, SESGD_OPT_WSM_HYBRID), so their slots are neither loaded nor streamed
  __device__ __forceinline__ bool skip(int s) const { return a.wsm_spanning_only && a.slot_kind[s] != 0; }

  // ---------------------------------------------------------------- P
  __device__ void run_p() const {
    if ((threadIdx.x & 31) != 0) return;
    unsigned long long *claim = ws_counter(a, a.my_rank, kClaimOff);
    for (int64_t k = 0;; ++k) {
      const uint64_t idx = atomicAdd(claim, 1ull) - a.claim_base;
      const int64_t u = idx < uint64_t(nunits) ? int64_t(idx) : -1;
      const int q = int(k % kQL);
      if (k >= kQL) mbar_spin(&sm->empty_ld[q], uint32_t((k / kQL - 1) & 1));
      Unit x{};
      if (u >= 0) x = decode(u);
      post_id(k, u, &x);
      if (u < 0) {
        dev::mbar_arrive_expect_tx(&sm->full_ld[q], 0);
        post_id(k + 1, -1);
        return;
      }
      if (!kTma) {
        mbar_arrive(&sm->full_ld[q]);
        continue;
      }
      const uint32_t bytes = uint32_t((x.phi - x.plo) / 4) * 16;  // whole float4s; tails via S
      uint32_t tx = 0;
      for (int s = 0; s < r; ++s)
        if (!skip(s)) tx += bytes * ((GRAD && a.slot_kind[s] == 0) ? 1u : 3u);
      dev::mbar_arrive_expect_tx(&sm->full_ld[q], tx);
      if (bytes) {
        for (int s = 0; s < r; ++s) {
          if (skip(s)) continue;
          const int64_t off = x.e0 + x.plo;
          dev::bulk_g2s(stage(q, s, 0), a.bg[x.b * r + s] + off, bytes, &sm->full_ld[q]);
          if (!(GRAD && a.slot_kind[s] == 0)) {
            dev::bulk_g2s(stage(q, s, 1), a.bv[x.b * r + s] + off, bytes, &sm->full_ld[q]);
            dev::bulk_g2s(stage(q, s, 2), a.bx[x.b * r + s] + off, bytes, &sm->full_ld[q]);
          }
        }
      }
    }
  }

  // element vector o (chunk offset, plo <= o < phi) of slot s, array arr (0 g, 1 v, 2 x)
  __device__ __forceinline__ void get(int q, int s, int arr, const Unit &x, int64_t o, int nv, int64_t len4,
                                      float (&r4)[W]) const {
    if (kTma && o + W <= len4) {
      const float4 t = *reinterpret_cast<const float4 *>(stage(q, s, arr) + (o - x.plo));
      r4[0] = t.x; r4[W > 1 ? 1 : 0] = t.y; r4[W > 2 ? 2 : 0] = t.z; r4[W > 3 ? 3 : 0] = t.w;
    } else {
      const float *src = (arr == 0 ? a.bg[x.b * r + s] : arr == 1 ? a.bv[x.b * r + s] : a.bx[x.b * r + s]);
      ldm<W>(src + x.e0 + o, r4, nv);
    }
  }

  // ---------------------------------------------------------------- S
  __device__ void run_s() const {
    const int t = threadIdx.x - kWarpsP * 32;
    const bool lead = a.prof && t == 0;
    const uint64_t ts = lead ? dev::globaltimer() : 0;
    uint64_t t_wait = 0;
    for (int64_t k = 0;; ++k) {
      const int q = int(k % kQL), qx = int(k % kQX);
      const uint64_t tw = lead ? dev::globaltimer() : 0;
      mbar_spin(&sm->full_ld[q], uint32_t((k / kQL) & 1));
      const int64_t u = sm->uid[k % kQI];
      if (u < 0) {
        for (int64_t kk = k; kk < k + kGroupsR; ++kk) {
          const int qq = int(kk % kQX);
          if (kk >= kQX) mbar_spin(&sm->empty_x[qq], uint32_t((kk / kQX - 1) & 1));
          if ((t & 31) == 0) {
            sm->xuid[qq] = -1;
            mbar_arrive(&sm->full_x[qq]);
          }
        }
        break;
      }
      if (k >= kQX) mbar_spin(&sm->empty_x[qx], uint32_t((k / kQX - 1) & 1));
      if (lead) t_wait += dev::globaltimer() - tw;
      const Unit x = sm->unit[k % kQI];
      const int64_t len4 = x.plo + ((x.phi - x.plo) & ~int64_t(3));
      const int64_t nvec = (x.phi - x.plo + W - 1) / W;
      // (local slot, vector) items of the unit, flattened so that every S thread has the same
      // share whatever r is (r * nvec items; nvec = 256 for a full piece at r <= 4)
      const int nvi = int(nvec);
      for (int it = t; it < r * nvi; it += kThS) {
        const int s = it / nvi, vi = it - s * nvi;
        const int kind = a.slot_kind[s];
        if (kind == 2 || skip(s)) continue;  // updated with its group's first member / by K6
        const int8_t *G = group(a.my_workers[s]);
        {
          const int64_t o = x.plo + int64_t(vi) * W;
          const int nv = int(min(int64_t(W), x.phi - o));
          const int64_t e = x.e0 + o;
          if (kind == 1) {  // every member here: the 1-GPU kernel's arithmetic in registers
            float acc[W];
            for (int rr = 0; rr < m; ++rr) {  // ascending member id
              const int sl = a.worker_slot[G[rr]];
              float gr[W];
              get(q, sl, 0, x, o, nv, len4, gr);
              if constexpr (!GRAD) {
                float v[W], xx[W];
                get(q, sl, 1, x, o, nv, len4, v);
                get(q, sl, 2, x, o, nv, len4, xx);
#pragma unroll
                for (int w = 0; w < W; ++w) {
                  v[w] = dev::momentum(a.mu, v[w], dev::decay(gr[w], a.wd, xx[w]));
                  const float xh = dev::sgd(xx[w], a.lr, v[w]);
                  acc[w] = (rr == 0) ? xh : __fadd_rn(acc[w], xh);
                }
                stm<W>(a.bv[x.b * r + sl] + e, v, nv);
              } else {
#pragma unroll
                for (int w = 0; w < W; ++w) acc[w] = (rr == 0) ? gr[w] : __fadd_rn(acc[w], gr[w]);
              }
            }
#pragma unroll
            for (int w = 0; w < W; ++w) acc[w] = dev::mean_rt(acc[w], m, inv_m);
            for (int rr = 0; rr < m; ++rr) {
              const int sl = a.worker_slot[G[rr]];
              if constexpr (!GRAD) {
                stm<W>(a.bx[x.b * r + sl] + e, acc, nv);
              } else {
                float v[W], xx[W];
                get(q, sl, 1, x, o, nv, len4, v);
                get(q, sl, 2, x, o, nv, len4, xx);
#pragma unroll
                for (int w = 0; w < W; ++w) {
                  v[w] = dev::momentum(a.mu, v[w], dev::decay(acc[w], a.wd, xx[w]));
                  xx[w] = dev::sgd(xx[w], a.lr, v[w]);
                }
                stm<W>(a.bv[x.b * r + sl] + e, v, nv);
                stm<W>(a.bx[x.b * r + sl] + e, xx, nv);
              }
            }
          } else {  // a group with remote members: reduce-scatter my contribution of slice j
            float val[W];
            get(q, s, 0, x, o, nv, len4, val);
            if constexpr (!GRAD) {
              float v[W], xx[W];
              get(q, s, 1, x, o, nv, len4, v);
              get(q, s, 2, x, o, nv, len4, xx);
#pragma unroll
              for (int w = 0; w < W; ++w) {
                v[w] = dev::momentum(a.mu, v[w], dev::decay(val[w], a.wd, xx[w]));
                val[w] = dev::sgd(xx[w], a.lr, v[w]);  // x_hat
              }
              stm<W>(a.bv[x.b * r + s] + e, v, nv);
            }
            const int w = G[x.j];  // the slice's owner
            if (local(w)) {
              float *dst = xent(qx, s) + (o - x.plo);
              SESGD_CHECK(o - x.plo + nv <= sub);
#pragma unroll
              for (int q2 = 0; q2 < W; ++q2)
                if (q2 < nv) dst[q2] = val[q2];
            } else {
              push<W>(recv(w, a.my_pos[s]) + x.soff + e, val, nv);
            }
          }
        }
      }
      __syncwarp();
      if ((t & 31) == 0) {
        mbar_arrive(&sm->empty_ld[q]);
        sm->xuid[qx] = u;
        sm->xunit[qx] = x;
        mbar_arrive(&sm->full_x[qx]);
      }
    }
    if (lead) {
      uint64_t *pr = a.prof + int64_t(cta) * 8;
      pr[0] += dev::globaltimer() - ts;
      pr[4] += t_wait;
    }
  }

  // ---------------------------------------------------------------- R
  __device__ void run_r(int grp, int t) const {
    const bool lead = a.prof && t == 0 && grp == 0;
    const uint64_t ts = lead ? dev::globaltimer() : 0;
    uint64_t t_wait = 0, t_spin = 0;
    uint64_t *spin = lead ? &t_spin : nullptr;
    bool delayed = false;
    for (int64_t k = grp;; k += kGroupsR) {
      const int qx = int(k % kQX);
      const uint64_t tw = lead ? dev::globaltimer() : 0;
      mbar_spin(&sm->full_x[qx], uint32_t((k / kQX) & 1));
      if (lead) t_wait += dev::globaltimer() - tw;
      const int64_t u = sm->xuid[qx];
      if (u < 0) break;
      if (!delayed && a.hop_delay_ns) {  // config 4: the all-gather round's injected hop
        const uint64_t t0 = dev::globaltimer();
        while (dev::globaltimer() - t0 < a.hop_delay_ns) {
        }
        delayed = true;
      }
      const Unit x = sm->xunit[qx];
      for (int o_s = 0; o_s < r; ++o_s) {  // every local owner of slice j in a group with remote members
        if (a.slot_kind[o_s] != 0 || a.my_pos[o_s] != x.j) continue;
        const int me = a.my_workers[o_s];
        const int8_t *G = group(me);
        for (int64_t base = x.plo; base < x.phi; base += int64_t(kThR) * W * kU) {
          float acc[kU][W];
          for (int rr = 0; rr < m; ++rr) {  // ascending position = ascending worker id
            const int w = G[rr];
            float y[kU][W];
            if (local(w)) {
              const float *ent = xent(qx, a.worker_slot[w]);
#pragma unroll
              for (int uu = 0; uu < kU; ++uu) {
                const int64_t o = base + (int64_t(uu) * kThR + t) * W;
                const int nv = int(max(int64_t(0), min(int64_t(W), x.phi - o)));
#pragma unroll
                for (int q2 = 0; q2 < W; ++q2) y[uu][q2] = (q2 < nv) ? ent[o - x.plo + q2] : 0.f;
              }
            } else {
              float *src = recv(me, rr) + x.soff + x.e0;
#pragma unroll
              for (int uu = 0; uu < kU; ++uu) {
                const int64_t o = base + (int64_t(uu) * kThR + t) * W;
                const int nv = int(max(int64_t(0), min(int64_t(W), x.phi - o)));
                if (nv > 0) ld_rel<W>(src + o, y[uu], nv);
              }
#pragma unroll
              for (int uu = 0; uu < kU; ++uu) {
                const int64_t o = base + (int64_t(uu) * kThR + t) * W;
                const int nv = int(max(int64_t(0), min(int64_t(W), x.phi - o)));
                if (nv <= 0) continue;
                wait_value<W>(a, cta, me, src + o, y[uu], nv, rr, spin);
                rearm<W>(src + o, nv);
              }
            }
#pragma unroll
            for (int uu = 0; uu < kU; ++uu)
#pragma unroll
              for (int q2 = 0; q2 < W; ++q2) acc[uu][q2] = (rr == 0) ? y[uu][q2] : __fadd_rn(acc[uu][q2], y[uu][q2]);
          }
#pragma unroll
          for (int uu = 0; uu < kU; ++uu) {
            const int64_t o = base + (int64_t(uu) * kThR + t) * W;
            const int nv = int(max(int64_t(0), min(int64_t(W), x.phi - o)));
            if (nv <= 0) continue;
            const int64_t e = x.e0 + o;
#pragma unroll
            for (int q2 = 0; q2 < W; ++q2) acc[uu][q2] = dev::mean_rt(acc[uu][q2], m, inv_m);
            for (int rr = 0; rr < m; ++rr) {
              const int w = G[rr];
              if (!local(w)) {
                push<W>(recv(w, x.j) + x.soff + e, acc[uu], nv);  // all-gather to a remote member
                continue;
              }
              const int sl = a.worker_slot[w];
              if constexpr (!GRAD) {
                stm<W>(a.bx[x.b * r + sl] + e, acc[uu], nv);
              } else {
                float v[W], xx[W];
                ldm<W>(a.bv[x.b * r + sl] + e, v, nv);
                ldm<W>(a.bx[x.b * r + sl] + e, xx, nv);
#pragma unroll
                for (int q2 = 0; q2 < W; ++q2) {
                  v[q2] = dev::momentum(a.mu, v[q2], dev::decay(acc[uu][q2], a.wd, xx[q2]));
                  xx[q2] = dev::sgd(xx[q2], a.lr, v[q2]);
                }
                stm<W>(a.bv[x.b * r + sl] + e, v, nv);
                stm<W>(a.bx[x.b * r + sl] + e, xx, nv);
              }
            }
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

  // ---------------------------------------------------------------- F
  __device__ void run_f(int grp, int t) const {
    const bool lead = a.prof && t == 0 && grp == 0;
    const uint64_t ts = lead ? dev::globaltimer() : 0;
    uint64_t t_spin = 0;
    uint64_t *spin = lead ? &t_spin : nullptr;
    for (int64_t k = grp;; k += kGroupsF) {
      const int qi = int(k % kQI);
      mbar_spin(&sm->full_id[qi], uint32_t((k / kQI) & 1));
      const int64_t u = sm->uid[qi];
      const Unit x = sm->unit[qi];
      __syncwarp();
      if ((t & 31) == 0) mbar_arrive(&sm->empty_id[qi]);
      if (u < 0) break;
      for (int s = 0; s < r; ++s) {  // every local worker whose slice-j owner is remote
        if (a.slot_kind[s] != 0) continue;
        const int me = a.my_workers[s];
        if (local(group(me)[x.j])) continue;
        float *src = recv(me, x.j) + x.soff + x.e0;
        for (int64_t base = x.plo; base < x.phi; base += int64_t(kThF) * W * kU) {
          float y[kU][W];
#pragma unroll
          for (int uu = 0; uu < kU; ++uu) {
            const int64_t o = base + (int64_t(uu) * kThF + t) * W;
            const int nv = int(max(int64_t(0), min(int64_t(W), x.phi - o)));
            if (nv > 0) ld_rel<W>(src + o, y[uu], nv);
          }
#pragma unroll
          for (int uu = 0; uu < kU; ++uu) {
            const int64_t o = base + (int64_t(uu) * kThF + t) * W;
            const int nv = int(max(int64_t(0), min(int64_t(W), x.phi - o)));
            if (nv <= 0) continue;
            wait_value<W>(a, cta, me, src + o, y[uu], nv, x.j, spin);
            rearm<W>(src + o, nv);
            const int64_t e = x.e0 + o;
            if constexpr (!GRAD) {
              stm<W>(a.bx[x.b * r + s] + e, y[uu], nv);
            } else {
              float v[W], xx[W];
              ldm<W>(a.bv[x.b * r + s] + e, v, nv);
              ldm<W>(a.bx[x.b * r + s] + e, xx, nv);
#pragma unroll
              for (int q2 = 0; q2 < W; ++q2) {
                v[q2] = dev::momentum(a.mu, v[q2], dev::decay(y[uu][q2], a.wd, xx[q2]));
                xx[q2] = dev::sgd(xx[q2], a.lr, v[q2]);
              }
              stm<W>(a.bv[x.b * r + s] + e, v, nv);
              stm<W>(a.bx[x.b * r + s] + e, xx, nv);
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
};

template <int W, bool GRAD>
__device__ __forceinline__ void k4w_multi_body(const P2PArgs &a, unsigned char *dsmem) {
  const WSM<W, GRAD> s(a, dsmem);
  if (s.cta == 0 && threadIdx.x == 0) count(a.counters, kCntLaunches);
  if (threadIdx.x == 0) {
    for (int q = 0; q < kQL; ++q) {
      dev::mbar_init(&s.sm->full_ld[q], 1);
      dev::mbar_init(&s.sm->empty_ld[q], s.kWarpsS);
    }
    for (int q = 0; q < kQX; ++q) {
      dev::mbar_init(&s.sm->full_x[q], s.kWarpsS);
      dev::mbar_init(&s.sm->empty_x[q], s.kWarpsR);
    }
    for (int q = 0; q < kQI; ++q) {
      dev::mbar_init(&s.sm->full_id[q], 1);
      dev::mbar_init(&s.sm->empty_id[q], s.kWarpsF);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // guard: every rank holding a remote member of one of my groups finished its launch of call - 2
  if (a.prev2_seq >= 0 && threadIdx.x < 32) {
    for (int p = threadIdx.x; p < a.r * a.m; p += 32) {
      const int sl = p / a.m, j = p % a.m;
      const int w = s.group(a.my_workers[sl])[j];
      if (!s.local(w)) wait_done(a, s.cta, a.worker_rank[w], w, j);
    }
  }
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
  const int kR0 = kWarpsP + s.kWarpsS, kF0 = kR0 + kGroupsR * s.kWarpsR;
  if (warp < kWarpsP) {
    s.run_p();
  } else if (warp < kR0) {
    s.run_s();
  } else if (warp < kF0) {
    const int w = warp - kR0;
    s.run_r(w / s.kWarpsR, (w % s.kWarpsR) * 32 + (threadIdx.x & 31));
  } else {
    const int w = warp - kF0;
    s.run_f(w / s.kWarpsF, (w % s.kWarpsF) * 32 + (threadIdx.x & 31));
  }
  __syncthreads();  // every re-arm of this CTA precedes the release
  if (threadIdx.x == 0) signal_done(a);
}

template <int W, bool GRAD>
__global__ void __launch_bounds__(kThreadsWSM, 1) k4w_multi(const __grid_constant__ P2PArgs a) {
  extern __shared__ __align__(128) unsigned char dsmem[];
  k4w_multi_body<W, GRAD>(a, dsmem);
}

// measurement harness (sesgd_sync_all_pair): two loopback virtual ranks in ONE grid (as k4w_pair)
template <int W, bool GRAD>
__global__ void __launch_bounds__(kThreadsWSM, 1) k4w_multi_pair(const __grid_constant__ P2PArgs a0,
                                                                const __grid_constant__ P2PArgs a1) {
  extern __shared__ __align__(128) unsigned char dsmem[];
  if (int(blockIdx.x) < a0.grid)
    k4w_multi_body<W, GRAD>(a0, dsmem);
  else
    k4w_multi_body<W, GRAD>(a1, dsmem);
}

// device-resident iteration state (SESGD_OPT_DEVICE_ITER, dev_iter.cuh)
template <int W, bool GRAD>
__global__ void __launch_bounds__(kThreadsWSM, 1) k4w_multi_dev(const __grid_constant__ P2PArgs a) {
  extern __shared__ __align__(128) unsigned char dsmem[];
  __shared__ P2PArgs sa;
  devit::load_patched(a, sa);
  __syncthreads();
  k4w_multi_body<W, GRAD>(sa, dsmem);
  if (threadIdx.x == 0) devit::finish(sa);
}

const void *pick_wsm(int mode, bool vec, bool devi = false) {
  const bool grad = (mode == SESGD_MODE_GRAD_AVG);
  if (devi) {
    if (vec)
      return grad ? reinterpret_cast<const void *>(&k4w_multi_dev<4, true>)
                  : reinterpret_cast<const void *>(&k4w_multi_dev<4, false>);
    return grad ? reinterpret_cast<const void *>(&k4w_multi_dev<1, true>)
                : reinterpret_cast<const void *>(&k4w_multi_dev<1, false>);
  }
  if (vec)
    return grad ? reinterpret_cast<const void *>(&k4w_multi<4, true>)
                : reinterpret_cast<const void *>(&k4w_multi<4, false>);
  return grad ? reinterpret_cast<const void *>(&k4w_multi<1, true>)
              : reinterpret_cast<const void *>(&k4w_multi<1, false>);
}

size_t wsm_smem(int r) {
  const size_t sub = size_t(sub_of(r));
  return kHeadM + size_t(kQL) * r * 3 * sub * 4 + size_t(kQX) * r * sub * 4;
}

}  // namespace

bool p2p_wsm_supported(int r, int m) {  // (+ the device-iteration variant's argument copy)
  return r >= 2 && r <= kMaxR && m >= 2 && wsm_smem(r) + sizeof(P2PArgs) <= 227 * 1024;
}

int p2p_wsm_occupancy(int r) {
  static_assert(sizeof(SmemM) <= kHeadM, "barrier block");
  const size_t smem = wsm_smem(r);
  int occ = 1 << 30;
  for (int mode = 0; mode < 2; ++mode)
    for (int vec = 0; vec < 4; ++vec) {  // bit 1: the device-iteration variant
      const void *k = pick_wsm(mode, (vec & 1) != 0, (vec & 2) != 0);
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      int b = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k, kThreadsWSM, smem) != cudaSuccess) b = 1;
      occ = b < occ ? b : occ;
    }
  return occ > 0 ? occ : 1;
}

int64_t p2p_wsm_units(int r, int m, int64_t chunks) {
  const int sub = sub_of(r);
  const int slice = (kChunkWSM / m) & ~31;
  int upc = 0;
  for (int j = 0; j < m; ++j) {
    const int lo = j * slice, hi = (j == m - 1) ? kChunkWSM : (j + 1) * slice;
    upc += (hi - lo + sub - 1) / sub;
  }
  return chunks * upc;
}

cudaError_t launch_p2p_wsm_pair(const P2PArgs &a0, const P2PArgs &a1, int mode, bool vec, cudaStream_t stream) {
  const bool grad = (mode == SESGD_MODE_GRAD_AVG);
  const void *k = vec ? (grad ? reinterpret_cast<const void *>(&k4w_multi_pair<4, true>)
                              : reinterpret_cast<const void *>(&k4w_multi_pair<4, false>))
                      : (grad ? reinterpret_cast<const void *>(&k4w_multi_pair<1, true>)
                              : reinterpret_cast<const void *>(&k4w_multi_pair<1, false>));
  const size_t smem = wsm_smem(a0.r);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  void *args[] = {const_cast<P2PArgs *>(&a0), const_cast<P2PArgs *>(&a1)};
  return launch_persistent(k, unsigned(a0.grid + a1.grid), kThreadsWSM, args, smem, stream, false);
}

cudaError_t launch_p2p_wsm(const P2PArgs &a, int mode, bool vec, cudaStream_t stream) {
  const void *k = pick_wsm(mode, vec, a.dev != nullptr);
  const size_t smem = wsm_smem(a.r);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  void *args[] = {const_cast<P2PArgs *>(&a)};
  return launch_persistent(k, unsigned(a.grid), kThreadsWSM, args, smem, stream, a.cooperative != 0);
}

}  // namespace sesgd
