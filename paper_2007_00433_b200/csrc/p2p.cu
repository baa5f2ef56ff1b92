// p2p.cu -- K3: fused local update + ONE-SHOT PUSH intra-group exchange over NVLink,
// SM-specialised: a few COMM CTAs move data over NVLink while the COMPUTE CTAs
// stream HBM, in one persistent kernel per bucket.
//
// Each iteration every group G = {a_0 < ... < a_{m-1}} of the shuffle-exchange
// partition (A1) averages its members' locally-stepped parameters (Eq. 6,
// P:204-207; Alg.1 line 11 "Ring-AllReduce(x_hat; G)").  The paper's ring over
// Ethernet is prior art: on NVSwitch every peer is one hop at full bandwidth, so one
// handshake round suffices (instead of the ring's 2(m-1)).
//
// Why this shape (measured on B200, profiles/r01_nvlink_probe_2gpu*.json):
//  * remote loads hold an SM's request slots for ~2.5 us and starve a local HBM
//    stream; remote STORES do not, and both-direction push keeps 705 GB/s/dir;
//  * 32 CTAs of pushes already reach 698 GB/s/dir and leave the other SMs free to
//    stream HBM concurrently (805 us vs 956 us serial); pushing from >= 64 CTAs
//    starves the local stream;
//  * a system-scope release stalls its warp until the CTA's remote stores drain,
//    so releases are batched (one per COMM batch of chunks).
//
// Roles (blockIdx < Q: COMM, else COMPUTE; all CTAs co-resident):
//  COMPUTE CTA i, chunks c = i, i+Gc, ... (chunk = 4096 floats):
//    stage(c):  load g, v, x ; v <- mu v + g ; x_hat <- x - lr v ; store v ;
//               x_hat -> own stage (L2) ; st.release staged[s][i] = E(seq, k)
//               (GRAD: g -> stage, v and x untouched)
//    fold(c) two chunks later: wait sent[s][c] (own COMM pushed it) and every peer's
//               ready[par][s][c][pos] ; fold the m contributions in ascending position
//               (= ascending worker id; own from the stage) ; (/) m ; store x
//               (GRAD: v, x update) ; discard the dead stage / receive lines from L2
//    end:       red.release.sys done[s][b] += 1   (consumption counter for senders)
//  COMM CTA q, batches of B chunks (batch j = q, q+Q, ...):
//    guard once per launch: every peer finished folding this bucket two calls ago
//               (done counter, read over NVLink)
//    wait staged for the batch ; copy own stage -> every peer's receive slot (NVLink
//    stores) ; one st.release.sys per (chunk, peer) ready flag + local sent flags
// All waits point to a strictly smaller chunk index (or an earlier step of the same
// chunk), so the smallest unfinished step can always progress: no deadlock.  Flags
// are keyed by the per-bucket call index (identical on every rank) and never reset.
// Every spin has a %globaltimer timeout that latches SESGD_ETIMEOUT.
#include "common.cuh"
#include "internal.h"

namespace sesgd {
namespace {

constexpr int kThreads = 256;
constexpr int kVec = 4;                                 // float4 items per thread per chunk
constexpr int64_t kChunk = int64_t(kThreads) * 4 * kVec;  // 4096 floats = 16 KiB
// fold(c) runs a.lag chunk steps after stage(c) (SESGD_OPT_FOLD_LAG)

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
__device__ __forceinline__ void red_add_release_sys(uint64_t *p, uint64_t v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_gpu(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(uint64_t *p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// what a timed-out wait was waiting for (reported through sesgd_last_error)
enum WaitKind : int { kWaitDone = 1, kWaitReady = 2, kWaitStaged = 3, kWaitSent = 4 };

// spin until *p >= target (sys-scope acquire); on timeout the first CTA to give up
// latches SESGD_ETIMEOUT plus a description of the flag in the host-mapped block
__device__ bool wait_geq(const P2PArgs &a, const uint64_t *p, uint64_t target, int kind,
                         int worker, int pos) {
  uint64_t v = dev::ld_acquire_sys(p);
  if (v >= target) return true;
  const uint64_t t0 = dev::globaltimer();
  for (;;) {
    v = dev::ld_acquire_sys(p);
    if (v >= target) return true;
    if (*reinterpret_cast<volatile unsigned int *>(a.abort_dev)) return false;
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
      return false;
    }
  }
}

__device__ __forceinline__ void hop_delay(const P2PArgs &a) {
  if (a.hop_delay_ns == 0) return;
  const uint64_t t0 = dev::globaltimer();
  while (dev::globaltimer() - t0 < a.hop_delay_ns) {
  }
}

template <int W, bool GRAD>
struct Split {
  static constexpr int kItems = int(kChunk / W) / kThreads;  // W-wide items per thread per chunk

  const P2PArgs &a;
  int gc;  // compute CTAs
  __device__ explicit Split(const P2PArgs &args) : a(args) { gc = a.grid - a.comm_ctas; }

  // ---- addressing (workspace layout: see sesgd_capi.cu freeze_layout) ----
  __device__ __forceinline__ const int8_t *group(int me) const {
    return a.canon + a.group_of[me] * a.m;
  }
  __device__ __forceinline__ float *stage(int s) const {
    return reinterpret_cast<float *>(a.ws[a.my_rank] + a.stage_off) + int64_t(s) * a.stage_slot_floats +
           a.stage_bucket_off;
  }
  __device__ __forceinline__ float *recv(int worker, int pos) const {
    char *base = a.ws[a.worker_rank[worker]] + a.recv_off;
    const int64_t region = (int64_t(a.parity) * a.r + a.worker_slot[worker]) * a.m + pos;
    return reinterpret_cast<float *>(base) + region * a.stage_slot_floats + a.stage_bucket_off;
  }
  __device__ __forceinline__ uint64_t *ready(int worker, int64_t c, int pos) const {
    uint64_t *f = reinterpret_cast<uint64_t *>(a.ws[a.worker_rank[worker]] + a.ready_off);
    const int64_t row = (int64_t(a.parity) * a.r + a.worker_slot[worker]) * a.total_chunks +
                        a.chunk_base + c;
    return f + row * a.m + pos;
  }
  __device__ __forceinline__ uint64_t *sent(int s, int64_t c) const {
    return reinterpret_cast<uint64_t *>(a.ws[a.my_rank] + a.sent_off) + int64_t(s) * a.total_chunks +
           a.chunk_base + c;
  }
  __device__ __forceinline__ uint64_t *staged(int s, int i) const {
    return reinterpret_cast<uint64_t *>(a.ws[a.my_rank] + a.staged_off) + int64_t(s) * gc + i;
  }
  __device__ __forceinline__ uint64_t *done(int worker) const {
    return reinterpret_cast<uint64_t *>(a.ws[a.worker_rank[worker]] + a.done_off) +
           int64_t(a.worker_slot[worker]) * a.nbuckets + a.bucket;
  }

  // ---------------------------------------------------------------- COMPUTE
  __device__ void stage_chunk(int i, int64_t k) const {
    const int64_t c = i + k * gc;
    const int64_t e0 = c * kChunk, e1 = min(e0 + kChunk, a.numel);
    for (int s = 0; s < a.r; ++s) {
      float *xs = a.x[s], *vs = a.v[s];
      const float *gs = a.g[s];
      float *st = stage(s);
#pragma unroll
      for (int it = 0; it < kItems; ++it) {
        const int64_t e = e0 + (int64_t(it) * kThreads + threadIdx.x) * W;
        const int nv = (int)min(int64_t(W), e1 - e);
        if (nv <= 0) continue;
        float g[W];
        load_m<W>(gs + e, g, nv);
        if constexpr (!GRAD) {
          float v[W], x[W];
          load_m<W>(vs + e, v, nv);
          load_m<W>(xs + e, x, nv);
#pragma unroll
          for (int w = 0; w < W; ++w) {
            v[w] = dev::momentum(a.mu, v[w], g[w]);
            x[w] = dev::sgd(x[w], a.lr, v[w]);  // x_hat
          }
          store_m<W>(vs + e, v, nv);
          st_slot<W>(st + e, x, nv);
        } else {
          st_slot<W>(st + e, g, nv);
        }
      }
    }
    __syncthreads();  // every stage store of chunk c precedes the release
    if (threadIdx.x < a.r) st_release_gpu(staged(threadIdx.x, i), a.seq_epoch0 + uint64_t(k));
  }

  __device__ void fold_chunk(int i, int64_t k) const {
    const int64_t c = i + k * gc;
    const int64_t e0 = c * kChunk, e1 = min(e0 + kChunk, a.numel);
    const uint64_t call = a.call + 1;
    // warp 0: my COMM pushed chunk c (stage no longer needed by it) and all peers' arrived
    if (threadIdx.x < 32) {
      const int pairs = a.r * a.m;
      for (int p = threadIdx.x; p < pairs; p += 32) {
        const int s = p / a.m, rr = p % a.m;
        const int me = a.my_workers[s];
        if (rr == a.my_pos[s])
          wait_geq(a, sent(s, c), call, kWaitSent, me, rr);
        else
          wait_geq(a, ready(me, c, rr), call, kWaitReady, me, rr);
      }
    }
    __syncthreads();
    for (int s = 0; s < a.r; ++s) {
      const int me = a.my_workers[s];
      const int mypos = a.my_pos[s];
      float *xs = a.x[s], *vs = a.v[s];
      const float *st = stage(s);
#pragma unroll
      for (int it = 0; it < kItems; ++it) {
        const int64_t e = e0 + (int64_t(it) * kThreads + threadIdx.x) * W;
        const int nv = (int)min(int64_t(W), e1 - e);
        if (nv <= 0) continue;
        float acc[W];
        for (int rr = 0; rr < a.m; ++rr) {  // ascending position = ascending worker id
          float y[W];
          ld_slot<W>((rr == mypos ? st : recv(me, rr)) + e, y, nv);
#pragma unroll
          for (int w = 0; w < W; ++w) acc[w] = (rr == 0) ? y[w] : __fadd_rn(acc[w], y[w]);
        }
#pragma unroll
        for (int w = 0; w < W; ++w) acc[w] = __fdiv_rn(acc[w], (float)a.m);
        if constexpr (!GRAD) {
          store_m<W>(xs + e, acc, nv);
        } else {
          float v[W], x[W];
          load_m<W>(vs + e, v, nv);
          load_m<W>(xs + e, x, nv);
#pragma unroll
          for (int w = 0; w < W; ++w) {
            v[w] = dev::momentum(a.mu, v[w], acc[w]);
            x[w] = dev::sgd(x[w], a.lr, v[w]);
          }
          store_m<W>(vs + e, v, nv);
          store_m<W>(xs + e, x, nv);
        }
      }
      // the stage and receive lines of this chunk are dead: drop them from L2 without
      // write-back.  A 128-byte line is read by 8 consecutive lanes of one warp.
      if constexpr (W == 4) {
        if (a.discard) {
          __syncwarp();
          if ((threadIdx.x & 7) == 0) {
#pragma unroll
            for (int it = 0; it < kItems; ++it) {
              const int64_t e = e0 + (int64_t(it) * kThreads + threadIdx.x) * W;
              if (e + 32 > e1) continue;
              for (int rr = 0; rr < a.m; ++rr) discard_l2((rr == mypos ? st : recv(me, rr)) + e);
            }
          }
        }
      }
    }
  }

  __device__ void compute(int i) const {
    const int64_t nk = (a.nchunks > i) ? (a.nchunks - i + gc - 1) / gc : 0;
    uint64_t t_stage = 0, t_fold = 0, t0 = a.prof ? dev::globaltimer() : 0, tstart = t0;
    for (int64_t k = 0; k < nk + a.lag; ++k) {
      if (k < nk) stage_chunk(i, k);
      if (a.prof) {
        const uint64_t t1 = dev::globaltimer();
        t_stage += t1 - t0;
        t0 = t1;
      }
      if (k >= a.lag) {
        fold_chunk(i, k - a.lag);
        __syncthreads();  // the fold's reads are complete before the next stage / done
      }
      if (a.prof) {
        const uint64_t t1 = dev::globaltimer();
        t_fold += t1 - t0;
        t0 = t1;
      }
    }
    if (a.prof && threadIdx.x == 0) {
      uint64_t *pr = a.prof + int64_t(blockIdx.x) * 8;
      pr[0] += t_stage;
      pr[1] += t_fold;
      pr[2] += t0 - tstart;
      pr[7] += 1;
    }
    // consumption counter (senders of call+2 wait for it); every compute CTA counts
    if (threadIdx.x < a.r) red_add_release_sys(done(a.my_workers[threadIdx.x]), 1);
  }

  // ---------------------------------------------------------------- COMM
  __device__ void comm(int q) const {
    // guard: every peer I push to has folded this bucket's call-2 data (one remote read
    // per peer per launch; normally long satisfied)
    if (a.call >= 2 && threadIdx.x < 32) {
      const uint64_t need = uint64_t(a.call - 1) * uint64_t(gc);
      const int pairs = a.r * a.m;
      for (int p = threadIdx.x; p < pairs; p += 32) {
        const int s = p / a.m, rr = p % a.m;
        const int me = a.my_workers[s];
        const int qw = group(me)[rr];
        if (qw != me) wait_geq(a, done(qw), need, kWaitDone, qw, rr);
      }
    }
    __syncthreads();
    const int B = a.comm_batch;
    const int64_t nbatches = (a.nchunks + B - 1) / B;
    uint64_t t_staged = 0, t_push = 0, t_rel = 0, t0 = a.prof ? dev::globaltimer() : 0, tstart = t0;
    for (int64_t j = q; j < nbatches; j += a.comm_ctas) {
      const int64_t c0 = j * B, c1 = min(c0 + B, a.nchunks);
      // wait until the compute CTAs staged every chunk of the batch
      if (threadIdx.x < 32) {
        const int n = int(c1 - c0) * a.r;
        for (int p = threadIdx.x; p < n; p += 32) {
          const int s = p % a.r;
          const int64_t c = c0 + p / a.r;
          wait_geq(a, staged(s, int(c % gc)), a.seq_epoch0 + uint64_t(c / gc), kWaitStaged,
                   a.my_workers[s], -1);
        }
      }
      __syncthreads();
      if (a.prof) {
        const uint64_t t1 = dev::globaltimer();
        t_staged += t1 - t0;
        t0 = t1;
      }
      // copy own stage -> every peer's receive slot (NVLink or local stores)
      for (int s = 0; s < a.r; ++s) {
        const int me = a.my_workers[s];
        const int8_t *G = group(me);
        const int mypos = a.my_pos[s];
        const float *st = stage(s);
        for (int64_t c = c0; c < c1; ++c) {
          const int64_t e0 = c * kChunk, e1 = min(e0 + kChunk, a.numel);
          float val[kItems][W];
          int nvs[kItems];
#pragma unroll
          for (int it = 0; it < kItems; ++it) {
            const int64_t e = e0 + (int64_t(it) * kThreads + threadIdx.x) * W;
            nvs[it] = (int)min(int64_t(W), e1 - e);
            if (nvs[it] > 0) ld_slot<W>(st + e, val[it], nvs[it]);
          }
          for (int rr = 0; rr < a.m; ++rr) {
            if (rr == mypos) continue;
            float *dst = recv(G[rr], mypos);
#pragma unroll
            for (int it = 0; it < kItems; ++it) {
              if (nvs[it] <= 0) continue;
              const int64_t e = e0 + (int64_t(it) * kThreads + threadIdx.x) * W;
              st_slot<W>(dst + e, val[it], nvs[it]);
            }
          }
        }
      }
      __syncthreads();  // all stores of the batch precede the releases (cumulativity)
      if (a.prof) {
        const uint64_t t1 = dev::globaltimer();
        t_push += t1 - t0;
        t0 = t1;
      }
      if (threadIdx.x < 32) {
        hop_delay(a);
        const uint64_t call = a.call + 1;
        const int n = int(c1 - c0) * a.r * a.m;
        for (int p = threadIdx.x; p < n; p += 32) {
          const int rr = p % a.m, s = (p / a.m) % a.r;
          const int64_t c = c0 + p / (a.m * a.r);
          const int me = a.my_workers[s];
          if (rr == a.my_pos[s])
            st_release_gpu(sent(s, c), call);
          else
            dev::st_release_sys(ready(group(me)[rr], c, a.my_pos[s]), call);
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
      pr[0] += t_staged;
      pr[1] += t_push;
      pr[2] += t_rel;
      pr[3] += t0 - tstart;
      pr[7] += 1;
    }
  }

  // m == 1: no exchange, the local step is the whole update (x / 1 = x)
  __device__ void local_only() const {
    const int64_t stride = int64_t(a.grid) * kThreads * W;
    for (int s = 0; s < a.r; ++s) {
      float *xs = a.x[s], *vs = a.v[s];
      const float *gs = a.g[s];
      for (int64_t e = (int64_t(blockIdx.x) * kThreads + threadIdx.x) * W; e < a.numel; e += stride) {
        const int nv = (int)min(int64_t(W), a.numel - e);
        float g[W], v[W], x[W];
        load_m<W>(gs + e, g, nv);
        load_m<W>(vs + e, v, nv);
        load_m<W>(xs + e, x, nv);
#pragma unroll
        for (int w = 0; w < W; ++w) {
          v[w] = dev::momentum(a.mu, v[w], g[w]);
          x[w] = dev::sgd(x[w], a.lr, v[w]);
        }
        store_m<W>(vs + e, v, nv);
        store_m<W>(xs + e, x, nv);
      }
    }
  }
};

template <int W, bool GRAD>
__global__ void __launch_bounds__(kThreads) k3_split(const __grid_constant__ P2PArgs a) {
  const Split<W, GRAD> p(a);
  if (a.m == 1) {
    p.local_only();
  } else if (int(blockIdx.x) < a.comm_ctas) {
    p.comm(blockIdx.x);
  } else {
    p.compute(blockIdx.x - a.comm_ctas);
  }
}

const void *pick(int mode, bool vec) {
  const bool grad = (mode == SESGD_MODE_GRAD_AVG);
  if (vec)
    return grad ? reinterpret_cast<const void *>(&k3_split<4, true>)
                : reinterpret_cast<const void *>(&k3_split<4, false>);
  return grad ? reinterpret_cast<const void *>(&k3_split<1, true>)
              : reinterpret_cast<const void *>(&k3_split<1, false>);
}

}  // namespace

bool p2p_variant_valid(int variant) { return variant >= 1 && variant <= 148; }
int p2p_block_threads(int) { return kThreads; }
int p2p_chunk_elems(int) { return int(kChunk); }

int p2p_occupancy(int variant, int r, int mode, bool vec) {
  (void)variant;
  (void)r;
  int blocks = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, pick(mode, vec), kThreads, 0) != cudaSuccess)
    return 1;
  return blocks > 0 ? blocks : 1;
}

cudaError_t launch_p2p_oneshot(const P2PArgs &a, int variant, int mode, bool vec,
                               cudaStream_t stream) {
  (void)variant;
  void *args[] = {const_cast<P2PArgs *>(&a)};
  return cudaLaunchKernel(pick(mode, vec), dim3(a.grid), dim3(kThreads), args, 0, stream);
}

}  // namespace sesgd
