// p2p.cu -- K3: fused local update + ONE-SHOT intra-group exchange over NVLink P2P.
//
// Workers live on several GPUs (one process per GPU, r workers per process).
// Each iteration every group G = {a_0 < ... < a_{m-1}} of the shuffle-exchange
// partition (A1) averages its members' locally-stepped parameters (Eq. 6,
// P:204-207; Alg.1 line 11 "Ring-AllReduce(x_hat; G)").  The paper's ring over
// Ethernet is prior art: on NVSwitch every peer is one hop at full bandwidth, so
// the group mean is computed "one-shot": every member publishes x_hat into its
// peer-visible stage and pulls the m-1 peer chunks directly (one handshake round
// instead of the ring's 2(m-1)).
//
// The bucket is cut into chunks of kChunk floats; CTA j of every rank handles
// chunks j, j+grid, ... in the same order (identical grid on every rank, all
// CTAs co-resident, so CTA j only ever waits on CTA j of its peers).  Per chunk:
//   (1) stage-reuse guard: the members of my group at t-2 have finished reading
//       my stage[t&1] chunk (done flags; normally already satisfied);
//   (2) phase A (HBM): v <- mu v + g ; x_hat <- x - lr v ; store v ; store x_hat
//       to stage[t&1]   (GRAD mode: copy g to the stage);
//   (3) publish: st.release.sys epoch into each peer's ready[slot][j][me];
//   (4) wait: ld.acquire.sys my ready[slot][j][q] >= epoch for every peer q;
//   (5) phase B (NVLink + HBM): fold the m stage chunks in ascending member id,
//       divide by m, store x   (GRAD: gb = fold/m, then v, x update);
//   (6) done: st.release.sys epoch into each peer's done[slot][j][me].
// Flags hold monotonic epochs E(t, b, k), never reset, so no flag is ever cleared
// and a slow peer can never be confused with a fast one.
// Every spin has a %globaltimer timeout that latches SESGD_ETIMEOUT (host-mapped
// word) instead of hanging the GPU.
#include "common.cuh"
#include "internal.h"

namespace sesgd {
namespace {

constexpr int kThreads = 512;
constexpr int kVecPerThread = 4;
constexpr int64_t kChunk = int64_t(kThreads) * 4 * kVecPerThread;  // 8192 floats = 32 KiB

template <int W>
__device__ __forceinline__ void load(const float *p, float (&r)[W]) {
  if constexpr (W == 4) {
    float4 t = dev::ld4(p);
    r[0] = t.x; r[1] = t.y; r[2] = t.z; r[3] = t.w;
  } else {
    r[0] = __ldcs(p);
  }
}
// peer / stage data: plain weak loads after the acquire (L1 is per-launch, L2 is
// bypassed for peer apertures), 128-bit
template <int W>
__device__ __forceinline__ void load_stage(const float *p, float (&r)[W]) {
  if constexpr (W == 4) {
    float4 t = *reinterpret_cast<const float4 *>(p);
    r[0] = t.x; r[1] = t.y; r[2] = t.z; r[3] = t.w;
  } else {
    r[0] = *p;
  }
}
template <int W>
__device__ __forceinline__ void store(float *p, const float (&r)[W]) {
  if constexpr (W == 4) {
    dev::st4(p, make_float4(r[0], r[1], r[2], r[3]));
  } else {
    __stcs(p, r[0]);
  }
}
template <int W>
__device__ __forceinline__ void store_stage(float *p, const float (&r)[W]) {
  if constexpr (W == 4) {
    *reinterpret_cast<float4 *>(p) = make_float4(r[0], r[1], r[2], r[3]);
  } else {
    *p = r[0];
  }
}

__device__ __forceinline__ float *stage_ptr(const P2PArgs &a, int worker, int parity) {
  char *base = a.ws[a.worker_rank[worker]] + a.stage_off;
  const int64_t region = int64_t(parity) * a.r + a.worker_slot[worker];
  return reinterpret_cast<float *>(base) + region * a.stage_slot_floats + a.stage_bucket_off;
}

__device__ __forceinline__ uint64_t *flag_ptr(const P2PArgs &a, int64_t off, int rank, int dst_slot,
                                              int src_worker) {
  uint64_t *f = reinterpret_cast<uint64_t *>(a.ws[rank] + off);
  return f + (int64_t(dst_slot) * a.grid + blockIdx.x) * a.n + src_worker;
}

// spin until *p >= target; false on timeout / abort (error latched)
__device__ bool wait_geq(const P2PArgs &a, const uint64_t *p, uint64_t target) {
  if (dev::ld_acquire_sys(p) >= target) return true;
  const uint64_t t0 = dev::globaltimer();
  for (;;) {
    if (dev::ld_acquire_sys(p) >= target) return true;
    if (*reinterpret_cast<volatile unsigned int *>(a.abort_dev)) return false;
    if (dev::globaltimer() - t0 > a.timeout_ns) {
      atomicExch(a.abort_dev, 1u);
      atomicExch(a.err_host, (unsigned int)(-SESGD_ETIMEOUT));
      __threadfence_system();
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

// Enumerate (local slot s, peer q) pairs of a partition; lane-parallel in warp 0.
template <typename F>
__device__ __forceinline__ void for_each_peer(const P2PArgs &a, const int8_t *canon,
                                              const int8_t *group_of, F &&f) {
  const int lane = threadIdx.x;
  const int pairs = a.r * a.m;
  for (int p = lane; p < pairs; p += 32) {
    const int s = p / a.m, rr = p % a.m;
    const int me = a.my_workers[s];
    const int q = canon[group_of[me] * a.m + rr];
    if (q != me) f(s, me, q);
  }
}

template <int W, bool GRAD>
__global__ void __launch_bounds__(kThreads) k3_oneshot(const __grid_constant__ P2PArgs a) {
  constexpr int kItems = int(kChunk / W) / kThreads;  // W-wide items per thread per chunk
  const int tid = threadIdx.x;
  const int parity = a.parity;

  for (int64_t k = 0, c = blockIdx.x; c < a.nchunks; ++k, c += a.grid) {
    const uint64_t epoch = a.epoch0 + uint64_t(k);
    const int64_t e0 = c * kChunk;
    const int64_t e1 = min(e0 + kChunk, a.numel);

    // (1) stage-reuse guard against the group of iteration t-2
    if (a.m > 1 && a.epoch_prev0 != 0 && tid < 32) {
      const uint64_t prev = a.epoch_prev0 + uint64_t(k);
      for_each_peer(a, a.canon_prev, a.group_of_prev, [&](int s, int, int q) {
        wait_geq(a, flag_ptr(a, a.done_off, a.my_rank, s, q), prev);
      });
    }
    __syncthreads();

    // (2) phase A: local momentum-SGD step, publish x_hat (or g) to my stage
    for (int s = 0; s < a.r; ++s) {
      float *xs = a.x[s], *vs = a.v[s];
      const float *gs = a.g[s];
      float *st = stage_ptr(a, a.my_workers[s], parity);
#pragma unroll
      for (int it = 0; it < kItems; ++it) {
        const int64_t e = e0 + (int64_t(it) * kThreads + tid) * W;
        if (e + W <= e1) {
          float g[W];
          load<W>(gs + e, g);
          if constexpr (!GRAD) {
            float v[W], x[W];
            load<W>(vs + e, v);
            load<W>(xs + e, x);
#pragma unroll
            for (int w = 0; w < W; ++w) {
              v[w] = dev::momentum(a.mu, v[w], g[w]);
              x[w] = dev::sgd(x[w], a.lr, v[w]);
            }
            store<W>(vs + e, v);
            if (a.m == 1)
              store<W>(xs + e, x);  // x / 1 = x: no exchange
            else
              store_stage<W>(st + e, x);
          } else {
            if (a.m == 1) {
              float v[W], x[W];
              load<W>(vs + e, v);
              load<W>(xs + e, x);
#pragma unroll
              for (int w = 0; w < W; ++w) {
                v[w] = dev::momentum(a.mu, v[w], g[w]);
                x[w] = dev::sgd(x[w], a.lr, v[w]);
              }
              store<W>(vs + e, v);
              store<W>(xs + e, x);
            } else {
              store_stage<W>(st + e, g);
            }
          }
        } else if (e < e1) {  // ragged tail (vector path only)
          for (int64_t ee = e; ee < e1; ++ee) {
            const float g = gs[ee];
            if constexpr (!GRAD) {
              const float v = dev::momentum(a.mu, vs[ee], g);
              const float xh = dev::sgd(xs[ee], a.lr, v);
              vs[ee] = v;
              if (a.m == 1) xs[ee] = xh; else st[ee] = xh;
            } else {
              if (a.m == 1) {
                const float v = dev::momentum(a.mu, vs[ee], g);
                vs[ee] = v;
                xs[ee] = dev::sgd(xs[ee], a.lr, v);
              } else {
                st[ee] = g;
              }
            }
          }
        }
      }
    }
    if (a.m == 1) continue;
    __syncthreads();

    // (3) publish + (4) wait, warp 0
    if (tid < 32) {
      hop_delay(a);
      for_each_peer(a, a.canon, a.group_of, [&](int, int me, int q) {
        dev::st_release_sys(flag_ptr(a, a.ready_off, a.worker_rank[q], a.worker_slot[q], me), epoch);
      });
      for_each_peer(a, a.canon, a.group_of, [&](int s, int, int q) {
        wait_geq(a, flag_ptr(a, a.ready_off, a.my_rank, s, q), epoch);
      });
    }
    __syncthreads();

    // (5) phase B: ascending fold of the m staged chunks (own + peers over NVLink)
    for (int s = 0; s < a.r; ++s) {
      const int me = a.my_workers[s];
      const int8_t *G = a.canon + a.group_of[me] * a.m;
      float *xs = a.x[s], *vs = a.v[s];
#pragma unroll
      for (int it = 0; it < kItems; ++it) {
        const int64_t e = e0 + (int64_t(it) * kThreads + tid) * W;
        if (e + W <= e1) {
          float acc[W];
          load_stage<W>(stage_ptr(a, G[0], parity) + e, acc);
          for (int r = 1; r < a.m; ++r) {
            float y[W];
            load_stage<W>(stage_ptr(a, G[r], parity) + e, y);
#pragma unroll
            for (int w = 0; w < W; ++w) acc[w] = __fadd_rn(acc[w], y[w]);
          }
#pragma unroll
          for (int w = 0; w < W; ++w) acc[w] = __fdiv_rn(acc[w], (float)a.m);
          if constexpr (!GRAD) {
            store<W>(xs + e, acc);
          } else {
            float v[W], x[W];
            load<W>(vs + e, v);
            load<W>(xs + e, x);
#pragma unroll
            for (int w = 0; w < W; ++w) {
              v[w] = dev::momentum(a.mu, v[w], acc[w]);
              x[w] = dev::sgd(x[w], a.lr, v[w]);
            }
            store<W>(vs + e, v);
            store<W>(xs + e, x);
          }
        } else if (e < e1) {
          for (int64_t ee = e; ee < e1; ++ee) {
            float acc = stage_ptr(a, G[0], parity)[ee];
            for (int r = 1; r < a.m; ++r) acc = __fadd_rn(acc, stage_ptr(a, G[r], parity)[ee]);
            acc = __fdiv_rn(acc, (float)a.m);
            if constexpr (!GRAD) {
              xs[ee] = acc;
            } else {
              const float v = dev::momentum(a.mu, vs[ee], acc);
              vs[ee] = v;
              xs[ee] = dev::sgd(xs[ee], a.lr, v);
            }
          }
        }
      }
    }
    __syncthreads();

    // (6) done: tell each peer its stage chunk has been consumed
    if (tid < 32) {
      for_each_peer(a, a.canon, a.group_of, [&](int, int me, int q) {
        dev::st_release_sys(flag_ptr(a, a.done_off, a.worker_rank[q], a.worker_slot[q], me), epoch);
      });
    }
  }
}

const void *pick(int mode, bool vec) {
  const bool grad = (mode == SESGD_MODE_GRAD_AVG);
  if (vec)
    return grad ? reinterpret_cast<const void *>(&k3_oneshot<4, true>)
                : reinterpret_cast<const void *>(&k3_oneshot<4, false>);
  return grad ? reinterpret_cast<const void *>(&k3_oneshot<1, true>)
              : reinterpret_cast<const void *>(&k3_oneshot<1, false>);
}

}  // namespace

int p2p_block_threads() { return kThreads; }
int p2p_chunk_elems() { return int(kChunk); }

int p2p_occupancy(int mode, bool vec) {
  int blocks = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, pick(mode, vec), kThreads, 0) !=
      cudaSuccess)
    return 1;
  return blocks > 0 ? blocks : 1;
}

cudaError_t launch_p2p_oneshot(const P2PArgs &a, int mode, bool vec, cudaStream_t stream) {
  void *args[] = {const_cast<P2PArgs *>(&a)};
  return cudaLaunchKernel(pick(mode, vec), dim3(a.grid), dim3(kThreads), args, 0, stream);
}

}  // namespace sesgd
