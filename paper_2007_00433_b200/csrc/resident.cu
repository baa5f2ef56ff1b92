// resident.cu -- K6: fused group sync + momentum-SGD update with all n workers
// resident on one GPU (the 1-GPU configuration: "k simulated workers are resident
// replicas", BASELINE north star).
//
// One launch covers one bucket for every group of the current iteration.  Each
// CTA row blockIdx.y is one group G = {a_0 < ... < a_{m-1}} of the canonical
// partition (A1); per element e it computes, entirely in registers
//   PARAM (Eq. 6; Alg.1 lines 3-11):
//     v_r = mu (x) v_r (+) g_r ; xh_r = x_r (-) lr (x) v_r      (R8, R11)
//     x_r = (xh_0 (+) xh_1 (+) ... (+) xh_{m-1}) (/) m           (R7, R10)
//   GRAD (Eq. 5 variant):
//     gb = (g_0 (+) ... (+) g_{m-1}) (/) m ; v_r = mu v_r + gb ; x_r = x_r - lr v_r
// so the HBM traffic is exactly the algorithmic 20 B per worker-element
// (read g, v, x; write v, x -- DESIGN.md "Algorithmic bytes"): x_hat never leaves
// registers.  Pure streaming: 128-bit coalesced loads/stores, several independent
// 16-byte loads in flight per thread, grid = SMs x occupancy (persistent-style
// grid-stride).  No tensor cores (nothing here is a contraction).
#include "common.cuh"
#include "internal.h"

namespace sesgd {
namespace {

constexpr int kThreads = 256;

template <int W>
__device__ __forceinline__ void load(const float *p, float (&r)[W]) {
  if constexpr (W == 4) {
    float4 t = dev::ld4(p);
    r[0] = t.x; r[1] = t.y; r[2] = t.z; r[3] = t.w;
  } else {
    r[0] = __ldcs(p);
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

// Registers of one W-wide item for a group of compile-time size M.
template <int M, int W, bool GRAD>
struct Item {
  float g[M][W], v[M][W], x[M][W];

  __device__ __forceinline__ void fetch(float *const *xp, float *const *vp,
                                        const float *const *gp, int64_t e) {
#pragma unroll
    for (int r = 0; r < M; ++r) {
      load<W>(gp[r] + e, g[r]);
      load<W>(vp[r] + e, v[r]);
      load<W>(xp[r] + e, x[r]);
    }
  }

  __device__ __forceinline__ void finish(float *const *xp, float *const *vp, int64_t e, float lr,
                                         float mu, float wd) {
    if constexpr (!GRAD) {
#pragma unroll
      for (int r = 0; r < M; ++r)
#pragma unroll
        for (int w = 0; w < W; ++w) {
          v[r][w] = dev::momentum(mu, v[r][w], dev::decay(g[r][w], wd, x[r][w]));
          x[r][w] = dev::sgd(x[r][w], lr, v[r][w]);  // x_hat, stays in registers
        }
      float mean[W];
#pragma unroll
      for (int w = 0; w < W; ++w) {
        float s = x[0][w];
#pragma unroll
        for (int r = 1; r < M; ++r) s = __fadd_rn(s, x[r][w]);  // ascending member order
        mean[w] = dev::mean_of<M>(s, M);
      }
#pragma unroll
      for (int r = 0; r < M; ++r) {
        store<W>(vp[r] + e, v[r]);
        store<W>(xp[r] + e, mean);
      }
    } else {
      float gb[W];
#pragma unroll
      for (int w = 0; w < W; ++w) {
        float s = g[0][w];
#pragma unroll
        for (int r = 1; r < M; ++r) s = __fadd_rn(s, g[r][w]);
        gb[w] = dev::mean_of<M>(s, M);
      }
#pragma unroll
      for (int r = 0; r < M; ++r) {
#pragma unroll
        for (int w = 0; w < W; ++w) {
          v[r][w] = dev::momentum(mu, v[r][w], dev::decay(gb[w], wd, x[r][w]));
          x[r][w] = dev::sgd(x[r][w], lr, v[r][w]);
        }
        store<W>(vp[r] + e, v[r]);
        store<W>(xp[r] + e, x[r]);
      }
    }
  }
};

// Runtime-m item (any group size): member loop, fold kept in registers.
template <int W, bool GRAD>
__device__ __forceinline__ void item_generic(const ResidentArgs &a, const int8_t *mem, int m,
                                             int64_t e) {
  float s[W];
  if constexpr (!GRAD) {
    for (int r = 0; r < m; ++r) {
      const int sl = mem[r];
      float g[W], v[W], x[W];
      load<W>(a.g[sl] + e, g);
      load<W>(a.v[sl] + e, v);
      load<W>(a.x[sl] + e, x);
#pragma unroll
      for (int w = 0; w < W; ++w) {
        v[w] = dev::momentum(a.mu, v[w], dev::decay(g[w], a.wd, x[w]));
        x[w] = dev::sgd(x[w], a.lr, v[w]);
        s[w] = (r == 0) ? x[w] : __fadd_rn(s[w], x[w]);
      }
      store<W>(a.v[sl] + e, v);
    }
#pragma unroll
    for (int w = 0; w < W; ++w) s[w] = __fdiv_rn(s[w], (float)m);
    for (int r = 0; r < m; ++r) store<W>(a.x[mem[r]] + e, s);
  } else {
    for (int r = 0; r < m; ++r) {
      float g[W];
      load<W>(a.g[mem[r]] + e, g);
#pragma unroll
      for (int w = 0; w < W; ++w) s[w] = (r == 0) ? g[w] : __fadd_rn(s[w], g[w]);
    }
#pragma unroll
    for (int w = 0; w < W; ++w) s[w] = __fdiv_rn(s[w], (float)m);
    for (int r = 0; r < m; ++r) {
      const int sl = mem[r];
      float v[W], x[W];
      load<W>(a.v[sl] + e, v);
      load<W>(a.x[sl] + e, x);
#pragma unroll
      for (int w = 0; w < W; ++w) {
        v[w] = dev::momentum(a.mu, v[w], dev::decay(s[w], a.wd, x[w]));
        x[w] = dev::sgd(x[w], a.lr, v[w]);
      }
      store<W>(a.v[sl] + e, v);
      store<W>(a.x[sl] + e, x);
    }
  }
}

// Default items per thread per trip.  M = 2 measured on B200 (cfg 2, all-bucket launch):
// U = 1 (62 regs, 4 CTAs/SM) 0.962 of HBM peak > U = 8 0.947 > U = 4 (128 regs) 0.933 > U = 2.
template <int M>
struct Unroll {
  static constexpr int value = M == 0 ? 1 : (M == 1 ? 4 : (M == 2 ? 1 : (M <= 4 ? 2 : 1)));
};

// One bucket for the group `mem` of this CTA row: grid-stride over W-wide items.
template <int M, int W, bool GRAD, int U, bool WD>
__device__ __forceinline__ void resident_bucket(const ResidentArgs &a, const int8_t *mem, int m,
                                                float *const *tx, float *const *tv,
                                                const float *const *tg, int64_t numel) {
  const int64_t nfull = numel / W;  // complete W-wide items
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if constexpr (M > 0) {
    float *xp[M], *vp[M];
    const float *gp[M];
#pragma unroll
    for (int r = 0; r < M; ++r) {
      xp[r] = tx[mem[r]];
      vp[r] = tv[mem[r]];
      gp[r] = tg[mem[r]];
    }
    // U independent items per trip: all 3*M*U loads are issued before the first store.
    for (; i + (U - 1) * stride < nfull; i += U * stride) {
      Item<M, W, GRAD> it[U];
#pragma unroll
      for (int u = 0; u < U; ++u) it[u].fetch(xp, vp, gp, (i + u * stride) * W);
#pragma unroll
      for (int u = 0; u < U; ++u) it[u].finish(xp, vp, (i + u * stride) * W, a.lr, a.mu, WD ? a.wd : 0.f);
    }
    for (; i < nfull; i += stride) {
      Item<M, W, GRAD> it;
      it.fetch(xp, vp, gp, i * W);
      it.finish(xp, vp, i * W, a.lr, a.mu, WD ? a.wd : 0.f);
    }
  } else {
    ResidentArgs b = a;  // runtime-m path reads the member tables through the args
    b.x = tx;
    b.v = tv;
    b.g = tg;
    for (; i < nfull; i += stride) item_generic<W, GRAD>(b, mem, m, i * W);
  }
  // ragged tail (numel % 4 elements) of the vector path
  if constexpr (W > 1) {
    const int64_t tail = numel - nfull * W;
    if (blockIdx.x == 0 && threadIdx.x < tail) {
      ResidentArgs b = a;
      b.x = tx;
      b.v = tv;
      b.g = tg;
      item_generic<1, GRAD>(b, mem, m, nfull * W + threadIdx.x);
    }
  }
}

// a.nb == 0: one bucket (a.x / a.v / a.g, a.numel).  a.nb > 0: every bucket of the iteration
// in one launch (tables bx/bv/bg[b * n_local + slot], numels[b]); elements are independent, so
// CTAs flow from one bucket into the next without any barrier (one launch tail per iteration).
// WD: weight decay compiled in (a.wd != 0); the WD = false kernels are the decay-free ones
template <int M, int W, bool GRAD, int U, bool WD>
__global__ void __launch_bounds__(kThreads) k6_resident(const __grid_constant__ ResidentArgs a) {
  const int m = M > 0 ? M : a.m;
  // device iteration state (SESGD_OPT_DEVICE_ITER): the iteration's groups from device memory
  const int8_t *mem = (a.dev ? a.dev->member_slot : a.member_slot) + blockIdx.y * m;
  if (a.nb == 0) {
    resident_bucket<M, W, GRAD, U, WD>(a, mem, m, a.x, a.v, a.g, a.numel);
  } else {
    for (int b = 0; b < a.nb; ++b)
      resident_bucket<M, W, GRAD, U, WD>(a, mem, m, a.bx + int64_t(b) * a.n_local,
                                     a.bv + int64_t(b) * a.n_local, a.bg + int64_t(b) * a.n_local,
                                     a.numels[b]);
  }
}

template <int M, int W, bool GRAD, int U>
const void *kernel_ptr(bool wd) {
  return wd ? reinterpret_cast<const void *>(&k6_resident<M, W, GRAD, U, true>)
            : reinterpret_cast<const void *>(&k6_resident<M, W, GRAD, U, false>);
}

// unroll 0 = default per M; 1 / 2 / 4 selectable for M = 2 (SESGD_OPT_RESIDENT_UNROLL)
template <int W, bool GRAD>
const void *pick_m(int m, int unroll, bool wd) {
  switch (m) {
    case 1: return kernel_ptr<1, W, GRAD, Unroll<1>::value>(wd);
    case 2:
      switch (unroll) {
        case 4: return kernel_ptr<2, W, GRAD, 4>(wd);
        case 2: return kernel_ptr<2, W, GRAD, 2>(wd);
        case 8: return kernel_ptr<2, W, GRAD, 8>(wd);
        default: return kernel_ptr<2, W, GRAD, Unroll<2>::value>(wd);
      }
    case 4: return kernel_ptr<4, W, GRAD, Unroll<4>::value>(wd);
    case 8: return kernel_ptr<8, W, GRAD, Unroll<8>::value>(wd);
    default: return kernel_ptr<0, W, GRAD, Unroll<0>::value>(wd);
  }
}

const void *pick(int mode, bool vec, int m, int unroll, bool wd) {
  const bool grad = (mode == SESGD_MODE_GRAD_AVG);
  if (vec) return grad ? pick_m<4, true>(m, unroll, wd) : pick_m<4, false>(m, unroll, wd);
  return grad ? pick_m<1, true>(m, unroll, wd) : pick_m<1, false>(m, unroll, wd);
}

// K8: Algorithm 1's last line, xbar = Ring-AllReduce(x_i; Global): per element, the
// left fold of the n workers' parameters in ascending worker id, one division by n (R7, R10),
// stored to every local worker.  Each thread reads all rows of its elements before writing them,
// so the rows may alias the outputs (one GPU, in place).
template <int W>
__global__ void __launch_bounds__(kThreads) k8_average(const __grid_constant__ AverageArgs a) {
  const int64_t items = (W == 4) ? a.numel / 4 : a.numel;
  const float nr = float(a.nrows);
  for (int64_t it = int64_t(blockIdx.x) * kThreads + threadIdx.x; it < items;
       it += int64_t(gridDim.x) * kThreads) {
    const int64_t e = it * W;
    float acc[W], y[W];
    load<W>(a.rows[0] + e, acc);
    for (int i = 1; i < a.nrows; ++i) {
      load<W>(a.rows[i] + e, y);
#pragma unroll
      for (int q = 0; q < W; ++q) acc[q] = __fadd_rn(acc[q], y[q]);
    }
#pragma unroll
    for (int q = 0; q < W; ++q) acc[q] = __fdiv_rn(acc[q], nr);
    for (int s = 0; s < a.nouts; ++s) store<W>(a.outs[s] + e, acc);
  }
  if constexpr (W == 4) {  // ragged tail of 1..3 elements
    const int64_t e = items * 4 + int64_t(blockIdx.x) * kThreads + threadIdx.x;
    if (blockIdx.x == 0 && e < a.numel) {
      float acc = a.rows[0][e];
      for (int i = 1; i < a.nrows; ++i) acc = __fadd_rn(acc, a.rows[i][e]);
      acc = __fdiv_rn(acc, nr);
      for (int s = 0; s < a.nouts; ++s) a.outs[s][e] = acc;
    }
  }
}

// K9: consistency of the workers' parameters: per element, the binary64 mean of
// the n rows, then out[0] += sum (x_i - mean)^2 and out[1] = max(out[1], |x_i - mean|) over the
// launch (warp-shuffle + shared-memory block reduction, one double atomic per CTA; the max via
// the order-preserving bit pattern of non-negative doubles).
__global__ void __launch_bounds__(kThreads) k9_consensus(const __grid_constant__ AverageArgs a,
                                                         double *out) {
  double ss = 0.0, mx = 0.0;
  for (int64_t e = int64_t(blockIdx.x) * kThreads + threadIdx.x; e < a.numel;
       e += int64_t(gridDim.x) * kThreads) {
    double mean = 0.0;
    for (int i = 0; i < a.nrows; ++i) mean += double(__ldcs(a.rows[i] + e));
    mean /= double(a.nrows);
    for (int i = 0; i < a.nrows; ++i) {
      const double d = double(__ldcs(a.rows[i] + e)) - mean;
      ss += d * d;
      mx = fmax(mx, fabs(d));
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  __shared__ double s_ss[kThreads / 32], s_mx[kThreads / 32];
  if ((threadIdx.x & 31) == 0) {
    s_ss[threadIdx.x >> 5] = ss;
    s_mx[threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kThreads / 32; ++w) {
      ss += s_ss[w];
      mx = fmax(mx, s_mx[w]);
    }
    atomicAdd(out, ss);
    atomicMax(reinterpret_cast<unsigned long long *>(out + 1),
              static_cast<unsigned long long>(__double_as_longlong(mx)));
  }
}

}  // namespace

cudaError_t launch_average(const AverageArgs &a, bool vec, int sm_count, cudaStream_t stream) {
  const int64_t items = vec ? a.numel / 4 : a.numel;
  int64_t blocks = (items + kThreads - 1) / kThreads;
  blocks = blocks < 1 ? 1 : (blocks > int64_t(sm_count) * 8 ? int64_t(sm_count) * 8 : blocks);
  void *args[] = {const_cast<AverageArgs *>(&a)};
  const void *k = vec ? reinterpret_cast<const void *>(&k8_average<4>)
                      : reinterpret_cast<const void *>(&k8_average<1>);
  return cudaLaunchKernel(k, dim3(unsigned(blocks)), dim3(kThreads), args, 0, stream);
}

cudaError_t launch_consensus(const AverageArgs &a, double *out, int sm_count, cudaStream_t stream) {
  int64_t blocks = (a.numel + kThreads - 1) / kThreads;
  blocks = blocks < 1 ? 1 : (blocks > int64_t(sm_count) * 4 ? int64_t(sm_count) * 4 : blocks);
  k9_consensus<<<unsigned(blocks), kThreads, 0, stream>>>(a, out);
  return cudaGetLastError();
}

int resident_block_threads() { return kThreads; }

int resident_occupancy(int mode, bool vec, int m, int unroll) {
  int blocks = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, pick(mode, vec, m, unroll, false), kThreads,
                                                    0) != cudaSuccess)
    return 1;
  return blocks > 0 ? blocks : 1;
}

cudaError_t launch_resident(const ResidentArgs &a, int mode, bool vec, int grid_x, int unroll,
                            cudaStream_t stream) {
  dim3 grid(grid_x, a.k), block(kThreads);
  void *args[] = {const_cast<ResidentArgs *>(&a)};
  return cudaLaunchKernel(pick(mode, vec, a.m, unroll, a.wd != 0.f), grid, block, args, 0, stream);
}

}  // namespace sesgd
