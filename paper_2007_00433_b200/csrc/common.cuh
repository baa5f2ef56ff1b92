// common.cuh -- device helpers shared by libsesgd's kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sesgd {
namespace dev {

// R10: every step is one binary32 round-to-nearest op; explicit intrinsics keep
// nvcc from contracting mul+add into FMA (which would change the bits).
__device__ __forceinline__ float momentum(float mu, float v, float g) {
  return __fadd_rn(__fmul_rn(mu, v), g);  // v <- mu (x) v (+) g        (R8)
}
__device__ __forceinline__ float sgd(float x, float lr, float v) {
  return __fsub_rn(x, __fmul_rn(lr, v));  // x <- x (-) lr (x) v        (Alg.1 line 7)
}

// group mean: one IEEE division by m after the fold (R7).  For m = 2^p the product with
// the exact reciprocal is the same correctly rounded value, so it is used instead.
template <int M>
__device__ __forceinline__ float mean_of(float s, int m) {
  if constexpr (M == 1) return s;
  if constexpr (M == 2) return __fmul_rn(s, 0.5f);
  if constexpr (M == 4) return __fmul_rn(s, 0.25f);
  if constexpr (M == 8) return __fmul_rn(s, 0.125f);
  return __fdiv_rn(s, (float)m);
}

// 128-bit streaming accesses (HBM-bound data touched once per launch)
__device__ __forceinline__ float4 ld4(const float *p) {
  return __ldcs(reinterpret_cast<const float4 *>(p));
}
__device__ __forceinline__ void st4(float *p, float4 v) { __stcs(reinterpret_cast<float4 *>(p), v); }

// ---- system-scope flags (NVLink P2P handshake) ----
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t *p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_sys() {
  asm volatile("fence.acq_rel.sys;" ::: "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

}  // namespace dev
}  // namespace sesgd
