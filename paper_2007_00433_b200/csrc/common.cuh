// common.cuh -- device helpers shared by libsesgd's kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

// Bounds / protocol checks of the checked build (_build.build(checked=True) compiles with
// -DSESGD_CHECKED: libsesgd_checked.so, selected with SESGD_LIB=checked).  compute-sanitizer is
// refused on this GPU pool, so the parity suite runs against this build instead: a failed check
// traps the kernel (the launch fails with an error the tests see).
#ifdef SESGD_CHECKED
#define SESGD_CHECK(cond)                                                                        \
  do {                                                                                           \
    if (!(cond)) {                                                                               \
      printf("SESGD_CHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__,  \
             int(blockIdx.x), int(threadIdx.x));                                                 \
      __trap();                                                                                  \
    }                                                                                            \
  } while (0)
#else
#define SESGD_CHECK(cond) \
  do {                    \
  } while (0)
#endif

namespace sesgd {
namespace dev {

// R10: every step is one binary32 round-to-nearest op; explicit intrinsics keep
// nvcc from contracting mul+add into FMA (which would change the bits).
__device__ __forceinline__ float momentum(float mu, float v, float g) {
  return __fadd_rn(__fmul_rn(mu, v), g);  // v <- mu (x) v (+) g        (R8)
}
// weight decay on the gradient term before momentum, as torch.optim.SGD (R20):
// d = g (+) wd (x) x; wd == 0 returns g unchanged (keeps the sign of a -0 gradient)
__device__ __forceinline__ float decay(float g, float wd, float x) {
  return wd == 0.f ? g : __fadd_rn(g, __fmul_rn(wd, x));
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

// runtime group size: inv_pow2 = 1/m when m is a power of two (exact), else 0.  s * 2^-p and
// s / 2^p are the same correctly rounded value (R7), and the multiply is one instruction
__host__ __device__ __forceinline__ float pow2_inverse(int m) { return (m & (m - 1)) == 0 ? 1.f / float(m) : 0.f; }
__device__ __forceinline__ float mean_rt(float s, int m, float inv_pow2) {
  return inv_pow2 != 0.f ? __fmul_rn(s, inv_pow2) : __fdiv_rn(s, float(m));
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

// ---- TMA bulk copies (cp.async.bulk) and mbarriers (sm_90+ / sm_100a) ----
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// the same with a suspend-time hint: the waiting warp is suspended (issues nothing) until the
// phase completes or the hint (ns) elapses -- a spinning consumer warp does not steal issue slots
// from the warps doing the work (measured: K4W-M spent ~1/3 of its issued instructions in spins)
__device__ __forceinline__ bool mbar_try_wait_suspend(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
      : "memory");
  return ok != 0;
}
// bounded wait: false after timeout_ns (the caller latches the error instead of hanging)
__device__ __forceinline__ bool mbar_wait(uint64_t *bar, uint32_t parity, uint64_t timeout_ns) {
  if (mbar_try_wait(bar, parity)) return true;
  const uint64_t t0 = globaltimer();
  while (!mbar_try_wait(bar, parity))
    if (globaltimer() - t0 > timeout_ns) return false;
  return true;
}
// global -> shared, completion counted on an mbarrier (bytes multiple of 16, 16-B aligned)
__device__ __forceinline__ void bulk_g2s(void *smem_dst, const void *gmem_src, uint32_t bytes,
                                         uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// shared -> global (any device-visible address, e.g. a peer GPU's buffer over NVLink)
__device__ __forceinline__ void bulk_s2g(void *gmem_dst, const void *smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem_dst),
               "r"(smem_u32(smem_src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {  // smem sources of all but N groups are free
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {  // every committed bulk write has completed
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
// every bulk group except (at most) the `newest` most recent ones has completed its writes
__device__ __forceinline__ void bulk_wait_upto(int newest) {
  switch (newest < 0 ? 0 : (newest > 15 ? 15 : newest)) {
    case 0: bulk_wait<0>(); break;
    case 1: bulk_wait<1>(); break;
    case 2: bulk_wait<2>(); break;
    case 3: bulk_wait<3>(); break;
    case 4: bulk_wait<4>(); break;
    case 5: bulk_wait<5>(); break;
    case 6: bulk_wait<6>(); break;
    case 7: bulk_wait<7>(); break;
    case 8: bulk_wait<8>(); break;
    case 9: bulk_wait<9>(); break;
    case 10: bulk_wait<10>(); break;
    case 11: bulk_wait<11>(); break;
    case 12: bulk_wait<12>(); break;
    case 13: bulk_wait<13>(); break;
    case 14: bulk_wait<14>(); break;
    default: bulk_wait<15>(); break;
  }
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
// generic-proxy shared-memory writes (st.shared) become visible to a following bulk copy
__device__ __forceinline__ void fence_proxy_async_shared() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

}  // namespace dev

// Persistent grids whose CTAs wait on each other or on peer GPUs' CTAs (K3, K4, K5) are launched
// cooperatively: the runtime rejects a grid that cannot be co-resident (instead of a hang) and
// starts it only when every CTA can be resident at once, e.g. on a side stream while backward
// kernels hold SMs (SESGDDataParallel's overlap).
inline cudaError_t launch_persistent(const void *kernel, unsigned grid, unsigned block, void **args,
                                     size_t smem, cudaStream_t stream, bool cooperative = true) {
  if (!cooperative) return cudaLaunchKernel(kernel, dim3(grid), dim3(block), args, smem, stream);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, kernel, args);
}
}  // namespace sesgd
