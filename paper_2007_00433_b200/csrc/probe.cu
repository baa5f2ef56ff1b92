// probe.cu -- K7: NVLink / HBM probes behind the C ABI (diagnostics, not the hot path).
//
// * sesgd_probe_copy: a streaming 128-bit copy between any two device-visible
//   addresses (local -> local, peer -> local = NVLink pull, local -> peer = NVLink
//   push).  The caller times it with events; it gives the bandwidth that bounds
//   the exchange of SURVEY Sec. 8(a) row a5.
// * sesgd_probe_pingpong: one-thread flag ping-pong between two GPUs through
//   system-scope release/acquire, the per-hop handshake latency t_tau of Eq. 2
//    on NVLink 5 (row a4).  Both ranks launch it concurrently.
#include "common.cuh"
#include "internal.h"

namespace sesgd {
namespace {

__global__ void __launch_bounds__(512) copy_kernel(float4 *__restrict__ dst,
                                                   const float4 *__restrict__ src, int64_t n4) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n4; i += 4 * stride) {
    float4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
    dst[i] = a;
    dst[i + stride] = b;
    dst[i + 2 * stride] = c;
    dst[i + 3 * stride] = d;
  }
  for (; i < n4; i += stride) dst[i] = src[i];
}

// initiator: for it: store(peer, 2it+1); wait(mine >= 2it+2).  responder: wait(mine >= 2it+1);
// store(peer, 2it+2).  Flags start at `base` (monotonic across calls).
__global__ void pingpong_kernel(uint64_t *mine, uint64_t *peer, int iters, int initiator,
                                uint64_t base, uint64_t *out_ns, uint64_t timeout_ns) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const uint64_t t0 = dev::globaltimer();
  for (int it = 0; it < iters; ++it) {
    const uint64_t ping = base + 2 * uint64_t(it) + 1, pong = ping + 1;
    if (initiator) {
      dev::st_release_sys(peer, ping);
      while (dev::ld_acquire_sys(mine) < pong)
        if (dev::globaltimer() - t0 > timeout_ns) { *out_ns = ~0ull; return; }
    } else {
      while (dev::ld_acquire_sys(mine) < ping)
        if (dev::globaltimer() - t0 > timeout_ns) { *out_ns = ~0ull; return; }
      dev::st_release_sys(peer, pong);
    }
  }
  *out_ns = dev::globaltimer() - t0;
}

}  // namespace

cudaError_t launch_pingpong(uint64_t *mine, uint64_t *peer, int iters, int initiator, uint64_t base,
                            uint64_t *out_ns, cudaStream_t stream) {
  pingpong_kernel<<<1, 32, 0, stream>>>(mine, peer, iters, initiator, base, out_ns, 10ull * 1000000000ull);
  return cudaGetLastError();
}
}  // namespace sesgd

extern "C" {

SESGD_API int sesgd_probe_copy(void *dst, const void *src, int64_t bytes, int32_t ctas,
                               void *stream) {
  if (!dst || !src || bytes < 0 || (bytes & 15) || ctas < 1) return SESGD_EINVAL;
  if ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) return SESGD_EINVAL;
  // ctas = CTA count | (threads per CTA / 32) << 16; threads default 512
  const int warps = (ctas >> 16) & 0x3f;
  ctas &= 0xffff;
  if (ctas < 1) return SESGD_EINVAL;
  sesgd::copy_kernel<<<ctas, warps ? warps * 32 : 512, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<float4 *>(dst), static_cast<const float4 *>(src), bytes / 16);
  return cudaGetLastError() == cudaSuccess ? SESGD_OK : SESGD_ECUDA;
}

SESGD_API int sesgd_probe_pingpong(uint64_t *my_flag, uint64_t *peer_flag, int32_t iters,
                                   int32_t initiator, uint64_t base, uint64_t *out_ns_device,
                                   void *stream) {
  if (!my_flag || !peer_flag || !out_ns_device || iters < 1) return SESGD_EINVAL;
  sesgd::pingpong_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(
      my_flag, peer_flag, iters, initiator, base, out_ns_device, 10ull * 1000000000ull);
  return cudaGetLastError() == cudaSuccess ? SESGD_OK : SESGD_ECUDA;
}

}  // extern "C"
