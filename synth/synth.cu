// synth.cu -- libsynth.so: seeded synthetic input fills (test / bench infrastructure).
//
// Wraps synth_gen.h (the shared input recipe) in
//   * device fill kernels: they stand in for the backward pass that would
//     produce each worker's gradient (Algorithm 1 lines 4-8)
//     and for the shared initial parameters x_0, and
//   * host fill functions with the same values, for tests that need host arrays.
// Holds none of SESGD's arithmetic: no schedule, no update, no averaging.
#include <cuda_runtime.h>
#include <stdint.h>

#include "synth_gen.h"

namespace {

__global__ void __launch_bounds__(256) fill_grad_kernel(float *__restrict__ out, int64_t numel,
                                                        int64_t e0, uint64_t key) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < numel; j += stride)
    out[j] = synth_grad(key, e0 + j);
}

// the same fill with the iteration read from device memory (*t_dev): a captured CUDA graph that
// replays every iteration (libsesgd's SESGD_OPT_DEVICE_ITER, sesgd_device_iter_ptr) regenerates
// the gradients of the device's current iteration
__global__ void __launch_bounds__(256) fill_grad_at_kernel(float *__restrict__ out, int64_t numel,
                                                           int64_t e0, uint64_t s_g, int32_t worker,
                                                           const int64_t *t_dev) {
  const uint64_t key = synth_grad_key(s_g, worker, *t_dev);
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < numel; j += stride)
    out[j] = synth_grad(key, e0 + j);
}

__global__ void __launch_bounds__(256) fill_x0_kernel(float *__restrict__ out, int64_t numel,
                                                      int64_t e0, uint64_t xkey) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < numel; j += stride)
    out[j] = synth_x0(xkey, e0 + j);
}

int grid_for(int64_t numel) {
  int64_t blocks = (numel + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  return (int)blocks;
}

}  // namespace

extern "C" {

// g[j] = gradient of `worker` at iteration `t`, global element e0 + j, for j < numel.
// `out` is a device pointer; enqueued on `stream`; returns a cudaError_t value.
int synth_fill_grad_device(float *out, int64_t numel, int64_t e0, uint64_t s_g, int32_t worker,
                           int64_t t, void *stream) {
  if (numel <= 0) return 0;
  fill_grad_kernel<<<grid_for(numel), 256, 0, (cudaStream_t)stream>>>(
      out, numel, e0, synth_grad_key(s_g, worker, t));
  return (int)cudaGetLastError();
}

// as synth_fill_grad_device with t = *t_dev (a device int64 read when the kernel runs)
int synth_fill_grad_device_at(float *out, int64_t numel, int64_t e0, uint64_t s_g, int32_t worker,
                              const int64_t *t_dev, void *stream) {
  if (numel <= 0) return 0;
  fill_grad_at_kernel<<<grid_for(numel), 256, 0, (cudaStream_t)stream>>>(out, numel, e0, s_g, worker, t_dev);
  return (int)cudaGetLastError();
}

int synth_fill_x0_device(float *out, int64_t numel, int64_t e0, uint64_t s_x, void *stream) {
  if (numel <= 0) return 0;
  fill_x0_kernel<<<grid_for(numel), 256, 0, (cudaStream_t)stream>>>(out, numel, e0,
                                                                     synth_x0_key(s_x));
  return (int)cudaGetLastError();
}

// Host versions, identical values.  `coords` (may be NULL = contiguous e0..e0+numel-1)
// lists global element indices.
void synth_fill_grad_host(float *out, int64_t numel, int64_t e0, const int64_t *coords,
                          uint64_t s_g, int32_t worker, int64_t t) {
  uint64_t key = synth_grad_key(s_g, worker, t);
  for (int64_t j = 0; j < numel; ++j) out[j] = synth_grad(key, coords ? coords[j] : e0 + j);
}

void synth_fill_x0_host(float *out, int64_t numel, int64_t e0, const int64_t *coords,
                        uint64_t s_x) {
  uint64_t key = synth_x0_key(s_x);
  for (int64_t j = 0; j < numel; ++j) out[j] = synth_x0(key, coords ? coords[j] : e0 + j);
}

}  // extern "C"
