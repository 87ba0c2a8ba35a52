/* synth_cuda.cu — device twin of the synthetic generator (see synth.h).
 * Fills a device buffer with the values synth_host.c produces for the same
 * (kind, seed, global index).  Bench/test infrastructure (the curandom role,
 * PAPER.md:381-383), not part of the method. */
#include <cuda_runtime.h>
#include <stdint.h>
#include "synth.h"

template <int KIND>
__global__ void __launch_bounds__(256) synth_fill_kernel(uint64_t seed, int64_t start, int64_t n,
                                                         int64_t lo, int64_t hi, void *out) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
    uint64_t i = (uint64_t)(start + k);
    uint64_t h = synth_hash(seed, i);
    if (KIND == SYNTH_F32_U01) ((float *)out)[k] = synth_f32_u01(h);
    if (KIND == SYNTH_F64_U01) ((double *)out)[k] = synth_f64_u01(h);
    if (KIND == SYNTH_F32_S11) ((float *)out)[k] = synth_f32_s11(h);
    if (KIND == SYNTH_F64_S11) ((double *)out)[k] = synth_f64_s11(h);
    if (KIND == SYNTH_I32_RANGE) ((int32_t *)out)[k] = (int32_t)synth_range(h, lo, hi);
    if (KIND == SYNTH_I64_RANGE) ((int64_t *)out)[k] = synth_range(h, lo, hi);
    if (KIND == SYNTH_I64_FULL) ((int64_t *)out)[k] = (int64_t)h;
    if (KIND == SYNTH_F32_RAMP) ((float *)out)[k] = (float)(int64_t)(i + (uint64_t)lo);
    if (KIND == SYNTH_F64_RAMP) ((double *)out)[k] = (double)(int64_t)(i + (uint64_t)lo);
    if (KIND == SYNTH_I32_RAMP) ((int32_t *)out)[k] = (int32_t)(uint32_t)(i + (uint64_t)lo);
    if (KIND == SYNTH_I64_RAMP) ((int64_t *)out)[k] = (int64_t)(i + (uint64_t)lo);
  }
}

extern "C" int synth_fill_cuda(int kind, uint64_t seed, int64_t start, int64_t n, int64_t lo,
                               int64_t hi, void *out, void *stream) {
  if (n < 0 || (n > 0 && !out) || kind < 0 || kind >= SYNTH_KIND_COUNT) return 1;
  if ((kind == SYNTH_I32_RANGE || kind == SYNTH_I64_RANGE) &&
      (hi < lo || (uint64_t)(hi - lo) > 0xffffffffULL)) return 1;
  if (n == 0) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t blocks = (n + 255) / 256;
  int grid = (int)(blocks < (int64_t)sms * 16 ? blocks : (int64_t)sms * 16);
  cudaStream_t s = (cudaStream_t)stream;
  switch (kind) {
#define SYNTH_CASE(K) case K: synth_fill_kernel<K><<<grid, 256, 0, s>>>(seed, start, n, lo, hi, out); break;
    SYNTH_CASE(0) SYNTH_CASE(1) SYNTH_CASE(2) SYNTH_CASE(3) SYNTH_CASE(4) SYNTH_CASE(5)
    SYNTH_CASE(6) SYNTH_CASE(7) SYNTH_CASE(8) SYNTH_CASE(9) SYNTH_CASE(10)
#undef SYNTH_CASE
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
