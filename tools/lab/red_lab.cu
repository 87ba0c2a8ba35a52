// red_lab.cu — tuning lab for fp32 sum / dot (not product code).
#include <cuda_runtime.h>
#include <stdint.h>

#include "ga_device.cuh"

using namespace ga;

template <int BLOCK>
__device__ float block_sum(float v, float *sm) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(~0u, v, o);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = v;
  __syncthreads();
  v = threadIdx.x < BLOCK / 32 ? sm[threadIdx.x] : 0.f;
  if (threadIdx.x < 32)
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(~0u, v, o);
  return v;
}

// one-shot: CTA b sums vectors [b*CH, (b+1)*CH), CH = BLOCK*K; last block folds partials.
template <int BLOCK, int K, bool DOT>
__global__ void __launch_bounds__(BLOCK) k_oneshot(int64_t nvec, const float *x, const float *y, float *out, float *partials,
                                                   unsigned *ticket) {
  __shared__ float sm[BLOCK / 32];
  __shared__ bool last;
  const int64_t base = (int64_t)blockIdx.x * BLOCK * K + threadIdx.x;
  V32 vx[K], vy[K];
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const int64_t v = base + j * BLOCK;
    if (v < nvec) {
      vx[j] = ld_nc_256(x + v * 8);
      if (DOT) vy[j] = ld_nc_256(y + v * 8);
    } else {
      for (int k = 0; k < 8; ++k) vx[j].r[k] = vy[j].r[k] = 0;
    }
  }
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
  for (int j = 0; j < K; ++j)
#pragma unroll
    for (int k = 0; k < 8; ++k)
      acc[k] = DOT ? __fmaf_rn(__uint_as_float(vx[j].r[k]), __uint_as_float(vy[j].r[k]), acc[k]) : acc[k] + __uint_as_float(vx[j].r[k]);
  float v = ((acc[0] + acc[4]) + (acc[2] + acc[6])) + ((acc[1] + acc[5]) + (acc[3] + acc[7]));
  v = block_sum<BLOCK>(v, sm);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = v;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  float w = 0.f;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += BLOCK) w += __ldcg(partials + i);
  __syncthreads();
  w = block_sum<BLOCK>(w, sm);
  if (threadIdx.x == 0) { *out = w; *ticket = 0; }
}

// persistent grid-stride (the previous product shape)
template <int BLOCK, int U, bool DOT>
__global__ void __launch_bounds__(BLOCK) k_persist(int64_t nvec, const float *x, const float *y, float *out, float *partials,
                                                   unsigned *ticket) {
  __shared__ float sm[BLOCK / 32];
  __shared__ bool last;
  const int64_t tid = (int64_t)blockIdx.x * BLOCK + threadIdx.x, nt = (int64_t)gridDim.x * BLOCK;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int64_t base = tid; base < nvec; base += nt * U) {
    V32 vx[U], vy[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int64_t v = base + j * nt;
      if (v < nvec) { vx[j] = ld_nc_256(x + v * 8); if (DOT) vy[j] = ld_nc_256(y + v * 8); }
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int64_t v = base + j * nt;
      if (v < nvec)
#pragma unroll
        for (int k = 0; k < 8; ++k)
          acc[k] = DOT ? __fmaf_rn(__uint_as_float(vx[j].r[k]), __uint_as_float(vy[j].r[k]), acc[k]) : acc[k] + __uint_as_float(vx[j].r[k]);
    }
  }
  float v = ((acc[0] + acc[4]) + (acc[2] + acc[6])) + ((acc[1] + acc[5]) + (acc[3] + acc[7]));
  v = block_sum<BLOCK>(v, sm);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = v;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  float w = 0.f;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += BLOCK) w += __ldcg(partials + i);
  __syncthreads();
  w = block_sum<BLOCK>(w, sm);
  if (threadIdx.x == 0) { *out = w; *ticket = 0; }
}

// balanced: grid = exactly `grid` CTAs, CTA b folds the contiguous vector
// range [b*per, (b+1)*per) in chunks of BLOCK*K (per rounded to a chunk).
template <int BLOCK, int K, bool DOT>
__global__ void __launch_bounds__(BLOCK) k_balanced(int64_t nvec, int64_t per, const float *x, const float *y, float *out,
                                                    float *partials, unsigned *ticket) {
  __shared__ float sm[BLOCK / 32];
  __shared__ bool last;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const int64_t beg = (int64_t)blockIdx.x * per, end = beg + per < nvec ? beg + per : nvec;
  for (int64_t base = beg + threadIdx.x; base < end; base += (int64_t)BLOCK * K) {
    V32 vx[K], vy[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const int64_t v = base + j * BLOCK;
      if (v < end) {
        vx[j] = ld_nc_256(x + v * 8);
        if (DOT) vy[j] = ld_nc_256(y + v * 8);
      } else {
        for (int k = 0; k < 8; ++k) vx[j].r[k] = vy[j].r[k] = 0;
      }
    }
#pragma unroll
    for (int j = 0; j < K; ++j)
#pragma unroll
      for (int k = 0; k < 8; ++k)
        acc[k] = DOT ? __fmaf_rn(__uint_as_float(vx[j].r[k]), __uint_as_float(vy[j].r[k]), acc[k]) : acc[k] + __uint_as_float(vx[j].r[k]);
  }
  float v = ((acc[0] + acc[4]) + (acc[2] + acc[6])) + ((acc[1] + acc[5]) + (acc[3] + acc[7]));
  v = block_sum<BLOCK>(v, sm);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = v;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  float w = 0.f;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += BLOCK) w += __ldcg(partials + i);
  __syncthreads();
  w = block_sum<BLOCK>(w, sm);
  if (threadIdx.x == 0) { *out = w; *ticket = 0; }
}

extern "C" int red_lab(int v, int64_t n, const float *x, const float *y, float *out, void *ws, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t nv = n / 8;
  unsigned *ticket = (unsigned *)ws;
  float *partials = (float *)((char *)ws + 128);
  switch (v) {
#define ONE(id, B, K, D) case id: k_oneshot<B, K, D><<<(int)((nv + B * K - 1) / (B * K)), B, 0, s>>>(nv, x, y, out, partials, ticket); break;
    ONE(0, 256, 4, false) ONE(1, 512, 4, false) ONE(2, 256, 8, false) ONE(3, 512, 2, false) ONE(4, 1024, 4, false)
    ONE(10, 256, 2, true) ONE(11, 512, 2, true) ONE(12, 256, 4, true) ONE(13, 512, 4, true) ONE(14, 1024, 2, true)
#define BAL(id, B, K, D, CTAS) case id: { const int64_t g = 148 * CTAS; int64_t per = (nv + g - 1) / g; \
      per = (per + B * K - 1) / (B * K) * (B * K); const int64_t grid = (nv + per - 1) / per; \
      k_balanced<B, K, D><<<(int)grid, B, 0, s>>>(nv, per, x, y, out, partials, ticket); break; }
    BAL(30, 512, 4, false, 2) BAL(31, 512, 4, false, 4) BAL(32, 512, 4, false, 8) BAL(33, 256, 4, false, 8)
    BAL(34, 512, 2, true, 2) BAL(35, 512, 2, true, 4) BAL(36, 256, 4, false, 4) BAL(37, 512, 4, false, 16)
#define PER(id, B, U, D, BPS) case id: k_persist<B, U, D><<<148 * BPS, B, 0, s>>>(nv, x, y, out, partials, ticket); break;
    PER(20, 256, 4, false, 4) PER(21, 256, 2, true, 4)
    default: return 2;
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
