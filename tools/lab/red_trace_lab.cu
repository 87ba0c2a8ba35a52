// red_trace_lab.cu — tuning lab only: where the fixed per-launch cost of a
// one-shot streaming reduction goes.  Same structure as the product sum
// kernel (256 threads, 8 x 32-byte vectors in flight per thread, one batch
// per CTA, block partial + atomic ticket), with per-CTA globaltimer stamps:
// trace[4b+0] = start, [4b+1] = last load returned, [4b+2] = end, [4b+3] = SM id.
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint64_t gt_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t smid() {
  uint32_t s;
  asm volatile("mov.u32 %0, %smid;" : "=r"(s));
  return s;
}

template <int BLOCK, int UNROLL>
__global__ void __launch_bounds__(BLOCK, 4) red_trace_kernel(const float4 *x, int64_t nvec, float *partials,
                                                             unsigned *ticket, float *out, uint64_t *trace) {
  __shared__ float sm[BLOCK / 32];
  __shared__ bool last;
  const uint64_t t0 = gt_ns();
  const int64_t base = (int64_t)blockIdx.x * BLOCK * UNROLL * 2 + threadIdx.x * 2;
  float acc = 0.f;
  float4 v[UNROLL][2];
#pragma unroll
  for (int u = 0; u < UNROLL; ++u) {
    const int64_t i = base + (int64_t)u * BLOCK * 2;
    if (i < nvec) {
      asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=f"(v[u][0].x), "=f"(v[u][0].y), "=f"(v[u][0].z), "=f"(v[u][0].w), "=f"(v[u][1].x),
                     "=f"(v[u][1].y), "=f"(v[u][1].z), "=f"(v[u][1].w)
                   : "l"(x + i));
    } else {
      v[u][0] = v[u][1] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
#pragma unroll
  for (int u = 0; u < UNROLL; ++u)
    acc += ((v[u][0].x + v[u][0].y) + (v[u][0].z + v[u][0].w)) + ((v[u][1].x + v[u][1].y) + (v[u][1].z + v[u][1].w));
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = acc;
  __syncthreads();
  const uint64_t t1 = gt_ns();
  if (threadIdx.x == 0) {
    float s = 0.f;
    for (int w = 0; w < BLOCK / 32; ++w) s += sm[w];
    partials[blockIdx.x] = s;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last) {
    float s = 0.f;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += BLOCK) s += __ldcg(partials + i);
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, s);
    if (threadIdx.x == 0) *ticket = 0;
  }
  if (threadIdx.x == 0) {
    trace[4 * blockIdx.x + 0] = t0;
    trace[4 * blockIdx.x + 1] = t1;
    trace[4 * blockIdx.x + 2] = gt_ns();
    trace[4 * blockIdx.x + 3] = smid();
  }
}

extern "C" int red_trace(int64_t n, const float *x, float *partials, unsigned *ticket, float *out, uint64_t *trace,
                         void *stream) {
  const int64_t nvec = n / 4;
  const int grid = (int)((nvec + 256 * 8 * 2 - 1) / (256 * 8 * 2));
  red_trace_kernel<256, 8><<<grid, 256, 0, (cudaStream_t)stream>>>((const float4 *)x, nvec, partials, ticket, out,
                                                                    trace);
  return cudaGetLastError() == cudaSuccess ? grid : -1;
}
