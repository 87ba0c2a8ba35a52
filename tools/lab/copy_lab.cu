// copy_lab.cu — tuning lab only: the 1 read : 1 write HBM ceiling that
// bounds the scan (8 B/elt int32 = a copy's traffic).  One-shot grids of
// 128-bit or 256-bit loads/stores, UNROLL vectors in flight per thread, plus
// a write-only fill for the single-direction limit.
#include <cuda_runtime.h>
#include <stdint.h>

template <int BLOCK, int UNROLL, bool WIDE>
__global__ void __launch_bounds__(BLOCK) copy_kernel(const uint4 *in, uint4 *out, int64_t nvec) {
  constexpr int V = WIDE ? 2 : 1;  // uint4 per access
  const int64_t base = (int64_t)blockIdx.x * BLOCK * UNROLL * V + threadIdx.x * V;
  uint4 r[UNROLL][V];
#pragma unroll
  for (int u = 0; u < UNROLL; ++u) {
    const int64_t i = base + (int64_t)u * BLOCK * V;
    if (i < nvec) {
      if constexpr (WIDE) {
        asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[u][0].x), "=r"(r[u][0].y), "=r"(r[u][0].z), "=r"(r[u][0].w), "=r"(r[u][V - 1].x),
                       "=r"(r[u][V - 1].y), "=r"(r[u][V - 1].z), "=r"(r[u][V - 1].w)
                     : "l"(in + i));
      } else {
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r[u][0].x), "=r"(r[u][0].y), "=r"(r[u][0].z), "=r"(r[u][0].w)
                     : "l"(in + i));
      }
    }
  }
#pragma unroll
  for (int u = 0; u < UNROLL; ++u) {
    const int64_t i = base + (int64_t)u * BLOCK * V;
    if (i < nvec) {
      if constexpr (WIDE) {
        asm volatile("st.global.L1::no_allocate.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(out + i),
                     "r"(r[u][0].x), "r"(r[u][0].y), "r"(r[u][0].z), "r"(r[u][0].w), "r"(r[u][V - 1].x),
                     "r"(r[u][V - 1].y), "r"(r[u][V - 1].z), "r"(r[u][V - 1].w)
                     : "memory");
      } else {
        asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(out + i), "r"(r[u][0].x),
                     "r"(r[u][0].y), "r"(r[u][0].z), "r"(r[u][0].w)
                     : "memory");
      }
    }
  }
}

template <int BLOCK, int UNROLL>
__global__ void __launch_bounds__(BLOCK) fill_kernel(uint4 *out, int64_t nvec, uint32_t v) {
  const int64_t base = (int64_t)blockIdx.x * BLOCK * UNROLL * 2 + threadIdx.x * 2;
#pragma unroll
  for (int u = 0; u < UNROLL; ++u) {
    const int64_t i = base + (int64_t)u * BLOCK * 2;
    if (i < nvec)
      asm volatile("st.global.L1::no_allocate.v8.u32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(out + i), "r"(v)
                   : "memory");
  }
}

// 2 reads : 1 write (axpbyz's traffic mix): out = a ^ b, 256-bit, UNROLL
// vectors per input in flight per thread.
template <int BLOCK, int UNROLL>
__global__ void __launch_bounds__(BLOCK) mix21_kernel(const uint4 *a, const uint4 *b, uint4 *out, int64_t nvec) {
  const int64_t base = (int64_t)blockIdx.x * BLOCK * UNROLL * 2 + threadIdx.x * 2;
  uint4 ra[UNROLL][2], rb[UNROLL][2];
#pragma unroll
  for (int u = 0; u < UNROLL; ++u) {
    const int64_t i = base + (int64_t)u * BLOCK * 2;
    if (i < nvec) {
      asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(ra[u][0].x), "=r"(ra[u][0].y), "=r"(ra[u][0].z), "=r"(ra[u][0].w), "=r"(ra[u][1].x),
                     "=r"(ra[u][1].y), "=r"(ra[u][1].z), "=r"(ra[u][1].w)
                   : "l"(a + i));
      asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(rb[u][0].x), "=r"(rb[u][0].y), "=r"(rb[u][0].z), "=r"(rb[u][0].w), "=r"(rb[u][1].x),
                     "=r"(rb[u][1].y), "=r"(rb[u][1].z), "=r"(rb[u][1].w)
                   : "l"(b + i));
    }
  }
#pragma unroll
  for (int u = 0; u < UNROLL; ++u) {
    const int64_t i = base + (int64_t)u * BLOCK * 2;
    if (i < nvec)
      asm volatile("st.global.L1::no_allocate.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(out + i),
                   "r"(ra[u][0].x ^ rb[u][0].x), "r"(ra[u][0].y ^ rb[u][0].y), "r"(ra[u][0].z ^ rb[u][0].z),
                   "r"(ra[u][0].w ^ rb[u][0].w), "r"(ra[u][1].x ^ rb[u][1].x), "r"(ra[u][1].y ^ rb[u][1].y),
                   "r"(ra[u][1].z ^ rb[u][1].z), "r"(ra[u][1].w ^ rb[u][1].w)
                   : "memory");
  }
}

extern "C" int copy_lab(int v, int64_t bytes, const void *in, void *out, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t nvec = bytes / 16;
  auto g = [&](int block, int unroll, int per) {
    return (int)((nvec + (int64_t)block * unroll * per - 1) / ((int64_t)block * unroll * per));
  };
  const uint4 *i4 = (const uint4 *)in;
  uint4 *o4 = (uint4 *)out;
  switch (v) {
    case 0: copy_kernel<256, 8, false><<<g(256, 8, 1), 256, 0, s>>>(i4, o4, nvec); break;
    case 1: copy_kernel<256, 4, true><<<g(256, 4, 2), 256, 0, s>>>(i4, o4, nvec); break;
    case 2: copy_kernel<256, 8, true><<<g(256, 8, 2), 256, 0, s>>>(i4, o4, nvec); break;
    case 3: copy_kernel<512, 4, true><<<g(512, 4, 2), 512, 0, s>>>(i4, o4, nvec); break;
    case 4: copy_kernel<256, 16, false><<<g(256, 16, 1), 256, 0, s>>>(i4, o4, nvec); break;
    case 5: copy_kernel<128, 8, true><<<g(128, 8, 2), 128, 0, s>>>(i4, o4, nvec); break;
    case 20: mix21_kernel<256, 2><<<g(256, 2, 2), 256, 0, s>>>(i4, i4 + nvec, o4, nvec); break;
    case 21: mix21_kernel<256, 4><<<g(256, 4, 2), 256, 0, s>>>(i4, i4 + nvec, o4, nvec); break;
    case 22: mix21_kernel<512, 2><<<g(512, 2, 2), 512, 0, s>>>(i4, i4 + nvec, o4, nvec); break;
    case 23: mix21_kernel<128, 4><<<g(128, 4, 2), 128, 0, s>>>(i4, i4 + nvec, o4, nvec); break;
    case 10: fill_kernel<256, 4><<<g(256, 4, 2), 256, 0, s>>>(o4, nvec, 7u); break;
    case 11: fill_kernel<256, 8><<<g(256, 8, 2), 256, 0, s>>>(o4, nvec, 7u); break;
    default: return 2;
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
