// ew_lab.cu — tuning lab for the fp32 axpbyz kernel (not product code).
#include <cuda_runtime.h>
#include <stdint.h>

#include "ga_device.cuh"

using namespace ga;

__device__ __forceinline__ uint4 ld128(const void *p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void st128(void *p, uint4 v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void st128cs(void *p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void st256cs(void *p, const V32 &v) {
  asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v.r[0]), "r"(v.r[1]), "r"(v.r[2]),
               "r"(v.r[3]), "r"(v.r[4]), "r"(v.r[5]), "r"(v.r[6]), "r"(v.r[7]) : "memory");
}
__device__ __forceinline__ V32 ld256ef(const void *p, uint64_t pol) {
  V32 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
               : "=r"(v.r[0]), "=r"(v.r[1]), "=r"(v.r[2]), "=r"(v.r[3]), "=r"(v.r[4]), "=r"(v.r[5]), "=r"(v.r[6]), "=r"(v.r[7])
               : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float f(float a, float x, float b, float y) { return __fadd_rn(__fmul_rn(a, x), __fmul_rn(b, y)); }

// A: one-shot grid, 256-bit, each thread K vectors spaced by blockDim (no loop)
template <int BLOCK, int K, int STORE>
__global__ void __launch_bounds__(BLOCK) k_oneshot256(int64_t nvec, float a, const float *x, float b, const float *y, float *z) {
  const int64_t base = (int64_t)blockIdx.x * BLOCK * K + threadIdx.x;
  V32 vx[K], vy[K];
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const int64_t v = base + j * BLOCK;
    if (v < nvec) {
      if (STORE == 2) { vx[j] = ld256ef(x + v * 8, pol); vy[j] = ld256ef(y + v * 8, pol); }
      else { vx[j] = ld_nc_256(x + v * 8); vy[j] = ld_nc_256(y + v * 8); }
    }
  }
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const int64_t v = base + j * BLOCK;
    if (v < nvec) {
      V32 o;
#pragma unroll
      for (int k = 0; k < 8; ++k) o.r[k] = __float_as_uint(f(a, __uint_as_float(vx[j].r[k]), b, __uint_as_float(vy[j].r[k])));
      if (STORE == 1) st256cs(z + v * 8, o);
      else st_256(z + v * 8, o);
    }
  }
}

// B: one-shot grid, 128-bit
template <int BLOCK, int K>
__global__ void __launch_bounds__(BLOCK) k_oneshot128(int64_t nvec, float a, const float *x, float b, const float *y, float *z) {
  const int64_t base = (int64_t)blockIdx.x * BLOCK * K + threadIdx.x;
  uint4 vx[K], vy[K];
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const int64_t v = base + j * BLOCK;
    if (v < nvec) { vx[j] = ld128(x + v * 4); vy[j] = ld128(y + v * 4); }
  }
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const int64_t v = base + j * BLOCK;
    if (v < nvec) {
      uint4 o;
      o.x = __float_as_uint(f(a, __uint_as_float(vx[j].x), b, __uint_as_float(vy[j].x)));
      o.y = __float_as_uint(f(a, __uint_as_float(vx[j].y), b, __uint_as_float(vy[j].y)));
      o.z = __float_as_uint(f(a, __uint_as_float(vx[j].z), b, __uint_as_float(vy[j].z)));
      o.w = __float_as_uint(f(a, __uint_as_float(vx[j].w), b, __uint_as_float(vy[j].w)));
      st128(z + v * 4, o);
    }
  }
}

// C: persistent grid-stride 256-bit (the product shape) with BLOCK/UNROLL/blocks-per-SM knobs
template <int BLOCK, int U>
__global__ void __launch_bounds__(BLOCK) k_persist256(int64_t nvec, float a, const float *x, float b, const float *y, float *z) {
  const int64_t tid = (int64_t)blockIdx.x * BLOCK + threadIdx.x;
  const int64_t nt = (int64_t)gridDim.x * BLOCK;
  for (int64_t base = tid; base < nvec; base += nt * U) {
    V32 vx[U], vy[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int64_t v = base + j * nt;
      if (v < nvec) { vx[j] = ld_nc_256(x + v * 8); vy[j] = ld_nc_256(y + v * 8); }
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int64_t v = base + j * nt;
      if (v < nvec) {
        V32 o;
#pragma unroll
        for (int k = 0; k < 8; ++k) o.r[k] = __float_as_uint(f(a, __uint_as_float(vx[j].r[k]), b, __uint_as_float(vy[j].r[k])));
        st_256(z + v * 8, o);
      }
    }
  }
}

extern "C" int ew_lab(int v, int64_t n, float a, const float *x, float b, const float *y, float *z, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  int sms = 148;
  const int64_t nv8 = n / 8, nv4 = n / 4;
  switch (v) {
#define ONE256(id, B, K, ST) case id: k_oneshot256<B, K, ST><<<(int)((nv8 + B * K - 1) / (B * K)), B, 0, s>>>(nv8, a, x, b, y, z); break;
#define ONE128(id, B, K) case id: k_oneshot128<B, K><<<(int)((nv4 + B * K - 1) / (B * K)), B, 0, s>>>(nv4, a, x, b, y, z); break;
#define PER(id, B, U, BPS) case id: k_persist256<B, U><<<sms * BPS, B, 0, s>>>(nv8, a, x, b, y, z); break;
    ONE256(0, 256, 1, 0) ONE256(1, 256, 2, 0) ONE256(2, 256, 4, 0) ONE256(3, 128, 2, 0) ONE256(4, 512, 2, 0)
    ONE256(5, 256, 2, 1) ONE256(6, 256, 2, 2) ONE256(7, 128, 4, 0)
    ONE128(10, 256, 2) ONE128(11, 256, 4) ONE128(12, 128, 4) ONE128(13, 512, 4) ONE128(14, 128, 8)
    PER(20, 256, 2, 4) PER(21, 256, 1, 8) PER(22, 256, 4, 2) PER(23, 512, 2, 2) PER(24, 128, 2, 8) PER(25, 256, 2, 8)
    PER(26, 256, 1, 4) PER(27, 1024, 1, 2)
    default: return 2;
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
