// ga_device.cuh — device helpers shared by the product kernels (NOT by the
// oracle): 256-bit global loads/stores, element arithmetic with explicit
// rounding, reduction operators with their neutral elements, warp folds.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "gpuarray.h"

namespace ga {

// ---------------------------------------------------------------------------
// Programmatic dependent launch.  Every product kernel is launched with
// programmatic stream serialization (ga_host.h launch()), so its CTAs may be
// scheduled while the previous grid of the stream is still finishing.  The
// first statement of every kernel is pdl_enter(): wait until the previous
// grid has completed and its memory operations are visible (nothing of this
// kernel touches global memory before that), then allow the next grid to
// begin launching — it fires once every CTA of this grid has started, i.e.
// during the last wave, so the next kernel's launch, CTA dispatch and
// prologue overlap this kernel's tail instead of following it.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---------------------------------------------------------------------------
// 256-bit memory operations (sm_100: LDG.E.NA.ENL2.256 / STG.E.NA.ENL2.256).
// Streaming data is touched once, so loads skip L1 allocation.
// ---------------------------------------------------------------------------
struct alignas(32) V32 {
  uint32_t r[8];
};

// Read-only (non-coherent) path: valid when the buffer is not written during
// the kernel.  .L2::256B asks L2 to fetch the full 256-byte line pair.
__device__ __forceinline__ V32 ld_nc_256(const void *p) {
  V32 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v.r[0]), "=r"(v.r[1]), "=r"(v.r[2]), "=r"(v.r[3]), "=r"(v.r[4]), "=r"(v.r[5]),
                 "=r"(v.r[6]), "=r"(v.r[7])
               : "l"(p));
  return v;
}

// Coherent path: for in-place calls where the same addresses are written.
__device__ __forceinline__ V32 ld_256(const void *p) {
  V32 v;
  asm volatile("ld.global.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v.r[0]), "=r"(v.r[1]), "=r"(v.r[2]), "=r"(v.r[3]), "=r"(v.r[4]), "=r"(v.r[5]),
                 "=r"(v.r[6]), "=r"(v.r[7])
               : "l"(p)
               : "memory");
  return v;
}

__device__ __forceinline__ void st_256(void *p, const V32 &v) {
  asm volatile("st.global.L1::no_allocate.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p),
               "r"(v.r[0]), "r"(v.r[1]), "r"(v.r[2]), "r"(v.r[3]), "r"(v.r[4]), "r"(v.r[5]), "r"(v.r[6]),
               "r"(v.r[7])
               : "memory");
}

// Complex element types (interleaved re, im), §8(f) NEXT-3.
struct alignas(8) c64 {
  float re, im;
};
struct alignas(16) c128 {
  double re, im;
};
template <typename T>
struct is_complex : std::false_type {};
template <>
struct is_complex<c64> : std::true_type {};
template <>
struct is_complex<c128> : std::true_type {};

template <bool NC>
__device__ __forceinline__ V32 ld_vec(const void *p) {
  if constexpr (NC) return ld_nc_256(p);
  else return ld_256(p);
}

// Element k of a 32-byte vector viewed as T[32/sizeof(T)].
template <typename T>
__device__ __forceinline__ T vget(const V32 &v, int k);
template <>
__device__ __forceinline__ float vget<float>(const V32 &v, int k) { return __uint_as_float(v.r[k]); }
template <>
__device__ __forceinline__ int32_t vget<int32_t>(const V32 &v, int k) { return (int32_t)v.r[k]; }
template <>
__device__ __forceinline__ double vget<double>(const V32 &v, int k) {
  return __hiloint2double((int)v.r[2 * k + 1], (int)v.r[2 * k]);
}
template <>
__device__ __forceinline__ int64_t vget<int64_t>(const V32 &v, int k) {
  return (int64_t)(((uint64_t)v.r[2 * k + 1] << 32) | v.r[2 * k]);
}

template <>
__device__ __forceinline__ c64 vget<c64>(const V32 &v, int k) {
  return c64{__uint_as_float(v.r[2 * k]), __uint_as_float(v.r[2 * k + 1])};
}
template <>
__device__ __forceinline__ c128 vget<c128>(const V32 &v, int k) {
  return c128{__hiloint2double((int)v.r[4 * k + 1], (int)v.r[4 * k]),
              __hiloint2double((int)v.r[4 * k + 3], (int)v.r[4 * k + 2])};
}

template <typename T>
__device__ __forceinline__ void vset(V32 &v, int k, T x);
template <>
__device__ __forceinline__ void vset<float>(V32 &v, int k, float x) { v.r[k] = __float_as_uint(x); }
template <>
__device__ __forceinline__ void vset<int32_t>(V32 &v, int k, int32_t x) { v.r[k] = (uint32_t)x; }
template <>
__device__ __forceinline__ void vset<double>(V32 &v, int k, double x) {
  v.r[2 * k] = (uint32_t)__double2loint(x);
  v.r[2 * k + 1] = (uint32_t)__double2hiint(x);
}
template <>
__device__ __forceinline__ void vset<int64_t>(V32 &v, int k, int64_t x) {
  v.r[2 * k] = (uint32_t)(uint64_t)x;
  v.r[2 * k + 1] = (uint32_t)((uint64_t)x >> 32);
}

template <>
__device__ __forceinline__ void vset<c64>(V32 &v, int k, c64 x) {
  v.r[2 * k] = __float_as_uint(x.re);
  v.r[2 * k + 1] = __float_as_uint(x.im);
}
template <>
__device__ __forceinline__ void vset<c128>(V32 &v, int k, c128 x) {
  v.r[4 * k] = (uint32_t)__double2loint(x.re);
  v.r[4 * k + 1] = (uint32_t)__double2hiint(x.re);
  v.r[4 * k + 2] = (uint32_t)__double2loint(x.im);
  v.r[4 * k + 3] = (uint32_t)__double2hiint(x.im);
}

// ---------------------------------------------------------------------------
// Element arithmetic with the rounding sequence DESIGN.md R1 fixes:
// mul = RN(a*b), add = RN(a+b), never contracted to FMA.  Integers wrap.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float e_mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double e_mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ int32_t e_mul(int32_t a, int32_t b) { return (int32_t)((uint32_t)a * (uint32_t)b); }
__device__ __forceinline__ int64_t e_mul(int64_t a, int64_t b) { return (int64_t)((uint64_t)a * (uint64_t)b); }
__device__ __forceinline__ float e_add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double e_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ int32_t e_add(int32_t a, int32_t b) { return (int32_t)((uint32_t)a + (uint32_t)b); }
__device__ __forceinline__ int64_t e_add(int64_t a, int64_t b) { return (int64_t)((uint64_t)a + (uint64_t)b); }
__device__ __forceinline__ int32_t e_sub(int32_t a, int32_t b) { return (int32_t)((uint32_t)a - (uint32_t)b); }
__device__ __forceinline__ int64_t e_sub(int64_t a, int64_t b) { return (int64_t)((uint64_t)a - (uint64_t)b); }
__device__ __forceinline__ float e_div(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double e_div(double a, double b) { return __ddiv_rn(a, b); }
// Complex (R24): the product written out component-wise, every operation RN:
// re(u*v) = RN(RN(ur*vr) - RN(ui*vi)), im(u*v) = RN(RN(ur*vi) + RN(ui*vr)).
__device__ __forceinline__ c64 e_mul(c64 u, c64 v) {
  return c64{__fsub_rn(__fmul_rn(u.re, v.re), __fmul_rn(u.im, v.im)),
             __fadd_rn(__fmul_rn(u.re, v.im), __fmul_rn(u.im, v.re))};
}
__device__ __forceinline__ c128 e_mul(c128 u, c128 v) {
  return c128{__dsub_rn(__dmul_rn(u.re, v.re), __dmul_rn(u.im, v.im)),
              __dadd_rn(__dmul_rn(u.re, v.im), __dmul_rn(u.im, v.re))};
}
__device__ __forceinline__ c64 e_add(c64 u, c64 v) { return c64{__fadd_rn(u.re, v.re), __fadd_rn(u.im, v.im)}; }
__device__ __forceinline__ c128 e_add(c128 u, c128 v) { return c128{__dadd_rn(u.re, v.re), __dadd_rn(u.im, v.im)}; }
// Fused multiply-add (one rounding) — used only where a tolerance, not
// bit-exactness, is the contract (float SUM reductions, R9).
__device__ __forceinline__ float e_fma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double e_fma(double a, double b, double c) { return __fma_rn(a, b, c); }

// ---------------------------------------------------------------------------
// Reduction operators "a+b" / max / min and their neutral elements
// (PAPER.md:479-485 footnote; R5, R6).
// ---------------------------------------------------------------------------
template <typename T>
struct Limits;
template <>
struct Limits<float> {
  __device__ static float lowest() { return -__int_as_float(0x7f800000); }
  __device__ static float highest() { return __int_as_float(0x7f800000); }
};
template <>
struct Limits<double> {
  __device__ static double lowest() { return -__longlong_as_double(0x7ff0000000000000LL); }
  __device__ static double highest() { return __longlong_as_double(0x7ff0000000000000LL); }
};
template <>
struct Limits<int32_t> {
  __device__ static int32_t lowest() { return INT32_MIN; }
  __device__ static int32_t highest() { return INT32_MAX; }
};
template <>
struct Limits<int64_t> {
  __device__ static int64_t lowest() { return INT64_MIN; }
  __device__ static int64_t highest() { return INT64_MAX; }
};

template <int OP, typename T>
struct Op;

template <typename T>
__device__ __forceinline__ T zero_of() {
  if constexpr (is_complex<T>::value) return T{0, 0};
  else return T(0);
}

template <typename T>
struct Op<GA_OP_SUM, T> {
  __device__ static T neutral() { return zero_of<T>(); }
  __device__ static T fold(T a, T b) { return e_add(a, b); }
};
// Floats: maximumNumber / minimumNumber of IEEE 754-2019 — a NaN operand
// loses (R6) and -0 < +0 (R7), a total order on the non-NaN values, so a
// fold gives the same bits in any order.  sm_100a's FMNMX / DMNMX (fmaxf,
// fminf, fmax, fmin) already order the zeros that way in both operand
// orders (tools/lab/zero_sign_probe.cu), so no tie-break is needed here.
template <typename T>
struct Op<GA_OP_MAX, T> {
  __device__ static T neutral() { return Limits<T>::lowest(); }
  __device__ static T fold(T a, T b) {
    if constexpr (std::is_same<T, float>::value) return fmaxf(a, b);
    else if constexpr (std::is_same<T, double>::value) return fmax(a, b);
    else return a > b ? a : b;
  }
};
template <typename T>
struct Op<GA_OP_MIN, T> {
  __device__ static T neutral() { return Limits<T>::highest(); }
  __device__ static T fold(T a, T b) {
    if constexpr (std::is_same<T, float>::value) return fminf(a, b);
    else if constexpr (std::is_same<T, double>::value) return fmin(a, b);
    else return a < b ? a : b;
  }
};

// Warp shuffle for scalar and complex elements.
template <typename T>
__device__ __forceinline__ T shfl_xor(T v, int off) {
  if constexpr (is_complex<T>::value)
    return T{__shfl_xor_sync(0xffffffffu, v.re, off), __shfl_xor_sync(0xffffffffu, v.im, off)};
  else return __shfl_xor_sync(0xffffffffu, v, off);
}
// L2 load (bypassing L1) of scalar and complex elements.
template <typename T>
__device__ __forceinline__ T ldcg(const T *p) {
  if constexpr (is_complex<T>::value) return T{__ldcg(&p->re), __ldcg(&p->im)};
  else return __ldcg(p);
}

// Warp-wide fold with a fixed xor-butterfly order: every lane ends with the
// same value, bit-identical run to run.
template <int OP, typename T>
__device__ __forceinline__ T warp_fold(T v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = Op<OP, T>::fold(v, shfl_xor<T>(v, off));
  return v;
}

// Coefficient with a device-resident factor (ga_dscalar_t): RN(scale *
// RN(num / den)), a missing pointer standing for 1, both missing: scale.  A
// zero numerator gives a zero factor whatever the denominator (a converged CG
// iteration has 0/0 and must stay finite).
template <typename T>
__device__ __forceinline__ T coef(T scale, const T *num, const T *den) {
  if constexpr (std::is_floating_point<T>::value) {
    if (!num && !den) return scale;
    const T nv = num ? *num : T(1);
    const T q = nv == T(0) ? T(0) : (den ? e_div(nv, *den) : nv);
    return e_mul(scale, q);
  } else {
    return scale;
  }
}

}  // namespace ga
