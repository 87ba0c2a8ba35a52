/* synth.h — the seeded, counter-based synthetic input generator.
 *
 * This module holds NONE of the method's arithmetic (no linear combination,
 * no reduction, no scan).  It is the one piece shared by the CUDA path (which
 * generates its inputs in HBM, see synth_cuda.cu) and the CPU oracle's tests
 * (which regenerate the same values on the host, see synth_host.c), so that
 * both sides see bit-identical data for every (seed, global index) and every
 * shard layout (SURVEY.md §0 fact 9, §8(d) "Synthetic inputs per config").
 *
 * Distribution: "arrays of approximately uniformly distributed random
 * numbers" (§3.2.1, pycuda.curandom).  Values are built
 * from integers only (no libm), so GPU and host agree bit for bit.
 *
 * h(seed, i) = splitmix64_finaliser(seed * 2^40 + i),  i < 2^40.
 */
#ifndef SYNTH_H
#define SYNTH_H
#include <stdint.h>

#if defined(__CUDACC__)
#define SYNTH_FN static __host__ __device__ __forceinline__
#else
#define SYNTH_FN static inline
#endif

/* Distribution kinds (the value recipe per kind is in synth_value_*). */
enum {
  SYNTH_F32_U01 = 0,   /* fp32 U[0,1) on the 2^-24 grid: (h>>40) * 2^-24         */
  SYNTH_F64_U01 = 1,   /* fp64 U[0,1) on the 2^-53 grid: (h>>11) * 2^-53         */
  SYNTH_F32_S11 = 2,   /* fp32 U[-1,1): ((h>>39) - 2^24) * 2^-24                  */
  SYNTH_F64_S11 = 3,   /* fp64 U[-1,1): ((h>>10) - 2^53) * 2^-53                  */
  SYNTH_I32_RANGE = 4, /* int32 U{lo..hi}, hi-lo+1 <= 2^32                         */
  SYNTH_I64_RANGE = 5, /* int64 U{lo..hi}, hi-lo+1 <= 2^32                         */
  SYNTH_I64_FULL = 6,  /* int64 full range: (int64_t)h                             */
  SYNTH_F32_RAMP = 7,  /* fp32 (float)(i + lo)  (closed-form pins; exact < 2^24)   */
  SYNTH_F64_RAMP = 8,  /* fp64 (double)(i + lo)                                     */
  SYNTH_I32_RAMP = 9,  /* int32 (int32_t)(uint32_t)(i + lo)                         */
  SYNTH_I64_RAMP = 10, /* int64 i + lo                                              */
  SYNTH_KIND_COUNT = 11
};

SYNTH_FN uint64_t synth_mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

SYNTH_FN uint64_t synth_hash(uint64_t seed, uint64_t i) {
  return synth_mix64((seed << 40) + i);
}

SYNTH_FN float synth_f32_u01(uint64_t h) { return (float)(h >> 40) * 5.9604644775390625e-08f; }
SYNTH_FN double synth_f64_u01(uint64_t h) { return (double)(h >> 11) * 1.1102230246251565e-16; }
SYNTH_FN float synth_f32_s11(uint64_t h) {
  return (float)((int64_t)(h >> 39) - (int64_t)16777216) * 5.9604644775390625e-08f;
}
SYNTH_FN double synth_f64_s11(uint64_t h) {
  return (double)((int64_t)(h >> 10) - (int64_t)9007199254740992LL) * 1.1102230246251565e-16;
}
/* lo + floor((h>>32) * span / 2^32), span = hi - lo + 1 in [1, 2^32]. */
SYNTH_FN int64_t synth_range(uint64_t h, int64_t lo, int64_t hi) {
  uint64_t span = (uint64_t)(hi - lo) + 1u;
  return lo + (int64_t)(((h >> 32) * span) >> 32);
}

#endif /* SYNTH_H */
