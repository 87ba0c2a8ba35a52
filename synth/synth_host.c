/* synth_host.c — host twin of the synthetic generator (see synth.h).
 * Test and bench infrastructure: the oracle's inputs are regenerated here, bit
 * identical to what synth_cuda.cu writes into HBM.  No method arithmetic. */
#include <stddef.h>
#include <stdint.h>
#include "synth.h"

int synth_fill_host(int kind, uint64_t seed, int64_t start, int64_t n, int64_t lo, int64_t hi,
                    void *out) {
  if (n < 0 || (n > 0 && !out) || kind < 0 || kind >= SYNTH_KIND_COUNT) return 1;
  if ((kind == SYNTH_I32_RANGE || kind == SYNTH_I64_RANGE) &&
      (hi < lo || (uint64_t)(hi - lo) > 0xffffffffULL)) return 1;
  for (int64_t k = 0; k < n; ++k) {
    uint64_t i = (uint64_t)(start + k);
    uint64_t h = synth_hash(seed, i);
    switch (kind) {
      case SYNTH_F32_U01: ((float *)out)[k] = synth_f32_u01(h); break;
      case SYNTH_F64_U01: ((double *)out)[k] = synth_f64_u01(h); break;
      case SYNTH_F32_S11: ((float *)out)[k] = synth_f32_s11(h); break;
      case SYNTH_F64_S11: ((double *)out)[k] = synth_f64_s11(h); break;
      case SYNTH_I32_RANGE: ((int32_t *)out)[k] = (int32_t)synth_range(h, lo, hi); break;
      case SYNTH_I64_RANGE: ((int64_t *)out)[k] = synth_range(h, lo, hi); break;
      case SYNTH_I64_FULL: ((int64_t *)out)[k] = (int64_t)h; break;
      case SYNTH_F32_RAMP: ((float *)out)[k] = (float)(int64_t)(i + (uint64_t)lo); break;
      case SYNTH_F64_RAMP: ((double *)out)[k] = (double)(int64_t)(i + (uint64_t)lo); break;
      case SYNTH_I32_RAMP: ((int32_t *)out)[k] = (int32_t)(uint32_t)(i + (uint64_t)lo); break;
      case SYNTH_I64_RAMP: ((int64_t *)out)[k] = (int64_t)(i + (uint64_t)lo); break;
    }
  }
  return 0;
}
