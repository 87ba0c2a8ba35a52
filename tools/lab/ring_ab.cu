// ring_ab.cu — tuning lab only: the product ring scan (csrc/scan_r.cu, built
// here with stub host helpers) callable for any (op, kind, dtype, n), to A/B
// it against the product dispatch and pick scan.cu's size window.
#include <cstdarg>
#include <cstdio>

#include "../../paper_1304_5553_b200/csrc/scan_r.cu"

namespace ga {
ga_status_t fail(ga_status_t s, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vfprintf(stderr, fmt, ap);
  va_end(ap);
  fputc('\n', stderr);
  return s;
}
ga_status_t check_launch(const char *what) {
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? GA_OK : fail(GA_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}
int sm_count() {
  static int n = 0;
  if (!n) {
    int d;
    cudaGetDevice(&d);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
  }
  return n;
}
void count_launch() {}
cudaError_t allow_dyn_smem(const void *kernel, size_t bytes) {
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}
}  // namespace ga

extern "C" int ring_ab(int op, int ex, int dt, int64_t n, const void *in, void *out, const void *carry, int64_t cc,
                       void *ws, void *stream) {
  // dt < 0: the widening scan from dtype -dt - 1 (int32 -> int64, float32 -> float64)
  const ga_dtype_t o = (ga_dtype_t)(dt < 0 ? (-dt - 1 == GA_I32 ? GA_I64 : GA_F64) : dt);
  const ga_dtype_t i = (ga_dtype_t)(dt < 0 ? -dt - 1 : dt);
  return (int)ga::scan_impl::launch_ring((ga_op_t)op, ex != 0, i, o, n, in, out, carry, cc, ws, (cudaStream_t)stream);
}

// shape variants (int32 / int64 SUM): v = 0 the product constants, else below
template <typename T, typename Tin = T>
static int ring_cfg(int v, int ex, int64_t n, const void *in, void *out, void *ws, cudaStream_t s) {
  using namespace ga::scan_impl;
#define RC(W, R, S, F, Q, PF, H)                                                                                \
  return (int)(ex ? ring_run<GA_OP_SUM, T, Tin, true, W, R, S, F, Q, PF, H>(n, in, out, nullptr, 0, ws, s)     \
                  : ring_run<GA_OP_SUM, T, Tin, false, W, R, S, F, Q, PF, H>(n, in, out, nullptr, 0, ws, s));
  switch (v) {
    case 1: RC(16, 0, 3, 2, 0, -1, 0)
    case 2: RC(16, 4, 3, 2, 0, -1, 1)
    case 3: RC(16, 2, 3, 2, 0, -1, 1)
    case 4: RC(16, 4, 3, 2, 3, 0, 1)
    case 5: RC(16, 2, 3, 2, 3, 0, 1)
  }
#undef RC
  return 2;
}
extern "C" int ring_ab_cfg(int v, int ex, int dt, int64_t n, const void *in, void *out, void *ws, void *stream) {
  if (dt == 0) return ring_cfg<float>(v, ex, n, in, out, ws, (cudaStream_t)stream);
  if (dt == -3) return ring_cfg<int64_t, int32_t>(v, ex, n, in, out, ws, (cudaStream_t)stream);
  return dt == 2 ? ring_cfg<int32_t>(v, ex, n, in, out, ws, (cudaStream_t)stream)
                 : ring_cfg<int64_t>(v, ex, n, in, out, ws, (cudaStream_t)stream);
}
