// cg_lab.cu — the PRODUCT fused CG kernels (csrc/cg_kernel.cuh) at other
// (vectors per thread, min CTAs per SM) shapes.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "cg_kernel.cuh"

using namespace ga;
using namespace ga::cg_detail;

static int grid_for(int64_t nvec, int unroll) {
  return (int)std::max<int64_t>(std::min<int64_t>((nvec + 256LL * unroll - 1) / (256LL * unroll), RED_MAX_PARTIALS), 1);
}

template <int U, int M, int LP>
static int dir(int64_t n, const float *r, const float *pin, float *pout, float *ap, float *out, void *ws,
               const float *num, const float *den, cudaStream_t s) {
  DirArgs<float> a{};
  a.n = n;
  a.nvec = n / 8;
  a.bscale = 1.0f;
  a.bnum = num;
  a.bden = den;
  a.l = -1.0f;
  a.d = 4.0f;
  a.u = -1.0f;
  a.diag = nullptr;
  a.r = r;
  a.pin = pin;
  a.pout = pout;
  a.ap = ap;
  a.out = out;
  a.fin = Finish{(char *)ws, RED_GROUP};  // = make_finish on a full B200
  cg_direction_kernel<float, U, M, false><<<grid_for(a.nvec, U * LP), CG_BLOCK, 0, s>>>(a);
  return (int)cudaGetLastError();
}

template <int U, int M, int LP>
static int upd(int64_t n, float *x, float *r, const float *p, const float *ap, float *out, void *ws,
               const float *num, const float *den, cudaStream_t s) {
  UpdArgs<float> a{};
  a.n = n;
  a.nvec = n / 8;
  a.ascale = 1.0f;
  a.anum = num;
  a.aden = den;
  a.x = x;
  a.r = r;
  a.p = p;
  a.ap = ap;
  a.out = out;
  a.fin = Finish{(char *)ws, RED_GROUP};  // = make_finish on a full B200
  cg_update_kernel<float, U, M><<<grid_for(a.nvec, U * LP), CG_BLOCK, 0, s>>>(a);
  return (int)cudaGetLastError();
}

#define V(X) X(0, 1, 4, 4) X(1, 1, 4, 8) X(2, 1, 4, 16) X(3, 2, 4, 8) X(4, 2, 2, 4) X(5, 1, 4, 2) X(6, 1, 6, 8) X(7, 2, 4, 16)

extern "C" int lab_dir(int v, int64_t n, const float *r, const float *pin, float *pout, float *ap, float *out,
                       void *ws, const float *num, const float *den, void *stream) {
  switch (v) {
#define C(id, U, M, LP) case id: return dir<U, M, LP>(n, r, pin, pout, ap, out, ws, num, den, (cudaStream_t)stream);
    V(C)
#undef C
  }
  return -1;
}
extern "C" int lab_upd(int v, int64_t n, float *x, float *r, const float *p, const float *ap, float *out, void *ws,
                       const float *num, const float *den, void *stream) {
  switch (v) {
#define C(id, U, M, LP) case id: return upd<U, M, LP>(n, x, r, p, ap, out, ws, num, den, (cudaStream_t)stream);
    V(C)
#undef C
  }
  return -1;
}
