// red_shape_lab.cu — times the product reduce_kernel at other CTA shapes.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "reduce_kernel.cuh"

using namespace ga;
using namespace ga::red_detail;

template <int MAP, int U, int B, int MINB>
static int run(int64_t n, const float *x, const float *y, float *out, void *ws, cudaStream_t s) {
  RedArgs<float, float> p;
  p.n = n;
  p.head = 0;
  p.nvec = n / 8;
  p.x = x;
  p.y = y;
  p.out = out;
  p.xg = Exchange();
  const int64_t units = (p.nvec + (int64_t)B * U - 1) / ((int64_t)B * U);
  const int grid = (int)std::max<int64_t>(std::min<int64_t>(units, RED_MAX_PARTIALS), 1);
  p.fin = Finish{(char *)ws, RED_GROUP};  // = make_finish on a full B200
  reduce_kernel<float, float, GA_OP_SUM, MAP, U, B, MINB><<<grid, B, 0, s>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

#define V(X) \
  X(0, GA_MAP_ID, 4, 512, 1) X(1, GA_MAP_ID, 4, 512, 2) X(2, GA_MAP_ID, 4, 512, 3) X(3, GA_MAP_ID, 4, 256, 4) \
  X(4, GA_MAP_ID, 4, 256, 6) X(5, GA_MAP_ID, 8, 256, 4) X(6, GA_MAP_ID, 2, 512, 3) X(7, GA_MAP_ID, 4, 1024, 1) \
  X(8, GA_MAP_ID, 2, 256, 8) X(9, GA_MAP_ID, 1, 256, 8) \
  X(10, GA_MAP_MUL, 2, 512, 1) X(11, GA_MAP_MUL, 2, 512, 2) X(12, GA_MAP_MUL, 2, 512, 3) X(13, GA_MAP_MUL, 2, 256, 4) \
  X(14, GA_MAP_MUL, 2, 256, 6) X(15, GA_MAP_MUL, 4, 256, 4) X(16, GA_MAP_MUL, 1, 512, 4) X(17, GA_MAP_MUL, 2, 1024, 1) X(18, GA_MAP_MUL, 1, 256, 8) \
  X(19, GA_MAP_ID, 8, 256, 3) X(20, GA_MAP_ID, 16, 256, 2) X(21, GA_MAP_MUL, 4, 256, 3) X(22, GA_MAP_MUL, 8, 256, 2) X(23, GA_MAP_ID, 8, 128, 8)

extern "C" int red_lab(int v, int64_t n, const float *x, const float *y, float *out, void *ws, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  switch (v) {
#define C(id, M, U, B, MB) case id: return run<M, U, B, MB>(n, x, y, out, ws, s);
    V(C)
#undef C
  }
  return 2;
}
