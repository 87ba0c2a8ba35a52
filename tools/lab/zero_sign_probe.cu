// zero_sign_probe.cu — lab probe: how the sm_100a min/max instructions order
// signed zeros (fmaxf/fminf/fmax/fmin on (+0,-0) and (-0,+0)).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(const float *f, const double *d, unsigned *o) {
  float p = f[0], m = f[1];
  double P = d[0], M = d[1];
  o[0] = __float_as_uint(fmaxf(p, m)); o[1] = __float_as_uint(fmaxf(m, p));
  o[2] = __float_as_uint(fminf(p, m)); o[3] = __float_as_uint(fminf(m, p));
  o[4] = (unsigned)(__double_as_longlong(fmax(P, M)) >> 32); o[5] = (unsigned)(__double_as_longlong(fmax(M, P)) >> 32);
  o[6] = (unsigned)(__double_as_longlong(fmin(P, M)) >> 32); o[7] = (unsigned)(__double_as_longlong(fmin(M, P)) >> 32);
}
int main() {
  float hf[2] = {0.0f, -0.0f}; double hd[2] = {0.0, -0.0};
  float *f; double *d; unsigned *o; unsigned h[8];
  cudaMalloc(&f, 8); cudaMalloc(&d, 16); cudaMalloc(&o, 32);
  cudaMemcpy(f, hf, 8, cudaMemcpyHostToDevice); cudaMemcpy(d, hd, 16, cudaMemcpyHostToDevice);
  k<<<1, 1>>>(f, d, o);
  cudaMemcpy(h, o, 32, cudaMemcpyDeviceToHost);
  const char *nm[8] = {"fmaxf(+0,-0)", "fmaxf(-0,+0)", "fminf(+0,-0)", "fminf(-0,+0)", "fmax(+0,-0)", "fmax(-0,+0)", "fmin(+0,-0)", "fmin(-0,+0)"};
  for (int i = 0; i < 8; ++i) printf("%s -> %s0\n", nm[i], (h[i] >> 31) ? "-" : "+");
  return 0;
}
