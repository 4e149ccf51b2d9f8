// Max relative error of MUFU.RSQ64H (rsqrt.approx.ftz.f64) and of one Newton step from it.
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
__global__ void k(const double* x, double* y0, double* y1, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double a = x[i], r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
  y0[i] = r;
  double h = a * r;
  double e = fma(-h, r, 1.0);
  y1[i] = fma(r * 0.5, e, r);  // Newton
}
int main() {
  const int n = 1 << 22;
  double *x, *y0, *y1;
  cudaMallocManaged(&x, n * 8); cudaMallocManaged(&y0, n * 8); cudaMallocManaged(&y1, n * 8);
  unsigned s = 12345;
  for (int i = 0; i < n; ++i) { s = s * 1664525u + 1013904223u; x[i] = std::ldexp(1.0 + (s >> 8) / 16777216.0, (int)(s % 40) - 20); }
  k<<<(n + 255) / 256, 256>>>(x, y0, y1, n);
  cudaDeviceSynchronize();
  long double m0 = 0, m1 = 0;
  for (int i = 0; i < n; ++i) {
    long double ex = 1.0L / sqrtl((long double)x[i]);
    long double e0 = fabsl((y0[i] - ex) / ex), e1 = fabsl((y1[i] - ex) / ex);
    if (e0 > m0) m0 = e0;
    if (e1 > m1) m1 = e1;
  }
  printf("{\"rsq64h_max_rel\": %.3Le, \"log2\": %.2f, \"newton1_max_rel\": %.3Le}\n", m0, (double)log2l(m0), m1);
}
