// Dependent-chain latency of DFMA / DMUL / MUFU.RSQ64H / LDS on this part (one warp, clock64).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* cyc, double a, double b, int n) {
  __shared__ double sm[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) sm[i] = 0.0;
  __syncthreads();
  double x = threadIdx.x * 1e-9 + 1.0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  double y = x;
  for (int i = 0; i < n; ++i) y = y * a;
  long long t2 = clock64();
  double z = y + 2.0;
  for (int i = 0; i < n; ++i) {
    double r;
    asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(z));
    z = r + 1.0;  // dependent: MUFU + DADD
  }
  long long t3 = clock64();
  int idx = ((int)z) & 0;
  double w = 0;
  for (int i = 0; i < n; ++i) {
    w = sm[idx];
    idx = ((int)w) & 255;  // dependent LDS chain (+ F2I + LOP)
  }
  long long t4 = clock64();
  out[threadIdx.x] = x + y + z + w;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3;
  }
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1024 * 8); cudaMallocManaged(&cyc, 4 * 8);
  const int n = 4096;
  lat<<<1, 32>>>(out, cyc, 0.9999999, 1e-9, n);
  cudaDeviceSynchronize();
  lat<<<1, 32>>>(out, cyc, 0.9999999, 1e-9, n);
  cudaDeviceSynchronize();
  printf("{\"dfma_lat\": %.2f, \"dmul_lat\": %.2f, \"rsq64h_plus_dadd_lat\": %.2f, \"lds_f2i_lop_lat\": %.2f}\n",
         (double)cyc[0] / n, (double)cyc[1] / n, (double)cyc[2] / n, (double)cyc[3] / n);
  return 0;
}
