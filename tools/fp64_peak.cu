// FP64 DFMA-throughput microbenchmark for the roofline denominator.
// Measures the B200's sustained FP64 FMA rate with many independent DFMA chains per
// thread, one persistent wave of CTAs per SM, CUDA-event timing after warm-up.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CHAINS 8
__global__ void __launch_bounds__(256) dfma_loop(double* out, int iters, double a, double b) {
  double x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-9 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
#pragma unroll
      for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 1234.5) out[0] = s;  // never true; keeps the loop alive
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("{\"device\": \"%s\", \"sms\": %d, \"clock_khz_attr\": %d, \"cc\": \"%d.%d\"",
         p.name, p.multiProcessorCount, clk_khz, p.major, p.minor);
  double* out;
  cudaMalloc(&out, 8);
  const int iters = 20000;
  int blocks_per_sm = 4;
  int blocks = p.multiProcessorCount * blocks_per_sm;
  for (int w = 0; w < 3; ++w) dfma_loop<<<blocks, 256>>>(out, iters / 10, 0.999999, 1e-7);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    dfma_loop<<<blocks, 256>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  double flops = 2.0 * (double)blocks * 256 * iters * 16 * CHAINS;
  printf(", \"dfma_tflops\": %.3f, \"ms\": %.3f", flops / (best * 1e-3) / 1e12, best);
  printf(", \"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
