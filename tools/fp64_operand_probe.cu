// DFMA throughput vs how many of its three 64-bit source operands change from one instruction to
// the next (register-file read bandwidth / operand reuse).  tools/fp64_peak.cu alternates two
// constants per operand and reaches 80-90% of the 64 DFMA/clk/SM rate; tools/dmma_probe.cu keeps
// the addend fixed and reaches 98%.  This probe separates the cases.
//   OPS = 0: fma(x_c, a, b)        a, b the same registers for every chain
//   OPS = 1: fma(x_c, a_c, b)      multiplier differs per chain
//   OPS = 2: fma(x_c, a_c, b_c)    multiplier and addend differ per chain
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_operand_probe tools/fp64_operand_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CH, int OPS>
__global__ void probe(double* out, int iters, double a0, double b0) {
  double x[CH], a[CH], b[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    x[c] = threadIdx.x * 1e-9 + c;
    a[c] = a0 * (1.0 + c * 1e-9);
    b[c] = b0 * (1.0 - c * 1e-9);
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        if (OPS == 0) x[c] = fma(x[c], a0, b0);
        if (OPS == 1) x[c] = fma(x[c], a[c], b0);
        if (OPS == 2) x[c] = fma(x[c], a[c], b[c]);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 1234.5) out[0] = s;
}

template <int CH, int OPS>
void run(int threads, int bps, int sms, double* out) {
  const int iters = 2000;
  const int blocks = sms * bps;
  probe<CH, OPS><<<blocks, threads>>>(out, iters / 10, 0.999999, 1e-7);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    probe<CH, OPS><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double inst = (double)blocks * threads * iters * 16 * CH;
  printf("{\"ops_varying\": %d, \"chains\": %d, \"threads\": %d, \"blocks_per_sm\": %d, \"tflops\": %.3f, "
         "\"dfma_per_clk_per_sm_at_1965\": %.2f}\n",
         OPS, CH, threads, bps, 2 * inst / (best * 1e-3) / 1e12, inst / (best * 1e-3) / (1.965e9 * sms));
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  printf("{\"device\": \"%s\", \"sms\": %d}\n", p.name, p.multiProcessorCount);
  double* out;
  cudaMalloc(&out, 8);
  const int S = p.multiProcessorCount;
  run<8, 0>(256, 4, S, out);
  run<8, 1>(256, 4, S, out);
  run<8, 2>(256, 4, S, out);
  run<16, 0>(128, 2, S, out);
  run<16, 1>(128, 2, S, out);
  run<16, 2>(128, 2, S, out);
  printf("{\"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
