// FP64 throughput microbenchmark for the roofline denominator.
// Measures DFMA / DMUL / DADD warp-instruction throughput with many independent chains per
// thread, several occupancies, CUDA-event timing after warm-up.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS, int OP>
__global__ void fp64_loop(double* out, int iters, double a, double b) {
  double x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-9 + c;
  double a2 = a * 1.0000001, b2 = b * 0.999;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
#pragma unroll
      for (int c = 0; c < CHAINS; ++c) {
        if (OP == 0) x[c] = fma(x[c], (c & 1) ? a : a2, (c & 2) ? b : b2);
        if (OP == 1) x[c] = x[c] * ((c & 1) ? a : a2);
        if (OP == 2) x[c] = x[c] + ((c & 1) ? b : b2);
        // operand patterns of the DFMA stream: OP 0 reads four distinct source registers across the
        // chains, OP 3 two multiplicands and one addend (tools/dmma_probe.cu's pattern), OP 4 one
        // of each -- register-bank conflicts of the 3-operand DFMA separate them (r02 reconciliation)
        if (OP == 3) x[c] = fma(x[c], (c & 1) ? a : a2, b);
        if (OP == 4) x[c] = fma(x[c], a, b);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 1234.5) out[0] = s;
}

template <int CHAINS, int OP>
void run(const char* name, int threads, int blocks_per_sm, int sms, double* out) {
  const int iters = 4000;
  int blocks = sms * blocks_per_sm;
  fp64_loop<CHAINS, OP><<<blocks, threads>>>(out, iters / 10, 0.999999, 1e-7);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    fp64_loop<CHAINS, OP><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  double inst = (double)blocks * threads * iters * 16 * CHAINS;
  double flops = inst * ((OP == 0 || OP >= 3) ? 2.0 : 1.0);
  printf("{\"op\": \"%s\", \"chains\": %d, \"threads\": %d, \"blocks_per_sm\": %d, \"ginst_per_s\": %.1f, "
         "\"tflops\": %.3f, \"inst_per_clk_per_sm_at_1965\": %.2f}\n",
         name, CHAINS, threads, blocks_per_sm, inst / (best * 1e-3) / 1e9, flops / (best * 1e-3) / 1e12,
         inst / (best * 1e-3) / (1.965e9 * sms));
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  printf("{\"device\": \"%s\", \"sms\": %d}\n", p.name, p.multiProcessorCount);
  double* out;
  cudaMalloc(&out, 8);
  const int S = p.multiProcessorCount;
  run<8, 0>("dfma", 256, 4, S, out);
  run<16, 0>("dfma", 256, 4, S, out);
  run<8, 0>("dfma", 256, 8, S, out);
  run<4, 0>("dfma", 128, 16, S, out);
  run<16, 0>("dfma", 128, 2, S, out);
  run<16, 0>("dfma", 128, 4, S, out);
  run<8, 3>("dfma_2src", 256, 4, S, out);
  run<16, 3>("dfma_2src", 256, 4, S, out);
  run<16, 3>("dfma_2src", 128, 4, S, out);
  run<8, 4>("dfma_1src", 256, 4, S, out);
  run<16, 4>("dfma_1src", 256, 4, S, out);
  run<8, 1>("dmul", 256, 4, S, out);
  run<8, 2>("dadd", 256, 4, S, out);
  printf("{\"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
