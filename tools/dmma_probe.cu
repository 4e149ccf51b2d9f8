// Does FP64 tensor-core work (DMMA, mma.sync m8n8k4 f64) run beside the FP64 vector pipe on
// B200, or on the same units?  (the pair dot products nu_i.nu_j, x_j.nu_i are
// 8x8x4 contractions; offloading them only pays if DMMA throughput adds to DFMA throughput.)
// Three kernels, same grid: DFMA chains only, DMMA chains only, and both interleaved in one
// warp (independent work).  If "both" takes ~max(dfma, dmma) time the units are separate; if it
// takes ~the sum, they share the pipe.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_probe tools/dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <int DF, int MM>
__global__ void probe(double* out, int iters, double a, double b) {
  double x[DF > 0 ? DF : 1];
  double acc[MM > 0 ? MM : 1][2];
#pragma unroll
  for (int c = 0; c < DF; ++c) x[c] = threadIdx.x * 1e-9 + c;
#pragma unroll
  for (int c = 0; c < MM; ++c) acc[c][0] = acc[c][1] = threadIdx.x * 1e-9 + c;
  const double a2 = a * 1.0000001;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
#pragma unroll
      for (int c = 0; c < MM; ++c) dmma(acc[c], (c & 1) ? a : a2, b);
#pragma unroll
      for (int c = 0; c < DF; ++c) x[c] = fma(x[c], (c & 1) ? a : a2, b);
#pragma unroll
      for (int c = 0; c < DF; ++c) x[c] = fma(x[c], (c & 1) ? a2 : a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < DF; ++c) s += x[c];
#pragma unroll
  for (int c = 0; c < MM; ++c) s += acc[c][0] + acc[c][1];
  if (s == 1234.5) out[0] = s;
}

template <int DF, int MM>
void run(const char* name, int threads, int bps, int sms, double* out) {
  const int iters = 2000;
  const int blocks = sms * bps;
  probe<DF, MM><<<blocks, threads>>>(out, iters / 10, 0.999999, 1e-7);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    probe<DF, MM><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double warps = (double)blocks * threads / 32;
  const double dfma_flops = warps * 32 * iters * 8 * 2 * DF * 2.0;
  const double dmma_flops = warps * iters * 8 * MM * (8 * 8 * 4 * 2.0);
  printf("{\"kernel\": \"%s\", \"dfma_chains\": %d, \"dmma_chains\": %d, \"threads\": %d, \"blocks_per_sm\": %d, "
         "\"ms\": %.3f, \"dfma_tflops\": %.3f, \"dmma_tflops\": %.3f, \"total_tflops\": %.3f}\n",
         name, DF, MM, threads, bps, best, dfma_flops / (best * 1e-3) / 1e12, dmma_flops / (best * 1e-3) / 1e12,
         (dfma_flops + dmma_flops) / (best * 1e-3) / 1e12);
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  printf("{\"device\": \"%s\", \"sms\": %d}\n", p.name, p.multiProcessorCount);
  double* out;
  cudaMalloc(&out, 8);
  const int S = p.multiProcessorCount;
  run<8, 0>("dfma", 256, 4, S, out);
  run<0, 4>("dmma", 256, 4, S, out);
  run<0, 8>("dmma", 256, 4, S, out);
  run<8, 4>("both", 256, 4, S, out);
  run<8, 2>("both", 256, 4, S, out);
  run<8, 1>("both", 256, 4, S, out);
  printf("{\"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
