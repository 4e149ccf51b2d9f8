// Accuracy of the device math routines the pair kernels use (bipb_kernels.cuh: rsqrt_fp64,
// exp_neg), against long double on the host, for whichever variant macros this binary is built
// with (DESIGN.md §6 "rsqrt", "exp").  Build, e.g.:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o tools/math_accuracy tools/math_accuracy.cu
//   nvcc ... -DBIPB_RSQ_INT=1 -DBIPB_EXP_F32K=1 -o tools/math_accuracy_int tools/math_accuracy.cu
#include <cmath>
#include <cstdio>
#include <vector>

#include "../paper_1301_5885_b200/csrc/bipb_kernels.cuh"

using namespace bipb;

__global__ void eval(const double* x, const double* t, double* rs, double* ex, int n) {
  __shared__ double s_tab[EXP_TAB];
  for (int i = threadIdx.x; i < EXP_TAB; i += blockDim.x) s_tab[i] = g_exp_tab[i];
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  rs[i] = rsqrt_fp64(x[i]);
  ex[i] = exp_neg(t[i], s_tab);
}

static double ulp_err(double got, long double ref) {
  const double r = (double)ref;
  const double u = std::nextafter(std::fabs(r), INFINITY) - std::fabs(r);
  return (double)(fabsl((long double)got - ref) / u);
}

int main() {
  const int n = 1 << 22;
  std::vector<double> tab(EXP_TAB);
  for (int j = 0; j < EXP_TAB; ++j) tab[j] = (double)exp2l(-(long double)j / EXP_TAB);
  cudaMemcpyToSymbol(g_exp_tab, tab.data(), sizeof(double) * EXP_TAB);
  double *x, *t, *rs, *ex;
  cudaMallocManaged(&x, n * 8);
  cudaMallocManaged(&t, n * 8);
  cudaMallocManaged(&rs, n * 8);
  cudaMallocManaged(&ex, n * 8);
  unsigned long long s = 88172645463325252ull;
  auto rnd = [&]() {
    s ^= s << 13;
    s ^= s >> 7;
    s ^= s << 17;
    return (s >> 11) * (1.0 / 9007199254740992.0);
  };
  // x = r^2 in [1e-10, 1e4] (log-uniform); t in three ranges: [0, 0.2), [0.2, 10), [10, 690)
  for (int i = 0; i < n; ++i) {
    x[i] = std::pow(10.0, -10.0 + 14.0 * rnd());
    const int band = i % 3;
    t[i] = band == 0 ? 0.2 * rnd() : (band == 1 ? 0.2 + 9.8 * rnd() : 10.0 + 680.0 * rnd());
  }
  eval<<<(n + 255) / 256, 256>>>(x, t, rs, ex, n);
  cudaDeviceSynchronize();
  double mr = 0, me[3] = {0, 0, 0}, mrel_e = 0;
  for (int i = 0; i < n; ++i) {
    mr = std::fmax(mr, ulp_err(rs[i], 1.0L / sqrtl((long double)x[i])));
    const long double er = expl(-(long double)t[i]);
    const int band = i % 3;
    if (band < 2) me[band] = std::fmax(me[band], ulp_err(ex[i], er));
    else me[2] = std::fmax(me[2], (double)fabsl((long double)ex[i] - er));  // absolute: values ~1e-5..1e-300
    if (band < 2) mrel_e = std::fmax(mrel_e, (double)fabsl(((long double)ex[i] - er) / er));
  }
  printf("{\"rsq_int\": %d, \"exp_f32k\": %d, \"rsqrt_max_ulp\": %.3f, \"exp_max_ulp_t_lt_0.2\": %.3f, "
         "\"exp_max_ulp_t_0.2_10\": %.3f, \"exp_max_abs_t_10_690\": %.3e, \"exp_max_rel_t_lt_10\": %.3e, \"err\": \"%s\"}\n",
         BIPB_RSQ_INT, BIPB_EXP_F32K, mr, me[0], me[1], me[2], mrel_e, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
