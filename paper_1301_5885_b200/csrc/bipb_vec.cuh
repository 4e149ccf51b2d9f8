// bipb_vec.cuh — O(N) kernels around the pair kernels: operand prescale (Eqs. (12)-(13)
// weights W_j), deterministic chunk reductions / row epilogues, and the device-side
// GMRES(m) vector work (MGS Arnoldi, Givens, back substitution).
// Every reduction has a fixed order (fixed grid, fixed tree, no atomics on values), so
// results are bitwise reproducible and identical on every rank.
#pragma once
#include <cstdint>
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "bipb_kernels.cuh"

namespace bipb {

constexpr int RED_BLOCKS = 296;  // 2 x 148 SMs
constexpr int RED_THREADS = 256;
constexpr double FOUR_PI = 12.566370614359172;
constexpr double C_E = 332.0716;  // kcal A / (mol e_c^2), reading R3

// a_j = W_j u_j, c_j = W_j u_{j+N}, A_j = a_j nu_j -> record {x,y,z,c,Ax,Ay,Az,0} (positions fixed)
__global__ void prescale_kernel(const double* __restrict__ u, const double* __restrict__ w,
                                const double* __restrict__ nx, const double* __restrict__ ny,
                                const double* __restrict__ nz, double* __restrict__ rec, int64_t n) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const double a = w[j] * u[j];
    const double c = w[j] * u[n + j];
    double4* r = reinterpret_cast<double4*>(rec + 8 * j);
    const double4 head = r[0];
    r[0] = make_double4(head.x, head.y, head.z, c);
    r[1] = make_double4(a * nx[j], a * ny[j], a * nz[j], 0.0);
  }
}

// Sum chunk partials in chunk order.  MATVEC: y_i = d1 u_i - P0/(4 pi), y_{i+N} = d2 u_{i+N} - P1/(4 pi)
// written to out0[l], out1[l] (out0 = y + r0, out1 = y + N + r0, or the all-gather stage).
__global__ void reduce_matvec_kernel(const double* __restrict__ part, int64_t nchunk, int64_t ntgt,
                                     const double* __restrict__ u0, const double* __restrict__ u1, double d1,
                                     double d2, double* __restrict__ out0, double* __restrict__ out1) {
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < ntgt; l += (int64_t)gridDim.x * blockDim.x) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll RED_UNROLL
    for (int64_t c = 0; c < nchunk; ++c) {
      s0 += part[(2 * c) * ntgt + l];
      s1 += part[(2 * c + 1) * ntgt + l];
    }
    out0[l] = d1 * u0[l] - s0 / FOUR_PI;
    out1[l] = d2 * u1[l] - s1 / FOUR_PI;
  }
}

// SOURCE: b_i = P0 / (4 pi eps1), b_{i+N} = P1 / (4 pi eps1)
__global__ void reduce_source_kernel(const double* __restrict__ part, int64_t nchunk, int64_t ntgt, double scale,
                                     double* __restrict__ out0, double* __restrict__ out1) {
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < ntgt; l += (int64_t)gridDim.x * blockDim.x) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll RED_UNROLL
    for (int64_t c = 0; c < nchunk; ++c) {
      s0 += part[(2 * c) * ntgt + l];
      s1 += part[(2 * c + 1) * ntgt + l];
    }
    out0[l] = s0 * scale;
    out1[l] = s1 * scale;
  }
}

// ENERGY: phi_tilde_k = 4 pi phi_reac(x_k) = sum_c P0
__global__ void reduce_energy_kernel(const double* __restrict__ part, int64_t nchunk, int64_t ntgt,
                                     double* __restrict__ out) {
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < ntgt; l += (int64_t)gridDim.x * blockDim.x) {
    double s0 = 0.0;
#pragma unroll RED_UNROLL
    for (int64_t c = 0; c < nchunk; ++c) s0 += part[(2 * c) * ntgt + l];
    out[l] = s0;
  }
}

// all-gather unpack: gathered [world][2*Np] -> y[r0_p + l], y[N + r0_p + l]
__global__ void unpack_kernel(const double* __restrict__ g, int64_t n, int64_t np, int world, double* __restrict__ y) {
  const int64_t total = (int64_t)world * np;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = q / np, l = q % np;
    const int64_t i = p * np + l;
    if (i < n) {
      y[i] = g[p * 2 * np + l];
      y[n + i] = g[p * 2 * np + np + l];
    }
  }
}
__global__ void unpack1_kernel(const double* __restrict__ g, int64_t n, int64_t np, int world, double* __restrict__ y) {
  const int64_t total = (int64_t)world * np;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    if (q < n) y[q] = g[q];
  }
}

// ------------------------------------------------------------ fixed-order reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double sh[RED_THREADS / 32];
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
  if (w == 0) {
    r = (l < RED_THREADS / 32) ? sh[l] : 0.0;
    r = warp_sum(r);
  }
  return r;  // valid in thread 0
}
// Last block (ticket) sums the per-block partials in index order -> *out; resets the counter.
__device__ __forceinline__ void finish_sum(double v, double* partials, unsigned* counter, double* out, double scale) {
  __shared__ bool last;
  const double bs = block_sum(v);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = bs;
    __threadfence();
    const unsigned ticket = atomicAdd(counter, 1u);
    last = (ticket == gridDim.x - 1);
  }
  __syncthreads();
  if (last && threadIdx.x < 32) {
    __threadfence();
    double s = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) s += __ldcg(partials + b);
    s = warp_sum(s);
    if (threadIdx.x == 0) {
      *out = s * scale;
      *counter = 0u;
    }
  }
}

// If alpha != nullptr: w -= (*alpha) * v (MGS step).  Then *out = sum(w .* z) (z may alias w).
__global__ void __launch_bounds__(RED_THREADS) axpy_dot_kernel(double* __restrict__ w, const double* __restrict__ v,
                                                               const double* alpha, const double* z, int64_t m,
                                                               double* partials, unsigned* counter, double* out) {
  double acc = 0.0;
  const double al = (alpha != nullptr) ? *alpha : 0.0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x) {
    double wt = w[t];
    if (alpha != nullptr) {
      wt = wt - al * v[t];
      w[t] = wt;
    }
    acc = fma(wt, z[t], acc);
  }
  finish_sum(acc, partials, counter, out, 1.0);
}

// *out = sum(a .* b) * scale
__global__ void __launch_bounds__(RED_THREADS) dot_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                                          int64_t m, double scale, double* partials,
                                                          unsigned* counter, double* out) {
  double acc = 0.0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x)
    acc = fma(a[t], b[t], acc);
  finish_sum(acc, partials, counter, out, scale);
}

// E_sol = 1/2 C_E sum_k Q_k phi_tilde_k  (Eq. (14), R3); charges [nc][4] with Q at [4k+3]
__global__ void __launch_bounds__(RED_THREADS) energy_sum_kernel(const double* __restrict__ q4,
                                                                 const double* __restrict__ phit, int64_t nc,
                                                                 double* partials, unsigned* counter, double* out) {
  double acc = 0.0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nc; k += (int64_t)gridDim.x * blockDim.x)
    acc = fma(q4[4 * k + 3], phit[k], acc);
  finish_sum(acc, partials, counter, out, 0.5 * C_E);
}

__global__ void sqrt_kernel(const double* in, double* out) { *out = sqrt(*in); }

// dst = src / (*den)
__global__ void scale_div_kernel(double* __restrict__ dst, const double* __restrict__ src, const double* den,
                                 int64_t m) {
  const double d = *den;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x)
    dst[t] = src[t] / d;
}
// r = b - ax
__global__ void residual_kernel(double* __restrict__ r, const double* __restrict__ b, const double* __restrict__ ax,
                                int64_t m) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x)
    r[t] = b[t] - ax[t];
}
__global__ void phi_scale_kernel(const double* __restrict__ phit, double* __restrict__ phi, int64_t nc) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nc; k += (int64_t)gridDim.x * blockDim.x)
    phi[k] = phit[k] / FOUR_PI;
}

// g = (beta, 0, ..., 0)
__global__ void init_g_kernel(double* g, const double* beta, int m) {
  for (int i = threadIdx.x; i <= m; i += blockDim.x) g[i] = (i == 0) ? *beta : 0.0;
}

// One Givens step on column k of H ((m+1) x m row-major), SURVEY.md §8(c) O4.
// hk1sq = ||w||^2 after orthogonalisation. info[0] = |g_{k+1}| / beta_b, info[1] = h_{k+1,k}.
__device__ __forceinline__ void givens_step(double* H, double* cs, double* sn, double* g, double hk1sq, double* hk1,
                                            int k, int m, double beta_b, double* info) {
  const double h = sqrt(hk1sq);
  H[(k + 1) * m + k] = h;
  for (int i = 0; i < k; ++i) {
    const double a = H[i * m + k], c = H[(i + 1) * m + k];
    H[i * m + k] = cs[i] * a + sn[i] * c;
    H[(i + 1) * m + k] = -sn[i] * a + cs[i] * c;
  }
  const double a = H[k * m + k], c = H[(k + 1) * m + k];
  const double delta = hypot(a, c);
  cs[k] = a / delta;
  sn[k] = c / delta;
  H[k * m + k] = delta;
  H[(k + 1) * m + k] = 0.0;
  g[k + 1] = -sn[k] * g[k];
  g[k] = cs[k] * g[k];
  *hk1 = h;
  info[0] = fabs(g[k + 1]) / beta_b;
  info[1] = h;
}
// Device-side Arnoldi cycle (BIPB_GRAPHS=2, bipb.cu run_cycle): after step k of a cycle graph,
// record the step's (|g_{k+1}|/beta_b, h_{k+1,k}) = S[6], S[7] in cyc[8 + 2k ..] and, when the host
// loop of bipb_gmres_solve would leave the cycle here, set the next step's IF condition to 0 (else
// to 1) so the remaining steps do not run.  The tests are the host loop's, on the same doubles:
// happy breakdown h_{k+1,k} <= 1e-14 beta_b, |g|/beta_b <= tol, its >= max_iters, NaN (exact sums).
// cyc[0..4] = beta_b, tol, iterations before the cycle, max_iters, exact-sums flag.
__global__ void cycle_check_kernel(const double* __restrict__ S, double* __restrict__ cyc, int k,
                                   cudaGraphConditionalHandle next, int has_next) {
  const double rel = S[6], hk1 = S[7];
  cyc[8 + 2 * k] = rel;
  cyc[9 + 2 * k] = hk1;
  const bool stop = (hk1 <= 1e-14 * cyc[0]) || (rel <= cyc[1]) || (cyc[2] + (k + 1) >= cyc[3]) ||
                    (cyc[4] != 0.0 && !(rel == rel));
  if (has_next) cudaGraphSetConditional(next, stop ? 0u : 1u);
}

__global__ void givens_kernel(double* H, double* cs, double* sn, double* g, const double* hk1sq, double* hk1,
                              int k, int m, const double* beta_b_ptr, double* info) {
  givens_step(H, cs, sn, g, *hk1sq, hk1, k, m, *beta_b_ptr, info);
}

// ------------------------------------------------ fused Arnoldi tail on one thread-block cluster
// For short Krylov vectors (2N <= ARN_CLUSTER * ARN_THREADS * E) the k + 2 dependent reductions
// of one MGS sweep (h_0 = <w, v_0>; for i = 0..k: w -= h_i v_i,
// h_{i+1} = <w, v_{i+1}> (i < k) or ||w||^2 (i = k)), the Givens step and w /= h_{k+1,k} run in ONE
// kernel on ONE cluster instead of k + 4 launches.  w and the current v_i stay in registers.  A
// reduction: warp partials (fixed shuffle tree) -> CTA partial in shared memory -> one cluster
// barrier -> warp 0 of every CTA reads the 8 CTA partials through distributed shared memory and
// sums them in rank order: bitwise the same total in every CTA, deterministic, no atomics.  The
// CTA-partial slot alternates by step parity, so one cluster barrier per reduction suffices.
// (Measured at C1: letting every warp read all 8 x 32 warp partials instead of the second
// __syncthreads is 15% slower; prefetching v_{i+1} one reduction ahead gains nothing.)  Same
// arithmetic per element as axpy_dot_kernel / scale_div_kernel; only the dots' summation order differs.
// The residual record is also stored to `info_host` (pinned, device-mapped) when non-null.
constexpr int ARN_THREADS = 1024;
constexpr int ARN_CLUSTER = 8;  // portable cluster size
template <int E>
__global__ void __cluster_dims__(ARN_CLUSTER, 1, 1) __launch_bounds__(ARN_THREADS, 1)
    arnoldi_fused_kernel(double* __restrict__ V, int64_t m2, int k, int m, double* H, double* cs, double* sn,
                         double* g, double* S, double* info_host) {
  namespace cg = cooperative_groups;
  static_assert(ARN_THREADS / 32 == 32, "one warp partial per lane");
  cg::cluster_group cl = cg::this_cluster();
  const int rank = static_cast<int>(cl.block_rank());
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ double ws[ARN_THREADS / 32];
  __shared__ double cpart[2];
  __shared__ double tot;
  auto reduce = [&](double acc, int step) -> double {
    acc = warp_sum(acc);
    if (lane == 0) ws[warp] = acc;
    __syncthreads();
    if (warp == 0) {
      const double r = warp_sum(ws[lane]);
      if (lane == 0) cpart[step & 1] = r;
    }
    cl.sync();  // every CTA's partial of this step is visible cluster-wide
    if (warp == 0) {
      double r = (lane < ARN_CLUSTER) ? *cl.map_shared_rank(&cpart[step & 1], lane) : 0.0;
      r = warp_sum(r);
      if (lane == 0) tot = r;
    }
    __syncthreads();
    return tot;
  };
  auto idx = [&](int e) { return ((int64_t)e * ARN_CLUSTER + rank) * ARN_THREADS + threadIdx.x; };
  double* wg = V + (int64_t)(k + 1) * m2;
  double w[E], z[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int64_t t = idx(e);
    w[e] = (t < m2) ? wg[t] : 0.0;
    z[e] = (t < m2) ? V[t] : 0.0;  // v_0
  }
  double acc = 0.0;
#pragma unroll
  for (int e = 0; e < E; ++e) acc = fma(w[e], z[e], acc);
  double h = reduce(acc, 0);
  const bool lead = (rank == 0 && threadIdx.x == 0);
  if (lead) H[0 * m + k] = h;
  for (int i = 0; i <= k; ++i) {
    acc = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      w[e] = w[e] - h * z[e];  // z = v_i
      if (i < k) {
        const int64_t t = idx(e);
        z[e] = (t < m2) ? V[(int64_t)(i + 1) * m2 + t] : 0.0;  // v_{i+1}
        acc = fma(w[e], z[e], acc);
      } else {
        acc = fma(w[e], w[e], acc);
      }
    }
    h = reduce(acc, i + 1);
    if (lead && i < k) H[(i + 1) * m + k] = h;
  }
  // h = ||w||^2: Givens on column k (one thread), then every thread normalises its elements
  if (lead) {
    givens_step(H, cs, sn, g, h, S + 3, k, m, S[0], S + 6);
    if (info_host) {
      info_host[0] = S[6];
      info_host[1] = S[7];
    }
  }
  const double hn = sqrt(h);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int64_t t = idx(e);
    if (t < m2) wg[t] = w[e] / hn;
  }
  cl.sync();  // no CTA exits while a peer may still read its shared memory
}

// ---------------------------------------- right preconditioning by the jump-term diagonal (opt-in)
// M = diag(1/2 (1 + eps) I_N, 1/2 (1 + 1/eps) I_N), s1 = M^-1 on the phi rows, s2 on the dphi rows
// (bipb_set_precond; Saad Alg. 9.5: z_k = M^-1 v_k before the product, x += M^-1 (V y) at the end
// of a cycle).  dst = M^-1 src
__global__ void jacobi_scale_kernel(double* __restrict__ dst, const double* __restrict__ src, int64_t n, double s1,
                                    double s2) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < 2 * n; t += (int64_t)gridDim.x * blockDim.x)
    dst[t] = ((t < n) ? s1 : s2) * src[t];
}
// x += M^-1 (V[0:k] y)  (per element: the combination j ascending, then the scaling, as the oracle)
__global__ void update_x_prec_kernel(double* __restrict__ x, const double* __restrict__ V,
                                     const double* __restrict__ y, int k, int64_t n, double s1, double s2) {
  const int64_t m = 2 * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < k; ++j) s = s + y[j] * V[(int64_t)j * m + t];
    x[t] = x[t] + ((t < n) ? s1 : s2) * s;
  }
}

// back substitution H[0:k,0:k] y = g[0:k]
__global__ void backsolve_kernel(const double* H, const double* g, double* y, int k, int m) {
  for (int i = k - 1; i >= 0; --i) {
    double s = g[i];
    for (int j = i + 1; j < k; ++j) s -= H[i * m + j] * y[j];
    y[i] = s / H[i * m + i];
  }
}

// x += V[0:k] y  (per element, j ascending, as the oracle)
__global__ void update_x_kernel(double* __restrict__ x, const double* __restrict__ V, const double* __restrict__ y,
                                int k, int64_t m) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x) {
    double xt = x[t];
    for (int j = 0; j < k; ++j) xt = xt + y[j] * V[(int64_t)j * m + t];
    x[t] = xt;
  }
}

// min over (element, charge) pairs of the squared distance (validation, reading R11)
__global__ void min_dist_kernel(const double* __restrict__ ex, const double* __restrict__ ey,
                                const double* __restrict__ ez, int64_t n, const double* __restrict__ q4, int64_t nc,
                                double lim2, int* flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double x = ex[i], y = ey[i], z = ez[i];
    double m = 1e300;
    for (int64_t k = 0; k < nc; ++k) {
      const double dx = x - q4[4 * k], dy = y - q4[4 * k + 1], dz = z - q4[4 * k + 2];
      m = fmin(m, fma(dx, dx, fma(dy, dy, dz * dz)));
    }
    if (m < lim2) atomicExch(flag, 1);
  }
}

}  // namespace bipb
