// bipb_sym.cuh — symmetric-pair matvec kernel (DESIGN.md §6 "symmetric kernel").
//
// Same product as pair_kernel<MATVEC> (Eqs. (12)-(13); kernels Eq. (10)), but each
// UNORDERED pair {i, j} is evaluated once: r, 1/r, exp(-kappa r), p1 - 1 and the kernel
// factors are shared by the two ordered pairs (i <- j) and (j <- i) (K1 and K4 are symmetric
// in (x, nu_x) <-> (y, nu_y), K2/K3 exchange roles under d -> -d).
//
// Work decomposition: the N elements are cut into nb blocks of B = TPB*T rows. Block pairs
// follow a circulant schedule (block I meets blocks I+o mod nb, o = 0..H(I)) so every
// unordered block pair is covered exactly once and every I has the same amount of work.
// A CTA owns one I-block (targets in registers: T per thread) and a run of W offsets;
// the J-blocks' records stream through a TMA-fed shared-memory ring as in pair_kernel.
// Forward sums (into i) stay in registers for the whole run -> Fwd[I][run][B] partials;
// reverse sums (into j) are accumulated by a rotating per-source register accumulator that
// travels around the warp with its source (32 steps per 32-source group; one 4-double
// shuffle per step, no add tree), then summed over the warps (fixed order) -> Rev[J][o][B].
// A reduce kernel adds the partials of every row in a fixed order: deterministic, no
// value atomics.  The diagonal block (o = 0) evaluates pairs i < j only.
#pragma once
#include "bipb_kernels.cuh"

namespace bipb {

#ifndef BIPB_SYM_PREFETCH
#define BIPB_SYM_PREFETCH 1
#endif
#ifndef BIPB_SYM_UNROLL
#define BIPB_SYM_UNROLL 1
#endif
constexpr int SYM_UNROLL = BIPB_SYM_UNROLL;
constexpr int SYM_REC = 8;  // fields per source: x,y,z (scaled), c = W u_dphi, a = W u_phi, nx,ny,nz (64 B)
// Global/shared layout is "tile-SoA": for every TILE-source tile, 8 contiguous field arrays
// of TILE doubles.  One TMA bulk copy moves a whole tile; lanes that read different sources
// (the rotation below) then hit consecutive 8-byte words: conflict-free LDS.64.
__host__ __device__ constexpr int64_t sym_idx(int64_t j, int f) { return (j / TILE) * (TILE * SYM_REC) + f * TILE + (j % TILE); }

struct SymArgs {
  const double* rec;  // tile-SoA [ceil(n/TILE)][8][TILE]
  int64_t n;          // elements
  int64_t nb;         // blocks of B rows
  int64_t B;          // rows per block (= TPB*T)
  int64_t runs;       // offset runs per I-block (grid.x = nb_local * runs)
  int64_t W;          // offsets per run
  int64_t I0;         // first I-block of this launch (rank sharding by I-blocks)
  int64_t hmax;       // max offsets per I (for Rev indexing)
  double eps, inveps;
  double sc1, sc2, sc3;
  double* fwd;        // [I1-I0][runs][2][B]    forward sums of tile run (I, run), rank-local I
  double* rev;        // [I1-I0][hmax+1][2][B]  reverse sums of tile (I, J = I+o), rank-local I
};

// number of offsets (including the diagonal o = 0) for block I in the circulant schedule
__host__ __device__ inline int64_t sym_noff(int64_t I, int64_t nb) {
  if (nb & 1) return (nb - 1) / 2 + 1;
  return nb / 2 - 1 + 1 + ((I < nb / 2) ? 1 : 0);
}

__device__ __forceinline__ void rec_load(const double* sb, int j, double4& a, double4& b) {
  a = make_double4(sb[j], sb[TILE + j], sb[2 * TILE + j], sb[3 * TILE + j]);              // x, y, z, c
  b = make_double4(sb[4 * TILE + j], sb[5 * TILE + j], sb[6 * TILE + j], sb[7 * TILE + j]);  // a, nx, ny, nz
}

struct SymTgt {
  double X, Y, Z, NX, NY, NZ, C, A;
};

struct Acc2 {
  double p0, p1;
};

// One unordered pair: target i (registers) and source j (smem record).
// Forward into f (row i), reverse into r (row j).  d = x_i - x_j (scaled by s = kappa),
// t = |d| = kappa r, c = W u_dphi, a' = s W u_phi (the record stores a' so that the four
// kernel sums of a row collapse into two accumulators of equal scale: p0 = K1 + K2 terms / s,
// p1 = K3 + K4 terms / s^2).  With A = a nu every normal-weighted product reduces to d.nu_i,
// d.nu_j and nu_i.nu_j:
//   i <- j:  p0 += rho(1-e) c_j + a'_j (d.nu_j) rho^3 (eps p1 - 1)
//            p1 += -(d.nu_i) rho^3 (1 - p1/eps) c_j + a'_j rho^3 Q
//   j <- i:  p0 += rho(1-e) c_i - a'_i (d.nu_i) rho^3 (eps p1 - 1)
//            p1 += (d.nu_j) rho^3 (1 - p1/eps) c_i + a'_i rho^3 Q
//   Q = (p1 - 1)(nu_i.nu_j - 3 (d.nu_i)(d.nu_j) rho^2) - e (d.nu_i)(d.nu_j)   (shared by both rows)
// kappa = 0 (s = 1): p0 = sum of the K2 geometry, p1 = sum of the K3 geometry; the constant
// factors (eps - 1), (1 - 1/eps) are applied per row.
template <bool SCREENED>
__device__ __forceinline__ void pair_sym(const SymTgt& ti, const double4 s0, const double4 s1, const PairConst& k,
                                         const double* __restrict__ tab, Acc2& f, Acc2& r) {
  const double dx = ti.X - s0.x, dy = ti.Y - s0.y, dz = ti.Z - s0.z;
  const double cj = s0.w, aj = s1.x;
  const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
  const double rho = rsqrt_fp64(r2);
  const double rho2 = rho * rho;
  const double rho3 = rho2 * rho;
  const double dni = fma(dx, ti.NX, fma(dy, ti.NY, dz * ti.NZ));  // d.nu_i
  const double dnj = fma(dx, s1.y, fma(dy, s1.z, dz * s1.w));     // d.nu_j
  if constexpr (SCREENED) {
    const double nij = fma(ti.NX, s1.y, fma(ti.NY, s1.z, ti.NZ * s1.w));  // nu_i.nu_j
    const double t = r2 * rho;
    const double e = exp_neg(t, tab);
    const double em1 = e - 1.0;
    const double p1m1 = fma(e, t, em1);                       // e (1 + t) - 1
    const double rem1 = rho * em1;                            // -rho (1 - e)
    const double r3f2 = rho3 * fma(k.eps, p1m1, k.epsm1);     // rho^3 (eps p1 - 1)
    const double r3f3 = rho3 * fma(-k.inveps, p1m1, k.omie);  // rho^3 (1 - p1/eps)
    const double dd = dni * dnj;
    const double r3q = rho3 * fma(p1m1, fma(dd * rho2, -3.0, nij), -(e * dd));
    f.p0 = fma(aj, dnj * r3f2, fma(-rem1, cj, f.p0));
    f.p1 = fma(aj, r3q, fma(-(dni * r3f3), cj, f.p1));
    r.p0 = fma(-ti.A, dni * r3f2, fma(-rem1, ti.C, r.p0));
    r.p1 = fma(ti.A, r3q, fma(dnj * r3f3, ti.C, r.p1));
  } else {
    f.p0 = fma(aj, dnj * rho3, f.p0);
    f.p1 = fma(dni * rho3, cj, f.p1);
    r.p0 = fma(-ti.A, dni * rho3, r.p0);
    r.p1 = fma(-(dnj * rho3), ti.C, r.p1);
  }
}

__device__ __forceinline__ double warp_allsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int TPB, int T, bool SCREENED, int MINB>
__global__ void __launch_bounds__(TPB, MINB) sym_kernel(const SymArgs a) {
  constexpr int NW = TPB / 32;
  constexpr int B = TPB * T;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ double s_tab[EXP_TAB];
  double* sbuf = reinterpret_cast<double*>(smem_raw);                           // [STAGES][TILE][10]
  double* rsum = sbuf + STAGES * TILE * SYM_REC;  // [NW][2][B] per-warp reverse sums of the current J-block
  uint64_t* full = reinterpret_cast<uint64_t*>(rsum + NW * 2 * B);
  for (int i = threadIdx.x; i < EXP_TAB; i += TPB) s_tab[i] = c_exp_tab[i];
  const PairConst kc{a.eps, a.inveps, a.eps - 1.0, 1.0 - a.inveps};
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  const int64_t I = a.I0 + blockIdx.x / a.runs;
  const int64_t run = blockIdx.x % a.runs;
  const int64_t noff = sym_noff(I, a.nb);
  const int64_t o0 = run * a.W;
  const int64_t o1 = (o0 + a.W < noff) ? o0 + a.W : noff;
  const int64_t i0 = I * B;
  const int64_t stages_per_block = B / TILE;

  // targets (registers); rows past n sit far away with c = A = 0 (exact zero reverse terms)
  SymTgt tg[T];
  int64_t gi[T];
  Acc2 fa[T];
#pragma unroll
  for (int k = 0; k < T; ++k) {
    const int64_t i = i0 + threadIdx.x + k * TPB;
    gi[k] = i;
    fa[k].p0 = fa[k].p1 = 0.0;
    if (i < a.n) {
      const double* p = a.rec + sym_idx(i, 0);
      tg[k] = SymTgt{p[0], p[TILE], p[2 * TILE], p[5 * TILE], p[6 * TILE], p[7 * TILE], p[3 * TILE], p[4 * TILE]};
    } else {
      tg[k] = SymTgt{1e6, 1e6, 1e6, 1.0, 0.0, 0.0, 0.0, 0.0};
    }
  }

  // the stage sequence: for o in [o0, o1): stages of block J = (I + o) mod nb
  const int64_t nstage = (o1 > o0) ? (o1 - o0) * stages_per_block : 0;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto stage_src = [&](int64_t q, int64_t& j0, int& cnt) {
    const int64_t o = o0 + q / stages_per_block;
    const int64_t J = (I + o) % a.nb;
    j0 = J * B + (q % stages_per_block) * TILE;
    const int64_t rem = a.n - j0;
    cnt = rem <= 0 ? 0 : (rem < TILE ? (int)rem : TILE);
  };
  auto issue = [&](int64_t q, int buf) {
    int64_t j0;
    int cnt;
    stage_src(q, j0, cnt);
    const uint32_t bytes = cnt > 0 ? static_cast<uint32_t>(TILE * SYM_REC * sizeof(double)) : 0u;  // whole tile
    if (bytes == 0) {
      // empty stage (ragged last block): arrive without a transfer
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[buf])) : "memory");
    } else {
      mbar_expect_tx(&full[buf], bytes);
      tma_bulk_g2s(sbuf + buf * TILE * SYM_REC, a.rec + (j0 / TILE) * (TILE * SYM_REC), bytes, &full[buf]);
    }
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES && s < nstage; ++s) issue(s, s);
  }

  for (int64_t q = 0; q < nstage; ++q) {
    const int buf = static_cast<int>(q % STAGES);
    mbar_wait(&full[buf], static_cast<uint32_t>((q / STAGES) & 1));
    const double* sb = sbuf + buf * TILE * SYM_REC;
    int64_t j0;
    int cnt;
    stage_src(q, j0, cnt);
    const int64_t o = o0 + q / stages_per_block;
    const int jl0 = static_cast<int>((q % stages_per_block) * TILE);  // offset of this stage in the J-block
    // Groups of 32 sources.  At step st lane l evaluates source (l + st) & 31 of the group
    // against its T targets; the reverse accumulator of that source travels with it
    // (handed from lane l+1 to lane l after every step), so after 32 steps lane l holds the
    // warp's complete reverse sum for source l: no shuffle-add reduction tree.
    for (int g0 = 0; g0 < cnt; g0 += 32) {
      const int gcnt = (cnt - g0 < 32) ? cnt - g0 : 32;
      Acc2 rv{0.0, 0.0};
      if (o != 0 && gcnt == 32) {
#if BIPB_SYM_PREFETCH
        // the next step's record is loaded while this step computes (software pipelining)
        double4 n0, n1;
        rec_load(sb, g0 + lane, n0, n1);
#pragma unroll 1
        for (int st = 0; st < 32; ++st) {
          const double4 s0 = n0, s1 = n1;
          rec_load(sb, g0 + ((lane + st + 1) & 31), n0, n1);  // wraps harmlessly at st = 31
#else
#pragma unroll(SYM_UNROLL)
        for (int st = 0; st < 32; ++st) {
          const int jq = g0 + ((lane + st) & 31);
          double4 s0, s1;
          rec_load(sb, jq, s0, s1);
#endif
#pragma unroll
          for (int k = 0; k < T; ++k) pair_sym<SCREENED>(tg[k], s0, s1, kc, s_tab, fa[k], rv);
          rv.p0 = __shfl_sync(0xffffffffu, rv.p0, (lane + 1) & 31);
          rv.p1 = __shfl_sync(0xffffffffu, rv.p1, (lane + 1) & 31);
        }
      } else {
        // diagonal block (pairs i < j only) or a partial group
#pragma unroll 1
        for (int st = 0; st < 32; ++st) {
          const int q32 = (lane + st) & 31;
          if (q32 < gcnt) {
            const int jq = g0 + q32;
            const int64_t gj = j0 + jq;
            double4 s0, s1;
            rec_load(sb, jq, s0, s1);
#pragma unroll
            for (int k = 0; k < T; ++k)
              if (o != 0 || gi[k] < gj) pair_sym<SCREENED>(tg[k], s0, s1, kc, s_tab, fa[k], rv);
          }
          rv.p0 = __shfl_sync(0xffffffffu, rv.p0, (lane + 1) & 31);
          rv.p1 = __shfl_sync(0xffffffffu, rv.p1, (lane + 1) & 31);
        }
      }
      if (lane < gcnt) {
        double* rs = rsum + (warp * 2) * B + jl0 + g0 + lane;
        rs[0] = rv.p0;
        rs[B] = rv.p1;
      }
    }
    __syncthreads();  // buffer `buf` consumed; rsum entries of this stage written
    if (threadIdx.x == 0 && q + STAGES < nstage) issue(q + STAGES, buf);
    if ((q + 1) % stages_per_block == 0) {
      // end of J-block: combine warps (fixed order), fold s powers, write Rev[J][o]
      const int64_t J = (I + o) % a.nb;
      double* rv0 = a.rev + (((I - a.I0) * (a.hmax + 1) + o) * 2) * B;  // stored at the tile's I (rank-local)
      double* rv1 = rv0 + B;
      for (int jl = threadIdx.x; jl < B; jl += TPB) {
        if (J * B + jl >= a.n) continue;
        double q0 = 0.0, q1 = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          q0 += rsum[(w * 2) * B + jl];
          q1 += rsum[(w * 2 + 1) * B + jl];
        }
        if constexpr (SCREENED) {
          rv0[jl] = a.sc1 * q0;
          rv1[jl] = a.sc2 * q1;
        } else {
          rv0[jl] = (a.eps - 1.0) * q0;
          rv1[jl] = -((1.0 - a.inveps) * q1);
        }
      }
      __syncthreads();  // rsum reused by the next J-block
    }
  }

  // forward partials of this run
  double* f0 = a.fwd + (((I - a.I0) * a.runs + run) * 2) * B;
  double* f1 = f0 + B;
#pragma unroll
  for (int k = 0; k < T; ++k) {
    const int l = threadIdx.x + k * TPB;
    if (SCREENED) {
      f0[l] = a.sc1 * fa[k].p0;
      f1[l] = a.sc2 * fa[k].p1;
    } else {
      f0[l] = (a.eps - 1.0) * fa[k].p0;
      f1[l] = -((1.0 - a.inveps) * fa[k].p1);
    }
  }
}

// records {x s, y s, z s, c = W u_dphi, a' = s W u_phi, nu}
__global__ void prescale_sym_kernel(const double* __restrict__ u, const double* __restrict__ w,
                                    const double* __restrict__ ex, const double* __restrict__ ey,
                                    const double* __restrict__ ez, const double* __restrict__ nx,
                                    const double* __restrict__ ny, const double* __restrict__ nz,
                                    double* __restrict__ rec, int64_t n, double s) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    double* r = rec + sym_idx(j, 0);
    r[0] = ex[j];
    r[TILE] = ey[j];
    r[2 * TILE] = ez[j];
    r[3 * TILE] = w[j] * u[n + j];
    r[4 * TILE] = s * (w[j] * u[j]);
    r[5 * TILE] = nx[j];
    r[6 * TILE] = ny[j];
    r[7 * TILE] = nz[j];
  }
}

// Row epilogue.  For global row i (block b, local l): forward runs of block b in run order,
// then reverse offsets o = 0..hmax of the tiles (I = b - o mod nb, J = b) that exist (o <= noff(I)-1)
// and whose I-block is in [I0, I1) (this rank's blocks).  out0/out1 get the partial sums for
// rows [r0, r1); with `final` the diagonal terms and 1/(4 pi) are applied (single GPU).
__global__ void reduce_sym_kernel(const double* __restrict__ fwd, const double* __restrict__ rev, int64_t n,
                                  int64_t nb, int64_t B, int64_t runs, int64_t hmax, int64_t I0, int64_t I1,
                                  const double* __restrict__ u, double d1, double d2, int final_,
                                  double* __restrict__ out0, double* __restrict__ out1) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = i / B, l = i % B;
    double s0 = 0.0, s1 = 0.0;
    if (b >= I0 && b < I1) {
      for (int64_t r = 0; r < runs; ++r) {
        const double* f = fwd + (((b - I0) * runs + r) * 2) * B;
        s0 += f[l];
        s1 += f[B + l];
      }
    }
    for (int64_t o = 0; o <= hmax; ++o) {
      const int64_t I = ((b - o) % nb + nb) % nb;
      if (o >= sym_noff(I, nb) || I < I0 || I >= I1) continue;
      const double* rv = rev + (((I - I0) * (hmax + 1) + o) * 2) * B;
      s0 += rv[l];
      s1 += rv[B + l];
    }
    if (final_) {
      out0[i] = d1 * u[i] - s0 / FOUR_PI;
      out1[i] = d2 * u[n + i] - s1 / FOUR_PI;
    } else {
      out0[i] = s0;
      out1[i] = s1;
    }
  }
}

// y = d u - P / (4 pi) after the cross-rank sum (P = [P0; P1] summed over ranks)
__global__ void finish_sym_kernel(const double* __restrict__ P, const double* __restrict__ u, int64_t n, double d1,
                                  double d2, double* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    y[i] = d1 * u[i] - P[i] / FOUR_PI;
    y[n + i] = d2 * u[n + i] - P[n + i] / FOUR_PI;
  }
}

}  // namespace bipb
