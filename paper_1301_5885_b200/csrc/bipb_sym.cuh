// bipb_sym.cuh — symmetric-pair matvec kernel (DESIGN.md §6 "symmetric kernel"), for R = 1, 2
// or 4 right-hand sides at once (multi-RHS).
//
// Same product as pair_kernel<MATVEC> (Eqs. (12)-(13); kernels Eq. (10)), but each
// UNORDERED pair {i, j} is evaluated once: r, 1/r, exp(-kappa r), p1 - 1 and the kernel
// factors are shared by the two ordered pairs (i <- j) and (j <- i) (K1 and K4 are symmetric
// in (x, nu_x) <-> (y, nu_y), K2/K3 exchange roles under d -> -d) and
// by all R operands u_1..u_R (only the 4 accumulate FMAs per direction are per operand).
//
// Work decomposition: the N elements are cut into nb blocks of B = TPB*T rows. Block pairs
// follow a circulant schedule (block I meets blocks I+o mod nb, o = 0..H(I)) so every
// unordered block pair is covered exactly once and every I has the same amount of work.
// A CTA owns one I-block (targets in registers: T per thread) and a run of W offsets;
// the J-blocks' records stream through a TMA-fed shared-memory ring.
// Forward sums (into i) stay in registers for the whole run -> Fwd[I][run] partials;
// reverse sums (into j) are accumulated by a rotating per-source register accumulator that
// travels around the warp with its source (32 steps per 32-source group; one shuffle per
// accumulator per step, no add tree), then summed over the warps (fixed order) -> Rev[I][o].
// Reduce kernels add the partials of every row in a fixed order: deterministic, no value
// atomics.  The diagonal block (o = 0) evaluates pairs i < j only.  Launches may cover the
// I-blocks in groups (bounded partial memory); groups are summed in order.
#pragma once
#include "bipb_kernels.cuh"
#include "bipb_p2p.cuh"
#include "bipb_exact.cuh"

namespace bipb {

#ifndef BIPB_SYM_PREFETCH
#define BIPB_SYM_PREFETCH 1
#endif
// unroll factor of the 32-step source rotation (tuning: > 1 lets the compiler overlap one step's
// reverse-accumulator chain + shuffles with the next step's independent work)
#ifndef BIPB_SYM_STUNROLL
#define BIPB_SYM_STUNROLL 1
#endif
#define BIPB_PRAGMA_(x) _Pragma(#x)
#define BIPB_UNROLL_(n) BIPB_PRAGMA_(unroll n)
// record prefetch of the 32-step rotation, per number of operands: 1 = load the next step's
// record while this one computes (register copy per step), 2 = ping-pong buffers (no copies, two
// records live), 0 = load at the top of each step (no copies, load latency exposed)
// (r02 session 4, profiles/r02/session4/tune_batch_C4.jsonl: ping-pong for R > 1 -- R = 4 320.4 ->
// 317.4 ms, R = 2 236.6 -> 235.1 per C4 product; R = 1 keeps 1: 191.1 vs 201.9 ms with 2, 198.1 with 0)
#ifndef BIPB_SYM_PREFETCH_MRHS
#define BIPB_SYM_PREFETCH_MRHS 2
#endif
__host__ __device__ constexpr int sym_prefetch(int R) { return R == 1 ? BIPB_SYM_PREFETCH : BIPB_SYM_PREFETCH_MRHS; }

// Record (tile-SoA): fields x, y, z (scaled by s), nx, ny, nz, then (c_r, a'_r) for r < R with
// c = W u_dphi and a' = s W u_phi.  For every TILE-source tile the F = 6 + 2R fields are
// contiguous arrays of TILE doubles: one TMA bulk copy moves a tile; lanes that read different
// sources (the rotation below) hit consecutive 8-byte words (conflict-free LDS.64).
template <int R>
struct SymLayout {
  static constexpr int F = 6 + 2 * R;
  // field order: R = 1 keeps {x, y, z, c, a', nx, ny, nz} (measured 2% faster register
  // allocation); R > 1 uses {x, y, z, nx, ny, nz, (c, a') x R}
  static constexpr int NX = (R == 1) ? 5 : 3;
  __host__ __device__ static constexpr int C(int r) { return (R == 1) ? 3 : 6 + 2 * r; }
  __host__ __device__ static constexpr int A(int r) { return (R == 1) ? 4 : 7 + 2 * r; }
};
// source rows per warp-combine of the reverse sums (see sym_kernel): the whole J-block for R = 1
// (one barrier per J-block), every stage for R > 1 -- or for R = 1 too with BIPB_SYM_RS_STAGE=1,
// which cuts the shared memory of a T = 5 CTA from ~82 KB to ~49 KB (3 CTAs per SM fit)
#ifndef BIPB_SYM_RS_STAGE
#define BIPB_SYM_RS_STAGE 0
#endif
__host__ __device__ constexpr int sym_rs_rows(int R, int B) { return (R == 1 && !BIPB_SYM_RS_STAGE) ? B : TILE; }
__host__ __device__ constexpr int64_t sym_idx(int64_t j, int f, int F) {
  return (j / TILE) * (TILE * F) + f * TILE + (j % TILE);
}

struct SymArgs {
  const double* rec;  // tile-SoA [ceil(n/TILE)][F][TILE]
  int64_t n;          // elements
  int64_t nb;         // blocks of B rows
  int64_t B;          // rows per block (= TPB*T)
  int64_t runs;       // offset runs per I-block (grid.x = nI * runs)
  int64_t W;          // offsets per run
  int64_t I0;         // first I-block of this launch
  int64_t hmax;       // max offsets per I (Rev indexing)
  double eps, inveps;
  double sc1, sc2;    // s, s^2
  double* fwd;        // [nI][runs][R][2][B]   forward sums of tile run (I, run), I - I0
  double* rev;        // [nI][hmax+1][R][2][B] reverse sums of tile (I, J = I+o), I - I0
  // exact sums (bipb_exact.cuh; R = 1 only): when xl != nullptr every partial is added to the
  // row limbs xl[3][2n] (+ overflow count) instead of being written to fwd / rev
  unsigned long long* xl;
  const int* xexp;    // largest exponent field of the operand weights (prescale_sym_kernel)
  int xbias;          // test hook: added to the shift S (forces the out-of-range fallback)
};

// number of offsets (including the diagonal o = 0) for block I in the circulant schedule
__host__ __device__ inline int64_t sym_noff(int64_t I, int64_t nb) {
  if (nb & 1) return (nb - 1) / 2 + 1;
  return nb / 2 - 1 + 1 + ((I < nb / 2) ? 1 : 0);
}

template <int R>
struct SymSrc {
  double x, y, z, nx, ny, nz, c[R], a[R];
};
template <int R>
__device__ __forceinline__ void rec_load(const double* sb, int j, SymSrc<R>& s) {
  using L = SymLayout<R>;
  s.x = sb[j];
  s.y = sb[TILE + j];
  s.z = sb[2 * TILE + j];
  s.nx = sb[L::NX * TILE + j];
  s.ny = sb[(L::NX + 1) * TILE + j];
  s.nz = sb[(L::NX + 2) * TILE + j];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    s.c[r] = sb[L::C(r) * TILE + j];
    s.a[r] = sb[L::A(r) * TILE + j];
  }
}

struct Acc2 {
  double p0, p1;
};

// One unordered pair: target i (registers) and source j (smem record).
// Forward into f[r] (row i), reverse into v[r] (row j).  d = x_i - x_j (scaled by s = kappa),
// t = |d| = kappa r, c = W u_dphi, a' = s W u_phi (the record stores a' so that the four kernel
// sums of a row collapse into two accumulators of equal scale: p0 = K1 + K2 terms / s,
// p1 = K3 + K4 terms / s^2).  With A = a nu every normal-weighted product reduces to d.nu_i,
// d.nu_j and nu_i.nu_j:
//   i <- j:  p0 += rho(1-e) c_j + a'_j (d.nu_j) rho^3 (eps p1 - 1)
//            p1 += -(d.nu_i) rho^3 (1 - p1/eps) c_j + a'_j rho^3 Q
//   j <- i:  p0 += rho(1-e) c_i - a'_i (d.nu_i) rho^3 (eps p1 - 1)
//            p1 += (d.nu_j) rho^3 (1 - p1/eps) c_i + a'_i rho^3 Q
//   Q = (p1 - 1)(nu_i.nu_j - 3 (d.nu_i)(d.nu_j) rho^2) - e (d.nu_i)(d.nu_j)   (shared by both rows)
// kappa = 0 (s = 1): p0 = sum of the K2 geometry, p1 = sum of the K3 geometry; the constant
// factors (eps - 1), (1 - 1/eps) are applied per row.
template <bool SCREENED, int R>
__device__ __forceinline__ void pair_sym(const SymSrc<R>& ti, const SymSrc<R>& sj, const PairConst& k,
                                         const double* __restrict__ tab, Acc2* f, Acc2* v) {
  const double dx = ti.x - sj.x, dy = ti.y - sj.y, dz = ti.z - sj.z;
  const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
  const double rho = rsqrt_fp64(r2);
  const double rho2 = rho * rho;
  const double rho3 = rho2 * rho;
  const double dni = fma(dx, ti.nx, fma(dy, ti.ny, dz * ti.nz));  // d.nu_i
  const double dnj = fma(dx, sj.nx, fma(dy, sj.ny, dz * sj.nz));  // d.nu_j
  if constexpr (SCREENED) {
    const double nij = fma(ti.nx, sj.nx, fma(ti.ny, sj.ny, ti.nz * sj.nz));  // nu_i.nu_j
    const double t = r2 * rho;
    const double e = exp_neg(t, tab);
    const double em1 = e - 1.0;
    const double p1m1 = fma(e, t, em1);                       // e (1 + t) - 1
    const double rem1 = rho * em1;                            // -rho (1 - e)
    const double r3f2 = rho3 * fma(k.eps, p1m1, k.epsm1);     // rho^3 (eps p1 - 1)
    const double r3f3 = rho3 * fma(-k.inveps, p1m1, k.omie);  // rho^3 (1 - p1/eps)
    const double dd = dni * dnj;
    const double r3q = rho3 * fma(p1m1, fma(dd * rho2, -3.0, nij), -(e * dd));
    if constexpr (R == 1) {
      f[0].p0 = fma(sj.a[0], dnj * r3f2, fma(-rem1, sj.c[0], f[0].p0));
      f[0].p1 = fma(sj.a[0], r3q, fma(-(dni * r3f3), sj.c[0], f[0].p1));
      v[0].p0 = fma(-ti.a[0], dni * r3f2, fma(-rem1, ti.c[0], v[0].p0));
      v[0].p1 = fma(ti.a[0], r3q, fma(dnj * r3f3, ti.c[0], v[0].p1));
    } else {
      const double g2f = dnj * r3f2, g2r = dni * r3f2, g3f = dni * r3f3, g3r = dnj * r3f3;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        f[r].p0 = fma(sj.a[r], g2f, fma(-rem1, sj.c[r], f[r].p0));
        f[r].p1 = fma(sj.a[r], r3q, fma(-g3f, sj.c[r], f[r].p1));
        v[r].p0 = fma(-ti.a[r], g2r, fma(-rem1, ti.c[r], v[r].p0));
        v[r].p1 = fma(ti.a[r], r3q, fma(g3r, ti.c[r], v[r].p1));
      }
    }
  } else {
    const double g2f = dnj * rho3, g2r = dni * rho3;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      f[r].p0 = fma(sj.a[r], g2f, f[r].p0);
      f[r].p1 = fma(g2r, sj.c[r], f[r].p1);
      v[r].p0 = fma(-ti.a[r], g2r, v[r].p0);
      v[r].p1 = fma(-g2f, ti.c[r], v[r].p1);
    }
  }
}

// BIPB_SYM_MAXNREG (tuning probe only): a per-kernel register cap instead of the occupancy bound
#ifdef BIPB_SYM_MAXNREG
#define BIPB_SYM_BOUNDS(TPB, MINB) __maxnreg__(BIPB_SYM_MAXNREG)
#else
#define BIPB_SYM_BOUNDS(TPB, MINB) __launch_bounds__(TPB, MINB)
#endif
template <int TPB, int T, bool SCREENED, int MINB, int R, bool EXACT = false>
__global__ void BIPB_SYM_BOUNDS(TPB, MINB) sym_kernel(const SymArgs a) {
  static_assert(!EXACT || R == 1, "exact sums: single operand only");
  constexpr int NW = TPB / 32;
  constexpr int B = TPB * T;
  constexpr int F = SymLayout<R>::F;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ double s_tab[EXP_TAB];
  double* sbuf = reinterpret_cast<double*>(smem_raw);  // [STAGES][F][TILE]
  // per-warp reverse sums [NW][R][2][RS], combined over the warps every RS source rows: the whole
  // J-block for R = 1 (one barrier per J-block), every stage for R > 1 (NW*R*2*TILE doubles instead
  // of NW*R*2*B: R = 4 needs 32 KB instead of 64-98 KB, which keeps 2 CTAs per SM; measured R = 4
  // at C4 456 -> 329 ms per product, R = 1 per stage would cost 0.7%)
  constexpr int RS = sym_rs_rows(R, B);
  double* rsum = sbuf + STAGES * TILE * F;
  uint64_t* full = reinterpret_cast<uint64_t*>(rsum + NW * R * 2 * RS);
  for (int i = threadIdx.x; i < EXP_TAB; i += TPB) s_tab[i] = g_exp_tab[i];
  const PairConst kc{a.eps, a.inveps, a.eps - 1.0, 1.0 - a.inveps};
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  const int64_t Il = blockIdx.x / a.runs;  // I-block relative to this launch
  const int64_t I = a.I0 + Il;
  const int64_t run = blockIdx.x % a.runs;
  const int64_t noff = sym_noff(I, a.nb);
  // the I-block's noff offsets split evenly over its runs (sizes differ by at most one, no tiny
  // last run: the CTAs have nearly equal work, which shortens the launch's tail)
  const int64_t o0 = run * noff / a.runs;
  const int64_t o1 = (run + 1) * noff / a.runs;
  const int64_t i0 = I * B;
  constexpr int64_t stages_per_block = B / TILE;

  // targets (registers); rows past n sit far away with c = a' = 0 (exact zero reverse terms)
  SymSrc<R> tg[T];
  int64_t gi[T];
  Acc2 fa[T][R];
#pragma unroll
  for (int k = 0; k < T; ++k) {
    const int64_t i = i0 + threadIdx.x + k * TPB;
    gi[k] = i;
#pragma unroll
    for (int r = 0; r < R; ++r) fa[k][r].p0 = fa[k][r].p1 = 0.0;
    if (i < a.n) {
      const double* p = a.rec + sym_idx(i, 0, F);
      tg[k].x = p[0];
      tg[k].y = p[TILE];
      tg[k].z = p[2 * TILE];
      tg[k].nx = p[SymLayout<R>::NX * TILE];
      tg[k].ny = p[(SymLayout<R>::NX + 1) * TILE];
      tg[k].nz = p[(SymLayout<R>::NX + 2) * TILE];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        tg[k].c[r] = p[SymLayout<R>::C(r) * TILE];
        tg[k].a[r] = p[SymLayout<R>::A(r) * TILE];
      }
    } else {
      tg[k].x = tg[k].y = tg[k].z = 1e6;
      tg[k].nx = 1.0;
      tg[k].ny = tg[k].nz = 0.0;
#pragma unroll
      for (int r = 0; r < R; ++r) tg[k].c[r] = tg[k].a[r] = 0.0;
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
    if (cnt == 0) {
      // empty stage (ragged last block): arrive without a transfer
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[buf])) : "memory");
    } else {
      const uint32_t bytes = static_cast<uint32_t>(TILE * F * sizeof(double));  // whole (padded) tile
      mbar_expect_tx(&full[buf], bytes);
      tma_bulk_g2s(sbuf + buf * TILE * F, a.rec + (j0 / TILE) * (TILE * F), bytes, &full[buf]);
    }
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES && s < nstage; ++s) issue(s, s);
  }

  for (int64_t q = 0; q < nstage; ++q) {
    const int buf = static_cast<int>(q % STAGES);
    mbar_wait(&full[buf], static_cast<uint32_t>((q / STAGES) & 1));
    const double* sb = sbuf + buf * TILE * F;
    int64_t j0;
    int cnt;
    stage_src(q, j0, cnt);
    const int64_t o = o0 + q / stages_per_block;
    const int jl0 = static_cast<int>((q % stages_per_block) * TILE);  // offset of this stage in the J-block
    // Groups of 32 sources.  At step st lane l evaluates source (l + st) & 31 of the group
    // against its T targets; the reverse accumulators of that source travel with it (handed
    // from lane l+1 to lane l after every step), so after 32 steps lane l holds the warp's
    // complete reverse sums for source l: no shuffle-add reduction tree.
    for (int g0 = 0; g0 < cnt; g0 += 32) {
      const int gcnt = (cnt - g0 < 32) ? cnt - g0 : 32;
      Acc2 rv[R];
#pragma unroll
      for (int r = 0; r < R; ++r) rv[r].p0 = rv[r].p1 = 0.0;
      if (o != 0 && gcnt == 32) {
        // one step: the T targets against source sj, then the reverse accumulators move one lane
        auto step = [&](const SymSrc<R>& sj) {
#pragma unroll
          for (int k = 0; k < T; ++k) pair_sym<SCREENED, R>(tg[k], sj, kc, s_tab, fa[k], rv);
#pragma unroll
          for (int r = 0; r < R; ++r) {
            rv[r].p0 = __shfl_sync(0xffffffffu, rv[r].p0, (lane + 1) & 31);
            rv[r].p1 = __shfl_sync(0xffffffffu, rv[r].p1, (lane + 1) & 31);
          }
        };
        constexpr int PF = sym_prefetch(R);
        if constexpr (PF == 2) {
          // ping-pong record buffers: the next step's record loads while this step computes, with
          // no register copies between steps (loop unrolled by two)
          SymSrc<R> ra, rb;
          rec_load<R>(sb, g0 + lane, ra);
#pragma unroll 1
          for (int st = 0; st < 32; st += 2) {
            rec_load<R>(sb, g0 + ((lane + st + 1) & 31), rb);
            step(ra);
            rec_load<R>(sb, g0 + ((lane + st + 2) & 31), ra);  // wraps harmlessly at st = 30
            step(rb);
          }
        } else if constexpr (PF == 1) {
          // the next step's record is loaded while this step computes (software pipelining)
          SymSrc<R> nxt;
          rec_load<R>(sb, g0 + lane, nxt);
          BIPB_UNROLL_(BIPB_SYM_STUNROLL)
          for (int st = 0; st < 32; ++st) {
            const SymSrc<R> sj = nxt;
            rec_load<R>(sb, g0 + ((lane + st + 1) & 31), nxt);  // wraps harmlessly at st = 31
            step(sj);
          }
        } else {
#pragma unroll 1
          for (int st = 0; st < 32; ++st) {
            SymSrc<R> sj;
            rec_load<R>(sb, g0 + ((lane + st) & 31), sj);
            step(sj);
          }
        }
      } else {
        // diagonal block (pairs i < j only) or a partial group
#pragma unroll 1
        for (int st = 0; st < 32; ++st) {
          const int q32 = (lane + st) & 31;
          if (q32 < gcnt) {
            const int jq = g0 + q32;
            const int64_t gj = j0 + jq;
            SymSrc<R> sj;
            rec_load<R>(sb, jq, sj);
#pragma unroll
            for (int k = 0; k < T; ++k)
              if (o != 0 || gi[k] < gj) pair_sym<SCREENED, R>(tg[k], sj, kc, s_tab, fa[k], rv);
          }
#pragma unroll
          for (int r = 0; r < R; ++r) {
            rv[r].p0 = __shfl_sync(0xffffffffu, rv[r].p0, (lane + 1) & 31);
            rv[r].p1 = __shfl_sync(0xffffffffu, rv[r].p1, (lane + 1) & 31);
          }
        }
      }
      if (lane < gcnt) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          double* rs = rsum + ((warp * R + r) * 2) * RS + (jl0 % RS) + g0 + lane;
          rs[0] = rv[r].p0;
          rs[RS] = rv[r].p1;
        }
      }
    }
    __syncthreads();  // buffer `buf` consumed; rsum entries of this stage written
    if (threadIdx.x == 0 && q + STAGES < nstage) issue(q + STAGES, buf);
    if ((q + 1) % (RS / TILE) == 0) {
      // combine the warps (fixed order), fold the s powers, write rows base .. base + RS of Rev[I][o]
      const int64_t J = (I + o) % a.nb;
      const int base = jl0 + TILE - RS;
      for (int jt = threadIdx.x; jt < RS; jt += TPB) {
        const int jl = base + jt;
        if (J * B + jl >= a.n) continue;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          double q0 = 0.0, q1 = 0.0;
#pragma unroll
          for (int w = 0; w < NW; ++w) {
            q0 += rsum[((w * R + r) * 2) * RS + jt];
            q1 += rsum[((w * R + r) * 2 + 1) * RS + jt];
          }
          const double v0 = SCREENED ? a.sc1 * q0 : (a.eps - 1.0) * q0;
          const double v1 = SCREENED ? a.sc2 * q1 : -((1.0 - a.inveps) * q1);
          if constexpr (EXACT) {
            const double p2s = exact_scale_dev(a.xexp, a.xbias);
            exact_add(a.xl, 2 * a.n, J * B + jl, v0, p2s);
            exact_add(a.xl, 2 * a.n, a.n + J * B + jl, v1, p2s);
            continue;
          }
          double* rv0 = a.rev + (((Il * (a.hmax + 1) + o) * R + r) * 2) * B;
          rv0[jl] = v0;
          rv0[B + jl] = v1;
        }
      }
      __syncthreads();  // rsum reused
    }
  }

  // forward partials of this run
#pragma unroll
  for (int k = 0; k < T; ++k) {
    const int l = threadIdx.x + k * TPB;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double v0 = SCREENED ? a.sc1 * fa[k][r].p0 : (a.eps - 1.0) * fa[k][r].p0;
      const double v1 = SCREENED ? a.sc2 * fa[k][r].p1 : -((1.0 - a.inveps) * fa[k][r].p1);
      if constexpr (EXACT) {
        if (gi[k] < a.n) {
          const double p2s = exact_scale_dev(a.xexp, a.xbias);
          exact_add(a.xl, 2 * a.n, gi[k], v0, p2s);
          exact_add(a.xl, 2 * a.n, a.n + gi[k], v1, p2s);
        }
        continue;
      }
      double* f0 = a.fwd + (((Il * a.runs + run) * R + r) * 2) * B;
      f0[l] = v0;
      f0[B + l] = v1;
    }
  }
}

// records {x s, y s, z s, nu, (c = W u_dphi, a' = s W u_phi) x R}; U = [R][2n]
template <int R>
__global__ void prescale_sym_kernel(const double* __restrict__ U, const double* __restrict__ w,
                                    const double* __restrict__ ex, const double* __restrict__ ey,
                                    const double* __restrict__ ez, const double* __restrict__ nx,
                                    const double* __restrict__ ny, const double* __restrict__ nz,
                                    double* __restrict__ rec, int64_t n, double s, int* __restrict__ xexp) {
  constexpr int F = SymLayout<R>::F;
  int emax = 0;  // exact sums: largest exponent field of the weights c, a'
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    using L = SymLayout<R>;
    double* p = rec + sym_idx(j, 0, F);
    p[0] = ex[j];
    p[TILE] = ey[j];
    p[2 * TILE] = ez[j];
    p[L::NX * TILE] = nx[j];
    p[(L::NX + 1) * TILE] = ny[j];
    p[(L::NX + 2) * TILE] = nz[j];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double cw = w[j] * U[(int64_t)r * 2 * n + n + j];
      const double aw = s * (w[j] * U[(int64_t)r * 2 * n + j]);
      p[L::C(r) * TILE] = cw;
      p[L::A(r) * TILE] = aw;
      emax = max(emax, max(exact_exp_field(cw), exact_exp_field(aw)));
    }
  }
  if (xexp) exact_note_exp(xexp, emax);
}

// Add one launch group's partials to the running row sums P = [R][2][n] (P0 | P1 blocks).
// For global row i (block b, local l): forward runs of block b (if b is in [Ia, Ib)) in run
// order, then reverse offsets o = 0..hmax of the tiles (I = b - o mod nb, J = b) with I in
// [Ia, Ib) and o < noff(I).  Fixed order -> deterministic.
// With nbox > 0 (last group, peer-store exchange) the row sums go to slot [rank] of every rank's
// mailbox (bipb_p2p.cuh) instead of P.
template <int R>
__global__ void reduce_sym_kernel(const double* __restrict__ fwd, const double* __restrict__ rev, int64_t n,
                                  int64_t nb, int64_t B, int64_t runs, int64_t hmax, int64_t Ia, int64_t Ib,
                                  int first, double* __restrict__ P, const PeerBoxes box, int nbox, int rank,
                                  int64_t stride, const unsigned long long* __restrict__ epoch) {
  const int64_t boff = nbox > 0 ? p2p_next_parity(epoch) * stride + (int64_t)rank * R * 2 * n : 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = i / B, l = i % B;
    double s0[R], s1[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      s0[r] = first ? 0.0 : P[(int64_t)(2 * r) * n + i];
      s1[r] = first ? 0.0 : P[(int64_t)(2 * r + 1) * n + i];
    }
    if (b >= Ia && b < Ib) {
      for (int64_t run = 0; run < runs; ++run) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const double* f = fwd + ((((b - Ia) * runs + run) * R + r) * 2) * B;
          s0[r] += f[l];
          s1[r] += f[B + l];
        }
      }
    }
    // offsets o whose source block I = b - o (mod nb) lies in [Ia, Ib): o = lo .. lo + L - 1
    // (mod nb), visited in ascending o (two segments when the range wraps)
    const int64_t L = Ib - Ia;
    const int64_t lo = ((b - (Ib - 1)) % nb + nb) % nb;
    const int64_t seg[2][2] = {{0, lo + L - 1 - nb}, {lo, lo + L - 1 < nb ? lo + L - 1 : nb - 1}};
    for (int sgi = 0; sgi < 2; ++sgi) {
      const int64_t oe = seg[sgi][1] < hmax ? seg[sgi][1] : hmax;
      for (int64_t o = seg[sgi][0]; o <= oe; ++o) {
        const int64_t I = ((b - o) % nb + nb) % nb;
        if (o >= sym_noff(I, nb)) continue;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const double* rv = rev + ((((I - Ia) * (hmax + 1) + o) * R + r) * 2) * B;
          s0[r] += rv[l];
          s1[r] += rv[B + l];
        }
      }
    }
    if (nbox > 0) {
      for (int p = 0; p < nbox; ++p) {
        double* b = box.p[p] + boff;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          b[(int64_t)(2 * r) * n + i] = s0[r];
          b[(int64_t)(2 * r + 1) * n + i] = s1[r];
        }
      }
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        P[(int64_t)(2 * r) * n + i] = s0[r];
        P[(int64_t)(2 * r + 1) * n + i] = s1[r];
      }
    }
  }
}

// Y[r] = d U[r] - P[r] / (4 pi)  (P after the cross-rank sum)
template <int R>
__global__ void finish_sym_kernel(const double* __restrict__ P, const double* __restrict__ U, int64_t n, double d1,
                                  double d2, double* __restrict__ Y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t o = (int64_t)r * 2 * n;
      Y[o + i] = d1 * U[o + i] - P[o + i] / FOUR_PI;
      Y[o + n + i] = d2 * U[o + n + i] - P[o + n + i] / FOUR_PI;
    }
  }
}

}  // namespace bipb
