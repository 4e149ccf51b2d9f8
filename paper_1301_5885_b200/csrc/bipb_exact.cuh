// bipb_exact.cuh — exact fixed-point accumulation of the symmetric kernel's row sums
// (DESIGN.md §6 "exact sums"; opt-in: bipb_set_sum_mode(ctx, 1) / BIPB_SUM=exact).
//
// The symmetric kernel (bipb_sym.cuh) produces, per product, one forward partial per (I-block,
// run) and one reverse partial per (I-block, offset) for every row: ~nb/2 + runs partials per
// row.  The default mode writes them to HBM as doubles and adds them in a fixed order (1.4 GB
// written and read back per C4 product).  This mode instead rounds every partial v to an
// integer multiple of 2^-S and adds it with 64-bit integer atomics (red.global.add.u64) into
// three limbs per row held in a 48N-byte buffer that stays in L2:
//     V = round(v 2^S) = sgn(v) (h 2^80 + m 2^40 + l),  0 <= l, m < 2^40 (l rounded), 0 <= h
//     row limbs L0 += +-l, L1 += +-m, L2 += +-h            (two's complement, wrap-free below)
// Integer addition is associative, so the row sums are exact and do not depend on the order
// in which CTAs finish, on the schedule (W, groups) or on the number of ranks: the final
// double is a fixed function of the exact integer (bitwise identical for any P).
//
// Scale: S = 80 - E_u where 2^E_u bounds every |c_j|, |a'_j| of the operand (one integer
// atomicMax over the exponent fields in the prescale kernel; the same on every rank because u
// is replicated).  Resolution U 2^-80 (U = max operand weight), far below the FP64 rounding of
// any row of size >= U 2^-27; range |v| < 2^118 2^-S = U 2^38 per partial.  Limb bounds: with
// K <= 2^23 partials per row, |L0|, |L1| < 2^63 and |L2| < 2^61.  A partial outside the range
// (or not finite) raises a device flag; the library then recomputes the product with the
// double partials (bipb.cu), so results are always correct.
#pragma once
#include <cmath>
#include <cstdint>
#ifdef __CUDACC__
#include "bipb_p2p.cuh"
#endif

#ifndef __CUDACC__
#define BIPB_HD
#else
#define BIPB_HD __host__ __device__
#endif

namespace bipb {

constexpr int EXACT_LIMB_BITS = 40;
constexpr long long EXACT_LIMB_MASK = (1LL << EXACT_LIMB_BITS) - 1;
constexpr int EXACT_S_TOP = 80;         // S = EXACT_S_TOP - E_u
constexpr double EXACT_MAX = 0x1p118;   // |v 2^S| must stay below this
constexpr int EXACT_S_CLAMP = 1000;     // |S| <= 1000 keeps 2^S and 2^-S normal doubles

struct ExactLimbs {
  long long l0, l1, l2;
};

// Split one partial v (scaled by p2s = 2^S) into signed limbs; returns false when out of range.
BIPB_HD inline bool exact_split(double v, double p2s, ExactLimbs& out) {
  const double ax = fabs(v * p2s);  // exact: power-of-two scaling (no overflow below the check)
  if (!(ax < EXACT_MAX)) {         // also catches NaN / inf
    out.l0 = out.l1 = out.l2 = 0;
    return false;
  }
  const double h = floor(ax * 0x1p-80);
  const double r1 = ax - h * 0x1p80;  // exact: the bits of ax below 2^80
  const double m = floor(r1 * 0x1p-40);
  const double r0 = r1 - m * 0x1p40;  // exact: the bits of ax below 2^40
  const double l = rint(r0);          // the one rounding (to the nearest multiple of 2^-S)
  long long L0 = static_cast<long long>(l), L1 = static_cast<long long>(m), L2 = static_cast<long long>(h);
  if (v < 0) {
    L0 = -L0;
    L1 = -L1;
    L2 = -L2;
  }
  out.l0 = L0;
  out.l1 = L1;
  out.l2 = L2;
  return true;
}

// The double nearest (within ~1 ulp) to (L2 2^80 + L1 2^40 + L0) 2^-S, a fixed function of the
// exact integer (the limbs are first carry-normalised, which is unique).
BIPB_HD inline double exact_value(long long L0, long long L1, long long L2, double p2ms) {
  const long long c0 = L0 >> EXACT_LIMB_BITS;  // arithmetic shift = floor division
  const long long t0 = L0 & EXACT_LIMB_MASK;
  L1 += c0;
  const long long c1 = L1 >> EXACT_LIMB_BITS;
  const long long t1 = L1 & EXACT_LIMB_MASK;
  L2 += c1;
  const double hi = static_cast<double>(L2) * 0x1p80;
  const double mid = static_cast<double>(t1) * 0x1p40;  // exact
  const double lo = static_cast<double>(t0);            // exact
  return ((hi + mid) + lo) * p2ms;
}

// S from the largest biased exponent field Eb of the operand weights (Eb = 0: a zero (or
// subnormal-only) operand, whose products are zero (resp. below 2^-1000) anyway).
BIPB_HD inline int exact_shift(int Eb) {
  if (Eb <= 0) return EXACT_S_CLAMP;
  const int Eu = Eb - 1022;  // every weight < 2^Eu
  int S = EXACT_S_TOP - Eu;
  if (S > EXACT_S_CLAMP) S = EXACT_S_CLAMP;
  if (S < -EXACT_S_CLAMP) S = -EXACT_S_CLAMP;
  return S;
}

BIPB_HD inline int exact_exp_field(double v) {
  union {
    double d;
    unsigned long long u;
  } b;
  b.d = v;
  return static_cast<int>((b.u >> 52) & 0x7ff);
}

BIPB_HD inline double exact_pow2(int S) {  // 2^S for |S| <= 1022
  union {
    double d;
    unsigned long long u;
  } b;
  b.u = static_cast<unsigned long long>(S + 1023) << 52;
  return b.d;
}

#ifdef __CUDACC__
// Row limbs: xl[k * 2n + row] (k = 0, 1, 2; row < 2n), xl[6n] = count of out-of-range partials.
__device__ __forceinline__ double exact_scale_dev(const int* xexp, int bias) {
  return exact_pow2(exact_shift(__ldg(xexp)) + bias);
}
__device__ __forceinline__ void exact_add(unsigned long long* __restrict__ xl, int64_t n2, int64_t row, double v,
                                          double p2s) {
  ExactLimbs l;
  if (!exact_split(v, p2s, l)) {
    atomicAdd(xl + 3 * n2, 1ull);
    return;
  }
  if (l.l0) atomicAdd(xl + row, static_cast<unsigned long long>(l.l0));  // result unused: RED
  if (l.l1) atomicAdd(xl + n2 + row, static_cast<unsigned long long>(l.l1));
  if (l.l2) atomicAdd(xl + 2 * n2 + row, static_cast<unsigned long long>(l.l2));
}

// Largest exponent field of the operand weights (one atomicMax per warp; max is order-free).
__device__ __forceinline__ void exact_note_exp(int* xexp, int e) {
  e = __reduce_max_sync(0xffffffffu, e);
  if ((threadIdx.x & 31) == 0 && e > 0) atomicMax(xexp, e);
}

// Peer-store exchange of the limbs: this rank's 6n + 1 words into slot [rank] of every rank's
// mailbox (next parity), exactly like reduce_sym_kernel's double partials (bipb_p2p.cuh).
__global__ void exact_publish_p2p_kernel(const unsigned long long* __restrict__ xl, int64_t words,
                                         const PeerBoxes box, int world, int rank, int64_t stride,
                                         const unsigned long long* __restrict__ epoch) {
  const int64_t off = static_cast<int64_t>(p2p_next_parity(epoch)) * stride + (int64_t)rank * words;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < words; i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long v = xl[i];
    for (int p = 0; p < world; ++p) reinterpret_cast<unsigned long long*>(box.p[p])[off + i] = v;
  }
}

// Y = d U - P / (4 pi), P the exact row sums: limbs summed over `nslots` slots (integer adds, so
// the order is irrelevant), carry-normalised and converted.  base: own limbs (1 slot) or the own
// mailbox (epoch != nullptr: current parity, one slot per rank).  Any out-of-range partial on any
// rank makes every row NaN and sets *sticky (the host then recomputes with double partials).
__global__ void finish_exact_kernel(const unsigned long long* __restrict__ base, int64_t stride,
                                    const unsigned long long* __restrict__ epoch, int nslots, int64_t words,
                                    const int* __restrict__ xexp, int bias, const double* __restrict__ U, int64_t n,
                                    double d1, double d2, double* __restrict__ Y, int* __restrict__ sticky) {
  if (epoch) base += static_cast<int64_t>(*epoch & 1ull) * stride;
  const int64_t n2 = 2 * n;
  unsigned long long F = 0;
  for (int p = 0; p < nslots; ++p) F += base[p * words + 3 * n2];
  const double p2ms = exact_pow2(-(exact_shift(*xexp) + bias));
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long L0 = 0, L1 = 0, L2 = 0;
    for (int p = 0; p < nslots; ++p) {
      const unsigned long long* b = base + p * words;
      L0 += b[i];
      L1 += b[n2 + i];
      L2 += b[2 * n2 + i];
    }
    const double v = exact_value(static_cast<long long>(L0), static_cast<long long>(L1), static_cast<long long>(L2), p2ms);
    Y[i] = F ? __longlong_as_double(0x7ff8000000000000LL) : (i < n ? d1 : d2) * U[i] - v / FOUR_PI;
  }
  if (F && blockIdx.x == 0 && threadIdx.x == 0) *sticky = 1;
}
#endif

}  // namespace bipb
