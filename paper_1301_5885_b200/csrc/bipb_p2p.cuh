// bipb_p2p.cuh — the per-product exchange done by the kernels themselves
// over peer memory (NVLink / NVSwitch P2P stores), instead of an NCCL collective after the
// product (DESIGN.md §8 "peer-store exchange").
//
// Every rank owns a mailbox in device memory, mapped into every other rank with CUDA IPC at
// setup: box[2 parities][stride] doubles plus a flag word per rank.  One exchange =
//   1. the product's epilogue kernel computes its values and STORES them straight into every
//      rank's mailbox (row kernel: rows [r0, r1) at their global positions; symmetric kernel:
//      this rank's partial sums of all rows into slot [rank]; likewise the source term's rows
//      and the energy's per-charge potentials);
//   2. p2p_signal_kernel: system-scope fence, epoch += 1, release-store the epoch into flag
//      [rank] of every rank;
//   3. p2p_wait_kernel: acquire-spin until every rank's flag in the OWN flag array reached the
//      epoch.  A peer that never arrives within BIPB_P2P_TIMEOUT_S seconds sets an error word in
//      mapped host memory and the kernel returns (no trap: the CUDA context stays usable); the
//      host turns the word into BIPB_ERR_NCCL and marks the context failed;
//   4. the consumer kernel reads the own mailbox (row kernel: copy y; symmetric kernel: sum the
//      ranks' slots in rank order, so every rank gets bitwise the same y).
// The mailbox parity alternates with the epoch so a fast rank can never overwrite a slot a slow
// rank is still reading (it needs the slow rank's next delivery first).  The epoch lives in
// device memory, so the sequence is CUDA-graph capturable.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "bipb_kernels.cuh"


#include "bipb_vec.cuh"

namespace bipb {

constexpr int P2P_MAX = 16;
struct PeerBoxes {
  double* p[P2P_MAX];  // every rank's mailbox base (own one included), mapped into this process
};
struct PeerFlags {
  unsigned long long* p[P2P_MAX];  // every rank's flag array [world]
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ int p2p_next_parity(const unsigned long long* epoch) {
  return static_cast<int>((*epoch + 1ull) & 1ull);
}

// Row kernel epilogue + exchange: the rank's rows (same arithmetic and chunk order as
// reduce_matvec_kernel, so values are bitwise those of the NCCL path) stored into every
// rank's mailbox at global rows r0 + l and n + r0 + l.
__global__ void reduce_matvec_p2p_kernel(const double* __restrict__ part, int64_t nchunk, int64_t ntgt,
                                         const double* __restrict__ u0, const double* __restrict__ u1, double d1,
                                         double d2, int64_t r0, int64_t n, const PeerBoxes box, int world,
                                         int64_t stride, const unsigned long long* __restrict__ epoch) {
  const int64_t off = static_cast<int64_t>(p2p_next_parity(epoch)) * stride;
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < ntgt; l += (int64_t)gridDim.x * blockDim.x) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll RED_UNROLL
    for (int64_t c = 0; c < nchunk; ++c) {
      s0 += part[(2 * c) * ntgt + l];
      s1 += part[(2 * c + 1) * ntgt + l];
    }
    const double v0 = d1 * u0[l] - s0 / FOUR_PI;
    const double v1 = d2 * u1[l] - s1 / FOUR_PI;
    for (int p = 0; p < world; ++p) {
      double* b = box.p[p] + off;
      b[r0 + l] = v0;
      b[n + r0 + l] = v1;
    }
  }
}

// Source term epilogue + exchange (same arithmetic as reduce_source_kernel): b rows r0 + l and
// n + r0 + l of every rank's mailbox.
__global__ void reduce_source_p2p_kernel(const double* __restrict__ part, int64_t nchunk, int64_t ntgt, double scale,
                                         int64_t r0, int64_t n, const PeerBoxes box, int world, int64_t stride,
                                         const unsigned long long* __restrict__ epoch) {
  const int64_t off = static_cast<int64_t>(p2p_next_parity(epoch)) * stride;
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < ntgt; l += (int64_t)gridDim.x * blockDim.x) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll RED_UNROLL
    for (int64_t c = 0; c < nchunk; ++c) {
      s0 += part[(2 * c) * ntgt + l];
      s1 += part[(2 * c + 1) * ntgt + l];
    }
    for (int p = 0; p < world; ++p) {
      double* b = box.p[p] + off;
      b[r0 + l] = s0 * scale;
      b[n + r0 + l] = s1 * scale;
    }
  }
}

// Energy epilogue + exchange (same arithmetic as reduce_energy_kernel): phi_tilde of charges
// k0 + l into every rank's mailbox.
__global__ void reduce_energy_p2p_kernel(const double* __restrict__ part, int64_t nchunk, int64_t ntgt, int64_t k0,
                                         const PeerBoxes box, int world, int64_t stride,
                                         const unsigned long long* __restrict__ epoch) {
  const int64_t off = static_cast<int64_t>(p2p_next_parity(epoch)) * stride;
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < ntgt; l += (int64_t)gridDim.x * blockDim.x) {
    double s0 = 0.0;
#pragma unroll RED_UNROLL
    for (int64_t c = 0; c < nchunk; ++c) s0 += part[(2 * c) * ntgt + l];
    for (int p = 0; p < world; ++p) box.p[p][off + k0 + l] = s0;
  }
}

// epoch += 1 and publish it to flag [rank] of every rank (one thread; after the producer kernel)
__global__ void p2p_signal_kernel(unsigned long long* epoch, const PeerFlags flags, int world, int rank) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  __threadfence_system();  // the producer's peer stores are ordered before the flags
  const unsigned long long e = *epoch + 1ull;
  *epoch = e;
  for (int p = 0; p < world; ++p) st_release_sys(flags.p[p] + rank, e);
}

// wait until every rank delivered the current epoch into this rank's mailbox.  err (mapped host
// memory): 0 while healthy; on a timeout 1 + the rank that did not deliver.  Once set, later
// waits return at once (the exchange protocol is broken; the host fails the context).
__global__ void p2p_wait_kernel(const unsigned long long* epoch, const unsigned long long* my_flags, int world,
                                unsigned long long timeout_ns, unsigned int* err) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (*reinterpret_cast<volatile unsigned int*>(err) != 0u) return;
  const unsigned long long e = *epoch;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int p = 0; p < world; ++p) {
    while (ld_acquire_sys(my_flags + p) < e) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > timeout_ns) {
        atomicExch(err, 1u + static_cast<unsigned int>(p));
        __threadfence_system();
        return;
      }
      __nanosleep(200);
    }
  }
  __threadfence_system();
}

// Setup self-test of the mappings: this rank writes probe_word(rank, p) into word [rank] of every
// rank p's mailbox and `magic + rank` into flag [rank] of every rank p.  After a barrier each rank
// checks its own mailbox and flags on the host (p2p_setup).
__host__ __device__ inline unsigned long long p2p_probe_word(int from, int to) {
  return 0xB1B0C0DE00000000ull ^ (static_cast<unsigned long long>(from) << 16) ^ static_cast<unsigned long long>(to);
}
__global__ void p2p_probe_kernel(const PeerBoxes box, const PeerFlags flags, int world, int rank,
                                 unsigned long long magic) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (int p = 0; p < world; ++p)
    reinterpret_cast<unsigned long long*>(box.p[p])[rank] = p2p_probe_word(rank, p);
  __threadfence_system();
  for (int p = 0; p < world; ++p) st_release_sys(flags.p[p] + rank, magic + static_cast<unsigned long long>(rank));
}

// row kernel consumer: y = own mailbox (current parity), 2n doubles
__global__ void p2p_take_kernel(const double* __restrict__ mybox, int64_t stride,
                                const unsigned long long* __restrict__ epoch, int64_t m2, double* __restrict__ y) {
  const double* b = mybox + static_cast<int64_t>(*epoch & 1ull) * stride;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m2; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = b[i];
}

// symmetric kernel consumer: P = sum over ranks (rank order) of the slots [R][2][n];
// Y[r] = d U[r] - P[r] / (4 pi)
template <int R>
__global__ void finish_sym_p2p_kernel(const double* __restrict__ mybox, int64_t stride,
                                      const unsigned long long* __restrict__ epoch, int world,
                                      const double* __restrict__ U, int64_t n, double d1, double d2,
                                      double* __restrict__ Y) {
  const double* b = mybox + static_cast<int64_t>(*epoch & 1ull) * stride;
  const int64_t slot = (int64_t)R * 2 * n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t o = (int64_t)r * 2 * n;
      double s0 = 0.0, s1 = 0.0;
      for (int p = 0; p < world; ++p) {
        s0 += b[p * slot + o + i];
        s1 += b[p * slot + o + n + i];
      }
      Y[o + i] = d1 * U[o + i] - s0 / FOUR_PI;
      Y[o + n + i] = d2 * U[o + n + i] - s1 / FOUR_PI;
    }
  }
}

}  // namespace bipb
