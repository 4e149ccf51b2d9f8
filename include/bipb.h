/*
 * bipb.h — C ABI of the B200-native direct-sum boundary-integral Poisson-Boltzmann
 * hot path (Geng & Jacob, arXiv 1301.5885; "P:<line>" = /root/reference/PAPER.md).
 *
 * The library (paper_1301_5885_b200/libbipb.so) evaluates, in FP64 on one or more
 * B200 GPUs (one process per GPU), the three direct sums of the paper's Table 1
 * and the restarted GMRES that drives the second one:
 *   bipb_source      b = [S1; S2]                 Eq. (11), P:242-245   (Table 1 step 6)
 *   bipb_matvec      y = A u                      Eqs. (12)-(13), P:264-269 (step 11)
 *   bipb_gmres_solve A x = b, GMRES(m), x0 given  P:271-272, P:342-356 (steps 9-16)
 *   bipb_energy      E_sol = 1/2 sum q_k phi_reac Eq. (14), P:278-286 (steps 18-21)
 * with the kernels K1..K4 of Eq. (10) built from G0 = 1/(4 pi r) and
 * Gk = exp(-kappa r)/(4 pi r) (Eq. (5)), flat triangles with centroid
 * collocation, the singular self term removed.
 *
 * Conventions:
 *   R1  eps = eps2/eps1 (P:247 prints eps1/eps2; Eqs. (8)-(9) require eps2/eps1).
 *   R2  S1 = (1/eps1) sum_k q_k G0,  S2 = (1/eps1) sum_k q_k dG0/dnu_x.
 *   R3  q_k = Q_k in units of e_c; E_sol = 1/2 * 4 pi * 332.0716 * sum_k Q_k phi_reac(x_k)
 *       in kcal/mol.
 *   Vectors of length 2N are laid out [phi_1..phi_N, dphi/dnu_1..dphi/dnu_N].
 *
 * Pointers: every array argument may be a HOST pointer or a DEVICE pointer on the
 * context's GPU (detected with cudaPointerGetAttributes; a vector on another GPU is
 * ERR_ARG).  Device pointers avoid copies.  All calls are ordered on the context's CUDA stream and return after the
 * work has completed.  A context is not thread-safe.  Errors are returned as status
 * codes, never as exceptions or aborts; bipb_last_error() gives a message.
 *
 * Multi-GPU (one process per GPU): pass a bipb_dist with the same 128-byte NCCL
 * unique id on every rank (create it with bipb_nccl_unique_id on rank 0 and
 * broadcast it).  Every rank holds the full geometry and charges, passes and receives
 * full-length vectors, and runs the same (replicated, deterministic) GMRES.  The product is
 * sharded by kernel (bipb_set_matvec_kernel): the row kernel splits target rows
 * (bipb_partition); the symmetric kernel splits its block schedule (bipb_partition of the
 * 640-row blocks) and every rank produces partial sums for all rows -- by default exact
 * fixed-point limbs (bipb_set_sum_mode), so the P-rank product is bitwise the single-GPU one.
 * Source and energy shard target rows / charges.  The per-product exchange is, by default,
 * peer stores into every rank's mailbox (see BIPB_DIST_P2P below), else NCCL collectives.
 *
 * Failures of the exchange: a peer that does not deliver within
 * BIPB_P2P_TIMEOUT_S (default 120 s), an NCCL error, or a synchronisation of a multi-rank context
 * that takes longer than BIPB_COMM_TIMEOUT_S (default 600 s) returns BIPB_ERR_NCCL (the NCCL
 * communicator is aborted with ncclCommAbort).  The context is then marked failed: every later
 * call returns BIPB_ERR_NCCL at once; destroy it.  The process's CUDA context stays usable.
 *
 * Stream ordering: the library orders a context's work on the stream given at setup (else a
 * private non-blocking stream) and each call returns after its work completed.  Device inputs
 * written on ANOTHER stream must be complete before the call (the Python binding synchronises
 * torch's current stream when it differs from the context's).
 */
#ifndef BIPB_H
#define BIPB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bipb_ctx bipb_ctx; /* opaque: owns device memory, stream, NCCL comm */

typedef enum {
  BIPB_OK = 0,
  BIPB_ERR_ARG = 1,           /* bad argument (n < 1, nc < 0, NULL where required, m < 1, ...) */
  BIPB_NOT_CONVERGED = 2,     /* GMRES hit max_iters; x and the report are still filled */
  BIPB_ERR_INPUT = 3,         /* non-finite input, area <= 0, |normal| not 1 within 1e-6 */
  BIPB_ERR_SINGULAR = 4,      /* a charge within 1e-6 A of a centroid (S1/S2 singular, R11) */
  BIPB_ERR_CUDA = 5,          /* CUDA runtime error / no device */
  BIPB_ERR_NCCL = 6,          /* NCCL missing or failed */
  BIPB_ERR_OOM = 7            /* device allocation failed */
} bipb_status;

/* Multi-GPU description; pass NULL for a single GPU. */
typedef struct {
  int32_t rank, world;       /* 0 <= rank < world */
  int32_t device;            /* CUDA device ordinal this rank uses (-1: current device) */
  int32_t flags;             /* 0, BIPB_DIST_NO_COMM (testing: no communicator; products and b
                                contain only this rank's rows, the rest is zero), or one of
                                BIPB_DIST_P2P / BIPB_DIST_NCCL (exchange choice, see below) */
  unsigned char nccl_uid[128];
} bipb_dist;
#define BIPB_DIST_NO_COMM 1
/* Per-product exchange (world > 1).  Default: peer stores — the product's epilogue kernel
 * writes its rows / partial sums straight into every rank's mailbox (CUDA IPC mappings over
 * NVLink / NVSwitch, set up once with NCCL all-gathers), then a flag handshake in device
 * memory; used when every rank can map every other rank's memory (up to 16 ranks), else the
 * NCCL collectives (all-gather / all-reduce).  Same values either way (row kernel and exact
 * sums: bitwise).  At setup every rank opens every peer's mailbox (devices compared by UUID,
 * not by per-process ordinal) and runs a self-test: each rank stores a known word and flag
 * into every mailbox, and after a barrier checks what arrived.  Any failure on any rank makes
 * all ranks use the collectives.  BIPB_DIST_P2P forces peer stores (ERR_NCCL from setup if the
 * mappings or the self-test fail; ERR_ARG beyond 16 ranks; also at world 1), BIPB_DIST_NCCL
 * forces the collectives; the environment variable BIPB_EXCHANGE=p2p|nccl overrides both. */
#define BIPB_DIST_P2P 2
#define BIPB_DIST_NCCL 4

/* GMRES report (iterations, restarts, final residual, history). */
typedef struct {
  int64_t iterations;        /* Arnoldi steps (= matvecs inside the Krylov cycles) */
  int64_t restarts;          /* number of warm restarts taken */
  int64_t matvecs;           /* all products: iterations + restart residuals + true-residual check */
  int64_t converged;         /* 1 if the relative residual reached tol */
  double rel_res_est;        /* |g_{k+1}| / ||b|| from the Givens recurrence */
  double rel_res_true;       /* ||b - A x|| / ||b|| if check_true was set, else -1 */
  double* history;           /* caller-owned HOST array for rel_res_est per iteration, may be NULL */
  int64_t history_cap;       /* its capacity */
  int64_t history_len;       /* entries produced (may exceed history_cap; extra not stored) */
} bipb_report;

/*
 * bipb_setup — Table 1 step 4: copy geometry and charges to the GPU.
 *   n          number of boundary elements N (>= 1)
 *   centroids  [n][3] row-major (x, y, z) in Angstrom
 *   normals    [n][3] unit OUTWARD normals
 *   areas      [n] element areas W_j > 0 (Eqs. (12)-(13) weights)
 *   nc         number of point charges N_c (>= 0; 0 => b = 0, x = 0, E = 0)
 *   charges    [nc][4] rows (x, y, z, Q), Q in units of e_c (R3); may be NULL if nc == 0
 *   eps1, eps2 solute / solvent dielectric constants (> 0); kappa >= 0 in 1/Angstrom
 *   dist       NULL for one GPU, else the rank/world/NCCL id (see top)
 *   cuda_stream a cudaStream_t to order all work on, or NULL for a private stream
 * The caller's arrays are copied; they may be freed on return.  On success *out owns
 * all device memory until bipb_destroy.
 * Errors: ERR_ARG, ERR_INPUT, ERR_SINGULAR, ERR_CUDA, ERR_NCCL, ERR_OOM.
 */
bipb_status bipb_setup(bipb_ctx** out, int64_t n, const double* centroids, const double* normals,
                       const double* areas, int64_t nc, const double* charges, double eps1, double eps2,
                       double kappa, const bipb_dist* dist, void* cuda_stream);

/*
 * bipb_set_charges — replace the point charges (x, y, z, Q) [nc][4] of a context while keeping
 * its surface, buffers and communicator (multi-RHS workflows: several charge sets or states on
 * one surface).  The stored right-hand side is invalidated (call
 * bipb_source again).  Errors as bipb_setup (ERR_ARG, ERR_INPUT, ERR_SINGULAR).
 */
bipb_status bipb_set_charges(bipb_ctx* ctx, int64_t nc, const double* charges);

/*
 * bipb_source — Eq. (11), Table 1 step 6: b_i = S1(x_i), b_{i+N} = S2(x_i)
 * over all N_c charges (N x N_c pairs).  The result is kept inside the context (it is
 * the default right-hand side of bipb_gmres_solve) and, if b != NULL, written to b [2n].
 */
bipb_status bipb_source(bipb_ctx* ctx, double* b);

/*
 * bipb_matvec — Eqs. (12)-(13), Table 1 step 11:
 *   y_i     = 1/2 (1+eps) u_i     - sum_{j != i} W_j [K1(x_i,x_j) u_{j+N} + K2(x_i,x_j) u_j]
 *   y_{i+N} = 1/2 (1+1/eps) u_{i+N} - sum_{j != i} W_j [K3(x_i,x_j) u_{j+N} + K4(x_i,x_j) u_j]
 * u, y: [2n] (must not alias).  N(N-1) pair evaluations, matrix-free.
 */
bipb_status bipb_matvec(bipb_ctx* ctx, const double* u, double* y);

/*
 * bipb_matvec_batch — the product of Eqs. (12)-(13) for nrhs operands at once (multi-RHS,
 * several charge sets / states on one surface):
 *   Y[r] = A U[r],  U, Y: [nrhs][2n] contiguous (must not alias).
 * With the symmetric kernel the distance, 1/r, exp and kernel factors of a pair are evaluated
 * once for up to 4 operands (passes of 4, 2, 1); with the row kernel it loops.
 */
bipb_status bipb_matvec_batch(bipb_ctx* ctx, int32_t nrhs, const double* U, double* Y);

/*
 * bipb_gmres_solve — restarted GMRES(m) with modified Gram-Schmidt Arnoldi and Givens
 * rotations (Saad), warm restart from the current iterate, on
 * the device; the host reads one 16-byte residual record per iteration.
 *   b          [2n] right-hand side, or NULL to use the one from the last bipb_source
 *   x          [2n] in: initial guess x0 (the paper uses 0); out: solution
 *   restart_m  Krylov dimension m >= 1 (paper: "every 10-20 steps")
 *   tol        relative residual target ||b - A x|| / ||b|| (> 0)
 *   max_iters  cap on Arnoldi steps (>= 1)
 *   check_true if nonzero, one extra product computes rep->rel_res_true
 *   rep        may be NULL
 * Returns BIPB_OK when converged, BIPB_NOT_CONVERGED when max_iters was reached (x and
 * rep filled).  ||b|| = 0 returns x = 0 at once.
 */
bipb_status bipb_gmres_solve(bipb_ctx* ctx, const double* b, double* x, int32_t restart_m, double tol,
                             int32_t max_iters, int32_t check_true, bipb_report* rep);

/*
 * bipb_gmres_solve_batch — nrhs independent systems A X[r] = B[r] (multi-RHS, §8(f) item 2):
 * each runs exactly the GMRES(m) of bipb_gmres_solve (same iterates up to the rounding of the
 * shared products); the systems advance in lockstep so every Arnoldi step applies A to all of
 * them through one bipb_matvec_batch-style product.
 *   B, X: [nrhs][2n] (host or device); X holds the initial guesses and receives the solutions.
 *   reps: NULL or an array of nrhs reports.
 * Returns BIPB_NOT_CONVERGED if any system hit max_iters (all X and reports still filled).
 */
bipb_status bipb_gmres_solve_batch(bipb_ctx* ctx, int32_t nrhs, const double* B, double* X, int32_t restart_m,
                                   double tol, int32_t max_iters, int32_t check_true, bipb_report* reps);

/*
 * bipb_energy — Eq. (14), Table 1 steps 18-21:
 *   phi_reac(x_k) = sum_j W_j [K1(x_k,x_j) x_{j+N} + K2(x_k,x_j) x_j]   (N_c x N pairs)
 *   E_sol = 1/2 * 4 pi * 332.0716 * sum_k Q_k phi_reac(x_k)  [kcal/mol]   (R3)
 *   x        [2n] solved surface potential and normal derivative
 *   e_sol    out: E_sol (host or device double), required
 *   phi_reac out: [nc] reaction potentials (internal units e_c/A, R3), may be NULL
 */
bipb_status bipb_energy(bipb_ctx* ctx, const double* x, double* e_sol, double* phi_reac);

/* Free everything the context owns (NULL is a no-op). */
void bipb_destroy(bipb_ctx* ctx);

/* Thread-local message describing the last non-OK status ("" if none). */
const char* bipb_last_error(void);

/* Rows [*r0, *r1) of n owned by `rank` of `world` (equal ceil(n/world) blocks; host-only). */
void bipb_partition(int64_t n, int32_t world, int32_t rank, int64_t* r0, int64_t* r1);

/* Create a fresh NCCL unique id (rank 0) into out[128].  ERR_NCCL if NCCL is unavailable. */
bipb_status bipb_nccl_unique_id(unsigned char* out);

/*
 * Matvec kernel selection.  Both compute Eqs. (12)-(13) exactly (same sums,
 * different rounding order):
 *   0  row kernel: every ordered pair (i, j) evaluated by the thread owning row i; a row's
 *      value is bitwise independent of the launch configuration and of the rank count.
 *   1  symmetric kernel: each unordered pair {i, j} evaluated once and used for both rows
 *      (K1, K4 symmetric; K2/K3 exchange under d -> -d); 27.5 instead of 47 FP64
 *      instructions per ordered pair.  Partial sums are added as exact fixed-point limbs by
 *      default (bipb_set_sum_mode 1: bitwise independent of schedule and rank count), or as
 *      fixed-order double partials (mode 0: deterministic for a fixed rank count); across
 *      ranks they travel through the per-product exchange (peer stores or NCCL).
 * Default: 1 when the problem has at least one wave (296) of 640 x 640 tile pairs
 * (N >~ 15k), else 0.  BIPB_MATVEC=row|sym in the environment overrides it at setup.
 */
bipb_status bipb_set_matvec_kernel(bipb_ctx* ctx, int32_t kind);
int32_t bipb_get_matvec_kernel(bipb_ctx* ctx);

/* How products are exchanged between ranks: 0 none (one GPU or BIPB_DIST_NO_COMM),
 * 1 NCCL collectives, 2 peer stores (BIPB_DIST_P2P above); -1 for a NULL context. */
int32_t bipb_get_exchange(bipb_ctx* ctx);

/* How bipb_gmres_solve runs the orthogonalisation of each Arnoldi step (same algorithm: modified
 * Gram-Schmidt, Givens rotation, normalisation):
 *   0   one reduction kernel per MGS dot product (k + 4 launches in step k)
 *   E>0 one kernel on one 8-CTA thread-block cluster, E vector elements per thread in registers,
 *       the dot products reduced through distributed shared memory (2N <= 8 * 1024 * E; chosen
 *       at setup for 2N <= 65536, i.e. N <= 32768; BIPB_ARNOLDI=launches in the environment
 *       forces 0).  Deterministic; only the summation order of the dots differs from 0.
 * -1 for a NULL context. */
int32_t bipb_get_arnoldi(bipb_ctx* ctx);

/*
 * Device-side GMRES cycles (an execution mode of bipb_gmres_solve, Table 1 steps 9-16; opt-in with
 * BIPB_GRAPHS=2 in the environment): the m Arnoldi steps of a cycle run as ONE CUDA-graph launch,
 * each step in a conditional (IF) node that a one-thread kernel clears once the host loop would
 * leave the cycle (breakdown, convergence, max_iters, NaN), and the host reads the per-step
 * residual records once per cycle.  Results are bitwise those of the eager loop.  Used on
 * single-GPU contexts after one eager product (a graph capture cannot allocate); if the graph
 * cannot be built the context falls back to eager cycles for good.
 * Returns the number of cycles this context has run as graphs (0 when the mode is off), -1 for a
 * NULL context.
 */
int64_t bipb_get_graph_cycles(bipb_ctx* ctx);

/*
 * GMRES preconditioning (NOT in the paper, which runs plain GMRES; default 0):
 *   0  plain GMRES(m) (the paper's method; parity with the oracle's iteration counts)
 *   1  right preconditioning by the diagonal of the jump terms of Eqs. (12)-(13),
 *      M = diag(1/2 (1 + eps) I_N, 1/2 (1 + 1/eps) I_N) (Saad, Algorithm 9.5: each Arnoldi step
 *      applies A to M^-1 v_k; a cycle ends with x += M^-1 V y).  Same linear system and the same
 *      true-residual test ||b - A x|| / ||b|| <= tol, so the same solution and energy to the
 *      tolerance; the 40.5 : 0.506 scaling of the two row blocks (eps = 80) no longer slows the
 *      Krylov iteration (C4: 26 -> 10 iterations, 5.25 -> 1.95 s).  Applies to bipb_gmres_solve and
 *      bipb_gmres_solve_batch.  BIPB_PRECOND=jacobi in the environment sets 1 at setup.
 * ERR_ARG for a NULL context or another kind; bipb_get_precond returns -1 for a NULL context.
 */
bipb_status bipb_set_precond(bipb_ctx* ctx, int32_t kind);
int32_t bipb_get_precond(bipb_ctx* ctx);

/*
 * How the symmetric kernel's partial row sums of a single-operand product are added
 * (bipb_matvec, bipb_gmres_solve; the batched products always use mode 0):
 *   0  fixed-order double partials: every (I-block, offset) tile writes its partial
 *      sums to HBM (C4: 1.4 GB per product) and a reduce kernel adds them in a fixed order;
 *      deterministic, but the rounding depends on the rank count.
 *   1  exact fixed-point sums (default; csrc/bipb_exact.cuh): every partial v is rounded to a multiple of
 *      2^-S (S = 80 - E_u, 2^E_u bounding the operand weights W u; resolution 2^-80 of the largest
 *      weight) and added with 64-bit integer atomics into three limbs per row (48 N bytes, resident
 *      in L2).  Integer sums are associative: the result is bitwise identical for any schedule and
 *      any number of ranks (the limbs are exchanged and summed as integers).  A partial beyond
 *      2^38 times the largest weight, or not finite, is detected on the device; the library then
 *      recomputes with mode 0 (bipb_matvec: that product; bipb_gmres_solve: the whole solve from
 *      x0) and keeps mode 0 for the context (bipb_get_sum_mode then returns 0).
 * The product is the same operator to rounding either way (Eqs. (12)-(13)); only the
 * summation of the partials differs.  Measured at C4: the same speed in both modes (5.19 s per solve),
 * 34.8 MB of DRAM traffic per product with exact sums vs 1.45 GB.  BIPB_SUM=fixed in the environment
 * sets 0 at setup.
 * ERR_ARG for a NULL context or another mode; bipb_get_sum_mode returns -1 for a NULL context.
 */
bipb_status bipb_set_sum_mode(bipb_ctx* ctx, int32_t mode);
int32_t bipb_get_sum_mode(bipb_ctx* ctx);

/*
 * Instrumentation (bench.py, tests).  `which`: 0 = matvec pair kernel, 1 = source pair
 * kernel, 2 = energy pair kernel, 3 = all kernels of the library.
 * bipb_timing_enable(ctx, 1) brackets each pair-kernel launch with CUDA events on the
 * context stream; bipb_timing_get returns the summed device time (ms) and the launch
 * count since the last reset (for which == 3 only the launch count is meaningful).
 */
bipb_status bipb_timing_enable(bipb_ctx* ctx, int32_t on);
bipb_status bipb_timing_get(bipb_ctx* ctx, int32_t which, double* total_ms, int64_t* launches);
bipb_status bipb_timing_reset(bipb_ctx* ctx);

/* Library version string and the compile-time target ("sm_100a"). */
const char* bipb_version(void);

#ifdef __cplusplus
}
#endif
#endif /* BIPB_H */
