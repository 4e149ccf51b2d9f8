/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU (FP64) implementation of the direct-sum
 * boundary-integral Poisson-Boltzmann method of Geng & Jacob, arXiv 1301.5885
 * (reference: /root/reference/PAPER.md, cited "P:<line>").  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load this library.  The product path (paper_1301_5885_b200/) never does, and this
 * file shares no code, header, table or constant generator with it.
 *
 * Every function is the plain definition written out in the paper's notation:
 *   - Green's functions G0, Gk: Eq. (5).
 *   - Normal derivatives: SURVEY.md Appendix A.1 (chain rule on the radial G),
 *     pinned by finite differences in tests/test_oracle_kernels.py.
 *   - Kernels K1..K4: Eq. (10), with eps = eps2/eps1 (reading R1;
 *     P:247 prints eps1/eps2, which contradicts Eqs. (8)-(9)).
 *   - Sources S1, S2: Eq. (11), with the 1/eps1 of reading R2.
 *   - Matvec: Eqs. (12)-(13); self term j=i "simply removed".
 *   - GMRES(m): Saad's restarted GMRES with MGS-Arnoldi + Givens rotations
 *     (restart/warm start P:342-347), step by step as SURVEY.md §8(c) O4.
 *   - Reaction potential + solvation energy: Eq. (14), units reading R3.
 * Loops are ascending, accumulation is left-to-right, compiled with
 * -O2 -fno-fast-math -ffp-contract=off (no FMA contraction), libm exp/sqrt.
 * OpenMP parallelises over independent target rows only (no reordering of any sum).
 *
 * Pins (tests/, -m "not gpu"): FD derivatives, kappa=0 & eps=1 structural zero,
 * K1 symmetry, dense assembly == matvec, single-charge source closed form,
 * Born / Kirkwood convergence under refinement, rotation invariance, GMRES on the
 * identity and the 2x2 example of SPEC.md S:183, GMRES vs LAPACK on the dense A.
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_PI 3.14159265358979323846

/* OpenMP threads of the following calls (timing legs: bench.py times the oracle on all host cores
 * and on one, the paper's "one CPU" framing).  No effect on any result: every parallel
 * loop is over independent rows with a fixed per-row order. */
void orc_set_threads(int64_t n) { omp_set_num_threads((int)(n > 0 ? n : 1)); }
int64_t orc_get_threads(void) { return (int64_t)omp_get_max_threads(); }

/* ---------------------------------------------------------------- vector helpers */
static double dot3(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
static double dist3(const double* x, const double* y) {
  double d0 = x[0] - y[0], d1 = x[1] - y[1], d2 = x[2] - y[2];
  return sqrt(d0 * d0 + d1 * d1 + d2 * d2);
}
/* (x - y) . v */
static double ddot3(const double* x, const double* y, const double* v) {
  return (x[0] - y[0]) * v[0] + (x[1] - y[1]) * v[1] + (x[2] - y[2]) * v[2];
}

/* ------------------------------------------------------ Eq. (5): G0, Gk */
double orc_G0(const double* x, const double* y) { return 1.0 / (4.0 * ORC_PI * dist3(x, y)); }

double orc_Gk(const double* x, const double* y, double kappa) {
  double r = dist3(x, y);
  return exp(-kappa * r) / (4.0 * ORC_PI * r);
}

/* ---------------------------- normal derivatives (d = x - y) */
/* dG0/dnu_y = (d . nu_y) / (4 pi r^3) */
double orc_dG0_dny(const double* x, const double* y, const double* ny) {
  double r = dist3(x, y);
  return ddot3(x, y, ny) / (4.0 * ORC_PI * r * r * r);
}
/* dGk/dnu_y = e^{-kr} (1 + kr) (d . nu_y) / (4 pi r^3) */
double orc_dGk_dny(const double* x, const double* y, const double* ny, double kappa) {
  double r = dist3(x, y);
  return exp(-kappa * r) * (1.0 + kappa * r) * ddot3(x, y, ny) / (4.0 * ORC_PI * r * r * r);
}
/* dG0/dnu_x = -(d . nu_x) / (4 pi r^3) */
double orc_dG0_dnx(const double* x, const double* nx, const double* y) {
  double r = dist3(x, y);
  return -ddot3(x, y, nx) / (4.0 * ORC_PI * r * r * r);
}
/* dGk/dnu_x = -e^{-kr} (1 + kr) (d . nu_x) / (4 pi r^3) */
double orc_dGk_dnx(const double* x, const double* nx, const double* y, double kappa) {
  double r = dist3(x, y);
  return -exp(-kappa * r) * (1.0 + kappa * r) * ddot3(x, y, nx) / (4.0 * ORC_PI * r * r * r);
}
/* d2G0/dnu_x dnu_y = [ (nu_x . nu_y)/r^3 - 3 (d . nu_x)(d . nu_y)/r^5 ] / (4 pi) */
double orc_d2G0_dnxdny(const double* x, const double* nx, const double* y, const double* ny) {
  double r = dist3(x, y);
  double r3 = r * r * r, r5 = r3 * r * r;
  return (dot3(nx, ny) / r3 - 3.0 * ddot3(x, y, nx) * ddot3(x, y, ny) / r5) / (4.0 * ORC_PI);
}
/* d2Gk/dnu_x dnu_y = e^{-kr} [ (1+kr)(nu_x . nu_y)/r^3 - (3+3kr+k^2r^2)(d . nu_x)(d . nu_y)/r^5 ] / (4 pi) */
double orc_d2Gk_dnxdny(const double* x, const double* nx, const double* y, const double* ny,
                       double kappa) {
  double r = dist3(x, y);
  double r3 = r * r * r, r5 = r3 * r * r;
  double kr = kappa * r;
  return exp(-kr) *
         ((1.0 + kr) * dot3(nx, ny) / r3 - (3.0 + 3.0 * kr + kr * kr) * ddot3(x, y, nx) * ddot3(x, y, ny) / r5) /
         (4.0 * ORC_PI);
}

/* ------------------------------------------------ Eq. (10): K1..K4 */
/* eps = eps2/eps1 (reading R1). K[0..3] = K1..K4 at target x (normal nx), source y (ny). */
void orc_kernels(const double* x, const double* nx, const double* y, const double* ny, double eps,
                 double kappa, double* K) {
  K[0] = orc_G0(x, y) - orc_Gk(x, y, kappa);
  K[1] = eps * orc_dGk_dny(x, y, ny, kappa) - orc_dG0_dny(x, y, ny);
  K[2] = orc_dG0_dnx(x, nx, y) - (1.0 / eps) * orc_dGk_dnx(x, nx, y, kappa);
  K[3] = orc_d2Gk_dnxdny(x, nx, y, ny, kappa) - orc_d2G0_dnxdny(x, nx, y, ny);
}

/* ------------------------------------- Eq. (11): b = [S1; S2] (R2) */
/* cen, nrm: [n][3]; chg: [nc][4] = (x, y, z, Q).  b: [2n]. */
void orc_source(int64_t n, const double* cen, const double* nrm, int64_t nc, const double* chg,
                double eps1, double* b) {
  int64_t i;
#pragma omp parallel for schedule(static)
  for (i = 0; i < n; ++i) {
    double s1 = 0.0, s2 = 0.0;
    for (int64_t k = 0; k < nc; ++k) {
      const double* yk = chg + 4 * k;
      double q = yk[3];
      s1 += q * orc_G0(cen + 3 * i, yk);
      s2 += q * orc_dG0_dnx(cen + 3 * i, nrm + 3 * i, yk);
    }
    b[i] = s1 / eps1;
    b[i + n] = s2 / eps1;
  }
}

/* ------------------------------ Eqs. (12)-(13): {Au}_i, {Au}_{i+N} */
static void matvec_row(int64_t n, const double* cen, const double* nrm, const double* area, double eps,
                       double kappa, const double* u, int64_t i, double* yi, double* yiN) {
  double s1 = 0.0, s2 = 0.0, K[4];
  for (int64_t j = 0; j < n; ++j) {
    if (j == i) continue; /* singular self term simply removed */
    orc_kernels(cen + 3 * i, nrm + 3 * i, cen + 3 * j, nrm + 3 * j, eps, kappa, K);
    s1 += area[j] * (K[0] * u[j + n] + K[1] * u[j]);
    s2 += area[j] * (K[2] * u[j + n] + K[3] * u[j]);
  }
  *yi = 0.5 * (1.0 + eps) * u[i] - s1;
  *yiN = 0.5 * (1.0 + 1.0 / eps) * u[i + n] - s2;
}

/* Full product y = A u (y: [2n]). */
void orc_matvec(int64_t n, const double* cen, const double* nrm, const double* area, double eps,
                double kappa, const double* u, double* y) {
  int64_t i;
#pragma omp parallel for schedule(static)
  for (i = 0; i < n; ++i) matvec_row(n, cen, nrm, area, eps, kappa, u, i, y + i, y + i + n);
}

/* Selected rows: out[2*t] = {Au}_{rows[t]}, out[2*t+1] = {Au}_{rows[t]+N}. */
void orc_matvec_rows(int64_t n, const double* cen, const double* nrm, const double* area, double eps,
                     double kappa, const double* u, int64_t nrows, const int64_t* rows, double* out) {
  int64_t t;
#pragma omp parallel for schedule(static)
  for (t = 0; t < nrows; ++t) matvec_row(n, cen, nrm, area, eps, kappa, u, rows[t], out + 2 * t, out + 2 * t + 1);
}

/* Explicit dense 2N x 2N matrix A (row-major), the test oracle of SPEC.md S:205-213. */
void orc_dense_assemble(int64_t n, const double* cen, const double* nrm, const double* area, double eps,
                        double kappa, double* A) {
  int64_t m = 2 * n, i;
  memset(A, 0, sizeof(double) * (size_t)(m * m));
#pragma omp parallel for schedule(static)
  for (i = 0; i < n; ++i) {
    double K[4];
    A[i * m + i] = 0.5 * (1.0 + eps);
    A[(i + n) * m + (i + n)] = 0.5 * (1.0 + 1.0 / eps);
    for (int64_t j = 0; j < n; ++j) {
      if (j == i) continue;
      orc_kernels(cen + 3 * i, nrm + 3 * i, cen + 3 * j, nrm + 3 * j, eps, kappa, K);
      A[i * m + (j + n)] = -area[j] * K[0];
      A[i * m + j] = -area[j] * K[1];
      A[(i + n) * m + (j + n)] = -area[j] * K[2];
      A[(i + n) * m + j] = -area[j] * K[3];
    }
  }
}

/* -------------------------------------------------- GMRES(m) */
typedef void (*orc_op_fn)(void* ctx, const double* x, double* y);

typedef struct {
  int64_t iterations, restarts, matvecs, converged;
  double rel_res_est, rel_res_true;
  double* history; /* caller-owned, may be NULL */
  int64_t history_cap, history_len;
} orc_report;

static double nrm2(int64_t m, const double* v) {
  double s = 0.0;
  for (int64_t i = 0; i < m; ++i) s += v[i] * v[i];
  return sqrt(s);
}
static double dotv(int64_t m, const double* a, const double* b) {
  double s = 0.0;
  for (int64_t i = 0; i < m; ++i) s += a[i] * b[i];
  return s;
}

/* Solve op(x) = b for x (length m); x holds x0 on entry. Returns 0 converged, 2 not.
 * minv != NULL: right-preconditioned GMRES with M = diag(1 / minv) (Saad, Iterative Methods for
 * Sparse Linear Systems, Algorithm 9.5): z_k = M^-1 v_k, w = op(z_k), ...; x = x0 + M^-1 (V y).
 * The residual the convergence test uses is still b - op(x) (right preconditioning leaves it
 * unchanged).  minv == NULL: plain GMRES as the paper. */
static int gmres_core(orc_op_fn op, void* ctx, int64_t m, const double* b, double* x, int64_t restart,
                      double tol, int64_t max_iters, int64_t check_true, const double* minv, orc_report* rep) {
  double* V = (double*)malloc(sizeof(double) * (size_t)(m * (restart + 1)));
  double* H = (double*)calloc((size_t)((restart + 1) * restart), sizeof(double)); /* H[i*restart+k] */
  double* cs = (double*)calloc((size_t)restart, sizeof(double));
  double* sn = (double*)calloc((size_t)restart, sizeof(double));
  double* g = (double*)calloc((size_t)(restart + 1), sizeof(double));
  double* yv = (double*)calloc((size_t)restart, sizeof(double));
  double* r = (double*)malloc(sizeof(double) * (size_t)m);
  double* z = minv ? (double*)malloc(sizeof(double) * (size_t)m) : NULL;
  int64_t its = 0, restarts = 0, matvecs = 0, converged = 0, hl = 0;
  double rel = 1.0;
  double beta_b = nrm2(m, b);
  rep->rel_res_true = -1.0;
  if (beta_b == 0.0) { /* b = 0 => x = 0 (R17) */
    for (int64_t i = 0; i < m; ++i) x[i] = 0.0;
    rep->iterations = 0; rep->restarts = 0; rep->matvecs = 0; rep->converged = 1;
    rep->rel_res_est = 0.0; rep->rel_res_true = 0.0; rep->history_len = 0;
    free(V); free(H); free(cs); free(sn); free(g); free(yv); free(r); free(z);
    return 0;
  }
  int first_cycle = 1;
  for (;;) {
    /* r = b - A x (x = 0 => r = b without a matvec) */
    int x_is_zero = 1;
    for (int64_t i = 0; i < m; ++i) if (x[i] != 0.0) { x_is_zero = 0; break; }
    if (x_is_zero) {
      memcpy(r, b, sizeof(double) * (size_t)m);
    } else {
      op(ctx, x, r);
      ++matvecs;
      for (int64_t i = 0; i < m; ++i) r[i] = b[i] - r[i];
    }
    if (!first_cycle) ++restarts;
    first_cycle = 0;
    double beta = nrm2(m, r);
    rel = beta / beta_b;
    if (rel <= tol) { converged = 1; break; }
    if (its >= max_iters) break;
    for (int64_t i = 0; i < m; ++i) V[i] = r[i] / beta;
    for (int64_t i = 0; i <= restart; ++i) g[i] = 0.0;
    g[0] = beta;
    int64_t k, kdone = 0;
    int stop = 0;
    for (k = 0; k < restart; ++k) {
      double* w = V + (k + 1) * m;
      if (minv) {
        for (int64_t t = 0; t < m; ++t) z[t] = minv[t] * V[k * m + t];
        op(ctx, z, w);
      } else {
        op(ctx, V + k * m, w);
      }
      ++matvecs;
      ++its;
      for (int64_t i = 0; i <= k; ++i) { /* modified Gram-Schmidt */
        double h = dotv(m, w, V + i * m);
        H[i * restart + k] = h;
        for (int64_t t = 0; t < m; ++t) w[t] -= h * V[i * m + t];
      }
      double hk1 = nrm2(m, w);
      H[(k + 1) * restart + k] = hk1;
      for (int64_t i = 0; i < k; ++i) { /* apply stored rotations to column k */
        double a = H[i * restart + k], c = H[(i + 1) * restart + k];
        H[i * restart + k] = cs[i] * a + sn[i] * c;
        H[(i + 1) * restart + k] = -sn[i] * a + cs[i] * c;
      }
      double a = H[k * restart + k], c = H[(k + 1) * restart + k];
      double delta = hypot(a, c);
      cs[k] = a / delta;
      sn[k] = c / delta;
      H[k * restart + k] = delta;
      H[(k + 1) * restart + k] = 0.0;
      g[k + 1] = -sn[k] * g[k];
      g[k] = cs[k] * g[k];
      kdone = k + 1;
      rel = fabs(g[k + 1]) / beta_b;
      if (rep->history && hl < rep->history_cap) rep->history[hl] = rel;
      ++hl;
      if (hk1 <= 1e-14 * beta_b) { stop = 1; break; } /* happy breakdown */
      for (int64_t t = 0; t < m; ++t) w[t] /= hk1;
      if (rel <= tol || its >= max_iters) { stop = 1; break; }
    }
    (void)stop;
    /* back substitution H[0:k,0:k] y = g[0:k]; x += V y (warm restart) */
    for (int64_t i = kdone - 1; i >= 0; --i) {
      double s = g[i];
      for (int64_t j = i + 1; j < kdone; ++j) s -= H[i * restart + j] * yv[j];
      yv[i] = s / H[i * restart + i];
    }
    if (minv) { /* x += M^-1 (V y) */
      for (int64_t t = 0; t < m; ++t) {
        double s = 0.0;
        for (int64_t j = 0; j < kdone; ++j) s += yv[j] * V[j * m + t];
        x[t] += minv[t] * s;
      }
    } else {
      for (int64_t j = 0; j < kdone; ++j)
        for (int64_t t = 0; t < m; ++t) x[t] += yv[j] * V[j * m + t];
    }
    if (rel <= tol) { converged = 1; break; }
    if (its >= max_iters) break;
  }
  if (check_true) { /* one extra product: ||b - A x|| / ||b|| */
    op(ctx, x, r);
    ++matvecs;
    for (int64_t i = 0; i < m; ++i) r[i] = b[i] - r[i];
    rep->rel_res_true = nrm2(m, r) / beta_b;
  }
  rep->iterations = its;
  rep->restarts = restarts;
  rep->matvecs = matvecs;
  rep->converged = converged;
  rep->rel_res_est = rel;
  rep->history_len = hl;
  free(V); free(H); free(cs); free(sn); free(g); free(yv); free(r); free(z);
  return converged ? 0 : 2;
}

typedef struct { int64_t m; const double* A; } dense_ctx;
static void dense_op(void* vctx, const double* x, double* y) {
  dense_ctx* c = (dense_ctx*)vctx;
  for (int64_t i = 0; i < c->m; ++i) {
    double s = 0.0;
    for (int64_t j = 0; j < c->m; ++j) s += c->A[i * c->m + j] * x[j];
    y[i] = s;
  }
}
/* GMRES on an explicit m x m matrix (SPEC.md S:182-183 examples). */
int orc_gmres_dense(int64_t m, const double* A, const double* b, double* x, int64_t restart, double tol,
                    int64_t max_iters, int64_t check_true, orc_report* rep) {
  dense_ctx c = {m, A};
  return gmres_core(dense_op, &c, m, b, x, restart, tol, max_iters, check_true, NULL, rep);
}
/* The same with right preconditioning M = diag(1 / minv). */
int orc_gmres_dense_prec(int64_t m, const double* A, const double* b, double* x, const double* minv,
                         int64_t restart, double tol, int64_t max_iters, int64_t check_true, orc_report* rep) {
  dense_ctx c = {m, A};
  return gmres_core(dense_op, &c, m, b, x, restart, tol, max_iters, check_true, minv, rep);
}

typedef struct {
  int64_t n; const double *cen, *nrm, *area; double eps, kappa;
} bem_ctx;
static void bem_op(void* vctx, const double* x, double* y) {
  bem_ctx* c = (bem_ctx*)vctx;
  orc_matvec(c->n, c->cen, c->nrm, c->area, c->eps, c->kappa, x, y);
}
/* GMRES on the BEM operator of Eqs. (12)-(13). */
int orc_gmres_bem(int64_t n, const double* cen, const double* nrm, const double* area, double eps,
                  double kappa, const double* b, double* x, int64_t restart, double tol, int64_t max_iters,
                  int64_t check_true, orc_report* rep) {
  bem_ctx c = {n, cen, nrm, area, eps, kappa};
  return gmres_core(bem_op, &c, 2 * n, b, x, restart, tol, max_iters, check_true, NULL, rep);
}
/* The same GMRES (gmres_core, unchanged) with the operator supplied by the caller: a C callback
 * op(ctx, x, y) that must set y = A x.  Used by oracle.gmres_checkpointed, whose callback is
 * orc_matvec behind an on-disk store of the products (so a long full-size solve can be split
 * across several processes and replays bitwise the same arithmetic). */
int orc_gmres_op(int64_t m, orc_op_fn op, void* ctx, const double* b, double* x, int64_t restart, double tol,
                 int64_t max_iters, int64_t check_true, orc_report* rep) {
  return gmres_core(op, ctx, m, b, x, restart, tol, max_iters, check_true, NULL, rep);
}
/* GMRES on the BEM operator, right-preconditioned by the diagonal of the jump terms of
 * Eqs. (12)-(13): M = diag(1/2 (1 + eps) I_N, 1/2 (1 + 1/eps) I_N) (not in the paper; the
 * library's opt-in bipb_set_precond(ctx, 1)).  Same linear system, same residual test. */
int orc_gmres_bem_jacobi(int64_t n, const double* cen, const double* nrm, const double* area, double eps,
                         double kappa, const double* b, double* x, int64_t restart, double tol, int64_t max_iters,
                         int64_t check_true, orc_report* rep) {
  bem_ctx c = {n, cen, nrm, area, eps, kappa};
  double* minv = (double*)malloc(sizeof(double) * (size_t)(2 * n));
  for (int64_t i = 0; i < n; ++i) {
    minv[i] = 1.0 / (0.5 * (1.0 + eps));
    minv[n + i] = 1.0 / (0.5 * (1.0 + 1.0 / eps));
  }
  int st = gmres_core(bem_op, &c, 2 * n, b, x, restart, tol, max_iters, check_true, minv, rep);
  free(minv);
  return st;
}

/* ---------------------- Eq. (14): phi_reac(x_k) and E_sol (reading R3) */
/* K1(x_k, x_j) and K2(x_k, x_j) use only the source normal nu_j (no normal at a charge). */
void orc_reaction_potential(int64_t n, const double* cen, const double* nrm, const double* area, double eps,
                            double kappa, int64_t nc, const double* chg, const double* x, double* phi) {
  int64_t k;
#pragma omp parallel for schedule(static)
  for (k = 0; k < nc; ++k) {
    const double* yk = chg + 4 * k;
    double s = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      double K1 = orc_G0(yk, cen + 3 * j) - orc_Gk(yk, cen + 3 * j, kappa);
      double K2 = eps * orc_dGk_dny(yk, cen + 3 * j, nrm + 3 * j, kappa) - orc_dG0_dny(yk, cen + 3 * j, nrm + 3 * j);
      s += area[j] * (K1 * x[j + n] + K2 * x[j]);
    }
    phi[k] = s;
  }
}

/* E_sol = 1/2 * 4 pi * C_E * sum_k Q_k phi_reac(x_k)   [kcal/mol], C_E = 332.0716 */
double orc_energy(int64_t n, const double* cen, const double* nrm, const double* area, double eps, double kappa,
                  int64_t nc, const double* chg, const double* x, double* phi_out /* nc or NULL */) {
  double* phi = (double*)malloc(sizeof(double) * (size_t)(nc > 0 ? nc : 1));
  orc_reaction_potential(n, cen, nrm, area, eps, kappa, nc, chg, x, phi);
  double s = 0.0;
  for (int64_t k = 0; k < nc; ++k) s += chg[4 * k + 3] * phi[k];
  if (phi_out) memcpy(phi_out, phi, sizeof(double) * (size_t)nc);
  free(phi);
  return 0.5 * 4.0 * ORC_PI * 332.0716 * s;
}
