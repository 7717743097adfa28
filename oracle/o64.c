/*
 * o64.c - fp64 CPU oracle (O64) for BiCGStab on the Jacobi-scaled 7-point
 * stencil.  TEST INFRASTRUCTURE ONLY (see oracle.h); plain and slow on purpose.
 *
 * Follows /root/reference/PAPER.md:
 *   Algorithm 1 "Standard BiCGStab", PAPER.md:172-186 - line numbers of the
 *   algorithm (l.174 ... l.184) are cited at each step below;
 *   unit diagonal after diagonal preconditioning, PAPER.md:195;
 *   SpMV as the local value plus six coefficient*neighbour products,
 *   PAPER.md:200-201.
 * Readings R1..R13 (paper silent / ambiguous) are listed in DESIGN.md.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* Thread count of the OpenMP loops (timing of the oracle on 1 thread vs all cores). */
void oracle_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

static int64_t idx3(int nx, int ny, int i, int j, int k) {
  return (int64_t)i + (int64_t)nx * ((int64_t)j + (int64_t)ny * (int64_t)k);
}

/* neighbour d in order xm, xp, ym, yp, zm, zp; returns 0 if outside the mesh */
static int neighbour(int nx, int ny, int nz, int i, int j, int k, int d, int64_t *q) {
  int ii = i, jj = j, kk = k;
  switch (d) {
    case 0: ii = i - 1; break;
    case 1: ii = i + 1; break;
    case 2: jj = j - 1; break;
    case 3: jj = j + 1; break;
    case 4: kk = k - 1; break;
    default: kk = k + 1; break;
  }
  if (ii < 0 || ii >= nx || jj < 0 || jj >= ny || kk < 0 || kk >= nz) return 0;
  *q = idx3(nx, ny, ii, jj, kk);
  return 1;
}

/* PAPER.md:195 "with diagonal preconditioning the main diagonal is all ones.
 * Therefore, we only store six other diagonals."  Scaled row P of D^-1 A. */
void o64_jacobi_scale(int nx, int ny, int nz, const double *diag,
                      const double *const off[6], double *const c[6]) {
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        int64_t P = idx3(nx, ny, i, j, k), q;
        for (int d = 0; d < 6; ++d) {
          if (neighbour(nx, ny, nz, i, j, k, d, &q))
            c[d][P] = diag ? off[d][P] / diag[P] : off[d][P];
          else
            c[d][P] = 0.0; /* R5: Dirichlet zero, coupling dropped */
        }
      }
}

/* "The local result of the SpMV is an array u ... computed
 * as the sum of seven vectors.  Six of these are elementwise products of a
 * vector of matrix elements and a vector of iterate elements."  The seventh
 * is the iterate itself (unit diagonal). */
void o64_apply(int nx, int ny, int nz, const double *const c[6],
               const double *v, double *u) {
#pragma omp parallel for schedule(static)
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        int64_t P = idx3(nx, ny, i, j, k), q;
        double s = v[P];
        for (int d = 0; d < 6; ++d)
          if (neighbour(nx, ny, nz, i, j, k, d, &q)) s += c[d][P] * v[q];
        u[P] = s;
      }
}

void o64_apply_raw(int nx, int ny, int nz, const double *diag,
                   const double *const off[6], const double *v, double *u) {
#pragma omp parallel for schedule(static)
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        int64_t P = idx3(nx, ny, i, j, k), q;
        double s = diag[P] * v[P];
        for (int d = 0; d < 6; ++d)
          if (neighbour(nx, ny, nz, i, j, k, d, &q)) s += off[d][P] * v[q];
        u[P] = s;
      }
}

double o64_dot(int64_t n, const double *a, const double *b) {
  double s = 0.0;
  for (int64_t P = 0; P < n; ++P) s += a[P] * b[P];
  return s;
}

double o64_true_residual(int nx, int ny, int nz, const double *const c[6],
                         const double *b, const double *x) {
  int64_t n = (int64_t)nx * ny * nz;
  double *t = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  o64_apply(nx, ny, nz, c, x, t);
  double rr = 0.0, bb = 0.0;
  for (int64_t P = 0; P < n; ++P) {
    double d = b[P] - t[P];
    rr += d * d;
    bb += b[P] * b[P];
  }
  free(t);
  return sqrt(rr) / sqrt(bb);
}

/* R7: first event is recorded; with tol > 0 the solve stops at it. */
static int on_event(int code, int i, double tol, int *ev, int *ev_it) {
  if (*ev < 0) {
    *ev = code;
    *ev_it = i;
  }
  return tol > 0.0;
}

int o64_bicgstab(int nx, int ny, int nz, const double *const c[6],
                 const double *b, const double *x0, double tol, int maxit,
                 double *x, double *hist, double *alpha_out, double *omega_out,
                 int *status, int *event_it) {
  int64_t n = (int64_t)nx * ny * nz;
  size_t bytes = sizeof(double) * (size_t)(n > 0 ? n : 1);
  double *r = (double *)malloc(bytes), *rh = (double *)malloc(bytes);
  double *p = (double *)malloc(bytes), *v = (double *)malloc(bytes);
  double *s = (double *)malloc(bytes), *t = (double *)malloc(bytes);
  int ev = -1, ev_it = 0, it = 0;

  /* Alg. 1 l.174: r0 := b, p0 := r0 (x0 = 0).  R1: general x0. */
  if (x0) {
    memcpy(x, x0, bytes);
    o64_apply(nx, ny, nz, c, x, t);
    for (int64_t P = 0; P < n; ++P) r[P] = b[P] - t[P];
  } else {
    for (int64_t P = 0; P < n; ++P) {
      x[P] = 0.0;
      r[P] = b[P];
    }
  }
  memcpy(rh, r, bytes); /* shadow residual r0 (Alg. 1 uses (r0, .)) */
  memcpy(p, r, bytes);
  double rho = o64_dot(n, rh, r);
  double nb = sqrt(o64_dot(n, b, b));
  if (nb == 0.0) { /* b = 0: x = 0 is exact */
    for (int64_t P = 0; P < n; ++P) x[P] = 0.0;
    hist[0] = 0.0;
    *status = ORC_CONVERGED;
    *event_it = 0;
    goto done;
  }
  hist[0] = sqrt(o64_dot(n, r, r)) / nb; /* R4: recurrence residual / ||b|| */
  if (tol > 0.0 && hist[0] <= tol) {
    *status = ORC_CONVERGED;
    *event_it = 0;
    goto done;
  }
  double alpha = 0.0, omega = 0.0, beta = 0.0;
  for (int i = 1; i <= maxit; ++i) {
    /* Alg. 1 l.184 (of the previous iteration): p := r + beta (p - omega s) */
    if (i > 1)
      for (int64_t P = 0; P < n; ++P) p[P] = r[P] + beta * (p[P] - omega * v[P]);
    o64_apply(nx, ny, nz, c, p, v);                 /* l.176  s_i := A p_i   (v) */
    double sigma = o64_dot(n, rh, v);               /* l.177  (r0, s_i)          */
    alpha = rho / sigma;                            /* l.177  alpha_i            */
    if (sigma == 0.0 || !isfinite(alpha)) {         /* R7 */
      alpha = 0.0;
      if (on_event(isfinite(sigma) ? ORC_BREAKDOWN : ORC_NONFINITE, i, tol, &ev, &ev_it)) {
        it = i - 1;
        break;
      }
    }
    for (int64_t P = 0; P < n; ++P) s[P] = r[P] - alpha * v[P]; /* l.178 q_i (s) */
    o64_apply(nx, ny, nz, c, s, t);                 /* l.179  y_i := A q_i   (t) */
    double ts = o64_dot(n, t, s), tt = o64_dot(n, t, t);
    if (tt == 0.0) {
      omega = 0.0;                                  /* R8: s == 0, lucky exit   */
    } else {
      omega = ts / tt;                              /* l.180 omega_i            */
      if (!isfinite(omega)) {
        omega = 0.0;
        if (on_event(ORC_NONFINITE, i, tol, &ev, &ev_it)) {
          it = i - 1;
          break;
        }
      }
    }
    for (int64_t P = 0; P < n; ++P) x[P] = (x[P] + alpha * p[P]) + omega * s[P]; /* l.181 (R2) */
    for (int64_t P = 0; P < n; ++P) r[P] = s[P] - omega * t[P];                  /* l.182 */
    double rhon = o64_dot(n, rh, r), rr = o64_dot(n, r, r);
    hist[i] = sqrt(rr) / nb;
    if (alpha_out) alpha_out[i] = alpha;
    if (omega_out) omega_out[i] = omega;
    it = i;
    int code = -1;
    if (!isfinite(rr) || !isfinite(rhon)) code = ORC_NONFINITE;
    else if (rr == 0.0 && rhon != 0.0) code = ORC_BREAKDOWN; /* R23: (r,r) underflowed, r != 0 */
    else if (rr == 0.0 || (tol > 0.0 && hist[i] <= tol)) code = ORC_CONVERGED;
    else if (omega == 0.0 || rhon == 0.0) code = ORC_BREAKDOWN;
    beta = (rhon / rho) * (alpha / omega);          /* l.183 beta_i             */
    if (!isfinite(beta)) beta = 0.0;                /* R7 guard                 */
    rho = rhon;
    if (code >= 0 && on_event(code, i, tol, &ev, &ev_it)) break;
  }
  *status = ev >= 0 ? ev : ORC_MAXIT;
  *event_it = ev_it;
done:
  free(r); free(rh); free(p); free(v); free(s); free(t);
  return it;
}
