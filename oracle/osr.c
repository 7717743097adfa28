/*
 * osr.c - CPU oracle of the SINGLE-REDUCTION BiCGStab schedule ("SR").
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Plain and slow on purpose.
 *
 * What it computes.  Alg. 1 needs three global reductions
 * per iteration (alpha l.177, omega l.180, beta l.183); the paper notes it did
 * NOT use a communication-hiding variant.  The SR schedule is
 * the same iteration rearranged so that ONE sweep over the mesh and ONE
 * reduction serve a whole iteration (reading R19):
 *
 *   with q_i := A r_i and y_i := A v_i (v_i = A p_i, Alg. 1's s_i), l.178-179 give
 *     s_i = r_i - alpha_i v_i            t_i = A s_i = q_i - alpha_i y_i
 *   so (t,s), (t,t) and (rhat, r_{i+1}) expand bilinearly into inner products
 *   of r_i, v_i, q_i, y_i, rhat, all available after the sweep that made them:
 *     (t,s)  = (q,r) - a (q,v) - a (y,r) + a^2 (y,v)
 *     (t,t)  = (q,q) - 2a (q,y) + a^2 (y,y)
 *     (rhat,r_{i+1}) = (rhat,s) - w (rhat,t) = rho - a sigma - w ((rhat,q) - a (rhat,y))
 *
 *   sweep i (scalars alpha_{i-1}, omega_{i-1}, beta_{i-1}; all 0 for i = 0):
 *     s  = r - alpha v                    (l.178)
 *     t  = q - alpha y                    (= A s, l.179)
 *     x  = (x + alpha p) + omega s        (l.181, R2)
 *     r  = s - omega t                    (l.182)
 *     p  = r + beta (p - omega v)         (l.184)
 *     v  = A p;  q = A r;  y = A v        (l.176 and the two products above)
 *     dots[0..11] = (rh,v) (rh,r) (rh,q) (rh,y) (q,r) (q,v) (y,r) (y,v)
 *                   (q,q) (q,y) (y,y) (r,r)
 *   then the scalar step: hist_i = sqrt((r,r))/||b||, alpha_i = (rh,r)/(rh,v)
 *   (l.177, rho taken from the direct inner product every sweep, so no
 *   scalar recurrence accumulates), omega_i from the expansions (l.180),
 *   beta_i = (rho_{i+1}/rho_i)(alpha_i/omega_i) (l.183).
 *
 * In exact arithmetic the iterates equal Alg. 1's; tests/test_oracle_sr.py pins
 * this file against the (separately pinned) classic oracle o64_bicgstab, the
 * LAPACK solve and closed-form special cases.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static int sr_on_event(int code, int i, double tol, int *ev, int *ev_it) {
  if (*ev < 0) {
    *ev = code;
    *ev_it = i;
  }
  return tol > 0.0;
}

/* ============================== fp64 (O64-SR) ============================== */

void o64_sr_sweep(int nx, int ny, int nz, const double *const c[6], double alpha,
                  double omega, double beta, const double *rh, double *x,
                  double *r, double *p, double *v, double *q, double *y,
                  double dots[12]) {
  int64_t n = (int64_t)nx * ny * nz;
  for (int64_t P = 0; P < n; ++P) {
    double s = r[P] - alpha * v[P];          /* l.178 */
    double t = q[P] - alpha * y[P];          /* A s (l.179) */
    x[P] = (x[P] + alpha * p[P]) + omega * s; /* l.181 */
    r[P] = s - omega * t;                    /* l.182 */
    p[P] = r[P] + beta * (p[P] - omega * v[P]); /* l.184 */
  }
  o64_apply(nx, ny, nz, c, p, v);            /* l.176: v = A p */
  o64_apply(nx, ny, nz, c, r, q);            /* q = A r */
  o64_apply(nx, ny, nz, c, v, y);            /* y = A v */
  const double *a[12] = {rh, rh, rh, rh, q, q, y, y, q, q, y, r};
  const double *b[12] = {v, r, q, y, r, v, r, v, q, y, y, r};
  for (int d = 0; d < 12; ++d) dots[d] = o64_dot(n, a[d], b[d]);
}

int o64_sr_bicgstab(int nx, int ny, int nz, const double *const c[6],
                    const double *b, const double *x0, double tol, int maxit,
                    double *x, double *hist, double *alpha_out, double *omega_out,
                    int *status, int *event_it) {
  int64_t n = (int64_t)nx * ny * nz;
  size_t bytes = sizeof(double) * (size_t)(n > 0 ? n : 1);
  double *r = (double *)malloc(bytes), *rh = (double *)malloc(bytes);
  double *p = (double *)malloc(bytes), *v = (double *)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
  double *q = (double *)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
  double *y = (double *)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
  int ev = -1, ev_it = 0, it = 0;

  if (x0) { /* R1: r0 = b - A x0 */
    memcpy(x, x0, bytes);
    o64_apply(nx, ny, nz, c, x, q);
    for (int64_t P = 0; P < n; ++P) r[P] = b[P] - q[P];
    memset(q, 0, bytes);
  } else { /* Alg. 1 l.174 */
    for (int64_t P = 0; P < n; ++P) {
      x[P] = 0.0;
      r[P] = b[P];
    }
  }
  memcpy(rh, r, bytes);
  memcpy(p, r, bytes); /* p0 = r0; sweep 0 (beta = 0) reproduces it */
  double nb = sqrt(o64_dot(n, b, b));
  if (nb == 0.0) {
    for (int64_t P = 0; P < n; ++P) x[P] = 0.0;
    hist[0] = 0.0;
    *status = ORC_CONVERGED;
    *event_it = 0;
    goto done;
  }
  double alpha = 0.0, omega = 0.0, beta = 0.0, dots[12];
  for (int i = 0; i <= maxit; ++i) {
    o64_sr_sweep(nx, ny, nz, c, alpha, omega, beta, rh, x, r, p, v, q, y, dots);
    const double sigma = dots[0], rho = dots[1], phi = dots[2], psi = dots[3];
    const double qr = dots[4], qv = dots[5], yr = dots[6], yv = dots[7];
    const double qq = dots[8], qy = dots[9], yy = dots[10], rr = dots[11];
    hist[i] = sqrt(rr) / nb; /* R4: ||r_i|| / ||b|| */
    it = i;
    int code = -1;
    if (!isfinite(rr) || !isfinite(rho)) code = ORC_NONFINITE;
    else if (rr == 0.0 && rho != 0.0) code = ORC_BREAKDOWN; /* R23: (r,r) underflowed, r != 0 */
    else if (rr == 0.0 || (tol > 0.0 && hist[i] <= tol)) code = ORC_CONVERGED;
    else if (i > 0 && (omega == 0.0 || rho == 0.0)) code = ORC_BREAKDOWN;
    if (code >= 0 && sr_on_event(code, i, tol, &ev, &ev_it)) break;
    if (i == maxit) break;
    /* iteration i+1 of Alg. 1 */
    alpha = rho / sigma; /* l.177 */
    if (sigma == 0.0 || !isfinite(alpha)) {
      alpha = 0.0;
      if (sr_on_event(isfinite(sigma) ? ORC_BREAKDOWN : ORC_NONFINITE, i + 1, tol, &ev, &ev_it)) break;
    }
    double ts = ((qr - alpha * qv) - alpha * yr) + (alpha * alpha) * yv;
    double tt = (qq - (2.0 * alpha) * qy) + (alpha * alpha) * yy;
    omega = 0.0; /* tt <= 0: t = A s = 0, so s = 0 (R8) */
    if (tt > 0.0) {
      omega = ts / tt; /* l.180 */
      if (!isfinite(omega)) {
        omega = 0.0;
        if (sr_on_event(ORC_NONFINITE, i + 1, tol, &ev, &ev_it)) break;
      }
    }
    double rhon = (rho - alpha * sigma) - omega * (phi - alpha * psi);
    beta = (rhon / rho) * (alpha / omega); /* l.183 */
    if (!isfinite(beta)) beta = 0.0;
    if (alpha_out) alpha_out[i + 1] = alpha;
    if (omega_out) omega_out[i + 1] = omega;
  }
  *status = ev >= 0 ? ev : ORC_MAXIT;
  *event_it = ev_it;
done:
  free(r); free(rh); free(p); free(v); free(q); free(y);
  return it;
}

/* ====================== fp16 mixed mirror (O16-SR) ========================= */
/* Every vector op is one fp16 FMAC (R11), in the GPU kernel's order:
 *   s = fma(-a, v, r); t = fma(-a, y, q); x = fma(w, s, fma(a, p, x));
 *   r = fma(-w, t, s); p = fma(b, fma(-w, v, p), r)
 * SpMVs as o16_apply_fused; inner products as o16_dot (fp16 products exact
 * in fp32, fp32 sums); scalars in fp32 (R12). */

static uint16_t sr_neg16(uint16_t a) { return a ^ 0x8000; }
static uint16_t sr_rn16f(float x) { return o16_from_double((double)x); }
static int sr_usable16(float s) {
  uint16_t h = sr_rn16f(s);
  return isfinite(s) && ((h >> 10) & 31) != 31;
}

/* ---- half dots (R22, the "16-bit mode" of
 * the paper's unpublished performance model) ----
 * The CS-1 PE forms its core-local part of a dot over its z pencil
 * (PAPER.md:394); in 16-bit mode that running sum is fp16: one fp16 FMAC per
 * point, acc = fma16(a, b, acc), z ascending from +0.  The pencil of column
 * (i, j) is cut into the z segments [seg[s], seg[s+1]) (the last one ends at
 * nz); the AllReduce stays 32-bit: here the segment sums are
 * added exactly in fp64 (*sum) -- the GPU adds them in fp32 in its own order,
 * a difference bounded by the fp32 rounding of that sum, for which *abs (the
 * sum of |segment sums|) is the scale. */
void o16h_dot(int nx, int ny, int nz, const uint16_t *a, const uint16_t *b, int nseg,
              const int *seg, double *sum, double *abs) {
  double t = 0.0, ta = 0.0;
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i)
      for (int sgi = 0; sgi < nseg; ++sgi) {
        const int z0 = seg[sgi], z1 = sgi + 1 < nseg ? seg[sgi + 1] : nz;
        uint16_t acc = 0; /* +0 */
        for (int k = z0; k < z1; ++k) {
          const int64_t P = (int64_t)i + (int64_t)nx * ((int64_t)j + (int64_t)ny * k);
          acc = o16_fma(a[P], b[P], acc);
        }
        const double d = o16_to_double(acc);
        t += d;
        ta += fabs(d);
      }
  *sum = t;
  if (abs) *abs = ta;
}

/* the twelve sums of a sweep: mixed (o16_dot) or, nseg > 0, half pencils
 * over the segments, rounded once to fp32 (dabs: their scales, may be NULL) */
static void sr16_dots(int nx, int ny, int nz, const uint16_t *const a[12], const uint16_t *const b[12],
                      int nseg, const int *seg, float dots[12], double *dabs) {
  for (int d = 0; d < 12; ++d) {
    if (nseg > 0) {
      double sm, ab;
      o16h_dot(nx, ny, nz, a[d], b[d], nseg, seg, &sm, &ab);
      dots[d] = (float)sm;
      if (dabs) dabs[d] = ab;
    } else {
      dots[d] = o16_dot(nx, ny, nz, a[d], b[d]);
      if (dabs) dabs[d] = 0.0;
    }
  }
}

void o16h_sr_sweep(int nx, int ny, int nz, const uint16_t *const c[6], float alpha,
                   float omega, float beta, const uint16_t *rh, uint16_t *x,
                   uint16_t *r, uint16_t *p, uint16_t *v, uint16_t *q, uint16_t *y,
                   int nseg, const int *seg, float dots[12], double dabs[12]) {
  int64_t n = (int64_t)nx * ny * nz;
  const uint16_t ah = sr_rn16f(alpha), wh = sr_rn16f(omega), bh = sr_rn16f(beta);
  for (int64_t P = 0; P < n; ++P) {
    uint16_t s = o16_fma(sr_neg16(ah), v[P], r[P]);
    uint16_t t = o16_fma(sr_neg16(ah), y[P], q[P]);
    x[P] = o16_fma(wh, s, o16_fma(ah, p[P], x[P]));
    r[P] = o16_fma(sr_neg16(wh), t, s);
    p[P] = o16_fma(bh, o16_fma(sr_neg16(wh), v[P], p[P]), r[P]);
  }
  o16_apply_fused(nx, ny, nz, c, p, v);
  o16_apply_fused(nx, ny, nz, c, r, q);
  o16_apply_fused(nx, ny, nz, c, v, y);
  const uint16_t *const a[12] = {rh, rh, rh, rh, q, q, y, y, q, q, y, r};
  const uint16_t *const b[12] = {v, r, q, y, r, v, r, v, q, y, y, r};
  sr16_dots(nx, ny, nz, a, b, nseg, seg, dots, dabs);
}

void o16_sr_sweep(int nx, int ny, int nz, const uint16_t *const c[6], float alpha,
                  float omega, float beta, const uint16_t *rh, uint16_t *x,
                  uint16_t *r, uint16_t *p, uint16_t *v, uint16_t *q, uint16_t *y,
                  float dots[12]) {
  o16h_sr_sweep(nx, ny, nz, c, alpha, omega, beta, rh, x, r, p, v, q, y, 0, NULL, dots, NULL);
}

/* The fp32 scalar step shared by the two fp32-scalar mirrors below.  Written
 * operation by operation (compiled with -ffp-contract=off: no FMA contraction). */
static float sr_omega32(const float *dots, float alpha, int *nonfinite) {
  const float qr = dots[4], qv = dots[5], yr = dots[6], yv = dots[7];
  const float qq = dots[8], qy = dots[9], yy = dots[10];
  const float a2 = alpha * alpha;
  const float ts = ((qr - alpha * qv) - alpha * yr) + a2 * yv;
  const float tt = (qq - (2.0f * alpha) * qy) + a2 * yy;
  *nonfinite = 0;
  if (!(tt > 0.0f)) {
    if (!isfinite(tt)) *nonfinite = 1;
    return 0.0f;
  }
  return ts / tt;
}

/* O16-SR with half dots over the segments seg[0..nseg) (nseg = 0: mixed dots,
 * = o16_sr_bicgstab).  ||b|| stays a mixed dot (setup, not an iteration op). */
int o16h_sr_bicgstab(int nx, int ny, int nz, const uint16_t *const c[6],
                     const uint16_t *b, const uint16_t *x0, double tol, int maxit,
                     int nseg, const int *seg,
                     uint16_t *x, double *hist, float *alpha_out, float *omega_out,
                     int *status, int *event_it) {
  int64_t n = (int64_t)nx * ny * nz;
  size_t bytes = sizeof(uint16_t) * (size_t)(n > 0 ? n : 1);
  uint16_t *r = (uint16_t *)malloc(bytes), *rh = (uint16_t *)malloc(bytes);
  uint16_t *p = (uint16_t *)malloc(bytes), *v = (uint16_t *)calloc((size_t)(n > 0 ? n : 1), 2);
  uint16_t *q = (uint16_t *)calloc((size_t)(n > 0 ? n : 1), 2);
  uint16_t *y = (uint16_t *)calloc((size_t)(n > 0 ? n : 1), 2);
  int ev = -1, ev_it = 0, it = 0;

  if (x0) { /* R1 */
    memcpy(x, x0, bytes);
    o16_apply_fused(nx, ny, nz, c, x, q);
    for (int64_t P = 0; P < n; ++P) r[P] = o16_add(b[P], sr_neg16(q[P]));
    memset(q, 0, bytes);
  } else {
    for (int64_t P = 0; P < n; ++P) {
      x[P] = 0;
      r[P] = b[P];
    }
  }
  memcpy(rh, r, bytes);
  memcpy(p, r, bytes);
  double nb = sqrt((double)o16_dot(nx, ny, nz, b, b));
  if (nb == 0.0) {
    for (int64_t P = 0; P < n; ++P) x[P] = 0;
    hist[0] = 0.0;
    *status = ORC_CONVERGED;
    *event_it = 0;
    goto done;
  }
  float alpha = 0.0f, omega = 0.0f, beta = 0.0f, dots[12];
  for (int i = 0; i <= maxit; ++i) {
    o16h_sr_sweep(nx, ny, nz, c, alpha, omega, beta, rh, x, r, p, v, q, y, nseg, seg, dots, NULL);
    const float sigma = dots[0], rho = dots[1], phi = dots[2], psi = dots[3], rr = dots[11];
    hist[i] = sqrt((double)rr) / nb;
    it = i;
    int code = -1;
    if (!isfinite(rr) || !isfinite(rho)) code = ORC_NONFINITE;
    else if (rr == 0.0f && rho != 0.0f) code = ORC_BREAKDOWN; /* R23: (r,r) underflowed, r != 0 */
    else if (rr == 0.0f || (tol > 0.0 && hist[i] <= tol)) code = ORC_CONVERGED;
    else if (i > 0 && (omega == 0.0f || rho == 0.0f)) code = ORC_BREAKDOWN;
    if (code >= 0 && sr_on_event(code, i, tol, &ev, &ev_it)) break;
    if (i == maxit) break;
    alpha = rho / sigma;
    if (sigma == 0.0f || !sr_usable16(alpha)) {
      alpha = 0.0f;
      if (sr_on_event(isfinite(sigma) ? ORC_BREAKDOWN : ORC_NONFINITE, i + 1, tol, &ev, &ev_it)) break;
    }
    int nf = 0;
    omega = sr_omega32(dots, alpha, &nf);
    if (nf || !sr_usable16(omega)) {
      omega = 0.0f;
      if (sr_on_event(ORC_NONFINITE, i + 1, tol, &ev, &ev_it)) break;
    }
    float rhon = (rho - alpha * sigma) - omega * (phi - alpha * psi);
    beta = (rhon / rho) * (alpha / omega);
    if (!sr_usable16(beta)) beta = 0.0f;
    if (alpha_out) alpha_out[i + 1] = alpha;
    if (omega_out) omega_out[i + 1] = omega;
  }
  *status = ev >= 0 ? ev : ORC_MAXIT;
  *event_it = ev_it;
done:
  free(r); free(rh); free(p); free(v); free(q); free(y);
  return it;
}

int o16_sr_bicgstab(int nx, int ny, int nz, const uint16_t *const c[6],
                    const uint16_t *b, const uint16_t *x0, double tol, int maxit,
                    uint16_t *x, double *hist, float *alpha_out, float *omega_out,
                    int *status, int *event_it) {
  return o16h_sr_bicgstab(nx, ny, nz, c, b, x0, tol, maxit, 0, NULL, x, hist, alpha_out, omega_out, status,
                          event_it);
}

/* ====================== fp32 mirror (vector ops only) ====================== */
/* The fp32 GPU path's element-wise order: fmaf (one rounding) per AXPY term,
 * SpMVs as o32_apply_fma.  Inner products in fp64 here (the GPU's fp32 sums
 * are compared with a tolerance, R13). */
void o32_sr_sweep(int nx, int ny, int nz, const float *const c[6], float alpha,
                  float omega, float beta, const float *rh, float *x, float *r,
                  float *p, float *v, float *q, float *y, double dots[12]) {
  int64_t n = (int64_t)nx * ny * nz;
  for (int64_t P = 0; P < n; ++P) {
    float s = fmaf(-alpha, v[P], r[P]);
    float t = fmaf(-alpha, y[P], q[P]);
    x[P] = fmaf(omega, s, fmaf(alpha, p[P], x[P]));
    r[P] = fmaf(-omega, t, s);
    p[P] = fmaf(beta, fmaf(-omega, v[P], p[P]), r[P]);
  }
  o32_apply_fma(nx, ny, nz, c, p, v);
  o32_apply_fma(nx, ny, nz, c, r, q);
  o32_apply_fma(nx, ny, nz, c, v, y);
  const float *a[12] = {rh, rh, rh, rh, q, q, y, y, q, q, y, r};
  const float *b[12] = {v, r, q, y, r, v, r, v, q, y, y, r};
  for (int d = 0; d < 12; ++d) {
    double s = 0.0;
    for (int64_t P = 0; P < n; ++P) s += (double)a[d][P] * (double)b[d][P];
    dots[d] = s;
  }
}
