/*
 * o16.c - IEEE binary16 primitives and the mixed-precision ("O16") oracle.
 * TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * The paper's mixed mode ("16-bit for all arithmetic except the
 * inner products and a mixed precision inner product with 16-bit multiply and
 * 32-bit add"; PAPER.md:116-118 fp16 FMAC "with no rounding of the product
 * prior to the add"; "mixed 16-bit multiply/32-bit add
 * precision, and we do the AllReduce at 32-bit precision").
 *
 * binary16 arithmetic is done EXACTLY in integers: every finite fp16 value is
 * an integer multiple of 2^-24, a product of two is a multiple of 2^-48 with
 * magnitude < 2^82, so a*b+c is held exactly in a 128-bit integer and rounded
 * once (round-to-nearest-even, subnormals kept, overflow to +-Inf).  No
 * _Float16 compiler arithmetic and no double-rounding path is involved.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef __int128 i128;
typedef unsigned __int128 u128;

static int bitlen128(u128 m) {
  uint64_t hi = (uint64_t)(m >> 64), lo = (uint64_t)m;
  if (hi) return 128 - __builtin_clzll(hi);
  if (lo) return 64 - __builtin_clzll(lo);
  return 0;
}

/* Round M * 2^E (M > 0) to binary16 magnitude bits, RNE. */
static uint16_t rn16_mag(u128 M, int E) {
  int L = bitlen128(M);
  int e = L - 1 + E;                      /* value in [2^e, 2^(e+1)) */
  int qexp = (e < -14 ? -14 : e) - 10;    /* weight of the last kept bit */
  int shift = qexp - E;
  u128 m;
  if (shift <= 0) {
    m = M << (-shift);                    /* exact */
  } else if (shift >= 128) {
    m = 0;                                /* below half the smallest subnormal */
  } else {
    m = M >> shift;
    u128 rem = M & ((((u128)1) << shift) - 1);
    u128 half = ((u128)1) << (shift - 1);
    if (rem > half || (rem == half && (m & 1))) m += 1;
  }
  if (e < -14) return (uint16_t)m;        /* subnormal; m == 1024 is the min normal */
  if (m == 2048) {
    m = 1024;
    e += 1;
  }
  if (e > 15) return 0x7C00;              /* overflow -> Inf */
  return (uint16_t)(((e + 15) << 10) | (int)(m - 1024));
}

double o16_to_double(uint16_t h) {
  int s = h >> 15, e = (h >> 10) & 31, m = h & 1023;
  double v;
  if (e == 0) v = ldexp((double)m, -24);
  else if (e == 31) v = m ? NAN : INFINITY;
  else v = ldexp((double)(m | 1024), e - 25);
  return s ? -v : v;
}

uint16_t o16_from_double(double x) {
  if (isnan(x)) return 0x7E00;
  uint16_t sign = signbit(x) ? 0x8000 : 0;
  double ax = fabs(x);
  if (isinf(ax)) return sign | 0x7C00;
  if (ax == 0.0) return sign;
  int ex;
  double f = frexp(ax, &ex);               /* ax = f * 2^ex, f in [0.5, 1) */
  uint64_t m = (uint64_t)ldexp(f, 53);     /* exact 53-bit integer */
  return sign | rn16_mag((u128)m, ex - 53);
}

/* value of a finite fp16 as a signed integer multiple of 2^-24 */
static int64_t units24(uint16_t h) {
  int e = (h >> 10) & 31, m = h & 1023;
  int64_t a = (e == 0) ? (int64_t)m : ((int64_t)(m | 1024) << (e - 1));
  return (h & 0x8000) ? -a : a;
}

static int finite16(uint16_t h) { return ((h >> 10) & 31) != 31; }

uint16_t o16_fma(uint16_t a, uint16_t b, uint16_t c) {
  if (!finite16(a) || !finite16(b) || !finite16(c)) {
    /* IEEE special cases: Inf/NaN results are exact in binary16 */
    return o16_from_double(fma(o16_to_double(a), o16_to_double(b), o16_to_double(c)));
  }
  int64_t A = units24(a), B = units24(b), C = units24(c);
  i128 N = (i128)A * (i128)B + (((i128)C) << 24); /* exact, units of 2^-48 */
  if (N == 0) {
    /* exact zero: (+-0)+(+-0) keeps the common sign, else +0 under RNE */
    int prod_neg = ((a ^ b) & 0x8000) != 0, c_neg = (c & 0x8000) != 0;
    if ((A == 0 || B == 0) && C == 0) return (prod_neg && c_neg) ? 0x8000 : 0;
    return 0;
  }
  uint16_t sign = N < 0 ? 0x8000 : 0;
  u128 M = N < 0 ? (u128)(-N) : (u128)N;
  return sign | rn16_mag(M, -48);
}

uint16_t o16_add(uint16_t a, uint16_t b) { return o16_fma(0x3C00 /* 1.0 */, a, b); }
uint16_t o16_mul(uint16_t a, uint16_t b) { return o16_fma(a, b, 0x8000 /* -0 */); }

void o16_from_double_array(int64_t n, const double *x, uint16_t *h) {
  for (int64_t i = 0; i < n; ++i) h[i] = o16_from_double(x[i]);
}
void o16_to_double_array(int64_t n, const uint16_t *h, double *x) {
  for (int64_t i = 0; i < n; ++i) x[i] = o16_to_double(h[i]);
}

static uint16_t neg16(uint16_t a) { return a ^ 0x8000; }
static float f16f(uint16_t h) { return (float)o16_to_double(h); } /* exact widening */
static uint16_t rn16f(float x) { return o16_from_double((double)x); }

static int64_t idx3(int nx, int ny, int i, int j, int k) {
  return (int64_t)i + (int64_t)nx * ((int64_t)j + (int64_t)ny * (int64_t)k);
}

/* value of neighbour d (xm,xp,ym,yp,zm,zp) or +0 outside the mesh */
static uint16_t nbv16(int nx, int ny, int nz, const uint16_t *v, int i, int j, int k, int d) {
  switch (d) {
    case 0: return i > 0 ? v[idx3(nx, ny, i - 1, j, k)] : 0;
    case 1: return i + 1 < nx ? v[idx3(nx, ny, i + 1, j, k)] : 0;
    case 2: return j > 0 ? v[idx3(nx, ny, i, j - 1, k)] : 0;
    case 3: return j + 1 < ny ? v[idx3(nx, ny, i, j + 1, k)] : 0;
    case 4: return k > 0 ? v[idx3(nx, ny, i, j, k - 1)] : 0;
    default: return k + 1 < nz ? v[idx3(nx, ny, i, j, k + 1)] : 0;
  }
}

void o16_apply_fused(int nx, int ny, int nz, const uint16_t *const c[6],
                     const uint16_t *v, uint16_t *u) {
#pragma omp parallel for schedule(static)
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        int64_t P = idx3(nx, ny, i, j, k);
        uint16_t acc = v[P];               /* unit diagonal: no multiply */
        for (int d = 0; d < 6; ++d) acc = o16_fma(c[d][P], nbv16(nx, ny, nz, v, i, j, k, d), acc);
        u[P] = acc;
      }
}

void o16_apply_unfused(int nx, int ny, int nz, const uint16_t *const c[6],
                       const uint16_t *v, uint16_t *u) {
#pragma omp parallel for schedule(static)
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        int64_t P = idx3(nx, ny, i, j, k);
        uint16_t acc = v[P];
        for (int d = 0; d < 6; ++d)
          acc = o16_add(acc, o16_mul(c[d][P], nbv16(nx, ny, nz, v, i, j, k, d)));
        u[P] = acc;
      }
}

float o16_dot(int nx, int ny, int nz, const uint16_t *a, const uint16_t *b) {
  float total = 0.0f;
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      float pencil = 0.0f;                 /* one core's Z-long local dot */
      for (int k = 0; k < nz; ++k) {
        int64_t P = idx3(nx, ny, i, j, k);
        pencil += f16f(a[P]) * f16f(b[P]); /* product exact in fp32 */
      }
      total += pencil;                     /* fp32 AllReduce */
    }
  return total;
}

static int on_event(int code, int i, double tol, int *ev, int *ev_it) {
  if (*ev < 0) {
    *ev = code;
    *ev_it = i;
  }
  return tol > 0.0;
}

/* R7 (mixed): the scalars enter fp16 FMACs, so a scalar whose fp16 rounding is
 * +-Inf (|s| >= 65520, the midpoint above the largest finite 65504) is as
 * unusable as an fp32 Inf/NaN. */
static int usable16(float s) { return isfinite(s) && finite16(rn16f(s)); }

/* The iteration's inner products: mixed (o16_dot: exact fp16 products summed in fp32)
 * or, nseg > 0, the half mode's fp16 column pencils over the z segments seg[0..nseg) (o16h_dot,
 * DESIGN.md R22), their exact sum rounded once to fp32. */
static float dot_it(int nx, int ny, int nz, const uint16_t *a, const uint16_t *b, int nseg, const int *seg) {
  if (nseg <= 0) return o16_dot(nx, ny, nz, a, b);
  double sm;
  o16h_dot(nx, ny, nz, a, b, nseg, seg, &sm, NULL);
  return (float)sm;
}

/* O16 (Alg. 1, in binary16) with the iteration's five inner products as half
 * pencils over seg[0..nseg) (nseg = 0: mixed dots, = o16_bicgstab); the setup's rho_0, ||b||,
 * hist[0] stay mixed (R28). */
int o16h_bicgstab(int nx, int ny, int nz, const uint16_t *const c[6],
                  const uint16_t *b, const uint16_t *x0, double tol, int maxit,
                  int unfused, int nseg, const int *seg, uint16_t *x, double *hist, float *alpha_out,
                  float *omega_out, int *status, int *event_it) {
  int64_t n = (int64_t)nx * ny * nz;
  size_t bytes = sizeof(uint16_t) * (size_t)(n > 0 ? n : 1);
  uint16_t *r = (uint16_t *)malloc(bytes), *rh = (uint16_t *)malloc(bytes);
  uint16_t *p = (uint16_t *)malloc(bytes), *v = (uint16_t *)malloc(bytes);
  uint16_t *s = (uint16_t *)malloc(bytes), *t = (uint16_t *)malloc(bytes);
  void (*apply)(int, int, int, const uint16_t *const *, const uint16_t *, uint16_t *) =
      unfused ? o16_apply_unfused : o16_apply_fused;
  int ev = -1, ev_it = 0, it = 0;

  if (x0) { /* R1 */
    memcpy(x, x0, bytes);
    apply(nx, ny, nz, c, x, t);
    for (int64_t P = 0; P < n; ++P) r[P] = o16_add(b[P], neg16(t[P]));
  } else { /* Alg. 1 l.174 */
    for (int64_t P = 0; P < n; ++P) {
      x[P] = 0;
      r[P] = b[P];
    }
  }
  memcpy(rh, r, bytes);
  memcpy(p, r, bytes);
  float rho = o16_dot(nx, ny, nz, rh, r);
  double nb = sqrt((double)o16_dot(nx, ny, nz, b, b));
  if (nb == 0.0) {
    for (int64_t P = 0; P < n; ++P) x[P] = 0;
    hist[0] = 0.0;
    *status = ORC_CONVERGED;
    *event_it = 0;
    goto done;
  }
  hist[0] = sqrt((double)o16_dot(nx, ny, nz, r, r)) / nb;
  if (tol > 0.0 && hist[0] <= tol) {
    *status = ORC_CONVERGED;
    *event_it = 0;
    goto done;
  }
  float alpha = 0.0f, omega = 0.0f, beta = 0.0f;
  for (int i = 1; i <= maxit; ++i) {
    if (i > 1) { /* l.184: p := r + beta (p - omega s), two fp16 FMACs (R11) */
      uint16_t bh = rn16f(beta), mwh = neg16(rn16f(omega));
      for (int64_t P = 0; P < n; ++P) p[P] = o16_fma(bh, o16_fma(mwh, v[P], p[P]), r[P]);
    }
    apply(nx, ny, nz, c, p, v);                       /* l.176 */
    float sigma = dot_it(nx, ny, nz, rh, v, nseg, seg); /* l.177 */
    alpha = rho / sigma;
    if (sigma == 0.0f || !usable16(alpha)) {
      alpha = 0.0f;
      if (on_event(isfinite(sigma) ? ORC_BREAKDOWN : ORC_NONFINITE, i, tol, &ev, &ev_it)) {
        it = i - 1;
        break;
      }
    }
    uint16_t ah = rn16f(alpha);
    for (int64_t P = 0; P < n; ++P) s[P] = o16_fma(neg16(ah), v[P], r[P]); /* l.178 */
    apply(nx, ny, nz, c, s, t);                       /* l.179 */
    float ts = dot_it(nx, ny, nz, t, s, nseg, seg), tt = dot_it(nx, ny, nz, t, t, nseg, seg);
    if (tt == 0.0f) {
      omega = 0.0f;
    } else {
      omega = ts / tt;                                /* l.180 */
      if (!usable16(omega)) {
        omega = 0.0f;
        if (on_event(ORC_NONFINITE, i, tol, &ev, &ev_it)) {
          it = i - 1;
          break;
        }
      }
    }
    uint16_t wh = rn16f(omega);
    for (int64_t P = 0; P < n; ++P) x[P] = o16_fma(wh, s[P], o16_fma(ah, p[P], x[P])); /* l.181 */
    for (int64_t P = 0; P < n; ++P) r[P] = o16_fma(neg16(wh), t[P], s[P]);            /* l.182 */
    float rhon = dot_it(nx, ny, nz, rh, r, nseg, seg), rr = dot_it(nx, ny, nz, r, r, nseg, seg);
    hist[i] = sqrt((double)rr) / nb;
    if (alpha_out) alpha_out[i] = alpha;
    if (omega_out) omega_out[i] = omega;
    it = i;
    int code = -1;
    if (!isfinite(rr) || !isfinite(rhon)) code = ORC_NONFINITE;
    else if (rr == 0.0f && rhon != 0.0f) code = ORC_BREAKDOWN; /* R23: (r,r) underflowed, r != 0 */
    else if (rr == 0.0f || (tol > 0.0 && hist[i] <= tol)) code = ORC_CONVERGED;
    else if (omega == 0.0f || rhon == 0.0f) code = ORC_BREAKDOWN;
    beta = (rhon / rho) * (alpha / omega);            /* l.183, fp32 */
    if (!usable16(beta)) beta = 0.0f;
    rho = rhon;
    if (code >= 0 && on_event(code, i, tol, &ev, &ev_it)) break;
  }
  *status = ev >= 0 ? ev : ORC_MAXIT;
  *event_it = ev_it;
done:
  free(r); free(rh); free(p); free(v); free(s); free(t);
  return it;
}

int o16_bicgstab(int nx, int ny, int nz, const uint16_t *const c[6],
                 const uint16_t *b, const uint16_t *x0, double tol, int maxit,
                 int unfused, uint16_t *x, double *hist, float *alpha_out,
                 float *omega_out, int *status, int *event_it) {
  return o16h_bicgstab(nx, ny, nz, c, b, x0, tol, maxit, unfused, 0, NULL, x, hist, alpha_out, omega_out, status,
                       event_it);
}

/* ---- fp32 mirror of the GPU fp32 SpMV evaluation order ---- */
static float nbv32(int nx, int ny, int nz, const float *v, int i, int j, int k, int d) {
  switch (d) {
    case 0: return i > 0 ? v[idx3(nx, ny, i - 1, j, k)] : 0.0f;
    case 1: return i + 1 < nx ? v[idx3(nx, ny, i + 1, j, k)] : 0.0f;
    case 2: return j > 0 ? v[idx3(nx, ny, i, j - 1, k)] : 0.0f;
    case 3: return j + 1 < ny ? v[idx3(nx, ny, i, j + 1, k)] : 0.0f;
    case 4: return k > 0 ? v[idx3(nx, ny, i, j, k - 1)] : 0.0f;
    default: return k + 1 < nz ? v[idx3(nx, ny, i, j, k + 1)] : 0.0f;
  }
}

void o32_apply_fma(int nx, int ny, int nz, const float *const c[6],
                   const float *v, float *u) {
#pragma omp parallel for schedule(static)
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        int64_t P = idx3(nx, ny, i, j, k);
        float acc = v[P];
        for (int d = 0; d < 6; ++d) acc = fmaf(c[d][P], nbv32(nx, ny, nz, v, i, j, k, d), acc);
        u[P] = acc;
      }
}

/* element-wise array forms (used by the exhaustive / sampled pin tests) */
void o16_fma_array(int64_t n, const uint16_t *a, const uint16_t *b, const uint16_t *c, uint16_t *out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = o16_fma(a[i], b[i], c[i]);
}
/* fp32 fused multiply-add, one rounding (C99 fmaf): the fp32 AXPY primitive of the
 * classic phases' mirrors (R11 in fp32: p' = fma(beta, fma(-omega, v, p), r), s = fma(-alpha, v, r)) */
void o32_fma_array(int64_t n, const float *a, const float *b, const float *c, float *out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = fmaf(a[i], b[i], c[i]);
}
void o16_add_array(int64_t n, const uint16_t *a, const uint16_t *b, uint16_t *out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = o16_add(a[i], b[i]);
}
void o16_mul_array(int64_t n, const uint16_t *a, const uint16_t *b, uint16_t *out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = o16_mul(a[i], b[i]);
}
