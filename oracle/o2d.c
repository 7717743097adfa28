/*
 * o2d.c - CPU oracle of the 2D 9-point SpMV.
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Plain and slow on purpose.
 *
 * PAPER.md:362-373, Sec. "SpMV (2D)": "an implementation of SpMV (u = Av as
 * above) for a 9-point stencil in 2D", a rectangular region of the mesh per
 * core, all 9 multiplies and adds of an element done with fused
 * multiply-accumulate, and "most problems will precondition the main diagonal
 * to unity".
 *
 * Mesh nx*ny, P = i + nx*j.  Neighbour order d = 0..7 (row-major over the 3x3
 * window without its centre): (-1,-1) (0,-1) (+1,-1) (-1,0) (+1,0) (-1,+1)
 * (0,+1) (+1,+1) as (dx, dy).  Dirichlet zero: couplings to points outside
 * the mesh are dropped (R5 in 2D).
 */
#include "oracle.h"

#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static const int DX9[8] = {-1, 0, 1, -1, 1, -1, 0, 1};
static const int DY9[8] = {-1, -1, -1, 0, 0, 1, 1, 1};

static int nb9(int nx, int ny, int i, int j, int d, int64_t *q) {
  const int ii = i + DX9[d], jj = j + DY9[d];
  if (ii < 0 || ii >= nx || jj < 0 || jj >= ny) return 0;
  *q = (int64_t)ii + (int64_t)nx * jj;
  return 1;
}

/* c_d[P] = off_d[P] / diag[P] for in-mesh neighbours, +0 otherwise (diag may be NULL) */
void o64_jacobi_scale9(int nx, int ny, const double *diag, const double *const off[8], double *const c[8]) {
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      const int64_t P = (int64_t)i + (int64_t)nx * j;
      int64_t q;
      for (int d = 0; d < 8; ++d)
        c[d][P] = nb9(nx, ny, i, j, d, &q) ? (diag ? off[d][P] / diag[P] : off[d][P]) : 0.0;
    }
}

/* u = v + sum_d c_d v_nb(d)  (unit diagonal), fp64 */
void o64_apply9(int nx, int ny, const double *const c[8], const double *v, double *u) {
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      const int64_t P = (int64_t)i + (int64_t)nx * j;
      int64_t q;
      double s = v[P];
      for (int d = 0; d < 8; ++d)
        if (nb9(nx, ny, i, j, d, &q)) s += c[d][P] * v[q];
      u[P] = s;
    }
}

/* mirror of the GPU kernel: u = v; u = fma16(c_d, v_nb(d), u) for d = 0..7
 * (one fp16 rounding per term), out-of-mesh neighbour values +0 */
void o16_apply9(int nx, int ny, const uint16_t *const c[8], const uint16_t *v, uint16_t *u) {
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      const int64_t P = (int64_t)i + (int64_t)nx * j;
      int64_t q;
      uint16_t acc = v[P];
      for (int d = 0; d < 8; ++d) acc = o16_fma(c[d][P], nb9(nx, ny, i, j, d, &q) ? v[q] : 0, acc);
      u[P] = acc;
    }
}

/* the same order in fp32 with single-rounding fmaf */
void o32_apply9(int nx, int ny, const float *const c[8], const float *v, float *u) {
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      const int64_t P = (int64_t)i + (int64_t)nx * j;
      int64_t q;
      float acc = v[P];
      for (int d = 0; d < 8; ++d) acc = fmaf(c[d][P], nb9(nx, ny, i, j, d, &q) ? v[q] : 0.0f, acc);
      u[P] = acc;
    }
}

/* ======================= the paper's tiled 2D SpMV ========================
 * "we map a rectangular region of the mesh of v to each core,
 * and store all elements of the corresponding columns of A.  After
 * multiplication of the local v with the local A we have generated products in
 * an output halo that must be sent to neighboring tiles. ... We complete a
 * round of send and add in one direction, then a round for the other
 * direction, and in this way avoid communication along diagonals of the tile
 * grid."  Written out step by step:
 *   tiles: a TX x TY grid; tile (a, b) owns columns [X_a, X_a+1) and rows
 *     [Y_b, Y_b+1), X_a = floor(a nx / TX), Y_b = floor(b ny / TY) (R24);
 *   step 1 (local product): for every point P of the tile's region grown by one
 *     point on each side (clipped to the mesh), w[P] = (P in tile ? v_P : 0)
 *     then, for d = 0..7 in order, w[P] += c_d[P] v_{P+d} for the neighbours
 *     P+d that lie IN the tile (the tile's columns of A);
 *   step 2 (x round): into each of its own columns, a tile adds the output halo
 *     column its left neighbour computed there, then its right neighbour's,
 *     over the full grown height (so diagonal products ride along);
 *   step 3 (y round): into each of its own rows (own columns only), a tile adds
 *     the output halo row of the tile below, then of the tile above;
 *   u_P = w[P] of the tile owning P.
 * Three precisions: fp64 (+, *), fp32 (fmaf for the products, + for the
 * rounds) and binary16 (o16_fma / o16_add), the last two the GPU's order. */
typedef struct {
  int x0, x1, y0, y1;   /* owned region [x0, x1) x [y0, y1) */
  int gx0, gx1, gy0, gy1; /* grown region, clipped to the mesh */
} Tile9;

static Tile9 tile9(int nx, int ny, int TX, int TY, int a, int b) {
  Tile9 t;
  t.x0 = (int)((int64_t)a * nx / TX);
  t.x1 = (int)((int64_t)(a + 1) * nx / TX);
  t.y0 = (int)((int64_t)b * ny / TY);
  t.y1 = (int)((int64_t)(b + 1) * ny / TY);
  t.gx0 = t.x0 > 0 ? t.x0 - 1 : 0;
  t.gx1 = t.x1 < nx ? t.x1 + 1 : nx;
  t.gy0 = t.y0 > 0 ? t.y0 - 1 : 0;
  t.gy1 = t.y1 < ny ? t.y1 + 1 : ny;
  return t;
}

static int in_tile(const Tile9 *t, int i, int j) { return i >= t->x0 && i < t->x1 && j >= t->y0 && j < t->y1; }
static int in_grown(const Tile9 *t, int i, int j) { return i >= t->gx0 && i < t->gx1 && j >= t->gy0 && j < t->gy1; }
static int64_t gidx(const Tile9 *t, int i, int j) {
  return (int64_t)(i - t->gx0) + (int64_t)(t->gx1 - t->gx0) * (j - t->gy0);
}

/* element type ops: 0 = fp64, 1 = fp32, 2 = binary16 (values carried as double
 * for fp64, float for fp32, uint16 bit patterns for fp16) */
typedef union {
  double d;
  float f;
  uint16_t h;
} Val9;

static Val9 zero9(int prec) {
  Val9 z;
  z.d = 0.0;
  if (prec == 1) z.f = 0.0f;
  if (prec == 2) z.h = 0;
  return z;
}
static Val9 ld9(int prec, const void *a, int64_t P) {
  Val9 v;
  if (prec == 0) v.d = ((const double *)a)[P];
  else if (prec == 1) v.f = ((const float *)a)[P];
  else v.h = ((const uint16_t *)a)[P];
  return v;
}
static void st9(int prec, void *a, int64_t P, Val9 v) {
  if (prec == 0) ((double *)a)[P] = v.d;
  else if (prec == 1) ((float *)a)[P] = v.f;
  else ((uint16_t *)a)[P] = v.h;
}
static Val9 fma9(int prec, Val9 a, Val9 b, Val9 c) { /* a*b + c */
  Val9 r;
  if (prec == 0) r.d = c.d + a.d * b.d;
  else if (prec == 1) r.f = fmaf(a.f, b.f, c.f);
  else r.h = o16_fma(a.h, b.h, c.h);
  return r;
}
static Val9 add9(int prec, Val9 a, Val9 b) {
  Val9 r;
  if (prec == 0) r.d = a.d + b.d;
  else if (prec == 1) r.f = a.f + b.f;
  else r.h = o16_add(a.h, b.h);
  return r;
}

static void apply9_tiles(int prec, int nx, int ny, int TX, int TY, const void *const c[8], const void *v, void *u) {
  const size_t es = prec == 0 ? 8 : (prec == 1 ? 4 : 2);
  const int NT = TX * TY;
  Tile9 *T = (Tile9 *)malloc(sizeof(Tile9) * (size_t)NT);
  void **W = (void **)malloc(sizeof(void *) * (size_t)NT);
  for (int b = 0; b < TY; ++b)
    for (int a = 0; a < TX; ++a) {
      Tile9 *t = &T[a + TX * b];
      *t = tile9(nx, ny, TX, TY, a, b);
      const size_t n = (size_t)(t->gx1 - t->gx0) * (size_t)(t->gy1 - t->gy0);
      W[a + TX * b] = calloc(n > 0 ? n : 1, es);
    }
  /* step 1: local products into the grown region */
  for (int k = 0; k < NT; ++k) {
    const Tile9 *t = &T[k];
    for (int j = t->gy0; j < t->gy1; ++j)
      for (int i = t->gx0; i < t->gx1; ++i) {
        const int64_t P = (int64_t)i + (int64_t)nx * j;
        Val9 w = in_tile(t, i, j) ? ld9(prec, v, P) : zero9(prec);
        int64_t q;
        for (int d = 0; d < 8; ++d)
          if (nb9(nx, ny, i, j, d, &q) && in_tile(t, i + DX9[d], j + DY9[d]))
            w = fma9(prec, ld9(prec, c[d], P), ld9(prec, v, q), w);
        st9(prec, W[k], gidx(t, i, j), w);
      }
  }
  /* step 2: x round - own columns += left neighbour's halo column, then the right one's */
  for (int b = 0; b < TY; ++b)
    for (int a = 0; a < TX; ++a) {
      const Tile9 *t = &T[a + TX * b];
      for (int side = 0; side < 2; ++side) {
        const int an = side == 0 ? a - 1 : a + 1;
        if (an < 0 || an >= TX) continue;
        const Tile9 *n = &T[an + TX * b];
        for (int j = t->gy0; j < t->gy1; ++j)
          for (int i = t->x0; i < t->x1; ++i)
            if (in_grown(n, i, j) && !in_tile(n, i, j)) {
              const Val9 s = add9(prec, ld9(prec, W[a + TX * b], gidx(t, i, j)), ld9(prec, W[an + TX * b], gidx(n, i, j)));
              st9(prec, W[a + TX * b], gidx(t, i, j), s);
            }
      }
    }
  /* step 3: y round - own rows (own columns) += the halo row of the tile below, then above */
  for (int b = 0; b < TY; ++b)
    for (int a = 0; a < TX; ++a) {
      const Tile9 *t = &T[a + TX * b];
      for (int side = 0; side < 2; ++side) {
        const int bn = side == 0 ? b - 1 : b + 1;
        if (bn < 0 || bn >= TY) continue;
        const Tile9 *n = &T[a + TX * bn];
        for (int j = t->y0; j < t->y1; ++j)
          for (int i = t->x0; i < t->x1; ++i)
            if (in_grown(n, i, j) && !in_tile(n, i, j)) {
              const Val9 s = add9(prec, ld9(prec, W[a + TX * b], gidx(t, i, j)), ld9(prec, W[a + TX * bn], gidx(n, i, j)));
              st9(prec, W[a + TX * b], gidx(t, i, j), s);
            }
      }
    }
  for (int k = 0; k < NT; ++k) {
    const Tile9 *t = &T[k];
    for (int j = t->y0; j < t->y1; ++j)
      for (int i = t->x0; i < t->x1; ++i) st9(prec, u, (int64_t)i + (int64_t)nx * j, ld9(prec, W[k], gidx(t, i, j)));
    free(W[k]);
  }
  free(W);
  free(T);
}

void o64_apply9_tiles(int nx, int ny, int TX, int TY, const double *const c[8], const double *v, double *u) {
  apply9_tiles(0, nx, ny, TX, TY, (const void *const *)c, v, u);
}
void o32_apply9_tiles(int nx, int ny, int TX, int TY, const float *const c[8], const float *v, float *u) {
  apply9_tiles(1, nx, ny, TX, TY, (const void *const *)c, v, u);
}
void o16_apply9_tiles(int nx, int ny, int TX, int TY, const uint16_t *const c[8], const uint16_t *v, uint16_t *u) {
  apply9_tiles(2, nx, ny, TX, TY, (const void *const *)c, v, u);
}

/* ====================== BiCGStab on the 2D operator =======================
 * each core holds "a matrix, halo, and vector (as well as all
 * terms needed for BiCG)" - Alg. 1 with the 9-point
 * operator in place of the 7-point one, under the readings of the 3D oracle
 * (R1-R8, R12, R23).  The SpMV is the gather, or with TX x TY > 1 the paper's
 * tiled output-halo form (apply9_tiles, R24: "all terms needed for BiCG" live with each tile's
 * columns of A).  fp64 (o2d64_bicgstab) and the binary16 mixed
 * mode in the GPU's operation order (o2d16_bicgstab: FMA-chain SpMV
 * o16_apply9, fp16 FMAC AXPYs with fp32 scalars rounded to fp16, dots of exact
 * fp16 products summed in fp32 over each row, then over rows). */
static int ev9(int code, int i, double tol, int *ev, int *ev_it) {
  if (*ev < 0) {
    *ev = code;
    *ev_it = i;
  }
  return tol > 0.0;
}

static double dot64_9(int64_t n, const double *a, const double *b) {
  double s = 0.0;
  for (int64_t P = 0; P < n; ++P) s += a[P] * b[P];
  return s;
}

/* the SpMV of the solve: the gather (one tile) or the paper's tiled output-halo form (R24) */
static void spmv64_9(int nx, int ny, int TX, int TY, const double *const c[8], const double *v, double *u) {
  if (TX * TY == 1) o64_apply9(nx, ny, c, v, u);
  else o64_apply9_tiles(nx, ny, TX, TY, c, v, u);
}
static void spmv16_9(int nx, int ny, int TX, int TY, const uint16_t *const c[8], const uint16_t *v, uint16_t *u) {
  if (TX * TY == 1) o16_apply9(nx, ny, c, v, u);
  else o16_apply9_tiles(nx, ny, TX, TY, c, v, u);
}

int o2d64_bicgstab_tiles(int nx, int ny, int TX, int TY, const double *const c[8], const double *b, const double *x0,
                         double tol, int maxit, double *x, double *hist, double *alpha_out, double *omega_out,
                         int *status, int *event_it) {
  const int64_t n = (int64_t)nx * ny;
  const size_t bytes = sizeof(double) * (size_t)(n > 0 ? n : 1);
  double *r = (double *)malloc(bytes), *rh = (double *)malloc(bytes);
  double *p = (double *)malloc(bytes), *v = (double *)malloc(bytes);
  double *s = (double *)malloc(bytes), *t = (double *)malloc(bytes);
  int ev = -1, ev_it = 0, it = 0;
  if (x0) { /* R1 */
    memcpy(x, x0, bytes);
    spmv64_9(nx, ny, TX, TY, c, x, t);
    for (int64_t P = 0; P < n; ++P) r[P] = b[P] - t[P];
  } else { /* l.174 */
    for (int64_t P = 0; P < n; ++P) {
      x[P] = 0.0;
      r[P] = b[P];
    }
  }
  memcpy(rh, r, bytes);
  memcpy(p, r, bytes);
  double rho = dot64_9(n, rh, r);
  const double nb = sqrt(dot64_9(n, b, b));
  if (nb == 0.0) {
    for (int64_t P = 0; P < n; ++P) x[P] = 0.0;
    hist[0] = 0.0;
    *status = ORC_CONVERGED;
    *event_it = 0;
    goto done;
  }
  hist[0] = sqrt(dot64_9(n, r, r)) / nb;
  if (tol > 0.0 && hist[0] <= tol) {
    *status = ORC_CONVERGED;
    *event_it = 0;
    goto done;
  }
  double alpha = 0.0, omega = 0.0, beta = 0.0;
  for (int i = 1; i <= maxit; ++i) {
    if (i > 1)
      for (int64_t P = 0; P < n; ++P) p[P] = r[P] + beta * (p[P] - omega * v[P]); /* l.184 */
    spmv64_9(nx, ny, TX, TY, c, p, v);                                                  /* l.176 */
    const double sigma = dot64_9(n, rh, v);                                       /* l.177 */
    alpha = rho / sigma;
    if (sigma == 0.0 || !isfinite(alpha)) {
      alpha = 0.0;
      if (ev9(isfinite(sigma) ? ORC_BREAKDOWN : ORC_NONFINITE, i, tol, &ev, &ev_it)) {
        it = i - 1;
        break;
      }
    }
    for (int64_t P = 0; P < n; ++P) s[P] = r[P] - alpha * v[P]; /* l.178 */
    spmv64_9(nx, ny, TX, TY, c, s, t);                                /* l.179 */
    const double ts = dot64_9(n, t, s), tt = dot64_9(n, t, t);
    if (tt == 0.0) {
      omega = 0.0; /* R8 */
    } else {
      omega = ts / tt; /* l.180 */
      if (!isfinite(omega)) {
        omega = 0.0;
        if (ev9(ORC_NONFINITE, i, tol, &ev, &ev_it)) {
          it = i - 1;
          break;
        }
      }
    }
    for (int64_t P = 0; P < n; ++P) x[P] = (x[P] + alpha * p[P]) + omega * s[P]; /* l.181 */
    for (int64_t P = 0; P < n; ++P) r[P] = s[P] - omega * t[P];                  /* l.182 */
    const double rhon = dot64_9(n, rh, r), rr = dot64_9(n, r, r);
    hist[i] = sqrt(rr) / nb;
    if (alpha_out) alpha_out[i] = alpha;
    if (omega_out) omega_out[i] = omega;
    it = i;
    int code = -1;
    if (!isfinite(rr) || !isfinite(rhon)) code = ORC_NONFINITE;
    else if (rr == 0.0 && rhon != 0.0) code = ORC_BREAKDOWN; /* R23 */
    else if (rr == 0.0 || (tol > 0.0 && hist[i] <= tol)) code = ORC_CONVERGED;
    else if (omega == 0.0 || rhon == 0.0) code = ORC_BREAKDOWN;
    beta = (rhon / rho) * (alpha / omega); /* l.183 */
    if (!isfinite(beta)) beta = 0.0;
    rho = rhon;
    if (code >= 0 && ev9(code, i, tol, &ev, &ev_it)) break;
  }
  *status = ev >= 0 ? ev : ORC_MAXIT;
  *event_it = ev_it;
done:
  free(r); free(rh); free(p); free(v); free(s); free(t);
  return it;
}

static uint16_t neg16_9(uint16_t a) { return a ^ 0x8000; }
static uint16_t rn16f_9(float x) { return o16_from_double((double)x); }
static int usable16_9(float s) { return isfinite(s) && (((rn16f_9(s) >> 10) & 31) != 31); }
/* fp16 values widened exactly; products exact in fp32; fp32 sums per row, then over rows */
static float dot16_9(int nx, int ny, const uint16_t *a, const uint16_t *b) {
  float total = 0.0f;
  for (int j = 0; j < ny; ++j) {
    float row = 0.0f;
    for (int i = 0; i < nx; ++i) {
      const int64_t P = (int64_t)i + (int64_t)nx * j;
      row += (float)o16_to_double(a[P]) * (float)o16_to_double(b[P]);
    }
    total += row;
  }
  return total;
}

int o2d16_bicgstab_tiles(int nx, int ny, int TX, int TY, const uint16_t *const c[8], const uint16_t *b,
                         const uint16_t *x0, double tol, int maxit, uint16_t *x, double *hist, float *alpha_out,
                         float *omega_out, int *status, int *event_it) {
  const int64_t n = (int64_t)nx * ny;
  const size_t bytes = sizeof(uint16_t) * (size_t)(n > 0 ? n : 1);
  uint16_t *r = (uint16_t *)malloc(bytes), *rh = (uint16_t *)malloc(bytes);
  uint16_t *p = (uint16_t *)malloc(bytes), *v = (uint16_t *)malloc(bytes);
  uint16_t *s = (uint16_t *)malloc(bytes), *t = (uint16_t *)malloc(bytes);
  int ev = -1, ev_it = 0, it = 0;
  if (x0) { /* R1 */
    memcpy(x, x0, bytes);
    spmv16_9(nx, ny, TX, TY, c, x, t);
    for (int64_t P = 0; P < n; ++P) r[P] = o16_add(b[P], neg16_9(t[P]));
  } else {
    for (int64_t P = 0; P < n; ++P) {
      x[P] = 0;
      r[P] = b[P];
    }
  }
  memcpy(rh, r, bytes);
  memcpy(p, r, bytes);
  float rho = dot16_9(nx, ny, rh, r);
  const double nb = sqrt((double)dot16_9(nx, ny, b, b));
  if (nb == 0.0) {
    for (int64_t P = 0; P < n; ++P) x[P] = 0;
    hist[0] = 0.0;
    *status = ORC_CONVERGED;
    *event_it = 0;
    goto done;
  }
  hist[0] = sqrt((double)dot16_9(nx, ny, r, r)) / nb;
  if (tol > 0.0 && hist[0] <= tol) {
    *status = ORC_CONVERGED;
    *event_it = 0;
    goto done;
  }
  float alpha = 0.0f, omega = 0.0f, beta = 0.0f;
  for (int i = 1; i <= maxit; ++i) {
    if (i > 1) { /* l.184, two fp16 FMACs (R11) */
      const uint16_t bh = rn16f_9(beta), mwh = neg16_9(rn16f_9(omega));
      for (int64_t P = 0; P < n; ++P) p[P] = o16_fma(bh, o16_fma(mwh, v[P], p[P]), r[P]);
    }
    spmv16_9(nx, ny, TX, TY, c, p, v);                   /* l.176 */
    const float sigma = dot16_9(nx, ny, rh, v);    /* l.177 */
    alpha = rho / sigma;
    if (sigma == 0.0f || !usable16_9(alpha)) {
      alpha = 0.0f;
      if (ev9(isfinite(sigma) ? ORC_BREAKDOWN : ORC_NONFINITE, i, tol, &ev, &ev_it)) {
        it = i - 1;
        break;
      }
    }
    const uint16_t ah = rn16f_9(alpha);
    for (int64_t P = 0; P < n; ++P) s[P] = o16_fma(neg16_9(ah), v[P], r[P]); /* l.178 */
    spmv16_9(nx, ny, TX, TY, c, s, t);                                             /* l.179 */
    const float ts = dot16_9(nx, ny, t, s), tt = dot16_9(nx, ny, t, t);
    if (tt == 0.0f) {
      omega = 0.0f;
    } else {
      omega = ts / tt; /* l.180 */
      if (!usable16_9(omega)) {
        omega = 0.0f;
        if (ev9(ORC_NONFINITE, i, tol, &ev, &ev_it)) {
          it = i - 1;
          break;
        }
      }
    }
    const uint16_t wh = rn16f_9(omega);
    for (int64_t P = 0; P < n; ++P) x[P] = o16_fma(wh, s[P], o16_fma(ah, p[P], x[P])); /* l.181 */
    for (int64_t P = 0; P < n; ++P) r[P] = o16_fma(neg16_9(wh), t[P], s[P]);           /* l.182 */
    const float rhon = dot16_9(nx, ny, rh, r), rr = dot16_9(nx, ny, r, r);
    hist[i] = sqrt((double)rr) / nb;
    if (alpha_out) alpha_out[i] = alpha;
    if (omega_out) omega_out[i] = omega;
    it = i;
    int code = -1;
    if (!isfinite(rr) || !isfinite(rhon)) code = ORC_NONFINITE;
    else if (rr == 0.0f && rhon != 0.0f) code = ORC_BREAKDOWN; /* R23 */
    else if (rr == 0.0f || (tol > 0.0 && hist[i] <= tol)) code = ORC_CONVERGED;
    else if (omega == 0.0f || rhon == 0.0f) code = ORC_BREAKDOWN;
    beta = (rhon / rho) * (alpha / omega); /* l.183, fp32 */
    if (!usable16_9(beta)) beta = 0.0f;
    rho = rhon;
    if (code >= 0 && ev9(code, i, tol, &ev, &ev_it)) break;
  }
  *status = ev >= 0 ? ev : ORC_MAXIT;
  *event_it = ev_it;
done:
  free(r); free(rh); free(p); free(v); free(s); free(t);
  return it;
}

/* the solves on the gather SpMV (one tile) */
int o2d64_bicgstab(int nx, int ny, const double *const c[8], const double *b, const double *x0, double tol,
                   int maxit, double *x, double *hist, double *alpha_out, double *omega_out, int *status,
                   int *event_it) {
  return o2d64_bicgstab_tiles(nx, ny, 1, 1, c, b, x0, tol, maxit, x, hist, alpha_out, omega_out, status, event_it);
}
int o2d16_bicgstab(int nx, int ny, const uint16_t *const c[8], const uint16_t *b, const uint16_t *x0, double tol,
                   int maxit, uint16_t *x, double *hist, float *alpha_out, float *omega_out, int *status,
                   int *event_it) {
  return o2d16_bicgstab_tiles(nx, ny, 1, 1, c, b, x0, tol, maxit, x, hist, alpha_out, omega_out, status, event_it);
}
