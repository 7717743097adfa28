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
