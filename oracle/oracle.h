/*
 * oracle.h - CPU oracle for BiCGStab on the Jacobi-scaled 7-point stencil.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.  The
 * product (paper_2010_03660_b200, libsten.so) never links, loads or calls it,
 * and shares no code with it.
 *
 * Written from the paper (arXiv 2010.03660, /root/reference/PAPER.md):
 *   - Algorithm 1 "Standard BiCGStab", PAPER.md:168-189 (Sec. III);
 *   - unit main diagonal by diagonal (Jacobi) preconditioning, six stored
 *     off-diagonals, PAPER.md:195 (Sec. IV);
 *   - SpMV u = A v as the sum of the local iterate and six coefficient-times-
 *     neighbour products, PAPER.md:198-201, 338-346 (Sec. SpMV(3D));
 *   - mixed precision: fp16 storage and arithmetic, inner products with fp16
 *     multiply / fp32 add, AllReduce in fp32, PAPER.md:82, 116-120, 397;
 *   - the single-reduction rearrangement of Alg. 1 (osr.c, R19), the 16-bit
 *     dot accumulation of the unpublished half mode (osr.c o16h_*, R22), the
 *     2D 9-point SpMV (o2d.c).
 * Readings where the paper is silent are numbered R1..R22 in DESIGN.md.
 *
 * Mesh: nx*ny*nz points, linear index P = i + nx*(j + ny*k), x fastest.
 * Coefficient arrays c[0..5] = (xm, xp, ym, yp, zm, zp): c_d[P] multiplies
 * v at the -x/+x/-y/+y/-z/+z neighbour of P.  Neighbours outside the mesh
 * contribute nothing (Dirichlet zero, R5).
 *
 * Parity pins: every function is pinned by tests/test_oracle_*.py (see the
 * "Pins" table in DESIGN.md).  Functions marked "mirror" reproduce one
 * specific evaluation order of the GPU kernels (bitwise tests); they are
 * independent re-statements of that order, not shared code.
 */
#ifndef STEN_ORACLE_H
#define STEN_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (same meaning as include/sten.h, restated here) */
#define ORC_CONVERGED 0
#define ORC_MAXIT 1
#define ORC_BREAKDOWN 2
#define ORC_NONFINITE 3

/* ---------------- fp64 reference (O64) ---------------- */

/* Jacobi scaling: c_d[P] = off_d[P] / diag[P] for in-mesh
 * neighbours, +0 where the neighbour is outside the mesh (R5). diag==NULL:
 * the off-diagonals are taken as already scaled (only the zeroing applies). */
void o64_jacobi_scale(int nx, int ny, int nz, const double *diag,
                      const double *const off[6], double *const c[6]);

/* u = v + sum_d c_d * v_nb(d)   (unit diagonal) */
void o64_apply(int nx, int ny, int nz, const double *const c[6],
               const double *v, double *u);

/* u = diag*v + sum_d off_d * v_nb(d)  (the un-scaled matrix; used to make a
 * manufactured right-hand side b = A x_true, config 1) */
void o64_apply_raw(int nx, int ny, int nz, const double *diag,
                   const double *const off[6], const double *v, double *u);

/* sum_P a[P]*b[P], P ascending, fp64 */
double o64_dot(int64_t n, const double *a, const double *b);

/* BiCGStab, Alg. 1 in fp64 with the stopping / breakdown
 * readings R6-R9.  x0 may be NULL (x0 = 0, Alg. 1 line 174 exactly).
 * hist[0..maxit] receives ||r_i||/||b||; alpha/omega (may be NULL) receive
 * alpha_i, omega_i at index i (1-based).  Returns the number of completed
 * iterations; *status one of ORC_*.  *event_it = iteration of the first event
 * (tol == 0 benchmark mode), 0 if none. */
int o64_bicgstab(int nx, int ny, int nz, const double *const c[6],
                 const double *b, const double *x0, double tol, int maxit,
                 double *x, double *hist, double *alpha, double *omega,
                 int *status, int *event_it);

/* ||b - A x||_2 / ||b||_2 in fp64 (unit-diagonal operator) */
double o64_true_residual(int nx, int ny, int nz, const double *const c[6],
                         const double *b, const double *x);

/* ---------------- IEEE binary16 primitives (exact integer arithmetic) ------ */
double o16_to_double(uint16_t h);
uint16_t o16_from_double(double x);              /* round-to-nearest-even */
uint16_t o16_fma(uint16_t a, uint16_t b, uint16_t c); /* a*b+c, one rounding */
uint16_t o16_add(uint16_t a, uint16_t b);
uint16_t o16_mul(uint16_t a, uint16_t b);
void o16_from_double_array(int64_t n, const double *x, uint16_t *h);
void o16_to_double_array(int64_t n, const uint16_t *h, double *x);
void o16_fma_array(int64_t n, const uint16_t *a, const uint16_t *b, const uint16_t *c, uint16_t *out);
void o32_fma_array(int64_t n, const float *a, const float *b, const float *c, float *out); /* fmaf */
void o16_add_array(int64_t n, const uint16_t *a, const uint16_t *b, uint16_t *out);
void o16_mul_array(int64_t n, const uint16_t *a, const uint16_t *b, uint16_t *out);

/* ---------------- fp16 "mixed" oracle (O16) ---------------- */

/* mirror: u = v; u = fma16(c_xm, v_xm, u); ... xp, ym, yp, zm, zp (R10);
 * out-of-mesh neighbour value taken as +0. */
void o16_apply_fused(int nx, int ny, int nz, const uint16_t *const c[6],
                     const uint16_t *v, uint16_t *u);
/* paper-faithful variant: each product rounded to fp16, then an fp16 add
 * (Table "Operations per meshpoint per iteration": HP x and HP + counted
 * separately; separate multiply threads + sumtask,
 * PAPER.md:340-346).  Diagonal term first, then xm..zp. */
void o16_apply_unfused(int nx, int ny, int nz, const uint16_t *const c[6],
                       const uint16_t *v, uint16_t *u);
/* mixed inner product: fp16 x fp16 product exact in fp32,
 * fp32 accumulation along each z-pencil (one CS-1 core's local dot,
 * PAPER.md:193-195), then an fp32 sum over pencils (the fp32 AllReduce). */
float o16_dot(int nx, int ny, int nz, const uint16_t *a, const uint16_t *b);

/* BiCGStab in mixed precision: every vector op in fp16 (fused FMAs, R11),
 * dots as o16_dot, scalars in fp32 (R12).  unfused != 0 selects
 * o16_apply_unfused and unfused AXPYs.  Same control flow as o64_bicgstab. */
int o16_bicgstab(int nx, int ny, int nz, const uint16_t *const c[6],
                 const uint16_t *b, const uint16_t *x0, double tol, int maxit,
                 int unfused, uint16_t *x, double *hist, float *alpha,
                 float *omega, int *status, int *event_it);
/* o16_bicgstab with the iteration's five inner products as half-mode fp16 pencils over the z
 * segments seg[0..nseg) (o16h_dot, R22; nseg = 0: mixed); rho_0, ||b|| and hist[0] stay mixed (R28) */
int o16h_bicgstab(int nx, int ny, int nz, const uint16_t *const c[6], const uint16_t *b, const uint16_t *x0,
                  double tol, int maxit, int unfused, int nseg, const int *seg, uint16_t *x, double *hist,
                  float *alpha_out, float *omega_out, int *status, int *event_it);

/* ---------------- fp32 mirror of the GPU fp32 kernels ---------------- */
/* u = v; u = fmaf(c_xm, v_xm, u); ... (same order as o16_apply_fused) */
void o32_apply_fma(int nx, int ny, int nz, const float *const c[6],
                   const float *v, float *u);

/* ---------------- single-reduction schedule (osr.c, R19) -------- */
/* One sweep: with scalars (alpha, omega, beta) of the previous iteration,
 * update x, r, p in place, then v = A p, q = A r, y = A v, and the twelve
 * inner products dots[] = (rh,v) (rh,r) (rh,q) (rh,y) (q,r) (q,v) (y,r) (y,v)
 * (q,q) (q,y) (y,y) (r,r).  See osr.c for the derivation from Alg. 1. */
void o64_sr_sweep(int nx, int ny, int nz, const double *const c[6], double alpha,
                  double omega, double beta, const double *rh, double *x,
                  double *r, double *p, double *v, double *q, double *y,
                  double dots[12]);
void o16_sr_sweep(int nx, int ny, int nz, const uint16_t *const c[6], float alpha,
                  float omega, float beta, const uint16_t *rh, uint16_t *x,
                  uint16_t *r, uint16_t *p, uint16_t *v, uint16_t *q, uint16_t *y,
                  float dots[12]);
void o32_sr_sweep(int nx, int ny, int nz, const float *const c[6], float alpha,
                  float omega, float beta, const float *rh, float *x, float *r,
                  float *p, float *v, float *q, float *y, double dots[12]);
/* Whole solves with the SR schedule; same arguments, outputs and control flow
 * (stopping, events) as o64_bicgstab / o16_bicgstab. */
int o64_sr_bicgstab(int nx, int ny, int nz, const double *const c[6],
                    const double *b, const double *x0, double tol, int maxit,
                    double *x, double *hist, double *alpha, double *omega,
                    int *status, int *event_it);
int o16_sr_bicgstab(int nx, int ny, int nz, const uint16_t *const c[6],
                    const uint16_t *b, const uint16_t *x0, double tol, int maxit,
                    uint16_t *x, double *hist, float *alpha, float *omega,
                    int *status, int *event_it);

/* Half dots (R22, NEXT-4): per (x, y) column and z segment
 * [seg[s], seg[s+1]) an fp16 running sum acc = fma16(a, b, acc) from +0, z
 * ascending; *sum = the exact (fp64) sum of the segment sums, *abs = the sum
 * of their magnitudes (may be NULL).  o16h_sr_sweep / o16h_sr_bicgstab: the
 * O16-SR sweep and solve with those dots rounded once to fp32 (nseg = 0: the
 * mixed dots of o16_sr_sweep / o16_sr_bicgstab); dabs may be NULL. */
void o16h_dot(int nx, int ny, int nz, const uint16_t *a, const uint16_t *b, int nseg,
              const int *seg, double *sum, double *abs);
void o16h_sr_sweep(int nx, int ny, int nz, const uint16_t *const c[6], float alpha,
                   float omega, float beta, const uint16_t *rh, uint16_t *x,
                   uint16_t *r, uint16_t *p, uint16_t *v, uint16_t *q, uint16_t *y,
                   int nseg, const int *seg, float dots[12], double dabs[12]);
int o16h_sr_bicgstab(int nx, int ny, int nz, const uint16_t *const c[6],
                     const uint16_t *b, const uint16_t *x0, double tol, int maxit,
                     int nseg, const int *seg,
                     uint16_t *x, double *hist, float *alpha, float *omega,
                     int *status, int *event_it);

/* ---------------- 2D 9-point SpMV (o2d.c; NEXT-3) ------- */
/* Mesh nx*ny, P = i + nx*j; c[0..7] couple P to its (dx,dy) neighbour in the
 * order (-1,-1) (0,-1) (+1,-1) (-1,0) (+1,0) (-1,+1) (0,+1) (+1,+1). */
void o64_jacobi_scale9(int nx, int ny, const double *diag, const double *const off[8], double *const c[8]);
void o64_apply9(int nx, int ny, const double *const c[8], const double *v, double *u);
void o16_apply9(int nx, int ny, const uint16_t *const c[8], const uint16_t *v, uint16_t *u);  /* mirror */
void o32_apply9(int nx, int ny, const float *const c[8], const float *v, float *u);           /* mirror */
/* the paper's tiled form: TX x TY tiles, local products of
 * each tile's columns into its grown region, then the output-halo rounds x
 * then y (see o2d.c); fp64, and the GPU's fp32 / binary16 orders */
void o64_apply9_tiles(int nx, int ny, int TX, int TY, const double *const c[8], const double *v, double *u);
void o32_apply9_tiles(int nx, int ny, int TX, int TY, const float *const c[8], const float *v, float *u);
void o16_apply9_tiles(int nx, int ny, int TX, int TY, const uint16_t *const c[8], const uint16_t *v, uint16_t *u);
/* BiCGStab (Alg. 1) on the 2D operator, readings as in 3D */
int o2d64_bicgstab(int nx, int ny, const double *const c[8], const double *b, const double *x0, double tol,
                   int maxit, double *x, double *hist, double *alpha, double *omega, int *status, int *event_it);
int o2d16_bicgstab(int nx, int ny, const uint16_t *const c[8], const uint16_t *b, const uint16_t *x0, double tol,
                   int maxit, uint16_t *x, double *hist, float *alpha, float *omega, int *status, int *event_it);
/* the same with the paper's tiled output-halo SpMV (apply9_tiles, R24) on TX x TY tiles */
int o2d64_bicgstab_tiles(int nx, int ny, int TX, int TY, const double *const c[8], const double *b, const double *x0,
                         double tol, int maxit, double *x, double *hist, double *alpha_out, double *omega_out,
                         int *status, int *event_it);
int o2d16_bicgstab_tiles(int nx, int ny, int TX, int TY, const uint16_t *const c[8], const uint16_t *b,
                         const uint16_t *x0, double tol, int maxit, uint16_t *x, double *hist, float *alpha_out,
                         float *omega_out, int *status, int *event_it);

/* informational */
int oracle_num_threads(void);
void oracle_set_threads(int n);

#ifdef __cplusplus
}
#endif
#endif
