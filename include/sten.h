/*
 * sten.h - C ABI of libsten.so: B200-native (sm_100a) BiCGStab for the linear
 * system of a 7-point finite-difference stencil on a regular 3D mesh, with the
 * main diagonal Jacobi-scaled to one.
 *
 * What is computed (arXiv 2010.03660, /root/reference/PAPER.md):
 *   - the operator: A x = b from a 7-point stencil; "with
 *     diagonal preconditioning the main diagonal is all ones.  Therefore, we
 *     only store six other diagonals" (Sec. IV);
 *   - stencil_apply: u = A v as the local value plus six coefficient-times-
 *     neighbour products (Sec. "SpMV (3D)");
 *   - bicgstab_solve: Algorithm 1 "Standard BiCGStab", as
 *     printed (STEN_SCHED_CLASSIC) or rearranged to one sweep and one
 *     reduction per iteration (STEN_SCHED_SR, R19);
 *   - bicgstab_refine: mixed-precision iterative refinement, the remedy the
 *     paper names for the fp16 plateau (R21);
 *   - stencil_create_const: a constant-coefficient operator (no coefficient
 *     streams in the SR sweep);
 *   - stencil2d_*: the paper's 2D 9-point SpMV;
 *   - precisions: fp32 throughout, or the paper's mixed mode - fp16 storage
 *     and arithmetic, inner products with fp16 multiply / fp32 accumulate, the
 *     cross-device reduction in fp32; optionally
 *     (sten_set_dot_precision) the unpublished 16-bit mode's fp16 dot
 *     accumulation (R22).
 * Readings of the paper where it is silent (stopping rule, breakdown, x0, the
 * order of floating-point operations ...) are R1..R22 in DESIGN.md.
 *
 * Layout.  A mesh (or a rank's slab of it) of nx*ny*nz points is a dense
 * array with linear index P = i + nx*(j + ny*k): x fastest, z slowest, so a
 * z-slab is contiguous.  Every vector argument (b, x0, x_out, x, y) is such a
 * dense array of this rank's points, in the precision's storage type:
 * float for STEN_FP32, IEEE binary16 (uint16 bit patterns) for STEN_MIXED.
 * Vector and coefficient pointers may be device pointers or host pointers
 * (pinned or pageable); the library classifies each with
 * cudaPointerGetAttributes and copies host data itself, inside the call.
 *
 * Multi-GPU.  With a communicator, rank r of R owns the z-planes directly
 * above rank r-1's (rank order = z order) and passes only its own planes;
 * the library exchanges halo planes with the z-neighbours over NCCL (one plane
 * per SpMV input for the classic schedule; two planes of five vectors once per
 * iteration for SR, overlapped with the interior z chunks) and all-reduces the
 * fp32 dot-product partial sums (1-3 per phase classic, 12 once per SR sweep).
 *
 * Errors.  Every int-returning entry point returns STEN_OK (0) or a negative
 * STEN_E* code; sten_last_error() then gives a thread-local message.
 * Numerical breakdown is NOT an error: bicgstab_solve returns STEN_OK and
 * reports it in *status.
 *
 * Threading.  A handle may be used by one host thread at a time.
 */
#ifndef STEN_H
#define STEN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define STEN_VERSION 3

/* precision of a solve / apply */
#define STEN_FP32 0   /* fp32 storage, fp32 arithmetic, fp32 dots */
#define STEN_MIXED 1  /* fp16 storage + arithmetic, fp16*fp16 products summed in fp32 */

/* iteration schedule of bicgstab_solve (sten_set_schedule) */
#define STEN_SCHED_CLASSIC 0 /* Alg. 1 as printed: 3 kernels, 3 reductions, 29 array passes / iteration */
#define STEN_SCHED_SR 1      /* single reduction: 1 sweep, 1 reduction, 19 array passes / iteration (R19) */

/* element type of the coefficient arrays passed to stencil_create */
#define STEN_DT_F64 0
#define STEN_DT_F32 1

/* return codes */
#define STEN_OK 0
#define STEN_EINVAL (-1)
#define STEN_ENOMEM (-2)
#define STEN_ECUDA (-3)
#define STEN_ENCCL (-4)
#define STEN_EUNSUPPORTED (-5)

/* solve status (R6-R8) */
#define STEN_CONVERGED 0 /* ||r_i||/||b|| <= tol, or r_i == 0 exactly (an
                            (r,r) of 0 with (rhat,r) != 0 is an fp16
                            underflow: BREAKDOWN, R23)                      */
#define STEN_MAXIT 1     /* maxit iterations done without an event             */
#define STEN_BREAKDOWN 2 /* (rhat, v) == 0, omega == 0 or (rhat, r_new) == 0   */
#define STEN_NONFINITE 3 /* a dot product or scalar became Inf/NaN             */
#define STEN_TIMEOUT 4   /* peer-memory all-reduce: a rank's sums never arrived
                            (bounded ~20 s wait; a dead or stalled peer) */

typedef struct sten_comm sten_comm;       /* opaque: NCCL communicator wrapper */
typedef struct sten_stencil sten_stencil; /* opaque: operator + solver workspace */

/* Performance counters of the last bicgstab_solve on a handle. */
typedef struct sten_stats {
  double phase_ms[3];     /* summed device time of phases H1, H2, H3 (timing on) */
  long long phase_launches[3]; /* launches of the H1/H2/H3 kernels timed      */
  double solve_ms;        /* device time from first to last kernel of the solve */
  long long kernel_launches; /* kernels of this library launched by the solve  */
  int event_iter;         /* iteration of the first breakdown event (0: none) */
  int graph_chunk;        /* iterations per CUDA-graph replay                  */
  int handover;           /* bicgstab_refine: outer step at which the inner
                             solves switched schedule after a stagnation
                             (-1: none; 0 after other calls)                  */
} sten_stats;

/* ---------------------------------------------------------------- misc -- */
int sten_version(void);
/* Thread-local message describing the last non-OK return on this thread. */
const char *sten_last_error(void);

/* ---------------------------------------------------------------- comm -- */
/* Write a fresh ncclUniqueId (128 bytes) into id_out; call on rank 0 and
 * broadcast the bytes to the other ranks by any means. */
int sten_comm_unique_id(void *id_out);
/* Create the communicator of rank `rank` of `nranks` on CUDA device
 * `cuda_device`, which becomes the calling thread's current device; handles
 * built on the communicator must be created and used with that device current.
 *   unique_id != NULL: NCCL (loaded at run time, libnccl.so.2) carries the
 *     halo planes and the fp32 all-reduces of every schedule;
 *   unique_id == NULL: a peer-memory-only communicator (no NCCL): after
 *     sten_p2p_import, halos and all-reduces go through CUDA IPC peer memory:
 *     the SR schedule with the fused exchange, or the classic schedule (halo
 *     planes pushed into the neighbours' buffers, a one-shot peer all-reduce
 *     per phase) in host lockstep (sten_set_host_barrier); x0 == NULL;
 *     everything else returns STEN_EUNSUPPORTED.
 * Errors: STEN_EINVAL (bad rank/nranks/cuda_device), STEN_ECUDA, STEN_ENCCL
 * (NCCL missing or ncclCommInitRank failed). */
int sten_comm_create(const void *unique_id, int nranks, int rank, int cuda_device, sten_comm **out);
void sten_comm_destroy(sten_comm *comm);

/* ------------------------------------------------------------- stencil -- */
/* Build the Jacobi-scaled operator of an nx*ny*nz_global mesh; this rank owns
 * planes [r*nz_global/R, (r+1)*nz_global/R) of it (R ranks of `comm`, 1
 * without one; rank order = z order) and passes only those planes.
 *   coeffs[0]   : main diagonal a_P of A, or NULL if A already has a unit
 *                 diagonal;
 *   coeffs[1..6]: off-diagonal entries of A coupling P to its -x, +x, -y, +y,
 *                 -z, +z neighbour (A[P, P-1], A[P, P+1], A[P, P-nx], ...);
 *   all dense (nz_global/R, ny, nx) arrays of coeff_dtype (STEN_DT_F64 or
 *   _F32), host or device; they are copied, the caller keeps ownership.
 * The library forms c_d = A_d / a_P in fp64 (c_d = A_d without a diagonal),
 * drops couplings to points outside the global mesh (Dirichlet zero), and
 * stores c_d rounded to nearest in fp32 AND in fp16 (R3, R5), plus a_P in fp64
 * to scale right-hand sides.
 *   nslabs >= 1: split this rank's planes into nslabs z-slabs with one-plane
 *                halos exchanged by device copies - the same halo/reduction
 *                path as multi-GPU, for testing it on one GPU ((nz_global/R)
 *                % nslabs must be 0; 1 for normal use);
 *   comm: NULL for a single rank, else this rank's communicator (its device
 *         must be current).
 * Errors: STEN_EINVAL (sizes <= 0, nz_global % R, (nz_global/R) % nslabs,
 * NULL coefficient, wrong current device), STEN_ENOMEM, STEN_ECUDA. */
int stencil_create(int nx, int ny, int nz_global, const void *const coeffs[7], int coeff_dtype,
                   int nslabs, sten_comm *comm, void *cuda_stream, sten_stencil **out);
/* The same for a CONSTANT-coefficient operator (e.g. the
 * Poisson stencil of BASELINE config 1): coeffs[0..6] = a_P, A_xm, A_xp,
 * A_ym, A_yp, A_zm, A_zp, the same at every point, with Dirichlet zero outside
 * the global mesh (couplings leaving it dropped, a_P unchanged: R5).  The
 * coefficient arrays are still built (for non-default classic tilings and
 * STEN_OPT_CLASSIC_CONST = 0), but the SR sweep reads none of them: it takes the six
 * scaled couplings (A_d / a_P in fp64, rounded once to fp32 / fp16) as
 * scalars and moves 13 instead of 19 arrays per iteration, and so do the
 * classic kernels (17 instead of 29; STEN_OPT_CLASSIC_CONST).  Results equal those
 * of stencil_create on the same constant fields (bitwise up to the sign of
 * zero).  Errors: STEN_EINVAL (non-finite coefficient, a_P == 0, sizes),
 * STEN_ENOMEM, STEN_ECUDA. */
int stencil_create_const(int nx, int ny, int nz_global, const double coeffs[7], int nslabs, sten_comm *comm,
                         void *cuda_stream, sten_stencil **out);
void stencil_destroy(sten_stencil *st);

/* y = A_hat x, A_hat the Jacobi-scaled operator (unit diagonal), one halo
 * exchange first when decomposed.  x, y: this rank's points in the storage
 * type of `precision`; x and y must not overlap.  Enqueued on cuda_stream and
 * synchronised before return.  Errors: STEN_EINVAL, STEN_ECUDA, STEN_ENCCL. */
int stencil_apply(sten_stencil *st, int precision, const void *x, void *y, void *cuda_stream);

/* Solve A x = b with BiCGStab (Alg. 1) on the Jacobi-scaled system
 * A_hat x = b_hat, b_hat = b / a_P rounded to the working precision (R3).
 *   b      : right-hand side of the ORIGINAL system (of A_hat if no diagonal
 *            was given), this rank's points;
 *   x0     : initial guess, or NULL for x0 = 0 (Alg. 1 l.174 exactly, R1);
 *   tol    : stop when ||r_i||_2 / ||b_hat||_2 <= tol (recurrence residual,
 *            R4); tol == 0 runs exactly maxit iterations (benchmark mode: a
 *            breakdown is recorded in sten_stats.event_iter and the scalars
 *            are guarded so the iteration stays finite, R7);
 *   maxit  : >= 0;
 *   x_out  : solution, this rank's points;
 *   iters  : completed iterations;
 *   res_hist: host array of >= maxit+1 doubles: ||r_i||/||b_hat||, i = 0..iters;
 *   status : STEN_CONVERGED / _MAXIT / _BREAKDOWN / _NONFINITE.
 * All work is enqueued on cuda_stream; returns after x_out, iters, res_hist
 * and status are final.  Errors: STEN_EINVAL (tol < 0 or NaN, maxit < 0),
 * STEN_ENOMEM, STEN_ECUDA, STEN_ENCCL. */
int bicgstab_solve(sten_stencil *st, int precision, const void *b, const void *x0, double tol,
                   int maxit, void *x_out, int *iters, double *res_hist, int *status,
                   void *cuda_stream);

/* n independent solves with the same operator (a serving batch): system i
 * is bicgstab_solve(b[i], x0 = NULL, tol, maxit) -> x_out[i], in order, with
 * identical results.  The host<->device traffic is pipelined: host vectors
 * (pinned memory, for the copies to be asynchronous) go through two device
 * staging buffers per direction, the upload of b[i+1] and the download of
 * x[i-1] running on a library copy stream while system i is solved.  Device
 * pointers are used in place.
 *   b, x_out : n pointers each (this rank's points, storage type of precision);
 *   iters, status : host, n ints each;
 *   res_hist : host, n * (maxit+1) doubles, row i = system i's history (NaN
 *              after iters[i]).
 * Extra device memory: 4 staging vectors.  Synchronises cuda_stream and the
 * copy stream before return.  Errors: as bicgstab_solve (a NULL vector:
 * STEN_EINVAL); n == 0 is a no-op. */
int bicgstab_solve_batch(sten_stencil *st, int precision, int n, const void *const *b, void *const *x_out,
                         double tol, int maxit, int *iters, double *res_hist, int *status, void *cuda_stream);

/* Mixed-precision iterative refinement (the remedy the paper names for the
 * fp16 plateau; R21).  Solves A x = b to an fp32
 * accuracy while the iterations run in the mixed mode:
 *   b_hat = rn32(b / a_P) (R3); x = x0 or 0 (fp32);
 *   for k = 0, 1, ...:
 *     r = b_hat - A_hat x in fp32 (fp32 coefficients, the FMA-chain SpMV of R10);
 *     res_hist[k] = ||r||_2 / ||b_hat||_2 (fp32 sums);
 *     stop: res <= tol -> STEN_CONVERGED; three consecutive steps without
 *           a 1% gain on the best residual so far -> STEN_BREAKDOWN
 *           (stagnation) - except the first time: the remaining inner
 *           solves then run the other schedule (classic <-> SR; they round
 *           differently, and on weakly dominant systems either fp16 iteration
 *           can stall where the other still gains) and the count restarts
 *           (sten_stats.handover = k; the handle's schedule is unchanged after
 *           the call; a handle whose configuration has no SR sweep stops
 *           instead); k == outer_maxit -> STEN_MAXIT;
 *           non-finite -> STEN_NONFINITE;
 *     sigma = 2^e, the power of two with max|r| <= sigma; r16 = rn16(r / sigma);
 *     d = the mixed-precision solve of A_hat d = r16 (the handle's schedule,
 *         relative tolerance inner_tol, at most inner_maxit iterations, x0 = 0);
 *     x = fma(sigma, d, x) in fp32 - unless the inner solve ended
 *         STEN_NONFINITE (its fp16 scalars overflowed, R7): then x is kept
 *         and inner_maxit halves for the rest of the call.
 *   b, x0, x_out: fp32, this rank's points (dense layout, host or device);
 *   outer_iters: refinement steps taken (k at exit); inner_iters: total
 *   mixed iterations; res_hist: host array of >= outer_maxit + 1 doubles.
 * b == 0 gives x = 0, CONVERGED, outer_iters = 0.  Errors: STEN_EINVAL (tol
 * <= 0, inner_tol < 0, outer_maxit < 0, inner_maxit < 1), STEN_ENOMEM,
 * STEN_ECUDA, STEN_ENCCL. */
int bicgstab_refine(sten_stencil *st, const void *b, const void *x0, double tol, int outer_maxit, double inner_tol,
                    int inner_maxit, void *x_out, int *outer_iters, int *inner_iters, double *res_hist,
                    int *status, void *cuda_stream);

/* Per-iteration scalars alpha_i, omega_i (i = 1..n) of the last solve, as
 * computed on the device (fp32), for parity checks.  n <= iters. */
int sten_scalar_history(sten_stencil *st, int n, double *alpha, double *omega);

/* Tuning options of a handle (the library reads no environment variables:
 * every knob is an explicit call).  Changing one drops the handle's cached
 * graphs.  Errors: STEN_EINVAL (NULL handle, unknown option, value out of
 * range).
 *   STEN_OPT_TMA_L2_PROMOTION  L2 promotion of every TMA tensor map: 0 none,
 *                              1 64 B, 2 128 B, 3 256 B (default 3)
 *   STEN_OPT_EW_CTAS_PER_SM    CTAs per SM of the element-wise kernels (H3,
 *                              init, refinement), 1..64 (default 64)
 *   STEN_OPT_COEF_PREFETCH     classic kernels with per-thread coefficient
 *                              loads (sten_set_tiling with explicit stages):
 *                              L2 prefetch distance in planes, 0..16 (default 0)
 *   STEN_OPT_SR_L2_PREFETCH    SR sweep: L2 prefetch distance, 0..16 (default 0)
 *   STEN_OPT_SR_LIGHT_LAST     SR on one slab: the last sweep of a solve
 *                              without its SpMVs (k_sr_last), 0 or 1 (default 1).
 *                              x and hist[0..maxit-1] are bitwise those of the
 *                              full sweep; hist[maxit] (and so a status decided
 *                              exactly at the tol boundary) may differ in the
 *                              last fp32 bit of its sum; the SR work vectors
 *                              (r, p, ...) are not valid after any solve
 *   STEN_OPT_CLASSIC_OVERLAP   classic schedule, decomposed (slabs >= 3
 *                              planes): the halo exchange before H1 / H2 runs
 *                              on a side stream with the two boundary planes,
 *                              concurrent with the interior planes, 0 or 1
 *                              (default 1).  Changes only the order in which
 *                              the phase sums are added.
 *   STEN_OPT_CLASSIC_FUSED     classic schedule, decomposed: 1 = fused compute +
 *                              collective over peer memory - H1 stores its
 *                              boundary planes of p', v' and H3 those of r
 *                              straight into the z-neighbours' halo planes (the
 *                              neighbour slab's buffers, or the neighbour rank's
 *                              through CUDA IPC after sten_p2p_import), and the
 *                              last CTA of every phase kernel writes the slab's
 *                              sums into every participant's inbox (one-shot
 *                              all-reduce, a 1-thread kernel per phase reads it);
 *                              no separate exchange.  Loopback slabs and 1-rank
 *                              communicators use it directly; across ranks it
 *                              needs sten_p2p_import (else the handle keeps the
 *                              NCCL exchange).  Bitwise equal to the serial
 *                              exchange (same sum order).  0 or 1 (default 0).
 *   STEN_OPT_CLASSIC_CONST     constant-coefficient handles (stencil_create_const),
 *                              classic schedule and stencil_apply with the default
 *                              tiling: 1 = the tile kernels take the six scaled
 *                              couplings as scalars and read no coefficient
 *                              tiles (H1 12 -> 6 passes, H2 10 -> 4: 17 per
 *                              iteration instead of 29);
 *                              0 = they read the coefficient arrays.  Results
 *                              are equal up to the sign of zero.  0 or 1
 *                              (default 1). */
#define STEN_OPT_TMA_L2_PROMOTION 1
#define STEN_OPT_EW_CTAS_PER_SM 2
#define STEN_OPT_COEF_PREFETCH 3
#define STEN_OPT_SR_L2_PREFETCH 4
#define STEN_OPT_SR_LIGHT_LAST 5
#define STEN_OPT_CLASSIC_OVERLAP 6
#define STEN_OPT_CLASSIC_FUSED 7
#define STEN_OPT_CLASSIC_CONST 8
int sten_set_option(sten_stencil *st, int option, int value);
int sten_get_option(sten_stencil *st, int option, int *value);

/* Record per-phase CUDA events inside the solve's graphs (enable != 0). */
int sten_set_timing(sten_stencil *st, int enable);
int sten_get_stats(sten_stencil *st, sten_stats *out);
/* Device time of each iteration of the last bicgstab_solve run with timing on,
 * in iteration order: phase 0/1/2 = the H1/H2/H3 kernel's events, -1 = their
 * sum (SR: phase 0 = the sweep, index 0 = sweep 0; phases 1, 2 read 0).
 * Writes min(cap, n) floats to out (host) and the number of iterations timed to
 * *n.  Iterations that the device state turned into no-ops (after a stop) are
 * not included; the SR solve's light last sweep (k_sr_last) is not timed.
 * Errors: STEN_EINVAL (NULL handle / n, out == NULL with cap > 0, phase not
 * in -1..2). */
int sten_iter_ms(sten_stencil *st, int phase, float *out, int cap, int *n);

/* Select the iteration schedule of later bicgstab_solve calls on this handle.
 *   STEN_SCHED_CLASSIC: Algorithm 1 exactly as printed:
 *     three fused kernels per iteration, one global reduction after each
 *     (alpha l.177, omega l.180, beta l.183).
 *   STEN_SCHED_SR: the same iteration rearranged so ONE sweep and ONE
 *     reduction serve it (R19; the paper notes it did not use a
 *     communication-hiding variant): with q = A r and y = A v the
 *     second product is t = A s = q - alpha y, and (t,s), (t,t), (rhat, r_new)
 *     expand into twelve inner products of one sweep.  Identical iterates in
 *     exact arithmetic; the rounding differs (oracle/osr.c is its oracle).
 *     Per iteration it moves 19 instead of 29 arrays through HBM.  Needs two
 *     halo planes per z-neighbour (exchanged once per iteration).
 * Errors: STEN_EINVAL. */
int sten_set_schedule(sten_stencil *st, int schedule);

/* Inner-product precision of STEN_MIXED solves (R22, R28; SURVEY
 * §8(f) NEXT-4, the "half" mode the paper sized but did not publish,
 * PAPER.md:427-441 (commented-out performance model: "16-bit mode")):
 *   STEN_DOTS_MIXED (default): fp16 products summed in fp32 (the paper's
 *     "mixed 16-bit multiply/32-bit add" instruction);
 *   STEN_DOTS_HALF: each point's product is added with ONE fp16 FMA into the
 *     running fp16 sum of its (x, y) column over one z segment (the CS-1 PE's
 *     core-local dot over its z pencil, in 16-bit); the column-segment sums
 *     are then added in fp32 (the AllReduce stays 32-bit).
 *     The segments are the chunk plan: sten_sr_segments for the SR schedule,
 *     sten_classic_segments for the classic one (one plan for H1, H2 and H3
 *     in this mode; the setup's rho_0, ||b||, hist[0] stay mixed, R28).
 * Vector arithmetic and HBM traffic are identical in both modes.  FP32
 * solves ignore the setting.  Supported with the field-coefficient operator:
 * SR with 16-B packs and the SERIAL/OVERLAP exchanges, classic on one slab
 * with the tile kernels; otherwise the solve / sweep returns
 * STEN_EUNSUPPORTED.
 * Errors: STEN_EINVAL. */
#define STEN_DOTS_MIXED 0
#define STEN_DOTS_HALF 1
int sten_set_dot_precision(sten_stencil *st, int dots);

/* The z segments of the SR chunk plan of `precision` on this rank: *n =
 * their number; z0 (host, room for cap ints, may be NULL to query *n)
 * receives each segment's first plane, relative to the rank's first plane,
 * ascending; a segment ends where the next one (or its slab) starts.  The
 * segments partition every (x, y) column into the pencils of
 * STEN_DOTS_HALF.  Errors: STEN_EINVAL (cap too small, NULL n). */
int sten_sr_segments(sten_stencil *st, int precision, int *z0, int cap, int *n);
/* The same for the classic kernels (H1, H2, apply): the first plane of every
 * z chunk a CTA of any of them marches (H2 may use longer chunks than H1 and
 * the apply: the union), per slab (the decomposed, overlapped schedule cuts
 * each slab into plane 0, the interior in chunks from plane 1, plane nz-1). */
int sten_classic_segments(sten_stencil *st, int precision, int *z0, int cap, int *n);

/* One phase of the classic schedule (Alg. 1) on caller
 * vectors, for parity tests, in the kernels and launch configuration a solve
 * uses (slabs, halo exchange and its overlap included).  The scalars are
 * rounded to fp32 (DevState), then to the working precision (R11):
 *   phase 1 (H1): out0 = p' = r + beta (p - omega v) (as fma(beta,
 *     fma(-omega, v, p), r)), out1 = v' = A p'; dots[0] = (rh, v');
 *   phase 2 (H2): out0 = s = r - alpha v (as fma(-alpha, v, r)),
 *     out1 = t = A s; dots[0] = (t, s), dots[1] = (t, t);
 * the SpMV as R10's FMA chain.  Vectors: this rank's points, dense, storage
 * type of `precision`, host or device; p and rh are read by H1 only (may be
 * NULL for H2).  dots (host) receives the fp32 sums over all slabs and ranks.
 * Synchronises cuda_stream.  Errors: STEN_EINVAL, STEN_ECUDA, STEN_ENCCL,
 * STEN_EUNSUPPORTED (p2p-only communicator). */
int sten_classic_phase(sten_stencil *st, int precision, int phase, double alpha, double omega, double beta,
                       const void *r, const void *p, const void *v, const void *rh, void *out0, void *out1,
                       float *dots, void *cuda_stream);

/* One SR sweep on caller vectors, for parity tests (oracle/osr.c
 * o16_sr_sweep / o32_sr_sweep).  With the scalars (alpha, omega, beta) of
 * the previous iteration (rounded to fp32, then to the working precision):
 *   s = r - alpha v; t = q - alpha y; x += alpha p + omega s (as
 *   fma(omega, s, fma(alpha, p, x))); r = s - omega t; p = r + beta (p - omega v);
 *   v = A p; q = A r; y = A v;
 * x, r, p, v, q, y are updated in place (this rank's points, dense layout,
 * storage type of `precision`; host or device); rh is read.  dots (host,
 * 12 floats) receives the fp32 sums (rh,v) (rh,r) (rh,q) (rh,y) (q,r) (q,v)
 * (y,r) (y,v) (q,q) (q,y) (y,y) (r,r) over this rank (all ranks when
 * decomposed).  Synchronises cuda_stream.  Errors: STEN_EINVAL, STEN_ECUDA. */
int sten_sr_sweep(sten_stencil *st, int precision, double alpha, double omega, double beta, const void *rh,
                  void *x, void *r, void *p, void *v, void *q, void *y, float *dots, void *cuda_stream);

/* How a decomposed SR sweep exchanges its halos and sums:
 *   STEN_XCHG_SERIAL : exchange (device copies / NCCL send-recv), then the sweep,
 *                      then the all-reduce of the slab sums;
 *   STEN_XCHG_OVERLAP: the exchange and the chunks that read halo planes on a side
 *                      stream, concurrent with the interior chunks;
 *   STEN_XCHG_FUSED  : ONE kernel per slab does the sweep, stores its boundary
 *                      planes straight into the z-neighbours' halo buffers (peer
 *                      memory) and deposits its sums in every participant's inbox
 *                      (one-shot all-reduce, flags with system-scope release /
 *                      acquire, inboxes double-buffered by the parity of the
 *                      sweep); a 1-thread kernel waits (bounded: ~20 s, then the
 *                      solve stops with status STEN_TIMEOUT) and runs the scalar
 *                      step.  Loopback slabs and 1-rank communicators use it
 *                      directly; across ranks it needs sten_p2p_import (else the
 *                      handle falls back to OVERLAP).
 * Default: FUSED.  SERIAL and FUSED add the slab sums in the same order: their
 * results are bitwise equal. */
/* Peer memory across ranks (one node, NVLink/NVSwitch): export writes CUDA IPC
 * handles of this rank's boundary-slab SR buffers, its inbox, its boundary
 * slabs' coefficient arrays and their classic halo'd vectors (r, p, v) for
 * `precision` (out == NULL: *bytes = the record
 * size); every rank passes all ranks' records, in rank order, to import, which
 * opens the z-neighbours' buffers and the other inboxes and selects
 * STEN_XCHG_FUSED across ranks.  With a peer-memory-only communicator
 * (sten_comm_create with unique_id == NULL) import also copies the
 * z-neighbours' boundary coefficient planes into this rank's coefficient halo
 * planes (NCCL does it at create otherwise), so every rank must have finished
 * stencil_create before any rank imports.  All ranks must import before the
 * next solve.  Errors: STEN_EINVAL, STEN_EUNSUPPORTED (> 8 ranks), STEN_ECUDA
 * (IPC). */
int sten_p2p_export(sten_stencil *st, int precision, void *out, size_t *bytes);
int sten_p2p_import(sten_stencil *st, int precision, const void *all, size_t bytes_per_rank);

#define STEN_XCHG_SERIAL 0
#define STEN_XCHG_OVERLAP 1
#define STEN_XCHG_FUSED 2
int sten_set_sr_exchange(sten_stencil *st, int mode);

/* Host lockstep for several ranks sharing ONE GPU (tests of the cross-rank
 * peer-memory path; fn == NULL turns it off).  Kernels that wait on a flag
 * written by another process's kernel are not guaranteed to make progress when
 * both processes share a GPU (a context-switch timeout, Xid 109, on B200), so
 * with a barrier set and a peer-memory-only communicator the solve runs sweep by
 * sweep (classic: iteration by iteration) without graphs and, before every
 * peer-memory all-reduce's waiting kernel, synchronises its stream and calls
 * fn(ctx) - which must return only after every rank has called it for the same
 * reduction (e.g. a gloo barrier).  The waiting kernel then finds every peer's
 * sums already deposited.  The classic schedule also calls it after every halo
 * push, so that the pushes have landed before any rank's stencil reads them; it
 * needs the barrier on a peer-memory-only communicator.  Results are bitwise
 * those of the unsynchronised path.  Errors: STEN_EINVAL. */
int sten_set_host_barrier(sten_stencil *st, void (*fn)(void *ctx), void *ctx);

/* SR kernel geometry for tuning (0 = default): by rows per tile (8 or 16),
 * stages input TMA stages, cstages coefficient stages, zc planes per CTA
 * (uniform chunks), pack bytes per thread vector (16, or 8 = twice the
 * threads per tile).  Errors: STEN_EINVAL for an unsupported combination. */
int sten_set_sr_tiling(sten_stencil *st, int precision, int by, int stages, int cstages, int zc, int pack);
/* SR chunk plan for tuning and tests: every CTA marches zc planes, except that
 * the last tail_planes planes of each slab (plus any remainder) go in chunks of
 * zc_tail (the default plan at config 3: 160, then 320 planes of 64-plane
 * chunks).  tail_planes = 0, or >= the slab's planes: uniform zc chunks (the
 * remainder in one zc_tail chunk).  Errors: STEN_EINVAL. */
int sten_set_sr_chunks(sten_stencil *st, int precision, int zc, int tail_planes, int zc_tail);

/* Tile geometry override for tuning (0 = library default).  bx: points per
 * tile in x (multiple of 8), by: rows per tile, zc: planes per CTA,
 * stages: TMA pipeline depth (2..8). */
int sten_set_tiling(sten_stencil *st, int precision, int bx, int by, int zc, int stages);

/* ------------------------------------------------- 2D 9-point SpMV ----- */
/* The paper's second kernel (Sec. "SpMV (2D)"; SURVEY
 * §8(f) NEXT-3): u = A v for a 9-point stencil on an nx x ny mesh, P = i + nx*j.
 *   coeffs[0]   : main diagonal A_P (or NULL: already unit); coeffs[1..8]: the
 *                 couplings to the (dx, dy) neighbours in the order (-1,-1)
 *                 (0,-1) (+1,-1) (-1,0) (+1,0) (-1,+1) (0,+1) (+1,+1); dense
 *                 (ny, nx) arrays of coeff_dtype, host or device, copied.
 * The operator is Jacobi-scaled as in 3D (c_d = A_d / A_P in fp64, couplings
 * leaving the mesh dropped, rounded RN to fp32 and fp16: "most
 * problems will precondition the main diagonal to unity").  Errors:
 * STEN_EINVAL, STEN_ENOMEM, STEN_ECUDA. */
typedef struct sten_stencil2d sten_stencil2d;
int stencil2d_create(int nx, int ny, const void *const coeffs[9], int coeff_dtype, void *cuda_stream,
                     sten_stencil2d **out);
/* y = A_hat x: u = x + sum_d c_d x_nb(d), one FMA per term in the order above
 * (fp32, or fp16 for STEN_MIXED; oracle/o2d.c mirrors it).  x, y: dense
 * (ny, nx), host or device, must not overlap.  Synchronises cuda_stream. */
int stencil2d_apply(sten_stencil2d *st, int precision, const void *x, void *y, void *cuda_stream);
/* device time (ms) of the last apply's kernels (CUDA events around them), or
 * of the last bicgstab2d_solve from S1 to its last iteration (b already in) */
int stencil2d_last_ms(sten_stencil2d *st, double *ms);
void stencil2d_destroy(sten_stencil2d *st);

/* The paper's tiled form of the 2D SpMV ("we map a
 * rectangular region of the mesh of v to each core, and store all elements of
 * the corresponding columns of A.  After multiplication of the local v with
 * the local A we have generated products in an output halo that must be sent
 * to neighboring tiles ... We complete a round of send and add in one
 * direction, then a round for the other direction").  DESIGN.md R24 fixes
 * what the paper leaves open: tile (a, b) of a tiles_x x tiles_y grid owns
 * columns [floor(a nx / tiles_x), floor((a+1) nx / tiles_x)) and rows likewise;
 * each tile forms, from ITS OWN v only, v_P + the products of its in-tile
 * neighbours at its points and the products landing one point outside it (its
 * output-halo ring); the x round adds the left, then the right neighbour's
 * halo column into a tile's edge columns over its grown rows (corners ride
 * along), then the y round adds the lower, then the upper neighbour's halo
 * row.  The tiles are loopback partitions of one device (each reads only its
 * own v and writes only its own u and ring; the rounds read the neighbours'
 * rings, the data a multi-device layout would send).  Results are bitwise
 * those of oracle/o2d.c o32/o16_apply9_tiles.  After this call
 * stencil2d_apply uses the tiled form; 1 x 1 restores the gather.
 * Errors: STEN_EINVAL (tiles_x not in 1..nx, tiles_y not in 1..ny),
 * STEN_ENOMEM.  Synchronises the device. */
int stencil2d_set_tiles(sten_stencil2d *st, int tiles_x, int tiles_y);

/* BiCGStab on the 2D operator (each core holds "a matrix, halo,
 * and vector (as well as all terms needed for BiCG)"; Alg. 1, PAPER.md:172-186,
 * with the 9-point operator, R25).  Arguments, precisions, status,
 * tol / maxit conventions and errors as bicgstab_solve; b, x0 (NULL: 0),
 * x_out: dense (ny, nx) vectors of the precision's type, host or device;
 * res_hist: host, maxit+1 doubles.  With a diagonal given at create, b_hat =
 * b / A_P (R3) and the residuals refer to the scaled system.  Schedule: H1 =
 * p' = r + beta (p - omega v), v' = A p', (rhat, v'); H2 = s = r - alpha v',
 * t = A s, (t, s), (t, t); H3 = x, r updates, (rhat, r), (r, r) - fused
 * kernels, 33 passes per iteration.  With tiles > 1 x 1 (stencil2d_set_tiles)
 * the SpMV is the paper's tiled output-halo form and the phases run unfused
 * around it (update, tiled SpMV, dots; oracle/o2d.c o2d16_bicgstab_tiles).
 * Synchronises cuda_stream. */
int bicgstab2d_solve(sten_stencil2d *st, int precision, const void *b, const void *x0, double tol, int maxit,
                     void *x_out, int *iters, double *res_hist, int *status, void *cuda_stream);
/* per-phase device timing of the 2D solve (CUDA events around H1, H2, H3 of
 * every iteration; off by default): mean ms of each phase over the
 * `iterations` iterations of the last timed solve */
int stencil2d_set_timing(sten_stencil2d *st, int enable);
int stencil2d_phase_ms(sten_stencil2d *st, double ms[3], long long *iterations);

#ifdef __cplusplus
}
#endif
#endif /* STEN_H */
