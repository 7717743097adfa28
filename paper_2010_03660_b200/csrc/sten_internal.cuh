// sten_internal.cuh - shared definitions of libsten.so (B200 / sm_100a).
//
// Device-side solver state, packed fp32x4 / fp16x8 vectors, TMA + mbarrier
// PTX wrappers, block/grid reductions and the scalar steps of Algorithm 1
// (PAPER.md:176-184).  Nothing here is shared with oracle/ (R13 in DESIGN.md).
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/sten.h"

namespace sten {

// ----------------------------------------------------------------------------
// Solver state living in device memory.  Written only by single-thread
// finalize code (last CTA of a reduction or the scalar kernel), read by every
// kernel of the next phase in stream order.
struct DevState {
  float rho, alpha, omega, beta;   // current BiCGStab scalars (fp32, R12)
  double nb;                       // ||b_hat||_2
  double tol;                      // stopping tolerance (0 = benchmark mode)
  int it;                          // completed iterations
  int maxit;
  int stop;                        // 1: later phases are no-ops
  int status;                      // STEN_* status when stop == 1
  int ev;                          // first event code (-1: none)
  int ev_it;                       // iteration of the first event
  int zero_x;                      // b_hat == 0: x must be returned as 0
  int sweep;                       // SR schedule: index of the next sweep
  int light;                       // SR: the last sweep (i = maxit) is k_sr_last, not k_sr
  int half;                        // mixed mode: scalars must be finite in fp16 (R7)
  double *hist;                    // [maxit+1] ||r_i|| / ||b_hat||
  float *ahist, *whist;            // [maxit+1] alpha_i, omega_i
};

enum Phase { PH_INIT = 0, PH_H1 = 1, PH_H2 = 2, PH_H3 = 3, PH_SR = 4 };
enum Mode { MODE_APPLY = 0, MODE_H1 = 1, MODE_H2 = 2 };
constexpr int kMaxDots = 12;  // SR sweep: 12 inner products (classic phases use 1-3)

// One participant's inbox of the peer-memory all-reduce (SR):
// sums[slot][kMaxDots] and flags[slot] (= the sequence number of the sweep
// whose sums landed in that slot).
constexpr int kMaxPeers = 8;
struct P2PBox {
  float *sums;
  unsigned *flags;
};

// Grid reduction plumbing of one kernel launch.
struct Reduce {
  float *partials;      // [gridDim.x * kMaxDots]
  unsigned *counter;    // zero between launches (reset by the last CTA)
  float *slab_out;      // decomposed solve: write the slab's sums here ...
  DevState *st;         // ... else finalize the scalars directly
  // peer-memory all-reduce (p2p_n > 0): the last CTA writes its sums into
  // slot p2p_slot of every inbox, then the flag (*p2p_seq + 1), after a
  // system-scope fence that also publishes the kernel's remote halo stores.
  // Inboxes are double-buffered by the parity of the sequence number
  // (p2p_nslots slots each), so a rank that has passed reduction i can deposit
  // its reduction-(i+1) sums while a slower rank still reads reduction i's.
  int p2p_n, p2p_slot, p2p_nslots;
  const unsigned *p2p_seq;
  P2PBox p2p[kMaxPeers];
};

// Geometry of one z-slab in the internal layout: planes 0 and nz+1 are the
// halo planes, rows have `pitch` elements (pitch % 8 == 0, x >= nx padded
// with zeros).  Coefficient arrays use the same rows but no halo planes.
struct Geom {
  int nx, ny, nz, pitch;
  long long plane;      // pitch * ny elements
};

// Arguments of the TMA z-march stencil kernel.
struct alignas(64) StencilArgs {
  CUtensorMap tm_in[3];   // halo'd inputs: box (BX+2H) x (BY+2) x 1 into shared memory
  CUtensorMap tm_c[6];    // coefficients xm,xp,ym,yp,zm,zp: box BX x BY x 1 (L2 prefetch)
  CUtensorMap tm_aux;     // rhat (H1): box BX x BY x 1 (L2 prefetch)
  const void *cptr[6];    // coefficient arrays (plane 0 at k = 0, no halo planes)
  const void *aux;        // rhat (H1), halo layout
  void *out0;             // APPLY: y   H1: v_new   H2: t
  void *out1;             // H1: p_new  H2: s
  Geom g;
  int zc, tiles_x, tiles_y;
  int zlo, zhi;           // planes [zlo, zhi) of the slab, in chunks of zc from zlo
  int pf;                 // L2 prefetch distance of the coefficient tiles (planes; 0 = off)
  // fused exchange (H1): interior plane 0 of out0 / out1 also to peer_lo[i] (the lower z-neighbour's
  // top halo plane), plane nz-1 to peer_hi[i] (the upper one's bottom halo plane); null: none
  void *peer_lo[2], *peer_hi[2];
  // constant-coefficient operator (stencil_create_const, NEXT-4): cc != 0 selects the kernels that
  // take the six scaled couplings as scalars (fp32 / fp16 bits) and read no coefficient tiles
  int cc;
  float cf32[6];
  uint16_t cf16[6];
  Reduce red;
};

struct EwArgs {           // element-wise kernels (H3, INIT)
  const void *x, *p, *s, *t, *rhat;   // H3 inputs
  void *xo, *ro;                       // H3 outputs
  const void *bw; const double *aP; const void *ax; // INIT inputs (ax = A x0 or null)
  void *r, *rh, *p0, *v0;              // INIT outputs
  long long nvec;                      // vectors of VEC elements holding mesh points
  long long rows;                      // ny * nz rows of the interior range
  int vpr;                             // vectors per row that hold points (ceil(nx/VEC))
  int pitch;                           // row pitch in elements (multiple of 64: 128-B rows)
  // fused exchange (H3): r's interior plane 0 also to peer_lo_r (the lower z-neighbour's top halo
  // plane), plane nz-1 to peer_hi_r; plane_elems = elements per plane, nzp = interior planes
  void *peer_lo_r, *peer_hi_r;
  long long plane_elems;
  int nzp;
  Reduce red;
};

// ---------------------------------------------------------------- packs --
// Two IEEE fp32 fused multiply-adds in one instruction (FFMA2, sm_100): d_i = rn(a_i * b_i + c_i),
// lane for lane the result of __fmaf_rn - half the issue slots of the fp32 element-wise work.
#ifndef STEN_FFMA2
#define STEN_FFMA2 1  // 0: two scalar FFMA (the experiment baseline; bitwise the same results)
#endif
__device__ __forceinline__ void ffma2(float &d0, float &d1, float a0, float a1, float b0, float b1, float c0,
                                      float c1) {
  if (!STEN_FFMA2) {
    d0 = __fmaf_rn(a0, b0, c0);
    d1 = __fmaf_rn(a1, b1, c1);
    return;
  }
  unsigned long long ra, rb, rc, rd;
  asm("mov.b64 %0, {%1, %2};" : "=l"(ra) : "f"(a0), "f"(a1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(rb) : "f"(b0), "f"(b1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(rc) : "f"(c0), "f"(c1));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(rd) : "l"(ra), "l"(rb), "l"(rc));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(d0), "=f"(d1) : "l"(rd));
}

template <typename T> struct Pack;

template <> struct Pack<float> {
  static constexpr int VEC = 4;
  float v[4];
  using S = float;
  static __device__ __forceinline__ Pack ld(const float *p) {
    float4 q = *reinterpret_cast<const float4 *>(p);
    return Pack{{q.x, q.y, q.z, q.w}};
  }
  static __device__ __forceinline__ Pack ldg(const float *p) {
    float4 q = __ldcs(reinterpret_cast<const float4 *>(p));
    return Pack{{q.x, q.y, q.z, q.w}};
  }
  __device__ __forceinline__ void st(float *p) const {
    *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
  static __device__ __forceinline__ Pack zero() { return Pack{{0.f, 0.f, 0.f, 0.f}}; }
  // neighbour at x-1 of each lane: (l3, c0, c1, c2); at x+1: (c1, c2, c3, r0)
  static __device__ __forceinline__ Pack shl(const Pack &l, const Pack &c) {
    return Pack{{l.v[3], c.v[0], c.v[1], c.v[2]}};
  }
  static __device__ __forceinline__ Pack shr(const Pack &c, const Pack &r) {
    return Pack{{c.v[1], c.v[2], c.v[3], r.v[0]}};
  }
  static __device__ __forceinline__ Pack fma(const Pack &a, const Pack &b, const Pack &c) {
    Pack o;
#pragma unroll
    for (int i = 0; i < 4; i += 2) ffma2(o.v[i], o.v[i + 1], a.v[i], a.v[i + 1], b.v[i], b.v[i + 1], c.v[i], c.v[i + 1]);
    return o;
  }
  static __device__ __forceinline__ S scalar(float a) { return a; }
  static __device__ __forceinline__ S neg(S a) { return -a; }
  static __device__ __forceinline__ Pack fmas(S a, const Pack &b, const Pack &c) {
    Pack o;
#pragma unroll
    for (int i = 0; i < 4; i += 2) ffma2(o.v[i], o.v[i + 1], a, a, b.v[i], b.v[i + 1], c.v[i], c.v[i + 1]);
    return o;
  }
  static __device__ __forceinline__ Pack sub(const Pack &a, const Pack &b) {
    Pack o;
#pragma unroll
    for (int i = 0; i < 4; ++i) o.v[i] = __fsub_rn(a.v[i], b.v[i]);
    return o;
  }
  // acc += a_i * b_i in lane order, fp32 FMA
  __device__ __forceinline__ float dot(const Pack &b, float acc) const {
#pragma unroll
    for (int i = 0; i < 4; ++i) acc = __fmaf_rn(v[i], b.v[i], acc);
    return acc;
  }
  // four independent partial sums (short dependency chains)
  __device__ __forceinline__ void dot4(const Pack &b, float (&acc)[4]) const {
    ffma2(acc[0], acc[1], v[0], v[1], b.v[0], b.v[1], acc[0], acc[1]);
    ffma2(acc[2], acc[3], v[2], v[3], b.v[2], b.v[3], acc[2], acc[3]);
  }
  __device__ __forceinline__ float mdot(const Pack &b, float acc) const { return dot(b, acc); }
};

template <> struct Pack<__half> {
  static constexpr int VEC = 8;
  uint32_t w[4];  // 4 x half2, lane 2i in the low half of w[i]
  using S = __half2;
  static __device__ __forceinline__ Pack ld(const __half *p) {
    uint4 q = *reinterpret_cast<const uint4 *>(p);
    return Pack{{q.x, q.y, q.z, q.w}};
  }
  static __device__ __forceinline__ Pack ldg(const __half *p) {
    uint4 q = __ldcs(reinterpret_cast<const uint4 *>(p));
    return Pack{{q.x, q.y, q.z, q.w}};
  }
  __device__ __forceinline__ void st(__half *p) const {
    *reinterpret_cast<uint4 *>(p) = make_uint4(w[0], w[1], w[2], w[3]);
  }
  static __device__ __forceinline__ Pack zero() { return Pack{{0u, 0u, 0u, 0u}}; }
  // x-1 neighbour of lanes (2i, 2i+1) = (lane 2i-1, lane 2i): low <- prev.hi, high <- cur.lo
  static __device__ __forceinline__ Pack shl(const Pack &l, const Pack &c) {
    return Pack{{__byte_perm(l.w[3], c.w[0], 0x5432), __byte_perm(c.w[0], c.w[1], 0x5432),
                 __byte_perm(c.w[1], c.w[2], 0x5432), __byte_perm(c.w[2], c.w[3], 0x5432)}};
  }
  static __device__ __forceinline__ Pack shr(const Pack &c, const Pack &r) {
    return Pack{{__byte_perm(c.w[0], c.w[1], 0x5432), __byte_perm(c.w[1], c.w[2], 0x5432),
                 __byte_perm(c.w[2], c.w[3], 0x5432), __byte_perm(c.w[3], r.w[0], 0x5432)}};
  }
  static __device__ __forceinline__ __half2 h2(uint32_t u) { return *reinterpret_cast<const __half2 *>(&u); }
  static __device__ __forceinline__ uint32_t u32(__half2 h) { return *reinterpret_cast<const uint32_t *>(&h); }
  static __device__ __forceinline__ Pack fma(const Pack &a, const Pack &b, const Pack &c) {
    Pack o;
#pragma unroll
    for (int i = 0; i < 4; ++i) o.w[i] = u32(__hfma2(h2(a.w[i]), h2(b.w[i]), h2(c.w[i])));
    return o;
  }
  static __device__ __forceinline__ S scalar(float a) { return __float2half2_rn(a); }
  static __device__ __forceinline__ S neg(S a) { return __hneg2(a); }
  static __device__ __forceinline__ Pack fmas(S a, const Pack &b, const Pack &c) {
    Pack o;
#pragma unroll
    for (int i = 0; i < 4; ++i) o.w[i] = u32(__hfma2(a, h2(b.w[i]), h2(c.w[i])));
    return o;
  }
  static __device__ __forceinline__ Pack sub(const Pack &a, const Pack &b) {
    Pack o;
#pragma unroll
    for (int i = 0; i < 4; ++i) o.w[i] = u32(__hsub2(h2(a.w[i]), h2(b.w[i])));
    return o;
  }
  // fp16 x fp16 products are exact in fp32; accumulate in fp32
  __device__ __forceinline__ float dot(const Pack &b, float acc) const {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 x = __half22float2(h2(w[i])), y = __half22float2(h2(b.w[i]));
      acc = __fmaf_rn(x.x, y.x, acc);
      acc = __fmaf_rn(x.y, y.y, acc);
    }
    return acc;
  }
  __device__ __forceinline__ void dot4(const Pack &b, float (&acc)[4]) const {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 x = __half22float2(h2(w[i])), y = __half22float2(h2(b.w[i]));
      acc[i] = __fmaf_rn(x.x, y.x, acc[i]);
      acc[i] = __fmaf_rn(x.y, y.y, acc[i]);
    }
  }
  // acc += a_i * b_i in lane order with the sm_100 mixed FMA (fma.rn.f32.f16:
  // fp16 x fp16 product, exact, added to fp32 with one rounding) - the same
  // value as dot(), one instruction per element
  __device__ __forceinline__ float mdot(const Pack &b, float acc) const {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm("{\n .reg .b16 al, ah, bl, bh;\n mov.b32 {al, ah}, %1;\n mov.b32 {bl, bh}, %2;\n"
          " fma.rn.f32.f16 %0, al, bl, %0;\n fma.rn.f32.f16 %0, ah, bh, %0;\n}"
          : "+f"(acc)
          : "r"(w[i]), "r"(b.w[i]));
    return acc;
  }
};

__device__ __forceinline__ float sum4(const float (&a)[4]) { return (a[0] + a[1]) + (a[2] + a[3]); }

// ------------------------------------------------------------- PTX: TMA --
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  uint32_t a = smem_u32(bar);
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!ok);
}
// 1D bulk copy global -> shared, completion on an mbarrier (complete_tx)
// the same with an L2 cache-policy hint (createpolicy), e.g. evict-first for data read exactly once
__device__ __forceinline__ void bulk_g2s_hint(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int x, int y, int z,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
// the same with an L2 eviction-priority policy (createpolicy)
__device__ __forceinline__ void tma_load_3d_hint(void *dst, const CUtensorMap *map, int x, int y, int z,
                                                 uint64_t *bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap *map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// ------------------------------------------------------------ reductions --
// Deterministic: fixed shuffle tree, fixed warp order.  Result valid in thread 0.
template <int ND>
__device__ __forceinline__ void block_sum(float (&v)[ND], float *scratch) {
#pragma unroll
  for (int d = 0; d < ND; ++d)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[d] += __shfl_xor_sync(0xffffffffu, v[d], o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();  // scratch may still be read by a previous call
  if (lane == 0)
#pragma unroll
    for (int d = 0; d < ND; ++d) scratch[warp * ND + d] = v[d];
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int d = 0; d < ND; ++d) {
      float x = lane < nw ? scratch[lane * ND + d] : 0.0f;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      v[d] = x;
    }
  }
}

// ------------------------------------------------ Algorithm 1 scalar steps --
// R6-R8 of DESIGN.md.  Run by ONE thread.
__device__ __forceinline__ void st_event(DevState *st, int code, int i, bool before_update) {
  if (st->ev < 0) {
    st->ev = code;
    st->ev_it = i;
  }
  if (st->tol > 0.0) {
    st->stop = 1;
    st->status = code;
    (void)before_update;  // `it` is only advanced by the H3 step
  }
}

// S1: rho = (rhat, r0), ||b_hat||, hist[0]  (Alg. 1 l.174)
__device__ __forceinline__ void fin_init(DevState *st, float rho, float bb, float rr) {
  st->rho = rho;
  st->alpha = 0.f;
  st->omega = 0.f;
  st->beta = 0.f;  // first H1 then computes p = r exactly (p_0 := r_0)
  double nb = sqrt((double)bb);
  st->nb = nb;
  if (nb == 0.0) {
    st->hist[0] = 0.0;
    st->zero_x = 1;
    st->stop = 1;
    st->status = STEN_CONVERGED;
    return;
  }
  double h0 = sqrt((double)rr) / nb;
  st->hist[0] = h0;
  if (st->tol > 0.0 && h0 <= st->tol) {
    st->stop = 1;
    st->status = STEN_CONVERGED;
  }
}

// A scalar is usable if finite in the working precision: in mixed mode it is
// rounded to fp16 before the AXPYs, and |s| >= 65520 rounds to Inf (R7).
__device__ __forceinline__ bool usable(const DevState *st, float s) {
  return isfinite(s) && (!st->half || fabsf(s) < 65520.0f);
}

// H1: alpha_i = rho_i / (rhat, s_i)   (l.177)
__device__ __forceinline__ void fin_h1(DevState *st, float sigma) {
  int i = st->it + 1;
  float alpha = st->rho / sigma;
  if (sigma == 0.0f || !usable(st, alpha)) {
    alpha = 0.0f;
    st_event(st, isfinite(sigma) ? STEN_BREAKDOWN : STEN_NONFINITE, i, true);
  }
  st->alpha = alpha;
  st->ahist[i] = alpha;
}

// H2: omega_i = (q_i, y_i) / (y_i, y_i)   (l.180)
__device__ __forceinline__ void fin_h2(DevState *st, float ts, float tt) {
  int i = st->it + 1;
  float omega = 0.0f;  // tt == 0: s == 0, x += alpha p is exact (R8)
  if (tt != 0.0f) {
    omega = ts / tt;
    if (!usable(st, omega)) {
      omega = 0.0f;
      st_event(st, STEN_NONFINITE, i, true);
    }
  }
  st->omega = omega;
  st->whist[i] = omega;
}

// H3: residual history, beta_i = (alpha/omega) (rhat,r_{i+1})/(rhat,r_i)  (l.183)
__device__ __forceinline__ void fin_h3(DevState *st, float rhon, float rr) {
  int i = st->it + 1;
  double h = sqrt((double)rr) / st->nb;
  st->hist[i] = h;
  st->it = i;
  int code = -1;
  if (!isfinite(rr) || !isfinite(rhon)) code = STEN_NONFINITE;
  else if (rr == 0.0f && rhon != 0.0f) code = STEN_BREAKDOWN;  // R23: (r,r) underflowed, r != 0
  else if (rr == 0.0f || (st->tol > 0.0 && h <= st->tol)) code = STEN_CONVERGED;
  else if (st->omega == 0.0f || rhon == 0.0f) code = STEN_BREAKDOWN;
  float beta = (rhon / st->rho) * (st->alpha / st->omega);
  if (!usable(st, beta)) beta = 0.0f;
  st->beta = beta;
  st->rho = rhon;
  if (code >= 0) st_event(st, code, i, false);
}

// SR schedule (R19, oracle/osr.c): the scalar step after sweep i,
// from its twelve inner products d = (rh,v) (rh,r) (rh,q) (rh,y) (q,r) (q,v)
// (y,r) (y,v) (q,q) (q,y) (y,y) (r,r).  fp32 arithmetic, no contraction, in
// the oracle's operation order.
__device__ __forceinline__ void fin_sr(DevState *st, const float *d) {
  const int i = st->sweep;
  const float sigma = d[0], rho = d[1], phi = d[2], psi = d[3];
  const float qr = d[4], qv = d[5], yr = d[6], yv = d[7], qq = d[8], qy = d[9], yy = d[10], rr = d[11];
  const double h = sqrt((double)rr) / st->nb;
  st->hist[i] = h;  // ||r_i|| / ||b_hat||, R4
  st->it = i;
  st->sweep = i + 1;
  int code = -1;
  if (!isfinite(rr) || !isfinite(rho)) code = STEN_NONFINITE;
  else if (rr == 0.0f && rho != 0.0f) code = STEN_BREAKDOWN;  // R23: (r,r) underflowed, r != 0
  else if (rr == 0.0f || (st->tol > 0.0 && h <= st->tol)) code = STEN_CONVERGED;
  else if (i > 0 && (st->omega == 0.0f || rho == 0.0f)) code = STEN_BREAKDOWN;
  if (code >= 0) st_event(st, code, i, false);
  if (st->stop || i >= st->maxit) return;
  float alpha = __fdiv_rn(rho, sigma);  // l.177
  if (sigma == 0.0f || !usable(st, alpha)) {
    alpha = 0.0f;
    st_event(st, isfinite(sigma) ? STEN_BREAKDOWN : STEN_NONFINITE, i + 1, true);
  }
  const float a2 = __fmul_rn(alpha, alpha);
  const float ts = __fadd_rn(__fsub_rn(__fsub_rn(qr, __fmul_rn(alpha, qv)), __fmul_rn(alpha, yr)), __fmul_rn(a2, yv));
  const float tt = __fadd_rn(__fsub_rn(qq, __fmul_rn(__fmul_rn(2.0f, alpha), qy)), __fmul_rn(a2, yy));
  float omega = 0.0f;  // tt <= 0: t = A s = 0, s = 0 (R8)
  bool nf = !isfinite(tt);
  if (tt > 0.0f) omega = __fdiv_rn(ts, tt);  // l.180
  if (nf || !usable(st, omega)) {
    omega = 0.0f;
    st_event(st, STEN_NONFINITE, i + 1, true);
  }
  const float rhon = __fsub_rn(__fsub_rn(rho, __fmul_rn(alpha, sigma)), __fmul_rn(omega, __fsub_rn(phi, __fmul_rn(alpha, psi))));
  float beta = __fmul_rn(__fdiv_rn(rhon, rho), __fdiv_rn(alpha, omega));  // l.183
  if (!usable(st, beta)) beta = 0.0f;
  st->alpha = alpha;
  st->omega = omega;
  st->beta = beta;
  st->rho = rho;
  st->ahist[i + 1] = alpha;
  st->whist[i + 1] = omega;
}

template <int PH>
__device__ __forceinline__ void finalize_phase(DevState *st, const float *s) {
  if (PH == PH_INIT) fin_init(st, s[0], s[1], s[2]);
  else if (PH == PH_H1) fin_h1(st, s[0]);
  else if (PH == PH_H2) fin_h2(st, s[0], s[1]);
  else if (PH == PH_H3) fin_h3(st, s[0], s[1]);
  else fin_sr(st, s);
}

__device__ __forceinline__ bool st_idle(const DevState *st) { return st->stop || st->it >= st->maxit; }
__device__ __forceinline__ bool sr_idle(const DevState *st) {
  return st->stop || st->sweep > st->maxit || (st->light && st->sweep == st->maxit);
}

// Grid-level end of a reduction: every CTA deposits its block sum; the last
// CTA to arrive sums the deposits in CTA order (deterministic) and either
// finalizes the phase or writes the slab's sums for the cross-slab step.
// peer_stores: this CTA may have stored into peer memory (halo planes of a z-neighbour); only then
// does it need the system-scope fence before its ticket (the last CTA fences before its flags anyway)
template <int ND, int PH>
__device__ __forceinline__ void grid_reduce_finalize(float (&v)[ND], const Reduce &red, float *scratch,
                                                     bool peer_stores = true) {
  block_sum<ND>(v, scratch);
  __shared__ int am_last;
  if (red.p2p_n > 0 && peer_stores) {
    __syncthreads();
    __threadfence_system();  // this CTA's stores to peer memory (halo planes) are visible before its ticket
  }
  if (threadIdx.x == 0) {
#pragma unroll
    for (int d = 0; d < ND; ++d) red.partials[blockIdx.x * kMaxDots + d] = v[d];
    __threadfence();
    unsigned t = atomicAdd(red.counter, 1u);
    am_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  float s[ND];
#pragma unroll
  for (int d = 0; d < ND; ++d) s[d] = 0.0f;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x)
#pragma unroll
    for (int d = 0; d < ND; ++d) s[d] += __ldcg(&red.partials[b * kMaxDots + d]);
  block_sum<ND>(s, scratch);
  if (threadIdx.x == 0) {
    *red.counter = 0u;
    if (red.p2p_n > 0) {  // one-shot all-reduce through peer memory: deposit, fence, flag
      const unsigned seq = *red.p2p_seq + 1u;
      const int slot = (int)(seq & 1u) * red.p2p_nslots + red.p2p_slot;
      for (int r = 0; r < red.p2p_n; ++r)
#pragma unroll
        for (int d = 0; d < ND; ++d) red.p2p[r].sums[slot * kMaxDots + d] = s[d];
      __threadfence_system();
      for (int r = 0; r < red.p2p_n; ++r)
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(red.p2p[r].flags + slot), "r"(seq) : "memory");
    } else if (red.slab_out) {
#pragma unroll
      for (int d = 0; d < ND; ++d) red.slab_out[d] = s[d];
    } else {
      float full[kMaxDots];
#pragma unroll
      for (int d = 0; d < kMaxDots; ++d) full[d] = d < ND ? s[d] : 0.0f;
      finalize_phase<PH>(red.st, full);
    }
  }
}

// ----------------------------------------------------------- host side --
// kernels.cu
// stencil.cu: x extent of a tile is fixed per precision (128-B rows of a tile:
// 128 fp16 / 64 fp32 points); rows per tile (by) and TMA stages are template
// instances chosen at run time.
template <typename T> constexpr int tile_bx() { return sizeof(T) == 2 ? 128 : 64; }
bool stencil_config_ok(int by, int stages, int cstages = 0);
template <typename T>
int stencil_launch(int mode, const StencilArgs &a, int by, int stages, int cstages, cudaStream_t s);
// the fused-exchange instance (MODE_H1 with peer stores), default geometry only
template <typename T> int stencil_launch_fused(const StencilArgs &a, int by, int stages, int cstages, cudaStream_t s);
// half dots (R22, R28): H1 / H2 with their inner products as fp16 column pencils over the chunk
int stencil_launch_half(int mode, const StencilArgs &a, int by, int stages, int cstages, cudaStream_t s);
// the classic H3 marching z over the same chunks, its two inner products as fp16 column pencils
struct H3zArgs {
  const void *x, *p, *s, *t, *rh;  // interior plane 0
  void *xo, *ro;
  Geom g;
  int zc, tiles_x, tiles_y;
  Reduce red;
};
int h3z_half_launch(const H3zArgs &a, int by, cudaStream_t s);
int h3z_half_grid(int sm_count, const H3zArgs &a);  // CTAs of h3z_half_launch
template <typename T> size_t stencil_smem_bytes(int mode, int by, int stages);
template <typename T> int stencil_threads(int by);
// row-strip kernel (no x halo): a CTA owns `by` full rows; used when a row fits
constexpr int kRowBoxElems = 64;
bool rows_config_ok(int by, int stages);
size_t rows_smem_bytes(int mode, int esz, int pitch, int by, int stages);
template <typename T> int rows_launch(int mode, const StencilArgs &a, int by, int stages, cudaStream_t s);
template <typename T> int rows_threads(int nx, int by);
template <typename T> int h3_launch(const EwArgs &a, int grid, int threads, cudaStream_t s);
template <typename T> int init_launch(const EwArgs &a, int grid, int threads, cudaStream_t s);
int scalars_launch(int phase, const float *slab_sums, int nslabs, DevState *st, cudaStream_t s);
// phase PH_SR (the fused SR sweep's all-reduce) or PH_INIT (a p2p-only communicator's init)
int p2p_fin_launch(int phase, P2PBox inbox, int nslots, unsigned *seq, DevState *st, cudaStream_t s);
// deposit the nslabs slab sums into slots base .. base+nslabs-1 of every inbox (peer-memory all-reduce)
int p2p_put_launch(const float *slab_sums, int nslabs, int base, int nslots, const P2PBox *boxes, int nboxes,
                   const unsigned *seq, cudaStream_t s);
int slabsum_launch(const float *slab_sums, int nslabs, float *out, cudaStream_t s);
// Iterative refinement (bicgstab_refine, R21): fp32 outer steps
// around the mixed inner solve.  All pointers at interior plane 0.
struct IrArgs {
  const float *b;        // ir_bhat: user b (fp32)      ir_resid: b_hat (fp32)
  const double *aP;      // ir_bhat: a_P or null
  const float *ax;       // ir_resid: A x (fp32)
  float *r;              // ir_bhat: b_hat out        ir_resid: r = b_hat - A x   ir_scale: r in
  __half *r16;           // ir_scale: r / sigma in fp16
  const __half *d16;     // ir_update: inner solution
  float *x;              // ir_update: x += sigma d
  unsigned *amax;        // ir_resid: atomicMax of |r| (float bits)
  float *sigma;          // ir_scale writes, ir_update reads: 2^e >= max|r|
  long long n;           // elements of the interior range (linear, padding holds zeros)
  Reduce red;            // ir_resid: (r, r) deposited in red.slab_out
};
int ir_launch(int which, const IrArgs &a, int grid, cudaStream_t s);
// pitched device-to-device copy of h x d rows of wbytes (kernels.cu); cudaErrorNotSupported if odd-aligned
int copy_rows_launch(void *dst, size_t dpitch, size_t dysize, const void *src, size_t spitch, size_t sysize,
                     size_t wbytes, size_t h, size_t d, int sms, cudaStream_t s);
enum { IR_BHAT = 0, IR_RESID = 1, IR_SCALE = 2, IR_UPDATE = 3 };

// sr.cu: the single-reduction sweep kernel (one launch per iteration)
struct alignas(64) SrArgs {
  CUtensorMap tm_in[5];   // r, p, v, q, y of the previous sweep: box (BX+2H) x (BY+4), 2 halo planes
  CUtensorMap tm_c[6];    // coefficients with one halo plane: box (BX+2H) x (BY+2)
  CUtensorMap tm_x;       // x (2 halo planes): box BX x BY, arrives with the input stage
  CUtensorMap tm_rh;      // r_hat, the same box
  void *x;                // in place (own points only), interior plane 0
  const void *rh;         // shadow residual, interior plane 0
  void *out[5];           // r, p, v, q, y of this sweep, interior plane 0
  Geom g;
  int zc, tiles_x, tiles_y;
  int nbig;               // chunks [0, nbig) have zc planes; the rest cover
  int zc_tail;            // [nbig*zc, nz) in zc_tail-plane chunks (fills the tail wave)
  int nch;                // chunks in this launch: its i-th chunk is i (i < ch_lo_n), else
  int ch_lo_n, ch_hi0;    // ch_hi0 + i - ch_lo_n (all / interior / boundary subsets)
  // constant-coefficient operator (stencil_create_const): the six scaled
  // couplings as scalars, no coefficient streams; v' is masked to zero outside
  // the global mesh (planes below/above exist only at slab interfaces)
  float cf32[6];
  unsigned short cf16[6];
  int has_below, has_above;
  int l2pf;               // input planes prefetched into L2 beyond the TMA stages (0: off)
  // fused halo exchange (peer memory): this sweep's planes 0, 1 also go to the
  // lower z-neighbour's top halo planes, planes nz-2, nz-1 to the upper one's
  // bottom halo planes (null: no neighbour or not fused).  Base = the
  // neighbour buffer's element of OUR plane 0 (resp. nz-2), same pitch/plane.
  void *peer_lo[5], *peer_hi[5];
  Reduce red;
};
bool sr_config_ok(int by, int stages, int cstages, int pack);
bool sr_hd_config_ok(int by, int stages, int cstages, int pack);
// the last SR sweep (i = maxit) without its three SpMVs: x_maxit, r_maxit and the two sums
// the scalar step still reads, (rhat, r) and (r, r) -- 8 passes instead of 19
struct SrLastArgs {
  void *x;                              // in place
  const void *rh, *r, *p, *v, *q, *y;   // the set sweep maxit reads
  long long nvec;                       // 16-B vectors of the interior range (padding holds zeros)
  Reduce red;
};
template <typename T> int sr_last_launch(const SrLastArgs &a, int grid, cudaStream_t s);
template <typename T>
int sr_launch(const SrArgs &a, int by, int stages, int cstages, int pack, bool cc, bool hd, cudaStream_t s);
template <typename T> size_t sr_smem_bytes(int by, int stages, int cstages, int pack);
template <typename T> int sr_threads(int by, int pack);

// sten2d.cu: the 2D 9-point SpMV and BiCGStab (NEXT-3)
struct alignas(64) Apply9Args {
  CUtensorMap tm_v;       // v: box (BX + 2H) x (BY + 2), one plane
  const void *c[8];       // scaled couplings, rows of `pitch`
  void *u;
  const unsigned char *xm, *ym;  // tiled product (R24): per column / row, bit 0 = the -1 neighbour
                                 // is in the same tile, bit 1 = the +1 neighbour (null: gather)
  int nx, ny, pitch, tiles_x;
};
// the tiled SpMV's output-halo ring and its two rounds (TX x TY tiles)
struct Ring9Args {
  const void *c[8];
  const void *v;          // ring: the input
  void *u;                // rounds: the output being completed
  void *ring;             // L[NT][HS] R[NT][HS] B[NT][WS] T[NT][WS]
  int nx, ny, pitch, TX, TY, HS, WS;
};
// the fused 2D BiCGStab phases H1 (inputs r, p, v) and H2 (inputs r, v')
#ifndef STEN_BICG9_BY
#define STEN_BICG9_BY 32
#endif
constexpr int kBicg9BY = STEN_BICG9_BY;  // rows per k_bicg9 tile
struct alignas(64) Bicg9Args {
  CUtensorMap tm_in[3];   // box (BX + 2H) x (BY + 2)
  const void *c[8];
  const void *rh;         // H1: rhat
  void *out0, *out1;      // H1: v', p'   H2: t, s
  int nx, ny, pitch, tiles_x, tiles_y;
  Reduce red;
};
// the tiled solve's unfused pieces: H1 p' = r + beta (p - omega v), H2 s = r - alpha v (k_upd9)
// and the phase's inner products (k_dot9: H1 (a0, b0); H2 (a0, b0), (a0, a0))
struct Upd9Args {
  const void *r, *p, *v;
  void *out;
  long long nvec;
  DevState *st;
};
struct Dot9Args {
  const void *a0, *b0;
  long long nvec;
  Reduce red;
};
template <typename T> int upd9_launch(int mode, const Upd9Args &a, int grid, cudaStream_t s);
template <typename T> int dot9_launch(int mode, const Dot9Args &a, int grid, cudaStream_t s);
struct Coef9In { const void *off[8]; };
struct Coef9Out { float *c32[8]; __half *c16[8]; };
template <typename T> int apply9_launch(const Apply9Args &a, cudaStream_t s);
template <typename T> int ring9_launch(const Ring9Args &a, cudaStream_t s);
template <typename T> int round9_launch(const Ring9Args &a, int dir, cudaStream_t s);
template <typename T> int bicg9_launch(int mode, const Bicg9Args &a, cudaStream_t s);
int create9_launch(int in_dtype, const void *diag, const Coef9In &in, int nx, int ny, int pitch, const Coef9Out &out,
                   double *aP, cudaStream_t s);

int create_coeffs_launch(int in_dtype, const void *diag, const void *const off[6], Geom g,
                         int has_below, int has_above, float *const c32[6], __half *const c16[6],
                         double *aP, const double *cconst, cudaStream_t s);
int device_sm_count();

}  // namespace sten
