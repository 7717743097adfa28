// kernels.cu - sm_100a kernels of the BiCGStab hot path.
//
//  (the fused stencil kernels k_stencil<T, MODE, BY, S> are in stencil.cu)
//  k_h3<T>, k_h3_bulk<T>: x += alpha p + omega s (l.181), r = s - omega t (l.182),
//           (rhat, r), (r, r) (l.183 and the stopping rule R4); the product runs
//           k_h3_bulk (the five input streams through a cp.async.bulk ring)
//  k_init<T>: b_hat = b / a_P (R3), r0 = b_hat - A x0 (R1), rhat = p = r0, v = 0
//  k_create_coeffs: Jacobi scaling c_d = A_d / a_P in fp64, rounded to fp32 and
//    fp16 (R3, R5).
#include "sten_internal.cuh"

#include <algorithm>

namespace sten {

// ------------------------------------------------------------------ H3 --
#ifndef STEN_H3_QUAD
#define STEN_H3_QUAD 1  // four vectors per trip: H3 1.284 -> 1.256 ms at config 3 (tools/h3_exp.sh)
#endif
// Element offset of the v-th vector of the interior range.  The element-wise
// kernels stream the whole 128-B-aligned range linearly, row padding included:
// the padding holds zeros in every vector (never written with anything else),
// and a linear aligned stream runs ~1.4x faster on B200 HBM than skipping the
// 80-B gap of every 1200-B row (tools/membench2.cu).
template <int VEC>
__device__ __forceinline__ long long vofs(long long v, const EwArgs &) {
  return v * VEC;
}

template <typename T>
__global__ void __launch_bounds__(256) k_h3(const __grid_constant__ EwArgs a) {
  using P = Pack<T>;
  constexpr int VEC = P::VEC;
  __shared__ float scratch[32 * kMaxDots];
  if (st_idle(a.red.st)) return;
  const typename P::S as = P::scalar(a.red.st->alpha);
  const typename P::S ws = P::scalar(a.red.st->omega);
  const typename P::S mws = P::neg(ws);
  const T *__restrict__ X = reinterpret_cast<const T *>(a.x);
  const T *__restrict__ Pp = reinterpret_cast<const T *>(a.p);
  const T *__restrict__ Sv = reinterpret_cast<const T *>(a.s);
  const T *__restrict__ Tv = reinterpret_cast<const T *>(a.t);
  const T *__restrict__ Rh = reinterpret_cast<const T *>(a.rhat);
  T *__restrict__ XO = reinterpret_cast<T *>(a.xo);
  T *__restrict__ RO = reinterpret_cast<T *>(a.ro);
  float d0[4] = {0.f, 0.f, 0.f, 0.f}, d1[4] = {0.f, 0.f, 0.f, 0.f};
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
#if STEN_H3_QUAD
  // four vectors per thread per trip: twenty loads in flight, then the pairs and the tail
  for (; v + 3 * stride < a.nvec; v += 4 * stride) {
    P xs[4], ps[4], ss[4], ts[4], rs[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long o = vofs<VEC>(v + u * stride, a);
      xs[u] = P::ldg(X + o); ps[u] = P::ldg(Pp + o); ss[u] = P::ldg(Sv + o); ts[u] = P::ldg(Tv + o); rs[u] = P::ldg(Rh + o);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long o = vofs<VEC>(v + u * stride, a);
      P xn = P::fmas(ws, ss[u], P::fmas(as, ps[u], xs[u])), rn = P::fmas(mws, ts[u], ss[u]);
#if STEN_H3_VARIANT == 1
      __stcs(reinterpret_cast<uint4 *>(XO + o), *reinterpret_cast<const uint4 *>(&xn));
      __stcs(reinterpret_cast<uint4 *>(RO + o), *reinterpret_cast<const uint4 *>(&rn));
#else
      xn.st(XO + o);
      rn.st(RO + o);
#endif
      rs[u].dot4(rn, d0);
      rn.dot4(rn, d1);
    }
  }
#endif
  // two vectors per thread per trip: all ten loads issued before any math
  for (; v + stride < a.nvec; v += 2 * stride) {
    const long long o0 = vofs<VEC>(v, a), o1 = vofs<VEC>(v + stride, a);
    P x0 = P::ldg(X + o0), p0 = P::ldg(Pp + o0), s0 = P::ldg(Sv + o0), t0 = P::ldg(Tv + o0), r0 = P::ldg(Rh + o0);
    P x1 = P::ldg(X + o1), p1 = P::ldg(Pp + o1), s1 = P::ldg(Sv + o1), t1 = P::ldg(Tv + o1), r1 = P::ldg(Rh + o1);
    P xn0 = P::fmas(ws, s0, P::fmas(as, p0, x0)), rn0 = P::fmas(mws, t0, s0);
    P xn1 = P::fmas(ws, s1, P::fmas(as, p1, x1)), rn1 = P::fmas(mws, t1, s1);
    xn0.st(XO + o0);
    rn0.st(RO + o0);
    xn1.st(XO + o1);
    rn1.st(RO + o1);
    r0.dot4(rn0, d0);
    rn0.dot4(rn0, d1);
    r1.dot4(rn1, d0);
    rn1.dot4(rn1, d1);
  }
  if (v < a.nvec) {
    const long long o0 = vofs<VEC>(v, a);
    P x0 = P::ldg(X + o0), p0 = P::ldg(Pp + o0), s0 = P::ldg(Sv + o0), t0 = P::ldg(Tv + o0), r0 = P::ldg(Rh + o0);
    P xn0 = P::fmas(ws, s0, P::fmas(as, p0, x0)), rn0 = P::fmas(mws, t0, s0);
    xn0.st(XO + o0);
    rn0.st(RO + o0);
    r0.dot4(rn0, d0);
    rn0.dot4(rn0, d1);
  }
  float d[2] = {sum4(d0), sum4(d1)};
  grid_reduce_finalize<2, PH_H3>(d, a.red, scratch);
}

// H3 implementation (tools/h3var.sh, config 3, paired runs at 1965 MHz): k_h3 1.24 ms; k_h3_bulk
// 1.17-1.19 ms for 2-3 stages of 256-512 vectors at 2-4 CTAs/SM, best 3 x 384 at 2 CTAs/SM.
#ifndef STEN_H3_VARIANT
#define STEN_H3_VARIANT 2  // 0: k_h3 (register streams); 1: k_h3 with .cs stores; 2: k_h3_bulk
#endif
#ifndef STEN_H3_SEGV
#define STEN_H3_SEGV 384   // k_h3_bulk: 16-B vectors per segment
#endif
#ifndef STEN_H3_NS
#define STEN_H3_NS 3       // k_h3_bulk: ring stages (3 x 5 x 6 KB = 90 KB)
#endif
#ifndef STEN_H3_CPS
#define STEN_H3_CPS 2      // k_h3_bulk: CTAs per SM
#endif
#ifndef STEN_H3_LDHINT
#define STEN_H3_LDHINT 0  // k_h3_bulk: the five input streams' bulk copies with an L2 evict-first hint
#endif
#ifndef STEN_H3_CSST
#define STEN_H3_CSST 1  // k_h3_bulk: streaming (.cs) stores of x, r
#endif

// H3 through 1D bulk copies: a persistent CTA streams segments of SEGV 16-B vectors of the five
// inputs (x, p, s, t, rhat) through an NS-stage shared ring (cp.async.bulk issued by one thread,
// mbarrier complete_tx), computes from shared memory and stores x, r with streaming stores.
template <typename T, int SEGV, int NS>
__global__ void __launch_bounds__(256) k_h3_bulk(const __grid_constant__ EwArgs a) {
  using P = Pack<T>;
  constexpr int VEC = P::VEC;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ float scratch[32 * kMaxDots];
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
  T *ring = reinterpret_cast<T *>(smem + 128);  // [NS][5][SEGV * VEC]
  if (st_idle(a.red.st)) return;
  const long long nseg = (a.nvec + SEGV - 1) / SEGV;
  const long long nmine = blockIdx.x < nseg ? (nseg - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const int tid = threadIdx.x;
  const T *src[5] = {reinterpret_cast<const T *>(a.x), reinterpret_cast<const T *>(a.p),
                     reinterpret_cast<const T *>(a.s), reinterpret_cast<const T *>(a.t),
                     reinterpret_cast<const T *>(a.rhat)};
  if (tid == 0) {
#pragma unroll
    for (int k = 0; k < NS; ++k) mbar_init(&bar[k], 1);
    fence_mbar_init();
  }
  __syncthreads();
  uint64_t pol = 0;
  if (STEN_H3_LDHINT) asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  auto issue = [&](long long i) {
    const int slot = (int)(i % NS);
    const long long v0 = (blockIdx.x + i * gridDim.x) * (long long)SEGV;
    const long long nv = min((long long)SEGV, a.nvec - v0);
    const uint32_t bytes = (uint32_t)(nv * 16);
    mbar_expect_tx(&bar[slot], 5u * bytes);
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      if (STEN_H3_LDHINT) bulk_g2s_hint(ring + ((size_t)slot * 5 + k) * SEGV * VEC, src[k] + v0 * VEC, bytes, &bar[slot], pol);
      else bulk_g2s(ring + ((size_t)slot * 5 + k) * SEGV * VEC, src[k] + v0 * VEC, bytes, &bar[slot]);
    }
  };
  if (tid == 0)
    for (long long i = 0; i < NS && i < nmine; ++i) issue(i);
  const typename P::S as = P::scalar(a.red.st->alpha);
  const typename P::S ws = P::scalar(a.red.st->omega);
  const typename P::S mws = P::neg(ws);
  T *__restrict__ XO = reinterpret_cast<T *>(a.xo);
  T *__restrict__ RO = reinterpret_cast<T *>(a.ro);
  T *const PLR = reinterpret_cast<T *>(a.peer_lo_r), *const PHR = reinterpret_cast<T *>(a.peer_hi_r);
  const long long top0 = (long long)(a.nzp - 1) * a.plane_elems;  // first element of the last plane
  bool peer = false;
  float d0[4] = {0.f, 0.f, 0.f, 0.f}, d1[4] = {0.f, 0.f, 0.f, 0.f};
  for (long long i = 0; i < nmine; ++i) {
    const int slot = (int)(i % NS);
    mbar_wait(&bar[slot], (uint32_t)((i / NS) & 1));
    const long long v0 = (blockIdx.x + i * gridDim.x) * (long long)SEGV;
    const int nv = (int)min((long long)SEGV, a.nvec - v0);
    const T *rb = ring + (size_t)slot * 5 * SEGV * VEC;
    for (int v = tid; v < nv; v += 256) {
      const int e = v * VEC;
      const P xs = P::ld(rb + e), ps = P::ld(rb + SEGV * VEC + e), ss = P::ld(rb + 2 * SEGV * VEC + e);
      const P ts = P::ld(rb + 3 * SEGV * VEC + e), rs = P::ld(rb + 4 * SEGV * VEC + e);
      const P xn = P::fmas(ws, ss, P::fmas(as, ps, xs)), rn = P::fmas(mws, ts, ss);
      const long long o = (v0 + v) * VEC;
      if (STEN_H3_CSST) {
        __stcs(reinterpret_cast<uint4 *>(XO + o), *reinterpret_cast<const uint4 *>(&xn));
        __stcs(reinterpret_cast<uint4 *>(RO + o), *reinterpret_cast<const uint4 *>(&rn));
      } else {
        xn.st(XO + o);
        rn.st(RO + o);
      }
      if (PLR && o < a.plane_elems) {  // fused exchange: r's boundary planes (H1's halos)
        rn.st(PLR + o);
        peer = true;
      }
      if (PHR && o >= top0) {
        rn.st(PHR + (o - top0));
        peer = true;
      }
      rs.dot4(rn, d0);
      rn.dot4(rn, d1);
    }
    __syncthreads();  // the slot is consumed
    if (tid == 0 && i + NS < nmine) issue(i + NS);
  }
  float d[2] = {sum4(d0), sum4(d1)};
  grid_reduce_finalize<2, PH_H3>(d, a.red, scratch, __syncthreads_or(peer) != 0);
}

template <typename T>
int h3_launch(const EwArgs &a, int grid, int threads, cudaStream_t s) {
#if STEN_H3_VARIANT == 2
  (void)grid;
  (void)threads;
  constexpr size_t smem = 128 + (size_t)STEN_H3_NS * 5 * STEN_H3_SEGV * 16;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_h3_bulk<T, STEN_H3_SEGV, STEN_H3_NS>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
    configured = true;
  }
  // persistent CTAs, but no more than there are segments (a small mesh would otherwise launch idle CTAs
  // that still take part in the last-CTA reduction)
  const long long nseg = (a.nvec + STEN_H3_SEGV - 1) / STEN_H3_SEGV;
  const int g = (int)std::max(1LL, std::min((long long)device_sm_count() * STEN_H3_CPS, nseg));
  k_h3_bulk<T, STEN_H3_SEGV, STEN_H3_NS><<<g, 256, smem, s>>>(a);
#else
  k_h3<T><<<grid, threads, 0, s>>>(a);
#endif
  return (int)cudaGetLastError();
}

// ---------------------------------------------------------------- INIT --
template <typename T> __device__ __forceinline__ T round_from_double(double x);
template <> __device__ __forceinline__ float round_from_double<float>(double x) { return __double2float_rn(x); }
template <> __device__ __forceinline__ __half round_from_double<__half>(double x) { return __double2half(x); }
template <typename T> __device__ __forceinline__ double widen(T x);
template <> __device__ __forceinline__ double widen<float>(float x) { return (double)x; }
template <> __device__ __forceinline__ double widen<__half>(__half x) { return (double)__half2float(x); }

template <typename T>
__global__ void __launch_bounds__(256) k_init(const __grid_constant__ EwArgs a) {
  using P = Pack<T>;
  constexpr int VEC = P::VEC;
  __shared__ float scratch[32 * kMaxDots];
  const T *__restrict__ B = reinterpret_cast<const T *>(a.bw);
  const T *__restrict__ AX = reinterpret_cast<const T *>(a.ax);
  T *R = reinterpret_cast<T *>(a.r);
  T *RH = reinterpret_cast<T *>(a.rh);
  T *P0 = reinterpret_cast<T *>(a.p0);
  T *V0 = reinterpret_cast<T *>(a.v0);
  float d[3] = {0.0f, 0.0f, 0.0f};
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < a.nvec; v += stride) {
    const long long o = vofs<VEC>(v, a);
    P bh = P::ld(B + o);
    if (a.aP) {  // b_hat = rn(b / a_P) in fp64 (R3)
      T e[VEC];
      *reinterpret_cast<P *>(e) = bh;
#pragma unroll
      for (int i = 0; i < VEC; ++i) e[i] = round_from_double<T>(widen<T>(e[i]) / a.aP[o + i]);
      bh = *reinterpret_cast<P *>(e);
    }
    P r = AX ? P::sub(bh, P::ld(AX + o)) : bh;
    r.st(R + o);
    r.st(RH + o);
    r.st(P0 + o);
    P::zero().st(V0 + o);
    d[0] = r.dot(r, d[0]);    // rho = (rhat, r0), rhat = r0
    d[1] = bh.dot(bh, d[1]);  // (b_hat, b_hat)
    d[2] = r.dot(r, d[2]);    // (r0, r0)
  }
  grid_reduce_finalize<3, PH_INIT>(d, a.red, scratch);
}

template <typename T>
int init_launch(const EwArgs &a, int grid, int threads, cudaStream_t s) {
  k_init<T><<<grid, threads, 0, s>>>(a);
  return (int)cudaGetLastError();
}

// ------------------------------------------- iterative refinement (R21) --
// The four streams run on 4-element vectors (the interior range is whole
// planes, a multiple of 64 elements, at a 256-B-aligned start); the element
// arithmetic is the scalar one, lane by lane.
// b_hat = rn32(b / a_P) in fp64 (R3); the refinement's fp32 right-hand side
__global__ void k_ir_bhat(const IrArgs a) {
  const long long nv = a.n >> 2;
  const float4 *B = reinterpret_cast<const float4 *>(a.b);
  const double2 *D = reinterpret_cast<const double2 *>(a.aP);
  float4 *R = reinterpret_cast<float4 *>(a.r);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += (long long)gridDim.x * blockDim.x) {
    float4 v = __ldcs(B + i);
    if (a.aP) {
      const double2 d0 = __ldcs(D + 2 * i), d1 = __ldcs(D + 2 * i + 1);
      v = make_float4(__double2float_rn((double)v.x / d0.x), __double2float_rn((double)v.y / d0.y),
                      __double2float_rn((double)v.z / d1.x), __double2float_rn((double)v.w / d1.y));
    }
    R[i] = v;
  }
}
// r = b_hat - A x in fp32 (ax null: x = 0, r = b_hat exactly); (r, r) by the
// deterministic grid reduction; max|r|
__global__ void __launch_bounds__(256) k_ir_resid(const IrArgs a) {
  __shared__ float scratch[32 * kMaxDots];
  float d[1] = {0.0f};
  float m = 0.0f;
  const long long nv = a.n >> 2;
  const float4 *B = reinterpret_cast<const float4 *>(a.b);
  const float4 *AX = reinterpret_cast<const float4 *>(a.ax);
  float4 *R = reinterpret_cast<float4 *>(a.r);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += (long long)gridDim.x * blockDim.x) {
    float4 r = __ldcs(B + i);
    if (AX) {
      const float4 ax = __ldcs(AX + i);
      r = make_float4(__fsub_rn(r.x, ax.x), __fsub_rn(r.y, ax.y), __fsub_rn(r.z, ax.z), __fsub_rn(r.w, ax.w));
    }
    R[i] = r;
    d[0] = __fmaf_rn(r.x, r.x, d[0]);
    d[0] = __fmaf_rn(r.y, r.y, d[0]);
    d[0] = __fmaf_rn(r.z, r.z, d[0]);
    d[0] = __fmaf_rn(r.w, r.w, d[0]);
    m = fmaxf(m, fmaxf(fmaxf(fabsf(r.x), fabsf(r.y)), fmaxf(fabsf(r.z), fabsf(r.w))));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.0f) atomicMax(a.amax, __float_as_uint(m));  // |r| >= 0: bits order as floats
  grid_reduce_finalize<1, PH_INIT>(d, a.red, scratch);
}
// r16 = rn16(r / sigma), sigma = 2^e the power of two with max|r| <= sigma
// (an exact scaling: the inner right-hand side uses the whole fp16 range)
__global__ void k_ir_scale(const IrArgs a) {
  const float m = __uint_as_float(*a.amax);
  int e = 0;
  frexpf(m, &e);  // m = f 2^e, f in [0.5, 1)
  const float inv = ldexpf(1.0f, -e);
  if (blockIdx.x == 0 && threadIdx.x == 0) *a.sigma = ldexpf(1.0f, e);
  const long long nv = a.n >> 2;
  const float4 *R = reinterpret_cast<const float4 *>(a.r);
  uint2 *R16 = reinterpret_cast<uint2 *>(a.r16);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += (long long)gridDim.x * blockDim.x) {
    const float4 r = __ldcs(R + i);
    const __half2 lo = __halves2half2(__float2half_rn(r.x * inv), __float2half_rn(r.y * inv));
    const __half2 hi = __halves2half2(__float2half_rn(r.z * inv), __float2half_rn(r.w * inv));
    R16[i] = make_uint2(*reinterpret_cast<const uint32_t *>(&lo), *reinterpret_cast<const uint32_t *>(&hi));
  }
}
// x = fma(sigma, d, x) in fp32
__global__ void k_ir_update(const IrArgs a) {
  const float sg = *a.sigma;
  const long long nv = a.n >> 2;
  const uint2 *D = reinterpret_cast<const uint2 *>(a.d16);
  float4 *X = reinterpret_cast<float4 *>(a.x);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += (long long)gridDim.x * blockDim.x) {
    const uint2 u = __ldcs(D + i);
    const float2 lo = __half22float2(*reinterpret_cast<const __half2 *>(&u.x));
    const float2 hi = __half22float2(*reinterpret_cast<const __half2 *>(&u.y));
    float4 x = X[i];
    x = make_float4(__fmaf_rn(sg, lo.x, x.x), __fmaf_rn(sg, lo.y, x.y), __fmaf_rn(sg, hi.x, x.z), __fmaf_rn(sg, hi.y, x.w));
    X[i] = x;
  }
}

// ------------------------------------------------ pitched device copies --
// d planes of h rows of W-byte words, dst <- src (the layouts' host-side
// copies: user vectors <-> halo'd pitched planes; cudaMemcpy3D moved them at
// ~2 TB/s).  blockIdx.y walks the planes; inside a plane either one linear
// stream (rows contiguous on both sides: the plane is one row of h*words) or
// one warp per row with the lanes over its words.
template <typename W>
__global__ void __launch_bounds__(256) k_copy_rows(char *__restrict__ dst, long long dplane, long long dpitch,
                                                   const char *__restrict__ src, long long splane, long long spitch,
                                                   int words, int h, long long d, int linear) {
  for (long long z = blockIdx.y; z < d; z += gridDim.y) {
    const char *sp0 = src + z * splane;
    char *dp0 = dst + z * dplane;
    if (linear) {
      const W *sp = reinterpret_cast<const W *>(sp0);
      W *dp = reinterpret_cast<W *>(dp0);
      const long long n = (long long)words * h;
      for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        dp[i] = __ldcs(sp + i);
    } else {
      const int lane = threadIdx.x & 31;
      for (int y = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); y < h; y += gridDim.x * (blockDim.x >> 5)) {
        const W *sp = reinterpret_cast<const W *>(sp0 + y * spitch);
        W *dp = reinterpret_cast<W *>(dp0 + y * dpitch);
        for (int i = lane; i < words; i += 32) dp[i] = __ldcs(sp + i);
      }
    }
  }
}

int copy_rows_launch(void *dst, size_t dpitch, size_t dysize, const void *src, size_t spitch, size_t sysize,
                     size_t wbytes, size_t h, size_t d, int sms, cudaStream_t s) {
  if (h == 0 || d == 0 || wbytes == 0) return (int)cudaSuccess;
  if (h > 0x7fffffff) return (int)cudaErrorNotSupported;
  const uintptr_t al = (uintptr_t)dst | (uintptr_t)src | dpitch | spitch | wbytes;
  const int ws = al % 16 == 0 ? 16 : al % 4 == 0 ? 4 : al % 2 == 0 ? 2 : 0;
  if (ws == 0 || wbytes / ws > 0x7fffffff) return (int)cudaErrorNotSupported;
  const int words = (int)(wbytes / ws);
  const int linear = (dpitch == wbytes && spitch == wbytes) ? 1 : 0;
  // about 8 resident 256-thread CTAs per SM in total, at least one per plane
  const long long gy = d < 65535 ? (long long)d : 65535;
  const long long per_plane = linear ? ((long long)words * (long long)h + 255) / 256 : ((long long)h + 7) / 8;
  long long gx = ((long long)sms * 8 + gy - 1) / gy;
  if (gx > per_plane) gx = per_plane;
  if (gx < 1) gx = 1;
  const dim3 grid((unsigned)gx, (unsigned)gy);
  char *D = static_cast<char *>(dst);
  const char *S = static_cast<const char *>(src);
  const long long dpl = (long long)(dpitch * dysize), spl = (long long)(spitch * sysize);
  if (ws == 16)
    k_copy_rows<uint4><<<grid, 256, 0, s>>>(D, dpl, (long long)dpitch, S, spl, (long long)spitch, words, (int)h, (long long)d, linear);
  else if (ws == 4)
    k_copy_rows<uint32_t><<<grid, 256, 0, s>>>(D, dpl, (long long)dpitch, S, spl, (long long)spitch, words, (int)h, (long long)d, linear);
  else
    k_copy_rows<unsigned short><<<grid, 256, 0, s>>>(D, dpl, (long long)dpitch, S, spl, (long long)spitch, words, (int)h, (long long)d, linear);
  return (int)cudaGetLastError();
}

int ir_launch(int which, const IrArgs &a, int grid, cudaStream_t s) {
  switch (which) {
    case IR_BHAT: k_ir_bhat<<<grid, 256, 0, s>>>(a); break;
    case IR_RESID: k_ir_resid<<<grid, 256, 0, s>>>(a); break;
    case IR_SCALE: k_ir_scale<<<grid, 256, 0, s>>>(a); break;
    default: k_ir_update<<<grid, 256, 0, s>>>(a); break;
  }
  return (int)cudaGetLastError();
}

// ------------------------------------------------- cross-slab scalar step --
__global__ void k_scalars(int phase, const float *__restrict__ slab_sums, int nslabs, DevState *st) {
  if (phase != PH_INIT && phase != PH_SR && st_idle(st)) return;
  if (phase == PH_SR && sr_idle(st)) return;
  float s[kMaxDots];
  for (int d = 0; d < kMaxDots; ++d) s[d] = 0.0f;
  for (int k = 0; k < nslabs; ++k)  // fixed slab order: deterministic
    for (int d = 0; d < kMaxDots; ++d) s[d] += slab_sums[k * kMaxDots + d];
  switch (phase) {
    case PH_INIT: finalize_phase<PH_INIT>(st, s); break;
    case PH_H1: finalize_phase<PH_H1>(st, s); break;
    case PH_H2: finalize_phase<PH_H2>(st, s); break;
    case PH_H3: finalize_phase<PH_H3>(st, s); break;
    default: finalize_phase<PH_SR>(st, s); break;
  }
}

__global__ void k_slabsum(const float *__restrict__ slab_sums, int nslabs, float *out) {
  float s[kMaxDots];
  for (int d = 0; d < kMaxDots; ++d) s[d] = 0.0f;
  for (int k = 0; k < nslabs; ++k)
    for (int d = 0; d < kMaxDots; ++d) s[d] += slab_sums[k * kMaxDots + d];
  for (int d = 0; d < kMaxDots; ++d) out[d] = s[d];
}

// Scalar step after a peer-memory all-reduce: wait (bounded) until every slot
// of this participant's inbox (the half of the sequence number's parity) holds
// the current reduction's sums, add them in slot order (deterministic,
// identical on every rank), finalise.  A peer that never arrives stops the
// solve with STEN_TIMEOUT after ~20 s instead of hanging the device.
template <int PH>
__global__ void k_p2p_fin(P2PBox inbox, int nslots, unsigned *seqp, DevState *st) {
  if (PH == PH_SR && sr_idle(st)) return;
  if ((PH == PH_H1 || PH == PH_H2 || PH == PH_H3) && st_idle(st)) return;  // every rank idles alike
  const unsigned seq = *seqp + 1u;
  const int base = (int)(seq & 1u) * nslots;
  const long long t0 = clock64();
  bool timeout = false;
  for (int k = 0; k < nslots && !timeout; ++k) {
    unsigned f;
    do {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(f) : "l"(inbox.flags + base + k) : "memory");
      if (f == seq) break;
      __nanosleep(200);
      if (clock64() - t0 > 40000000000ll) timeout = true;  // ~20 s: a peer never arrived
    } while (!timeout);
  }
  float s[kMaxDots];
  for (int d = 0; d < kMaxDots; ++d) s[d] = 0.0f;
  for (int k = 0; k < nslots; ++k)
    for (int d = 0; d < kMaxDots; ++d) s[d] += __ldcv(&inbox.sums[(base + k) * kMaxDots + d]);
  if (timeout) {  // never hang the device: report and stop the solve
    st_event(st, STEN_TIMEOUT, PH == PH_SR ? st->sweep : 0, false);
    st->stop = 1;
    st->status = STEN_TIMEOUT;
    return;
  }
  *seqp = seq;
  finalize_phase<PH>(st, s);
}

int p2p_fin_launch(int phase, P2PBox inbox, int nslots, unsigned *seq, DevState *st, cudaStream_t s) {
  switch (phase) {
    case PH_INIT: k_p2p_fin<PH_INIT><<<1, 1, 0, s>>>(inbox, nslots, seq, st); break;
    case PH_H1: k_p2p_fin<PH_H1><<<1, 1, 0, s>>>(inbox, nslots, seq, st); break;
    case PH_H2: k_p2p_fin<PH_H2><<<1, 1, 0, s>>>(inbox, nslots, seq, st); break;
    case PH_H3: k_p2p_fin<PH_H3><<<1, 1, 0, s>>>(inbox, nslots, seq, st); break;
    default: k_p2p_fin<PH_SR><<<1, 1, 0, s>>>(inbox, nslots, seq, st); break;
  }
  return (int)cudaGetLastError();
}

struct P2PBoxes {
  P2PBox b[kMaxPeers];
};
__global__ void k_p2p_put(const float *__restrict__ slab_sums, int nslabs, int base, int nslots, P2PBoxes boxes,
                          int nboxes, const unsigned *seqp) {
  const unsigned seq = *seqp + 1u;
  const int half = (int)(seq & 1u) * nslots;
  for (int r = 0; r < nboxes; ++r)
    for (int k = 0; k < nslabs; ++k)
      for (int d = 0; d < kMaxDots; ++d) boxes.b[r].sums[(half + base + k) * kMaxDots + d] = slab_sums[k * kMaxDots + d];
  __threadfence_system();
  for (int r = 0; r < nboxes; ++r)
    for (int k = 0; k < nslabs; ++k)
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(boxes.b[r].flags + half + base + k), "r"(seq) : "memory");
}

int p2p_put_launch(const float *slab_sums, int nslabs, int base, int nslots, const P2PBox *boxes, int nboxes,
                   const unsigned *seq, cudaStream_t s) {
  if (nboxes > kMaxPeers) return (int)cudaErrorInvalidValue;
  P2PBoxes bx;
  for (int r = 0; r < nboxes; ++r) bx.b[r] = boxes[r];
  k_p2p_put<<<1, 1, 0, s>>>(slab_sums, nslabs, base, nslots, bx, nboxes, seq);
  return (int)cudaGetLastError();
}

int scalars_launch(int phase, const float *slab_sums, int nslabs, DevState *st, cudaStream_t s) {
  k_scalars<<<1, 1, 0, s>>>(phase, slab_sums, nslabs, st);
  return (int)cudaGetLastError();
}
int slabsum_launch(const float *slab_sums, int nslabs, float *out, cudaStream_t s) {
  k_slabsum<<<1, 1, 0, s>>>(slab_sums, nslabs, out);
  return (int)cudaGetLastError();
}

// -------------------------------------------------- Jacobi scaling (S0) --
template <typename TIN>
__global__ void k_create_coeffs(const TIN *__restrict__ diag, const TIN *o0, const TIN *o1, const TIN *o2,
                                const TIN *o3, const TIN *o4, const TIN *o5, Geom g, int has_below,
                                int has_above, float *c32_0, float *c32_1, float *c32_2, float *c32_3,
                                float *c32_4, float *c32_5, __half *c16_0, __half *c16_1, __half *c16_2,
                                __half *c16_3, __half *c16_4, __half *c16_5, double *aP, const double *cconst) {
  const TIN *off[6] = {o0, o1, o2, o3, o4, o5};
  float *c32[6] = {c32_0, c32_1, c32_2, c32_3, c32_4, c32_5};
  __half *c16[6] = {c16_0, c16_1, c16_2, c16_3, c16_4, c16_5};
  const long long total = g.plane * g.nz;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const long long inplane = q % g.plane;
    const int x = (int)(inplane % g.pitch);
    const int y = (int)(inplane / g.pitch), z = (int)(q / g.plane);
    if (x >= g.nx || y >= g.ny) {  // row / plane padding: zero couplings, unit diagonal
      for (int d = 0; d < 6; ++d) {
        c32[d][q] = 0.0f;
        c16[d][q] = __float2half(0.0f);
      }
      if (aP) aP[q] = 1.0;
      continue;
    }
    const long long P = x + (long long)g.nx * (y + (long long)g.ny * z);
    const bool inside[6] = {x > 0, x + 1 < g.nx, y > 0, y + 1 < g.ny, z > 0 || has_below != 0,
                            z + 1 < g.nz || has_above != 0};
    // cconst: a constant operator (diag, xm..zp), the same scaling per point
    const bool hasd = cconst ? cconst[0] != 0.0 : diag != nullptr;
    const double dP = cconst ? (hasd ? cconst[0] : 1.0) : (diag ? (double)diag[P] : 1.0);
    for (int d = 0; d < 6; ++d) {
      double c = 0.0;  // R5: couplings leaving the mesh are dropped
      const double od = cconst ? cconst[1 + d] : (double)off[d][P];
      if (inside[d]) c = hasd ? __ddiv_rn(od, dP) : od;
      c32[d][q] = __double2float_rn(c);
      c16[d][q] = __double2half(c);
    }
    if (aP) aP[q] = dP;
  }
}

int create_coeffs_launch(int in_dtype, const void *diag, const void *const off[6], Geom g, int has_below,
                         int has_above, float *const c32[6], __half *const c16[6], double *aP,
                         const double *cconst, cudaStream_t s) {
  const long long total = g.plane * g.nz;
  int grid = (int)((total + 255) / 256);
  if (grid > 148 * 32) grid = 148 * 32;
  if (grid < 1) grid = 1;
  if (in_dtype == STEN_DT_F64) {
    const double *const *o = reinterpret_cast<const double *const *>(off);
    k_create_coeffs<double><<<grid, 256, 0, s>>>((const double *)diag, o[0], o[1], o[2], o[3], o[4], o[5], g,
                                                 has_below, has_above, c32[0], c32[1], c32[2], c32[3], c32[4],
                                                 c32[5], c16[0], c16[1], c16[2], c16[3], c16[4], c16[5], aP,
                                                 cconst);
  } else {
    const float *const *o = reinterpret_cast<const float *const *>(off);
    k_create_coeffs<float><<<grid, 256, 0, s>>>((const float *)diag, o[0], o[1], o[2], o[3], o[4], o[5], g,
                                                has_below, has_above, c32[0], c32[1], c32[2], c32[3], c32[4],
                                                c32[5], c16[0], c16[1], c16[2], c16[3], c16[4], c16[5], aP,
                                                cconst);
  }
  return (int)cudaGetLastError();
}

int device_sm_count() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

template int h3_launch<float>(const EwArgs &, int, int, cudaStream_t);
template int h3_launch<__half>(const EwArgs &, int, int, cudaStream_t);
template int init_launch<float>(const EwArgs &, int, int, cudaStream_t);
template int init_launch<__half>(const EwArgs &, int, int, cudaStream_t);

}  // namespace sten
