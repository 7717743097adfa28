// sr.cu - the single-reduction BiCGStab sweep (R19, "SR schedule").
//
// One launch = one whole iteration of Alg. 1, rearranged
// so that it needs ONE pass over the mesh and ONE global reduction:
//
//   with the previous iteration's scalars (alpha, omega, beta), per point
//     s  = r - alpha v            (l.178)       t = q - alpha y   (= A s, l.179)
//     x += alpha p + omega s      (l.181)       r' = s - omega t  (l.182)
//     p' = r' + beta (p - omega v)                                 (l.184)
//   then three 7-point products in the same sweep
//     v' = A p'  (l.176)          q' = A r'          y' = A v'  (= A^2 p')
//   and twelve inner products of rh, r', v', q', y' (fp32 sums), from which the
//   last CTA forms alpha, omega (bilinear expansions of (t,s), (t,t)) and beta
//   (fin_sr in sten_internal.cuh).
//
// HBM traffic per point and iteration: read x r p v q y rh + 6 coefficients,
// write x r p v q y = 19 arrays (the classic three-kernel schedule moves 29).
//
// Structure of a CTA (an xy tile of BX x BY points marching z over a chunk):
//  * r, p, v, q, y of plane k+2 arrive by TMA as (BX+2H) x (BY+4) boxes - a
//    two-point xy halo, because y' = A(A p') needs p' two points away - into an
//    S-stage mbarrier ring; the six coefficient tiles of plane k+1 arrive as
//    (BX+2H) x (BY+2) boxes (one-point halo, for v' on the halo ring) into an
//    SC-stage ring.  Out-of-mesh elements are TMA zero fill; vectors carry two
//    zero/halo planes and coefficients one, so z needs no bound test.
//  * step k: (A) form p', r' of plane k+2 on the whole halo'd box and update
//    x, r, p of the own points; (B) v' of plane k+1 on the one-point halo ring;
//    (C) q', y' of plane k and the twelve dot products of plane k.  Formed
//    planes live in small shared rings (p' 3 planes, r' 4, v' 2); each thread
//    keeps its own z column of p', r', v' and its coefficients in registers.
//  * Two __syncthreads per plane.  Operation order of every element-wise op
//    and SpMV is the one oracle/osr.c mirrors (bitwise test).
//  * The z loop is unrolled by 6 (the period of every ring and window: input
//    stages 2|3, coefficient stages 2|3, p' ring 3, r' ring 6, v' ring 2), so
//    every shared-memory slot and register window is a compile-time name: no
//    modulo arithmetic and no register rotation per plane.
#include "sten_internal.cuh"

#include <type_traits>

namespace sten {

namespace {

constexpr int a128(int b) { return (b + 127) & ~127; }


template <int V> struct IC { static constexpr int value = V; };

#ifndef STEN_SR_DIAG
#define STEN_SR_DIAG 0
#endif
#ifndef STEN_SR_XTMA
#define STEN_SR_XTMA 1  // x arrives with the input stage by TMA (else a direct load three planes ahead)
#endif
#ifndef STEN_SR_RHTMA
#define STEN_SR_RHTMA 1  // r_hat too, into a 6-plane ring (it is used two steps after its stage lands)
#endif

// Per-thread vectors of the SR sweep: NB = 16 (8 fp16 / 4 fp32 lanes) or 8
// bytes (4 / 2 lanes).  The 8-B form gives a tile twice the threads (16 warps
// per SM for a 16-row tile) for the same shared-memory pipeline.
template <typename T, int NB> struct SPack;
template <int NB> struct SPack<__half, NB> {
  static constexpr int NW = NB / 4;  // 32-bit words (half2)
  static constexpr int VEC = 2 * NW;
  using S = __half2;
  uint32_t w[NW];
  static __device__ __forceinline__ __half2 h2(uint32_t u) { return *reinterpret_cast<const __half2 *>(&u); }
  static __device__ __forceinline__ uint32_t u32(__half2 h) { return *reinterpret_cast<const uint32_t *>(&h); }
  static __device__ __forceinline__ SPack ld(const __half *p) {
    SPack o;
    if (NB == 16) {
      const uint4 q = *reinterpret_cast<const uint4 *>(p);
      o.w[0] = q.x; o.w[1] = q.y; o.w[NW > 2 ? 2 : 0] = q.z; o.w[NW > 3 ? 3 : 1] = q.w;
    } else {
      const uint2 q = *reinterpret_cast<const uint2 *>(p);
      o.w[0] = q.x; o.w[1] = q.y;
    }
    return o;
  }
  static __device__ __forceinline__ SPack ldg(const __half *p) {
    SPack o;
    if (NB == 16) {
      const uint4 q = __ldcs(reinterpret_cast<const uint4 *>(p));
      o.w[0] = q.x; o.w[1] = q.y; o.w[NW > 2 ? 2 : 0] = q.z; o.w[NW > 3 ? 3 : 1] = q.w;
    } else {
      const uint2 q = __ldcs(reinterpret_cast<const uint2 *>(p));
      o.w[0] = q.x; o.w[1] = q.y;
    }
    return o;
  }
  __device__ __forceinline__ void st(__half *p) const {
    if (NB == 16) *reinterpret_cast<uint4 *>(p) = make_uint4(w[0], w[1], w[NW > 2 ? 2 : 0], w[NW > 3 ? 3 : 1]);
    else *reinterpret_cast<uint2 *>(p) = make_uint2(w[0], w[1]);
  }
  static __device__ __forceinline__ SPack zero() {
    SPack o;
#pragma unroll
    for (int i = 0; i < NW; ++i) o.w[i] = 0u;
    return o;
  }
  static __device__ __forceinline__ SPack fma(const SPack &a, const SPack &b, const SPack &c) {
    SPack o;
#pragma unroll
    for (int i = 0; i < NW; ++i) o.w[i] = u32(__hfma2(h2(a.w[i]), h2(b.w[i]), h2(c.w[i])));
    return o;
  }
  static __device__ __forceinline__ S scalar(float a) { return __float2half2_rn(a); }
  static __device__ __forceinline__ S neg(S a) { return __hneg2(a); }
  static __device__ __forceinline__ SPack fmas(S a, const SPack &b, const SPack &c) {
    SPack o;
#pragma unroll
    for (int i = 0; i < NW; ++i) o.w[i] = u32(__hfma2(a, h2(b.w[i]), h2(c.w[i])));
    return o;
  }
  // acc += a_i b_i in lane order: fma.rn.f32.f16 (exact fp16 product, fp32 add)
  __device__ __forceinline__ float mdot(const SPack &b, float acc) const {
#pragma unroll
    for (int i = 0; i < NW; ++i)
      asm("{\n .reg .b16 al, ah, bl, bh;\n mov.b32 {al, ah}, %1;\n mov.b32 {bl, bh}, %2;\n"
          " fma.rn.f32.f16 %0, al, bl, %0;\n fma.rn.f32.f16 %0, ah, bh, %0;\n}"
          : "+f"(acc)
          : "r"(w[i]), "r"(b.w[i]));
    return acc;
  }
};
template <int NB> struct SPack<float, NB> {
  static constexpr int VEC = NB / 4;
  using S = float;
  float v[VEC];
  static __device__ __forceinline__ SPack ld(const float *p) {
    SPack o;
    if (NB == 16) {
      const float4 q = *reinterpret_cast<const float4 *>(p);
      o.v[0] = q.x; o.v[1] = q.y; o.v[VEC > 2 ? 2 : 0] = q.z; o.v[VEC > 3 ? 3 : 1] = q.w;
    } else {
      const float2 q = *reinterpret_cast<const float2 *>(p);
      o.v[0] = q.x; o.v[1] = q.y;
    }
    return o;
  }
  static __device__ __forceinline__ SPack ldg(const float *p) {
    SPack o;
    if (NB == 16) {
      const float4 q = __ldcs(reinterpret_cast<const float4 *>(p));
      o.v[0] = q.x; o.v[1] = q.y; o.v[VEC > 2 ? 2 : 0] = q.z; o.v[VEC > 3 ? 3 : 1] = q.w;
    } else {
      const float2 q = __ldcs(reinterpret_cast<const float2 *>(p));
      o.v[0] = q.x; o.v[1] = q.y;
    }
    return o;
  }
  __device__ __forceinline__ void st(float *p) const {
    if (NB == 16) *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[VEC > 2 ? 2 : 0], v[VEC > 3 ? 3 : 1]);
    else *reinterpret_cast<float2 *>(p) = make_float2(v[0], v[1]);
  }
  static __device__ __forceinline__ SPack zero() {
    SPack o;
#pragma unroll
    for (int i = 0; i < VEC; ++i) o.v[i] = 0.0f;
    return o;
  }
  static __device__ __forceinline__ SPack fma(const SPack &a, const SPack &b, const SPack &c) {
    SPack o;  // FFMA2: two RN fp32 FMAs per instruction, lane for lane __fmaf_rn
#pragma unroll
    for (int i = 0; i < VEC; i += 2) ffma2(o.v[i], o.v[i + 1], a.v[i], a.v[i + 1], b.v[i], b.v[i + 1], c.v[i], c.v[i + 1]);
    return o;
  }
  static __device__ __forceinline__ S scalar(float a) { return a; }
  static __device__ __forceinline__ S neg(S a) { return -a; }
  static __device__ __forceinline__ SPack fmas(S a, const SPack &b, const SPack &c) {
    SPack o;
#pragma unroll
    for (int i = 0; i < VEC; i += 2) ffma2(o.v[i], o.v[i + 1], a, a, b.v[i], b.v[i + 1], c.v[i], c.v[i + 1]);
    return o;
  }
  __device__ __forceinline__ float mdot(const SPack &b, float acc) const {
#pragma unroll
    for (int i = 0; i < VEC; ++i) acc = __fmaf_rn(v[i], b.v[i], acc);
    return acc;
  }
};

__device__ __forceinline__ void tma_prefetch_l2(const CUtensorMap *map, int x, int y, int z) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(z)
               : "memory");
}

template <typename T, int BY, int NB>
struct SrGeo {
  static constexpr int VEC = SPack<T, NB>::VEC;
  static constexpr int BX = tile_bx<T>();
  static constexpr int H = 16 / (int)sizeof(T);  // x halo pad of the boxes: 16 B (TMA rows stay 16-B multiples)
  static constexpr int VOFF = H - VEC;           // element offset of halo vector column 0 (x0 - VEC)
  static constexpr int VPR = BX / VEC;           // own vectors per tile row
  static constexpr int VW = VPR + 2;             // vectors per box row (incl. the x halo)
  static constexpr int HW = BX + 2 * H;          // box row (elements)
  static constexpr int NT = VPR * BY;            // threads: one own vector each
  static constexpr int RI = BY + 4;              // rows of input / formed boxes: y0-2 .. y0+BY+1
  static constexpr int RC = BY + 2;              // rows of coefficient / v' boxes: y0-1 .. y0+BY
  static constexpr int IE = a128(HW * RI * (int)sizeof(T)) / (int)sizeof(T);  // elements per input box
  static constexpr int CE = a128(HW * RC * (int)sizeof(T)) / (int)sizeof(T);  // elements per coef box
  static constexpr int NHF = RI * VW - NT;       // formed vectors outside the own tile
  static constexpr int NHV = RC * VW - NT;       // v' vectors outside the own tile
  static constexpr int NR = 6;                   // r' ring slots (= unroll period)
  static constexpr int XE = a128(BX * BY * (int)sizeof(T)) / (int)sizeof(T);  // x tile per input stage
  static constexpr int SE = 5 * IE + (STEN_SR_XTMA ? XE : 0);                  // elements per input stage
  static_assert(NHF <= NT && NHV <= NT, "halo work must fit one extra item per thread");
};

template <typename T, int BY, int S, int SC, bool CC, int NB>
constexpr size_t sr_smem_c() {
  using G = SrGeo<T, BY, NB>;
  return 128 + (size_t)sizeof(T) * ((size_t)S * G::SE + (CC ? 0 : (size_t)SC * 6 * G::CE) +
                                    (STEN_SR_RHTMA ? 6 * (size_t)G::XE : 0) +
                                    (3 + G::NR) * (size_t)G::IE + 2 * (size_t)G::CE);
}

// constant coefficients as packs, and lane masks (keep lanes [lo, hi))
template <typename T, int NB> struct SrConst;
template <int NB> struct SrConst<float, NB> {
  using P = SPack<float, NB>;
  static __device__ __forceinline__ P splat(const SrArgs &a, int d) {
    P o;
#pragma unroll
    for (int i = 0; i < P::VEC; ++i) o.v[i] = a.cf32[d];
    return o;
  }
  static __device__ __forceinline__ P keep(const P &v, int lo, int hi) {
    P o;
#pragma unroll
    for (int i = 0; i < P::VEC; ++i) o.v[i] = (i >= lo && i < hi) ? v.v[i] : 0.0f;
    return o;
  }
};
template <int NB> struct SrConst<__half, NB> {
  using P = SPack<__half, NB>;
  static __device__ __forceinline__ P splat(const SrArgs &a, int d) {
    const uint32_t h = a.cf16[d];
    P o;
#pragma unroll
    for (int i = 0; i < P::NW; ++i) o.w[i] = h | (h << 16);
    return o;
  }
  static __device__ __forceinline__ P keep(const P &v, int lo, int hi) {
    P o;
#pragma unroll
    for (int i = 0; i < P::NW; ++i) {
      const uint32_t m = ((2 * i >= lo && 2 * i < hi) ? 0x0000FFFFu : 0u) | ((2 * i + 1 >= lo && 2 * i + 1 < hi) ? 0xFFFF0000u : 0u);
      o.w[i] = v.w[i] & m;
    }
    return o;
  }
};

// L2 eviction hints (bit 0: the sweep's stores evict-first -- the product
// default, +0.5%: the outputs are next read a whole sweep later, so they
// should not displace the input planes that neighbouring tiles still read as
// halos; experiments: bit 1 x / r_hat TMA loads evict-first (-4%), bit 2 the
// coefficient loads evict-first (-20%), bit 3 the halo'd inputs evict-last
// (+-0), bit 4 at fraction 0.5; keeping the four planes the next chunk of a tile
// stages again evict-last cost 2-4%)
#ifndef STEN_SR_EVF
#define STEN_SR_EVF 1
#endif
template <typename PK, typename T>
__device__ __forceinline__ void sr_st(const PK &v, T *p, uint64_t pol) {
  if (STEN_SR_EVF & 1) {
    if (sizeof(PK) == 16) {
      uint4 u;
      memcpy(&u, &v, 16);
      asm volatile("st.global.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(u.x), "r"(u.y),
                   "r"(u.z), "r"(u.w), "l"(pol)
                   : "memory");
    } else {
      uint2 u;
      memcpy(&u, &v, 8);
      asm volatile("st.global.L2::cache_hint.v2.b32 [%0], {%1, %2}, %3;" ::"l"(p), "r"(u.x), "r"(u.y), "l"(pol)
                   : "memory");
    }
  } else {
    v.st(p);
  }
}

// half-dot mode (HD, DESIGN R22): the lane pencils of a pack, each an fp16
// running sum over the thread's z range, widened and added in lane order
template <int NB> __device__ __forceinline__ float sr_lanesum(const SPack<__half, NB> &a) {
  float s = 0.0f;
#pragma unroll
  for (int i = 0; i < SPack<__half, NB>::NW; ++i) {
    const float2 f = __half22float2(SPack<__half, NB>::h2(a.w[i]));
    s += f.x;
    s += f.y;
  }
  return s;
}
template <int NB> __device__ __forceinline__ float sr_lanesum(const SPack<float, NB> &a) {
  float s = 0.0f;
#pragma unroll
  for (int i = 0; i < SPack<float, NB>::VEC; ++i) s += a.v[i];
  return s;
}

template <typename T, int NB> struct SrShift;
template <int NB> struct SrShift<float, NB> {
  using E = float;
  using P = SPack<float, NB>;
  static __device__ __forceinline__ P left(const P &c, float l) {
    P o;
    o.v[0] = l;
#pragma unroll
    for (int i = 1; i < P::VEC; ++i) o.v[i] = c.v[i - 1];
    return o;
  }
  static __device__ __forceinline__ P right(const P &c, float r) {
    P o;
#pragma unroll
    for (int i = 0; i + 1 < P::VEC; ++i) o.v[i] = c.v[i + 1];
    o.v[P::VEC - 1] = r;
    return o;
  }
  static __device__ __forceinline__ float ld1(const float *p) { return *p; }
};
template <int NB> struct SrShift<__half, NB> {
  using E = uint32_t;
  using P = SPack<__half, NB>;
  static __device__ __forceinline__ P left(const P &c, uint32_t l) {
    P o;
    o.w[0] = __byte_perm(l, c.w[0], 0x5410);
#pragma unroll
    for (int i = 1; i < P::NW; ++i) o.w[i] = __byte_perm(c.w[i - 1], c.w[i], 0x5432);
    return o;
  }
  static __device__ __forceinline__ P right(const P &c, uint32_t r) {
    P o;
#pragma unroll
    for (int i = 0; i + 1 < P::NW; ++i) o.w[i] = __byte_perm(c.w[i], c.w[i + 1], 0x5432);
    o.w[P::NW - 1] = __byte_perm(c.w[P::NW - 1], r, 0x5432);
    return o;
  }
  static __device__ __forceinline__ uint32_t ld1(const __half *p) {
    return (uint32_t)*reinterpret_cast<const unsigned short *>(p);
  }
};

// u = m; u = fma(c_xm, x-1, u); ... xp, ym, yp, zm, zp (R10, oracle o16/o32 mirrors)
template <typename P>
__device__ __forceinline__ P spmv(const P (&c)[6], const P &m, const P &xl, const P &xr, const P &ym, const P &yp,
                                  const P &zm, const P &zp) {
  P acc = m;
  acc = P::fma(c[0], xl, acc);
  acc = P::fma(c[1], xr, acc);
  acc = P::fma(c[2], ym, acc);
  acc = P::fma(c[3], yp, acc);
  acc = P::fma(c[4], zm, acc);
  acc = P::fma(c[5], zp, acc);
  return acc;
}

}  // namespace

template <typename T, int BY, int S, int SC, bool CC, int NB, bool FU, bool HD>
__global__ void __launch_bounds__(SrGeo<T, BY, NB>::NT, 1) k_sr(const __grid_constant__ SrArgs a) {
  using P = SPack<T, NB>;
  using G = SrGeo<T, BY, NB>;
  using SH = SrShift<T, NB>;
  using SCn = SrConst<T, NB>;
  constexpr int VEC = G::VEC, H = G::H, HW = G::HW, VW = G::VW, VPR = G::VPR, IE = G::IE, CE = G::CE;
  static_assert(6 % S == 0 && 6 % SC == 0, "stage counts must divide the unroll period");

  if (sr_idle(a.red.st)) return;

  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t *mbar = reinterpret_cast<uint64_t *>(smem);           // [S] inputs, [SC] coefficients
  T *const IN = reinterpret_cast<T *>(smem + 128);               // [S][SE]: 5 boxes of IE (+ the x tile)
  T *const CF = IN + S * G::SE;                                  // [SC][6][CE]
  T *const PR = CF + (CC ? 0 : SC * 6 * CE);                     // p' ring [3][IE]
  T *const RR = PR + 3 * IE;                                     // r' ring [6][IE]
  T *const VR = RR + G::NR * IE;                                 // v' ring [2][CE]
  T *const RHR = VR + 2 * CE;                                    // r_hat ring [6][XE] (RHTMA)
  __shared__ float scratch[32 * kMaxDots];

  int b = blockIdx.x;
  const int tx = b % a.tiles_x;
  b /= a.tiles_x;
  const int ty = b % a.tiles_y;
  const int ci = b / a.tiles_y;
  const int ch = ci < a.ch_lo_n ? ci : a.ch_hi0 + (ci - a.ch_lo_n);
  const int x0 = tx * G::BX, y0 = ty * BY;
  const int z0 = ch < a.nbig ? ch * a.zc : a.nbig * a.zc + (ch - a.nbig) * a.zc_tail;
  const int z1 = min(z0 + (ch < a.nbig ? a.zc : a.zc_tail), a.g.nz);
  const int npi = z1 - z0 + 4;  // steps = staged input planes z0-2 .. z1+1
  const int npc = z1 - z0 + 2;  // staged coefficient planes z0-1 .. z1
  const int tid = threadIdx.x;
  uint64_t pol = 0;
  if (STEN_SR_EVF) asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  uint64_t pol_in = 0;  // bit 3: the halo'd inputs evict-last (bit 4: at fraction 0.5)
  if (STEN_SR_EVF & 16) asm("createpolicy.fractional.L2::evict_last.b64 %0, 0.5;" : "=l"(pol_in));
  else if (STEN_SR_EVF & 8) asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_in));

  // own vector: tile row ry, vector column cx
  const int ry = tid / VPR, cx = tid - (tid / VPR) * VPR;
  const int ei = (ry + 2) * HW + H + cx * VEC;  // in input / formed boxes
  const int ec = (ry + 1) * HW + H + cx * VEC;  // in coefficient / v' boxes
  // one halo item of the formed region (rows 0..RI-1, vector cols 0..VW-1 minus the own tile)
  int hf = -1;
  if (tid < G::NHF) {
    int r, c;
    if (tid < 2 * VW) { r = tid / VW; c = tid % VW; }
    else if (tid < 4 * VW) { r = BY + 2 + (tid - 2 * VW) / VW; c = (tid - 2 * VW) % VW; }
    else { const int m = tid - 4 * VW; r = 2 + m / 2; c = (m & 1) ? VW - 1 : 0; }
    hf = r * HW + G::VOFF + c * VEC;
  }
  // one halo item of the v' region (coef-box rows 0..RC-1, cols 0..VW-1 minus the own tile)
  int hv = -1, hvc = 0;
  if (tid < G::NHV) {
    int r, c;
    if (tid < VW) { r = 0; c = tid; }
    else if (tid < 2 * VW) { r = G::RC - 1; c = tid - VW; }
    else { const int m = tid - 2 * VW; r = 1 + m / 2; c = (m & 1) ? VW - 1 : 0; }
    hv = r * HW + G::VOFF + c * VEC;
    hvc = c;
  }
  const int gx = x0 + cx * VEC, gy = y0 + ry;
  const bool inside = gy < a.g.ny && gx < a.g.nx;
  const long long gofs = (long long)gy * a.g.pitch + gx;
  const long long plane = a.g.plane;
  const int nzl = a.g.nz;
  const bool hb = a.has_below != 0, ha = a.has_above != 0;

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < S + SC; ++s) mbar_init(&mbar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  // STEN_SR_DIAG (traffic diagnostics only - wrong results): bit 0 input boxes without the x halo,
  // bit 1 without the y halo, bit 2 coefficient boxes without halos (the host maps match)
  constexpr int DXH = (STEN_SR_DIAG & 1) ? 0 : H, DYH = (STEN_SR_DIAG & 2) ? 0 : 2;
  constexpr int CXH = (STEN_SR_DIAG & 4) ? 0 : H, CYH = (STEN_SR_DIAG & 4) ? 0 : 1;
  auto issue_in = [&](int qi) {  // plane z0-2+qi of r, p, v, q, y (vectors: 2 halo planes)
    const int slot = qi % S, m = z0 - 2 + qi;
    // x and r_hat only on the chunk's own planes (the four halo planes need neither)
    const bool own = m >= z0 && m < z1;
    mbar_expect_tx(&mbar[slot], (5u * (G::BX + 2 * DXH) * (BY + 2 * DYH) + (own && STEN_SR_XTMA ? G::BX * BY : 0) +
                                 (own && STEN_SR_RHTMA ? G::BX * BY : 0)) *
                                    (uint32_t)sizeof(T));
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      if (STEN_SR_EVF & 8) tma_load_3d_hint(IN + slot * G::SE + i * IE, &a.tm_in[i], x0 - DXH, y0 - DYH, m + 2, &mbar[slot], pol_in);
      else tma_load_3d(IN + slot * G::SE + i * IE, &a.tm_in[i], x0 - DXH, y0 - DYH, m + 2, &mbar[slot]);
    }
    if (!own) {
    } else if (STEN_SR_EVF & 2) {
      tma_load_3d_hint(IN + slot * G::SE + 5 * IE, &a.tm_x, x0, y0, m + 2, &mbar[slot], pol);
      tma_load_3d_hint(RHR + (qi % 6) * G::XE, &a.tm_rh, x0, y0, m + 2, &mbar[slot], pol);
    } else {
      if (STEN_SR_XTMA) tma_load_3d(IN + slot * G::SE + 5 * IE, &a.tm_x, x0, y0, m + 2, &mbar[slot]);
      if (STEN_SR_RHTMA) tma_load_3d(RHR + (qi % 6) * G::XE, &a.tm_rh, x0, y0, m + 2, &mbar[slot]);
    }
  };
  auto issue_c = [&](int qc) {  // plane z0-1+qc of the six coefficient arrays (1 halo plane)
    const int slot = qc % SC, m = z0 - 1 + qc;
    mbar_expect_tx(&mbar[S + slot], 6u * (G::BX + 2 * CXH) * (BY + 2 * CYH) * (uint32_t)sizeof(T));
#pragma unroll
    for (int d = 0; d < 6; ++d) {
      if (STEN_SR_EVF & 4) tma_load_3d_hint(CF + (slot * 6 + d) * CE, &a.tm_c[d], x0 - CXH, y0 - CYH, m + 1, &mbar[S + slot], pol);
      else tma_load_3d(CF + (slot * 6 + d) * CE, &a.tm_c[d], x0 - CXH, y0 - CYH, m + 1, &mbar[S + slot]);
    }
  };
  // optional L2 prefetch (cp.async.bulk.prefetch.tensor) of input planes beyond
  // the shared-memory stages: bytes in flight to HBM without shared memory
  const int l2pf = a.l2pf;
  auto prefetch_in = [&](int qi) {
    if (qi < npi) {
#pragma unroll
      for (int i = 0; i < 5; ++i) tma_prefetch_l2(&a.tm_in[i], x0 - H, y0 - 2, z0 - 2 + qi + 2);
    }
  };
  if (tid == 0) {
    for (int q = 0; q < min(S, npi); ++q) issue_in(q);
    if (!CC)
      for (int q = 0; q < min(SC, npc); ++q) issue_c(q);
    for (int q = S; q < S + l2pf; ++q) prefetch_in(q);
  }
  // CC: the couplings as packs; v' is zero outside the global mesh (lanes
  // [vlo, vhi) of an item's vector are in x, vrow says the row is in y)
  P cst[6];
  int olo = 0, ohi = VEC, hlo = 0, hhi = VEC;
  bool orow = true, hrow = true;
  if (CC) {
#pragma unroll
    for (int d = 0; d < 6; ++d) cst[d] = SCn::splat(a, d);
    const int gxo = x0 + cx * VEC;
    ohi = min(VEC, a.g.nx - gxo);
    orow = (y0 + ry) < a.g.ny;
    if (hv >= 0) {
      const int gxh = x0 + (hvc - 1) * VEC, gyh = y0 - 1 + hv / HW;
      hlo = max(0, -gxh);
      hhi = min(VEC, a.g.nx - gxh);
      hrow = gyh >= 0 && gyh < a.g.ny;
    }
  }

  const typename P::S al_s = P::scalar(a.red.st->alpha), mal_s = P::neg(al_s);
  const typename P::S om_s = P::scalar(a.red.st->omega), mom_s = P::neg(om_s);
  const typename P::S be_s = P::scalar(a.red.st->beta);

  T *const Xg = reinterpret_cast<T *>(a.x);
  const T *const RHg = reinterpret_cast<const T *>(a.rh);
  T *const Og[5] = {reinterpret_cast<T *>(a.out[0]), reinterpret_cast<T *>(a.out[1]), reinterpret_cast<T *>(a.out[2]),
                    reinterpret_cast<T *>(a.out[3]), reinterpret_cast<T *>(a.out[4])};
  // own x / r_hat arrive by plain 16-B loads three planes ahead of their use
  // (x at the step that forms its plane, r_hat at the dots of its plane)
  // fused halo exchange: planes 0, 1 / nz-2, nz-1 of the outputs also to the
  // z-neighbours' halo planes (peer memory)
  T *const PL[5] = {reinterpret_cast<T *>(a.peer_lo[0]), reinterpret_cast<T *>(a.peer_lo[1]),
                    reinterpret_cast<T *>(a.peer_lo[2]), reinterpret_cast<T *>(a.peer_lo[3]),
                    reinterpret_cast<T *>(a.peer_lo[4])};
  T *const PH[5] = {reinterpret_cast<T *>(a.peer_hi[0]), reinterpret_cast<T *>(a.peer_hi[1]),
                    reinterpret_cast<T *>(a.peer_hi[2]), reinterpret_cast<T *>(a.peer_hi[3]),
                    reinterpret_cast<T *>(a.peer_hi[4])};
  auto halo_st = [&](int i, int m, const P &val) {
    if (FU) {  // a compile-time switch: the checks cost 4.7% in the single-GPU sweep
      if (m < 2 && PL[i]) val.st(PL[i] + (long long)m * plane + gofs);
      if (m >= nzl - 2 && PH[i]) val.st(PH[i] + (long long)(m - (nzl - 2)) * plane + gofs);
    }
  };
  // (measured: unconditional loads from clamped addresses with branch-free
  // dots ran 14% slower than these predicated loads)
  auto ld_x = [&](int m) {
    P v = P::zero();
    if (inside && m >= z0 && m < z1) v = P::ldg(Xg + (long long)m * plane + gofs);
    return v;
  };
  auto ld_rh = [&](int k) {
    P v = P::zero();
    if (inside && k < z1) v = P::ldg(RHg + (long long)k * plane + gofs);
    return v;
  };

  // register windows, named by step mod 6 (or mod 3 / mod 2)
  P pw[3], rw[6], vw[3], cw[2][6], xq[3], rq[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    pw[i] = vw[i] = P::zero();
    xq[i] = STEN_SR_XTMA ? P::zero() : ld_x(z0 - 2 + i);  // x of the plane formed at step i
    rq[i] = STEN_SR_RHTMA ? P::zero() : ld_rh(z0 + i);  // r_hat of the plane of the dots at step 4 + i
  }
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    rw[i] = P::zero();
    cw[0][i] = cw[1][i] = P::zero();
  }
  float dacc[12];
#pragma unroll
  for (int d = 0; d < 12; ++d) dacc[d] = 0.0f;
  P hacc[HD ? 12 : 1];  // HD: per-lane fp16 pencils of the twelve sums
#pragma unroll
  for (int d = 0; d < (HD ? 12 : 1); ++d) hacc[d] = P::zero();

  // one step j (= J mod 6): (A) form p', r' of plane m = k+2 and update the own
  // x, r, p; (B) v' = A p' on plane k+1; (C) q' = A r', y' = A v' and the
  // twelve inner products on plane k.  k = z0 - 4 + j.
  auto step = [&](auto JC, int j) {
    constexpr int J = decltype(JC)::value;
    const int k = z0 - 4 + j, m = k + 2;
    // ---------------- (A) ----------------
    mbar_wait(&mbar[J % S], (uint32_t)((j / S) & 1));
    {
      const T *st = IN + (J % S) * G::SE;
      T *pr = PR + (J % 3) * IE;
      T *rr = RR + J * IE;
      const P r = P::ld(st + ei), p = P::ld(st + IE + ei), v = P::ld(st + 2 * IE + ei);
      const P q = P::ld(st + 3 * IE + ei), y = P::ld(st + 4 * IE + ei);
      const P s = P::fmas(mal_s, v, r);
      const P t = P::fmas(mal_s, y, q);
      const P rn = P::fmas(mom_s, t, s);
      const P pn = P::fmas(be_s, P::fmas(mom_s, v, p), rn);
      rn.st(rr + ei);
      pn.st(pr + ei);
      pw[J % 3] = pn;
      rw[J] = rn;
      if (inside && m >= z0 && m < z1) {
        const long long o = (long long)m * plane + gofs;
        const P xv = STEN_SR_XTMA ? P::ld(st + 5 * IE + ry * G::BX + cx * VEC) : xq[J % 3];
        sr_st(P::fmas(om_s, s, P::fmas(al_s, p, xv)), Xg + o, pol);
        sr_st(rn, Og[0] + o, pol);
        sr_st(pn, Og[1] + o, pol);
        halo_st(0, m, rn);
        halo_st(1, m, pn);
      }
      if (!STEN_SR_XTMA) xq[J % 3] = ld_x(m + 3);
      if (hf >= 0) {
        const P hr = P::ld(st + hf), hp = P::ld(st + IE + hf), hv_ = P::ld(st + 2 * IE + hf);
        const P hq = P::ld(st + 3 * IE + hf), hy = P::ld(st + 4 * IE + hf);
        const P hs = P::fmas(mal_s, hv_, hr);
        const P ht = P::fmas(mal_s, hy, hq);
        const P hrn = P::fmas(mom_s, ht, hs);
        P::fmas(be_s, P::fmas(mom_s, hv_, hp), hrn).st(pr + hf);
        hrn.st(rr + hf);
      }
    }
    __syncthreads();
    if (tid == 0) {
      if (j + S < npi) issue_in(j + S);
      if (l2pf) prefetch_in(j + S + l2pf);
    }

    // ---------------- (B) ----------------
    if (j >= 2) {
      constexpr int CS = (J + 6 - 2) % SC;  // coefficient slot of plane k+1 (ordinal j-2)
      if (!CC) mbar_wait(&mbar[S + CS], (uint32_t)(((j - 2) / SC) & 1));
      const T *cf = CF + CS * 6 * CE;
      // CC: plane k+1 exists (a neighbour slab's plane at an interface)?
      const bool zin = (k + 1 >= 0 || hb) && (k + 1 < nzl || ha);
      const T *p0 = PR + ((J + 1) % 3) * IE;  // plane k
      const T *p1 = PR + ((J + 2) % 3) * IE;  // plane k+1
      const T *p2 = PR + (J % 3) * IE;        // plane k+2
      T *vr = VR + ((J + 1) & 1) * CE;
      P (&cn)[6] = cw[J & 1];
      if (!CC) {
#pragma unroll
        for (int d = 0; d < 6; ++d) cn[d] = P::ld(cf + d * CE + ec);
      }
      const P &c1 = pw[(J + 2) % 3];
      const P xl = SH::left(c1, SH::ld1(p1 + ei - 1)), xr = SH::right(c1, SH::ld1(p1 + ei + VEC));
      P vn = spmv<P>(CC ? cst : cn, c1, xl, xr, P::ld(p1 + ei - HW), P::ld(p1 + ei + HW), pw[(J + 1) % 3], pw[J % 3]);
      if (CC) vn = (orow && zin) ? SCn::keep(vn, olo, ohi) : P::zero();
      vn.st(vr + ec);
      vw[J % 3] = vn;
      if (inside && k + 1 >= z0 && k + 1 < z1) {
        sr_st(vn, Og[2] + (long long)(k + 1) * plane + gofs, pol);
        halo_st(2, k + 1, vn);
      }
      if (hv >= 0) {
        const int hp = hv + HW;  // same point in the input-box layout
        P c[6];
#pragma unroll
        for (int d = 0; d < 6; ++d) c[d] = CC ? cst[d] : P::ld(cf + d * CE + hv);
        const P m1 = P::ld(p1 + hp);
        const typename SH::E zl = hvc == 0 ? (typename SH::E)0 : SH::ld1(p1 + hp - 1);
        const typename SH::E zr = hvc == VW - 1 ? (typename SH::E)0 : SH::ld1(p1 + hp + VEC);
        P hvn = spmv<P>(c, m1, SH::left(m1, zl), SH::right(m1, zr), P::ld(p1 + hp - HW), P::ld(p1 + hp + HW),
                        P::ld(p0 + hp), P::ld(p2 + hp));
        if (CC) hvn = (hrow && zin) ? SCn::keep(hvn, hlo, hhi) : P::zero();
        hvn.st(vr + hv);
      }
      __syncthreads();
      if (!CC && tid == 0 && j - 2 + SC < npc) issue_c(j - 2 + SC);
    }

    // ---------------- (C) ----------------
    if (j >= 4) {
      const T *r1 = RR + ((J + 4) % 6) * IE;  // r' plane k
      const T *v1 = VR + (J & 1) * CE;        // v' plane k
      const P (&cc)[6] = CC ? cst : cw[(J + 1) & 1];  // coefficients of plane k (loaded at step j-1)
      const P &rm = rw[(J + 3) % 6], &rc = rw[(J + 4) % 6], &rp = rw[(J + 5) % 6];
      const P &vm = vw[(J + 1) % 3], &vc = vw[(J + 2) % 3], &vp = vw[J % 3];
      P qn = spmv<P>(cc, rc, SH::left(rc, SH::ld1(r1 + ei - 1)), SH::right(rc, SH::ld1(r1 + ei + VEC)),
                     P::ld(r1 + ei - HW), P::ld(r1 + ei + HW), rm, rp);
      P yn = spmv<P>(cc, vc, SH::left(vc, SH::ld1(v1 + ec - 1)), SH::right(vc, SH::ld1(v1 + ec + VEC)),
                     P::ld(v1 + ec - HW), P::ld(v1 + ec + HW), vm, vp);
      if (CC) {  // constant couplings do not vanish outside the mesh: zero q', y' there (lanes >= nx, rows >= ny)
        qn = orow ? SCn::keep(qn, olo, ohi) : P::zero();
        yn = orow ? SCn::keep(yn, olo, ohi) : P::zero();
      }
      // r_hat of plane k: from the ring (it arrived with stage j-2), or loaded three steps ago
      const P rh = STEN_SR_RHTMA ? P::ld(RHR + ((J + 4) % 6) * G::XE + ry * G::BX + cx * VEC) : rq[(J + 2) % 3];
      if (!STEN_SR_RHTMA) rq[(J + 2) % 3] = ld_rh(k + 3);
      if (inside) {
        const long long o = (long long)k * plane + gofs;
        sr_st(qn, Og[3] + o, pol);
        sr_st(yn, Og[4] + o, pol);
        halo_st(3, k, qn);
        halo_st(4, k, yn);
        if constexpr (HD) {  // one fp16 FMA per point into the lane's pencil (R22)
          hacc[0] = P::fma(rh, vc, hacc[0]);
          hacc[1] = P::fma(rh, rc, hacc[1]);
          hacc[2] = P::fma(rh, qn, hacc[2]);
          hacc[3] = P::fma(rh, yn, hacc[3]);
          hacc[4] = P::fma(qn, rc, hacc[4]);
          hacc[5] = P::fma(qn, vc, hacc[5]);
          hacc[6] = P::fma(yn, rc, hacc[6]);
          hacc[7] = P::fma(yn, vc, hacc[7]);
          hacc[8] = P::fma(qn, qn, hacc[8]);
          hacc[9] = P::fma(qn, yn, hacc[9]);
          hacc[10] = P::fma(yn, yn, hacc[10]);
          hacc[11] = P::fma(rc, rc, hacc[11]);
        } else {
          dacc[0] = rh.mdot(vc, dacc[0]);    // (rh, v)
          dacc[1] = rh.mdot(rc, dacc[1]);    // (rh, r)
          dacc[2] = rh.mdot(qn, dacc[2]);    // (rh, q)
          dacc[3] = rh.mdot(yn, dacc[3]);    // (rh, y)
          dacc[4] = qn.mdot(rc, dacc[4]);    // (q, r)
          dacc[5] = qn.mdot(vc, dacc[5]);    // (q, v)
          dacc[6] = yn.mdot(rc, dacc[6]);    // (y, r)
          dacc[7] = yn.mdot(vc, dacc[7]);    // (y, v)
          dacc[8] = qn.mdot(qn, dacc[8]);    // (q, q)
          dacc[9] = qn.mdot(yn, dacc[9]);    // (q, y)
          dacc[10] = yn.mdot(yn, dacc[10]);  // (y, y)
          dacc[11] = rc.mdot(rc, dacc[11]);  // (r, r)
        }
      }
    }
  };

  for (int j = 0; j < npi; j += 6) {
    step(IC<0>{}, j);
    if (j + 1 < npi) step(IC<1>{}, j + 1);
    if (j + 2 < npi) step(IC<2>{}, j + 2);
    if (j + 3 < npi) step(IC<3>{}, j + 3);
    if (j + 4 < npi) step(IC<4>{}, j + 4);
    if (j + 5 < npi) step(IC<5>{}, j + 5);
  }
  if constexpr (HD) {
#pragma unroll
    for (int d = 0; d < 12; ++d) dacc[d] = sr_lanesum(hacc[d]);
  }
  // only the chunks holding a slab's two boundary planes on either side stored to peers
  grid_reduce_finalize<12, PH_SR>(dacc, a.red, scratch, FU && (z0 < 2 || z1 > nzl - 2));
}

// The last sweep of a solve (i = maxit, DevState::light): phase A of k_sr -- the
// same element-wise operations in the same order -- and the sums (rhat, r_maxit)
// and (r_maxit, r_maxit), the only ones the scalar step reads at i = maxit (fin_sr
// stops there); v', q', y' are never used.  A linear stream over the interior.
template <typename T>
__global__ void __launch_bounds__(256) k_sr_last(const __grid_constant__ SrLastArgs a) {
  using P = SPack<T, 16>;
  __shared__ float scratch[32 * kMaxDots];
  const DevState *st = a.red.st;
  if (st->stop || !st->light || st->sweep != st->maxit) return;
  const typename P::S al_s = P::scalar(st->alpha), mal_s = P::neg(al_s);
  const typename P::S om_s = P::scalar(st->omega), mom_s = P::neg(om_s);
  constexpr int VEC = P::VEC;
  T *X = reinterpret_cast<T *>(a.x);
  const T *RH = reinterpret_cast<const T *>(a.rh), *R = reinterpret_cast<const T *>(a.r);
  const T *Pp = reinterpret_cast<const T *>(a.p), *V = reinterpret_cast<const T *>(a.v);
  const T *Q = reinterpret_cast<const T *>(a.q), *Y = reinterpret_cast<const T *>(a.y);
  float dacc[12];
#pragma unroll
  for (int d = 0; d < 12; ++d) dacc[d] = 0.0f;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < a.nvec; i += stride) {
    const long long o = i * VEC;
    const P r = P::ldg(R + o), p = P::ldg(Pp + o), v = P::ldg(V + o), q = P::ldg(Q + o), y = P::ldg(Y + o);
    const P x = P::ldg(X + o), rh = P::ldg(RH + o);
    const P s = P::fmas(mal_s, v, r);
    const P t = P::fmas(mal_s, y, q);
    const P rn = P::fmas(mom_s, t, s);
    P::fmas(om_s, s, P::fmas(al_s, p, x)).st(X + o);
    dacc[1] = rh.mdot(rn, dacc[1]);   // (rh, r)
    dacc[11] = rn.mdot(rn, dacc[11]);  // (r, r)
  }
  grid_reduce_finalize<12, PH_SR>(dacc, a.red, scratch);
}

template <typename T>
int sr_last_launch(const SrLastArgs &a, int grid, cudaStream_t s) {
  k_sr_last<T><<<grid, 256, 0, s>>>(a);
  return (int)cudaGetLastError();
}
template int sr_last_launch<float>(const SrLastArgs &, int, cudaStream_t);
template int sr_last_launch<__half>(const SrLastArgs &, int, cudaStream_t);

// ------------------------------------------------------------ host side --
namespace {
template <typename T, int BY, int S, int SC, bool CC, int NB, bool FU, bool HD = false>
int launch_sr_one(const SrArgs &a, cudaStream_t s) {
  constexpr size_t smem = sr_smem_c<T, BY, S, SC, CC, NB>();
  static_assert(smem <= 227 * 1024, "shared memory budget");
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_sr<T, BY, S, SC, CC, NB, FU, HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return (int)e;
    configured = true;
  }
  const int grid = a.tiles_x * a.tiles_y * a.nch;
  if (grid == 0) return (int)cudaSuccess;
  k_sr<T, BY, S, SC, CC, NB, FU, HD><<<grid, SrGeo<T, BY, NB>::NT, smem, s>>>(a);
  return (int)cudaGetLastError();
}
}  // namespace

// (rows per tile, input stages, coefficient stages, bytes per thread vector)
#define STEN_SR_CONFIGS(X) \
  X(16, 2, 2, 16) X(16, 2, 2, 8) X(8, 2, 2, 16) X(8, 3, 2, 16) X(8, 3, 3, 16) X(8, 2, 2, 8) X(8, 3, 2, 8)

bool sr_config_ok(int by, int stages, int cstages, int pack) {
#define X(B, S_, C_, N_) if (by == B && stages == S_ && cstages == C_ && pack == N_) return true;
  STEN_SR_CONFIGS(X)
#undef X
  return false;
}

// the half-dot variant (R22): fp16 sweeps with the general operator, 16-B packs
#define STEN_SR_HD_CONFIGS(X) X(16, 2, 2, 16) X(8, 2, 2, 16) X(8, 3, 2, 16) X(8, 3, 3, 16)

bool sr_hd_config_ok(int by, int stages, int cstages, int pack) {
#define X(B, S_, C_, N_) if (by == B && stages == S_ && cstages == C_ && pack == N_) return true;
  STEN_SR_HD_CONFIGS(X)
#undef X
  return false;
}

template <typename T>
int sr_launch(const SrArgs &a, int by, int stages, int cstages, int pack, bool cc, bool hd, cudaStream_t s) {
  const bool fu = a.peer_lo[0] || a.peer_hi[0];
  if (hd) {
    if constexpr (std::is_same<T, __half>::value) {
      if (cc || fu) return (int)cudaErrorNotSupported;
#define X(B, S_, C_, N_) \
  if (by == B && stages == S_ && cstages == C_ && pack == N_) return launch_sr_one<T, B, S_, C_, false, N_, false, true>(a, s);
      STEN_SR_HD_CONFIGS(X)
#undef X
    }
    return (int)cudaErrorNotSupported;
  }
#define X(B, S_, C_, N_)                                                                              \
  if (by == B && stages == S_ && cstages == C_ && pack == N_) {                                       \
    if (fu) return cc ? launch_sr_one<T, B, S_, C_, true, N_, true>(a, s)                             \
                      : launch_sr_one<T, B, S_, C_, false, N_, true>(a, s);                           \
    return cc ? launch_sr_one<T, B, S_, C_, true, N_, false>(a, s) : launch_sr_one<T, B, S_, C_, false, N_, false>(a, s); \
  }
  STEN_SR_CONFIGS(X)
#undef X
  return (int)cudaErrorInvalidValue;
}

template <typename T>
size_t sr_smem_bytes(int by, int stages, int cstages, int pack) {
#define X(B, S_, C_, N_) \
  if (by == B && stages == S_ && cstages == C_ && pack == N_) return sr_smem_c<T, B, S_, C_, false, N_>();
  STEN_SR_CONFIGS(X)
#undef X
  return 0;
}

template <typename T>
int sr_threads(int by, int pack) {
  return (tile_bx<T>() / (pack / (int)sizeof(T))) * by;
}

template int sr_launch<float>(const SrArgs &, int, int, int, int, bool, bool, cudaStream_t);
template int sr_launch<__half>(const SrArgs &, int, int, int, int, bool, bool, cudaStream_t);
template size_t sr_smem_bytes<float>(int, int, int, int);
template size_t sr_smem_bytes<__half>(int, int, int, int);
template int sr_threads<float>(int, int);
template int sr_threads<__half>(int, int);

}  // namespace sten
