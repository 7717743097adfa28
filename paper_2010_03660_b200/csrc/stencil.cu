// stencil.cu - the fused 7-point SpMV kernels of the BiCGStab hot path (sm_100a).
//
// u = A v with the unit diagonal left implicit:
//   u_P = v_P + c_xm v_{P-x} + c_xp v_{P+x} + c_ym v_{P-y} + c_yp v_{P+y}
//             + c_zm v_{P-z} + c_zp v_{P+z}
// evaluated as one FMA chain in that order (R10), fp32 FFMA or fp16 HFMA2.
//
// Structure:
//  * A CTA owns an xy tile of BX x BY points (BX = 128 fp16 / 64 fp32, i.e. a
//    256-B row segment) and marches z over a chunk of planes, one 16-byte vector
//    of VEC points per thread.
//  * The operands the SpMV input is built from (halo'd: H1 r, p, v; H2 r, v;
//    APPLY x) arrive plane by plane through a TMA ring of S stages
//    (cp.async.bulk.tensor.3d, mbarrier complete_tx, out-of-mesh zero fill).
//  * The SpMV input plane (H1: p' = r + beta (p - omega v), Alg. 1 l.184;
//    H2: s = r - alpha v, l.178) is formed once per point into a 3-deep shared
//    ring for the xy neighbours; each thread keeps its own column k-1, k, k+1 in
//    registers for the z terms.  One __syncthreads per plane.
//  * The six coefficient arrays (and rhat for H1) are read once per point, as
//    BX x BY TMA tiles into an SC-stage ring of their own (the default, SC = 2;
//    per-thread 16-B loads straddle 32-B sectors on unpadded 1200-B rows).  The
//    older variant (SC = 0, selected by sten_set_tiling with explicit stages)
//    prefetches the tiles into L2 (cp.async.bulk.prefetch.tensor) and each
//    thread loads its 16-B vectors straight into registers one plane ahead.
//  * A launch covers planes [zlo, zhi) of its slab in chunks of zc (the
//    decomposed classic schedule launches the interior and the two boundary
//    planes separately, so the halo exchange overlaps the interior).
//  * The dot products that follow each SpMV in Alg. 1 are accumulated in fp32
//    registers and reduced by the deterministic last-CTA reduction.
#include "sten_internal.cuh"

#include <algorithm>

namespace sten {

namespace {

constexpr int align128c(int b) { return (b + 127) & ~127; }

template <typename T, int MODE, int BY>
struct Geo {
  static constexpr int VEC = Pack<T>::VEC;
  static constexpr int BX = tile_bx<T>();
  static constexpr int H = VEC;                 // x halo pad (keeps 16-B vectors aligned)
  static constexpr int VPR = BX / VEC;          // vectors per tile row
  static constexpr int NT = VPR * BY;           // threads: one output vector each
  static constexpr int HW = BX + 2 * H;         // halo box width (elements)
  static constexpr int HBOX = HW * (BY + 2);    // halo box elements
  static constexpr int HBYTES = align128c(HBOX * (int)sizeof(T));
  static constexpr int NIN = MODE == MODE_H1 ? 3 : (MODE == MODE_H2 ? 2 : 1);
  static constexpr int NHALO = 2 * VPR + 2 * BY;  // halo vectors formed per plane
};

// SC > 0: the six coefficient tiles (and rhat for H1) of a plane arrive by TMA
// into an SC-stage ring (no per-thread global loads on misaligned rows)
// (CC: constant couplings - only rhat's tile for H1, none for H2 / APPLY)
template <typename T, int MODE, int BY, bool CC = false>
struct CGeo {
  static constexpr int NC = CC ? (MODE == MODE_H1 ? 1 : 0) : (MODE == MODE_H1 ? 7 : 6);  // tiles per plane
  static constexpr int RH = CC ? 0 : 6;                                                 // rhat's tile index
  static constexpr int XE = align128c(tile_bx<T>() * BY * (int)sizeof(T)) / (int)sizeof(T);  // elements per tile
};

template <typename T, int MODE, int BY, int S, int SC = 0, bool CC = false>
constexpr size_t smem_bytes_c() {
  using G = Geo<T, MODE, BY>;
  using C = CGeo<T, MODE, BY, CC>;
  return 128 /* mbarriers */ + (size_t)S * G::NIN * G::HBYTES + 3 * (size_t)G::HBYTES +
         (size_t)SC * C::NC * C::XE * sizeof(T);
}

__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap *map, int x, int y, int z) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(z)
               : "memory");
}

// x-1 / x+1 neighbours of a vector given the single elements left and right of it
template <typename T> struct Shift;
template <> struct Shift<float> {
  static __device__ __forceinline__ Pack<float> left(const Pack<float> &c, float l) {
    return Pack<float>{{l, c.v[0], c.v[1], c.v[2]}};
  }
  static __device__ __forceinline__ Pack<float> right(const Pack<float> &c, float r) {
    return Pack<float>{{c.v[1], c.v[2], c.v[3], r}};
  }
  static __device__ __forceinline__ float ld1(const float *p) { return *p; }
};
template <> struct Shift<__half> {
  static __device__ __forceinline__ Pack<__half> left(const Pack<__half> &c, uint32_t l) {
    return Pack<__half>{{__byte_perm(l, c.w[0], 0x5410), __byte_perm(c.w[0], c.w[1], 0x5432),
                         __byte_perm(c.w[1], c.w[2], 0x5432), __byte_perm(c.w[2], c.w[3], 0x5432)}};
  }
  static __device__ __forceinline__ Pack<__half> right(const Pack<__half> &c, uint32_t r) {
    return Pack<__half>{{__byte_perm(c.w[0], c.w[1], 0x5432), __byte_perm(c.w[1], c.w[2], 0x5432),
                         __byte_perm(c.w[2], c.w[3], 0x5432), __byte_perm(c.w[3], r, 0x5432)}};
  }
  static __device__ __forceinline__ uint32_t ld1(const __half *p) {
    return (uint32_t)*reinterpret_cast<const unsigned short *>(p);
  }
};

}  // namespace

// the lanes of an fp16 pencil pack widened and added in fp32, in lane order (half dots, R22)
__device__ __forceinline__ float pencil_sum(const Pack<__half> &h) {
  float s = 0.0f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __half22float2(Pack<__half>::h2(h.w[i]));
    s += f.x;
    s += f.y;
  }
  return s;
}
__device__ __forceinline__ float pencil_sum(const Pack<float> &h) { return (h.v[0] + h.v[1]) + (h.v[2] + h.v[3]); }

// constant couplings as packs, and "keep the first n lanes" (CC outputs outside the mesh are 0)
template <typename T> struct CcPack;
template <> struct CcPack<float> {
  static __device__ __forceinline__ Pack<float> splat(const StencilArgs &a, int d) {
    const float c = a.cf32[d];
    return Pack<float>{{c, c, c, c}};
  }
  static __device__ __forceinline__ Pack<float> keep(const Pack<float> &v, int n) {
    Pack<float> o;
#pragma unroll
    for (int i = 0; i < 4; ++i) o.v[i] = i < n ? v.v[i] : 0.0f;
    return o;
  }
};
template <> struct CcPack<__half> {
  static __device__ __forceinline__ Pack<__half> splat(const StencilArgs &a, int d) {
    const uint32_t h = a.cf16[d];
    return Pack<__half>{{h | (h << 16), h | (h << 16), h | (h << 16), h | (h << 16)}};
  }
  static __device__ __forceinline__ Pack<__half> keep(const Pack<__half> &v, int n) {
    Pack<__half> o;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      o.w[i] = v.w[i] & ((2 * i < n ? 0x0000FFFFu : 0u) | (2 * i + 1 < n ? 0xFFFF0000u : 0u));
    return o;
  }
};

template <typename T, int MODE, int BY, int S, int SC, bool FU = false, bool HD = false, bool CC = false>
__global__ void __launch_bounds__(Geo<T, MODE, BY>::NT, 2) k_stencil(const __grid_constant__ StencilArgs a) {
  using P = Pack<T>;
  using G = Geo<T, MODE, BY>;
  using CG = CGeo<T, MODE, BY, CC>;
  constexpr int VEC = G::VEC, BX = G::BX, H = G::H, HW = G::HW, NIN = G::NIN;
  constexpr int HSTR = G::HBYTES / (int)sizeof(T);  // elements between halo boxes
  constexpr int ND = MODE == MODE_H2 ? 2 : 1;
  static_assert(!CC || SC > 0, "the constant-coefficient kernels take rhat through the tile ring");

  if (MODE != MODE_APPLY && st_idle(a.red.st)) return;

  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t *mbar = reinterpret_cast<uint64_t *>(smem);
  T *stage0 = reinterpret_cast<T *>(smem + 128);         // [S][NIN][HSTR]
  T *U = stage0 + S * NIN * HSTR;                       // [3][HSTR]
  T *CF = U + 3 * HSTR;                                  // [SC][NC][XE] coefficient (+ rhat) tiles
  __shared__ float scratch[32 * kMaxDots];

  int b = blockIdx.x;
  const int tx = b % a.tiles_x;
  b /= a.tiles_x;
  const int ty = b % a.tiles_y;
  const int ch = b / a.tiles_y;
  const int x0 = tx * BX, y0 = ty * BY;
  const int z0 = a.zlo + ch * a.zc, z1 = min(z0 + a.zc, a.zhi);
  const int np = z1 - z0 + 2;  // staged planes z0-1 .. z1
  const int tid = threadIdx.x;

  // own output vector and (for the first NHALO threads) one halo vector
  const int ry = tid / G::VPR, cx = tid - (tid / G::VPR) * G::VPR;
  const int hown = (ry + 1) * HW + H + cx * VEC;
  int hhalo = -1;
  if (tid < G::VPR) hhalo = H + tid * VEC;                                     // row y0-1
  else if (tid < 2 * G::VPR) hhalo = (BY + 1) * HW + H + (tid - G::VPR) * VEC;  // row y0+BY
  else if (tid < 2 * G::VPR + BY) hhalo = (tid - 2 * G::VPR + 1) * HW;          // x0-H .. x0-1
  else if (tid < G::NHALO) hhalo = (tid - 2 * G::VPR - BY + 1) * HW + H + BX;   // x0+BX ..
  const int gx = x0 + cx * VEC, gy = y0 + ry;
  const bool inside = gy < a.g.ny && gx < a.g.nx;
  const long long gofs = (long long)gy * a.g.pitch + gx;

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < S + SC; ++s) mbar_init(&mbar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  auto issue_c = [&](int k) {  // coefficient (+ rhat) tiles of plane k, one thread
    if (CG::NC == 0) return;
    const int s = (k - z0) % (SC > 0 ? SC : 1);
    mbar_expect_tx(&mbar[S + s], CG::NC * BX * BY * (uint32_t)sizeof(T));
    if (!CC)
#pragma unroll
      for (int d = 0; d < 6; ++d) tma_load_3d(CF + (s * CG::NC + d) * CG::XE, &a.tm_c[d], x0, y0, k, &mbar[S + s]);
    if (MODE == MODE_H1) tma_load_3d(CF + (s * CG::NC + CG::RH) * CG::XE, &a.tm_aux, x0, y0, k + 1, &mbar[S + s]);
  };
  auto issue = [&](int q) {  // planes z0-1+q of every halo'd operand, one thread
    const int s = q % S, p = z0 - 1 + q;
    mbar_expect_tx(&mbar[s], NIN * G::HBOX * (uint32_t)sizeof(T));
#pragma unroll
    for (int i = 0; i < NIN; ++i) tma_load_3d(stage0 + (s * NIN + i) * HSTR, &a.tm_in[i], x0 - H, y0 - 1, p + 1, &mbar[s]);
  };
  auto prefetch = [&](int k) {  // coefficient (+ rhat) tiles of plane k into L2
    if (k < z1) {
#pragma unroll
      for (int d = 0; d < 6; ++d) tma_prefetch_3d(&a.tm_c[d], x0, y0, k);
      if (MODE == MODE_H1) tma_prefetch_3d(&a.tm_aux, x0, y0, k + 1);
    }
  };
  if (tid == 0) {
    for (int q = 0; q < min(S, np); ++q) issue(q);
    if (SC > 0)
      for (int k = z0; k < min(z0 + SC, z1); ++k) issue_c(k);
    else
      for (int k = z0; k < z0 + a.pf; ++k) prefetch(k);
  }
  // coefficients (+ rhat) of a plane straight into registers, one plane ahead
  const T *const *cp = reinterpret_cast<const T *const *>(a.cptr);
  P cn[6], rhn;
  auto load_coefs = [&](int k) {
    if (inside && k < z1) {
      const long long o = (long long)k * a.g.plane + gofs;
#pragma unroll
      for (int d = 0; d < 6; ++d) cn[d] = P::ldg(cp[d] + o);
      if (MODE == MODE_H1) rhn = P::ldg(reinterpret_cast<const T *>(a.aux) + o + a.g.plane);
    } else {
#pragma unroll
      for (int d = 0; d < 6; ++d) cn[d] = P::zero();
      rhn = P::zero();
    }
  };
  if (SC == 0) load_coefs(z0);

  typename P::S beta_s{}, momega_s{}, malpha_s{};
  if (MODE == MODE_H1) {
    beta_s = P::scalar(a.red.st->beta);
    momega_s = P::neg(P::scalar(a.red.st->omega));
  } else if (MODE == MODE_H2) {
    malpha_s = P::neg(P::scalar(a.red.st->alpha));
  }
  // SpMV input at box offset h of staged plane q
  auto form = [&](int q, int h) -> P {
    const T *in = stage0 + (q % S) * NIN * HSTR;
    P o = P::ld(in + h);
    if (MODE == MODE_H1) o = P::fmas(beta_s, P::fmas(momega_s, P::ld(in + 2 * HSTR + h), P::ld(in + HSTR + h)), o);
    else if (MODE == MODE_H2) o = P::fmas(malpha_s, P::ld(in + HSTR + h), o);
    return o;
  };
  auto wait = [&](int q) { mbar_wait(&mbar[q % S], (uint32_t)((q / S) & 1)); };

  // prologue: planes z0-1 (own column only) and z0 (own + halo into U ring)
  wait(0);
  P um = form(0, hown);
  wait(1);
  P uc = form(1, hown);
  uc.st(U + 1 * HSTR + hown);
  if (hhalo >= 0) form(1, hhalo).st(U + 1 * HSTR + hhalo);
  __syncthreads();
  if (tid == 0) {
    if (S < np) issue(S);
    if (S + 1 < np) issue(S + 1);
  }

  float dacc[ND][4];
#pragma unroll
  for (int d = 0; d < ND; ++d)
#pragma unroll
    for (int i = 0; i < 4; ++i) dacc[d][i] = 0.0f;
  P hacc[ND];  // HD: the column pencils, fp16 running sums from +0 (R22)
#pragma unroll
  for (int d = 0; d < ND; ++d) hacc[d] = P::zero();

  for (int k = z0; k < z1; ++k) {
    const int qc = k - z0 + 1, qn = qc + 1;
    P c[6], rh;
    if (CC) {  // constant couplings; rhat (H1) from the ring
#pragma unroll
      for (int d = 0; d < 6; ++d) c[d] = CcPack<T>::splat(a, d);
      if (MODE == MODE_H1) {
        const int cs = (k - z0) % (SC > 0 ? SC : 1);
        mbar_wait(&mbar[S + cs], (uint32_t)(((k - z0) / (SC > 0 ? SC : 1)) & 1));
        rh = P::ld(CF + cs * CG::NC * CG::XE + ry * BX + cx * VEC);
      }
    } else if (SC > 0) {  // this plane's tiles from the ring (slot refilled after the barrier below)
      const int cs = (k - z0) % (SC > 0 ? SC : 1);
      mbar_wait(&mbar[S + cs], (uint32_t)(((k - z0) / (SC > 0 ? SC : 1)) & 1));
      const T *cf = CF + cs * CG::NC * CG::XE + ry * BX + cx * VEC;
#pragma unroll
      for (int d = 0; d < 6; ++d) c[d] = P::ld(cf + d * CG::XE);
      if (MODE == MODE_H1) rh = P::ld(cf + 6 * CG::XE);
    } else {
#pragma unroll
      for (int d = 0; d < 6; ++d) c[d] = cn[d];
      rh = rhn;
      load_coefs(k + 1);  // in flight during this plane's work
      if (tid == 0 && a.pf > 0) prefetch(k + a.pf);
    }
    // SpMV input of plane k+1
    wait(qn);
    T *Un = U + (qn % 3) * HSTR;
    const P up = form(qn, hown);
    up.st(Un + hown);
    if (hhalo >= 0) form(qn, hhalo).st(Un + hhalo);
    __syncthreads();
    if (tid == 0 && qn + S < np) issue(qn + S);  // stage of plane k+1 is consumed
    if (SC > 0 && tid == 0 && k + SC < z1) issue_c(k + SC);  // and the coefficient slot of plane k
    // u_k = v_k + sum of the six products (order xm, xp, ym, yp, zm, zp)
    const T *Uc = U + (qc % 3) * HSTR;
    P acc = uc;
    acc = P::fma(c[0], Shift<T>::left(uc, Shift<T>::ld1(Uc + hown - 1)), acc);
    acc = P::fma(c[1], Shift<T>::right(uc, Shift<T>::ld1(Uc + hown + VEC)), acc);
    acc = P::fma(c[2], P::ld(Uc + hown - HW), acc);
    acc = P::fma(c[3], P::ld(Uc + hown + HW), acc);
    acc = P::fma(c[4], um, acc);
    acc = P::fma(c[5], up, acc);
    // CC: the couplings are not zero outside the mesh (the arrays' are), so points past nx / ny
    // would see their in-mesh neighbours: they are 0 here, as the array kernels compute them
    if (CC) acc = inside ? CcPack<T>::keep(acc, a.g.nx - gx) : P::zero();
    if (inside) {
      const long long o = (long long)(k + 1) * a.g.plane + gofs;
      acc.st(reinterpret_cast<T *>(a.out0) + o);
      if (MODE != MODE_APPLY) uc.st(reinterpret_cast<T *>(a.out1) + o);
      if (FU) {  // fused exchange: the slab's boundary planes into the z-neighbours' halo planes
        if (k == 0 && a.peer_lo[0]) {
          acc.st(reinterpret_cast<T *>(a.peer_lo[0]) + gofs);
          uc.st(reinterpret_cast<T *>(a.peer_lo[1]) + gofs);
        }
        if (k == a.g.nz - 1 && a.peer_hi[0]) {
          acc.st(reinterpret_cast<T *>(a.peer_hi[0]) + gofs);
          uc.st(reinterpret_cast<T *>(a.peer_hi[1]) + gofs);
        }
      }
    }
    if (HD) {  // one fp16 FMA per point into the lane's pencil (o16h_dot order: fma16(a, b, acc))
      if (MODE == MODE_H1) {
        hacc[0] = P::fma(rh, acc, hacc[0]);  // (rhat, v')
      } else if (MODE == MODE_H2) {
        hacc[0] = P::fma(acc, uc, hacc[0]);       // (t, s)
        hacc[ND - 1] = P::fma(acc, acc, hacc[ND - 1]);  // (t, t)
      }
    } else if (MODE == MODE_H1) {
      rh.dot4(acc, dacc[0]);  // (rhat, v')
    } else if (MODE == MODE_H2) {
      acc.dot4(uc, dacc[0]);        // (t, s)
      acc.dot4(acc, dacc[ND - 1]);  // (t, t)
    }
    um = uc;
    uc = up;
  }

  if (MODE != MODE_APPLY) {
    float v[ND];
#pragma unroll
    for (int d = 0; d < ND; ++d) v[d] = HD ? pencil_sum(hacc[d]) : sum4(dacc[d]);
    const bool peer = FU && (z0 == 0 || z1 == a.g.nz);  // only boundary-plane chunks stored to peers
    if (MODE == MODE_H1) grid_reduce_finalize<ND, PH_H1>(v, a.red, scratch, peer);
    else grid_reduce_finalize<ND, PH_H2>(v, a.red, scratch, peer);
  }
}

// ============================================================ row strips ==
// k_rows: a CTA owns BY complete mesh rows (all of x) and marches z.  With no x
// halo every TMA box row is whole 128-B lines of this CTA's own rows, and the
// only re-read data are the two y-halo rows, which the y-neighbour CTAs (next
// blockIdx) read at about the same time (L2 hits).  A strip plane of one
// operand arrives as pitch/64 TMA boxes of 64 x (BY+2) elements; shared memory
// holds them box-major, element (row r, x) at (x/64)*(BY+2)*64 + r*64 + x%64.
constexpr int kRowBox = 64;  // elements per TMA box row (128 B fp16, 256 B fp32)

template <typename T, int MODE, int BY, int S>
__global__ void __launch_bounds__(512, 1) k_rows(const __grid_constant__ StencilArgs a) {
  using P = Pack<T>;
  constexpr int VEC = P::VEC, W = kRowBox, RB = BY + 2;
  constexpr int NIN = MODE == MODE_H1 ? 3 : (MODE == MODE_H2 ? 2 : 1);
  constexpr int ND = MODE == MODE_H2 ? 2 : 1;

  if (MODE != MODE_APPLY && st_idle(a.red.st)) return;

  const int pitch = a.g.pitch;
  const int nb = (a.g.nx + W - 1) / W;      // boxes per strip row (last one zero-filled past nx)
  const int astr = nb * RB * W;             // elements per staged operand (128-B multiple)
  const int vpr = (a.g.nx + VEC - 1) / VEC; // point-holding vectors per row
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t *mbar = reinterpret_cast<uint64_t *>(smem);
  T *stage0 = reinterpret_cast<T *>(smem + 128);  // [S][NIN][astr]
  T *U = stage0 + S * NIN * astr;                 // [3][astr]
  __shared__ float scratch[32 * kMaxDots];

  const int ty = blockIdx.x % a.tiles_y;  // y-neighbours are consecutive CTAs
  const int ch = blockIdx.x / a.tiles_y;
  const int y0 = ty * BY;
  const int z0 = a.zlo + ch * a.zc, z1 = min(z0 + a.zc, a.zhi);
  const int np = z1 - z0 + 2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  auto sidx = [&](int r, int x) { return (x / W) * (RB * W) + r * W + (x % W); };
  const int ry = tid / vpr, cx = tid - (tid / vpr) * vpr;
  const int x = cx * VEC;
  const bool active = ry < BY;  // blockDim may be rounded up to whole warps
  const int hown = active ? sidx(ry + 1, x) : 0;
  const int hleft = (active && x > 0) ? sidx(ry + 1, x - 1) : -1;
  // U columns >= vpr*VEC are never formed: a right neighbour at x+VEC >= nx is
  // outside the mesh and must be an exact zero (0 * stale data could be NaN)
  const int hright = (active && x + VEC < a.g.nx) ? sidx(ry + 1, x + VEC) : -1;
  int hhalo = -1;
  if (tid < 2 * vpr) hhalo = sidx(tid < vpr ? 0 : RB - 1, (tid % vpr) * VEC);
  const int gy = y0 + ry;
  const bool inside = active && gy < a.g.ny;
  const long long gofs = (long long)gy * pitch + x;

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < S; ++s) mbar_init(&mbar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  auto issue = [&](int q) {  // warp 0: lane j issues box j of every operand
    const int s = q % S, p = z0 - 1 + q;
    if (lane == 0) mbar_expect_tx(&mbar[s], (uint32_t)(NIN * nb * RB * W * (int)sizeof(T)));
    __syncwarp();
    for (int j = lane; j < nb; j += 32)
#pragma unroll
      for (int i = 0; i < NIN; ++i)
        tma_load_3d(stage0 + (s * NIN + i) * astr + j * RB * W, &a.tm_in[i], j * W, y0 - 1, p + 1, &mbar[s]);
  };
  if (warp == 0)
    for (int q = 0; q < min(S, np); ++q) issue(q);

  const T *const *cp = reinterpret_cast<const T *const *>(a.cptr);
  P cn[6], rhn;
  auto load_coefs = [&](int k) {
    if (inside && k < z1) {
      const long long o = (long long)k * a.g.plane + gofs;
#pragma unroll
      for (int d = 0; d < 6; ++d) cn[d] = P::ldg(cp[d] + o);
      if (MODE == MODE_H1) rhn = P::ldg(reinterpret_cast<const T *>(a.aux) + o + a.g.plane);
    } else {
#pragma unroll
      for (int d = 0; d < 6; ++d) cn[d] = P::zero();
      rhn = P::zero();
    }
  };
  load_coefs(z0);

  typename P::S beta_s{}, momega_s{}, malpha_s{};
  if (MODE == MODE_H1) {
    beta_s = P::scalar(a.red.st->beta);
    momega_s = P::neg(P::scalar(a.red.st->omega));
  } else if (MODE == MODE_H2) {
    malpha_s = P::neg(P::scalar(a.red.st->alpha));
  }
  auto form = [&](int q, int h) -> P {
    const T *in = stage0 + (q % S) * NIN * astr;
    P o = P::ld(in + h);
    if (MODE == MODE_H1) o = P::fmas(beta_s, P::fmas(momega_s, P::ld(in + 2 * astr + h), P::ld(in + astr + h)), o);
    else if (MODE == MODE_H2) o = P::fmas(malpha_s, P::ld(in + astr + h), o);
    return o;
  };
  auto wait = [&](int q) { mbar_wait(&mbar[q % S], (uint32_t)((q / S) & 1)); };

  wait(0);
  P um = form(0, hown);
  wait(1);
  P uc = form(1, hown);
  if (active) uc.st(U + 1 * astr + hown);
  if (hhalo >= 0) form(1, hhalo).st(U + 1 * astr + hhalo);
  __syncthreads();
  if (warp == 0) {
    if (S < np) issue(S);
    if (S + 1 < np) issue(S + 1);
  }

  float dacc[ND][4];
#pragma unroll
  for (int d = 0; d < ND; ++d)
#pragma unroll
    for (int i = 0; i < 4; ++i) dacc[d][i] = 0.0f;

  for (int k = z0; k < z1; ++k) {
    const int qc = k - z0 + 1, qn = qc + 1;
    P c[6], rh;
#pragma unroll
    for (int d = 0; d < 6; ++d) c[d] = cn[d];
    rh = rhn;
    load_coefs(k + 1);
    wait(qn);
    T *Un = U + (qn % 3) * astr;
    const P up = form(qn, hown);
    if (active) up.st(Un + hown);
    if (hhalo >= 0) form(qn, hhalo).st(Un + hhalo);
    __syncthreads();
    if (warp == 0 && qn + S < np) issue(qn + S);
    const T *Uc = U + (qc % 3) * astr;
    P acc = uc;
    const auto zl = Shift<T>::ld1(Uc + (hleft >= 0 ? hleft : hown)), zr = Shift<T>::ld1(Uc + (hright >= 0 ? hright : hown));
    acc = P::fma(c[0], Shift<T>::left(uc, hleft >= 0 ? zl : decltype(zl)(0)), acc);
    acc = P::fma(c[1], Shift<T>::right(uc, hright >= 0 ? zr : decltype(zr)(0)), acc);
    acc = P::fma(c[2], P::ld(Uc + hown - W), acc);
    acc = P::fma(c[3], P::ld(Uc + hown + W), acc);
    acc = P::fma(c[4], um, acc);
    acc = P::fma(c[5], up, acc);
    if (inside) {
      const long long o = (long long)(k + 1) * a.g.plane + gofs;
      acc.st(reinterpret_cast<T *>(a.out0) + o);
      if (MODE != MODE_APPLY) uc.st(reinterpret_cast<T *>(a.out1) + o);
    }
    if (MODE == MODE_H1 && active) {
      rh.dot4(acc, dacc[0]);
    } else if (MODE == MODE_H2 && active) {
      acc.dot4(uc, dacc[0]);
      acc.dot4(acc, dacc[ND - 1]);
    }
    um = uc;
    uc = up;
  }

  if (MODE != MODE_APPLY) {
    float v[ND];
#pragma unroll
    for (int d = 0; d < ND; ++d) v[d] = sum4(dacc[d]);
    if (MODE == MODE_H1) grid_reduce_finalize<ND, PH_H1>(v, a.red, scratch);
    else grid_reduce_finalize<ND, PH_H2>(v, a.red, scratch);
  }
}

size_t rows_smem_bytes(int mode, int esz, int pitch, int by, int stages) {
  const int nin = mode == MODE_H1 ? 3 : (mode == MODE_H2 ? 2 : 1);
  const size_t astr = (size_t)((pitch + kRowBox - 1) / kRowBox) * (by + 2) * kRowBox * esz;
  return 128 + (size_t)stages * nin * astr + 3 * astr;
}

template <typename T>
int rows_threads(int nx, int by) {
  const int vpr = (nx + Pack<T>::VEC - 1) / Pack<T>::VEC;
  return (vpr * by + 31) / 32 * 32;
}

// ------------------------------------------------------------ host side --
namespace {
template <typename T, int MODE, int BY, int S>
int launch_rows(const StencilArgs &a, cudaStream_t s) {
  const size_t smem = rows_smem_bytes(MODE, (int)sizeof(T), a.g.pitch, BY, S);
  static size_t configured = 0;
  if (configured < smem) {
    cudaError_t e = cudaFuncSetAttribute(k_rows<T, MODE, BY, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
    configured = smem;
  }
  const int grid = a.tiles_y * ((a.zhi - a.zlo + a.zc - 1) / a.zc);
  k_rows<T, MODE, BY, S><<<grid, rows_threads<T>(a.g.nx, BY), smem, s>>>(a);
  return (int)cudaGetLastError();
}
template <typename T, int MODE>
int launch_rows_mode(const StencilArgs &a, int by, int stages, cudaStream_t s) {
  if (by == 2 && stages == 3) return launch_rows<T, MODE, 2, 3>(a, s);
  if (by == 2 && stages == 4) return launch_rows<T, MODE, 2, 4>(a, s);
  if (by == 4 && stages == 3) return launch_rows<T, MODE, 4, 3>(a, s);
  if (by == 4 && stages == 4) return launch_rows<T, MODE, 4, 4>(a, s);
  if (by == 8 && stages == 3) return launch_rows<T, MODE, 8, 3>(a, s);
  return (int)cudaErrorInvalidValue;
}
}  // namespace

bool rows_config_ok(int by, int stages) {
  return ((by == 2 || by == 4) && (stages == 3 || stages == 4)) || (by == 8 && stages == 3);
}

template <typename T>
int rows_launch(int mode, const StencilArgs &a, int by, int stages, cudaStream_t s) {
  if (mode == MODE_H1) return launch_rows_mode<T, MODE_H1>(a, by, stages, s);
  if (mode == MODE_H2) return launch_rows_mode<T, MODE_H2>(a, by, stages, s);
  return launch_rows_mode<T, MODE_APPLY>(a, by, stages, s);
}
template int rows_launch<float>(int, const StencilArgs &, int, int, cudaStream_t);
template int rows_launch<__half>(int, const StencilArgs &, int, int, cudaStream_t);
template int rows_threads<float>(int, int);
template int rows_threads<__half>(int, int);

// ------------------------------------------------------------ host side --
namespace {
template <typename T, int MODE, int BY, int S, int SC = 0, bool FU = false, bool HD = false, bool CC = false>
int launch_one(const StencilArgs &a, cudaStream_t s) {
  using G = Geo<T, MODE, BY>;
  constexpr size_t smem = smem_bytes_c<T, MODE, BY, S, SC, CC>();
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_stencil<T, MODE, BY, S, SC, FU, HD, CC>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
    configured = true;
  }
  const int grid = a.tiles_x * a.tiles_y * ((a.zhi - a.zlo + a.zc - 1) / a.zc);
  k_stencil<T, MODE, BY, S, SC, FU, HD, CC><<<grid, G::NT, smem, s>>>(a);
  return (int)cudaGetLastError();
}
template <typename T, int MODE>
int launch_mode(const StencilArgs &a, int by, int stages, int cstages, cudaStream_t s) {
  if (a.cc) {  // constant couplings: the default tiling only
    if (by == 16 && stages == 2 && cstages == 2) return launch_one<T, MODE, 16, 2, 2, false, false, true>(a, s);
    return (int)cudaErrorNotSupported;
  }
  if (cstages) {  // coefficient tiles by TMA
    if (by == 16 && stages == 2 && cstages == 2) return launch_one<T, MODE, 16, 2, 2>(a, s);
    if (by == 16 && stages == 3 && cstages == 1) return launch_one<T, MODE, 16, 3, 1>(a, s);
    if (by == 16 && stages == 2 && cstages == 1) return launch_one<T, MODE, 16, 2, 1>(a, s);
    if (by == 8 && stages == 3 && cstages == 2) return launch_one<T, MODE, 8, 3, 2>(a, s);
    return (int)cudaErrorInvalidValue;
  }
  if (by == 8 && stages == 3) return launch_one<T, MODE, 8, 3>(a, s);
  if (by == 8 && stages == 4) return launch_one<T, MODE, 8, 4>(a, s);
  if (by == 16 && stages == 3) return launch_one<T, MODE, 16, 3>(a, s);
  if (by == 16 && stages == 4) return launch_one<T, MODE, 16, 4>(a, s);
  if (by == 4 && stages == 4) return launch_one<T, MODE, 4, 4>(a, s);
  return (int)cudaErrorInvalidValue;
}
template <typename T, int MODE>
size_t smem_mode(int by, int stages) {
  if (by == 8 && stages == 3) return smem_bytes_c<T, MODE, 8, 3>();
  if (by == 8 && stages == 4) return smem_bytes_c<T, MODE, 8, 4>();
  if (by == 16 && stages == 3) return smem_bytes_c<T, MODE, 16, 3>();
  if (by == 16 && stages == 4) return smem_bytes_c<T, MODE, 16, 4>();
  if (by == 4 && stages == 4) return smem_bytes_c<T, MODE, 4, 4>();
  return 0;
}
}  // namespace

bool stencil_config_ok(int by, int stages, int cstages) {
  if (cstages)
    return (by == 16 && ((stages == 2 && (cstages == 1 || cstages == 2)) || (stages == 3 && cstages == 1))) ||
           (by == 8 && stages == 3 && cstages == 2);
  return (by == 8 && (stages == 3 || stages == 4)) || (by == 16 && (stages == 3 || stages == 4)) ||
         (by == 4 && stages == 4);
}

template <typename T>
int stencil_launch(int mode, const StencilArgs &a, int by, int stages, int cstages, cudaStream_t s) {
  if (mode == MODE_H1) return launch_mode<T, MODE_H1>(a, by, stages, cstages, s);
  if (mode == MODE_H2) return launch_mode<T, MODE_H2>(a, by, stages, cstages, s);
  return launch_mode<T, MODE_APPLY>(a, by, stages, cstages, s);
}
template <typename T>
size_t stencil_smem_bytes(int mode, int by, int stages) {
  if (mode == MODE_H1) return smem_mode<T, MODE_H1>(by, stages);
  if (mode == MODE_H2) return smem_mode<T, MODE_H2>(by, stages);
  return smem_mode<T, MODE_APPLY>(by, stages);
}
template <typename T>
int stencil_threads(int by) {
  return (tile_bx<T>() / Pack<T>::VEC) * by;
}

template <typename T>
int stencil_launch_fused(const StencilArgs &a, int by, int stages, int cstages, cudaStream_t s) {
  if (by == 16 && stages == 2 && cstages == 2)
    return a.cc ? launch_one<T, MODE_H1, 16, 2, 2, true, false, true>(a, s) : launch_one<T, MODE_H1, 16, 2, 2, true>(a, s);
  return (int)cudaErrorNotSupported;
}
int stencil_launch_half(int mode, const StencilArgs &a, int by, int stages, int cstages, cudaStream_t s) {
  if (!(by == 16 && stages == 2 && cstages == 2)) return (int)cudaErrorNotSupported;
  if (mode == MODE_H1) return launch_one<__half, MODE_H1, 16, 2, 2, false, true>(a, s);
  if (mode == MODE_H2) return launch_one<__half, MODE_H2, 16, 2, 2, false, true>(a, s);
  return (int)cudaErrorNotSupported;
}

// ---------------------------------------------- H3 half (R28): a z-march --
// x += alpha p + omega s, r = s - omega t (the k_h3 operation order), with (rhat, r) and (r, r) as
// fp16 column pencils over the chunk (one fp16 FMA per point, z ascending from +0), so that the
// classic half mode's pencils follow one z-chunk plan in all three phases.  A CTA owns a BX x BY
// tile and marches its chunk; two planes per trip keep ten loads in flight.
template <int BY>
__global__ void __launch_bounds__((128 / 8) * BY) k_h3z_half(const __grid_constant__ H3zArgs a) {
  using P = Pack<__half>;
  constexpr int VEC = 8, BX = 128, VPR = BX / VEC;  // = tile_bx<__half>(): the classic tiles
  __shared__ float scratch[32 * kMaxDots];
  if (st_idle(a.red.st)) return;
  int b = blockIdx.x;
  const int tx = b % a.tiles_x;
  b /= a.tiles_x;
  const int ty = b % a.tiles_y;
  const int ch = b / a.tiles_y;
  const int z0 = ch * a.zc, z1 = min(z0 + a.zc, a.g.nz);
  const int ry = threadIdx.x / VPR, cx = threadIdx.x - ry * VPR;
  const int gx = tx * BX + cx * VEC, gy = ty * BY + ry;
  P h0 = P::zero(), h1 = P::zero();
  if (gx < a.g.nx && gy < a.g.ny) {
    const typename P::S as = P::scalar(a.red.st->alpha), ws = P::scalar(a.red.st->omega), mws = P::neg(ws);
    const __half *X = reinterpret_cast<const __half *>(a.x), *Pp = reinterpret_cast<const __half *>(a.p);
    const __half *Sv = reinterpret_cast<const __half *>(a.s), *Tv = reinterpret_cast<const __half *>(a.t);
    const __half *Rh = reinterpret_cast<const __half *>(a.rh);
    __half *XO = reinterpret_cast<__half *>(a.xo), *RO = reinterpret_cast<__half *>(a.ro);
    const long long g0 = (long long)gy * a.g.pitch + gx;
    int k = z0;
    constexpr int U = 4;  // planes per trip: twenty 16-B loads in flight per thread
    for (; k + U - 1 < z1; k += U) {
      P xs[U], ps[U], ss[U], ts[U], rs[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long o = (long long)(k + u) * a.g.plane + g0;
        xs[u] = P::ldg(X + o);
        ps[u] = P::ldg(Pp + o);
        ss[u] = P::ldg(Sv + o);
        ts[u] = P::ldg(Tv + o);
        rs[u] = P::ldg(Rh + o);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {  // z ascending: the pencils' order
        const long long o = (long long)(k + u) * a.g.plane + g0;
        const P xn = P::fmas(ws, ss[u], P::fmas(as, ps[u], xs[u])), rn = P::fmas(mws, ts[u], ss[u]);
        xn.st(XO + o);
        rn.st(RO + o);
        h0 = P::fma(rs[u], rn, h0);  // (rhat, r)
        h1 = P::fma(rn, rn, h1);     // (r, r)
      }
    }
    for (; k < z1; ++k) {
      const long long o0 = (long long)k * a.g.plane + g0;
      const P x0 = P::ldg(X + o0), p0 = P::ldg(Pp + o0), s0 = P::ldg(Sv + o0), t0 = P::ldg(Tv + o0), r0 = P::ldg(Rh + o0);
      const P xn0 = P::fmas(ws, s0, P::fmas(as, p0, x0)), rn0 = P::fmas(mws, t0, s0);
      xn0.st(XO + o0);
      rn0.st(RO + o0);
      h0 = P::fma(r0, rn0, h0);
      h1 = P::fma(rn0, rn0, h1);
    }
  }
  float v[2] = {pencil_sum(h0), pencil_sum(h1)};
  grid_reduce_finalize<2, PH_H3>(v, a.red, scratch);
}

// The same operation and the same pencils through a 1D bulk-copy ring (the k_h3_bulk stream):
// a work item is (segment j of a plane, z chunk c) - SEGV consecutive 16-B vectors of every
// plane of the chunk; thread tid owns vector j*SEGV + tid, i.e. one (x, y) column over the
// chunk, so its two fp16 pencils run z ascending from +0 exactly as in k_h3z_half (the pencil
// values are identical; only the fp32 order in which pencils are added differs).  Persistent
// CTAs; one thread issues the five 6-KB copies of the step NS ahead (crossing items).
// Planes hold whole padded rows: padding is zero and stays zero (x += a 0 + w 0, r = 0 - w 0).
template <int SEGV, int NS>
__global__ void __launch_bounds__(SEGV) k_h3s_half(const __grid_constant__ H3zArgs a) {
  using P = Pack<__half>;
  constexpr int VEC = 8, SE = SEGV * VEC;  // elements per input per step
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ float scratch[32 * kMaxDots];
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
  __half *ring = reinterpret_cast<__half *>(smem + 128);  // [NS][5][SE]
  if (st_idle(a.red.st)) return;
  const long long pv = a.g.plane / VEC;           // vectors per plane
  const int nsp = (int)((pv + SEGV - 1) / SEGV);  // segments per plane
  const int nch = (a.g.nz + a.zc - 1) / a.zc;
  const long long nitems = (long long)nsp * nch;
  const int tid = threadIdx.x;
  const __half *src[5] = {reinterpret_cast<const __half *>(a.x), reinterpret_cast<const __half *>(a.p),
                          reinterpret_cast<const __half *>(a.s), reinterpret_cast<const __half *>(a.t),
                          reinterpret_cast<const __half *>(a.rh)};
  if (tid == 0) {
#pragma unroll
    for (int k = 0; k < NS; ++k) mbar_init(&bar[k], 1);
    fence_mbar_init();
  }
  __syncthreads();
  // producer cursor (thread 0): the item and plane of the next step to issue
  long long pit = blockIdx.x, pstep = 0;
  int pz = 0;
  auto issue_next = [&]() {
    if (pit >= nitems) return;
    const int c = (int)(pit / nsp), j = (int)(pit - (long long)c * nsp);
    const int z0 = c * a.zc, nzc = min(a.zc, a.g.nz - z0);
    const long long v0 = (long long)j * SEGV;
    const uint32_t bytes = (uint32_t)(min((long long)SEGV, pv - v0) * 16);
    const int slot = (int)(pstep % NS);
    const long long o = (long long)(z0 + pz) * a.g.plane + v0 * VEC;
    mbar_expect_tx(&bar[slot], 5u * bytes);
#pragma unroll
    for (int k = 0; k < 5; ++k) bulk_g2s(ring + ((size_t)slot * 5 + k) * SE, src[k] + o, bytes, &bar[slot]);
    ++pstep;
    if (++pz == nzc) {
      pz = 0;
      pit += gridDim.x;
    }
  };
  if (tid == 0)
    for (int k = 0; k < NS; ++k) issue_next();
  const typename P::S as = P::scalar(a.red.st->alpha), ws = P::scalar(a.red.st->omega), mws = P::neg(ws);
  __half *XO = reinterpret_cast<__half *>(a.xo), *RO = reinterpret_cast<__half *>(a.ro);
  float acc0 = 0.0f, acc1 = 0.0f;
  long long step = 0;
  for (long long it = blockIdx.x; it < nitems; it += gridDim.x) {
    const int c = (int)(it / nsp), j = (int)(it - (long long)c * nsp);
    const int z0 = c * a.zc, z1 = min(z0 + a.zc, a.g.nz);
    const long long v0 = (long long)j * SEGV;
    const bool own = v0 + tid < pv;
    P h0 = P::zero(), h1 = P::zero();
    for (int z = z0; z < z1; ++z, ++step) {
      const int slot = (int)(step % NS);
      mbar_wait(&bar[slot], (uint32_t)((step / NS) & 1));
      if (own) {
        const __half *rb = ring + (size_t)slot * 5 * SE + tid * VEC;
        const P xs = P::ld(rb), ps = P::ld(rb + SE), ss = P::ld(rb + 2 * SE), ts = P::ld(rb + 3 * SE),
                rs = P::ld(rb + 4 * SE);
        const P xn = P::fmas(ws, ss, P::fmas(as, ps, xs)), rn = P::fmas(mws, ts, ss);
        const long long o = (long long)z * a.g.plane + (v0 + tid) * VEC;
        __stcs(reinterpret_cast<uint4 *>(XO + o), *reinterpret_cast<const uint4 *>(&xn));
        __stcs(reinterpret_cast<uint4 *>(RO + o), *reinterpret_cast<const uint4 *>(&rn));
        h0 = P::fma(rs, rn, h0);  // (rhat, r)
        h1 = P::fma(rn, rn, h1);  // (r, r)
      }
      __syncthreads();  // the slot is consumed
      if (tid == 0) issue_next();
    }
    acc0 += pencil_sum(h0);
    acc1 += pencil_sum(h1);
  }
  float v[2] = {acc0, acc1};
  grid_reduce_finalize<2, PH_H3>(v, a.red, scratch);
}

#ifndef STEN_H3Z_VARIANT
#define STEN_H3Z_VARIANT 1  // 0: k_h3z_half (tile z-march, direct loads); 1: k_h3s_half (bulk ring)
#endif
#ifndef STEN_H3S_SEGV
#define STEN_H3S_SEGV 384  // k_h3s_half: 16-B vectors per segment (= threads)
#endif
#ifndef STEN_H3S_NS
#define STEN_H3S_NS 3      // k_h3s_half: ring stages (3 x 5 x 6 KB = 90 KB)
#endif
#ifndef STEN_H3S_CPS
#define STEN_H3S_CPS 2     // k_h3s_half: CTAs per SM
#endif

int h3z_half_grid(int sm_count, const H3zArgs &a) {
  const int nch = (a.g.nz + a.zc - 1) / a.zc;
  if (STEN_H3Z_VARIANT != 1) return a.tiles_x * a.tiles_y * nch;
  const long long items = (a.g.plane / 8 + STEN_H3S_SEGV - 1) / STEN_H3S_SEGV * nch;  // (segment, chunk) items
  return (int)std::max(1LL, std::min((long long)sm_count * STEN_H3S_CPS, items));
}

int h3z_half_launch(const H3zArgs &a, int by, cudaStream_t s) {
  if (by != 16) return (int)cudaErrorNotSupported;
#if STEN_H3Z_VARIANT == 1
  constexpr size_t smem = 128 + (size_t)STEN_H3S_NS * 5 * STEN_H3S_SEGV * 16;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_h3s_half<STEN_H3S_SEGV, STEN_H3S_NS>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
    configured = true;
  }
  k_h3s_half<STEN_H3S_SEGV, STEN_H3S_NS><<<h3z_half_grid(device_sm_count(), a), STEN_H3S_SEGV, smem, s>>>(a);
#else
  const int grid = a.tiles_x * a.tiles_y * ((a.g.nz + a.zc - 1) / a.zc);
  k_h3z_half<16><<<grid, (tile_bx<__half>() / 8) * 16, 0, s>>>(a);
#endif
  return (int)cudaGetLastError();
}


template int stencil_launch_fused<float>(const StencilArgs &, int, int, int, cudaStream_t);
template int stencil_launch_fused<__half>(const StencilArgs &, int, int, int, cudaStream_t);
template int stencil_launch<float>(int, const StencilArgs &, int, int, int, cudaStream_t);
template int stencil_launch<__half>(int, const StencilArgs &, int, int, int, cudaStream_t);
template size_t stencil_smem_bytes<float>(int, int, int);
template size_t stencil_smem_bytes<__half>(int, int, int);
template int stencil_threads<float>(int);
template int stencil_threads<__half>(int);

}  // namespace sten
