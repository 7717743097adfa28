// sten2d.cu - the 2D 9-point SpMV (PAPER.md:362-373,
// Sec. "SpMV (2D)").
//
//   u_P = v_P + sum_d c_d[P] v_{P+d},  d over the 8 neighbours in the order
//   (-1,-1) (0,-1) (+1,-1) (-1,0) (+1,0) (-1,+1) (0,+1) (+1,+1)   [(dx, dy)]
//
// with the main diagonal Jacobi-scaled to one ("most problems will
// precondition the main diagonal to unity"), one FMA per term
// in that order (fp32 FFMA / fp16 HFMA2), as oracle/o2d.c mirrors.
//
// The CS-1 maps a rectangular block per core and pushes output-halo products
// to the neighbours.  On B200 the gather form needs no
// output halo: a CTA owns a BX x BY tile (one 16-B vector per thread), its
// input v arrives by TMA as a (BX+2H) x (BY+2) box (one-point halo, zero fill
// outside the mesh), the eight coefficient vectors are streaming 16-B loads
// issued before the TMA wait.  HBM traffic per point: 8 coefficient arrays +
// v + u = 10 arrays (v's halo rows come from L2).
#include "sten_internal.cuh"

namespace sten {

namespace {

template <typename T> struct Sh2;
template <> struct Sh2<float> {
  static __device__ __forceinline__ Pack<float> left(const Pack<float> &c, float l) {
    return Pack<float>{{l, c.v[0], c.v[1], c.v[2]}};
  }
  static __device__ __forceinline__ Pack<float> right(const Pack<float> &c, float r) {
    return Pack<float>{{c.v[1], c.v[2], c.v[3], r}};
  }
  static __device__ __forceinline__ float ld1(const float *p) { return *p; }
};
template <> struct Sh2<__half> {
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

__host__ __device__ constexpr int a128_2d(int b) { return (b + 127) & ~127; }

}  // namespace

template <typename T> struct Tile2 { static constexpr int BX = sizeof(T) == 2 ? 128 : 64; };

// Per-lane selection for the tiled (output-halo) product: a term whose
// neighbour lies outside the point's tile is SKIPPED (R24: "the tile's columns
// of A" only), i.e. the accumulator keeps its value, sign of zero included.
template <typename T> struct Mask9;
template <> struct Mask9<__half> {
  // lanes gx .. gx+7: bit 0 of xm = left neighbour in the tile, bit 1 = right
  static __device__ __forceinline__ void lanes(const unsigned char *xm, long long gx, uint32_t (&mL)[4],
                                               uint32_t (&mR)[4]) {
    const uint2 q = *reinterpret_cast<const uint2 *>(xm + gx);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t w = (i < 2 ? q.x : q.y) >> (16 * (i & 1));
      const uint32_t lo = w & 0xFFu, hi = (w >> 8) & 0xFFu;
      mL[i] = ((lo & 1u) ? 0x0000FFFFu : 0u) | ((hi & 1u) ? 0xFFFF0000u : 0u);
      mR[i] = ((lo & 2u) ? 0x0000FFFFu : 0u) | ((hi & 2u) ? 0xFFFF0000u : 0u);
    }
  }
  static __device__ __forceinline__ Pack<__half> sel(const uint32_t (&m)[4], const Pack<__half> &f,
                                                     const Pack<__half> &u) {
    Pack<__half> o;
#pragma unroll
    for (int i = 0; i < 4; ++i) o.w[i] = (f.w[i] & m[i]) | (u.w[i] & ~m[i]);
    return o;
  }
};
template <> struct Mask9<float> {
  static __device__ __forceinline__ void lanes(const unsigned char *xm, long long gx, uint32_t (&mL)[4],
                                               uint32_t (&mR)[4]) {
    const uint32_t q = *reinterpret_cast<const uint32_t *>(xm + gx);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t b = (q >> (8 * i)) & 0xFFu;
      mL[i] = (b & 1u) ? ~0u : 0u;
      mR[i] = (b & 2u) ? ~0u : 0u;
    }
  }
  static __device__ __forceinline__ Pack<float> sel(const uint32_t (&m)[4], const Pack<float> &f,
                                                    const Pack<float> &u) {
    Pack<float> o;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      o.v[i] = __uint_as_float((__float_as_uint(f.v[i]) & m[i]) | (__float_as_uint(u.v[i]) & ~m[i]));
    return o;
  }
};

// u = c * vn + u on the lanes of mask m (the others keep u)
template <typename T>
__device__ __forceinline__ Pack<T> fma_m(const uint32_t (&m)[4], const Pack<T> &c, const Pack<T> &vn, const Pack<T> &u) {
  return Mask9<T>::sel(m, Pack<T>::fma(c, vn, u), u);
}
__device__ __forceinline__ void and4(uint32_t (&o)[4], const uint32_t (&a)[4], uint32_t b) {
#pragma unroll
  for (int i = 0; i < 4; ++i) o[i] = a[i] & b;
}

// The nine-term FMA chain of one 16-B vector from a box holding the input with
// a one-point halo (row stride HW, own vector at element e).  TILED: terms
// whose neighbour leaves the point's tile are skipped (masks from xm / ym).
template <typename T, int HW, bool TILED>
__device__ __forceinline__ Pack<T> chain9(const T *box, int e, const Pack<T> (&c)[8], const unsigned char *xm,
                                          const unsigned char *ym, long long gx, int gy, bool inside) {
  using P = Pack<T>;
  using SH = Sh2<T>;
  constexpr int VEC = P::VEC;
  const P vm = P::ld(box + e - HW), vc = P::ld(box + e), vp = P::ld(box + e + HW);
  P u = vc;
  if (!TILED) {
    u = P::fma(c[0], SH::left(vm, SH::ld1(box + e - HW - 1)), u);
    u = P::fma(c[1], vm, u);
    u = P::fma(c[2], SH::right(vm, SH::ld1(box + e - HW + VEC)), u);
    u = P::fma(c[3], SH::left(vc, SH::ld1(box + e - 1)), u);
    u = P::fma(c[4], SH::right(vc, SH::ld1(box + e + VEC)), u);
    u = P::fma(c[5], SH::left(vp, SH::ld1(box + e + HW - 1)), u);
    u = P::fma(c[6], vp, u);
    u = P::fma(c[7], SH::right(vp, SH::ld1(box + e + HW + VEC)), u);
  } else {
    uint32_t mL[4] = {0u, 0u, 0u, 0u}, mR[4] = {0u, 0u, 0u, 0u}, m[4];
    uint32_t yb = 0u;
    if (inside) {
      Mask9<T>::lanes(xm, gx, mL, mR);
      yb = ym[gy];
    }
    const uint32_t yD = (yb & 1u) ? ~0u : 0u, yU = (yb & 2u) ? ~0u : 0u;
    const uint32_t mD[4] = {yD, yD, yD, yD}, mU[4] = {yU, yU, yU, yU};
    and4(m, mL, yD);
    u = fma_m<T>(m, c[0], SH::left(vm, SH::ld1(box + e - HW - 1)), u);
    u = fma_m<T>(mD, c[1], vm, u);
    and4(m, mR, yD);
    u = fma_m<T>(m, c[2], SH::right(vm, SH::ld1(box + e - HW + VEC)), u);
    u = fma_m<T>(mL, c[3], SH::left(vc, SH::ld1(box + e - 1)), u);
    u = fma_m<T>(mR, c[4], SH::right(vc, SH::ld1(box + e + VEC)), u);
    and4(m, mL, yU);
    u = fma_m<T>(m, c[5], SH::left(vp, SH::ld1(box + e + HW - 1)), u);
    u = fma_m<T>(mU, c[6], vp, u);
    and4(m, mR, yU);
    u = fma_m<T>(m, c[7], SH::right(vp, SH::ld1(box + e + HW + VEC)), u);
  }
  return u;
}

template <typename T, int BY, bool TILED>
__global__ void __launch_bounds__((Tile2<T>::BX / Pack<T>::VEC) * BY) k_apply9(const __grid_constant__ Apply9Args a) {
  using P = Pack<T>;
  constexpr int VEC = P::VEC, BX = Tile2<T>::BX, H = 16 / (int)sizeof(T), HW = BX + 2 * H, VPR = BX / VEC;
  __shared__ __align__(128) T box[a128_2d(HW * (BY + 2) * (int)sizeof(T)) / (int)sizeof(T)];
  __shared__ __align__(8) uint64_t bar;
  const int tx = blockIdx.x % a.tiles_x, ty = blockIdx.x / a.tiles_x;
  const int x0 = tx * BX, y0 = ty * BY;
  const int tid = threadIdx.x, ry = tid / VPR, cx = tid - (tid / VPR) * VPR;
  const int gx = x0 + cx * VEC, gy = y0 + ry;
  const bool inside = gx < a.nx && gy < a.ny;
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    mbar_expect_tx(&bar, (uint32_t)(HW * (BY + 2) * sizeof(T)));
    tma_load_3d(box, &a.tm_v, x0 - H, y0 - 1, 0, &bar);
  }
  // the eight coefficient vectors, in flight while the box arrives
  P c[8];
  const long long o = (long long)gy * a.pitch + gx;
#pragma unroll
  for (int d = 0; d < 8; ++d) c[d] = inside ? P::ldg(reinterpret_cast<const T *>(a.c[d]) + o) : P::zero();
  mbar_wait(&bar, 0);
  const int e = (ry + 1) * HW + H + cx * VEC;  // own vector in the box
  const P u = chain9<T, HW, TILED>(box, e, c, a.xm, a.ym, gx, gy, inside);
  if (inside) u.st(reinterpret_cast<T *>(a.u) + o);
}

// ----------------------------------------------- tiled SpMV: output halo --
// R24 (oracle/o2d.c apply9_tiles): tile (ta, tb) owns [X_ta, X_ta+1) x
// [Y_tb, Y_tb+1), X_a = floor(a nx / TX).  Its output-halo ring - the points
// one step outside the tile that its columns of A reach - is computed here:
// w = +0, then one FMA per neighbour d = 0..7 (in order) that lies IN the
// tile.  Ring storage, tile k = ta + TX tb: L[k][HS], R[k][HS] (columns x0-1 and
// x1 over the grown rows gy0 .. gy1-1), B[k][WS], T[k][WS] (rows y0-1 and y1
// over the own columns).
__device__ __forceinline__ int tbound(int a, int n, int t) { return (int)((long long)a * n / t); }

template <typename T> struct S9;
template <> struct S9<float> {
  static __device__ __forceinline__ float fma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float zero() { return 0.0f; }
};
template <> struct S9<__half> {
  static __device__ __forceinline__ __half fma(__half a, __half b, __half c) { return __hfma(a, b, c); }
  static __device__ __forceinline__ __half add(__half a, __half b) { return __hadd(a, b); }
  static __device__ __forceinline__ __half zero() { return __ushort_as_half((unsigned short)0); }
};

struct TileBox {
  int ta, tb, x0, x1, y0, y1, gy0, gy1;
};
__device__ __forceinline__ TileBox tile_box(const Ring9Args &a, int k) {
  TileBox t;
  t.ta = k % a.TX;
  t.tb = k / a.TX;
  t.x0 = tbound(t.ta, a.nx, a.TX);
  t.x1 = tbound(t.ta + 1, a.nx, a.TX);
  t.y0 = tbound(t.tb, a.ny, a.TY);
  t.y1 = tbound(t.tb + 1, a.ny, a.TY);
  t.gy0 = t.y0 > 0 ? t.y0 - 1 : 0;
  t.gy1 = t.y1 < a.ny ? t.y1 + 1 : a.ny;
  return t;
}

template <typename T>
__global__ void k_ring9(const Ring9Args a) {
  const int DX[8] = {-1, 0, 1, -1, 1, -1, 0, 1}, DY[8] = {-1, -1, -1, 0, 0, 1, 1, 1};
  const int NT = a.TX * a.TY, E = 2 * a.HS + 2 * a.WS;
  const T *v = reinterpret_cast<const T *>(a.v);
  T *ring = reinterpret_cast<T *>(a.ring);
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < (long long)NT * E;
       q += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(q / E), e = (int)(q % E);
    const TileBox t = tile_box(a, k);
    int px, py;
    bool ok;
    long long slot;
    if (e < a.HS) {  // L: column x0-1
      px = t.x0 - 1;
      py = t.gy0 + e;
      ok = t.ta > 0 && py < t.gy1;
      slot = (long long)k * a.HS + e;
    } else if (e < 2 * a.HS) {  // R: column x1
      px = t.x1;
      py = t.gy0 + e - a.HS;
      ok = t.ta < a.TX - 1 && py < t.gy1;
      slot = (long long)NT * a.HS + (long long)k * a.HS + (e - a.HS);
    } else if (e < 2 * a.HS + a.WS) {  // B: row y0-1
      px = t.x0 + e - 2 * a.HS;
      py = t.y0 - 1;
      ok = t.tb > 0 && px < t.x1;
      slot = 2LL * NT * a.HS + (long long)k * a.WS + (e - 2 * a.HS);
    } else {  // T: row y1
      px = t.x0 + e - 2 * a.HS - a.WS;
      py = t.y1;
      ok = t.tb < a.TY - 1 && px < t.x1;
      slot = 2LL * NT * a.HS + (long long)NT * a.WS + (long long)k * a.WS + (e - 2 * a.HS - a.WS);
    }
    if (!ok) continue;
    const long long P = (long long)py * a.pitch + px;
    T w = S9<T>::zero();
#pragma unroll
    for (int d = 0; d < 8; ++d) {
      const int qx = px + DX[d], qy = py + DY[d];
      if (qx >= t.x0 && qx < t.x1 && qy >= t.y0 && qy < t.y1)
        w = S9<T>::fma(reinterpret_cast<const T *>(a.c[d])[P], v[(long long)qy * a.pitch + qx], w);
    }
    ring[slot] = w;
  }
}

// The two rounds of PAPER.md:367-368 ("a round of send and add in one
// direction, then a round for the other direction").  dir 0 (x round): a
// tile's columns x0 and x1-1, over its grown rows (halo rows B / T included:
// the diagonal products ride along), += the left neighbour's R column, then
// the right neighbour's L column.  dir 1 (y round): its rows y0 and y1-1 (own
// columns) += the lower neighbour's T row, then the upper neighbour's B row.
// One thread per (tile, row / column): the two adds of a width-1 / height-1
// tile hit the same point in the oracle's order.
template <typename T>
__global__ void k_round9(const Ring9Args a, int dir) {
  const int NT = a.TX * a.TY, E = dir == 0 ? a.HS : a.WS;
  T *u = reinterpret_cast<T *>(a.u);
  T *ring = reinterpret_cast<T *>(a.ring);
  const long long oL = 0, oR = (long long)NT * a.HS, oB = 2LL * NT * a.HS, oT = oB + (long long)NT * a.WS;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < (long long)NT * E;
       q += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(q / E), e = (int)(q % E);
    const TileBox t = tile_box(a, k);
    if (dir == 0) {
      const int j = t.gy0 + e;
      if (j >= t.gy1) continue;
      auto at = [&](int x) -> T * {  // the tile's value at (x, j), x in its own columns
        if (j >= t.y0 && j < t.y1) return u + (long long)j * a.pitch + x;
        return ring + (j < t.y0 ? oB : oT) + (long long)k * a.WS + (x - t.x0);
      };
      if (t.ta > 0) {
        T *p = at(t.x0);
        *p = S9<T>::add(*p, ring[oR + (long long)(k - 1) * a.HS + e]);
      }
      if (t.ta < a.TX - 1) {
        T *p = at(t.x1 - 1);
        *p = S9<T>::add(*p, ring[oL + (long long)(k + 1) * a.HS + e]);
      }
    } else {
      const int i = t.x0 + e;
      if (i >= t.x1) continue;
      if (t.tb > 0) {
        T *p = u + (long long)t.y0 * a.pitch + i;
        *p = S9<T>::add(*p, ring[oT + (long long)(k - a.TX) * a.WS + e]);
      }
      if (t.tb < a.TY - 1) {
        T *p = u + (long long)(t.y1 - 1) * a.pitch + i;
        *p = S9<T>::add(*p, ring[oB + (long long)(k + a.TX) * a.WS + e]);
      }
    }
  }
}

// ------------------------------------------- BiCGStab on the 2D operator --
// PAPER.md:373 ("all terms needed for BiCG"), R25: Alg. 1 with the 9-point
// operator.  The two SpMV phases, fused like the 3D ones:
//   H1: p' = r + beta (p - omega v) (l.184) on the whole box, v' = A p'
//       (l.176), (rhat, v')  -> alpha (l.177)
//   H2: s = r - alpha v' (l.178) on the whole box, t = A s (l.179),
//       (t, s), (t, t)       -> omega (l.180)
// A persistent CTA (2 per SM) walks the BX x BY tiles b, b + G, b + 2G, ... (G = grid size; the G
// tiles in flight are consecutive in row-major order, so y-neighbours run together and share halo
// rows in L2).  Per tile the NIN inputs arrive by TMA as (BX+2H) x (BY+2) boxes (zero fill outside
// the mesh) into a 2-stage ring - the next tile's boxes are in flight while this one is computed -
// the SpMV input is formed once per box element into one of two shared boxes (ping-pong: one
// barrier per tile), the eight couplings (and rhat) of the next tile are streaming 16-B loads
// issued as soon as this tile's FMA chain has consumed its own.  The inner products accumulate
// over all of a CTA's tiles: one deposit per CTA.  H3 and S1 are the 3D element-wise kernels
// (k_h3_bulk, k_init) over the pitched plane.
#ifndef STEN_BICG9_MINB
#define STEN_BICG9_MINB 1  // CTAs per SM (measured: 1 per SM 5.44 ms per mixed iteration at 22800^2, 2 per SM 5.79)
#endif
#ifndef STEN_BICG9_NS
#define STEN_BICG9_NS 2  // input stages
#endif
template <typename T, int MODE, int BY>
__global__ void __launch_bounds__((Tile2<T>::BX / Pack<T>::VEC) * BY, STEN_BICG9_MINB) k_bicg9(const __grid_constant__ Bicg9Args a) {
  using P = Pack<T>;
  constexpr int VEC = P::VEC, BX = Tile2<T>::BX, H = 16 / (int)sizeof(T), HW = BX + 2 * H, VPR = BX / VEC;
  constexpr int NT = VPR * BY, NIN = MODE == MODE_H1 ? 3 : 2, ND = MODE == MODE_H1 ? 1 : 2;
  constexpr int HSTR = a128_2d(HW * (BY + 2) * (int)sizeof(T)) / (int)sizeof(T);
  constexpr int NVB = (HW / VEC) * (BY + 2);  // 16-B vectors per box
  if (st_idle(a.red.st)) return;
  extern __shared__ __align__(128) unsigned char smem2[];
  constexpr int NS = STEN_BICG9_NS;
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem2);  // [NS]
  T *stage = reinterpret_cast<T *>(smem2 + 128);        // [NS][NIN][HSTR]
  T *Ub = stage + NS * NIN * HSTR;                      // [2][HSTR]
  __shared__ float scratch[32 * kMaxDots];
  const int ntiles = a.tiles_x * a.tiles_y;
  const int tid = threadIdx.x, ry = tid / VPR, cx = tid - (tid / VPR) * VPR;
  if (tid == 0) {
#pragma unroll
    for (int q = 0; q < NS; ++q) mbar_init(&bar[q], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](int tile, int slot) {  // one thread
    const int x0 = (tile % a.tiles_x) * BX, y0 = (tile / a.tiles_x) * BY;
    mbar_expect_tx(&bar[slot], (uint32_t)(NIN * HW * (BY + 2) * sizeof(T)));
#pragma unroll
    for (int i = 0; i < NIN; ++i) tma_load_3d(stage + (slot * NIN + i) * HSTR, &a.tm_in[i], x0 - H, y0 - 1, 0, &bar[slot]);
  };
  const int t0 = blockIdx.x, G = gridDim.x;
  if (tid == 0)
    for (int q = 0; q < NS; ++q)
      if (t0 + q * G < ntiles) issue(t0 + q * G, q);
  typename P::S s1{}, s2{};
  if (MODE == MODE_H1) {
    s1 = P::scalar(a.red.st->beta);
    s2 = P::neg(P::scalar(a.red.st->omega));
  } else {
    s1 = P::neg(P::scalar(a.red.st->alpha));
  }
  P c[8], rh = P::zero();
  auto load_own = [&](int tile, long long &o, bool &inside, int &gx, int &gy) {
    gx = (tile % a.tiles_x) * BX + cx * VEC;
    gy = (tile / a.tiles_x) * BY + ry;
    inside = tile < ntiles && gx < a.nx && gy < a.ny;
    o = (long long)gy * a.pitch + gx;
#pragma unroll
    for (int d = 0; d < 8; ++d) c[d] = inside ? P::ldg(reinterpret_cast<const T *>(a.c[d]) + o) : P::zero();
    if (MODE == MODE_H1) rh = inside ? P::ldg(reinterpret_cast<const T *>(a.rh) + o) : P::zero();
  };
  long long o;
  bool inside;
  int gx, gy;
  load_own(t0, o, inside, gx, gy);
  float dacc[ND][4];
#pragma unroll
  for (int d = 0; d < ND; ++d)
#pragma unroll
    for (int i = 0; i < 4; ++i) dacc[d][i] = 0.0f;
  const int e = (ry + 1) * HW + H + cx * VEC;
  int k = 0;
  for (int tile = t0; tile < ntiles; tile += G, ++k) {
    const int slot = k % NS;
    mbar_wait(&bar[slot], (uint32_t)((k / NS) & 1));
    const T *box = stage + slot * NIN * HSTR;
    T *U = Ub + (k & 1) * HSTR;
    for (int q = tid; q < NVB; q += NT) {  // the SpMV input on the whole box
      const int h = q * VEC;
      P f = P::ld(box + h);  // r
      if (MODE == MODE_H1) f = P::fmas(s1, P::fmas(s2, P::ld(box + 2 * HSTR + h), P::ld(box + HSTR + h)), f);
      else f = P::fmas(s1, P::ld(box + HSTR + h), f);
      f.st(U + h);
    }
    __syncthreads();  // U complete, the stage consumed (and every thread is past the previous tile)
    if (tid == 0 && tile + NS * G < ntiles) issue(tile + NS * G, slot);
    const P w = P::ld(U + e);  // p' (H1) / s (H2) at the own points
    const P u = chain9<T, HW, false>(U, e, c, nullptr, nullptr, gx, gy, inside);
    const P rh_ = rh;
    const long long o_ = o;
    const bool in_ = inside;
    load_own(tile + G, o, inside, gx, gy);  // the next tile's couplings in flight
    if (in_) {
      u.st(reinterpret_cast<T *>(a.out0) + o_);
      w.st(reinterpret_cast<T *>(a.out1) + o_);
      if (MODE == MODE_H1) {
        rh_.dot4(u, dacc[0]);  // (rhat, v')
      } else {
        u.dot4(w, dacc[0]);       // (t, s)
        u.dot4(u, dacc[ND - 1]);  // (t, t)
      }
    }
  }
  float v[ND];
#pragma unroll
  for (int d = 0; d < ND; ++d) v[d] = sum4(dacc[d]);
  if (MODE == MODE_H1) grid_reduce_finalize<ND, PH_H1>(v, a.red, scratch);
  else grid_reduce_finalize<ND, PH_H2>(v, a.red, scratch);
}

// ------------------------------- BiCGStab on the tiled SpMV (R24, R25) --
// With the paper's tiled output-halo SpMV the phases cannot fuse the update into the product (the
// rounds complete a tile's edge values after its kernel), so a tiled solve runs them unfused over
// the pitched plane (linear 16-B vectors; padding holds zeros): H1 = k_upd9<P> (p' = r + beta (p -
// omega v), l.184), the tiled apply of p', k_dot9 (rhat, v'); H2 = k_upd9<S> (s = r - alpha v',
// l.178), the tiled apply of s, k_dot9 (t, s), (t, t); H3 = k_h3_bulk.  Same roundings as the
// fused kernels (oracle/o2d.c o2d16_bicgstab_tiles).
template <typename T, int MODE>
__global__ void __launch_bounds__(256) k_upd9(const __grid_constant__ Upd9Args a) {
  using P = Pack<T>;
  constexpr int VEC = P::VEC;
  if (st_idle(a.st)) return;
  typename P::S s1{}, s2{};
  if (MODE == MODE_H1) {
    s1 = P::scalar(a.st->beta);
    s2 = P::neg(P::scalar(a.st->omega));
  } else {
    s1 = P::neg(P::scalar(a.st->alpha));
  }
  const T *R = reinterpret_cast<const T *>(a.r), *V = reinterpret_cast<const T *>(a.v);
  const T *Pp = reinterpret_cast<const T *>(a.p);
  T *O = reinterpret_cast<T *>(a.out);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < a.nvec; i += (long long)gridDim.x * blockDim.x) {
    const long long o = i * VEC;
    P f = P::ldg(R + o);
    if (MODE == MODE_H1) f = P::fmas(s1, P::fmas(s2, P::ldg(V + o), P::ldg(Pp + o)), f);
    else f = P::fmas(s1, P::ldg(V + o), f);
    f.st(O + o);
  }
}

template <typename T, int ND, int PH>
__global__ void __launch_bounds__(256) k_dot9(const __grid_constant__ Dot9Args a) {
  using P = Pack<T>;
  constexpr int VEC = P::VEC;
  __shared__ float scratch[32 * kMaxDots];
  if (st_idle(a.red.st)) return;
  const T *A0 = reinterpret_cast<const T *>(a.a0), *B0 = reinterpret_cast<const T *>(a.b0);
  float d0[4] = {0.f, 0.f, 0.f, 0.f}, d1[4] = {0.f, 0.f, 0.f, 0.f};
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < a.nvec; i += (long long)gridDim.x * blockDim.x) {
    const long long o = i * VEC;
    const P x = P::ldg(A0 + o), y = P::ldg(B0 + o);
    x.dot4(y, d0);              // H1: (rhat, v')   H2: (t, s)
    if (ND == 2) x.dot4(x, d1);  // H2: (t, t)
  }
  float v[ND];
  v[0] = sum4(d0);
  if (ND == 2) v[ND - 1] = sum4(d1);
  grid_reduce_finalize<ND, PH>(v, a.red, scratch);
}

template <typename T>
int upd9_launch(int mode, const Upd9Args &a, int grid, cudaStream_t s) {
  if (mode == MODE_H1) k_upd9<T, MODE_H1><<<grid, 256, 0, s>>>(a);
  else k_upd9<T, MODE_H2><<<grid, 256, 0, s>>>(a);
  return (int)cudaGetLastError();
}
template <typename T>
int dot9_launch(int mode, const Dot9Args &a, int grid, cudaStream_t s) {
  if (mode == MODE_H1) k_dot9<T, 1, PH_H1><<<grid, 256, 0, s>>>(a);
  else k_dot9<T, 2, PH_H2><<<grid, 256, 0, s>>>(a);
  return (int)cudaGetLastError();
}
template int upd9_launch<float>(int, const Upd9Args &, int, cudaStream_t);
template int upd9_launch<__half>(int, const Upd9Args &, int, cudaStream_t);
template int dot9_launch<float>(int, const Dot9Args &, int, cudaStream_t);
template int dot9_launch<__half>(int, const Dot9Args &, int, cudaStream_t);

// Jacobi scaling of the 9-point operator (R3/R5 in 2D): c_d = A_d / A_P in
// fp64, couplings leaving the mesh dropped, rounded RN to fp32 and fp16;
// padding columns hold zero couplings
template <typename TIN>
__global__ void k_create9(const TIN *diag, Coef9In in, int nx, int ny, int pitch, Coef9Out out, double *aP) {
  const int DX[8] = {-1, 0, 1, -1, 1, -1, 0, 1}, DY[8] = {-1, -1, -1, 0, 0, 1, 1, 1};
  const long long total = (long long)pitch * ny;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(q % pitch), y = (int)(q / pitch);
    for (int d = 0; d < 8; ++d) {
      double cv = 0.0;
      if (x < nx) {
        const long long P = x + (long long)nx * y;
        const int xx = x + DX[d], yy = y + DY[d];
        if (xx >= 0 && xx < nx && yy >= 0 && yy < ny) {
          const double od = (double)reinterpret_cast<const TIN *>(in.off[d])[P];
          cv = diag ? __ddiv_rn(od, (double)diag[P]) : od;
        }
      }
      out.c32[d][q] = __double2float_rn(cv);
      out.c16[d][q] = __double2half(cv);
    }
    if (aP) aP[q] = (x < nx && diag) ? (double)diag[x + (long long)nx * y] : 1.0;  // R3: b_hat = b / a_P
  }
}

template <typename T>
int apply9_launch(const Apply9Args &a, cudaStream_t s) {
  constexpr int BY = 32;  // = kApply9BY of the host's tensor maps
  const int ty = (a.ny + BY - 1) / BY;
  if (a.xm) k_apply9<T, BY, true><<<a.tiles_x * ty, (Tile2<T>::BX / Pack<T>::VEC) * BY, 0, s>>>(a);
  else k_apply9<T, BY, false><<<a.tiles_x * ty, (Tile2<T>::BX / Pack<T>::VEC) * BY, 0, s>>>(a);
  return (int)cudaGetLastError();
}
template int apply9_launch<float>(const Apply9Args &, cudaStream_t);
template int apply9_launch<__half>(const Apply9Args &, cudaStream_t);

static int small_grid(long long work) {
  long long g = (work + 255) / 256;
  if (g > 148 * 8) g = 148 * 8;
  return (int)(g < 1 ? 1 : g);
}
template <typename T>
int ring9_launch(const Ring9Args &a, cudaStream_t s) {
  const long long work = (long long)a.TX * a.TY * (2 * a.HS + 2 * a.WS);
  k_ring9<T><<<small_grid(work), 256, 0, s>>>(a);
  return (int)cudaGetLastError();
}
template <typename T>
int round9_launch(const Ring9Args &a, int dir, cudaStream_t s) {
  const long long work = (long long)a.TX * a.TY * (dir == 0 ? a.HS : a.WS);
  k_round9<T><<<small_grid(work), 256, 0, s>>>(a, dir);
  return (int)cudaGetLastError();
}
template int ring9_launch<float>(const Ring9Args &, cudaStream_t);
template int ring9_launch<__half>(const Ring9Args &, cudaStream_t);
template int round9_launch<float>(const Ring9Args &, int, cudaStream_t);
template int round9_launch<__half>(const Ring9Args &, int, cudaStream_t);

template <typename T, int MODE, int BY>
static int bicg9_one(const Bicg9Args &a, cudaStream_t s) {
  constexpr int NIN = MODE == MODE_H1 ? 3 : 2, H = 16 / (int)sizeof(T), HW = Tile2<T>::BX + 2 * H;
  constexpr size_t smem = 128 + (size_t)(STEN_BICG9_NS * NIN + 2) * (a128_2d(HW * (BY + 2) * (int)sizeof(T)));
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_bicg9<T, MODE, BY>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
    configured = true;
  }
  const int tiles = a.tiles_x * a.tiles_y, nt = (Tile2<T>::BX / Pack<T>::VEC) * BY;
  int grid = device_sm_count() * STEN_BICG9_MINB;
  if (grid > tiles) grid = tiles;
  k_bicg9<T, MODE, BY><<<grid, nt, smem, s>>>(a);
  return (int)cudaGetLastError();
}
template <typename T>
int bicg9_launch(int mode, const Bicg9Args &a, cudaStream_t s) {
  constexpr int BY = kBicg9BY;
  if (mode == MODE_H1) return bicg9_one<T, MODE_H1, BY>(a, s);
  return bicg9_one<T, MODE_H2, BY>(a, s);
}
template int bicg9_launch<float>(int, const Bicg9Args &, cudaStream_t);
template int bicg9_launch<__half>(int, const Bicg9Args &, cudaStream_t);

int create9_launch(int in_dtype, const void *diag, const Coef9In &in, int nx, int ny, int pitch, const Coef9Out &out,
                   double *aP, cudaStream_t s) {
  const long long total = (long long)pitch * ny;
  int grid = (int)((total + 255) / 256);
  if (grid > 148 * 32) grid = 148 * 32;
  if (grid < 1) grid = 1;
  if (in_dtype == STEN_DT_F64) k_create9<double><<<grid, 256, 0, s>>>((const double *)diag, in, nx, ny, pitch, out, aP);
  else k_create9<float><<<grid, 256, 0, s>>>((const float *)diag, in, nx, ny, pitch, out, aP);
  return (int)cudaGetLastError();
}

}  // namespace sten
