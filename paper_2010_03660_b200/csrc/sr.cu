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
#include "sten_internal.cuh"

namespace sten {

namespace {

constexpr int a128(int b) { return (b + 127) & ~127; }

#ifndef STEN_SR_MMA
#define STEN_SR_MMA 1  // 0: fp16 dots on the FMA pipe (fma.rn.f32.f16), for comparison
#endif

// Gram of (rh, r', v', q', y') over one tile row of BX points on the tensor
// cores.  ldmatrix.x2 at `row` + 16 i gives rows = vectors (lanes 0-7: points
// 16i..16i+7, lanes 8-15: 16i+8..16i+15): at once the A fragment (rows 0-7;
// rows 8-15 zero) and the B fragment of mma.m16n8k16 (fp16 x fp16 products,
// fp32 sums).  D[a][b] = sum_k U[a][k] U[b][k] lands in lane
// 4a + b/2.  Every mma starts from C = 0 and its D is added to the running
// sums with round-to-nearest fp32 adds: the tensor core's internal 16-term sum
// truncates, so the accumulator is never carried through it (R20).
template <int NB>
__device__ __forceinline__ void gram_row(uint32_t row_addr, float (&acc)[2]) {
  uint32_t m0[NB], m1[NB];
#pragma unroll
  for (int i = 0; i < NB; ++i)
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0, %1}, [%2];"
                 : "=r"(m0[i]), "=r"(m1[i])
                 : "r"(row_addr + 32u * i));
  float d0[NB], d1[NB];
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    float d2, d3;
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
        "{%10, %10, %10, %10};"
        : "=f"(d0[i]), "=f"(d1[i]), "=f"(d2), "=f"(d3)
        : "r"(m0[i]), "r"(0u), "r"(m1[i]), "r"(0u), "r"(m0[i]), "r"(m1[i]), "f"(0.0f));
  }
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    acc[0] = __fadd_rn(acc[0], d0[i]);
    acc[1] = __fadd_rn(acc[1], d1[i]);
  }
}

template <typename T, int BY>
struct SrGeo {
  static constexpr int VEC = Pack<T>::VEC;
  static constexpr int BX = tile_bx<T>();
  static constexpr int H = VEC;                  // x halo pad: one vector (keeps 16-B alignment)
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
  static_assert(NHF <= NT && NHV <= NT, "halo work must fit one extra item per thread");
  // tensor-core Gram (fp16): rh, v', q', y' of one plane staged as 4 dense
  // BY x BX arrays (16-B staggered to spread ldmatrix rows over banks) + one
  // zero row; r' is read from its ring
  static constexpr bool MMA = sizeof(T) == 2 && STEN_SR_MMA;
  static constexpr int GSV = BX * BY + 8;        // elements between staged vectors
  static constexpr int GSE = MMA ? 4 * GSV + BX + 8 : 0;  // staging elements (+ a zero row of BX+8)
};

template <typename T, int BY, int S, int SC>
constexpr size_t sr_smem_c() {
  using G = SrGeo<T, BY>;
  return 128 + (size_t)sizeof(T) * ((size_t)S * 5 * G::IE + (size_t)SC * 6 * G::CE + 7 * (size_t)G::IE +
                                    2 * (size_t)G::CE + (size_t)G::GSE);
}

template <typename T> struct SrShift;
template <> struct SrShift<float> {
  using E = float;
  static __device__ __forceinline__ Pack<float> left(const Pack<float> &c, float l) {
    return Pack<float>{{l, c.v[0], c.v[1], c.v[2]}};
  }
  static __device__ __forceinline__ Pack<float> right(const Pack<float> &c, float r) {
    return Pack<float>{{c.v[1], c.v[2], c.v[3], r}};
  }
  static __device__ __forceinline__ float ld1(const float *p) { return *p; }
};
template <> struct SrShift<__half> {
  using E = uint32_t;
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

// u = c0 l + ... in the fixed order: u = m; fma xm, xp, ym, yp, zm, zp (R10)
template <typename T>
__device__ __forceinline__ Pack<T> spmv(const Pack<T> (&c)[6], const Pack<T> &m, const Pack<T> &xl,
                                        const Pack<T> &xr, const Pack<T> &ym, const Pack<T> &yp,
                                        const Pack<T> &zm, const Pack<T> &zp) {
  using P = Pack<T>;
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

template <typename T, int BY, int S, int SC>
__global__ void __launch_bounds__(SrGeo<T, BY>::NT, 1) k_sr(const __grid_constant__ SrArgs a) {
  using P = Pack<T>;
  using G = SrGeo<T, BY>;
  using SH = SrShift<T>;
  constexpr int VEC = G::VEC, H = G::H, HW = G::HW, VW = G::VW, VPR = G::VPR, IE = G::IE, CE = G::CE;

  if (sr_idle(a.red.st)) return;

  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t *mbar = reinterpret_cast<uint64_t *>(smem);           // [S] inputs, [SC] coefficients
  T *const IN = reinterpret_cast<T *>(smem + 128);               // [S][5][IE]
  T *const CF = IN + S * 5 * IE;                                 // [SC][6][CE]
  T *const PR = CF + SC * 6 * CE;                                // p' ring [3][IE]
  T *const RR = PR + 3 * IE;                                     // r' ring [4][IE]
  T *const VR = RR + 4 * IE;                                     // v' ring [2][CE]
  T *const GS = VR + 2 * CE;                                     // Gram staging (MMA): [4][GSV] + zero row
  __shared__ float scratch[32 * kMaxDots];

  int b = blockIdx.x;
  const int tx = b % a.tiles_x;
  b /= a.tiles_x;
  const int ty = b % a.tiles_y;
  const int ch = b / a.tiles_y;
  const int x0 = tx * G::BX, y0 = ty * BY;
  const int z0 = ch * a.zc, z1 = min(z0 + a.zc, a.g.nz);
  const int npi = z1 - z0 + 4;  // staged input planes z0-2 .. z1+1
  const int npc = z1 - z0 + 2;  // staged coefficient planes z0-1 .. z1
  const int tid = threadIdx.x;

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
    hf = r * HW + c * VEC;
  }
  // one halo item of the v' region (coef-box rows 0..RC-1, cols 0..VW-1 minus the own tile)
  int hv = -1, hvc = 0;
  if (tid < G::NHV) {
    int r, c;
    if (tid < VW) { r = 0; c = tid; }
    else if (tid < 2 * VW) { r = G::RC - 1; c = tid - VW; }
    else { const int m = tid - 2 * VW; r = 1 + m / 2; c = (m & 1) ? VW - 1 : 0; }
    hv = r * HW + c * VEC;
    hvc = c;
  }
  const int gx = x0 + cx * VEC, gy = y0 + ry;
  const bool inside = gy < a.g.ny && gx < a.g.nx;
  const long long gofs = (long long)gy * a.g.pitch + gx;
  const long long plane = a.g.plane;

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < S + SC; ++s) mbar_init(&mbar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  auto issue_in = [&](int qi) {  // plane z0-2+qi of r, p, v, q, y (vectors: 2 halo planes)
    const int slot = qi % S, m = z0 - 2 + qi;
    mbar_expect_tx(&mbar[slot], 5u * HW * G::RI * (uint32_t)sizeof(T));
#pragma unroll
    for (int i = 0; i < 5; ++i) tma_load_3d(IN + (slot * 5 + i) * IE, &a.tm_in[i], x0 - H, y0 - 2, m + 2, &mbar[slot]);
  };
  auto issue_c = [&](int qc) {  // plane z0-1+qc of the six coefficient arrays (1 halo plane)
    const int slot = qc % SC, m = z0 - 1 + qc;
    mbar_expect_tx(&mbar[S + slot], 6u * HW * G::RC * (uint32_t)sizeof(T));
#pragma unroll
    for (int d = 0; d < 6; ++d) tma_load_3d(CF + (slot * 6 + d) * CE, &a.tm_c[d], x0 - H, y0 - 1, m + 1, &mbar[S + slot]);
  };
  if (tid == 0) {
    for (int q = 0; q < min(S, npi); ++q) issue_in(q);
    for (int q = 0; q < min(SC, npc); ++q) issue_c(q);
  }

  typename P::S al_s = P::scalar(a.red.st->alpha), mal_s = P::neg(al_s);
  typename P::S om_s = P::scalar(a.red.st->omega), mom_s = P::neg(om_s);
  typename P::S be_s = P::scalar(a.red.st->beta);

  T *const Xg = reinterpret_cast<T *>(a.x);
  const T *const RHg = reinterpret_cast<const T *>(a.rh);
  T *const Og[5] = {reinterpret_cast<T *>(a.out[0]), reinterpret_cast<T *>(a.out[1]), reinterpret_cast<T *>(a.out[2]),
                    reinterpret_cast<T *>(a.out[3]), reinterpret_cast<T *>(a.out[4])};

  // own x of the plane formed at the next step, r_hat of the plane of the next dots
  P xn = P::zero(), rhn = P::zero();
  auto load_x = [&](int m) {
    if (inside && m >= z0 && m < z1) xn = P::ldg(Xg + (long long)m * plane + gofs);
  };
  auto load_rh = [&](int k) {
    if (inside && k < z1) rhn = P::ldg(RHg + (long long)k * plane + gofs);
  };
  load_x(z0 - 2);
  load_rh(z0);

  P pw0 = P::zero(), pw1 = P::zero(), pw2 = P::zero();                   // own p' at k, k+1, k+2
  P rw0 = P::zero(), rw1 = P::zero(), rw2 = P::zero(), rw3 = P::zero();  // own r' at k-1 .. k+2
  P vw0 = P::zero(), vw1 = P::zero(), vw2 = P::zero();                   // own v' at k-1, k, k+1
  P cc[6], cn[6];                                                        // own coefficients at k, k+1
#pragma unroll
  for (int d = 0; d < 6; ++d) cc[d] = cn[d] = P::zero();
  float dacc[12];
#pragma unroll
  for (int d = 0; d < 12; ++d) dacc[d] = 0.0f;
  float gacc[2] = {0.f, 0.f};  // MMA path: this lane's part (row g, cols 2c, 2c+1) of the warp's Gram
  if (G::MMA) {
    for (int e = tid; e < G::BX + 8; e += blockDim.x) GS[4 * G::GSV + e] = T(0.0f);
  }
  // MMA path: warp w reduces rows 2w, 2w+1 of the staged plane (16 points per
  // mma), r' of that plane from ring slot `rslot`.  Lane l (< 16) points at
  // row l%8 (rh r' v' q' y' 0 0 0) of the 8 points starting at 8*(l/8).
  auto gram_plane = [&](int rslot) {
    const int lane = tid & 31, w = tid >> 5, vrow = lane & 7, half = (lane >> 3) & 1;
#pragma unroll
    for (int rr2 = 0; rr2 < 2; ++rr2) {
      const int row = 2 * w + rr2;
      const T *addr;
      if (vrow == 1) addr = RR + rslot * IE + (row + 2) * HW + H + 8 * half;
      else if (vrow == 0) addr = GS + row * G::BX + 8 * half;
      else if (vrow < 5) addr = GS + (vrow - 1) * G::GSV + row * G::BX + 8 * half;
      else addr = GS + 4 * G::GSV;
      gram_row<G::BX / 16>(smem_u32(addr), gacc);  // rows 5-7 walk the zero row
    }
  };
  for (int j = 0; j < npi; ++j) {
    const int k = z0 - 4 + j;  // step k: form plane k+2, v' of plane k+1, q'/y'/dots of plane k
    // ---------------- (A) form p', r' of plane k+2; update own x, r, p ----------------
    mbar_wait(&mbar[j % S], (uint32_t)((j / S) & 1));
    {
      const T *st = IN + (j % S) * 5 * IE;
      T *pr = PR + (j % 3) * IE;
      T *rr = RR + (j & 3) * IE;
      const int m = k + 2;
      {
        const P r = P::ld(st + ei), p = P::ld(st + IE + ei), v = P::ld(st + 2 * IE + ei);
        const P q = P::ld(st + 3 * IE + ei), y = P::ld(st + 4 * IE + ei);
        const P s = P::fmas(mal_s, v, r);
        const P t = P::fmas(mal_s, y, q);
        const P rn = P::fmas(mom_s, t, s);
        const P pn = P::fmas(be_s, P::fmas(mom_s, v, p), rn);
        rn.st(rr + ei);
        pn.st(pr + ei);
        pw2 = pn;
        rw3 = rn;
        if (inside && m >= z0 && m < z1) {
          const long long o = (long long)m * plane + gofs;
          P::fmas(om_s, s, P::fmas(al_s, p, xn)).st(Xg + o);
          rn.st(Og[0] + o);
          pn.st(Og[1] + o);
        }
      }
      if (hf >= 0) {
        const P r = P::ld(st + hf), p = P::ld(st + IE + hf), v = P::ld(st + 2 * IE + hf);
        const P q = P::ld(st + 3 * IE + hf), y = P::ld(st + 4 * IE + hf);
        const P s = P::fmas(mal_s, v, r);
        const P t = P::fmas(mal_s, y, q);
        const P rn = P::fmas(mom_s, t, s);
        P::fmas(be_s, P::fmas(mom_s, v, p), rn).st(pr + hf);
        rn.st(rr + hf);
      }
      load_x(m + 1);
    }
    __syncthreads();
    if (tid == 0 && j + S < npi) issue_in(j + S);

    // ---------------- (B) v' = A p' on plane k+1 (own tile + one-point ring) ----------------
    if (j >= 2) {
      const int qc = j - 2;  // coefficient plane k+1
      mbar_wait(&mbar[S + qc % SC], (uint32_t)((qc / SC) & 1));
      const T *cf = CF + (qc % SC) * 6 * CE;
      const T *p0 = PR + ((j + 1) % 3) * IE;  // plane k
      const T *p1 = PR + ((j + 2) % 3) * IE;  // plane k+1
      const T *p2 = PR + (j % 3) * IE;        // plane k+2
      T *vr = VR + ((j + 1) & 1) * CE;
      {
#pragma unroll
        for (int d = 0; d < 6; ++d) cn[d] = P::ld(cf + d * CE + ec);
        const P xl = SH::left(pw1, SH::ld1(p1 + ei - 1)), xr = SH::right(pw1, SH::ld1(p1 + ei + VEC));
        const P vn = spmv<T>(cn, pw1, xl, xr, P::ld(p1 + ei - HW), P::ld(p1 + ei + HW), pw0, pw2);
        vn.st(vr + ec);
        vw2 = vn;
        if (inside && k + 1 >= z0 && k + 1 < z1) vn.st(Og[2] + (long long)(k + 1) * plane + gofs);
      }
      if (hv >= 0) {
        const int hp = hv + HW;  // same point in the input-box layout
        P c[6];
#pragma unroll
        for (int d = 0; d < 6; ++d) c[d] = P::ld(cf + d * CE + hv);
        const P m1 = P::ld(p1 + hp);
        const typename SH::E zl = hvc == 0 ? (typename SH::E)0 : SH::ld1(p1 + hp - 1);
        const typename SH::E zr = hvc == VW - 1 ? (typename SH::E)0 : SH::ld1(p1 + hp + VEC);
        spmv<T>(c, m1, SH::left(m1, zl), SH::right(m1, zr), P::ld(p1 + hp - HW), P::ld(p1 + hp + HW),
                P::ld(p0 + hp), P::ld(p2 + hp))
            .st(vr + hv);
      }
      if (G::MMA && j >= 5) gram_plane((j + 1) & 3);  // plane k-1, staged in C(k-1)
      __syncthreads();
      if (tid == 0 && qc + SC < npc) issue_c(qc + SC);
    }

    // ---------------- (C) q' = A r', y' = A v' on plane k; the twelve dots ----------------
    if (j >= 4) {
      const T *r1 = RR + ((j + 2) & 3) * IE;  // r' plane k
      const T *v1 = VR + (j & 1) * CE;        // v' plane k
      const P qn = spmv<T>(cc, rw1, SH::left(rw1, SH::ld1(r1 + ei - 1)), SH::right(rw1, SH::ld1(r1 + ei + VEC)),
                           P::ld(r1 + ei - HW), P::ld(r1 + ei + HW), rw0, rw2);
      const P yn = spmv<T>(cc, vw1, SH::left(vw1, SH::ld1(v1 + ec - 1)), SH::right(vw1, SH::ld1(v1 + ec + VEC)),
                           P::ld(v1 + ec - HW), P::ld(v1 + ec + HW), vw0, vw2);
      const P rh = rhn;
      load_rh(k + 1);
      if (inside) {
        const long long o = (long long)k * plane + gofs;
        qn.st(Og[3] + o);
        yn.st(Og[4] + o);
      }
      if (G::MMA) {  // stage rh, v', q', y' of plane k for the tensor-core Gram (read in B(k+1))
        T *g = GS + ry * G::BX + cx * VEC;
        (inside ? rh : P::zero()).st(g);
        (inside ? vw1 : P::zero()).st(g + G::GSV);
        (inside ? qn : P::zero()).st(g + 2 * G::GSV);
        (inside ? yn : P::zero()).st(g + 3 * G::GSV);
      } else if (inside) {
        dacc[0] = rh.mdot(vw1, dacc[0]);   // (rh, v)
        dacc[1] = rh.mdot(rw1, dacc[1]);   // (rh, r)
        dacc[2] = rh.mdot(qn, dacc[2]);    // (rh, q)
        dacc[3] = rh.mdot(yn, dacc[3]);    // (rh, y)
        dacc[4] = qn.mdot(rw1, dacc[4]);   // (q, r)
        dacc[5] = qn.mdot(vw1, dacc[5]);   // (q, v)
        dacc[6] = yn.mdot(rw1, dacc[6]);   // (y, r)
        dacc[7] = yn.mdot(vw1, dacc[7]);   // (y, v)
        dacc[8] = qn.mdot(qn, dacc[8]);    // (q, q)
        dacc[9] = qn.mdot(yn, dacc[9]);    // (q, y)
        dacc[10] = yn.mdot(yn, dacc[10]);  // (y, y)
        dacc[11] = rw1.mdot(rw1, dacc[11]);  // (r, r)
      }
    }
    pw0 = pw1;
    pw1 = pw2;
    rw0 = rw1;
    rw1 = rw2;
    rw2 = rw3;
    vw0 = vw1;
    vw1 = vw2;
#pragma unroll
    for (int d = 0; d < 6; ++d) cc[d] = cn[d];
  }
  if (G::MMA) {
    __syncthreads();
    gram_plane((npi + 1) & 3);  // the last plane, staged in C of the last step
    // G[a][b] sits in lane 4a + b/2, register b%2 (a, b: 0 rh, 1 r, 2 v, 3 q, 4 y)
    constexpr int A_[12] = {0, 0, 0, 0, 3, 3, 4, 4, 3, 3, 4, 1};
    constexpr int B_[12] = {2, 1, 3, 4, 1, 2, 1, 2, 3, 4, 4, 1};
    const int lane = tid & 31;
#pragma unroll
    for (int d = 0; d < 12; ++d)
      dacc[d] = (lane == 4 * A_[d] + B_[d] / 2) ? gacc[B_[d] & 1] : 0.0f;
  }
  grid_reduce_finalize<12, PH_SR>(dacc, a.red, scratch);
}

// ------------------------------------------------------------ host side --
namespace {
template <typename T, int BY, int S, int SC>
int launch_sr_one(const SrArgs &a, cudaStream_t s) {
  constexpr size_t smem = sr_smem_c<T, BY, S, SC>();
  static_assert(smem <= 227 * 1024, "shared memory budget");
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_sr<T, BY, S, SC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
    configured = true;
  }
  const int grid = a.tiles_x * a.tiles_y * ((a.g.nz + a.zc - 1) / a.zc);
  k_sr<T, BY, S, SC><<<grid, SrGeo<T, BY>::NT, smem, s>>>(a);
  return (int)cudaGetLastError();
}
}  // namespace

#define STEN_SR_CONFIGS(X) X(16, 3, 2) X(16, 2, 2) X(8, 2, 2) X(8, 3, 2) X(8, 4, 3)

bool sr_config_ok(int by, int stages, int cstages) {
#define X(B, S_, C_) if (by == B && stages == S_ && cstages == C_) return true;
  STEN_SR_CONFIGS(X)
#undef X
  return false;
}

template <typename T>
int sr_launch(const SrArgs &a, int by, int stages, int cstages, cudaStream_t s) {
#define X(B, S_, C_) if (by == B && stages == S_ && cstages == C_) return launch_sr_one<T, B, S_, C_>(a, s);
  STEN_SR_CONFIGS(X)
#undef X
  return (int)cudaErrorInvalidValue;
}

template <typename T>
size_t sr_smem_bytes(int by, int stages, int cstages) {
#define X(B, S_, C_) if (by == B && stages == S_ && cstages == C_) return sr_smem_c<T, B, S_, C_>();
  STEN_SR_CONFIGS(X)
#undef X
  return 0;
}

template <typename T>
int sr_threads(int by) {
  return (tile_bx<T>() / Pack<T>::VEC) * by;
}

template int sr_launch<float>(const SrArgs &, int, int, int, cudaStream_t);
template int sr_launch<__half>(const SrArgs &, int, int, int, cudaStream_t);
template size_t sr_smem_bytes<float>(int, int, int);
template size_t sr_smem_bytes<__half>(int, int, int);
template int sr_threads<float>(int);
template int sr_threads<__half>(int);

}  // namespace sten
