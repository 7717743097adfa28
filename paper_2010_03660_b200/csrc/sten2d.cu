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

template <typename T, int BY>
__global__ void __launch_bounds__((Tile2<T>::BX / Pack<T>::VEC) * BY) k_apply9(const __grid_constant__ Apply9Args a) {
  using P = Pack<T>;
  using SH = Sh2<T>;
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
  const P vm = P::ld(box + e - HW), vc = P::ld(box + e), vp = P::ld(box + e + HW);
  P u = vc;
  u = P::fma(c[0], SH::left(vm, SH::ld1(box + e - HW - 1)), u);
  u = P::fma(c[1], vm, u);
  u = P::fma(c[2], SH::right(vm, SH::ld1(box + e - HW + VEC)), u);
  u = P::fma(c[3], SH::left(vc, SH::ld1(box + e - 1)), u);
  u = P::fma(c[4], SH::right(vc, SH::ld1(box + e + VEC)), u);
  u = P::fma(c[5], SH::left(vp, SH::ld1(box + e + HW - 1)), u);
  u = P::fma(c[6], vp, u);
  u = P::fma(c[7], SH::right(vp, SH::ld1(box + e + HW + VEC)), u);
  if (inside) u.st(reinterpret_cast<T *>(a.u) + o);
}

// Jacobi scaling of the 9-point operator (R3/R5 in 2D): c_d = A_d / A_P in
// fp64, couplings leaving the mesh dropped, rounded RN to fp32 and fp16;
// padding columns hold zero couplings
template <typename TIN>
__global__ void k_create9(const TIN *diag, Coef9In in, int nx, int ny, int pitch, Coef9Out out) {
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
  }
}

template <typename T>
int apply9_launch(const Apply9Args &a, cudaStream_t s) {
  constexpr int BY = 32;
  const int ty = (a.ny + BY - 1) / BY;
  k_apply9<T, BY><<<a.tiles_x * ty, (Tile2<T>::BX / Pack<T>::VEC) * BY, 0, s>>>(a);
  return (int)cudaGetLastError();
}
template int apply9_launch<float>(const Apply9Args &, cudaStream_t);
template int apply9_launch<__half>(const Apply9Args &, cudaStream_t);

int create9_launch(int in_dtype, const void *diag, const Coef9In &in, int nx, int ny, int pitch, const Coef9Out &out,
                   cudaStream_t s) {
  const long long total = (long long)pitch * ny;
  int grid = (int)((total + 255) / 256);
  if (grid > 148 * 32) grid = 148 * 32;
  if (grid < 1) grid = 1;
  if (in_dtype == STEN_DT_F64) k_create9<double><<<grid, 256, 0, s>>>((const double *)diag, in, nx, ny, pitch, out);
  else k_create9<float><<<grid, 256, 0, s>>>((const float *)diag, in, nx, ny, pitch, out);
  return (int)cudaGetLastError();
}

}  // namespace sten
