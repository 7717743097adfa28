// gen_cuda.cu - device twin of inputs/gen.py (seeded synthetic problem fields).
//
// Input synthesis only: no step of the method (no Jacobi scaling, SpMV or
// BiCGStab arithmetic) lives here.  Every value is a pure function of
// (seed, stream, global index) and is bit-identical to gen.py: SplitMix64
// finalizer, 53-bit uniform, a + (b-a)*u with separately rounded fp64 ops
// (__dmul_rn/__dadd_rn so nvcc cannot contract them into an FMA).
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

constexpr uint64_t C_GOLD = 0x9E3779B97F4A7C15ull;
constexpr uint64_t C_STREAM = 0xD1B54A32D192ED03ull;
constexpr uint64_t C_OFF = 0x632BE59BD9B4E019ull;

__host__ __device__ inline uint64_t mix(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}
__host__ __device__ inline uint64_t key(uint64_t seed, uint64_t stream) {
  return mix(seed * C_GOLD + stream * C_STREAM + C_OFF);
}
__device__ inline double uniform(uint64_t k, uint64_t idx, double a, double b) {
  uint64_t h = mix(k + (idx + 1ull) * C_GOLD);
  double u = __dmul_rn((double)(h >> 11), 1.1102230246251565e-16 /* 2^-53 */);
  return __dadd_rn(a, __dmul_rn(__dadd_rn(b, -a), u));
}

__global__ void k_fields(int kind, int nx, int ny, int nz, long long z0, uint64_t seed, double factor,
                         const double *__restrict__ kz, double *diag, double *o0, double *o1, double *o2,
                         double *o3, double *o4, double *o5) {
  double *off[6] = {o0, o1, o2, o3, o4, o5};
  const long long n = (long long)nx * ny * nz;
  const uint64_t kK = key(seed, 1), kX = key(seed, 2), kY = key(seed, 3), kZ = key(seed, 4), kN = key(seed, 5);
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x) {
    if (kind == 0) {  // Poisson
      diag[q] = 6.0;
      for (int d = 0; d < 6; ++d) off[d][q] = -1.0;
      continue;
    }
    const long long kl = q / ((long long)nx * ny);
    const uint64_t idx = (uint64_t)(q + z0 * (long long)nx * ny);  // global linear index
    double kd;
    if (kind == 1) {
      kd = uniform(kK, idx, 0.5, 2.0);
    } else {
      double xi = uniform(kN, idx, -1.0, 1.0);
      kd = __dmul_rn(kz[z0 + kl], __dadd_rn(1.0, __dmul_rn(0.1, xi)));
    }
    const double ux = uniform(kX, idx, -1.0, 1.0), uy = uniform(kY, idx, -1.0, 1.0), uz = uniform(kZ, idx, -1.0, 1.0);
    double a[6] = {__dadd_rn(kd, fmax(ux, 0.0)), __dadd_rn(kd, fmax(-ux, 0.0)), __dadd_rn(kd, fmax(uy, 0.0)),
                   __dadd_rn(kd, fmax(-uy, 0.0)), __dadd_rn(kd, fmax(uz, 0.0)), __dadd_rn(kd, fmax(-uz, 0.0))};
    double s = __dadd_rn(a[0], a[1]);
    s = __dadd_rn(s, a[2]);
    s = __dadd_rn(s, a[3]);
    s = __dadd_rn(s, a[4]);
    s = __dadd_rn(s, a[5]);
    diag[q] = __dmul_rn(factor, s);
    for (int d = 0; d < 6; ++d) off[d][q] = -a[d];
  }
}

// the 2D 9-point stand-in (gen.py problem_fields_2d); offs in the o2d.c order
__global__ void k_fields2d(int nx, int ny, uint64_t seed, double factor, double *diag, double *o0, double *o1,
                           double *o2, double *o3, double *o4, double *o5, double *o6, double *o7) {
  double *off[8] = {o0, o1, o2, o3, o4, o5, o6, o7};
  const long long n = (long long)nx * ny;
  const uint64_t kK = key(seed, 1), kX = key(seed, 2), kY = key(seed, 3);
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x) {
    const uint64_t idx = (uint64_t)q;
    const double kd = uniform(kK, idx, 0.5, 2.0);
    const double ux = uniform(kX, idx, -1.0, 1.0), uy = uniform(kY, idx, -1.0, 1.0);
    const double c = __dmul_rn(0.25, kd);
    double a[8] = {c, __dadd_rn(kd, fmax(uy, 0.0)), c, __dadd_rn(kd, fmax(ux, 0.0)), __dadd_rn(kd, fmax(-ux, 0.0)),
                   c, __dadd_rn(kd, fmax(-uy, 0.0)), c};
    double s = __dadd_rn(a[0], a[1]);
    for (int d = 2; d < 8; ++d) s = __dadd_rn(s, a[d]);
    diag[q] = __dmul_rn(factor, s);
    for (int d = 0; d < 8; ++d) off[d][q] = -a[d];
  }
}

__global__ void k_uniform(int nx, int ny, int nz, long long z0, uint64_t seed, uint64_t stream, double lo, double hi,
                          int out_dtype, void *out) {
  const long long n = (long long)nx * ny * nz;
  const uint64_t k = key(seed, stream);
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x) {
    double v = uniform(k, (uint64_t)(q + z0 * (long long)nx * ny), lo, hi);
    if (out_dtype == 0) reinterpret_cast<double *>(out)[q] = v;
    else reinterpret_cast<float *>(out)[q] = __double2float_rn(v);
  }
}

int grid_for(long long n) {
  long long g = (n + 255) / 256;
  if (g > 148 * 64) g = 148 * 64;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace

extern "C" {
// kind: 0 Poisson, 1 convection-diffusion, 2 weak-scaling variant (kz indexed by
// global plane, device pointer).  Writes dense (nz,ny,nx) fp64 arrays.
int sten_inputs_fields(int kind, int nx, int ny, int nz, long long z0, unsigned long long seed, double factor,
                       const double *kz_dev, double *diag, double *const off[6], void *stream) {
  long long n = (long long)nx * ny * nz;
  k_fields<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(kind, nx, ny, nz, z0, seed, factor, kz_dev, diag, off[0],
                                                          off[1], off[2], off[3], off[4], off[5]);
  return (int)cudaGetLastError();
}
// the 2D 9-point stand-in: dense (ny,nx) fp64 arrays, off[8] in the o2d.c order
int sten_inputs_fields2d(int nx, int ny, unsigned long long seed, double factor, double *diag, double *const off[8],
                         void *stream) {
  long long n = (long long)nx * ny;
  k_fields2d<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(nx, ny, seed, factor, diag, off[0], off[1], off[2],
                                                            off[3], off[4], off[5], off[6], off[7]);
  return (int)cudaGetLastError();
}
// U(lo,hi) of `stream` on planes [z0, z0+nz); out_dtype 0: fp64, 1: fp32 (RN of the fp64 value)
int sten_inputs_uniform(int nx, int ny, int nz, long long z0, unsigned long long seed, unsigned long long stream_id,
                        double lo, double hi, int out_dtype, void *out, void *stream) {
  long long n = (long long)nx * ny * nz;
  k_uniform<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(nx, ny, nz, z0, seed, stream_id, lo, hi, out_dtype, out);
  return (int)cudaGetLastError();
}
}
