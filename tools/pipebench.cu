// Throughput of the candidate dot-product instructions on sm_100a (one SM,
// 8 warps, 8 independent chains per thread): FHFMA (fma.rn.f32.f16), FFMA,
// FFMA2 (fma.rn.f32x2), HFMA2, HADD2.F32 conversion, mma.sync m16n8k16.
#include <cstdio>
#include <cuda_fp16.h>
#define N 4096
__global__ void k_fhfma(unsigned *io, float *out, long long *cyc) {
  unsigned a = io[threadIdx.x], b = io[threadIdx.x + 1];
  float acc[8] = {0, 1, 2, 3, 4, 5, 6, 7};
  long long t0 = clock64();
  for (int i = 0; i < N; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("{ .reg .b16 l, h; mov.b32 {l, h}, %1; fma.rn.f32.f16 %0, l, h, %0; }" : "+f"(acc[j]) : "r"(a ^ j));
  }
  long long t1 = clock64();
  float s = 0; for (int j = 0; j < 8; ++j) s += acc[j];
  out[threadIdx.x] = s; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_ffma(unsigned *io, float *out, long long *cyc) {
  float a = __int_as_float(io[threadIdx.x]), b = __int_as_float(io[threadIdx.x + 1]);
  float acc[8] = {0, 1, 2, 3, 4, 5, 6, 7};
  long long t0 = clock64();
  for (int i = 0; i < N; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(acc[j]) : "f"(a), "f"(b));
  }
  long long t1 = clock64();
  float s = 0; for (int j = 0; j < 8; ++j) s += acc[j];
  out[threadIdx.x] = s; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_ffma2(unsigned *io, float *out, long long *cyc) {
  unsigned long long a = ((unsigned long long)io[threadIdx.x] << 32) | io[threadIdx.x + 1];
  unsigned long long acc[8];
  for (int j = 0; j < 8; ++j) acc[j] = j;
  long long t0 = clock64();
  for (int i = 0; i < N; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) asm volatile("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(acc[j]) : "l"(a));
  }
  long long t1 = clock64();
  unsigned long long s = 0; for (int j = 0; j < 8; ++j) s ^= acc[j];
  out[threadIdx.x] = (float)s; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_hfma2(unsigned *io, float *out, long long *cyc) {
  unsigned a = io[threadIdx.x];
  unsigned acc[8];
  for (int j = 0; j < 8; ++j) acc[j] = j;
  long long t0 = clock64();
  for (int i = 0; i < N; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) asm volatile("fma.rn.f16x2 %0, %1, %1, %0;" : "+r"(acc[j]) : "r"(a));
  }
  long long t1 = clock64();
  unsigned s = 0; for (int j = 0; j < 8; ++j) s ^= acc[j];
  out[threadIdx.x] = (float)s; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_cvt(unsigned *io, float *out, long long *cyc) {
  unsigned a = io[threadIdx.x];
  float acc[8] = {0, 1, 2, 3, 4, 5, 6, 7};
  long long t0 = clock64();
  for (int i = 0; i < N; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float2 f = __half22float2(*reinterpret_cast<__half2 *>(&a));
      acc[j] += f.x;  // FADD + 2 conversions
      a += j;
    }
  }
  long long t1 = clock64();
  float s = 0; for (int j = 0; j < 8; ++j) s += acc[j];
  out[threadIdx.x] = s; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_mma(unsigned *io, float *out, long long *cyc) {
  unsigned a = io[threadIdx.x], b = io[threadIdx.x + 1];
  float c[8][4] = {};
  long long t0 = clock64();
  for (int i = 0; i < N / 4; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%4,%5,%5}, {%4,%5}, {%0,%1,%2,%3};"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3]) : "r"(a), "r"(b));
  }
  long long t1 = clock64();
  float s = 0; for (int j = 0; j < 8; ++j) s += c[j][0];
  out[threadIdx.x] = s; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
template <typename K> void run(const char *name, K k, int iters_per_thread, unsigned *io, float *out, long long *cyc) {
  k<<<1, 256>>>(io, out, cyc);
  cudaDeviceSynchronize();
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  // 8 warps on 4 SMSPs: warp-instructions per SMSP per cycle
  double wi = 8.0 * iters_per_thread * 8 / 4;
  printf("%-8s %8lld cycles  %.3f warp-instr/cycle/SMSP\n", name, c, wi / c);
}
int main() {
  unsigned *io; float *out; long long *cyc;
  cudaMalloc(&io, 4096); cudaMalloc(&out, 4096); cudaMalloc(&cyc, 8);
  cudaMemset(io, 0x3c, 4096);
  run("FHFMA", k_fhfma, N, io, out, cyc);
  run("FFMA", k_ffma, N, io, out, cyc);
  run("FFMA2", k_ffma2, N, io, out, cyc);
  run("HFMA2", k_hfma2, N, io, out, cyc);
  run("CVT+FADD", k_cvt, N, io, out, cyc);
  run("MMA", k_mma, N / 4, io, out, cyc);
  return 0;
}
