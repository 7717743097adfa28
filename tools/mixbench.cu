// mixbench.cu - HBM bandwidth of a streaming kernel with R read and W written
// arrays per element (16-B vectors, grid-stride), to know the ceiling of the SR
// sweep's read/write mix (13 reads : 6 writes per point) next to the plain copy
// (1 : 1) that MEASURED_PEAKS.json quotes.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/mixbench.cu -o tools/mixbench
#include <cstdio>
#include <cstdint>
#include <vector>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int kMax = 20;
struct Args { const uint4 *in[kMax]; uint4 *out[kMax]; long long n; };

template <int R, int W>
__global__ void __launch_bounds__(256) k_mix(const __grid_constant__ Args a) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += stride) {
    uint4 acc = make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const uint4 v = __ldcs(a.in[r] + i);
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
#pragma unroll
    for (int w = 0; w < W; ++w) __stcs(a.out[w] + i, make_uint4(acc.x + w, acc.y, acc.z, acc.w));
  }
}

template <int R, int W>
int run(const std::vector<void *> &bufs, long long n, int sms) {
  Args a;
  for (int r = 0; r < R; ++r) a.in[r] = (const uint4 *)bufs[r];
  for (int w = 0; w < W; ++w) a.out[w] = (uint4 *)bufs[R + w];
  a.n = n;
  float best = 1e30f;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int ctas : {8, 16, 32}) {
    for (int rep = 0; rep < 6; ++rep) {
      CK(cudaEventRecord(e0));
      k_mix<R, W><<<sms * ctas, 256>>>(a);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (rep > 0 && ms < best) best = ms;
    }
  }
  const double bytes = (double)(R + W) * n * 16;
  printf("R=%2d W=%2d  %.3f ms  %.0f GB/s\n", R, W, best, bytes / best / 1e6);
  return 0;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const long long elems = 548352000LL;  // one fp16 vector of config 3
  const long long n = elems * 2 / 16;   // 16-B vectors
  std::vector<void *> bufs(19);
  for (auto &b : bufs) {
    CK(cudaMalloc(&b, n * 16));
    CK(cudaMemset(b, 1, n * 16));
  }
  run<1, 1>(bufs, n, sms);
  run<13, 6>(bufs, n, sms);
  run<19, 0>(bufs, n, sms);
  run<2, 1>(bufs, n, sms);
  run<5, 2>(bufs, n, sms);
  run<9, 1>(bufs, n, sms);
  return 0;
}
