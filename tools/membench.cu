// membench.cu - streaming-pattern microbenchmark for the H3-like kernel shape
// (5 fp16 input streams, 2 output streams, 1.1 GB each) on B200.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membench membench.cu
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

struct P { const uint4 *a, *b, *c, *d, *e; uint4 *x, *y; long long n; };

__device__ __forceinline__ uint4 op(uint4 a, uint4 b, uint4 c) {
  uint4 r;
  __half2 *pa = (__half2 *)&a, *pb = (__half2 *)&b, *pc = (__half2 *)&c, *pr = (__half2 *)&r;
  for (int i = 0; i < 4; ++i) pr[i] = __hfma2(pa[i], pb[i], pc[i]);
  return r;
}

// A: grid-stride, U vectors per trip
template <int U>
__global__ void __launch_bounds__(256) k_gridstride(P p) {
  long long stride = (long long)gridDim.x * blockDim.x;
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < p.n; v += U * stride) {
    uint4 A[U], B[U], C[U], D[U], E[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      long long w = v + u * stride;
      if (w < p.n) { A[u] = __ldcs(p.a + w); B[u] = __ldcs(p.b + w); C[u] = __ldcs(p.c + w); D[u] = __ldcs(p.d + w); E[u] = __ldcs(p.e + w); }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      long long w = v + u * stride;
      if (w < p.n) { p.x[w] = op(A[u], B[u], C[u]); p.y[w] = op(C[u], D[u], E[u]); }
    }
  }
}

// B: block-contiguous chunks of CH vectors per block iteration
template <int U>
__global__ void __launch_bounds__(256) k_chunked(P p, long long chunk) {
  long long nchunks = (p.n + chunk - 1) / chunk;
  for (long long c = blockIdx.x; c < nchunks; c += gridDim.x) {
    long long base = c * chunk, end = min(base + chunk, p.n);
    for (long long v = base + threadIdx.x; v < end; v += U * blockDim.x) {
      uint4 A[U], B[U], C[U], D[U], E[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        long long w = v + u * blockDim.x;
        if (w < end) { A[u] = __ldcs(p.a + w); B[u] = __ldcs(p.b + w); C[u] = __ldcs(p.c + w); D[u] = __ldcs(p.d + w); E[u] = __ldcs(p.e + w); }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        long long w = v + u * blockDim.x;
        if (w < end) { p.x[w] = op(A[u], B[u], C[u]); p.y[w] = op(C[u], D[u], E[u]); }
      }
    }
  }
}

// C: TMA 1D bulk copies into smem, S stages of CH vectors per array
__device__ __forceinline__ uint32_t s32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int S, int CH>
__global__ void __launch_bounds__(256) k_bulk(P p) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t *bar = (uint64_t *)sm;
  uint4 *buf = (uint4 *)(sm + 128);
  const uint4 *src[5] = {p.a, p.b, p.c, p.d, p.e};
  long long nchunks = p.n / CH;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  auto issue = [&](long long c, int s) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar[s])), "r"(5 * CH * 16));
    for (int i = 0; i < 5; ++i)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       s32(buf + (s * 5 + i) * CH)), "l"(src[i] + c * CH), "r"(CH * 16), "r"(s32(&bar[s])) : "memory");
  };
  int k = 0;
  long long c0 = blockIdx.x;
  if (threadIdx.x == 0)
    for (int s = 0; s < S; ++s) if (c0 + (long long)s * gridDim.x < nchunks) issue(c0 + (long long)s * gridDim.x, s);
  for (long long c = c0; c < nchunks; c += gridDim.x, ++k) {
    int s = k % S; uint32_t par = (k / S) & 1, ok = 0;
    do { asm volatile("{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0,1,0,q; }" : "=r"(ok) : "r"(s32(&bar[s])), "r"(par) : "memory"); } while (!ok);
    uint4 *bs = buf + s * 5 * CH;
    for (int v = threadIdx.x; v < CH; v += blockDim.x) {
      uint4 A = bs[v], B = bs[CH + v], C = bs[2 * CH + v], D = bs[3 * CH + v], E = bs[4 * CH + v];
      p.x[c * CH + v] = op(A, B, C);
      p.y[c * CH + v] = op(C, D, E);
    }
    __syncthreads();
    long long cn = c + (long long)S * gridDim.x;
    if (threadIdx.x == 0 && cn < nchunks) issue(cn, s);
  }
}

__global__ void k_copy(const uint4 *a, uint4 *x, long long n) {
  long long stride = (long long)gridDim.x * blockDim.x;
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride) x[v] = __ldcs(a + v);
}

__global__ void k_fill(uint4 *x, long long n, unsigned seed) {
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (long long)gridDim.x * blockDim.x) {
    unsigned h = (unsigned)(v * 2654435761u) ^ seed;
    uint4 r;
    h = h * 1664525u + 1013904223u; r.x = (h & 0x3bff3bffu);
    h = h * 1664525u + 1013904223u; r.y = (h & 0x3bff3bffu);
    h = h * 1664525u + 1013904223u; r.z = (h & 0x3bff3bffu);
    h = h * 1664525u + 1013904223u; r.w = (h & 0x3bff3bffu);
    x[v] = r;
  }
}

int main(int argc, char **argv) {
  const int random_fill = argc > 1 ? atoi(argv[1]) : 0;
  const long long offset_vec = argc > 2 ? atoll(argv[2]) : 0;
  const long long npts = 600LL * 595 * 1536;  // fp16 points
  const long long n = npts / 8;               // uint4 vectors
  std::vector<void *> bufs(7);
  unsigned sd = 1;
  for (auto &b : bufs) {
    CK(cudaMalloc(&b, (n + 64) * 16)); CK(cudaMemset(b, 0, (n + 64) * 16));
    if (random_fill) k_fill<<<148 * 16, 256>>>((uint4 *)b, n + 64, sd++);
    b = (char *)b + offset_vec * 16;
  }
  CK(cudaDeviceSynchronize());
  printf("random_fill=%d offset=%lld B\n", random_fill, offset_vec * 16);
  P p{(uint4 *)bufs[0], (uint4 *)bufs[1], (uint4 *)bufs[2], (uint4 *)bufs[3], (uint4 *)bufs[4], (uint4 *)bufs[5], (uint4 *)bufs[6], n};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = 148;
  auto run = [&](const char *name, double bytes, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    cudaEventRecord(e0);
    const int R = 10;
    for (int i = 0; i < R; ++i) launch();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    printf("%-36s %8.3f ms  %7.1f GB/s %s\n", name, ms / R, bytes / (ms / R * 1e-3) / 1e9, err ? cudaGetErrorString(err) : "");
  };
  double b7 = 7.0 * n * 16, b2 = 2.0 * n * 16;
  run("copy 1R1W grid 148x8x256", b2, [&] { k_copy<<<sms * 8, 256>>>(p.a, p.x, n); });
  run("copy 1R1W grid 148x32x256", b2, [&] { k_copy<<<sms * 32, 256>>>(p.a, p.x, n); });
  run("gridstride U1 148x8", b7, [&] { k_gridstride<1><<<sms * 8, 256>>>(p); });
  run("gridstride U2 148x8", b7, [&] { k_gridstride<2><<<sms * 8, 256>>>(p); });
  run("gridstride U2 148x4", b7, [&] { k_gridstride<2><<<sms * 4, 256>>>(p); });
  run("gridstride U4 148x4", b7, [&] { k_gridstride<4><<<sms * 4, 256>>>(p); });
  run("gridstride U1 148x64 (1 pass)", b7, [&] { k_gridstride<1><<<(int)((n + 255) / 256 < sms * 64 ? (n + 255) / 256 : sms * 64), 256>>>(p); });
  for (long long ch : {1024LL, 4096LL, 16384LL}) {
    char nm[64]; snprintf(nm, 64, "chunked U2 148x4 chunk %lld", ch);
    run(nm, b7, [&] { k_chunked<2><<<sms * 4, 256>>>(p, ch); });
    snprintf(nm, 64, "chunked U1 148x8 chunk %lld", ch);
    run(nm, b7, [&] { k_chunked<1><<<sms * 8, 256>>>(p, ch); });
  }
  {
    constexpr int S = 4, CH = 512;  // 8 KB per array per stage, 160 KB smem
    size_t smem = 128 + (size_t)S * 5 * CH * 16;
    CK(cudaFuncSetAttribute(k_bulk<S, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    run("bulk S4 CH512 (8KB) 1 blk/SM", b7, [&] { k_bulk<S, CH><<<sms, 256, smem>>>(p); });
  }
  {
    constexpr int S = 3, CH = 256;  // 4 KB per array per stage, 60 KB smem
    size_t smem = 128 + (size_t)S * 5 * CH * 16;
    CK(cudaFuncSetAttribute(k_bulk<S, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    run("bulk S3 CH256 (4KB) 3 blk/SM", b7, [&] { k_bulk<S, CH><<<sms * 3, 256, smem>>>(p); });
  }
  {
    constexpr int S = 4, CH = 128;  // 2 KB per array per stage
    size_t smem = 128 + (size_t)S * 5 * CH * 16;
    CK(cudaFuncSetAttribute(k_bulk<S, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    run("bulk S4 CH128 (2KB) 4 blk/SM", b7, [&] { k_bulk<S, CH><<<sms * 4, 256, smem>>>(p); });
  }
  return 0;
}
