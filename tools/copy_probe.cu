// Local HBM copy variants (developer tool): what reaches the measured copy
// peak on B200 for the p = 1 all_reduce floor (256 MiB out-of-place).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

template <int U, int MODE>
__global__ void __launch_bounds__(512) cp(uint4* __restrict__ d, const uint4* __restrict__ s, long n) {
  const long stride = long(gridDim.x) * blockDim.x;
  long i = long(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (MODE == 0) v[u] = __ldcs(s + i + u * stride);
      else if (MODE == 1) v[u] = s[i + u * stride];
      else v[u] = __ldg(s + i + u * stride);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (MODE == 0) __stcs(d + i + u * stride, v[u]);
      else d[i + u * stride] = v[u];
    }
  }
  for (; i < n; i += stride) d[i] = s[i];
}

// 32-byte per thread (two uint4 adjacent) to test wider per-thread sectors
template <int U>
__global__ void __launch_bounds__(256) cp32(uint4* __restrict__ d, const uint4* __restrict__ s, long n2) {
  const long stride = long(gridDim.x) * blockDim.x;
  long i = long(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n2; i += U * stride) {
    uint4 a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      a[u] = __ldcs(s + 2 * (i + u * stride));
      b[u] = __ldcs(s + 2 * (i + u * stride) + 1);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      __stcs(d + 2 * (i + u * stride), a[u]);
      __stcs(d + 2 * (i + u * stride) + 1, b[u]);
    }
  }
}

typedef void (*kfn)(uint4*, const uint4*, long);

float timeit(kfn f, int grid, int block, uint4* d, uint4* s, long n, cudaStream_t st) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  f<<<grid, block, 0, st>>>(d, s, n);
  CK(cudaEventRecord(a, st));
  for (int i = 0; i < 20; ++i) f<<<grid, block, 0, st>>>(d, s, n);
  CK(cudaEventRecord(b, st));
  CK(cudaEventSynchronize(b));
  float ms;
  CK(cudaEventElapsedTime(&ms, a, b));
  return 2.0 * n * 16 / (ms / 20) / 1e6;
}

int main() {
  const long bytes = 256l << 20, n = bytes / 16;
  uint4 *s, *d;
  CK(cudaMalloc(&s, bytes));
  CK(cudaMalloc(&d, bytes));
  CK(cudaMemset(s, 1, bytes));
  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  int grids[] = {148, 296, 444, 592, 1184, 2368};
  struct K { const char* name; kfn f; int block; long nn; } ks[] = {
      {"U4 cs", cp<4, 0>, 512, n}, {"U8 cs", cp<8, 0>, 512, n}, {"U4 plain", cp<4, 1>, 512, n},
      {"U8 plain", cp<8, 1>, 512, n}, {"U4 ldg", cp<4, 2>, 512, n}, {"U2 cs", cp<2, 0>, 512, n},
      {"32B U4 cs", cp32<4>, 256, n / 2}};
  for (auto& k : ks) {
    printf("%-10s", k.name);
    for (int g : grids) printf("  g%-4d %6.0f", g, timeit(k.f, g, k.block, d, s, k.nn, st));
    printf("  GB/s (read+write)\n");
  }
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaEventRecord(a, st));
  for (int i = 0; i < 20; ++i) CK(cudaMemcpyAsync(d, s, bytes, cudaMemcpyDeviceToDevice, st));
  CK(cudaEventRecord(b, st));
  CK(cudaEventSynchronize(b));
  float ms;
  CK(cudaEventElapsedTime(&ms, a, b));
  printf("cudaMemcpyAsync D2D: %6.0f GB/s\n", 2.0 * bytes / (ms / 20) / 1e6);
  return 0;
}
