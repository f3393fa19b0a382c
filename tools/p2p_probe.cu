// NVLink peer bandwidth probe (developer tool, not part of the library).
// One process, two GPUs with peer access; measures GB/s per direction for
// SM push-stores, SM pull-loads, bidirectional push, and cudaMemcpyPeerAsync,
// over grid sizes and unroll factors. Nothing here waits on another kernel.
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e));  \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

template <int U>
__global__ void __launch_bounds__(512) copy16(uint4* __restrict__ dst, const uint4* __restrict__ src,
                                              long n) {
  long i = long(blockIdx.x) * blockDim.x + threadIdx.x;
  const long stride = long(gridDim.x) * blockDim.x;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = src[i + u * stride];
#pragma unroll
    for (int u = 0; u < U; ++u) dst[i + u * stride] = v[u];
  }
  for (; i < n; i += stride) dst[i] = src[i];
}

// contiguous chunk per block (like the library's byte_share)
template <int U>
__global__ void __launch_bounds__(512) copy16_chunk(uint4* __restrict__ dst, const uint4* __restrict__ src,
                                                    long n) {
  long per = (n + gridDim.x - 1) / gridDim.x;
  long s = per * blockIdx.x, e = s + per < n ? s + per : n;
  const int nt = blockDim.x;
  long i = s + threadIdx.x;
  for (; i + (U - 1) * nt < e; i += U * nt) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = src[i + u * nt];
#pragma unroll
    for (int u = 0; u < U; ++u) dst[i + u * nt] = v[u];
  }
  for (; i < e; i += nt) dst[i] = src[i];
}

typedef void (*kfn)(uint4*, const uint4*, long);

static float run(int dev, kfn k, int grid, uint4* dst, const uint4* src, long n, cudaStream_t s,
                 int iters) {
  CK(cudaSetDevice(dev));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  k<<<grid, 512, 0, s>>>(dst, src, n);
  CK(cudaEventRecord(a, s));
  for (int i = 0; i < iters; ++i) k<<<grid, 512, 0, s>>>(dst, src, n);
  CK(cudaEventRecord(b, s));
  CK(cudaEventSynchronize(b));
  float ms;
  CK(cudaEventElapsedTime(&ms, a, b));
  return ms / iters;
}

int main() {
  int ndev;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) {
    printf("need 2 GPUs\n");
    return 0;
  }
  const long bytes = 256l << 20;
  const long n = bytes / 16;
  uint4 *a0, *b0, *a1, *b1;
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaMalloc(&a0, bytes));
  CK(cudaMalloc(&b0, bytes));
  CK(cudaMemset(a0, 1, bytes));
  cudaStream_t s0, s1;
  CK(cudaStreamCreate(&s0));
  CK(cudaSetDevice(1));
  CK(cudaDeviceEnablePeerAccess(0, 0));
  CK(cudaMalloc(&a1, bytes));
  CK(cudaMalloc(&b1, bytes));
  CK(cudaMemset(a1, 2, bytes));
  CK(cudaStreamCreate(&s1));
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("SMs %d, %ld MiB per transfer\n", sms, bytes >> 20);
  int grids[] = {sms / 2, sms, 2 * sms, 4 * sms, 8 * sms};
  struct K { const char* name; kfn f; } ks[] = {
      {"grid-stride U1", copy16<1>}, {"grid-stride U4", copy16<4>}, {"grid-stride U8", copy16<8>},
      {"chunk U4", copy16_chunk<4>}, {"chunk U8", copy16_chunk<8>}};
  for (auto& k : ks) {
    for (int g : grids) {
      float push = run(0, k.f, g, b1, a0, n, s0, 10);  // GPU0 stores into GPU1
      float pull = run(0, k.f, g, b0, a1, n, s0, 10);  // GPU0 loads from GPU1
      float local = run(0, k.f, g, b0, a0, n, s0, 10);
      printf("%-16s grid %4d: push %6.1f GB/s  pull %6.1f GB/s  local(copy rd+wr) %7.1f GB/s\n",
             k.name, g, bytes / push / 1e6, bytes / pull / 1e6, 2 * bytes / local / 1e6);
    }
  }
  // bidirectional push: both GPUs store into each other at the same time
  for (int g : grids) {
    CK(cudaSetDevice(0));
    cudaEvent_t e0a, e0b;
    CK(cudaEventCreate(&e0a));
    CK(cudaEventCreate(&e0b));
    CK(cudaEventRecord(e0a, s0));
    for (int i = 0; i < 10; ++i) copy16<4><<<g, 512, 0, s0>>>(b1, a0, n);
    CK(cudaEventRecord(e0b, s0));
    CK(cudaSetDevice(1));
    for (int i = 0; i < 10; ++i) copy16<4><<<g, 512, 0, s1>>>(b0, a1, n);
    CK(cudaStreamSynchronize(s1));
    CK(cudaSetDevice(0));
    CK(cudaEventSynchronize(e0b));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0a, e0b));
    printf("bidir push U4 grid %4d: %6.1f GB/s per direction (GPU0 clock)\n", g,
           bytes / (ms / 10) / 1e6);
  }
  CK(cudaSetDevice(0));
  cudaEvent_t x, y;
  CK(cudaEventCreate(&x));
  CK(cudaEventCreate(&y));
  CK(cudaEventRecord(x, s0));
  for (int i = 0; i < 10; ++i) CK(cudaMemcpyPeerAsync(b1, 1, a0, 0, bytes, s0));
  CK(cudaEventRecord(y, s0));
  CK(cudaEventSynchronize(y));
  float ms;
  CK(cudaEventElapsedTime(&ms, x, y));
  printf("cudaMemcpyPeerAsync 0->1: %6.1f GB/s\n", bytes / (ms / 10) / 1e6);
  return 0;
}
