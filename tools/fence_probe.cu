// Cost of per-chunk release flags on NVLink push bandwidth (developer tool).
// GPU0 pushes 256 MiB into GPU1 in chunks; after each chunk the CTA (or warp)
// publishes a flag into GPU1 memory. Variants: CTA-level chunk + syncthreads +
// fence + st.release; warp-level chunk + syncwarp + st.release; no flags.
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// MODE 0: no flags; 1: CTA chunk + syncthreads + threadfence_system + release;
// 2: CTA chunk + syncthreads + release only; 3: warp chunk + syncwarp + release
template <int MODE>
__global__ void __launch_bounds__(512) push(uint4* dst, const uint4* src, long n, long chunk_packs,
                                            uint64_t* flags) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const long per = (n + gridDim.x - 1) / gridDim.x;
  const long s = per * blockIdx.x, e = min(n, s + per);
  if (MODE == 3) {
    const int w = tid / 32, lane = tid % 32, nw = nt / 32;
    const long wper = (e - s + nw - 1) / nw;
    const long ws = s + w * wper, we = min(e, ws + wper);
    uint64_t step = 0;
    for (long c0 = ws; c0 < we; c0 += chunk_packs) {
      const long c1 = min(we, c0 + chunk_packs);
      long i = c0 + lane;
      for (; i + 3 * 32 < c1; i += 4 * 32) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = src[i + u * 32];
#pragma unroll
        for (int u = 0; u < 4; ++u) dst[i + u * 32] = v[u];
      }
      for (; i < c1; i += 32) dst[i] = src[i];
      __syncwarp();
      if (lane == 0) st_release_sys(&flags[blockIdx.x * 16 + w], ++step);
    }
    return;
  }
  uint64_t step = 0;
  for (long c0 = s; c0 < e; c0 += chunk_packs) {
    const long c1 = min(e, c0 + chunk_packs);
    long i = c0 + tid;
    for (; i + 3 * nt < c1; i += 4 * nt) {
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = src[i + u * nt];
#pragma unroll
      for (int u = 0; u < 4; ++u) dst[i + u * nt] = v[u];
    }
    for (; i < c1; i += nt) dst[i] = src[i];
    if (MODE == 1 || MODE == 2) {
      __syncthreads();
      if (tid == 0) {
        if (MODE == 1) __threadfence_system();
        st_release_sys(&flags[blockIdx.x], ++step);
      }
    }
  }
}

typedef void (*kfn)(uint4*, const uint4*, long, long, uint64_t*);

int main() {
  const long bytes = 256l << 20, n = bytes / 16;
  uint4 *a0, *b1;
  uint64_t* f1;
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&b1, bytes));
  CK(cudaMalloc(&f1, 1 << 20));
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaMalloc(&a0, bytes));
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  cudaEvent_t x, y;
  CK(cudaEventCreate(&x));
  CK(cudaEventCreate(&y));
  struct { const char* name; kfn f; } ks[] = {{"noflag", push<0>}, {"cta+fence+rel", push<1>},
                                             {"cta+rel", push<2>}, {"warp+rel", push<3>}};
  long chunks[] = {1024, 4096, 16384, 65536};  // packs: 16K, 64K, 256K, 1M bytes
  int grids[] = {74, 148, 296};
  for (auto& k : ks)
    for (int g : grids)
      for (long ch : chunks) {
        long cp = ch;
        if (k.f == push<3>) cp = ch / 16;  // warp chunk = CTA chunk / 16 warps
        if (cp < 32) cp = 32;
        k.f<<<g, 512, 0, s>>>(b1, a0, n, cp, f1);
        CK(cudaEventRecord(x, s));
        for (int i = 0; i < 10; ++i) k.f<<<g, 512, 0, s>>>(b1, a0, n, cp, f1);
        CK(cudaEventRecord(y, s));
        CK(cudaEventSynchronize(y));
        float ms;
        CK(cudaEventElapsedTime(&ms, x, y));
        printf("%-14s grid %3d chunk %7ld B: %6.1f GB/s\n", k.name, g, cp * 16, bytes / (ms / 10) / 1e6);
        if (k.f == push<0>) break;
      }
  return 0;
}
