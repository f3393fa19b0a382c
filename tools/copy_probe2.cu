// Local HBM copy, round 2 (developer tool): the p = 1 all_reduce floor is a
// 256 MiB out-of-place copy timed back to back (bench.py). Compares the
// shipped k_copy geometry (grid-stride, 16 x SMs) with block-contiguous
// batches (no grid-stride tail) and a TMA bulk-copy ring.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/copy_probe2.cu -o copy_probe2
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

// shipped: grid-stride, 8 in flight, single-load tail loop
__global__ void __launch_bounds__(512) k_stride8(uint4* d, const uint4* s, long np) {
  const long stride = long(gridDim.x) * blockDim.x;
  long i = long(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + 7 * stride < np; i += 8 * stride) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = s[i + u * stride];
#pragma unroll
    for (int u = 0; u < 8; ++u) d[i + u * stride] = v[u];
  }
  for (; i < np; i += stride) d[i] = s[i];
}

// block-contiguous: CTA b copies packs [b*T*U, (b+1)*T*U), U loads in flight
template <int T, int U, int HINT>
__global__ void __launch_bounds__(T) k_block(uint4* d, const uint4* s, long np) {
  const long base = long(blockIdx.x) * T * U + threadIdx.x;
  uint4 v[U];
  if (base + (U - 1) * T < np) {
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = HINT ? __ldcs(s + base + u * T) : s[base + u * T];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (HINT) __stcs(d + base + u * T, v[u]);
      else d[base + u * T] = v[u];
    }
  } else {
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (base + u * T < np) v[u] = s[base + u * T];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (base + u * T < np) d[base + u * T] = v[u];
  }
}

// persistent block-contiguous: grid = resident CTAs, each loops over tiles
template <int T, int U>
__global__ void __launch_bounds__(T) k_persist(uint4* d, const uint4* s, long np) {
  const long tiles = (np + long(T) * U - 1) / (long(T) * U);
  for (long t = blockIdx.x; t < tiles; t += gridDim.x) {
    const long base = t * T * U + threadIdx.x;
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (base + u * T < np) v[u] = s[base + u * T];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (base + u * T < np) d[base + u * T] = v[u];
  }
}

// TMA ring: one elected thread per CTA, S stages of P bytes, contiguous share
__device__ __forceinline__ uint32_t sm32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
template <int P, int S>
__global__ void __launch_bounds__(32) k_tma(uint8_t* d, const uint8_t* s, long bytes) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar[S];
  if (threadIdx.x != 0) return;
  const long per = (bytes / gridDim.x + P - 1) / P * P;
  const long lo = long(blockIdx.x) * per;
  const long hi = lo + per < bytes ? lo + per : bytes;
  if (lo >= hi) return;
  const long np = (hi - lo + P - 1) / P;
  for (int k = 0; k < S; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sm32(&bar[k])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  auto load = [&](long k) {
    const int st = int(k % S);
    const long off = lo + k * P;
    const uint32_t sz = uint32_t(hi - off < P ? hi - off : P);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm32(&bar[st])), "r"(sz) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sm32(smem + st * P)), "l"(s + off), "r"(sz), "r"(sm32(&bar[st])) : "memory");
  };
  for (long k = 0; k < S && k < np; ++k) load(k);
  for (long k = 0; k < np; ++k) {
    const int st = int(k % S);
    const uint32_t ph = uint32_t((k / S) & 1);
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(ok) : "r"(sm32(&bar[st])), "r"(ph) : "memory");
    const long off = lo + k * P;
    const uint32_t sz = uint32_t(hi - off < P ? hi - off : P);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d + off), "r"(sm32(smem + st * P)), "r"(sz) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    // refill the stage the PREVIOUS store read (one store may stay in flight)
    if (k >= 1 && k - 1 + S < np) {
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      load(k - 1 + S);
    } else if (k == 0 && S == 1 && np > 1) {
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      load(1);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

static cudaStream_t g_st;
static cudaEvent_t g_a, g_b;

template <typename F>
static double timeit(F launch, long bytes, int reps = 20) {
  launch();
  launch();
  CK(cudaEventRecord(g_a, g_st));
  for (int i = 0; i < reps; ++i) launch();
  CK(cudaEventRecord(g_b, g_st));
  CK(cudaEventSynchronize(g_b));
  CK(cudaGetLastError());
  float ms;
  CK(cudaEventElapsedTime(&ms, g_a, g_b));
  return 2.0 * bytes / (ms / reps) / 1e6;
}

int main() {
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaStreamCreate(&g_st));
  CK(cudaEventCreate(&g_a));
  CK(cudaEventCreate(&g_b));
  const long sizes[] = {256l << 20, 1l << 30};
  for (long bytes : sizes) {
    const long np = bytes / 16;
    uint4 *s, *d;
    CK(cudaMalloc(&s, bytes));
    CK(cudaMalloc(&d, bytes));
    CK(cudaMemset(s, 1, bytes));
    printf("== %ld MiB, GB/s (read + write)\n", bytes >> 20);
    {
      long g = (bytes + 512l * 128 - 1) / (512l * 128);
      if (g > 16 * sms) g = 16 * sms;
      printf("shipped k_copy grid %ld          %7.0f\n", g, timeit([&] { k_stride8<<<g, 512, 0, g_st>>>(d, s, np); }, bytes));
    }
#define BLK(T, U, H)                                                                                   \
  {                                                                                                    \
    long g = (np + long(T) * U - 1) / (long(T) * U);                                                   \
    printf("block T%-4d U%-2d hint%d grid %-7ld  %7.0f\n", T, U, H, g,                                  \
           timeit([&] { k_block<T, U, H><<<g, T, 0, g_st>>>(d, s, np); }, bytes));                     \
  }
    BLK(512, 8, 0) BLK(512, 4, 0) BLK(256, 8, 0) BLK(256, 16, 0) BLK(128, 16, 0) BLK(512, 8, 1) BLK(256, 8, 1)
    BLK(1024, 4, 0) BLK(512, 2, 0)
#define PER(T, U, M)                                                                                   \
  {                                                                                                    \
    long g = long(M) * sms;                                                                            \
    printf("persist T%-4d U%-2d grid %-7ld       %7.0f\n", T, U, g,                                      \
           timeit([&] { k_persist<T, U><<<g, T, 0, g_st>>>(d, s, np); }, bytes));                      \
  }
    PER(512, 8, 2) PER(512, 8, 4) PER(256, 8, 8) PER(512, 4, 4)
#define TMA(P, S, M)                                                                                   \
  {                                                                                                    \
    auto k = k_tma<P, S>;                                                                              \
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, P * S));                  \
    long g = long(M) * sms;                                                                            \
    printf("tma P%-6d S%-2d grid %-7ld         %7.0f\n", P, S, g,                                       \
           timeit([&] { k<<<g, 32, P * S, g_st>>>((uint8_t*)d, (const uint8_t*)s, bytes); }, bytes));  \
  }
    TMA(16384, 8, 1) TMA(32768, 6, 1) TMA(16384, 6, 2) TMA(8192, 8, 4) TMA(32768, 3, 2) TMA(65536, 3, 1)
    TMA(16384, 4, 3) TMA(8192, 6, 4)
    printf("cudaMemcpyAsync D2D                %7.0f\n",
           timeit([&] { CK(cudaMemcpyAsync(d, s, bytes, cudaMemcpyDeviceToDevice, g_st)); }, bytes));
    CK(cudaFree(s));
    CK(cudaFree(d));
  }
  return 0;
}
