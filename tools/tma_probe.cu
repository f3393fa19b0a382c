// TMA bulk-copy push bandwidth over NVLink (developer tool).
// GPU0 pushes 256 MiB into GPU1: local HBM --cp.async.bulk--> smem ring
// --cp.async.bulk (bulk_group)--> peer HBM, one elected thread per CTA driving
// a STAGES-deep pipeline. Compared with SM LD/ST push (p2p_probe.cu).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int STAGES, int CHUNK>
__global__ void __launch_bounds__(32) tma_push(uint8_t* dst, const uint8_t* src, long bytes) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar[STAGES];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < STAGES; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const long nchunks = bytes / CHUNK;
  uint32_t phase[STAGES];
  for (int s = 0; s < STAGES; ++s) phase[s] = 0;
  // chunks owned by this CTA: c = blockIdx.x + k * gridDim.x
  long issued = 0, done = 0;
  long my_total = 0;
  for (long c = blockIdx.x; c < nchunks; c += gridDim.x) ++my_total;
  auto chunk_of = [&](long k) { return long(blockIdx.x) + k * gridDim.x; };
  // prologue: fill the ring with loads
  for (; issued < my_total && issued < STAGES; ++issued) {
    const int s = int(issued % STAGES);
    const long c = chunk_of(issued);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&bar[s])),
                 "r"(CHUNK));
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(smem + s * CHUNK)),
        "l"(src + c * CHUNK), "r"(CHUNK), "r"(smem_addr(&bar[s]))
        : "memory");
  }
  for (; done < my_total; ++done) {
    const int s = int(done % STAGES);
    // wait for the load of chunk `done`
    uint32_t ok = 0;
    while (!ok) {
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(ok)
          : "r"(smem_addr(&bar[s])), "r"(phase[s])
          : "memory");
    }
    phase[s] ^= 1;
    const long c = chunk_of(done);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + c * CHUNK),
                 "r"(smem_addr(smem + s * CHUNK)), "r"(CHUNK)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (issued < my_total) {
      // the slot we refill is `s` (ring): its store must have read smem first
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      const long c2 = chunk_of(issued);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&bar[s])),
                   "r"(CHUNK));
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_addr(smem + s * CHUNK)),
          "l"(src + c2 * CHUNK), "r"(CHUNK), "r"(smem_addr(&bar[s]))
          : "memory");
      ++issued;
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int STAGES, int CHUNK>
float run(int grid, uint8_t* dst, const uint8_t* src, long bytes, cudaStream_t st) {
  const int smem = STAGES * CHUNK;
  CK(cudaFuncSetAttribute(tma_push<STAGES, CHUNK>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  tma_push<STAGES, CHUNK><<<grid, 32, smem, st>>>(dst, src, bytes);
  CK(cudaGetLastError());
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaEventRecord(a, st));
  for (int i = 0; i < 10; ++i) tma_push<STAGES, CHUNK><<<grid, 32, smem, st>>>(dst, src, bytes);
  CK(cudaEventRecord(b, st));
  CK(cudaEventSynchronize(b));
  float ms;
  CK(cudaEventElapsedTime(&ms, a, b));
  return bytes / (ms / 10) / 1e6;
}

int main() {
  const long bytes = 256l << 20;
  uint8_t *a0, *b0, *b1, *a1;
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&b1, bytes));
  CK(cudaMalloc(&a1, bytes));
  CK(cudaMemset(a1, 9, bytes));
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaMalloc(&a0, bytes));
  CK(cudaMalloc(&b0, bytes));
  CK(cudaMemset(a0, 7, bytes));
  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  int grids[] = {8, 16, 32, 64, 148, 296};
  for (int g : grids) {
    printf("grid %3d: push 4x32K %6.1f  4x48K %6.1f  6x32K %6.1f  3x64K %6.1f GB/s | local 4x32K %7.1f GB/s\n", g,
           run<4, 32768>(g, b1, a0, bytes, st), run<4, 49152>(g, b1, a0, bytes, st),
           run<6, 32768>(g, b1, a0, bytes, st), run<3, 65536>(g, b1, a0, bytes, st),
           2 * run<4, 32768>(g, b0, a0, bytes, st));
  }
  for (int g : grids) {  // pull: GPU0 reads GPU1's buffer into its own memory
    printf("grid %3d: pull 4x32K %6.1f  3x64K %6.1f GB/s\n", g, run<4, 32768>(g, b0, a1, bytes, st),
           run<3, 65536>(g, b0, a1, bytes, st));
  }
  // bidirectional pull (both GPUs pull from each other at once)
  {
    cudaStream_t st1;
    CK(cudaSetDevice(1));
    CK(cudaDeviceEnablePeerAccess(0, 0));
    CK(cudaStreamCreate(&st1));
    const int smem = 4 * 32768;
    CK(cudaFuncSetAttribute(tma_push<4, 32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaSetDevice(0));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaEventRecord(a, st));
    for (int i = 0; i < 10; ++i) tma_push<4, 32768><<<148, 32, smem, st>>>(b0, a1, bytes);
    CK(cudaEventRecord(b, st));
    CK(cudaSetDevice(1));
    for (int i = 0; i < 10; ++i) tma_push<4, 32768><<<148, 32, smem, st1>>>(b1, a0, bytes);
    CK(cudaSetDevice(0));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    printf("bidir pull grid 148: %6.1f GB/s per direction\n", bytes / (ms / 10) / 1e6);
    CK(cudaSetDevice(1));
    CK(cudaStreamSynchronize(st1));
    CK(cudaSetDevice(0));
  }
  // verify a copy
  CK(cudaMemset(b0, 0, bytes));
  run<4, 32768>(148, b0, a0, bytes, st);
  uint8_t h[16];
  CK(cudaMemcpy(h, b0 + bytes - 16, 16, cudaMemcpyDeviceToHost));
  printf("verify last byte: %d (expect 7)\n", h[15]);
  return 0;
}
