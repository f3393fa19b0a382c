// NVLS (NVLink SHARP multicast) throughput probe (developer tool).
// One process drives all visible GPUs (one stream each). Every GPU owns a
// S-byte buffer bound to one multicast object; GPU d reduces shard d with
// multimem.ld_reduce and broadcasts it with multimem.st: the reduce-scatter +
// all-gather core of the NVLS all_reduce with no staging copies. Also times
// the two halves alone and a local HBM copy for reference.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/nvls_probe tools/nvls_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s (line %d)\n", #x, cudaGetErrorString(e), __LINE__); exit(1);} } while (0)
#define DK(x) do { CUresult e = (x); if (e != CUDA_SUCCESS) { const char* s; cuGetErrorString(e, &s); printf("%s: %s (line %d)\n", #x, s, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint4 ld_reduce(const void* p) {
  uint4 r;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ void mst(void* p, const uint4& v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// mode 0: ld_reduce + st (same address); 1: ld_reduce -> local; 2: local -> st
template <int U>
__global__ void __launch_bounds__(512) k_nvls(int mode, uint8_t* mc, uint8_t* uc_other, int64_t n16) {
  const int64_t nt = int64_t(gridDim.x) * blockDim.x;
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * nt < n16; i += U * nt) {
    uint4 v[U];
    if (mode == 2) {
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = reinterpret_cast<const uint4*>(uc_other)[i + u * nt];
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ld_reduce(mc + (i + u * nt) * 16);
    }
    if (mode == 1) {
#pragma unroll
      for (int u = 0; u < U; ++u) reinterpret_cast<uint4*>(uc_other)[i + u * nt] = v[u];
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u) mst(mc + (i + u * nt) * 16, v[u]);
    }
  }
  for (; i < n16; i += nt) {
    uint4 v = mode == 2 ? reinterpret_cast<const uint4*>(uc_other)[i] : ld_reduce(mc + i * 16);
    if (mode == 1) reinterpret_cast<uint4*>(uc_other)[i] = v; else mst(mc + i * 16, v);
  }
}

__global__ void k_fill(float* p, int64_t n, float v) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) p[i] = v;
}

typedef void (*KFn)(int, uint8_t*, uint8_t*, int64_t);

int main(int argc, char** argv) {
  int N = 0;
  CK(cudaGetDeviceCount(&N));
  const int64_t S = (argc > 1 ? atoll(argv[1]) : 256) << 20;  // MiB per GPU buffer
  printf("devices=%d S=%lld MiB\n", N, (long long)(S >> 20));
  DK(cuInit(0));
  std::vector<CUdevice> dev(N);
  for (int d = 0; d < N; ++d) { CK(cudaSetDevice(d)); CK(cudaFree(0)); DK(cuDeviceGet(&dev[d], d)); }
  CUmulticastObjectProp mp;
  memset(&mp, 0, sizeof(mp));
  mp.numDevices = N;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  mp.size = S;
  DK(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  const size_t bytes = (S + gran - 1) / gran * gran;
  mp.size = bytes;
  CUmemGenericAllocationHandle mc;
  DK(cuMulticastCreate(&mc, &mp));
  for (int d = 0; d < N; ++d) DK(cuMulticastAddDevice(mc, dev[d]));
  std::vector<CUmemGenericAllocationHandle> mem(N);
  std::vector<uint8_t*> mcva(N), ucva(N), scratch(N);
  for (int d = 0; d < N; ++d) {
    CK(cudaSetDevice(d));
    CUmemAllocationProp ap;
    memset(&ap, 0, sizeof(ap));
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = d;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    DK(cuMemCreate(&mem[d], bytes, &ap, 0));
    DK(cuMulticastBindMem(mc, 0, mem[d], 0, bytes, 0));
  }
  for (int d = 0; d < N; ++d) {
    CK(cudaSetDevice(d));
    CUmemAccessDesc ad;
    memset(&ad, 0, sizeof(ad));
    ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ad.location.id = d;
    ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CUdeviceptr a;
    DK(cuMemAddressReserve(&a, bytes, gran, 0, 0));
    DK(cuMemMap(a, bytes, 0, mc, 0));
    DK(cuMemSetAccess(a, bytes, &ad, 1));
    mcva[d] = reinterpret_cast<uint8_t*>(a);
    DK(cuMemAddressReserve(&a, bytes, gran, 0, 0));
    DK(cuMemMap(a, bytes, 0, mem[d], 0));
    DK(cuMemSetAccess(a, bytes, &ad, 1));
    ucva[d] = reinterpret_cast<uint8_t*>(a);
    CK(cudaMalloc(&scratch[d], bytes));
    k_fill<<<1024, 256>>>(reinterpret_cast<float*>(ucva[d]), int64_t(bytes / 4), float(d + 1));
    CK(cudaDeviceSynchronize());
  }
  std::vector<cudaStream_t> st(N);
  std::vector<cudaEvent_t> e0(N), e1(N);
  for (int d = 0; d < N; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[d]));
    CK(cudaEventCreate(&e1[d]));
  }
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int64_t shard16 = int64_t(bytes) / 16 / N;
  struct V { const char* name; int mode; int u; KFn fn; };
  V vs[] = {{"rsag", 0, 1, k_nvls<1>}, {"rsag", 0, 2, k_nvls<2>}, {"rsag", 0, 4, k_nvls<4>},
            {"rsag", 0, 8, k_nvls<8>}, {"ldred", 1, 4, k_nvls<4>}, {"ldred", 1, 8, k_nvls<8>},
            {"st", 2, 4, k_nvls<4>}, {"st", 2, 8, k_nvls<8>}};
  const int grids[] = {sms / 2, sms, 2 * sms, 3 * sms, 4 * sms};
  printf("%-6s %2s %5s %9s %10s %10s %12s\n", "mode", "U", "grid", "ms", "algbw", "busbw", "link_GB/s");
  for (const V& v : vs) {
    for (int g : grids) {
      float best = 1e30f;
      for (int it = 0; it < 4; ++it) {
        for (int d = 0; d < N; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
        for (int d = 0; d < N; ++d) {
          CK(cudaSetDevice(d));
          CK(cudaEventRecord(e0[d], st[d]));
          v.fn<<<g, 512, 0, st[d]>>>(v.mode, mcva[d] + int64_t(d) * shard16 * 16, scratch[d], shard16);
          CK(cudaEventRecord(e1[d], st[d]));
        }
        float mx = 0;
        for (int d = 0; d < N; ++d) {
          CK(cudaSetDevice(d));
          CK(cudaEventSynchronize(e1[d]));
          float ms;
          CK(cudaEventElapsedTime(&ms, e0[d], e1[d]));
          mx = std::max(mx, ms);
        }
        if (it > 0) best = std::min(best, mx);
      }
      // rsag moves the whole all_reduce of `bytes`; per-GPU link egress =
      // bytes (switch reads of every shard copy) + bytes/N (own shard st)
      const double sec = best * 1e-3;
      const double alg = double(bytes) / sec / 1e9;
      const double bus = alg * 2.0 * (N - 1) / N;
      const double link = v.mode == 0 ? double(bytes) * (1.0 + 1.0 / N) / sec / 1e9
                                      : double(bytes) / sec / 1e9;
      printf("%-6s %2d %5d %9.4f %10.1f %10.1f %12.1f\n", v.name, v.u, g, best, alg, bus, link);
    }
  }
  // single-source multicast store: only GPU 0 stores the WHOLE buffer (the
  // NVLS bcast root's egress); others idle
  for (int g : grids) {
    float best = 1e30f;
    for (int it = 0; it < 4; ++it) {
      for (int d = 0; d < N; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
      CK(cudaSetDevice(0));
      CK(cudaEventRecord(e0[0], st[0]));
      k_nvls<4><<<g, 512, 0, st[0]>>>(2, mcva[0], scratch[0], int64_t(bytes) / 16);
      CK(cudaEventRecord(e1[0], st[0]));
      CK(cudaEventSynchronize(e1[0]));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0[0], e1[0]));
      if (it > 0) best = std::min(best, ms);
    }
    printf("st1    %2d %5d %9.4f  root egress %8.1f GB/s\n", 4, g, best, double(bytes) / (best * 1e-3) / 1e9);
  }
  // sanity: after rsag, every element = sum(d+1) * (#rsag iterations) ... just check finite
  CK(cudaSetDevice(0));
  float h = 0;
  CK(cudaMemcpy(&h, ucva[0], 4, cudaMemcpyDeviceToHost));
  printf("ucva[0][0]=%g\n", h);
  return 0;
}
