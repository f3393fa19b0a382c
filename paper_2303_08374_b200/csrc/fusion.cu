// Tensor-fusion pack / unpack (K9 building blocks).
//
// Reference: FusionManager._flush_locked concatenates member snapshots with
// np.concatenate (middleware.py:316) and _scatter_back copies each member's
// slice out again (middleware.py:329-341). On the device both are one launch
// over a segment table; the fused all_reduce (allreduce.cu, k_ar_fused)
// removes them from the hot path for groups whose one-shot slots fit a
// workspace half; larger groups (nvl/backend.py post_fused) pack, run the
// two-shot / NVLS all_reduce on the packed buffer, and unpack.
#include "internal.h"

namespace mcrdl {

// CTAs per member: members are at most one fusion buffer (FusionConfig B)
constexpr int kFusionCtasPerMember = 32;

// grid.y = segment, grid.x = CTA share of that segment.
__global__ void __launch_bounds__(kThreads)
    k_pack(const uint8_t* const* src, const int64_t* nbytes, const int64_t* offs, uint8_t* dst) {
  const int m = blockIdx.y;
  int64_t s, e;
  byte_share(nbytes[m], blockIdx.x, gridDim.x, s, e);
  block_copy<4>(dst + offs[m] + s, src[m] + s, e - s);
}

__global__ void __launch_bounds__(kThreads)
    k_unpack(const uint8_t* src, uint8_t* const* dst, const int64_t* nbytes, const int64_t* offs) {
  const int m = blockIdx.y;
  int64_t s, e;
  byte_share(nbytes[m], blockIdx.x, gridDim.x, s, e);
  block_copy<4>(dst[m] + s, src + offs[m] + s, e - s);
}

}  // namespace mcrdl

using namespace mcrdl;

extern "C" {

mcrdl_status_t mcrdl_fusion_pack(const void* const* d_src_ptrs, const int64_t* d_nbytes,
                                 const int64_t* d_offsets, int n, void* dst, void* stream) {
  if (n <= 0) return MCRDL_OK;
  if (n > 65535) return set_error(MCRDL_ERR_VALIDATION, "too many fusion members (%d)", n);
  dim3 grid(kFusionCtasPerMember, n);
  k_pack<<<grid, kThreads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const uint8_t* const*>(d_src_ptrs), d_nbytes, d_offsets,
      reinterpret_cast<uint8_t*>(dst));
  count_launch();
  MCRDL_CUDA_CHECK(cudaGetLastError());
  return MCRDL_OK;
}

mcrdl_status_t mcrdl_fusion_unpack(const void* src, void* const* d_dst_ptrs, const int64_t* d_nbytes,
                                   const int64_t* d_offsets, int n, void* stream) {
  if (n <= 0) return MCRDL_OK;
  if (n > 65535) return set_error(MCRDL_ERR_VALIDATION, "too many fusion members (%d)", n);
  dim3 grid(kFusionCtasPerMember, n);
  k_unpack<<<grid, kThreads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const uint8_t*>(src), reinterpret_cast<uint8_t* const*>(d_dst_ptrs), d_nbytes,
      d_offsets);
  count_launch();
  MCRDL_CUDA_CHECK(cudaGetLastError());
  return MCRDL_OK;
}

}  // extern "C"
