// Zero-copy exchange into symmetric outputs: all_to_all_single and
// all_gather(v) whose output lies in a user symmetric allocation
// (mcrdl_symm_alloc, same offset on every rank). Every receiver's placement is
// known to every sender (fixed blocks / common displacements), so sender CTAs
// store straight into the peers' output buffers over NVLink — no workspace
// slot, no receiver copy-out. Per-CTA entry barrier (a rank's output is not
// written before that rank's previous work ended) and exit barrier (all data
// destined to me landed) as in k_ar_symm (allreduce.cu).
// Reference: _alltoall_* (collectives.py:648-733), _allgather_* (:446-512).
#include <algorithm>
#include <cstring>

#include "internal.h"

namespace mcrdl {

struct XSymmArgs {
  const uint8_t* src[kMaxRanks];  // what this rank sends to rank q
  uint8_t* dst[kMaxRanks];        // where it lands (rank q's output, mapped here)
  int64_t bytes[kMaxRanks];
};

__device__ __forceinline__ void x_symm_body(DevComm c, const XSymmArgs& a, uint32_t epoch,
                                            uint32_t sig) {
  __shared__ int s_err;
  __shared__ SComm S;
  __shared__ const uint8_t* s_src[kMaxRanks];
  __shared__ uint8_t* s_dst[kMaxRanks];
  __shared__ int64_t s_b[kMaxRanks];
  const int par = epoch & 1, rank = c.rank, world = c.world;
  const int s = int(blockIdx.x), G = int(gridDim.x), tid = threadIdx.x;
  if (tid == 0) s_err = 0;
  if (tid < kMaxRanks) {
    s_src[tid] = a.src[tid];
    s_dst[tid] = a.dst[tid];
    s_b[tid] = a.bytes[tid];
  }
  stage_comm(c, S);
  __syncthreads();
  if (tid < world) publish(&S.pad[tid]->flag[par][s][rank], make_flag(epoch, sig, 1));
  if (tid < world) {
    int e = wait_flag(&S.pad[rank]->flag[par][s][tid], S.pad[rank], c.timeout_ns, c.err, epoch, sig, 1);
    if (e) atomicCAS(&s_err, 0, e);
  }
  __syncthreads();
  if (s_err) {
    if (tid == 0) raise_error(S.pad, world, c.err, s_err, epoch);
    return;
  }
  for (int k = 0; k < world; ++k) {  // own block last-but-not-special: k = 0 is self
    const int q = (rank + k) % world;
    int64_t lo, hi;
    byte_share(s_b[q], s, G, lo, hi);
    block_copy<8>(s_dst[q] + lo, s_src[q] + lo, hi - lo);
  }
  __syncthreads();
  if (tid < world) publish(&S.pad[tid]->flag2[par][s][rank], make_flag(epoch, sig, 1));
  if (tid < world) {
    int e = wait_flag(&S.pad[rank]->flag2[par][s][tid], S.pad[rank], c.timeout_ns, c.err, epoch,
                      sig, 1);
    if (e) atomicCAS(&s_err, 0, e);
  }
  __syncthreads();
  if (s_err && tid == 0) raise_error(S.pad, world, c.err, s_err, epoch);
}

__global__ void __launch_bounds__(kThreads) k_x_symm(DevComm c, XSymmArgs a, uint32_t sig) {
  const uint32_t epoch = epoch_enter(c);
  x_symm_body(c, a, epoch, sig);
  epoch_exit(c, epoch);
}

// `send_off[q]`/`recv_off[q]`: byte offsets of the block this rank sends to q
// (in `in`) and of where it lands in q's output; bytes[q] its size. Returns
// true (and *st) when `out` is symmetric and the zero-copy kernel took the op.
bool try_exchange_symm(mcrdl_comm* c, const void* in, void* out, uint64_t out_bytes,
                       const int64_t* send_off, const int64_t* recv_off, const int64_t* bytes,
                       int64_t grid_bytes, uint32_t sig, cudaStream_t stream, mcrdl_status_t* st) {
  static const int64_t on = env_int("MCRDL_SYMM", 1);
  if (!on || c->world == 1 || out == nullptr) return false;
  uint64_t oo = 0;
  const Region* ro = find_symm(c, out, out_bytes, &oo);
  if (ro == nullptr) return false;
  XSymmArgs a{};
  for (int q = 0; q < c->world; ++q) {
    a.src[q] = static_cast<const uint8_t*>(in) + send_off[q];
    a.dst[q] = reinterpret_cast<uint8_t*>(ro->ptr[q]) + oo + recv_off[q];
    a.bytes[q] = bytes[q];
  }
  // the output offset is part of the agreement (ranks passing different
  // slices of the symmetric allocation fail with ORDER_MISMATCH)
  sig = mix32(sig, oo) & ~kSigCodecBit;
  if ((*st = begin_op(c, stream)) != MCRDL_OK) return true;
  // grid from a size EVERY rank agrees on (the per-CTA barriers pair CTA s
  // of every rank with CTA s of every peer)
  int64_t g = (grid_bytes + (32 << 10) - 1) / (32 << 10);
  g = std::max<int64_t>(1, std::min<int64_t>(g, c->num_sms));
  k_x_symm<<<int(g), kThreads, 0, stream>>>(c->dc, a, sig);
  count_launch();
  *st = cudaGetLastError() == cudaSuccess ? MCRDL_OK
                                           : set_error(MCRDL_ERR_CUDA, "k_x_symm launch failed");
  return true;
}

}  // namespace mcrdl
