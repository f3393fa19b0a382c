// Direct-write exchange engine: alltoall(v) (K5), allgatherv (K6), gatherv
// (K7), bcast (K8, push variant) and the 0-byte barrier, all as one kernel
// over per-peer (pointer, bytes) spans.
//
// Reference algorithms being replaced (collectives.py):
//   _alltoall_pairwise/_naive/_bruck + _BlockView   :648-733
//   _allgather_ring/_bruck/_naive + _gather_counts   :446-512
//   _gather_linear                                   :515-525
//   _bcast_linear/_binomial                          :418-443
//   pairwise count cross-check in _cross_check       :229-241
// NVSwitch gives every pair full bandwidth, so there is no ring/tree
// schedule: every rank writes its chunk for peer j straight into j's
// workspace slot `rank` over NVLink, raises one flag per (block, pair), and
// the receiver lands the slot into its output. Pairs larger than a slot move
// in rounds, the receiver acknowledging each round (bounded workspace, any
// message size). Counts may live in device memory (MoE routing) and are
// read by the kernel itself.
#include <algorithm>

#include "internal.h"

namespace mcrdl {

struct XArgs {
  const uint8_t* sptr[kMaxRanks];
  int64_t sbytes[kMaxRanks];
  uint8_t* rptr[kMaxRanks];
  int64_t rbytes[kMaxRanks];
  const int64_t* d_counts;  // [scounts | sdispls | rcounts | rdispls] in elements, or null
  const uint8_t* in_base;
  uint8_t* out_base;
  int64_t in_count;   // element capacity of in/out (device-count bounds check)
  int64_t out_count;
  int64_t slot;
  int esize;
  int gmax;
  uint32_t sig_base;
};

constexpr int64_t kPairCtaBytes = 64 << 10;  // one CTA per 64 KiB of a pair

__device__ __forceinline__ int64_t rounds_for(int64_t bytes, int64_t slot) {
  return bytes <= slot ? 1 : (bytes + slot - 1) / slot;
}
__device__ __forceinline__ uint32_t pair_sig(uint32_t base, int64_t bytes) {
  return mix32(base, uint64_t(bytes)) & 0xFFFFFu;
}

// CTAs that serve one pair: a function of the pair's byte count only, so the
// sender (which knows its scount) and the receiver (its rcount) partition the
// pair identically without exchanging anything. Capped by gmax, a
// communicator-wide constant.
__device__ __host__ __forceinline__ int pair_ctas(int64_t bytes, int gmax) {
  int64_t g = (bytes + kPairCtaBytes - 1) / kPairCtaBytes;
  if (g < 1) g = 1;
  if (g > gmax) g = gmax;
  return int(g);
}

__global__ void __launch_bounds__(kThreads) k_exchange(DevComm c, XArgs a, uint32_t epoch) {
  __shared__ const uint8_t* s_sp[kMaxRanks];
  __shared__ uint8_t* s_rp[kMaxRanks];
  __shared__ int64_t s_sb[kMaxRanks];
  __shared__ int64_t s_rb[kMaxRanks];
  __shared__ int s_gs[kMaxRanks];
  __shared__ int s_gr[kMaxRanks];
  __shared__ int s_err;
  __shared__ SComm S;
  const int par = epoch & 1, rank = c.rank, world = c.world;
  const int b = blockIdx.x, G = gridDim.x, tid = threadIdx.x;
  const int64_t hoff = int64_t(par) * c.half_bytes;
  const int64_t slot = a.slot;
  if (tid == 0) s_err = 0;
  stage_comm(c, S);
  if (tid < world) {
    if (a.d_counts != nullptr) {
      const int64_t sc = a.d_counts[tid], sd = a.d_counts[world + tid];
      const int64_t rc = a.d_counts[2 * world + tid], rd = a.d_counts[3 * world + tid];
      s_sp[tid] = a.in_base + sd * a.esize;
      s_sb[tid] = sc * a.esize;
      s_rp[tid] = a.out_base + rd * a.esize;
      s_rb[tid] = rc * a.esize;
      if (sc < 0 || sd < 0 || rc < 0 || rd < 0 || (sd + sc) > a.in_count ||
          (rd + rc) > a.out_count)
        s_err = MCRDL_ERR_VALIDATION;
    } else {
      s_sp[tid] = a.sptr[tid];
      s_sb[tid] = a.sbytes[tid];
      s_rp[tid] = a.rptr[tid];
      s_rb[tid] = a.rbytes[tid];
    }
    s_gs[tid] = pair_ctas(s_sb[tid], a.gmax);
    s_gr[tid] = pair_ctas(s_rb[tid], a.gmax);
  }
  __syncthreads();
  if (tid == 0 && s_sb[rank] != s_rb[rank]) s_err = MCRDL_ERR_VALIDATION;
  __syncthreads();
  if (s_err) {
    if (tid == 0) raise_error(S.pad, world, c.err, s_err, epoch);
    return;
  }

  // Rounds this CTA takes part in (block-uniform).
  int64_t rmax = 0;
  for (int j = 0; j < world; ++j) {
    if (j == rank) continue;
    if (b < s_gs[j]) rmax = max(rmax, rounds_for(s_sb[j], slot));
    if (b < s_gr[j]) rmax = max(rmax, rounds_for(s_rb[j], slot));
  }

  // Local segment: straight copy over every launched CTA, no workspace
  // (skipped when in place).
  {
    int64_t s, e;
    byte_share(s_sb[rank], b, G, s, e);
    block_copy<4>(s_rp[rank] + s, s_sp[rank] + s, e - s);
  }

  const uint8_t* my_ws = S.ws[rank] + hoff;
  for (int64_t t = 0; t < rmax; ++t) {
    // Slot reuse: wait until receiver j consumed round t-1.
    if (t > 0) {
      if (tid < world && tid != rank && b < s_gs[tid] && t < rounds_for(s_sb[tid], slot)) {
        int e = wait_flag(&S.pad[rank]->ack[par][b][tid], S.pad[rank], c.timeout_ns, epoch,
                          pair_sig(a.sig_base, s_sb[tid]), uint32_t(t - 1));
        if (e) atomicCAS(&s_err, 0, e);
      }
      __syncthreads();
      if (s_err) {
        if (tid == 0) raise_error(S.pad, world, c.err, s_err, epoch);
        return;
      }
    }
    // Send round t to every peer (rotated start spreads the traffic).
    for (int k = 1; k < world; ++k) {
      const int j = (rank + k) % world;
      if (b >= s_gs[j] || t >= rounds_for(s_sb[j], slot)) continue;
      const int64_t off = t * slot;
      const int64_t len = min(slot, s_sb[j] - off);
      int64_t s, e;
      byte_share(len, b, s_gs[j], s, e);
      block_copy<4>(S.ws[j] + hoff + int64_t(rank) * slot + s, s_sp[j] + off + s, e - s);
    }
    __syncthreads();
    if (tid < world && tid != rank && b < s_gs[tid] && t < rounds_for(s_sb[tid], slot))
      publish(&S.pad[tid]->flag[par][b][rank],
              make_flag(epoch, pair_sig(a.sig_base, s_sb[tid]), uint32_t(t)));
    if (tid < world && tid != rank && b < s_gr[tid] && t < rounds_for(s_rb[tid], slot)) {
      int e = wait_flag(&S.pad[rank]->flag[par][b][tid], S.pad[rank], c.timeout_ns, epoch,
                        pair_sig(a.sig_base, s_rb[tid]), uint32_t(t));
      if (e) atomicCAS(&s_err, 0, e);
    }
    __syncthreads();
    if (s_err) {
      if (tid == 0) raise_error(S.pad, world, c.err, s_err, epoch);
      return;
    }
    // Receive round t from every peer into the output.
    for (int k = 1; k < world; ++k) {
      const int i = (rank - k + world) % world;
      if (b >= s_gr[i] || t >= rounds_for(s_rb[i], slot)) continue;
      const int64_t off = t * slot;
      const int64_t len = min(slot, s_rb[i] - off);
      int64_t s, e;
      byte_share(len, b, s_gr[i], s, e);
      block_copy<4>(s_rp[i] + off + s, my_ws + int64_t(i) * slot + s, e - s);
    }
    if (t + 1 < rmax) {
      __syncthreads();
      if (tid < world && tid != rank && b < s_gr[tid] && t + 1 < rounds_for(s_rb[tid], slot))
        publish(&S.pad[tid]->ack[par][b][rank],
                make_flag(epoch, pair_sig(a.sig_base, s_rb[tid]), uint32_t(t)));
    }
  }
}

mcrdl_status_t launch_local_copy(void* dst, const void* src, int64_t nbytes, int num_sms,
                                 cudaStream_t stream);

mcrdl_status_t launch_exchange(mcrdl_comm* c, const ExchangeSpec& sp, int64_t total_hint,
                               cudaStream_t stream) {
  if (c->world == 1 && sp.d_counts == nullptr) {
    if (sp.sbytes[0] != sp.rbytes[0])
      return set_error(MCRDL_ERR_VALIDATION, "self segment: send %lld bytes, receive %lld bytes",
                       (long long)sp.sbytes[0], (long long)sp.rbytes[0]);
    return launch_local_copy(sp.rptr[0], sp.sptr[0], sp.sbytes[0], c->num_sms, stream);
  }
  uint32_t epoch;
  mcrdl_status_t st = begin_op(c, &epoch);
  if (st != MCRDL_OK) return st;
  XArgs a;
  memset(&a, 0, sizeof(a));
  for (int r = 0; r < c->world; ++r) {
    a.sptr[r] = sp.sptr[r];
    a.sbytes[r] = sp.sbytes[r];
    a.rptr[r] = sp.rptr[r];
    a.rbytes[r] = sp.rbytes[r];
  }
  a.d_counts = sp.d_counts;
  a.in_base = sp.in_base;
  a.out_base = sp.out_base;
  a.esize = sp.esize;
  a.sig_base = sp.sig_base;
  a.slot = c->dc.half_bytes / c->world / 256 * 256;
  a.in_count = sp.in_count;
  a.out_count = sp.out_count;
  a.gmax = 2 * c->num_sms < kMaxBlocks ? 2 * c->num_sms : kMaxBlocks;
  // Grid: enough CTAs for the widest pair (pairs agree on their own CTA
  // count, see pair_ctas); device-resident counts are unknown here -> gmax.
  int64_t g = 1;
  if (sp.d_counts != nullptr) {
    g = a.gmax;
  } else {
    for (int r = 0; r < c->world; ++r) {
      g = std::max<int64_t>(g, pair_ctas(sp.sbytes[r], a.gmax));
      g = std::max<int64_t>(g, pair_ctas(sp.rbytes[r], a.gmax));
    }
  }
  (void)total_hint;
  k_exchange<<<int(g), kThreads, 0, stream>>>(c->dc, a, epoch);
  count_launch();
  MCRDL_CUDA_CHECK(cudaGetLastError());
  return MCRDL_OK;
}

static bool check_counts(const int64_t* counts, const int64_t* displs, int world, const char* what) {
  for (int r = 0; r < world; ++r) {
    if (counts[r] < 0 || displs[r] < 0) {
      set_error(MCRDL_ERR_VALIDATION, "%s: counts and displacements must be >= 0", what);
      return false;
    }
  }
  return true;
}

static ExchangeSpec empty_spec(int esize, uint32_t sig_base) {
  ExchangeSpec s;
  memset(&s, 0, sizeof(s));
  s.esize = esize;
  s.sig_base = sig_base;
  return s;
}

}  // namespace mcrdl

using namespace mcrdl;

extern "C" {

mcrdl_status_t mcrdl_all_to_allv(mcrdl_comm* c, const void* in, void* out, const int64_t* scounts,
                                 const int64_t* sdispls, const int64_t* rcounts,
                                 const int64_t* rdispls, mcrdl_dtype_t dtype, mcrdl_algo_t algo,
                                 uint64_t seq, void* stream) {
  (void)algo;
  if (c == nullptr) return set_error(MCRDL_ERR_NOT_INITIALIZED, "communicator is NULL");
  const int es = elem_size(dtype);
  if (es == 0) return set_error(MCRDL_ERR_VALIDATION, "unknown dtype %d", int(dtype));
  if (!check_counts(scounts, sdispls, c->world, "scounts") ||
      !check_counts(rcounts, rdispls, c->world, "rcounts"))
    return MCRDL_ERR_VALIDATION;
  if (in == out) {
    for (int r = 0; r < c->world; ++r)
      if (scounts[r] != rcounts[r] || sdispls[r] != rdispls[r])
        return set_error(MCRDL_ERR_VALIDATION,
                         "in-place all_to_allv needs identical send/recv layouts (snapshot the input)");
  }
  ExchangeSpec s = empty_spec(es, op_sig(kKindA2AV, dtype, 0, -1, 0, seq));
  int64_t ts = 0, tr = 0;
  for (int r = 0; r < c->world; ++r) {
    s.sptr[r] = reinterpret_cast<const uint8_t*>(in) + sdispls[r] * es;
    s.sbytes[r] = scounts[r] * es;
    s.rptr[r] = reinterpret_cast<uint8_t*>(out) + rdispls[r] * es;
    s.rbytes[r] = rcounts[r] * es;
    ts += s.sbytes[r];
    tr += s.rbytes[r];
  }
  return launch_exchange(c, s, ts > tr ? ts : tr, reinterpret_cast<cudaStream_t>(stream));
}

mcrdl_status_t mcrdl_all_to_allv_dev(mcrdl_comm* c, const void* in, uint64_t in_count, void* out,
                                     uint64_t out_count, const int64_t* d_counts,
                                     mcrdl_dtype_t dtype, mcrdl_algo_t algo,
                                     uint64_t seq, void* stream) {
  (void)algo;
  if (c == nullptr) return set_error(MCRDL_ERR_NOT_INITIALIZED, "communicator is NULL");
  const int es = elem_size(dtype);
  if (es == 0) return set_error(MCRDL_ERR_VALIDATION, "unknown dtype %d", int(dtype));
  if (d_counts == nullptr) return set_error(MCRDL_ERR_VALIDATION, "NULL device count array");
  ExchangeSpec s = empty_spec(es, op_sig(kKindA2AV, dtype, 0, -1, 0, seq));
  s.d_counts = d_counts;
  s.in_base = reinterpret_cast<const uint8_t*>(in);
  s.out_base = reinterpret_cast<uint8_t*>(out);
  s.in_count = int64_t(in_count);
  s.out_count = int64_t(out_count);
  return launch_exchange(c, s, -1, reinterpret_cast<cudaStream_t>(stream));
}

mcrdl_status_t mcrdl_all_to_all_single(mcrdl_comm* c, const void* in, void* out, uint64_t count,
                                       mcrdl_dtype_t dtype, mcrdl_algo_t algo, uint64_t seq,
                                       void* stream) {
  (void)algo;
  if (c == nullptr) return set_error(MCRDL_ERR_NOT_INITIALIZED, "communicator is NULL");
  const int es = elem_size(dtype);
  if (es == 0) return set_error(MCRDL_ERR_VALIDATION, "unknown dtype %d", int(dtype));
  if (count % uint64_t(c->world) != 0)
    return set_error(MCRDL_ERR_VALIDATION, "count %llu not divisible by %d",
                     (unsigned long long)count, c->world);
  const int64_t m = int64_t(count) / c->world;
  ExchangeSpec s = empty_spec(es, op_sig(kKindA2ASingle, dtype, 0, -1, uint64_t(m), seq));
  for (int r = 0; r < c->world; ++r) {
    s.sptr[r] = reinterpret_cast<const uint8_t*>(in) + r * m * es;
    s.sbytes[r] = m * es;
    s.rptr[r] = reinterpret_cast<uint8_t*>(out) + r * m * es;
    s.rbytes[r] = m * es;
  }
  return launch_exchange(c, s, int64_t(count) * es, reinterpret_cast<cudaStream_t>(stream));
}

mcrdl_status_t mcrdl_all_to_all_ptrs(mcrdl_comm* c, const void* const* in_ptrs,
                                     const int64_t* in_counts, void* const* out_ptrs,
                                     const int64_t* out_counts, mcrdl_dtype_t dtype,
                                     mcrdl_algo_t algo, uint64_t seq, void* stream) {
  (void)algo;
  if (c == nullptr) return set_error(MCRDL_ERR_NOT_INITIALIZED, "communicator is NULL");
  const int es = elem_size(dtype);
  if (es == 0) return set_error(MCRDL_ERR_VALIDATION, "unknown dtype %d", int(dtype));
  ExchangeSpec s = empty_spec(es, op_sig(kKindA2AList, dtype, 0, -1, 0, seq));
  int64_t ts = 0, tr = 0;
  for (int r = 0; r < c->world; ++r) {
    if (in_counts[r] < 0 || out_counts[r] < 0)
      return set_error(MCRDL_ERR_VALIDATION, "negative block count");
    s.sptr[r] = reinterpret_cast<const uint8_t*>(in_ptrs[r]);
    s.sbytes[r] = in_counts[r] * es;
    s.rptr[r] = reinterpret_cast<uint8_t*>(out_ptrs[r]);
    s.rbytes[r] = out_counts[r] * es;
    ts += s.sbytes[r];
    tr += s.rbytes[r];
  }
  return launch_exchange(c, s, ts > tr ? ts : tr, reinterpret_cast<cudaStream_t>(stream));
}

mcrdl_status_t mcrdl_all_gatherv(mcrdl_comm* c, const void* in, void* out, const int64_t* rcounts,
                                 const int64_t* displs, mcrdl_dtype_t dtype, mcrdl_algo_t algo,
                                 uint64_t seq, void* stream) {
  (void)algo;
  if (c == nullptr) return set_error(MCRDL_ERR_NOT_INITIALIZED, "communicator is NULL");
  const int es = elem_size(dtype);
  if (es == 0) return set_error(MCRDL_ERR_VALIDATION, "unknown dtype %d", int(dtype));
  if (!check_counts(rcounts, displs, c->world, "rcounts")) return MCRDL_ERR_VALIDATION;
  ExchangeSpec s = empty_spec(es, op_sig(kKindAllGatherv, dtype, 0, -1, 0, seq));
  int64_t total = 0;
  for (int r = 0; r < c->world; ++r) {
    s.sptr[r] = reinterpret_cast<const uint8_t*>(in);
    s.sbytes[r] = rcounts[c->rank] * es;
    s.rptr[r] = reinterpret_cast<uint8_t*>(out) + displs[r] * es;
    s.rbytes[r] = rcounts[r] * es;
    total += s.rbytes[r];
  }
  return launch_exchange(c, s, total, reinterpret_cast<cudaStream_t>(stream));
}

mcrdl_status_t mcrdl_gatherv(mcrdl_comm* c, const void* in, void* out, const int64_t* rcounts,
                             const int64_t* displs, int root, mcrdl_dtype_t dtype, mcrdl_algo_t algo,
                             uint64_t seq, void* stream) {
  (void)algo;
  if (c == nullptr) return set_error(MCRDL_ERR_NOT_INITIALIZED, "communicator is NULL");
  const int es = elem_size(dtype);
  if (es == 0) return set_error(MCRDL_ERR_VALIDATION, "unknown dtype %d", int(dtype));
  if (root < 0 || root >= c->world)
    return set_error(MCRDL_ERR_VALIDATION, "root %d outside world %d", root, c->world);
  if (!check_counts(rcounts, displs, c->world, "rcounts")) return MCRDL_ERR_VALIDATION;
  if (c->rank == root && out == nullptr && rcounts[root] > 0)
    return set_error(MCRDL_ERR_VALIDATION, "root must supply the output buffer");
  ExchangeSpec s = empty_spec(es, op_sig(kKindGatherv, dtype, 0, root, 0, seq));
  int64_t total = 0;
  if (c->rank == root) {
    for (int r = 0; r < c->world; ++r) {
      s.rptr[r] = reinterpret_cast<uint8_t*>(out) + displs[r] * es;
      s.rbytes[r] = rcounts[r] * es;
      total += s.rbytes[r];
    }
    s.sptr[root] = reinterpret_cast<const uint8_t*>(in);
    s.sbytes[root] = rcounts[root] * es;
  } else {
    s.sptr[root] = reinterpret_cast<const uint8_t*>(in);
    s.sbytes[root] = rcounts[c->rank] * es;
    total = s.sbytes[root];
  }
  return launch_exchange(c, s, total, reinterpret_cast<cudaStream_t>(stream));
}

mcrdl_status_t mcrdl_bcast(mcrdl_comm* c, void* buf, uint64_t count, mcrdl_dtype_t dtype, int root,
                           mcrdl_algo_t algo, uint64_t seq, void* stream) {
  (void)algo;
  if (c == nullptr) return set_error(MCRDL_ERR_NOT_INITIALIZED, "communicator is NULL");
  const int es = elem_size(dtype);
  if (es == 0) return set_error(MCRDL_ERR_VALIDATION, "unknown dtype %d", int(dtype));
  if (root < 0 || root >= c->world)
    return set_error(MCRDL_ERR_VALIDATION, "root %d outside world %d", root, c->world);
  if (c->world == 1) return MCRDL_OK;
  ExchangeSpec s = empty_spec(es, op_sig(kKindBcast, dtype, 0, root, count, seq));
  const int64_t nb = int64_t(count) * es;
  if (c->rank == root) {
    for (int r = 0; r < c->world; ++r) {
      if (r == root) continue;
      s.sptr[r] = reinterpret_cast<const uint8_t*>(buf);
      s.sbytes[r] = nb;
    }
  } else {
    s.rptr[root] = reinterpret_cast<uint8_t*>(buf);
    s.rbytes[root] = nb;
  }
  return launch_exchange(c, s, nb, reinterpret_cast<cudaStream_t>(stream));
}

mcrdl_status_t mcrdl_barrier(mcrdl_comm* c, uint64_t seq, void* stream) {
  if (c == nullptr) return set_error(MCRDL_ERR_NOT_INITIALIZED, "communicator is NULL");
  if (c->world == 1) return MCRDL_OK;
  ExchangeSpec s = empty_spec(1, op_sig(kKindBarrier, 0, 0, -1, 0, seq));
  return launch_exchange(c, s, 0, reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
