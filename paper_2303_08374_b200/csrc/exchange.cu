// Direct-write exchange engine: alltoall(v) (K5), allgatherv (K6), gatherv
// (K7), scatter(v), bcast (K8, push variant) and the 0-byte barrier — one
// kernel over per-peer (pointer, bytes) spans.
//
// Reference algorithms being replaced (collectives.py):
//   _alltoall_pairwise/_naive/_bruck + _BlockView   :648-733
//   _allgather_ring/_bruck/_naive + _gather_counts   :446-512
//   _gather_linear                                   :515-525
//   _bcast_linear/_binomial                          :418-443
//   pairwise count cross-check in _cross_check       :229-241
// NVSwitch gives every pair full bandwidth, so there is no ring/tree
// schedule. The grid is split into two roles that run concurrently:
//   sender CTAs   [0, Gp)    push share s of every outgoing pair into the
//                            peer's workspace slot `rank`, one release flag
//                            per 64 KiB chunk;
//   receiver CTAs [Gp, 2Gp)  copy their share of the local segment, then land
//                            each incoming chunk as soon as its flag arrives.
// So the NVLink push, the local copy and the copy-out overlap; senders never
// wait except for slot reuse (pairs larger than a workspace slot move in
// rounds the receiver acknowledges), so forward progress does not depend on
// CTA co-residency. Pairs agree on their geometry from their own byte count
// (sender: scount, receiver: rcount) — no extra exchange.
#include <algorithm>
#include <cstring>

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
  int64_t in_count;  // element capacity of in/out (device-count bounds check)
  int64_t out_count;
  int64_t slot;      // workspace bytes per (sender) slot per round
  int esize;
  int gmax;          // communicator-wide cap on CTAs per pair
  int gp;            // CTAs per role in this launch
  uint32_t sig_base;
};

constexpr int64_t kPairCtaBytes = 32 << 10;   // one CTA per 32 KiB of a pair
constexpr int64_t kChunkBytes = 256 << 10;    // flag granularity inside a share
constexpr int64_t kMaxSteps = 4000;           // < 4096 (12-bit flag step)

__device__ __host__ __forceinline__ int64_t rounds_for(int64_t bytes, int64_t slot) {
  return bytes <= slot ? 1 : (bytes + slot - 1) / slot;
}
__device__ __forceinline__ uint32_t pair_sig(uint32_t base, int64_t bytes) {
  return mix32(base, uint64_t(bytes)) & 0xFFFFFu;
}
// CTAs serving one pair: a function of the pair's byte count only.
__device__ __host__ __forceinline__ int pair_ctas(int64_t bytes, int gmax) {
  int64_t g = (bytes + kPairCtaBytes - 1) / kPairCtaBytes;
  return int(g < 1 ? 1 : (g > gmax ? gmax : g));
}
__device__ __forceinline__ int64_t pair_chunk(int64_t bytes, int g) {
  int64_t per = (bytes + g - 1) / g;
  int64_t ch = (per + kMaxSteps - 1) / kMaxSteps;
  ch = (ch + 15) & ~int64_t(15);
  return ch > kChunkBytes ? ch : kChunkBytes;
}

// Share s of round t of a pair moving B bytes: [a, e) relative to the round,
// in n chunks of `ch` bytes. A 0-byte pair still carries one empty chunk on
// share 0 (its flag is the order check / barrier).
struct Span {
  int64_t a, e;
  int n;
};
__device__ __forceinline__ Span span_of(int64_t B, int64_t slot, int g, int64_t ch, int64_t t, int s) {
  Span sp{0, 0, 0};
  if (s >= g || t >= rounds_for(B, slot)) return sp;
  const int64_t len = min(slot, B - t * slot);
  byte_share(len, s, g, sp.a, sp.e);
  sp.n = int((sp.e - sp.a + ch - 1) / ch);
  if (B == 0 && s == 0 && t == 0) sp.n = 1;
  return sp;
}

__global__ void __launch_bounds__(kThreads, 2) k_exchange(DevComm c, XArgs a, uint32_t epoch) {
  __shared__ const uint8_t* s_sp[kMaxRanks];
  __shared__ uint8_t* s_rp[kMaxRanks];
  __shared__ int64_t s_sb[kMaxRanks];
  __shared__ int64_t s_rb[kMaxRanks];
  __shared__ int s_err;
  __shared__ SComm S;
  const int par = epoch & 1, rank = c.rank, world = c.world;
  const int tid = threadIdx.x;
  const bool sender = int(blockIdx.x) < a.gp;
  const int s = sender ? int(blockIdx.x) : int(blockIdx.x) - a.gp;  // share index
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
      if (sc < 0 || sd < 0 || rc < 0 || rd < 0 || sd + sc > a.in_count || rd + rc > a.out_count)
        s_err = MCRDL_ERR_VALIDATION;
    } else {
      s_sp[tid] = a.sptr[tid];
      s_sb[tid] = a.sbytes[tid];
      s_rp[tid] = a.rptr[tid];
      s_rb[tid] = a.rbytes[tid];
    }
  }
  __syncthreads();
  if (tid == 0 && s_sb[rank] != s_rb[rank]) s_err = MCRDL_ERR_VALIDATION;
  __syncthreads();
  if (s_err) {
    if (tid == 0) raise_error(S.pad, world, c.err, s_err, epoch);
    return;
  }

  // Per-peer state lives in thread `peer` (tid < world) and is mirrored by
  // every thread from shared memory when computing block-uniform loop bounds.
  const int me = tid;  // peer index handled by this thread in flag duties
  if (sender) {
    int64_t rmax = 0;
    for (int j = 0; j < world; ++j)
      if (j != rank && s < pair_ctas(s_sb[j], a.gmax)) rmax = max(rmax, rounds_for(s_sb[j], slot));
    int sent = 0;  // chunks published to peer `me` (thread-local, tid < world)
    for (int64_t t = 0; t < rmax; ++t) {
      if (t > 0) {  // slot reuse: receiver share s consumed round t-1
        if (me < world && me != rank) {
          const int g = pair_ctas(s_sb[me], a.gmax);
          if (s < g && t < rounds_for(s_sb[me], slot)) {
            int e = wait_flag(&S.pad[rank]->ack[par][s][me], S.pad[rank], c.timeout_ns, epoch,
                              pair_sig(a.sig_base, s_sb[me]), uint32_t(t));
            if (e) atomicCAS(&s_err, 0, e);
          }
        }
        __syncthreads();
        if (s_err) {
          if (tid == 0) raise_error(S.pad, world, c.err, s_err, epoch);
          return;
        }
      }
      int rows = 0;
      for (int j = 0; j < world; ++j) {
        if (j == rank) continue;
        const int g = pair_ctas(s_sb[j], a.gmax);
        rows = max(rows, span_of(s_sb[j], slot, g, pair_chunk(s_sb[j], g), t, s).n);
      }
      for (int r = 0; r < rows; ++r) {
        for (int k = 1; k < world; ++k) {
          const int j = (rank + k) % world;
          const int g = pair_ctas(s_sb[j], a.gmax);
          const int64_t ch = pair_chunk(s_sb[j], g);
          const Span sp = span_of(s_sb[j], slot, g, ch, t, s);
          if (r >= sp.n) continue;
          const int64_t lo = sp.a + r * ch, hi = min(sp.e, lo + ch);
          block_copy<4>(S.ws[j] + hoff + int64_t(rank) * slot + lo, s_sp[j] + t * slot + lo, hi - lo);
        }
        __syncthreads();
        if (me < world && me != rank) {
          const int g = pair_ctas(s_sb[me], a.gmax);
          const Span sp = span_of(s_sb[me], slot, g, pair_chunk(s_sb[me], g), t, s);
          if (r < sp.n) {
            ++sent;
            publish(&S.pad[me]->flag[par][s][rank],
                    make_flag(epoch, pair_sig(a.sig_base, s_sb[me]), uint32_t(sent)));
          }
        }
      }
    }
    return;
  }

  // ------------------------------------------------------------- receiver
  {  // local segment: straight copy (skipped when in place)
    int64_t lo, hi;
    byte_share(s_sb[rank], s, a.gp, lo, hi);
    block_copy<4>(s_rp[rank] + lo, s_sp[rank] + lo, hi - lo);
  }
  int64_t rmax = 0;
  for (int i = 0; i < world; ++i)
    if (i != rank && s < pair_ctas(s_rb[i], a.gmax)) rmax = max(rmax, rounds_for(s_rb[i], slot));
  int got = 0;  // chunks consumed from peer `me`
  const uint8_t* my_ws = S.ws[rank] + hoff;
  for (int64_t t = 0; t < rmax; ++t) {
    int rows = 0;
    for (int i = 0; i < world; ++i) {
      if (i == rank) continue;
      const int g = pair_ctas(s_rb[i], a.gmax);
      rows = max(rows, span_of(s_rb[i], slot, g, pair_chunk(s_rb[i], g), t, s).n);
    }
    for (int r = 0; r < rows; ++r) {
      if (me < world && me != rank) {
        const int g = pair_ctas(s_rb[me], a.gmax);
        const Span sp = span_of(s_rb[me], slot, g, pair_chunk(s_rb[me], g), t, s);
        if (r < sp.n) {
          int e = wait_flag(&S.pad[rank]->flag[par][s][me], S.pad[rank], c.timeout_ns, epoch,
                            pair_sig(a.sig_base, s_rb[me]), uint32_t(got + 1));
          if (e) atomicCAS(&s_err, 0, e);
          ++got;
        }
      }
      __syncthreads();
      if (s_err) {
        if (tid == 0) raise_error(S.pad, world, c.err, s_err, epoch);
        return;
      }
      for (int k = 1; k < world; ++k) {
        const int i = (rank - k + world) % world;
        const int g = pair_ctas(s_rb[i], a.gmax);
        const int64_t ch = pair_chunk(s_rb[i], g);
        const Span sp = span_of(s_rb[i], slot, g, ch, t, s);
        if (r >= sp.n) continue;
        const int64_t lo = sp.a + r * ch, hi = min(sp.e, lo + ch);
        block_copy<4>(s_rp[i] + t * slot + lo, my_ws + int64_t(i) * slot + lo, hi - lo);
      }
    }
    // Round t of every pair fully landed: let senders reuse the slot.
    bool more = false;
    for (int i = 0; i < world; ++i)
      if (i != rank && s < pair_ctas(s_rb[i], a.gmax) && t + 1 < rounds_for(s_rb[i], slot)) more = true;
    if (more) {
      __syncthreads();
      if (me < world && me != rank && s < pair_ctas(s_rb[me], a.gmax) &&
          t + 1 < rounds_for(s_rb[me], slot))
        publish(&S.pad[me]->ack[par][s][rank],
                make_flag(epoch, pair_sig(a.sig_base, s_rb[me]), uint32_t(t + 1)));
    }
  }
}

mcrdl_status_t launch_local_copy(void* dst, const void* src, int64_t nbytes, int num_sms,
                                 cudaStream_t stream);

mcrdl_status_t launch_exchange(mcrdl_comm* c, const ExchangeSpec& sp, int64_t total_hint,
                               cudaStream_t stream) {
  (void)total_hint;
  if (c->world == 1 && sp.d_counts == nullptr) {
    if (sp.sbytes[0] != sp.rbytes[0])
      return set_error(MCRDL_ERR_VALIDATION, "self segment: send %lld bytes, receive %lld bytes",
                       (long long)sp.sbytes[0], (long long)sp.rbytes[0]);
    return launch_local_copy(sp.rptr[0], sp.sptr[0], sp.sbytes[0], c->num_sms, stream);
  }
  uint32_t epoch;
  mcrdl_status_t st = begin_op(c, stream, &epoch);
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
  a.in_count = sp.in_count;
  a.out_count = sp.out_count;
  a.esize = sp.esize;
  a.sig_base = sp.sig_base;
  a.slot = c->dc.half_bytes / c->world / 256 * 256;
  a.gmax = c->num_sms < kMaxBlocks ? c->num_sms : kMaxBlocks;  // 2 roles -> 2 CTAs/SM
  if (a.gmax < 1) a.gmax = 1;
  // CTAs per role: the widest pair (sender and receiver agree per pair,
  // see pair_ctas); device-resident counts are unknown here -> gmax. The
  // local copy also spreads over the receiver CTAs.
  int64_t g = 1;
  if (sp.d_counts != nullptr) {
    g = a.gmax;
  } else {
    for (int r = 0; r < c->world; ++r) {
      if (r == c->rank) {
        g = std::max<int64_t>(g, std::min<int64_t>(a.gmax, (sp.sbytes[r] + (1 << 20) - 1) >> 20));
        continue;
      }
      g = std::max<int64_t>(g, pair_ctas(sp.sbytes[r], a.gmax));
      g = std::max<int64_t>(g, pair_ctas(sp.rbytes[r], a.gmax));
    }
  }
  a.gp = int(g);
  k_exchange<<<int(2 * g), kThreads, 0, stream>>>(c->dc, a, epoch);
  count_launch();
  MCRDL_CUDA_CHECK(cudaGetLastError());
  return MCRDL_OK;
}

}  // namespace mcrdl
