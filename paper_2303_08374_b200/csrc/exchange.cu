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
//                            per 256 KiB chunk;
//   receiver CTAs [Gp, 2Gp)  copy their share of the local segment, then land
//                            each incoming chunk as soon as its flag arrives.
// So the NVLink push, the local copy and the copy-out overlap; senders never
// wait except for slot reuse (pairs larger than a workspace slot move in
// rounds the receiver acknowledges), so forward progress does not depend on
// CTA co-residency. Pairs agree on their geometry from their own byte count
// (sender: scount, receiver: rcount) — no extra exchange.
#include <algorithm>
#include <cstring>

#include "ll.cuh"

namespace mcrdl {

struct XArgs {
  const uint8_t* sptr[kMaxRanks];
  int64_t sbytes[kMaxRanks];
  uint8_t* rptr[kMaxRanks];
  int64_t rbytes[kMaxRanks];
  const int64_t* d_counts;  // device counts in elements (layout: d_layout), or null
  const int64_t* d_displs;  // all_gatherv / gatherv layouts: device displs
  int d_layout;
  int d_root;
  const uint8_t* in_base;
  uint8_t* out_base;
  int64_t in_count;  // element capacity of in/out (device-count bounds check)
  int64_t out_count;
  int64_t slot;      // workspace bytes per (sender) slot per round
  int esize;
  int gmax;          // communicator-wide cap on CTAs per pair
  int gp;            // CTAs per role in this launch
  int codec;         // 1: trunc16 on peer pairs (2 wire bytes per f32)
  int64_t ll_max;    // pairs of <= ll_max bytes use LL lines (-1: none)
  int64_t pair_cta;  // bytes of a pair per serving CTA (kPairCtaBytes)
  int64_t chunk_min; // minimum flag chunk (kChunkBytes)
  int64_t wide_min;  // pairs of >= wide_min bytes get 4x pair_cta per CTA (0: off)
  uint32_t sig_base;
};

constexpr int64_t kPairCtaBytes = 32 << 10;   // one CTA per 32 KiB of a pair
// Flag granularity inside a share: 128 KiB (p = 4 all_to_allv 256 MiB: 393 vs
// 418 us at 256 KiB, 64 KiB equal to 128 KiB, <= 16 MiB neutral;
// profiles/xgeo_ab_r1_p4.log).
constexpr int64_t kChunkBytes = 128 << 10;
__device__ __forceinline__ uint32_t pair_sig(uint32_t base, int64_t bytes) {
  // user (not wire) bytes, codec bit carried through from the base
  return (mix32(base, uint64_t(bytes)) & 0x7FFFFu) | (base & kSigCodecBit);
}

// Trunc16Codec fused into the copies (reference middleware.py:43-75): the
// wire carries the top 16 bits of each f32 (sign, exponent, 7 mantissa
// bits), widened back with zero fill. `wire` = 2 bytes per element; user
// f32 buffers are at least 4-byte aligned, workspace offsets 16-byte.
__device__ __forceinline__ void block_encode16(uint8_t* dst, const uint8_t* src, int64_t wire) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t ne = wire / 2;
  int64_t done = 0;
  if (((uintptr_t(dst) | uintptr_t(src)) & 15) == 0) {
    const int64_t np = wire / 16;  // 8 elements per wire pack
    const uint4* s = reinterpret_cast<const uint4*>(src);
    uint4* d = reinterpret_cast<uint4*>(dst);
    int64_t i = tid;
    for (; i + nt < np; i += 2 * nt) {
      uint4 a[2], b[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        a[u] = s[2 * (i + u * nt)];
        b[u] = s[2 * (i + u * nt) + 1];
      }
#pragma unroll
      for (int u = 0; u < 2; ++u)
        d[i + u * nt] = make_uint4(__byte_perm(a[u].x, a[u].y, 0x7632), __byte_perm(a[u].z, a[u].w, 0x7632),
                                   __byte_perm(b[u].x, b[u].y, 0x7632), __byte_perm(b[u].z, b[u].w, 0x7632));
    }
    for (; i < np; i += nt) {
      const uint4 a = s[2 * i], b = s[2 * i + 1];
      d[i] = make_uint4(__byte_perm(a.x, a.y, 0x7632), __byte_perm(a.z, a.w, 0x7632),
                        __byte_perm(b.x, b.y, 0x7632), __byte_perm(b.z, b.w, 0x7632));
    }
    done = np * 8;
  }
  const uint32_t* s32 = reinterpret_cast<const uint32_t*>(src);
  uint16_t* d16 = reinterpret_cast<uint16_t*>(dst);
  for (int64_t e = done + tid; e < ne; e += nt) d16[e] = uint16_t(s32[e] >> 16);
}

__device__ __forceinline__ void block_decode16(uint8_t* dst, const uint8_t* src, int64_t wire) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t ne = wire / 2;
  int64_t done = 0;
  if (((uintptr_t(dst) | uintptr_t(src)) & 15) == 0) {
    const int64_t np = wire / 16;
    const uint4* s = reinterpret_cast<const uint4*>(src);
    uint4* d = reinterpret_cast<uint4*>(dst);
    for (int64_t i = tid; i < np; i += nt) {
      const uint4 w = __ldcg(s + i);
      d[2 * i] = make_uint4(w.x << 16, w.x & 0xFFFF0000u, w.y << 16, w.y & 0xFFFF0000u);
      d[2 * i + 1] = make_uint4(w.z << 16, w.z & 0xFFFF0000u, w.w << 16, w.w & 0xFFFF0000u);
    }
    done = np * 8;
  }
  const unsigned short* s16 = reinterpret_cast<const unsigned short*>(src);
  uint32_t* d32 = reinterpret_cast<uint32_t*>(dst);
  for (int64_t e = done + tid; e < ne; e += nt) d32[e] = uint32_t(__ldcg(s16 + e)) << 16;
}
// Per-peer geometry of this CTA's role, computed once by thread `peer`:
// 64-bit divisions are ~70-instruction subroutines, and every thread of
// every row recomputing them cost ~8 us of latency per op.
struct PeerGeo {
  int64_t ch[kMaxRanks];  // chunk bytes
  int64_t R[kMaxRanks];   // rounds this CTA takes part in (0: not serving the pair)
  int64_t a[kMaxRanks];   // current round's share [a, e)
  int64_t e[kMaxRanks];
  int g[kMaxRanks];
  int n[kMaxRanks];       // chunks of the current round's share
  int rows;
  int more;               // some pair continues past the current round
  int64_t rmax;
};

__device__ __forceinline__ void geo_init(PeerGeo& G, const int64_t* bytes, const int64_t* user,
                                         int world, int rank, int s, int gmax, int64_t slot,
                                         int64_t ll_max, int64_t per_cta, int64_t chunk_min,
                                         int64_t wide_min) {
  const int tid = threadIdx.x;
  if (tid < world) {
    const int64_t B = bytes[tid];  // wire bytes
    const int g = pair_ctas(B, gmax, per_cta, wide_min);
    G.g[tid] = g;
    G.ch[tid] = pair_chunk(B, g, chunk_min);
    // LL pairs (<= ll_max USER bytes, as both LL ends decide) move as LL lines.
    G.R[tid] = (tid != rank && s < g && user[tid] > ll_max) ? rounds_for(B, slot) : 0;
  }
  __syncthreads();
  if (tid == 0) {
    int64_t m = 0;
    for (int j = 0; j < world; ++j) m = max(m, G.R[j]);
    G.rmax = m;
  }
  __syncthreads();
}

__device__ __forceinline__ void geo_round(PeerGeo& G, const int64_t* bytes, int world, int s,
                                          int64_t slot, int64_t t) {
  const int tid = threadIdx.x;
  if (tid < world) {
    Span sp{0, 0, 0};
    if (t < G.R[tid]) sp = span_of(bytes[tid], slot, G.g[tid], G.ch[tid], t, s);
    G.a[tid] = sp.a;
    G.e[tid] = sp.e;
    G.n[tid] = sp.n;
  }
  __syncthreads();
  if (tid == 0) {
    int rows = 0, more = 0;
    for (int j = 0; j < world; ++j) {
      rows = max(rows, G.n[j]);
      if (t + 1 < G.R[j]) more = 1;
    }
    G.rows = rows;
    G.more = more;
  }
  __syncthreads();
}

__device__ __forceinline__ void exchange_body(DevComm c, XArgs a, uint32_t epoch) {
  __shared__ const uint8_t* s_sp[kMaxRanks];
  __shared__ uint8_t* s_rp[kMaxRanks];
  __shared__ int64_t s_sb[kMaxRanks];
  __shared__ int64_t s_rb[kMaxRanks];
  __shared__ int64_t s_sw[kMaxRanks];  // wire bytes per pair (== user bytes without codec)
  __shared__ int64_t s_rw[kMaxRanks];
  __shared__ int s_err;
  __shared__ SComm S;
  __shared__ PeerGeo G;
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
      int64_t sc, sd, rc, rd;
      if (a.d_layout == kDevA2AV) {
        sc = a.d_counts[tid], sd = a.d_counts[world + tid];
        rc = a.d_counts[2 * world + tid], rd = a.d_counts[3 * world + tid];
      } else {
        // gathers: my block (rcounts[rank]) goes to every receiving peer;
        // block tid lands at displs[tid] (gatherv: root <-> everyone only)
        const bool gv = a.d_layout == kDevGatherv;
        const bool to_peer = !gv || tid == a.d_root;
        const bool from_peer = !gv || rank == a.d_root;
        sc = to_peer ? a.d_counts[rank] : 0, sd = 0;
        rc = from_peer ? a.d_counts[tid] : 0, rd = from_peer ? a.d_displs[tid] : 0;
      }
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
  if (tid < world) {
    s_sw[tid] = (a.codec && tid != rank) ? s_sb[tid] / 2 : s_sb[tid];
    s_rw[tid] = (a.codec && tid != rank) ? s_rb[tid] / 2 : s_rb[tid];
  }
  if (tid == 0 && s_sb[rank] != s_rb[rank]) s_err = MCRDL_ERR_VALIDATION;
  __syncthreads();
  // LL carries small pairs (truncated values when the codec is on)
  const int64_t ll_max = a.ll_max;
  if (s_err) {
    if (tid == 0) raise_error(S.pad, world, c.err, s_err, epoch);
    return;
  }

  const int me = tid;  // peer index this thread handles in flag duties (tid < world)
  const int bid = int(blockIdx.x);
  MCRDL_TRACE_AT(c, bid, 0);
  if (sender) {
    if (ll_max >= 0)
      exchange_ll_send_pairs(S.pad, rank, world, par, s_sp, s_sb, a.sig_base, epoch, ll_max, s,
                             a.gp);
    geo_init(G, s_sw, s_sb, world, rank, s, a.gmax, slot, ll_max, a.pair_cta, a.chunk_min,
             a.wide_min);
    int sent = 0;  // chunks published to peer `me`
    for (int64_t t = 0; t < G.rmax; ++t) {
      if (t > 0) {  // slot reuse: receiver share s consumed round t-1
        if (me < world && t < G.R[me]) {
          int e = wait_flag(&S.pad[rank]->ack[par][s][me], S.pad[rank], c.timeout_ns, c.err, epoch,
                            pair_sig(a.sig_base, s_sb[me]), uint32_t(t));
          if (e) atomicCAS(&s_err, 0, e);
        }
        __syncthreads();
        if (s_err) {
          if (tid == 0) raise_error(S.pad, world, c.err, s_err, epoch);
          return;
        }
      }
      geo_round(G, s_sw, world, s, slot, t);
      for (int r = 0; r < G.rows; ++r) {
        for (int k = 1; k < world; ++k) {
          const int j = (rank + k) % world;
          if (r >= G.n[j]) continue;
          const int64_t lo = G.a[j] + r * G.ch[j], hi = min(G.e[j], lo + G.ch[j]);
          uint8_t* dst = S.ws[j] + hoff + int64_t(rank) * slot + lo;
          if (a.codec)
            block_encode16(dst, s_sp[j] + 2 * (t * slot + lo), hi - lo);
          else
            block_copy<4>(dst, s_sp[j] + t * slot + lo, hi - lo);
        }
        __syncthreads();
        if (me < world && me != rank && r < G.n[me]) {
          ++sent;
          publish(&S.pad[me]->flag[par][s][rank],
                  make_flag(epoch, pair_sig(a.sig_base, s_sb[me]), uint32_t(sent)));
        }
        MCRDL_TRACE_AT(c, bid, 1 + r);
      }
    }
    MCRDL_TRACE_AT(c, bid, kTraceSlots - 1);
    return;
  }

  // ------------------------------------------------------------- receiver
  {  // local segment: straight copy (skipped when in place). (Interleaving it
     // with the row-flag waits measured neutral: tools/trace_x.py.)
    int64_t lo, hi;
    byte_share(s_sb[rank], s, a.gp, lo, hi);
    block_copy<4>(s_rp[rank] + lo, s_sp[rank] + lo, hi - lo);
  }
  MCRDL_TRACE_AT(c, bid, 1);
  if (ll_max >= 0) {
    const int e = exchange_ll_recv_pairs(S.pad, rank, world, par, s_rp, s_rb, a.sig_base, epoch,
                                         c.timeout_ns, ll_max, s, a.gp);
    if (e) {  // abort now: other threads may be polling lines that will never come
      atomicCAS(&s_err, 0, e);
      raise_error(S.pad, world, c.err, e, epoch);
    }
  }
  __syncthreads();
  if (s_err) {
    if (tid == 0) raise_error(S.pad, world, c.err, s_err, epoch);
    return;
  }
  geo_init(G, s_rw, s_rb, world, rank, s, a.gmax, slot, ll_max, a.pair_cta, a.chunk_min,
           a.wide_min);
  int got = 0;  // chunks consumed from peer `me`
  const uint8_t* my_ws = S.ws[rank] + hoff;
  for (int64_t t = 0; t < G.rmax; ++t) {
    geo_round(G, s_rw, world, s, slot, t);
    for (int r = 0; r < G.rows; ++r) {
      if (me < world && me != rank && r < G.n[me]) {
        int e = wait_flag(&S.pad[rank]->flag[par][s][me], S.pad[rank], c.timeout_ns, c.err, epoch,
                          pair_sig(a.sig_base, s_rb[me]), uint32_t(got + 1));
        if (e) atomicCAS(&s_err, 0, e);
        ++got;
      }
      __syncthreads();
      MCRDL_TRACE_AT(c, bid, 2 + 2 * r);
      if (s_err) {
        if (tid == 0) raise_error(S.pad, world, c.err, s_err, epoch);
        return;
      }
      for (int k = 1; k < world; ++k) {
        const int i = (rank - k + world) % world;
        if (r >= G.n[i]) continue;
        const int64_t lo = G.a[i] + r * G.ch[i], hi = min(G.e[i], lo + G.ch[i]);
        if (a.codec)
          block_decode16(s_rp[i] + 2 * (t * slot + lo), my_ws + int64_t(i) * slot + lo, hi - lo);
        else
          block_copy<4>(s_rp[i] + t * slot + lo, my_ws + int64_t(i) * slot + lo, hi - lo);
      }
      MCRDL_TRACE_AT(c, bid, 3 + 2 * r);
    }
    // Round t of every pair fully landed: let senders reuse the slot.
    if (G.more) {
      __syncthreads();
      if (me < world && t + 1 < G.R[me])
        publish(&S.pad[me]->ack[par][s][rank],
                make_flag(epoch, pair_sig(a.sig_base, s_rb[me]), uint32_t(t + 1)));
    }
  }
  MCRDL_TRACE_AT(c, bid, kTraceSlots - 1);
}

__global__ void __launch_bounds__(kThreads, 2) k_exchange(DevComm c, XArgs a) {
  const uint32_t epoch = epoch_enter(c);
  exchange_body(c, a, epoch);
  epoch_exit(c, epoch);
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
  mcrdl_status_t st = begin_op(c, stream);
  if (st != MCRDL_OK) return st;
  // Geometry knobs (tools/xgeo_ab.sh); every rank must see the same values.
  static const int64_t pair_kb = env_int("MCRDL_X_PAIR_KB", kPairCtaBytes >> 10);
  static const int64_t chunk_kb = env_int("MCRDL_X_CHUNK_KB", kChunkBytes >> 10);
  // Pairs >= 8 MiB: 128 KiB of pair per CTA (fewer, longer shares). p = 4
  // 32/64 MiB all_to_allv +11/+8 %, p = 2 16/32 MiB +17/+13 %, other sizes
  // neutral; a 4 MiB threshold costs p = 4 16 MiB (profiles/xwide_ab_r1_p2p4.log).
  static const int64_t wide_mb = env_int("MCRDL_X_WIDE_MB", 8);
  const int64_t pair_cta = (pair_kb > 0 ? pair_kb : kPairCtaBytes >> 10) << 10;
  const int64_t chunk_min = (chunk_kb > 0 ? chunk_kb : kChunkBytes >> 10) << 10;
  const int64_t wide_min = wide_mb > 0 ? wide_mb << 20 : 0;
  // The knobs are part of the pair agreement: ranks with different MCRDL_X_*
  // values raise ORDER_MISMATCH instead of landing half-written shares.
  ExchangeSpec spg = sp;
  spg.sig_base =
      (mix32(mix32(mix32(sp.sig_base, uint64_t(pair_cta)), uint64_t(chunk_min)), uint64_t(wide_min)) &
       ~kSigCodecBit) |
      (sp.codec ? kSigCodecBit : 0u);
  // LL pairs carry the codec too (truncated values in raw LL lines): both
  // ends pick LL from the pair's user bytes, so a codec disagreement on a
  // small pair meets a header with the other codec bit -> CODEC_MISMATCH.
  const int64_t ll_max = exchange_ll_max();
  if (ll_max >= 0 && try_exchange_ll(c, spg, ll_max, stream, &st)) return st;
  XArgs a;
  memset(&a, 0, sizeof(a));
  for (int r = 0; r < c->world; ++r) {
    a.sptr[r] = sp.sptr[r];
    a.sbytes[r] = sp.sbytes[r];
    a.rptr[r] = sp.rptr[r];
    a.rbytes[r] = sp.rbytes[r];
  }
  a.d_counts = sp.d_counts;
  a.d_displs = sp.d_displs;
  a.d_layout = sp.d_layout;
  a.d_root = sp.d_root;
  a.in_base = sp.in_base;
  a.out_base = sp.out_base;
  a.in_count = sp.in_count;
  a.out_count = sp.out_count;
  a.esize = sp.esize;
  a.codec = sp.codec;
  a.ll_max = ll_max;
  a.pair_cta = pair_cta;
  a.chunk_min = chunk_min;
  a.wide_min = wide_min;
  a.sig_base = spg.sig_base;
  a.slot = c->dc.half_bytes / c->world / 256 * 256;
  a.gmax = c->num_sms < kMaxBlocks ? c->num_sms : kMaxBlocks;  // 2 roles -> 2 CTAs/SM
  if (a.gmax < 1) a.gmax = 1;
  // CTAs per role: the widest pair (sender and receiver agree per pair,
  // see pair_ctas); device-resident counts are unknown here -> gmax. The
  // local copy also spreads over the receiver CTAs.
  int64_t g = 1;
  if (sp.d_counts != nullptr) {
    // counts live on the device: no pair can exceed the larger buffer, so
    // size for that instead of always the full grid
    // (pair_ctas is not monotonic: the largest narrow pair below the wide
    // threshold may need more CTAs than the capacity itself)
    const int64_t cap = std::max(sp.in_count, sp.out_count) * sp.esize;
    const int64_t wire = sp.codec ? cap / 2 : cap;
    const int64_t narrow = a.wide_min > 0 ? std::min(wire, a.wide_min - 1) : wire;
    g = std::max<int64_t>(pair_ctas(wire, a.gmax, a.pair_cta, a.wide_min),
                          pair_ctas(narrow, a.gmax, a.pair_cta, a.wide_min));
    g = std::max<int64_t>(g, std::min<int64_t>(a.gmax, (cap + (1 << 20) - 1) >> 20));
  } else {
    for (int r = 0; r < c->world; ++r) {
      if (r == c->rank) {
        g = std::max<int64_t>(g, std::min<int64_t>(a.gmax, (sp.sbytes[r] + (1 << 20) - 1) >> 20));
        continue;
      }
      // wire bytes, as the kernel computes them: pair_ctas is not monotonic
      // in the byte count (wide pairs), so user bytes would under-size the grid
      const int64_t sw = sp.codec ? sp.sbytes[r] / 2 : sp.sbytes[r];
      const int64_t rw = sp.codec ? sp.rbytes[r] / 2 : sp.rbytes[r];
      g = std::max<int64_t>(g, pair_ctas(sw, a.gmax, a.pair_cta, a.wide_min));
      g = std::max<int64_t>(g, pair_ctas(rw, a.gmax, a.pair_cta, a.wide_min));
    }
  }
  a.gp = int(g);
  k_exchange<<<int(2 * g), kThreads, 0, stream>>>(c->dc, a);
  count_launch();
  MCRDL_CUDA_CHECK(cudaGetLastError());
  return MCRDL_OK;
}

}  // namespace mcrdl
