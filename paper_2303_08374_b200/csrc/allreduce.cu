// all_reduce over NVLink peer memory: one-shot (K1), two-shot (K2) and the
// fused pack -> reduce -> unpack variant (K9).
//
// Reference algorithms being replaced (collectives.py):
//   _allreduce_naive   :296-312  gather to rank 0, fold ascending, send back
//   _allreduce_ring    :355-382  ring RS + AG over even_segments (:163-171)
//   FusionManager flush (middleware.py:311-344) concat -> all_reduce -> scatter
// Both kernels here fold the p contributions in ASCENDING rank order with a
// single pass per element, exactly the sequential oracle's fold
// (reference.py:16-20, tests/seqref.py:13-24), so f32/f64 results are
// bit-identical to the oracle (bf16: f32 accumulation, one RNE rounding).
#include "internal.h"

namespace mcrdl {

// ----------------------------------------------------------------- one-shot
// Block b owns packs [pb, pe) of the message. Phase 1 pushes them into every
// peer's workspace slot `rank`; phase 2 folds slots 0..p-1 (own input for
// slot == rank) into `out`. Latency: one NVLink write + one flag per peer.
template <typename T, int OP, bool VEC>
__device__ __forceinline__ void ar_oneshot_body(DevComm c, const T* in, T* out, int64_t n, int64_t slot_bytes, uint32_t epoch,
                 uint32_t sig) {
  constexpr int N = Pack<T>::N;
  __shared__ int s_err;
  __shared__ SComm S;
  const int par = epoch & 1, rank = c.rank, world = c.world;
  const int b = blockIdx.x, G = gridDim.x, tid = threadIdx.x, nt = blockDim.x;
  const int64_t npk = (n + N - 1) / N;
  const int64_t pb = npk * b / G, pe = npk * (b + 1) / G;
  const int64_t hoff = int64_t(par) * c.half_bytes;
  if (tid == 0) s_err = 0;
  stage_comm(c, S);
  __syncthreads();

  // Phase 1: each pack read once from HBM, written to p-1 peers (kBatch
  // loads in flight per thread before the stores).
  constexpr int kBatch = 4;
  for (int64_t i0 = pb + tid; i0 < pe; i0 += kBatch * nt) {
    uint4 v[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u)
      if (i0 + u * nt < pe) v[u] = load_pack<T, VEC>(in, i0 + u * nt, n);
    for (int k = 1; k < world; ++k) {
      uint8_t* dst = S.ws[(rank + k) % world] + hoff + int64_t(rank) * slot_bytes;
#pragma unroll
      for (int u = 0; u < kBatch; ++u)
        if (i0 + u * nt < pe) st16(dst + (i0 + u * nt) * 16, v[u]);
    }
  }
  __syncthreads();
  const uint64_t f = make_flag(epoch, sig, 0);
  if (tid < world && tid != rank) publish(&S.pad[tid]->flag[par][b][rank], f);
  if (tid < world && tid != rank) {
    int e = wait_flag(&S.pad[rank]->flag[par][b][tid], S.pad[rank], c.timeout_ns, c.err, epoch, sig, 0);
    if (e) atomicCAS(&s_err, 0, e);
  }
  __syncthreads();
  if (s_err) {
    if (tid == 0) raise_error(S.pad, world, c.err, s_err, epoch);
    return;
  }
  // Phase 2: ascending fold; all p loads of a pack are issued before the
  // first fold (a fold-per-load loop waits one HBM latency per rank).
  const uint8_t* ws = S.ws[rank] + hoff;
  for (int64_t i = pb + tid; i < pe; i += nt) {
    uint4 raw[kMaxRanks];
#pragma unroll
    for (int r = 0; r < kMaxRanks; ++r)
      if (r < world)
        raw[r] = (r == rank) ? load_pack<T, VEC>(in, i, n)
                             : ld16_cg(ws + int64_t(r) * slot_bytes + i * 16);
    Pack<T> acc;
    acc.from_raw(raw[0]);
#pragma unroll
    for (int r = 1; r < kMaxRanks; ++r)
      if (r < world) acc.template fold<OP>(raw[r]);
    store_pack<T, VEC>(out, i, n, acc.to_raw());
  }
}

template <typename T, int OP, bool VEC>
__global__ void __launch_bounds__(kThreads) k_ar_oneshot(DevComm c, const T* in, T* out, int64_t n, int64_t slot_bytes, uint32_t sig) {
  const uint32_t epoch = epoch_enter(c);
  ar_oneshot_body<T, OP, VEC>(c, in, out, n, slot_bytes, epoch, sig);
  epoch_exit(c, epoch);
}

// ------------------------------------------------ pipelined two-shot (K2)
// Three CTA roles run concurrently over the same share s of every segment,
// handing off 64 KiB chunks through per-chunk release flags:
//   senders   [0, gp)     RS push: my copy of segment q, chunk r -> rank q
//   reducers  [gp, 2gp)   fold chunk r of my segment (ascending ranks) ->
//                         out + every peer's AG area
//   gatherers [2gp, 3gp)  land every peer's reduced chunk r into out
// NVLink carries RS and AG traffic at the same time and local HBM work hides
// under it. Senders never wait; reducers wait only for senders; gatherers
// only for reducers: progress does not need CTA co-residency.
template <typename T, bool VEC, int U = 4>
__device__ __forceinline__ void push_packs(const T* in, int64_t n, int64_t g0, int64_t cnt,
                                           uint8_t* dst) {
  // packs [g0, g0+cnt) of `in` -> dst (16-byte aligned, pack i at dst + 16*(i-g0));
  // U packs in flight per thread
  const int tid = threadIdx.x, nt = blockDim.x;
  int64_t i = tid;
  for (; i + (U - 1) * nt < cnt; i += U * nt) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = load_pack<T, VEC>(in, g0 + i + u * nt, n);
#pragma unroll
    for (int u = 0; u < U; ++u) st16(dst + (i + u * nt) * 16, v[u]);
  }
  for (; i < cnt; i += nt) st16(dst + i * 16, load_pack<T, VEC>(in, g0 + i, n));
}

// TMA bulk-copy streaming (one elected thread): contiguous global -> smem ring
// (cp.async.bulk + mbarrier) -> global, possibly a peer over NVLink
// (cp.async.bulk.global.shared::cta). Measured on B200: 16 single-thread CTAs
// saturate NVLink push (697 GB/s, tools/tma_probe.cu) where LD/ST push needs
// ~74 full CTAs, so the SMs stay free for the fold/gather roles.
constexpr int kTmaStages = 4;
constexpr int kTmaPiece = 8192;
struct TmaRing {
  uint8_t* buf;    // smem, kTmaStages * kTmaPiece
  uint64_t* bar;   // smem mbarriers [kTmaStages]
  uint32_t phase;  // parity bit per stage
  uint32_t n;      // pieces issued
};
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void tma_init(TmaRing& R) {
  for (int s = 0; s < kTmaStages; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&R.bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  R.phase = 0;
  R.n = 0;
}
__device__ __forceinline__ void tma_stream(TmaRing& R, uint8_t* dst, const uint8_t* src,
                                           int64_t bytes) {
  for (int64_t off = 0; off < bytes; off += kTmaPiece) {
    const uint32_t sz = uint32_t(min(int64_t(kTmaPiece), bytes - off));
    const int st = int(R.n % kTmaStages);
    // the store issued from this stage kTmaStages pieces ago must have read smem
    if (R.n >= kTmaStages)
      asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kTmaStages - 1) : "memory");
    uint8_t* buf = R.buf + st * kTmaPiece;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&R.bar[st])),
                 "r"(sz)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(buf)),
        "l"(src + off), "r"(sz), "r"(smem_u32(&R.bar[st]))
        : "memory");
    const uint32_t ph = (R.phase >> st) & 1u;
    uint32_t ok = 0;
    while (!ok) {
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(ok)
          : "r"(smem_u32(&R.bar[st])), "r"(ph)
          : "memory");
    }
    R.phase ^= (1u << st);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + off),
                 "r"(smem_u32(buf)), "r"(sz)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    ++R.n;
  }
}
// A list of contiguous copies (one row: a chunk for every peer) streamed as
// kTmaPiece pieces with up to kTmaStages loads in flight: piece k loads into
// stage k % kTmaStages once the store that last used that stage has read it.
struct TmaList {
  uint8_t* dst[kMaxRanks];
  const uint8_t* src[kMaxRanks];
  int64_t bytes[kMaxRanks];
  int n;
};
__device__ __forceinline__ void tma_wait_stage(TmaRing& R, int st) {
  const uint32_t ph = (R.phase >> st) & 1u;
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_u32(&R.bar[st])), "r"(ph)
        : "memory");
  }
  R.phase ^= (1u << st);
}
__device__ __forceinline__ void tma_copy_list(TmaRing& R, const TmaList& L) {
  uint8_t* qdst[kTmaStages];
  uint32_t qsz[kTmaStages];
  int si = 0;
  int64_t off = 0;
  int loaded = 0, stored = 0;  // pieces of this list
  auto next = [&](uint8_t*& d, const uint8_t*& s, uint32_t& sz) -> bool {
    while (si < L.n && off >= L.bytes[si]) {
      ++si;
      off = 0;
    }
    if (si >= L.n) return false;
    d = L.dst[si] + off;
    s = L.src[si] + off;
    sz = uint32_t(min(int64_t(kTmaPiece), L.bytes[si] - off));
    off += sz;
    return true;
  };
  auto issue_load = [&](uint8_t* d, const uint8_t* s, uint32_t sz) {
    const int st = int((R.n + loaded) % kTmaStages);
    if (R.n + loaded >= kTmaStages)  // stage reused: its last store must have read smem
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&R.bar[st])),
                 "r"(sz)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(R.buf + st * kTmaPiece)),
        "l"(s), "r"(sz), "r"(smem_u32(&R.bar[st]))
        : "memory");
    qdst[st] = d;
    qsz[st] = sz;
    ++loaded;
  };
  uint8_t* d;
  const uint8_t* s;
  uint32_t sz;
  while (loaded < kTmaStages - 1 && next(d, s, sz)) issue_load(d, s, sz);
  while (stored < loaded) {
    const int st = int((R.n + stored) % kTmaStages);
    tma_wait_stage(R, st);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(qdst[st]),
                 "r"(smem_u32(R.buf + st * kTmaPiece)), "r"(qsz[st])
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    ++stored;
    if (next(d, s, sz)) issue_load(d, s, sz);
  }
  R.n += loaded;
}

// All bulk stores issued so far are complete and ordered before the thread's
// following generic-proxy operations (the release flag).
__device__ __forceinline__ void tma_drain() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

template <typename T, int OP, bool VEC, bool TMA>
__device__ __forceinline__ void ar_pipe_body(DevComm c, const T* in, T* out, int64_t n, int64_t sp,
                                             int64_t segb, int gp, int gs, int64_t chp,
                                             int root, uint32_t epoch, uint32_t sig, T* rs_out,
                                             int64_t rs_n) {
  constexpr int N = Pack<T>::N;
  __shared__ int s_err;
  __shared__ SComm S;
  __shared__ __align__(128) uint8_t s_ring[TMA ? kTmaStages * kTmaPiece : 16];
  __shared__ __align__(8) uint64_t s_bar[kTmaStages];
  const int par = epoch & 1, rank = c.rank, world = c.world;
  const int tid = threadIdx.x, nt = blockDim.x;
  // CTA roles: [0, gs) senders, [gs, gs+gp) reducers, [gs+gp, gs+2gp) gatherers
  const int bid = int(blockIdx.x);
  const int role = bid < gs ? 0 : (bid < gs + gp ? 1 : 2);
  const int s = role == 0 ? bid : (role == 1 ? bid - gs : bid - gs - gp);
  const int64_t npk = (n + N - 1) / N;
  const int64_t rb = sp * s / gp, re = sp * (s + 1) / gp;
  const int64_t hoff = int64_t(par) * c.half_bytes;
  const int64_t ag = int64_t(world) * segb;
  if (tid == 0) s_err = 0;
  stage_comm(c, S);
  __syncthreads();
  const uint8_t* ws = S.ws[rank] + hoff;
  MCRDL_TRACE_AT(c, bid, 0);

  if (TMA && role == 0) {  // ---------------------------- sender (TMA bulk)
    if (tid != 0) return;
    TmaRing R{s_ring, s_bar, 0, 0};
    tma_init(R);
    const uint8_t* src = reinterpret_cast<const uint8_t*>(in);
    for (int sh = s; sh < gp; sh += gs) {  // shares served by this CTA
      const int64_t b0 = sp * sh / gp, b1 = sp * (sh + 1) / gp;
      int rows = 0;
      for (int q = 0; q < world; ++q)
        if (q != rank) rows = max(rows, nchunks(seg_len(npk, sp, q, b0, b1), chp, sh));
      for (int r = 0; r < rows; ++r) {
        TmaList L;
        L.n = 0;
        for (int k = 1; k < world; ++k) {
          const int q = (rank + k) % world;
          const int64_t len = seg_len(npk, sp, q, b0, b1);
          const int64_t lo = int64_t(r) * chp;
          if (lo >= len) continue;
          const int64_t cnt = min(chp, len - lo);
          const int64_t g0 = int64_t(q) * sp + b0 + lo;
          // full packs by TMA, a trailing partial pack (end of the message) by hand
          const int64_t full = min(cnt, n / N - g0 > 0 ? n / N - g0 : int64_t(0));
          uint8_t* dst = S.ws[q] + hoff + int64_t(rank) * segb + (b0 + lo) * 16;
          if (full > 0) {
            L.dst[L.n] = dst;
            L.src[L.n] = src + g0 * 16;
            L.bytes[L.n] = full * 16;
            ++L.n;
          }
          for (int64_t i = full; i < cnt; ++i) st16(dst + i * 16, load_pack<T, VEC>(in, g0 + i, n));
        }
        tma_copy_list(R, L);
        tma_drain();
        for (int q = 0; q < world; ++q)
          if (q != rank && r < nchunks(seg_len(npk, sp, q, b0, b1), chp, sh))
            publish(&S.pad[q]->flag[par][sh][rank], make_flag(epoch, sig, uint32_t(r + 1)));
        MCRDL_TRACE_AT(c, bid, 1 + r);
      }
    }
    MCRDL_TRACE_AT(c, bid, kTraceSlots - 1);
    return;
  }

  if (role == 0) {  // ---------------------------------------------- sender
    int rows = 0;
    for (int q = 0; q < world; ++q)
      if (q != rank) rows = max(rows, nchunks(seg_len(npk, sp, q, rb, re), chp, s));
    for (int r = 0; r < rows; ++r) {
      for (int k = 1; k < world; ++k) {
        const int q = (rank + k) % world;
        const int64_t len = seg_len(npk, sp, q, rb, re);
        const int64_t lo = int64_t(r) * chp;
        if (lo >= len) continue;
        const int64_t cnt = min(chp, len - lo);
        push_packs<T, VEC>(in, n, int64_t(q) * sp + rb + lo, cnt,
                           S.ws[q] + hoff + int64_t(rank) * segb + (rb + lo) * 16);
      }
      __syncthreads();
      if (tid < world && tid != rank && r < nchunks(seg_len(npk, sp, tid, rb, re), chp, s))
        publish(&S.pad[tid]->flag[par][s][rank], make_flag(epoch, sig, uint32_t(r + 1)));
      MCRDL_TRACE_AT(c, bid, 1 + r);
    }
    MCRDL_TRACE_AT(c, bid, kTraceSlots - 1);
    return;
  }

  if (role == 1) {  // --------------------------------------------- reducer
    const int64_t len = seg_len(npk, sp, rank, rb, re);
    const int rows = nchunks(len, chp, s);
    for (int r = 0; r < rows; ++r) {
      if (tid < world && tid != rank) {
        int e = wait_flag(&S.pad[rank]->flag[par][s][tid], S.pad[rank], c.timeout_ns, c.err, epoch, sig,
                          uint32_t(r + 1));
        if (e) atomicCAS(&s_err, 0, e);
      }
      __syncthreads();
      MCRDL_TRACE_AT(c, bid, 1 + 2 * r);
      if (s_err) {
        if (tid == 0) raise_error(S.pad, world, c.err, s_err, epoch);
        return;
      }
      const int64_t lo = int64_t(r) * chp, hi = min(len, lo + chp);
      // RU packs per thread in flight: each rank's RU loads issue before the fold.
      constexpr int RU = sizeof(T) == 2 ? 2 : 4;
      int64_t i0 = rb + lo + tid;
      for (; i0 < rb + hi; i0 += RU * nt) {
        Pack<T> acc[RU];
        uint4 v[RU];
#pragma unroll
        for (int u = 0; u < RU; ++u) {
          const int64_t i = i0 + u * nt;
          if (i < rb + hi)
            v[u] = rank == 0 ? load_pack<T, VEC>(in, int64_t(rank) * sp + i, n) : ld16_cg(ws + i * 16);
        }
#pragma unroll
        for (int u = 0; u < RU; ++u) acc[u].from_raw(v[u]);
        for (int q = 1; q < world; ++q) {
#pragma unroll
          for (int u = 0; u < RU; ++u) {
            const int64_t i = i0 + u * nt;
            if (i < rb + hi)
              v[u] = (q == rank) ? load_pack<T, VEC>(in, int64_t(rank) * sp + i, n)
                                 : ld16_cg(ws + int64_t(q) * segb + i * 16);
          }
#pragma unroll
          for (int u = 0; u < RU; ++u) acc[u].template fold<OP>(v[u]);
        }
#pragma unroll
        for (int u = 0; u < RU; ++u) {
          const int64_t i = i0 + u * nt;
          if (i >= rb + hi) break;
          const uint4 res = acc[u].to_raw();
          if (rs_out != nullptr) {  // reduce_scatter: my segment is my output
            store_pack<T, VEC>(rs_out, i, rs_n, res);
            continue;
          }
          if (root >= 0) {  // reduce: the segment goes to the root only
            if (rank == root)
              store_pack<T, VEC>(out, int64_t(rank) * sp + i, n, res);
            else
              st16(S.ws[root] + hoff + ag + int64_t(rank) * segb + i * 16, res);
            continue;
          }
          for (int k = 1; k < world; ++k) {
            const int q = (rank + k) % world;
            st16(S.ws[q] + hoff + ag + int64_t(rank) * segb + i * 16, res);
          }
          store_pack<T, VEC>(out, int64_t(rank) * sp + i, n, res);
        }
      }
      if (rs_out != nullptr) continue;
      __syncthreads();
      if (tid < world && tid != rank && (root < 0 || tid == root))
        publish(&S.pad[tid]->flag2[par][s][rank], make_flag(epoch, sig, uint32_t(r + 1)));
      MCRDL_TRACE_AT(c, bid, 2 + 2 * r);
    }
    MCRDL_TRACE_AT(c, bid, kTraceSlots - 1);
    return;
  }

  // ------------------------------------------------------------- gatherer
  if (rs_out != nullptr) return;  // reduce_scatter has no all-gather phase
  if (root >= 0 && rank != root) return;  // reduce: only the root gathers
  int rows = 0;
  for (int q = 0; q < world; ++q)
    if (q != rank) rows = max(rows, nchunks(seg_len(npk, sp, q, rb, re), chp, s));
  for (int r = 0; r < rows; ++r) {
    if (tid < world && tid != rank && r < nchunks(seg_len(npk, sp, tid, rb, re), chp, s)) {
      int e = wait_flag(&S.pad[rank]->flag2[par][s][tid], S.pad[rank], c.timeout_ns, c.err, epoch, sig,
                        uint32_t(r + 1));
      if (e) atomicCAS(&s_err, 0, e);
    }
    __syncthreads();
    MCRDL_TRACE_AT(c, bid, 1 + 2 * r);
    if (s_err) {
      if (tid == 0) raise_error(S.pad, world, c.err, s_err, epoch);
      return;
    }
    for (int k = 1; k < world; ++k) {
      const int q = (rank + k) % world;
      const int64_t len = seg_len(npk, sp, q, rb, re);
      const int64_t lo = int64_t(r) * chp;
      if (lo >= len) continue;
      const int64_t hi = min(len, lo + chp);
      int64_t i = rb + lo + tid;
      const uint8_t* src = ws + ag + int64_t(q) * segb;
      for (; i + 3 * nt < rb + hi; i += 4 * nt) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = ld16_cg(src + (i + u * nt) * 16);
#pragma unroll
        for (int u = 0; u < 4; ++u) store_pack<T, VEC>(out, int64_t(q) * sp + i + u * nt, n, v[u]);
      }
      for (; i < rb + hi; i += nt) store_pack<T, VEC>(out, int64_t(q) * sp + i, n, ld16_cg(src + i * 16));
    }
    MCRDL_TRACE_AT(c, bid, 2 + 2 * r);
  }
  MCRDL_TRACE_AT(c, bid, kTraceSlots - 1);
}

template <typename T, int OP, bool VEC, bool TMA>
__global__ void __launch_bounds__(kThreads, 2)
    k_ar_pipe(DevComm c, const T* in, T* out, int64_t n, int64_t sp, int64_t segb, int gp, int gs,
              int64_t chp, int root, uint32_t sig, T* rs_out = nullptr,
              int64_t rs_n = 0) {
  const uint32_t epoch = epoch_enter(c);
  ar_pipe_body<T, OP, VEC, TMA>(c, in, out, n, sp, segb, gp, gs, chp, root, epoch, sig,
                                rs_out, rs_n);
  epoch_exit(c, epoch);
}

// ----------------------------------------------------------- NVLS (switch)
// All-reduce through the NVSwitch multicast object (sum, f32 / bf16):
//   copiers   [0, gp)     my input, chunk r of share s of EVERY segment ->
//                         my NVLS buffer (local HBM copy); flag to all ranks
//   reducers  [gp, 2gp)   chunk r of MY segment: multimem.ld_reduce (the
//                         switch sums the p replicas) -> multimem.st (the
//                         switch writes the sum to every rank); flag2 to all
//   gatherers [2gp, 3gp)  chunk r of segment q once rank q's flag2 arrived:
//                         NVLS buffer -> out
// NVLink bytes per rank ~S each way instead of 2(p-1)/p*S for two-shot.
// The switch's summation order is unspecified: results are within the
// float tolerance, not bit-identical to the ascending fold.
template <typename T>
__device__ __forceinline__ uint4 mm_ld_reduce_sum(const void* mc) {
  uint4 r;
  if constexpr (sizeof(T) == 4) {
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(mc)
                 : "memory");
  } else {
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(mc)
                 : "memory");
  }
  return r;
}
__device__ __forceinline__ void mm_st(void* mc, const uint4& v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc),
               "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

template <typename T, bool VEC>
__device__ __forceinline__ void ar_nvls_body(DevComm c, uint8_t* uc, uint8_t* mc, const T* in,
                                             T* out, int64_t n, int64_t sp, int gp, int gc, int gg,
                                             int64_t chp, int fence, uint32_t epoch, uint32_t sig) {
  // CTA roles: [0, gc) copiers, [gc, gc+gp) reducers (one per share),
  // [gc+gp, gc+gp+gg) gatherers. Copier / gatherer CTA k serves shares
  // k, k+gc (k+gg), ... row by row, so the local staging copies can run on
  // fewer SMs than the switch reductions.
  constexpr int N = Pack<T>::N;
  __shared__ int s_err;
  __shared__ SComm S;
  const int par = epoch & 1, rank = c.rank, world = c.world;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int bid = int(blockIdx.x);
  const int role = bid < gc ? 0 : (bid < gc + gp ? 1 : 2);
  const int k = role == 0 ? bid : (role == 1 ? bid - gc : bid - gc - gp);
  const int64_t npk = (n + N - 1) / N;
  if (tid == 0) s_err = 0;
  stage_comm(c, S);
  __syncthreads();

  if (role == 0) {  // ---------------------------------------------- copier
    int rows = 0;
    for (int sh = k; sh < gp; sh += gc) {
      const int64_t rb = sp * sh / gp, re = sp * (sh + 1) / gp;
      for (int q = 0; q < world; ++q) rows = max(rows, nchunks(seg_len(npk, sp, q, rb, re), chp, sh));
    }
    for (int r = 0; r < rows; ++r) {
      for (int sh = k; sh < gp; sh += gc) {
        const int64_t rb = sp * sh / gp, re = sp * (sh + 1) / gp;
        int my_rows = 0;
        for (int q = 0; q < world; ++q)
          my_rows = max(my_rows, nchunks(seg_len(npk, sp, q, rb, re), chp, sh));
        if (r >= my_rows) continue;
        for (int q = 0; q < world; ++q) {
          const int64_t len = seg_len(npk, sp, q, rb, re);
          const int64_t lo = int64_t(r) * chp;
          if (lo >= len) continue;
          const int64_t g0 = int64_t(q) * sp + rb + lo;
          push_packs<T, VEC, 8>(in, n, g0, min(chp, len - lo), uc + g0 * 16);
        }
        __syncthreads();
        if (tid < world)
          publish(&S.pad[tid]->flag[par][sh][rank], make_flag(epoch, sig, uint32_t(r + 1)));
      }
    }
    return;
  }

  if (role == 1) {  // --------------------------------------------- reducer
    const int s = k;
    const int64_t rb = sp * s / gp, re = sp * (s + 1) / gp;
    const int64_t len = seg_len(npk, sp, rank, rb, re);
    const int rows = nchunks(len, chp, s);
    for (int r = 0; r < rows; ++r) {
      if (tid < world) {
        int e = wait_flag(&S.pad[rank]->flag[par][s][tid], S.pad[rank], c.timeout_ns, c.err, epoch, sig,
                          uint32_t(r + 1));
        if (e) atomicCAS(&s_err, 0, e);
      }
      __syncthreads();
      if (s_err) {
        if (tid == 0) raise_error(S.pad, world, c.err, s_err, epoch);
        return;
      }
      const int64_t lo = int64_t(r) * chp, hi = min(len, lo + chp);
      const int64_t base = int64_t(rank) * sp + rb;
      // own segment: the result goes to the peers through the switch and
      // straight into `out` here (the gatherers skip it)
      int64_t i = lo + tid;
      for (; i + 3 * nt < hi; i += 4 * nt) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = mm_ld_reduce_sum<T>(mc + (base + i + u * nt) * 16);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          mm_st(mc + (base + i + u * nt) * 16, v[u]);
          store_pack<T, VEC>(out, base + i + u * nt, n, v[u]);
        }
      }
      for (; i < hi; i += nt) {
        const uint4 v = mm_ld_reduce_sum<T>(mc + (base + i) * 16);
        mm_st(mc + (base + i) * 16, v);
        store_pack<T, VEC>(out, base + i, n, v);
      }
      if (fence) __threadfence_system();  // multicast stores complete on every rank before the flag
      __syncthreads();
      if (tid < world) publish(&S.pad[tid]->flag2[par][s][rank], make_flag(epoch, sig, uint32_t(r + 1)));
    }
    return;
  }

  // ------------------------------------------------------------- gatherer
  int rows = 0;
  for (int sh = k; sh < gp; sh += gg) {
    const int64_t rb = sp * sh / gp, re = sp * (sh + 1) / gp;
    for (int q = 0; q < world; ++q) rows = max(rows, nchunks(seg_len(npk, sp, q, rb, re), chp, sh));
  }
  for (int r = 0; r < rows; ++r) {
    for (int sh = k; sh < gp; sh += gg) {
      const int64_t rb = sp * sh / gp, re = sp * (sh + 1) / gp;
      if (tid < world && r < nchunks(seg_len(npk, sp, tid, rb, re), chp, sh)) {
        int e = wait_flag(&S.pad[rank]->flag2[par][sh][tid], S.pad[rank], c.timeout_ns, c.err, epoch,
                          sig, uint32_t(r + 1));
        if (e) atomicCAS(&s_err, 0, e);
      }
      __syncthreads();
      if (s_err) {
        if (tid == 0) raise_error(S.pad, world, c.err, s_err, epoch);
        return;
      }
      for (int q = 0; q < world; ++q) {
        if (q == rank) continue;  // written by this rank's reducer
        const int64_t len = seg_len(npk, sp, q, rb, re);
        const int64_t lo = int64_t(r) * chp;
        if (lo >= len) continue;
        const int64_t hi = min(len, lo + chp);
        const int64_t base = int64_t(q) * sp + rb;
        int64_t i = lo + tid;
        for (; i + 7 * nt < hi; i += 8 * nt) {
          uint4 v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = ld16_cg(uc + (base + i + u * nt) * 16);
#pragma unroll
          for (int u = 0; u < 8; ++u) store_pack<T, VEC>(out, base + i + u * nt, n, v[u]);
        }
        for (; i < hi; i += nt) store_pack<T, VEC>(out, base + i, n, ld16_cg(uc + (base + i) * 16));
      }
    }
  }
}

template <typename T, bool VEC>
__global__ void __launch_bounds__(kThreads, 2)
    k_ar_nvls(DevComm c, uint8_t* uc, uint8_t* mc, int64_t nv_half, const T* in, T* out, int64_t n,
              int64_t sp, int gp, int gc, int gg, int64_t chp, int fence, uint32_t sig) {
  const uint32_t epoch = epoch_enter(c);
  const int64_t hoff = int64_t(epoch & 1) * nv_half;
  ar_nvls_body<T, VEC>(c, uc + hoff, mc + hoff, in, out, n, sp, gp, gc, gg, chp, fence, epoch, sig);
  epoch_exit(c, epoch);
}

// -------------------------------------------------------------- NVLS bcast
// The root stores every 16-byte pack ONCE into the multicast mapping and the
// switch replicates it into every rank's NVLS buffer: root egress S instead of
// (p-1)·S for a push broadcast. Chunk r of CTA share s is signalled by a
// multicast release store of the flag word (same path as the data: the
// CUTLASS multimem pattern, multimem.st + bar.sync + release). Non-roots wait
// on their unicast view of the flag, copy the chunk out, and ack their share
// to the root at the end: the NVLS half is free again before the root reuses
// it two launches later. Reference: Runtime.bcast (runtime.py:528-532).
__device__ __forceinline__ void mm_st_release_u64(uint64_t* mc, uint64_t v) {
  asm volatile("multimem.st.release.sys.global.u64 [%0], %1;" ::"l"(mc), "l"(v) : "memory");
}

// Byte-wise pack access for unaligned user buffers and the final partial
// pack (the protocol choice must not depend on a rank's own alignment).
__device__ __forceinline__ uint4 ld_bytes16(const uint8_t* p, int64_t valid) {
  uint4 v = make_uint4(0, 0, 0, 0);
  uint8_t* b = reinterpret_cast<uint8_t*>(&v);
  for (int k = 0; k < 16 && k < valid; ++k) b[k] = p[k];
  return v;
}
__device__ __forceinline__ void st_bytes16(uint8_t* p, const uint4& v, int64_t valid) {
  const uint8_t* b = reinterpret_cast<const uint8_t*>(&v);
  for (int k = 0; k < 16 && k < valid; ++k) p[k] = b[k];
}

__device__ __forceinline__ void bcast_nvls_body(DevComm c, uint8_t* uc, uint8_t* mc,
                                                const uint64_t* uc_flags, uint64_t* mc_flags,
                                                uint8_t* buf, int64_t nbytes, int root,
                                                int64_t chp, uint32_t epoch, uint32_t sig) {
  __shared__ int s_err;
  __shared__ SComm S;
  const int rank = c.rank, world = c.world, par = epoch & 1;
  const int s = int(blockIdx.x), G = int(gridDim.x), tid = threadIdx.x, nt = blockDim.x;
  const int64_t npk = (nbytes + 15) / 16;
  // full packs reachable with 16-byte accesses (0 when buf is unaligned)
  const int64_t nfast = (reinterpret_cast<uintptr_t>(buf) & 15) ? 0 : nbytes / 16;
  const int64_t pb = npk * s / G, pe = npk * (s + 1) / G;
  const int rows = int((pe - pb + chp - 1) / chp);
  if (tid == 0) s_err = 0;
  stage_comm(c, S);
  __syncthreads();
  if (rank == root) {
    for (int r = 0; r < rows; ++r) {
      const int64_t lo = pb + int64_t(r) * chp, hi = min(pe, lo + chp);
      const int64_t hf = max(lo, min(hi, nfast));
      int64_t i = lo + tid;
      for (; i + 3 * nt < hf; i += 4 * nt) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = ld16(buf + (i + u * nt) * 16);
#pragma unroll
        for (int u = 0; u < 4; ++u) mm_st(mc + (i + u * nt) * 16, v[u]);
      }
      for (; i < hf; i += nt) mm_st(mc + i * 16, ld16(buf + i * 16));
      for (i = hf + tid; i < hi; i += nt) mm_st(mc + i * 16, ld_bytes16(buf + i * 16, nbytes - i * 16));
      __syncthreads();
      if (tid == 0) mm_st_release_u64(mc_flags + s, make_flag(epoch, sig, uint32_t(r + 1)));
    }
    if (tid < world && tid != root) {
      int e = wait_flag(&S.pad[rank]->flag2[par][s][tid], S.pad[rank], c.timeout_ns, c.err, epoch,
                        sig, 1);
      if (e) atomicCAS(&s_err, 0, e);
    }
    __syncthreads();
    if (s_err && tid == 0) raise_error(S.pad, world, c.err, s_err, epoch);
    return;
  }
  for (int r = 0; r < rows; ++r) {
    if (tid == 0) {
      int e = wait_flag(uc_flags + s, S.pad[rank], c.timeout_ns, c.err, epoch, sig, uint32_t(r + 1));
      if (e) s_err = e;
    }
    __syncthreads();
    if (s_err) {
      if (tid == 0) raise_error(S.pad, world, c.err, s_err, epoch);
      return;
    }
    const int64_t lo = pb + int64_t(r) * chp, hi = min(pe, lo + chp);
    const int64_t hf = max(lo, min(hi, nfast));
    int64_t i = lo + tid;
    for (; i + 3 * nt < hf; i += 4 * nt) {
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = ld16_cg(uc + (i + u * nt) * 16);
#pragma unroll
      for (int u = 0; u < 4; ++u) st16(buf + (i + u * nt) * 16, v[u]);
    }
    for (; i < hf; i += nt) st16(buf + i * 16, ld16_cg(uc + i * 16));
    for (i = hf + tid; i < hi; i += nt) st_bytes16(buf + i * 16, ld16_cg(uc + i * 16), nbytes - i * 16);
  }
  __syncthreads();
  if (tid == 0) publish(&S.pad[root]->flag2[par][s][rank], make_flag(epoch, sig, 1));
}

__global__ void __launch_bounds__(kThreads)
    k_bcast_nvls(DevComm c, uint8_t* uc, uint8_t* mc, int64_t nv_half, int64_t room, uint8_t* buf,
                 int64_t nbytes, int root, int64_t chp, uint32_t sig) {
  const uint32_t epoch = epoch_enter(c);
  const int64_t hoff = int64_t(epoch & 1) * nv_half;
  bcast_nvls_body(c, uc + hoff, mc + hoff, reinterpret_cast<const uint64_t*>(uc + hoff + room),
                  reinterpret_cast<uint64_t*>(mc + hoff + room), buf, nbytes, root, chp, epoch, sig);
  epoch_exit(c, epoch);
}

mcrdl_status_t launch_bcast_nvls(mcrdl_comm* c, uint8_t* buf, int64_t nbytes, int root, int dtype,
                                 uint64_t count, uint64_t seq, cudaStream_t stream) {
  const int64_t nv_half = int64_t(c->nvls.bytes / 2);
  const int64_t room = (nv_half - kNvlsFlagBytes) / 256 * 256;
  uint8_t* uc = reinterpret_cast<uint8_t*>(c->nvls.uc_ptr);
  uint8_t* mc = reinterpret_cast<uint8_t*>(c->nvls.mc_ptr);
  int64_t done = 0;
  int sub = 0;
  do {
    const int64_t nb = std::min(nbytes - done, room);
    mcrdl_status_t st = begin_op(c, stream);
    if (st != MCRDL_OK) return st;
    const uint32_t sig = op_sig(kKindBcast, dtype, sub, root, count, seq);
    const int64_t npk = (nb + 15) / 16;
    static const int64_t bc_ctas = env_int("MCRDL_BCAST_CTAS", 0);
    static const int64_t bc_chunk_kb = env_int("MCRDL_BCAST_CHUNK_KB", 256);
    // measured (tools/bcast_knobs.sh, p=4): 74 CTAs best at 16 MiB, 32 at 256 MiB
    const int64_t gdef = nb >= (int64_t(64) << 20) ? 32 : c->num_sms / 2;
    int64_t g = (nb + (256 << 10) - 1) / (256 << 10);
    g = std::max<int64_t>(1, std::min<int64_t>(g, bc_ctas > 0 ? bc_ctas : gdef));
    int64_t chp = ((npk + g - 1) / g + 3999) / 4000;  // <= 4000 chunks per share
    if (chp < bc_chunk_kb * 64) chp = bc_chunk_kb * 64;
    k_bcast_nvls<<<int(g), kThreads, 0, stream>>>(c->dc, uc, mc, nv_half, room, buf + done, nb,
                                                  root, chp, sig);
    count_launch();
    MCRDL_CUDA_CHECK(cudaGetLastError());
    done += nb;
    ++sub;
  } while (done < nbytes);
  return MCRDL_OK;
}

// ------------------------------------------------------------ chain bcast
// Large bcast as a pipelined chain root -> root+1 -> ... -> root+p-1 (at p = 2
// just root -> peer, still ahead of the exchange push: 128 CTAs, no
// receiver role, the copy-out fused per chunk): chunk j
// is pushed into the next rank's workspace as soon as it landed in this
// rank's, so every link carries S once and the root's egress is S (direct
// write pushes (p-1)·S from the root; NVLS is bound by one GPU's multicast
// stores). Each rank: NVLink ingress S + egress S, HBM ws -> buf copy fused
// with the forward (one load, two stores).
// Workspace reuse: every CTA first exchanges a start flag with EVERY peer, so
// finishing op e proves each peer started op e (the all-pairs guarantee the
// exchange engine relies on, §7 "Why bcast keeps an all-pairs handshake").
__device__ __forceinline__ void copy2(uint8_t* d1, uint8_t* d2, const uint8_t* src, int64_t n) {
  const int tid = threadIdx.x, nt = blockDim.x;
  int64_t done = 0;
  if (((uintptr_t(d1) | uintptr_t(d2) | uintptr_t(src)) & 15) == 0) {
    const int64_t np = n >> 4;
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    uint4* a4 = reinterpret_cast<uint4*>(d1);
    uint4* b4 = reinterpret_cast<uint4*>(d2);
    constexpr int U = 4;
    int64_t i = tid;
    for (; i + (U - 1) * nt < np; i += U * nt) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = __ldcg(s4 + i + u * nt);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        a4[i + u * nt] = v[u];
        b4[i + u * nt] = v[u];
      }
    }
    for (; i < np; i += nt) {
      const uint4 v = __ldcg(s4 + i);
      a4[i] = v;
      b4[i] = v;
    }
    done = np << 4;
  }
  for (int64_t i = done + tid; i < n; i += nt) {
    const uint8_t v = src[i];
    d1[i] = v;
    d2[i] = v;
  }
}

__global__ void __launch_bounds__(kThreads)
    k_bcast_chain(DevComm c, uint8_t* buf, int64_t nb, int root, int64_t chunk, uint32_t sig) {
  const uint32_t epoch = epoch_enter(c);
  __shared__ SComm S;
  __shared__ int s_err;
  const int par = epoch & 1, rank = c.rank, world = c.world, tid = threadIdx.x;
  const int b = blockIdx.x;
  const int pos = (rank - root + world) % world;
  const int pred = (rank - 1 + world) % world, succ = (rank + 1) % world;
  const bool last = pos == world - 1;
  const int64_t hoff = int64_t(par) * c.half_bytes;
  if (tid == 0) s_err = 0;
  stage_comm(c, S);
  __syncthreads();
  // all-pairs start handshake (per CTA)
  if (tid < world && tid != rank) {
    publish(&S.pad[tid]->ack[par][b][rank], make_flag(epoch, sig, 1));
    const int e = wait_flag(&S.pad[rank]->ack[par][b][tid], S.pad[rank], c.timeout_ns, c.err,
                            epoch, sig, 1);
    if (e) atomicCAS(&s_err, 0, e);
  }
  __syncthreads();
  if (s_err) {
    if (tid == 0) raise_error(S.pad, world, c.err, s_err, epoch);
    epoch_exit(c, epoch);
    return;
  }
  uint8_t* my_ws = S.ws[rank] + hoff;
  uint8_t* succ_ws = S.ws[succ] + hoff;
  const int64_t nch = (nb + chunk - 1) / chunk;
  uint32_t step = 0;
  for (int64_t j = b; j < nch; j += gridDim.x) {
    const int64_t lo = j * chunk, len = min(chunk, nb - lo);
    ++step;
    if (pos == 0) {
      block_copy<4>(succ_ws + lo, buf + lo, len);
    } else {
      if (tid == 0) {
        const int e = wait_flag(&S.pad[rank]->flag[par][b][pred], S.pad[rank], c.timeout_ns,
                                c.err, epoch, sig, step);
        if (e) s_err = e;
      }
      __syncthreads();
      if (s_err) {
        if (tid == 0) raise_error(S.pad, world, c.err, s_err, epoch);
        break;
      }
      if (last)
        block_copy<4>(buf + lo, my_ws + lo, len);
      else
        copy2(succ_ws + lo, buf + lo, my_ws + lo, len);
    }
    if (!last) {
      __syncthreads();
      if (tid == 0) publish(&S.pad[succ]->flag[par][b][rank], make_flag(epoch, sig, step));
    }
  }
  epoch_exit(c, epoch);
}

mcrdl_status_t launch_bcast_chain(mcrdl_comm* c, uint8_t* buf, int64_t nbytes, int root,
                                  int dtype, uint64_t count, uint64_t seq, cudaStream_t stream) {
  // 128 CTAs x 128 KiB chunks (profiles/r2_bcast_chain_ab.csv, p = 4: 1 GiB
  // 644 GB/s, 256 MiB 537; 256 KiB chunks deepen the pipeline fill, 64 KiB
  // ones cost flag round trips at 1 GiB). Knobs: every rank must agree
  // (folded into the flag signature).
  static const int64_t ch_ctas = env_int("MCRDL_BCAST_CHAIN_CTAS", 128);
  static const int64_t ch_kb = env_int("MCRDL_BCAST_CHAIN_KB", 128);
  const int64_t chunk = std::max<int64_t>(16, ch_kb) << 10;
  const int64_t room = c->dc.half_bytes / 256 * 256;
  int64_t done = 0;
  int sub = 0;
  do {
    const int64_t nb = std::min(nbytes - done, room);
    mcrdl_status_t st = begin_op(c, stream);
    if (st != MCRDL_OK) return st;
    // CTAs and chunk (<= kMaxSteps chunks per CTA: 12-bit flag steps), geometry.h
    const ChainGeo geo = chain_geo(nb, chunk, ch_ctas, c->num_sms, kMaxBlocks);
    const int64_t g = geo.g, ch = geo.ch;
    const uint32_t sig = mix32(mix32(mix32(op_sig(kKindBcast, dtype, sub, root, count, seq),
                                           uint64_t(MCRDL_ALGO_CHAIN)),
                                     uint64_t(ch)),
                               uint64_t(g)) &
                         ~kSigCodecBit;
    k_bcast_chain<<<int(g), kThreads, 0, stream>>>(c->dc, buf + done, nb, root, ch, sig);
    count_launch();
    MCRDL_CUDA_CHECK(cudaGetLastError());
    done += nb;
    ++sub;
  } while (done < nbytes);
  return MCRDL_OK;
}

// ------------------------------------------------------------- fused (K9)
// Members laid out back to back in a virtual packed buffer (element offsets
// d_off[m], 16-byte aligned). One-shot protocol over the packed index space:
// phase 1 packs member inputs straight into every peer's workspace; phase 2
// folds and unpacks straight into member outputs. No staging buffer, one
// launch (reference: np.concatenate + all_reduce + _scatter_back,
// middleware.py:316-341).
template <typename T, int OP>
__device__ __forceinline__ void ar_fused_body(DevComm c, const T* const* in_ptrs, T* const* out_ptrs, const int64_t* counts,
               const int64_t* offs, int nmem, int64_t total, int64_t slot_bytes, uint32_t epoch,
               uint32_t sig) {
  constexpr int N = Pack<T>::N;
  __shared__ int s_err;
  __shared__ SComm S;
  __shared__ int s_m0;
  const int par = epoch & 1, rank = c.rank, world = c.world;
  const int b = blockIdx.x, G = gridDim.x, tid = threadIdx.x, nt = blockDim.x;
  const int64_t npk = (total + N - 1) / N;
  const int64_t pb = npk * b / G, pe = npk * (b + 1) / G;
  const int64_t hoff = int64_t(par) * c.half_bytes;
  if (tid == 0) {
    s_err = 0;
    // first member whose packed range ends after pb
    int lo = 0, hi = nmem;
    while (lo < hi) {
      int mid = (lo + hi) / 2;
      if ((offs[mid] + counts[mid] + N - 1) / N <= pb) lo = mid + 1;
      else hi = mid;
    }
    s_m0 = lo;
  }
  stage_comm(c, S);
  __syncthreads();
  const int m0 = s_m0;

  for (int m = m0; m < nmem; ++m) {
    const int64_t mp0 = offs[m] / N;                      // member's first pack
    const int64_t mpn = (counts[m] + N - 1) / N;          // member packs
    if (mp0 >= pe) break;
    const int64_t a = max(pb, mp0), z = min(pe, mp0 + mpn);
    const T* src = in_ptrs[m];
    const bool vec = (uintptr_t(src) & 15) == 0;
    for (int64_t i = a + tid; i < z; i += nt) {
      const uint4 v = vec ? load_pack<T, true>(src, i - mp0, counts[m])
                          : load_pack<T, false>(src, i - mp0, counts[m]);
      for (int k = 1; k < world; ++k) {
        const int q = (rank + k) % world;
        st16(S.ws[q] + hoff + int64_t(rank) * slot_bytes + i * 16, v);
      }
    }
  }
  __syncthreads();
  if (tid < world && tid != rank) publish(&S.pad[tid]->flag[par][b][rank], make_flag(epoch, sig, 0));
  if (tid < world && tid != rank) {
    int e = wait_flag(&S.pad[rank]->flag[par][b][tid], S.pad[rank], c.timeout_ns, c.err, epoch, sig, 0);
    if (e) atomicCAS(&s_err, 0, e);
  }
  __syncthreads();
  if (s_err) {
    if (tid == 0) raise_error(S.pad, world, c.err, s_err, epoch);
    return;
  }
  const uint8_t* ws = S.ws[rank] + hoff;
  for (int m = m0; m < nmem; ++m) {
    const int64_t mp0 = offs[m] / N;
    const int64_t mpn = (counts[m] + N - 1) / N;
    if (mp0 >= pe) break;
    const int64_t a = max(pb, mp0), z = min(pe, mp0 + mpn);
    const T* src = in_ptrs[m];
    T* dst = out_ptrs[m];
    const int64_t cnt = counts[m];
    const bool vec = ((uintptr_t(src) | uintptr_t(dst)) & 15) == 0;
    for (int64_t i = a + tid; i < z; i += nt) {
      const int64_t li = i - mp0;
      Pack<T> acc;
      auto own = [&]() {
        return vec ? load_pack<T, true>(src, li, cnt) : load_pack<T, false>(src, li, cnt);
      };
      uint4 raw[kMaxRanks];  // every rank's pack loaded before the first fold
#pragma unroll
      for (int r = 0; r < kMaxRanks; ++r)
        if (r < world) raw[r] = (r == rank) ? own() : ld16_cg(ws + int64_t(r) * slot_bytes + i * 16);
      acc.from_raw(raw[0]);
#pragma unroll
      for (int r = 1; r < kMaxRanks; ++r)
        if (r < world) acc.template fold<OP>(raw[r]);
      if (vec) store_pack<T, true>(dst, li, cnt, acc.to_raw());
      else store_pack<T, false>(dst, li, cnt, acc.to_raw());
    }
  }
}

template <typename T, int OP>
__global__ void __launch_bounds__(kThreads) k_ar_fused(DevComm c, const T* const* in_ptrs, T* const* out_ptrs, const int64_t* counts,
               const int64_t* offs, int nmem, int64_t total, int64_t slot_bytes, uint32_t sig) {
  const uint32_t epoch = epoch_enter(c);
  ar_fused_body<T, OP>(c, in_ptrs, out_ptrs, counts, offs, nmem, total, slot_bytes, epoch, sig);
  epoch_exit(c, epoch);
}

// Local copy used for world == 1 (the p = 1 floor: out[:] = in).
// One 16 KiB tile per CTA (512 threads x 2 x 16 B, both loads issued before
// the stores), no grid-stride loop: tools/copy_probe2.cu on B200, 256 MiB back
// to back: 6.68 TB/s read+write against 5.94 for the former grid-stride
// kernel (16 x SMs CTAs, whose single-load tail loop ran most of the copy)
// and 6.38 for cudaMemcpyAsync D2D.
constexpr int kCopyUnroll = 2;
constexpr int64_t kCopyTile = int64_t(kThreads) * kCopyUnroll * 16;
__global__ void __launch_bounds__(kThreads) k_copy(uint8_t* dst, const uint8_t* src, int64_t n) {
  if (((uintptr_t(dst) | uintptr_t(src)) & 15) != 0) {
    int64_t s, e;
    byte_share(n, blockIdx.x, gridDim.x, s, e);
    block_copy<4>(dst + s, src + s, e - s);
    return;
  }
  const int64_t np = n >> 4;
  const uint4* s4 = reinterpret_cast<const uint4*>(src);
  uint4* d4 = reinterpret_cast<uint4*>(dst);
  const int64_t base = int64_t(blockIdx.x) * (kThreads * kCopyUnroll) + threadIdx.x;
  uint4 v[kCopyUnroll];
#pragma unroll
  for (int u = 0; u < kCopyUnroll; ++u)
    if (base + u * kThreads < np) v[u] = s4[base + u * kThreads];
#pragma unroll
  for (int u = 0; u < kCopyUnroll; ++u)
    if (base + u * kThreads < np) d4[base + u * kThreads] = v[u];
  if (blockIdx.x == gridDim.x - 1)
    for (int64_t k = (np << 4) + threadIdx.x; k < n; k += blockDim.x) dst[k] = src[k];
}

// ----------------------------------------------------------------- launch
static int grid_for(int64_t packs, int num_sms, int max_blocks) {
  // ~2 packs per thread per block for small messages, up to 2 CTAs per SM.
  int64_t g = (packs + int64_t(kThreads) * 2 - 1) / (int64_t(kThreads) * 2);
  int cap = max_blocks;
  if (cap > 2 * num_sms) cap = 2 * num_sms;
  if (cap > kMaxBlocks) cap = kMaxBlocks;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return int(g);
}

mcrdl_status_t launch_local_copy(void* dst, const void* src, int64_t nbytes, int num_sms,
                                 cudaStream_t stream) {
  if (nbytes <= 0 || dst == src) return MCRDL_OK;
  // aligned: one tile per CTA; misaligned: byte shares over 16 CTAs per SM
  const bool aligned = ((uintptr_t(dst) | uintptr_t(src)) & 15) == 0;
  int64_t g = aligned ? (nbytes + kCopyTile - 1) / kCopyTile : int64_t(16) * num_sms;
  if (!aligned && g > (nbytes + 4095) / 4096) g = (nbytes + 4095) / 4096;
  if (g < 1) g = 1;
  if (g > INT32_MAX) return set_error(MCRDL_ERR_VALIDATION, "local copy too large");
  k_copy<<<int(g), kThreads, 0, stream>>>(reinterpret_cast<uint8_t*>(dst),
                                          reinterpret_cast<const uint8_t*>(src), nbytes);
  count_launch();
  MCRDL_CUDA_CHECK(cudaGetLastError());
  return MCRDL_OK;
}

// LL threshold for one-shot all_reduce (MCRDL_LL_MAX_BYTES overrides).
static int64_t ll_max_bytes() {
  static int64_t v = [] {
    const char* e = getenv("MCRDL_LL_MAX_BYTES");
    const int64_t want = e ? int64_t(strtoll(e, nullptr, 10)) : kLLMaxAllReduceBytes;
    return want < kLLMaxPayload ? want : kLLMaxPayload;
  }();
  return v;
}

// ------------------------------------------ symmetric zero-copy all_reduce
// `in` and `out` lie in user symmetric allocations (mcrdl_symm_alloc) at the
// same offsets on every rank: no workspace and no staging copies. Rank q owns
// shard q of the packs:
//  NVLS: multimem.ld_reduce of shard q straight from the inputs' multicast
//        view, multimem.st straight into the outputs' (f32 / bf16 sum) —
//        HBM traffic 2·S instead of 6·S for the staged k_ar_nvls;
//  P2P:  ascending fold of shard q loaded from every rank's input over
//        NVLink, stored into every rank's output (any dtype / op, bit-exact).
// Per-CTA entry barrier (every peer entered: its input is final and nobody
// writes a rank's output before that rank's previous work ended) and exit
// barrier (every store into my output landed, every read of my input done).
struct SymmArgs {
  const uint8_t* in[kMaxRanks];
  uint8_t* out[kMaxRanks];
  const uint8_t* mc_in;
  uint8_t* mc_out;
};

template <typename T, int OP, bool VEC, bool NVLS>
__device__ __forceinline__ void ar_symm_body(DevComm c, const SymmArgs& a, int64_t n,
                                             uint32_t epoch, uint32_t sig) {
  constexpr int N = Pack<T>::N;
  __shared__ int s_err;
  __shared__ SComm S;
  __shared__ const T* s_in[kMaxRanks];
  __shared__ T* s_out[kMaxRanks];
  const int par = epoch & 1, rank = c.rank, world = c.world;
  const int s = int(blockIdx.x), G = int(gridDim.x), tid = threadIdx.x, nt = blockDim.x;
  if (tid == 0) {
    s_err = 0;
#pragma unroll
    for (int r = 0; r < kMaxRanks; ++r) {
      s_in[r] = reinterpret_cast<const T*>(a.in[r]);
      s_out[r] = reinterpret_cast<T*>(a.out[r]);
    }
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
  const int64_t npk = (n + N - 1) / N;
  const int64_t sp = (npk + world - 1) / world;
  const int64_t q0 = min(npk, int64_t(rank) * sp), q1 = min(npk, q0 + sp);
  const int64_t lo = q0 + (q1 - q0) * s / G, hi = q0 + (q1 - q0) * (s + 1) / G;
  if constexpr (NVLS) {
    int64_t i = lo + tid;
    for (; i + 3 * nt < hi; i += 4 * nt) {
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = mm_ld_reduce_sum<T>(a.mc_in + (i + u * nt) * 16);
#pragma unroll
      for (int u = 0; u < 4; ++u) mm_st(a.mc_out + (i + u * nt) * 16, v[u]);
    }
    for (; i < hi; i += nt) mm_st(a.mc_out + i * 16, mm_ld_reduce_sum<T>(a.mc_in + i * 16));
  } else {
    constexpr int RU = sizeof(T) == 2 ? 2 : 4;
    for (int64_t i0 = lo + tid; i0 < hi; i0 += RU * nt) {
      Pack<T> acc[RU];
      uint4 v[RU];
#pragma unroll
      for (int u = 0; u < RU; ++u)
        if (i0 + u * nt < hi) v[u] = load_pack<T, VEC>(s_in[0], i0 + u * nt, n);
#pragma unroll
      for (int u = 0; u < RU; ++u) acc[u].from_raw(v[u]);
      for (int q = 1; q < world; ++q) {
#pragma unroll
        for (int u = 0; u < RU; ++u)
          if (i0 + u * nt < hi) v[u] = load_pack<T, VEC>(s_in[q], i0 + u * nt, n);
#pragma unroll
        for (int u = 0; u < RU; ++u) acc[u].template fold<OP>(v[u]);
      }
#pragma unroll
      for (int u = 0; u < RU; ++u) {
        if (i0 + u * nt >= hi) break;
        const uint4 res = acc[u].to_raw();
        for (int k = 0; k < world; ++k) {
          const int q = (rank + k) % world;
          store_pack<T, VEC>(s_out[q], i0 + u * nt, n, res);
        }
      }
    }
  }
  __syncthreads();
  if (tid < world) publish(&S.pad[tid]->flag2[par][s][rank], make_flag(epoch, sig, 1));
  if (tid < world) {
    int e = wait_flag(&S.pad[rank]->flag2[par][s][tid], S.pad[rank], c.timeout_ns, c.err, epoch, sig,
                      1);
    if (e) atomicCAS(&s_err, 0, e);
  }
  __syncthreads();
  if (s_err && tid == 0) raise_error(S.pad, world, c.err, s_err, epoch);
}

template <typename T, int OP, bool VEC, bool NVLS>
__global__ void __launch_bounds__(kThreads) k_ar_symm(DevComm c, SymmArgs a, int64_t n, uint32_t sig) {
  const uint32_t epoch = epoch_enter(c);
  ar_symm_body<T, OP, VEC, NVLS>(c, a, n, epoch, sig);
  epoch_exit(c, epoch);
}

// Returns true (and *st) when the symmetric path took the op.
template <typename T, int OP>
static bool try_ar_symm(mcrdl_comm* c, const T* in, T* out, int64_t n, mcrdl_algo_t algo,
                        uint64_t seq, int dt, cudaStream_t stream, mcrdl_status_t* st) {
  static const int64_t symm_on = env_int("MCRDL_SYMM", 1);
  static const int64_t symm_ctas = env_int("MCRDL_SYMM_CTAS", 0);
  const int64_t bytes = n * int64_t(sizeof(T));
  if (!symm_on || c->world == 1 || bytes == 0) return false;
  uint64_t oi = 0, oo = 0;
  const Region* ri = find_symm(c, in, uint64_t(bytes), &oi);
  const Region* ro = find_symm(c, out, uint64_t(bytes), &oo);
  if (ri == nullptr || ro == nullptr) return false;
  // Measured (tools: tuner --symm, profiles/symm_*_p{2,4}.log): the extra
  // entry/exit barriers lose to LL / one-shot below ~2 MiB (8 MiB at p = 2,
  // where one-shot stays ahead longer); explicit one_shot keeps the standard
  // path too.
  const int64_t min_bytes = c->world == 2 ? (int64_t(8) << 20) : (int64_t(2) << 20);
  if (algo == MCRDL_ALGO_ONE_SHOT || (algo == MCRDL_ALGO_AUTO && bytes < min_bytes)) return false;
  SymmArgs a{};
  for (int q = 0; q < c->world; ++q) {
    a.in[q] = reinterpret_cast<const uint8_t*>(ri->ptr[q]) + oi;
    a.out[q] = reinterpret_cast<uint8_t*>(ro->ptr[q]) + oo;
  }
  const bool vec = ((oi | oo) & 15) == 0;
  constexpr bool kNvlsType = (sizeof(T) == 4 && T(0.5) != T(0)) || sizeof(T) == 2;
  // NVLS needs >= 3 ranks to pay off: at p = 2 its traffic (1.5 S per link
  // direction) exceeds the peer path's S (355 vs 610 GB/s at 1 GiB).
  const bool nv = kNvlsType && OP == MCRDL_SUM && ri->mc_ptr && ro->mc_ptr && vec &&
                  bytes % 16 == 0 &&
                  (algo == MCRDL_ALGO_NVLS || (algo == MCRDL_ALGO_AUTO && c->world >= 3));
  if (nv) {
    a.mc_in = reinterpret_cast<const uint8_t*>(ri->mc_ptr) + oi;
    a.mc_out = reinterpret_cast<uint8_t*>(ro->mc_ptr) + oo;
  }
  // signature folds the buffer offsets: ranks passing different slices of
  // the symmetric allocation fail with ORDER_MISMATCH instead of mixing data
  uint32_t sig = op_sig(kKindAllReduce, dt, OP, nv ? -3 : -2, uint64_t(n), seq);
  sig = mix32(mix32(sig, oi), oo) & ~kSigCodecBit;
  if ((*st = begin_op(c, stream)) != MCRDL_OK) return true;
  c->last_algo[MCRDL_TUNE_ALL_REDUCE] = nv ? MCRDL_ALGO_NVLS : MCRDL_ALGO_DIRECT_WRITE;  // zero-copy
  constexpr int N = Pack<T>::N;
  const int64_t shard = ((n + N - 1) / N + c->world - 1) / c->world * 16;  // bytes per rank
  // CTAs: the switch path peaks with ~32 (p = 4: 656 GB/s at 256 MiB vs 566
  // with 148); the peer path wants every SM (576 vs 532 with 32).
  int64_t g = (shard + (64 << 10) - 1) / (64 << 10);
  g = std::max<int64_t>(1, std::min<int64_t>(g, symm_ctas > 0 ? symm_ctas : nv ? 32 : c->num_sms));
  if constexpr (kNvlsType && OP == MCRDL_SUM) {
    if (nv) {
      k_ar_symm<T, OP, true, true><<<int(g), kThreads, 0, stream>>>(c->dc, a, n, sig);
      count_launch();
      *st = cudaGetLastError() == cudaSuccess ? MCRDL_OK
                                               : set_error(MCRDL_ERR_CUDA, "k_ar_symm launch failed");
      return true;
    }
  }
  if (vec)
    k_ar_symm<T, OP, true, false><<<int(g), kThreads, 0, stream>>>(c->dc, a, n, sig);
  else
    k_ar_symm<T, OP, false, false><<<int(g), kThreads, 0, stream>>>(c->dc, a, n, sig);
  count_launch();
  *st = cudaGetLastError() == cudaSuccess ? MCRDL_OK
                                           : set_error(MCRDL_ERR_CUDA, "k_ar_symm launch failed");
  return true;
}

template <typename T, int OP>
static mcrdl_status_t ar_typed(mcrdl_comm* c, const T* in, T* out, int64_t n, mcrdl_algo_t algo,
                               uint64_t seq, int dt, cudaStream_t stream, int root = -1) {
  constexpr int N = Pack<T>::N;
  const int world = c->world;
  const int64_t half = c->dc.half_bytes;
  const bool vec = ((uintptr_t(in) | uintptr_t(out)) & 15) == 0;
  // p = 1: AUTO is the local copy; an explicitly requested algorithm runs its
  // real kernel (no peers: flags and folds degenerate to the own input), so
  // every kernel can be exercised and profiled on a single GPU.
  if (world == 1 && algo != MCRDL_ALGO_ONE_SHOT && algo != MCRDL_ALGO_TWO_SHOT)
    return launch_local_copy(out, in, n * int64_t(sizeof(T)), c->num_sms, stream);
  if (root < 0) {
    mcrdl_status_t sst;
    if (try_ar_symm<T, OP>(c, in, out, n, algo, seq, dt, stream, &sst)) return sst;
  } else {
    algo = MCRDL_ALGO_TWO_SHOT;  // reduce: RS + gather to the root (k_ar_pipe root mode)
  }
  const int64_t bytes = n * int64_t(sizeof(T));
  const int64_t oneshot_max = half / world / 256 * 256;
  // AUTO: the installed tuning table first (mcrdl_comm_set_tuning), then the
  // built-in crossovers
  if (algo == MCRDL_ALGO_AUTO) algo = tuned_algo(c, MCRDL_TUNE_ALL_REDUCE, uint64_t(bytes));
  if (algo == MCRDL_ALGO_AUTO) {
    // Crossovers measured by the tuner on B200 (profiles/tune_p{2,4}.csv):
    // one-shot pushes (p-1)*S, two-shot 2(p-1)/p*S, so it wins longer at small p.
    const int64_t thr = world == 2 ? (int64_t(8) << 20) : world <= 4 ? (int64_t(2) << 20)
                                                                      : (int64_t(1) << 20);
    algo = bytes <= thr ? MCRDL_ALGO_ONE_SHOT : MCRDL_ALGO_TWO_SHOT;
    // NVLS for large f32/bf16 sums: its link traffic is (1 + 1/p)·S against
    // 2(p-1)/p·S for two-shot. Measured at p = 4 (profiles/nvls_vs_twoshot_r1_p4.csv,
    // full_sweep_r1_p4.csv): ahead from ~256 MiB (582-592 vs 540-572 GB/s),
    // behind at 64 MiB; at p >= 6 the traffic ratio (1.125 vs 1.75 at p = 8)
    // moves the crossover down, taken here as 16 MiB.
    const int64_t nvls_thr = world >= 6 ? (int64_t(16) << 20) : (int64_t(128) << 20);
    if (world >= 4 && bytes >= nvls_thr) algo = MCRDL_ALGO_NVLS;
  }
  // NVLS: the switch reduces; sum of f32/bf16 only, and only when every rank
  // built the multicast object (caps.nvls_supported). Otherwise two-shot.
  constexpr bool kNvlsType = (sizeof(T) == 4 && T(0.5) != T(0)) || sizeof(T) == 2;
  if (algo == MCRDL_ALGO_NVLS && !(kNvlsType && OP == MCRDL_SUM && c->nvls.ok))
    algo = MCRDL_ALGO_TWO_SHOT;
  if (algo == MCRDL_ALGO_ONE_SHOT && bytes > oneshot_max) algo = MCRDL_ALGO_TWO_SHOT;
  if (algo >= MCRDL_ALGO_DIRECT_WRITE || algo == MCRDL_ALGO_AUTO) algo = MCRDL_ALGO_TWO_SHOT;
  if (root < 0) c->last_algo[MCRDL_TUNE_ALL_REDUCE] = int(algo);

  // Host chunking keeps every launch inside one workspace (or NVLS) half.
  const int64_t room =
      (algo == MCRDL_ALGO_NVLS) ? int64_t(c->nvls.bytes / 2) - kNvlsFlagBytes : half / 2;
  const int64_t chunk_elems = (algo == MCRDL_ALGO_ONE_SHOT)
                                  ? n
                                  : ((room - int64_t(world) * 1024) / int64_t(sizeof(T))) /
                                        (int64_t(world) * 4 * N) * (int64_t(world) * 4 * N);
  int64_t done = 0;
  int sub = 0;
  do {
    const int64_t m = (n - done < chunk_elems) ? (n - done) : chunk_elems;
    mcrdl_status_t st = begin_op(c, stream);
    if (st != MCRDL_OK) return st;
    // the algorithm is part of the agreement: ranks that resolved AUTO
    // differently (different tuning rows) raise ORDER_MISMATCH
    const uint32_t sig =
        mix32(root < 0 ? op_sig(kKindAllReduce, dt, OP, sub, uint64_t(m), seq)
                       : mix32(op_sig(kKindReduce, dt, OP, sub, uint64_t(m), seq), uint64_t(root)),
              uint64_t(algo)) &
        ~kSigCodecBit;
    const T* ip = in + done;
    T* op = out + done;
    const int64_t npk = (m + N - 1) / N;
    if (algo == MCRDL_ALGO_ONE_SHOT && m * int64_t(sizeof(T)) <= ll_max_bytes()) {
      // LL vs bulk one-shot is part of the agreement (MCRDL_LL_MAX_BYTES)
      st = launch_ar_ll<T, OP>(c, ip, op, m, mix32(sig, 0x4C4Cu) & ~kSigCodecBit, stream);
      if (st != MCRDL_OK) return st;
      done += m;
      ++sub;
      continue;
    }
    if (algo == MCRDL_ALGO_ONE_SHOT) {
      const int64_t slot = (npk * 16 + 255) / 256 * 256;
      // one pack per thread up to 128 CTAs (profiles/r2_oneshot_geo_ab.csv:
      // p = 4 8 MiB 61.6 -> 56.8 us, 1 MiB 20.3 -> 19.9 against 64 CTAs x 2
      // packs; MCRDL_AR_ONESHOT_CTAS / _PPT override)
      static const int64_t os_ctas = env_int("MCRDL_AR_ONESHOT_CTAS", 128);
      static const int64_t os_ppt = env_int("MCRDL_AR_ONESHOT_PPT", 1);
      const int G = grid_for((npk * 2 + os_ppt - 1) / (os_ppt > 0 ? os_ppt : 1), c->num_sms,
                             int(os_ctas > 0 ? os_ctas : 128));
      const uint32_t gsig = mix32(sig, uint64_t(G)) & ~kSigCodecBit;  // flags are per CTA
      if (vec)
        k_ar_oneshot<T, OP, true><<<G, kThreads, 0, stream>>>(c->dc, ip, op, m, slot, gsig);
      else
        k_ar_oneshot<T, OP, false><<<G, kThreads, 0, stream>>>(c->dc, ip, op, m, slot, gsig);
    } else {
      // CTAs per role: one per 32 KiB of segment; 3 roles x gp <= 2 CTAs/SM
      // (MCRDL_AR_GPMAX / MCRDL_AR_CHUNK_KB override, for tuning).
      static const int64_t gp_env = env_int("MCRDL_AR_GPMAX", 0);
      // Flag chunk: 256 KiB, but 128 KiB for mid-size launches at p >= 4 so a
      // CTA share spans several rows and RS / AG overlap (tools/chunk_ab.sh,
      // profiles/chunk_ab_r1_p{2,4}.log: p = 4, 64 MiB 464 vs 439 GB/s; 256 MiB
      // and p = 2 prefer 256 KiB). MCRDL_AR_CHUNK_KB overrides.
      static const int64_t chunk_env = env_int("MCRDL_AR_CHUNK_KB", 0);
      const int64_t chunk_kb =
          chunk_env > 0 ? chunk_env
                        : (world >= 4 && m * int64_t(sizeof(T)) < (int64_t(128) << 20) ? 128 : 256);
      // RS senders on TMA bulk copies for large launches (aligned buffers):
      // measured +2-3% at >= 256 MiB, slower below 64 MiB (profiles/tma_ab_r1.log).
      // MCRDL_AR_TMA=0 disables, =2 forces; MCRDL_AR_TMA_CTAS sets the sender CTAs.
      static const int64_t tma_on = env_int("MCRDL_AR_TMA", 1);
      static const int64_t tma_ctas = env_int("MCRDL_AR_TMA_CTAS", 64);
      const bool big = m * int64_t(sizeof(T)) >= (int64_t(256) << 20);
      // Share geometry (shares, chunk) comes only from values every rank
      // agrees on (size, SM budget, env); buffer alignment only picks the
      // sender flavour (geometry.h two_shot_geo).
      const bool tma_geo = algo != MCRDL_ALGO_NVLS && (tma_on == 2 || (tma_on == 1 && big));
      const TwoShotGeo geo =
          two_shot_geo(npk, world, c->num_sms, chunk_kb, tma_geo, gp_env, tma_ctas, kMaxBlocks);
      const int64_t sp = geo.sp, segb = geo.segb, gp = geo.gp;
      bool launched = false;
      if constexpr (kNvlsType && OP == MCRDL_SUM) {
        if (algo == MCRDL_ALGO_NVLS) {
          // the kernel picks the multicast half by its device epoch's parity
          const int64_t nv_half = int64_t(c->nvls.bytes / 2);
          uint8_t* uc = reinterpret_cast<uint8_t*>(c->nvls.uc_ptr);
          uint8_t* mc = reinterpret_cast<uint8_t*>(c->nvls.mc_ptr);
          // Measured (tools/nvls_knobs.sh, profiles/nvls_knobs_r1_p4.log): the
          // switch path peaks with ~32 CTAs per role (p=4, 256 MiB: 575 GB/s vs
          // 497 with 98), and the per-chunk system fence before the release
          // flag costs ~3% (multimem.st + bar.sync + st.release.sys is the
          // ordering the CUTLASS multimem all-reduce uses as well).
          static const int64_t nv_gp = env_int("MCRDL_NVLS_GP", 32);
          static const int fence = int(env_int("MCRDL_NVLS_FENCE", 0));
          // copier / gatherer CTAs: the staging copies are local HBM work with 8
          // packs in flight per thread; 16 each matched or beat 32 each
          // (profiles/nvls_roles_r1_p4.log: 592 vs 581 GB/s at 256 MiB)
          static const int64_t nv_gc = env_int("MCRDL_NVLS_GC", 16);
          static const int64_t nv_gg = env_int("MCRDL_NVLS_GG", 16);
          const int64_t gpn = std::max<int64_t>(1, std::min<int64_t>(gp, nv_gp));
          const int gcn = int(std::max<int64_t>(1, std::min<int64_t>(nv_gc > 0 ? nv_gc : gpn, gpn)));
          const int ggn = int(std::max<int64_t>(1, std::min<int64_t>(nv_gg > 0 ? nv_gg : gpn, gpn)));
          const int64_t chpn = chunk_packs(sp, gpn, chunk_kb);
          const int Gn = int(gcn + gpn + ggn);
          if (vec)
            k_ar_nvls<T, true><<<Gn, kThreads, 0, stream>>>(c->dc, uc, mc, nv_half, ip, op, m, sp,
                                                            int(gpn), gcn, ggn, chpn, fence, sig);
          else
            k_ar_nvls<T, false><<<Gn, kThreads, 0, stream>>>(c->dc, uc, mc, nv_half, ip, op, m, sp,
                                                             int(gpn), gcn, ggn, chpn, fence, sig);
          launched = true;
        }
      }
      if (!launched) {
        {
          const int gs = geo.gs;
          const int64_t shares = geo.shares, chs = geo.chp;
          // Any geometry disagreement (env knobs) fails as ORDER_MISMATCH
          // instead of folding bytes that have not landed.
          const uint32_t gsig = mix32(mix32(sig, uint64_t(shares)), uint64_t(chs)) & ~kSigCodecBit;
          if (tma_geo && vec) {
            k_ar_pipe<T, OP, true, true><<<int(gs + 2 * shares), kThreads, 0, stream>>>(
                c->dc, ip, op, m, sp, segb, int(shares), gs, chs, root, gsig);
          } else if (vec) {
            k_ar_pipe<T, OP, true, false><<<int(3 * shares), kThreads, 0, stream>>>(
                c->dc, ip, op, m, sp, segb, int(shares), int(shares), chs, root, gsig);
          } else {
            k_ar_pipe<T, OP, false, false><<<int(3 * shares), kThreads, 0, stream>>>(
                c->dc, ip, op, m, sp, segb, int(shares), int(shares), chs, root, gsig);
          }
        }
      }
    }
    count_launch();
    MCRDL_CUDA_CHECK(cudaGetLastError());
    done += m;
    ++sub;
  } while (done < n);
  return MCRDL_OK;
}

template <typename T>
static mcrdl_status_t ar_op(mcrdl_comm* c, const void* in, void* out, int64_t n, mcrdl_redop_t op,
                            mcrdl_algo_t algo, uint64_t seq, int dt, cudaStream_t s,
                            int root = -1) {
  const T* i = reinterpret_cast<const T*>(in);
  T* o = reinterpret_cast<T*>(out);
  switch (op) {
    case MCRDL_SUM: return ar_typed<T, MCRDL_SUM>(c, i, o, n, algo, seq, dt, s, root);
    case MCRDL_PROD: return ar_typed<T, MCRDL_PROD>(c, i, o, n, algo, seq, dt, s, root);
    case MCRDL_MIN: return ar_typed<T, MCRDL_MIN>(c, i, o, n, algo, seq, dt, s, root);
    case MCRDL_MAX: return ar_typed<T, MCRDL_MAX>(c, i, o, n, algo, seq, dt, s, root);
  }
  return set_error(MCRDL_ERR_VALIDATION, "unknown reduce op %d", int(op));
}

// reduce_scatter (reference _reduce_scatter_ring/_naive, collectives.py:609-645):
// the RS half of the two-shot pipeline; rank r's reduced segment (ascending
// fold, bit-exact) lands straight in its m-element output. Needs 16-byte
// aligned buffers, m*sizeof(T) % 16 == 0 and one workspace half; otherwise
// MCRDL_ERR_UNSUPPORTED (the caller composes all_reduce + slice).
template <typename T, int OP>
static mcrdl_status_t rs_typed(mcrdl_comm* c, const T* in, T* out, int64_t m, uint64_t seq, int dt,
                               cudaStream_t stream) {
  const int world = c->world;
  if (world == 1) return launch_local_copy(out, in, m * int64_t(sizeof(T)), c->num_sms, stream);
  const int64_t segbytes = m * int64_t(sizeof(T));
  if (((uintptr_t(in) | uintptr_t(out)) & 15) != 0 || segbytes % 16 != 0 ||
      2 * int64_t(world) * ((segbytes + 255) / 256 * 256) > c->dc.half_bytes)
    return set_error(MCRDL_ERR_UNSUPPORTED, "reduce_scatter kernel needs aligned 16-byte segments "
                                            "within one workspace half");
  mcrdl_status_t st = begin_op(c, stream);
  if (st != MCRDL_OK) return st;
  const uint32_t sig = op_sig(kKindReduceScatter, dt, OP, -1, uint64_t(m), seq);
  const int64_t sp = segbytes / 16;
  const int64_t segb = (sp * 16 + 255) / 256 * 256;
  int64_t gp = (segbytes + (32 << 10) - 1) / (32 << 10);
  gp = std::max<int64_t>(1, std::min<int64_t>(gp, 2 * c->num_sms / 3));
  int64_t chp = ((sp + gp - 1) / gp + 3999) / 4000;
  if (chp < 16384) chp = 16384;
  // senders + reducers only (reduce_scatter has no all-gather role)
  k_ar_pipe<T, OP, true, false><<<int(2 * gp), kThreads, 0, stream>>>(
      c->dc, in, out, int64_t(world) * m, sp, segb, int(gp), int(gp), chp, -1, sig, out, m);
  count_launch();
  MCRDL_CUDA_CHECK(cudaGetLastError());
  return MCRDL_OK;
}

template <typename T>
static mcrdl_status_t rs_op(mcrdl_comm* c, const void* in, void* out, int64_t m, mcrdl_redop_t op,
                            uint64_t seq, int dt, cudaStream_t s) {
  const T* i = reinterpret_cast<const T*>(in);
  T* o = reinterpret_cast<T*>(out);
  switch (op) {
    case MCRDL_SUM: return rs_typed<T, MCRDL_SUM>(c, i, o, m, seq, dt, s);
    case MCRDL_PROD: return rs_typed<T, MCRDL_PROD>(c, i, o, m, seq, dt, s);
    case MCRDL_MIN: return rs_typed<T, MCRDL_MIN>(c, i, o, m, seq, dt, s);
    case MCRDL_MAX: return rs_typed<T, MCRDL_MAX>(c, i, o, m, seq, dt, s);
  }
  return set_error(MCRDL_ERR_VALIDATION, "unknown reduce op %d", int(op));
}

template <typename T, int OP>
static mcrdl_status_t fused_typed(mcrdl_comm* c, const void* const* in_ptrs, void* const* out_ptrs,
                                  const int64_t* counts, const int64_t* offs, int nmem,
                                  int64_t total, uint64_t seq, int dt, cudaStream_t stream) {
  constexpr int N = Pack<T>::N;
  mcrdl_status_t st = begin_op(c, stream);
  if (st != MCRDL_OK) return st;
  const int64_t npk = (total + N - 1) / N;
  const int64_t slot = (npk * 16 + 255) / 256 * 256;
  if (slot * c->world > c->dc.half_bytes)
    return set_error(MCRDL_ERR_VALIDATION, "fused all_reduce of %lld elements exceeds workspace",
                     (long long)total);
  const uint32_t sig = op_sig(kKindAllReduce, dt, OP, -2, uint64_t(total), seq);
  const int G = grid_for(npk, c->num_sms, 64);
  k_ar_fused<T, OP><<<G, kThreads, 0, stream>>>(
      c->dc, reinterpret_cast<const T* const*>(in_ptrs), reinterpret_cast<T* const*>(out_ptrs), counts,
      offs, nmem, total, slot, sig);
  count_launch();
  MCRDL_CUDA_CHECK(cudaGetLastError());
  return MCRDL_OK;
}

template <typename T>
static mcrdl_status_t fused_op(mcrdl_comm* c, const void* const* ip, void* const* op_, const int64_t* cn,
                               const int64_t* of, int nm, int64_t total, mcrdl_redop_t op,
                               uint64_t seq, int dt, cudaStream_t s) {
  switch (op) {
    case MCRDL_SUM: return fused_typed<T, MCRDL_SUM>(c, ip, op_, cn, of, nm, total, seq, dt, s);
    case MCRDL_PROD: return fused_typed<T, MCRDL_PROD>(c, ip, op_, cn, of, nm, total, seq, dt, s);
    case MCRDL_MIN: return fused_typed<T, MCRDL_MIN>(c, ip, op_, cn, of, nm, total, seq, dt, s);
    case MCRDL_MAX: return fused_typed<T, MCRDL_MAX>(c, ip, op_, cn, of, nm, total, seq, dt, s);
  }
  return set_error(MCRDL_ERR_VALIDATION, "unknown reduce op %d", int(op));
}

}  // namespace mcrdl

using namespace mcrdl;

extern "C" {

mcrdl_status_t mcrdl_all_reduce(mcrdl_comm* c, const void* in, void* out, uint64_t count,
                                mcrdl_dtype_t dtype, mcrdl_redop_t op, mcrdl_algo_t algo,
                                uint64_t seq, void* stream) {
  if (c == nullptr) return set_error(MCRDL_ERR_NOT_INITIALIZED, "communicator is NULL");
  if (count == 0) return mcrdl_barrier(c, seq, stream);
  if (in == nullptr || out == nullptr) return set_error(MCRDL_ERR_VALIDATION, "NULL buffer");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t n = int64_t(count);
  switch (dtype) {
    case MCRDL_F32: return ar_op<float>(c, in, out, n, op, algo, seq, int(dtype), s);
    case MCRDL_F64: return ar_op<double>(c, in, out, n, op, algo, seq, int(dtype), s);
    case MCRDL_I32: return ar_op<int32_t>(c, in, out, n, op, algo, seq, int(dtype), s);
    case MCRDL_I64: return ar_op<int64_t>(c, in, out, n, op, algo, seq, int(dtype), s);
    case MCRDL_U8: return ar_op<uint8_t>(c, in, out, n, op, algo, seq, int(dtype), s);
    case MCRDL_BF16: return ar_op<__nv_bfloat16>(c, in, out, n, op, algo, seq, int(dtype), s);
  }
  return set_error(MCRDL_ERR_VALIDATION, "unknown dtype %d", int(dtype));
}

// reduce (runtime.py:519-526; collectives.py _reduce_linear/_binomial; oracle
// reference.py:27-33): the two-shot pipeline in root mode — reduce-scatter as
// for all_reduce, then every rank sends its reduced segment to the root only
// (non-roots move (p-1)/p·S + S/p instead of 2(p-1)/p·S; only the root's
// gatherers run). Ascending fold: bit-exact. out may be NULL off the root.
mcrdl_status_t mcrdl_reduce(mcrdl_comm* c, const void* in, void* out, uint64_t count,
                            mcrdl_dtype_t dtype, mcrdl_redop_t op, int root, mcrdl_algo_t algo,
                            uint64_t seq, void* stream) {
  (void)algo;
  if (c == nullptr) return set_error(MCRDL_ERR_NOT_INITIALIZED, "communicator is NULL");
  if (root < 0 || root >= c->world)
    return set_error(MCRDL_ERR_VALIDATION, "root %d outside world %d", root, c->world);
  if (count == 0) return mcrdl_barrier(c, seq, stream);
  if (in == nullptr || (out == nullptr && c->rank == root))
    return set_error(MCRDL_ERR_VALIDATION, "NULL buffer");
  if (out == nullptr) out = const_cast<void*>(in);  // never written off the root
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t n = int64_t(count);
  switch (dtype) {
    case MCRDL_F32: return ar_op<float>(c, in, out, n, op, algo, seq, int(dtype), s, root);
    case MCRDL_F64: return ar_op<double>(c, in, out, n, op, algo, seq, int(dtype), s, root);
    case MCRDL_I32: return ar_op<int32_t>(c, in, out, n, op, algo, seq, int(dtype), s, root);
    case MCRDL_I64: return ar_op<int64_t>(c, in, out, n, op, algo, seq, int(dtype), s, root);
    case MCRDL_U8: return ar_op<uint8_t>(c, in, out, n, op, algo, seq, int(dtype), s, root);
    case MCRDL_BF16: return ar_op<__nv_bfloat16>(c, in, out, n, op, algo, seq, int(dtype), s, root);
  }
  return set_error(MCRDL_ERR_VALIDATION, "unknown dtype %d", int(dtype));
}

mcrdl_status_t mcrdl_reduce_scatter(mcrdl_comm* c, const void* in, void* out, uint64_t recvcount,
                                    mcrdl_dtype_t dtype, mcrdl_redop_t op, mcrdl_algo_t algo,
                                    uint64_t seq, void* stream) {
  (void)algo;
  if (c == nullptr) return set_error(MCRDL_ERR_NOT_INITIALIZED, "communicator is NULL");
  if (recvcount == 0) return mcrdl_barrier(c, seq, stream);
  if (in == nullptr || out == nullptr) return set_error(MCRDL_ERR_VALIDATION, "NULL buffer");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t m = int64_t(recvcount);
  switch (dtype) {
    case MCRDL_F32: return rs_op<float>(c, in, out, m, op, seq, int(dtype), s);
    case MCRDL_F64: return rs_op<double>(c, in, out, m, op, seq, int(dtype), s);
    case MCRDL_I32: return rs_op<int32_t>(c, in, out, m, op, seq, int(dtype), s);
    case MCRDL_I64: return rs_op<int64_t>(c, in, out, m, op, seq, int(dtype), s);
    case MCRDL_U8: return rs_op<uint8_t>(c, in, out, m, op, seq, int(dtype), s);
    case MCRDL_BF16: return rs_op<__nv_bfloat16>(c, in, out, m, op, seq, int(dtype), s);
  }
  return set_error(MCRDL_ERR_VALIDATION, "unknown dtype %d", int(dtype));
}

mcrdl_status_t mcrdl_all_reduce_fused(mcrdl_comm* c, const void* const* d_in_ptrs,
                                      void* const* d_out_ptrs, const int64_t* d_counts,
                                      const int64_t* d_offsets, int n, uint64_t total_count,
                                      mcrdl_dtype_t dtype, mcrdl_redop_t op, mcrdl_algo_t algo,
                                      uint64_t seq, void* stream) {
  (void)algo;
  if (c == nullptr) return set_error(MCRDL_ERR_NOT_INITIALIZED, "communicator is NULL");
  if (n <= 0 || total_count == 0) return mcrdl_barrier(c, seq, stream);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t t = int64_t(total_count);
  switch (dtype) {
    case MCRDL_F32: return fused_op<float>(c, d_in_ptrs, d_out_ptrs, d_counts, d_offsets, n, t, op, seq, int(dtype), s);
    case MCRDL_F64: return fused_op<double>(c, d_in_ptrs, d_out_ptrs, d_counts, d_offsets, n, t, op, seq, int(dtype), s);
    case MCRDL_I32: return fused_op<int32_t>(c, d_in_ptrs, d_out_ptrs, d_counts, d_offsets, n, t, op, seq, int(dtype), s);
    case MCRDL_I64: return fused_op<int64_t>(c, d_in_ptrs, d_out_ptrs, d_counts, d_offsets, n, t, op, seq, int(dtype), s);
    case MCRDL_U8: return fused_op<uint8_t>(c, d_in_ptrs, d_out_ptrs, d_counts, d_offsets, n, t, op, seq, int(dtype), s);
    case MCRDL_BF16:
      return fused_op<__nv_bfloat16>(c, d_in_ptrs, d_out_ptrs, d_counts, d_offsets, n, t, op, seq, int(dtype), s);
  }
  return set_error(MCRDL_ERR_VALIDATION, "unknown dtype %d", int(dtype));
}

}  // extern "C"
