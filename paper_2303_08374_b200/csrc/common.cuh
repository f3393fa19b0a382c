// Device-side building blocks shared by every collective kernel.
//
// Memory model of the backend:
//  * Every rank owns one cuMem VMM region = [signal pad | workspace]. Every
//    peer's region is mapped into every rank's address space, so a kernel
//    reaches a peer with plain ld/st over NVLink (NVSwitch routes them).
//  * The workspace is split into two halves; op with epoch e uses half e&1.
//    Every op ends only after receiving a flag from every peer, so when a rank
//    starts op e+2 in half (e&1), every peer has finished op e (stream order).
//  * Flags are 64-bit words in the RECEIVER's pad, one per (parity, block,
//    sender), value = epoch<<32 | sig20<<12 | step12. `sig` folds the op
//    signature (kind, dtype, op, root, count, reference seq) — the device
//    restatement of the reference's header agreement (collectives.py:178-285):
//    a rank that posted a different op at the same slot sees a sig mismatch
//    and raises ORDER_MISMATCH instead of corrupting data.
//  * Release/acquire at .sys scope; every spin is bounded by the comm timeout
//    (reference: MCRDL_TIMEOUT_SECS, runtime.py:65) and by a peer abort word.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/mcrdl_nvl.h"
#include "geometry.h"

namespace mcrdl {

constexpr int kMaxRanks = MCRDL_MAX_RANKS;
constexpr int kMaxBlocks = 512;  // flag slots per parity
// Device-timed op log (CommLog durations): a ring of {start, end} stamps in
// the pad, mirrored to a host-mapped copy every kOpLogFlush ops by the op's
// own last CTA and fully by mcrdl_comm_log_flush.
constexpr int kOpLogSlots = 4096;
constexpr int kOpLogFlush = 64;
constexpr int kThreads = 512;
// Point-to-point mailboxes (p2p.cu): every rank owns one ring of kP2PSlots x
// kP2PChunk bytes per sender; kP2PHdr message headers per sender.
constexpr int kP2PSlots = 512;
constexpr int64_t kP2PChunk = 64 << 10;  // one CTA pass (512 thr x 16 B x 8)
constexpr int kP2PHdr = 256;
// Small messages (<= kP2PLLMax bytes) take the LL path: a ring of kP2PLLSlots
// slots per sender, each a header line + 16-byte {data, tag} lines.
constexpr int kP2PLLSlots = 64;
constexpr int64_t kP2PLLMax = 256 << 10;
constexpr int64_t kP2PLLCtaBytes = 8 << 10;  // payload per CTA of an LL message
constexpr int64_t kP2PLLSlotBytes = 2 * kP2PLLMax + 256;
constexpr int64_t kP2PLLSenderBytes = int64_t(kP2PLLSlots) * kP2PLLSlotBytes;

struct Pad {
  uint64_t flag[2][kMaxBlocks][kMaxRanks];   // data-ready, phase 1
  uint64_t flag2[2][kMaxBlocks][kMaxRanks];  // data-ready, phase 2
  uint64_t ack[2][kMaxBlocks][kMaxRanks];    // slot consumed (multi-round)
  uint64_t abort_word[2][2];                 // [par] = {epoch, code}
  uint64_t poison;                           // any rank's error code, never cleared
  // Local-only words (never written by peers): the device-resident op epoch
  // (epoch of the last completed launch) and the exit counter of the running
  // launch. Keeping the epoch on the device makes every launch replayable
  // from a CUDA graph: no host-baked argument changes between ops.
  uint32_t dev_epoch;
  uint32_t done_ctas;
  // Point-to-point channel (p2p.cu). Written by the peer named in [.]:
  uint64_t p2p_full[kMaxRanks][kP2PSlots];   // [src][slot] = chunk index + 1 now in the slot
  uint64_t p2p_free[kMaxRanks][kP2PSlots];   // [dst][slot] = chunk index + 1 dst consumed
  uint64_t p2p_hdr[kMaxRanks][kP2PHdr][2];   // [src][msg % H] = {msg + 1, bytes}
  uint64_t p2p_hdr_ack[kMaxRanks];           // [dst] = messages dst has matched
  // Local-only per-peer stream counters (device-resident: graph-safe).
  uint64_t p2p_tx_chunks[kMaxRanks], p2p_tx_msgs[kMaxRanks];
  uint64_t p2p_rx_chunks[kMaxRanks], p2p_rx_msgs[kMaxRanks];
  uint32_t p2p_done[2];  // exit counters of the running send / recv launch
  uint64_t oplog[kOpLogSlots][2];  // local: {start, end} stamps by log id % slots
};
// Region layout: [flag pad | LL area | workspace]. The LL area is written
// only by LL kernels (ll.cu), so a stale LL line always carries an older
// epoch and can never be mistaken for a current one (raw bulk payloads could
// contain any bit pattern, including a small epoch value).
constexpr size_t kLLOffset = size_t(1) << 20;
constexpr int64_t kLLMaxPayload = 256 << 10;               // per (sender -> receiver) slot
constexpr int64_t kLLSlotBytes = 129 * 4096;               // >= 16 + 2 * kLLMaxPayload
constexpr int64_t kLLParityBytes = int64_t(kMaxRanks) * kLLSlotBytes;
constexpr size_t kPadBytes = size_t(16) << 20;             // workspace starts 16 MiB in
static_assert(sizeof(Pad) <= kLLOffset, "pad too large");
static_assert(16 + 2 * kLLMaxPayload <= kLLSlotBytes, "LL slot too small");
static_assert(kLLOffset + 2 * kLLParityBytes <= kPadBytes, "LL area too large");

struct DevComm {
  uint8_t* ws[kMaxRanks];  // rank r's workspace, mapped in this address space
  Pad* pad[kMaxRanks];     // rank r's signal pad
  Pad* self;               // == pad[rank] (no runtime-indexed param access)
  int* err;                // host-mapped latched error word
  uint64_t* trace;         // host-mapped timeline (trace builds only), else null
  uint64_t timeout_ns;
  int64_t half_bytes;      // bytes per workspace half
  int64_t mbox_bytes;      // p2p mailbox per sender (at ws + 2 * half_bytes)
  uint64_t* oplog;         // host-mapped op log ring (kOpLogSlots x {start, end} words)
  uint64_t log_id;         // this launch's log id (0: not logged, e.g. graph capture)
  int rank;
  int world;
};

// Developer timeline (build.py --trace defines MCRDL_TRACE): thread 0 of a CTA
// stamps %globaltimer into slot [cta][idx] of a host-mapped buffer.
constexpr int kTraceSlots = 256;
#ifdef MCRDL_TRACE
#define MCRDL_TRACE_AT(c, cta, idx)                                                       \
  do {                                                                                    \
    if ((c).trace && threadIdx.x == 0 && (idx) < kTraceSlots)                             \
      (c).trace[int64_t(cta) * kTraceSlots + (idx)] = globaltimer_ns();                   \
  } while (0)
#else
#define MCRDL_TRACE_AT(c, cta, idx) \
  do {                              \
  } while (0)
#endif

// ------------------------------------------------------------ primitives
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_relaxed_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// 16-byte loads/stores. Workspace reads use .cg (L2, the coherence point for
// peer writes); user-buffer reads use the default path.
__device__ __forceinline__ uint4 ld16(const void* p) { return *reinterpret_cast<const uint4*>(p); }
__device__ __forceinline__ uint4 ld16_cg(const void* p) {
  return __ldcg(reinterpret_cast<const uint4*>(p));
}
__device__ __forceinline__ void st16(void* p, const uint4& v) { *reinterpret_cast<uint4*>(p) = v; }

// Bit 19 of the 20-bit flag signature carries the payload codec (trunc16),
// every other bit the op hash: a flag that differs ONLY in that bit is a
// codec disagreement (the reference's CodecMismatch), not an order mismatch.
constexpr uint32_t kSigCodecBit = 1u << 19;

__device__ __forceinline__ uint64_t make_flag(uint32_t epoch, uint32_t sig, uint32_t step) {
  return (uint64_t(epoch) << 32) | (uint64_t(sig & 0xFFFFFu) << 12) | uint64_t(step & 0xFFFu);
}

__host__ __device__ __forceinline__ uint32_t mix32(uint32_t h, uint64_t v) {
  // FNV-1a style mix of a 64-bit value into a 32-bit hash.
  for (int i = 0; i < 8; ++i) {
    h ^= uint32_t((v >> (8 * i)) & 0xFF);
    h *= 16777619u;
  }
  return h;
}

// Per-CTA shared copy of the peer pointer tables. Indexing the kernel-param
// arrays with a runtime rank would spill DevComm to local memory; the staged
// copy is loaded with constant indices once per CTA.
struct SComm {
  uint8_t* ws[kMaxRanks];
  Pad* pad[kMaxRanks];
};
__device__ __forceinline__ void stage_comm(const DevComm& c, SComm& s) {
  if (threadIdx.x == 0) {
#pragma unroll
    for (int r = 0; r < kMaxRanks; ++r) {
      s.ws[r] = c.ws[r];
      s.pad[r] = c.pad[r];
    }
  }
}

// Device-resident epoch. Every CTA of a launch reads the local pad's
// dev_epoch at entry (the launch's epoch = last + 1, skipping 0); the last CTA
// to leave stores it back. The store happens only after all gridDim.x CTAs
// have arrived at the exit counter, i.e. after every CTA has read the old
// value. Launches of one comm never overlap (stream-ordered; begin_op chains
// streams), so launch k+1 always sees launch k's store.
// Device-timed op log (CommLog durations, reference middleware.py:100-124):
// block 0 stamps %globaltimer at entry, the last CTA to exit at exit, into a
// ring in the LOCAL pad (each stamp is ONE 64-bit store: id tag in the top 16
// bits, 48-bit ns time below). Every kOpLogFlush-th op's last CTA mirrors the
// last kOpLogFlush entries into the host-mapped ring (the host reads it
// lazily; mcrdl_comm_log_flush mirrors the rest on demand). Stamping straight
// into host-mapped memory cost every op its end-of-kernel system-memory flush
// (0.4-1.8 us measured at p = 2-4, profiles/r2_latency_log_*).
__device__ __forceinline__ uint64_t oplog_word(uint64_t id) {
  return (id << 48) | (globaltimer_ns() & 0xFFFFFFFFFFFFull);
}
__device__ __forceinline__ void oplog_start(const DevComm& c) {
  if (c.log_id != 0 && blockIdx.x == 0 && threadIdx.x == 0)
    *reinterpret_cast<volatile uint64_t*>(&c.self->oplog[c.log_id % kOpLogSlots][0]) =
        oplog_word(c.log_id);
}
__device__ __forceinline__ void oplog_end(const DevComm& c) {  // last CTA, one thread
  if (c.log_id == 0) return;
  *reinterpret_cast<volatile uint64_t*>(&c.self->oplog[c.log_id % kOpLogSlots][1]) =
      oplog_word(c.log_id);
  if (c.log_id % kOpLogFlush == 0 && c.oplog != nullptr) {
    for (uint64_t k = c.log_id + 1 - kOpLogFlush; k <= c.log_id; ++k) {
      const uint64_t s = k % kOpLogSlots;
      volatile const uint64_t* src = c.self->oplog[s];
      c.oplog[s * 2] = src[0];
      c.oplog[s * 2 + 1] = src[1];
    }
  }
}

__device__ __forceinline__ uint32_t epoch_enter(const DevComm& c) {
  __shared__ uint32_t s_epoch;
  oplog_start(c);
  if (threadIdx.x == 0) {
    const uint32_t e = *reinterpret_cast<const volatile uint32_t*>(&c.self->dev_epoch) + 1u;
    s_epoch = e == 0u ? 1u : e;
  }
  __syncthreads();
  return s_epoch;
}
__device__ __forceinline__ void epoch_exit(const DevComm& c, uint32_t epoch) {
  __syncthreads();
  if (gridDim.x == 1) {  // one CTA (small messages): no exit counter, no fences —
    // the kernel boundary orders the store before the comm's next launch
    if (threadIdx.x == 0) {
      *reinterpret_cast<volatile uint32_t*>(&c.self->dev_epoch) = epoch;
      oplog_end(c);
    }
    return;
  }
  if (threadIdx.x == 0) {
    __threadfence();
    const uint32_t prev = atomicAdd(&c.self->done_ctas, 1u);
    if (prev == gridDim.x - 1) {
      *reinterpret_cast<volatile uint32_t*>(&c.self->done_ctas) = 0u;
      *reinterpret_cast<volatile uint32_t*>(&c.self->dev_epoch) = epoch;
      __threadfence();
      oplog_end(c);
    }
  }
}

// Record an error: latch it in the host-visible word and tell every peer to
// stop spinning on this op (abort word carries the epoch + code).
static __device__ __noinline__ void raise_error(Pad* const* pads, int world, int* err, int code,
                                                uint32_t epoch) {
  const int par = epoch & 1;
  if (atomicCAS(err, 0, code) == 0)
    printf("[mcrdl] raise_error: code %d epoch %u (pad %p, block %d)\n", code, epoch,
           (const void*)pads[0], int(blockIdx.x));
  for (int r = 0; r < world; ++r) {
    st_relaxed_sys(&pads[r]->abort_word[par][1], uint64_t(code));
    __threadfence_system();
    st_release_sys(&pads[r]->abort_word[par][0], uint64_t(epoch));
    // Poison every rank: ops already enqueued behind this one (other epochs)
    // then drain at once instead of each waiting out its timeout.
    st_release_sys(&pads[r]->poison, uint64_t(code));
  }
}

// Spin until the flag at `p` carries (epoch, sig, >= step). Returns MCRDL_OK
// or an error code; never spins past the timeout or a peer abort (`me` is
// the local pad).
// A communicator whose host-mapped error word is set is poisoned: ops that
// were already enqueued behind the failing one must drain at once instead
// of each waiting out its own timeout (their epochs never see the abort).
__device__ __forceinline__ int poisoned(const int* err) {
  return *reinterpret_cast<const volatile int*>(err);
}

static __device__ __noinline__ int wait_flag(const uint64_t* p, const Pad* me, uint64_t timeout_ns,
                                             const int* err, uint32_t epoch, uint32_t sig,
                                             uint32_t step) {
  const int par = epoch & 1;
  uint64_t start = 0;
  int spins = 0;
  for (;;) {
    const uint64_t v = ld_acquire_sys(p);
    if (uint32_t(v >> 32) == epoch) {
      const uint32_t lo = uint32_t(v);
      if ((lo >> 12) != (sig & 0xFFFFFu))
        return (((lo >> 12) ^ sig) & 0xFFFFFu) == kSigCodecBit ? MCRDL_ERR_CODEC_MISMATCH
                                                                : MCRDL_ERR_ORDER_MISMATCH;
      if ((lo & 0xFFFu) >= (step & 0xFFFu)) return MCRDL_OK;
    }
    if (++spins >= 32) {
      spins = 0;
      if (ld_acquire_sys(&me->abort_word[par][0]) == epoch) {
        int code = int(ld_relaxed_sys(&me->abort_word[par][1]));
        return code ? code : MCRDL_ERR_INTERNAL;
      }
      // (the host-mapped `err` word is NOT polled here: a PCIe read in every
      // spinning thread measurably slowed the bandwidth kernels; raise_error
      // mirrors the code into every rank's device-side pad->poison instead)
      (void)err;
      if (const uint64_t pz = ld_relaxed_sys(&me->poison)) return int(pz);
      const uint64_t now = globaltimer_ns();
      if (start == 0) {
        start = now;
      } else if (now - start > timeout_ns) {
        // one diagnostic line per timed-out waiter (exceptional path only)
        printf("[mcrdl] flag timeout: pad %p word %p want epoch %u sig %05x step>=%u, saw %016llx "
               "(block %d thread %d)\n",
               (const void*)me, (const void*)p, epoch, sig & 0xFFFFFu, step & 0xFFFu,
               (unsigned long long)v, int(blockIdx.x), int(threadIdx.x));
        return MCRDL_ERR_TIMEOUT;
      }
    }
  }
}

// Spin until the monotone counter at `p` reaches `target` (p2p channel);
// bounded by the timeout and by the poison word like wait_flag.
static __device__ __noinline__ int wait_geq(const uint64_t* p, const Pad* me, uint64_t timeout_ns,
                                            uint64_t target) {
  uint64_t start = 0;
  int spins = 0;
  for (;;) {
    if (ld_acquire_sys(p) >= target) return MCRDL_OK;
    if (++spins >= 32) {
      spins = 0;
      if (const uint64_t pz = ld_relaxed_sys(&me->poison)) return int(pz);
      const uint64_t now = globaltimer_ns();
      if (start == 0) {
        start = now;
      } else if (now - start > timeout_ns) {
        printf("[mcrdl] counter timeout: pad %p word %p want >= %llu, saw %llu (block %d thread %d)\n",
               (const void*)me, (const void*)p, (unsigned long long)target,
               (unsigned long long)ld_relaxed_sys(p), int(blockIdx.x), int(threadIdx.x));
        return MCRDL_ERR_TIMEOUT;
      }
    }
  }
}

// Publish flag value `val` into a peer's slot. Caller must __syncthreads()
// (or __syncwarp for warp-private data) first: the barrier orders every
// thread's payload stores before this thread's release, and a .sys release
// is cumulative over them. No separate fence.sc: measured on B200 NVLink
// (tools/fence_probe.cu) a __threadfence_system per 64 KiB chunk cost ~40%
// of push bandwidth, the release alone ~1%.
__device__ __forceinline__ void publish(uint64_t* peer_slot, uint64_t val) {
  st_release_sys(peer_slot, val);
}

// ------------------------------------------------------------ reduce ops
template <typename T>
struct AccT {
  using type = T;
};
template <>
struct AccT<__nv_bfloat16> {
  using type = float;
};

template <typename A>
__device__ __forceinline__ A op_sum(A a, A b) { return a + b; }
template <>
__device__ __forceinline__ int32_t op_sum(int32_t a, int32_t b) {
  return int32_t(uint32_t(a) + uint32_t(b));
}
template <>
__device__ __forceinline__ int64_t op_sum(int64_t a, int64_t b) {
  return int64_t(uint64_t(a) + uint64_t(b));
}
template <>
__device__ __forceinline__ uint8_t op_sum(uint8_t a, uint8_t b) { return uint8_t(a + b); }

template <typename A>
__device__ __forceinline__ A op_prod(A a, A b) { return a * b; }
template <>
__device__ __forceinline__ int32_t op_prod(int32_t a, int32_t b) {
  return int32_t(uint32_t(a) * uint32_t(b));
}
template <>
__device__ __forceinline__ int64_t op_prod(int64_t a, int64_t b) {
  return int64_t(uint64_t(a) * uint64_t(b));
}
template <>
__device__ __forceinline__ uint8_t op_prod(uint8_t a, uint8_t b) { return uint8_t(a * b); }

// numpy minimum/maximum semantics: NaN propagates, ties return the second
// operand (np.minimum(0.0, -0.0) == -0.0).
template <typename A>
__device__ __forceinline__ A op_min(A a, A b) { return (a != a || a < b) ? a : b; }
template <typename A>
__device__ __forceinline__ A op_max(A a, A b) { return (a != a || a > b) ? a : b; }

template <int OP, typename A>
__device__ __forceinline__ A apply_op(A a, A b) {
  if constexpr (OP == MCRDL_SUM) return op_sum<A>(a, b);
  else if constexpr (OP == MCRDL_PROD) return op_prod<A>(a, b);
  else if constexpr (OP == MCRDL_MIN) return op_min<A>(a, b);
  else return op_max<A>(a, b);
}

// A 16-byte pack of T, unpacked into accumulator registers.
template <typename T>
struct Pack {
  static constexpr int N = 16 / int(sizeof(T));
  using A = typename AccT<T>::type;
  A v[N];

  __device__ __forceinline__ void from_raw(const uint4& raw) {
    const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = to_acc(e[i]);
  }
  __device__ __forceinline__ uint4 to_raw() const {
    uint4 raw;
    T* e = reinterpret_cast<T*>(&raw);
#pragma unroll
    for (int i = 0; i < N; ++i) e[i] = from_acc(v[i]);
    return raw;
  }
  template <int OP>
  __device__ __forceinline__ void fold(const uint4& raw) {
    const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = apply_op<OP, A>(v[i], to_acc(e[i]));
  }
  static __device__ __forceinline__ A to_acc(T x) {
    if constexpr (sizeof(T) == 2) return __bfloat162float(x);
    else return x;
  }
  static __device__ __forceinline__ T from_acc(A x) {
    if constexpr (sizeof(T) == 2) return __float2bfloat16_rn(x);  // one RNE rounding
    else return x;
  }
};

// Load pack i of an n-element array; partial/misaligned packs go element-wise
// (unused lanes zero). VEC: the base pointer is 16-byte aligned.
template <typename T, bool VEC>
__device__ __forceinline__ uint4 load_pack(const T* base, int64_t i, int64_t n) {
  constexpr int N = 16 / int(sizeof(T));
  if (VEC && (i + 1) * N <= n) return ld16(base + i * N);
  uint4 raw = make_uint4(0, 0, 0, 0);
  T* e = reinterpret_cast<T*>(&raw);
  const int64_t lim = n - i * N;
#pragma unroll
  for (int k = 0; k < N; ++k)
    if (k < lim) e[k] = base[i * N + k];
  return raw;
}
template <typename T, bool VEC>
__device__ __forceinline__ void store_pack(T* base, int64_t i, int64_t n, const uint4& raw) {
  constexpr int N = 16 / int(sizeof(T));
  if (VEC && (i + 1) * N <= n) {
    st16(base + i * N, raw);
    return;
  }
  const T* e = reinterpret_cast<const T*>(&raw);
  const int64_t lim = n - i * N;
#pragma unroll
  for (int k = 0; k < N; ++k)
    if (k < lim) base[i * N + k] = e[k];
}

// Block-cooperative byte copy, widest access the alignment of dst, src and n
// allows. Loads are batched (UNROLL in flight per thread) before the stores.
template <int UNROLL = 4>
__device__ __forceinline__ void block_copy(uint8_t* dst, const uint8_t* src, int64_t n) {
  if (n <= 0 || dst == src) return;
  const uintptr_t a = uintptr_t(dst) | uintptr_t(src);
  const int tid = threadIdx.x, nt = blockDim.x;
  int64_t done = 0;
  if ((a & 15) == 0) {
    const int64_t np = n >> 4;
    const uint4* s = reinterpret_cast<const uint4*>(src);
    uint4* d = reinterpret_cast<uint4*>(dst);
    int64_t i = tid;
    for (; i + (UNROLL - 1) * nt < np; i += UNROLL * nt) {
      uint4 v[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) v[u] = __ldcg(s + i + u * nt);
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) d[i + u * nt] = v[u];
    }
    for (; i < np; i += nt) d[i] = __ldcg(s + i);
    done = np << 4;
  } else if ((a & 7) == 0) {
    const int64_t np = n >> 3;
    const uint2* s = reinterpret_cast<const uint2*>(src);
    uint2* d = reinterpret_cast<uint2*>(dst);
    for (int64_t i = tid; i < np; i += nt) d[i] = __ldcg(s + i);
    done = np << 3;
  } else if ((a & 3) == 0) {
    const int64_t np = n >> 2;
    const uint32_t* s = reinterpret_cast<const uint32_t*>(src);
    uint32_t* d = reinterpret_cast<uint32_t*>(dst);
    for (int64_t i = tid; i < np; i += nt) d[i] = __ldcg(s + i);
    done = np << 2;
  }
  for (int64_t i = done + tid; i < n; i += nt) dst[i] = src[i];
}


}  // namespace mcrdl
