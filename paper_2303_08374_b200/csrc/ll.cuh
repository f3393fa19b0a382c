// LL protocol device helpers shared by ll.cu (LL kernels) and exchange.cu
// (LL pairs inside the bulk exchange kernel). See ll.cu for the protocol.
#pragma once

#include "internal.h"

namespace mcrdl {

constexpr int64_t kLLHeader = 16;
constexpr int kLLThreads = 256;

struct LLArgs {
  const uint8_t* sptr[kMaxRanks];
  int64_t sbytes[kMaxRanks];
  uint8_t* rptr[kMaxRanks];
  int64_t rbytes[kMaxRanks];
  uint32_t sig_base;
};

__device__ __forceinline__ void st_ll(void* p, uint32_t d0, uint32_t d1, uint32_t f) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(d0), "r"(f),
               "r"(d1), "r"(f)
               : "memory");
}
__device__ __forceinline__ uint4 ld_ll(const void* p) {
  uint4 v;
  asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ bool ll_ready(const uint4& v, uint32_t epoch) {
  return v.y == epoch && v.w == epoch;
}

// Spin on one LL line until both flags carry `epoch`; false on timeout /
// peer abort (code in *err).
static __device__ __noinline__ bool poll_ll(const void* p, uint32_t epoch, const Pad* me,
                                            uint64_t timeout_ns, uint2& out, int* err) {
  uint64_t start = 0;
  int spins = 0;
  for (;;) {
    const uint4 v = ld_ll(p);
    if (ll_ready(v, epoch)) {
      out = make_uint2(v.x, v.z);
      return true;
    }
    if (++spins >= 64) {
      spins = 0;
      if (ld_acquire_sys(&me->abort_word[epoch & 1][0]) == epoch) {
        *err = int(ld_relaxed_sys(&me->abort_word[epoch & 1][1]));
        if (*err == 0) *err = MCRDL_ERR_INTERNAL;
        return false;
      }
      if (const uint64_t pz = ld_relaxed_sys(&me->poison)) {  // an earlier op failed
        *err = int(pz);
        return false;
      }
      const uint64_t now = globaltimer_ns();
      if (start == 0) start = now;
      else if (now - start > timeout_ns) {
        printf("[mcrdl] LL timeout: pad %p line %p want epoch %u, saw {%08x %08x %08x %08x} "
               "(block %d thread %d)\n",
               (const void*)me, p, epoch, v.x, v.y, v.z, v.w, int(blockIdx.x), int(threadIdx.x));
        *err = MCRDL_ERR_TIMEOUT;
        return false;
      }
    }
  }
}

__device__ __forceinline__ uint8_t* ll_slot(Pad* pad, int par, int sender) {
  return reinterpret_cast<uint8_t*>(pad) + kLLOffset + par * kLLParityBytes +
         int64_t(sender) * kLLSlotBytes;
}

__device__ __forceinline__ uint2 load8(const uint8_t* src, int64_t u, int64_t B) {
  uint2 v = make_uint2(0, 0);
  if ((uintptr_t(src) & 7) == 0 && (u + 1) * 8 <= B) {
    v = *reinterpret_cast<const uint2*>(src + u * 8);
  } else {
    uint8_t* b = reinterpret_cast<uint8_t*>(&v);
    for (int q = 0; q < 8; ++q)
      if (u * 8 + q < B) b[q] = src[u * 8 + q];
  }
  return v;
}
__device__ __forceinline__ void store8(uint8_t* dst, int64_t u, int64_t B, uint2 v) {
  if ((uintptr_t(dst) & 7) == 0 && (u + 1) * 8 <= B) {
    *reinterpret_cast<uint2*>(dst + u * 8) = v;
  } else {
    const uint8_t* b = reinterpret_cast<const uint8_t*>(&v);
    for (int q = 0; q < 8; ++q)
      if (u * 8 + q < B) dst[u * 8 + q] = b[q];
  }
}

// Header signature of an LL pair: the op hash mixed with the pair's byte
// count, with bit 19 carrying the payload codec (as the bulk pair_sig), so a
// codec disagreement is told apart from an order mismatch.
__device__ __forceinline__ uint32_t ll_pair_sig(uint32_t sig_base, int64_t B) {
  return (mix32(sig_base & ~kSigCodecBit, uint64_t(B)) & ~kSigCodecBit) | (sig_base & kSigCodecBit);
}
__device__ __forceinline__ int ll_header_error(uint32_t got, uint32_t want) {
  return ((got ^ want) == kSigCodecBit) ? MCRDL_ERR_CODEC_MISMATCH : MCRDL_ERR_ORDER_MISMATCH;
}

// LL-send units [u0, u1) of a B-byte pair; `hdr` also writes the header.
// trunc: trunc16 codec on an f32 payload (middleware.py:43-75) — each f32
// keeps its top 16 bits (the LL line carries raw words, so the wire size is
// unchanged; the values match the compressed bulk path).
__device__ __forceinline__ void ll_send(uint8_t* slot, const uint8_t* src, int64_t B, int64_t u0,
                                        int64_t u1, bool hdr, uint32_t sig, uint32_t epoch,
                                        bool trunc = false) {
  const uint32_t mask = trunc ? 0xFFFF0000u : 0xFFFFFFFFu;
  for (int64_t u = u0 + threadIdx.x; u < u1; u += blockDim.x) {
    const uint2 v = load8(src, u, B);
    st_ll(slot + kLLHeader + u * 16, v.x & mask, v.y & mask, epoch);
  }
  if (hdr && threadIdx.x == 0) st_ll(slot, sig, uint32_t(B), epoch);
}

// LL-receive units [u0, u1) (4 lines in flight per thread); `hdr` also
// checks the header. Returns an error code (0 ok).
__device__ __forceinline__ int ll_recv(const uint8_t* slot, uint8_t* dst, int64_t B, int64_t u0,
                                       int64_t u1, bool hdr, uint32_t sig, uint32_t epoch,
                                       const Pad* me, uint64_t tmo) {
  int err = 0;
  if (hdr && threadIdx.x == 0) {
    uint2 h;
    if (!poll_ll(slot, epoch, me, tmo, h, &err)) return err;
    if (h.x != sig) return ll_header_error(h.x, sig);
    if (h.y != uint32_t(B)) return MCRDL_ERR_ORDER_MISMATCH;
  }
  const int nt = blockDim.x;
  for (int64_t u = u0 + threadIdx.x; u < u1; u += 4 * nt) {
    uint4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (u + k * nt < u1) v[k] = ld_ll(slot + kLLHeader + (u + k * nt) * 16);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t uk = u + k * nt;
      if (uk >= u1) break;
      uint2 d;
      if (ll_ready(v[k], epoch)) {
        d = make_uint2(v[k].x, v[k].z);
      } else if (!poll_ll(slot + kLLHeader + uk * 16, epoch, me, tmo, d, &err)) {
        return err;
      }
      store8(dst, uk, B, d);
    }
  }
  return 0;
}

// Device helpers for the mixed case (k_exchange handles bulk pairs and
// calls these for its LL pairs from sender / receiver CTA 0).
// LL pairs (<= ll_max bytes) inside the bulk exchange kernel: CTA b of the
// role's G CTAs moves units [nu*b/G, nu*(b+1)/G) of every LL pair; CTA 0
// writes / checks the header.
__device__ __forceinline__ void exchange_ll_send_pairs(Pad* const* pads, int rank, int world, int par,
                                       const uint8_t* const* sptr, const int64_t* sbytes,
                                       uint32_t sig_base, uint32_t epoch, int64_t ll_max, int b,
                                       int G) {
  for (int k = 1; k < world; ++k) {
    const int j = (rank + k) % world;
    const int64_t B = sbytes[j];
    if (B > ll_max) continue;
    const int64_t nu = (B + 7) / 8;
    ll_send(ll_slot(pads[j], par, rank), sptr[j], B, nu * b / G, nu * (b + 1) / G, b == 0,
            ll_pair_sig(sig_base, B), epoch, (sig_base & kSigCodecBit) != 0);
  }
}
__device__ __forceinline__ int exchange_ll_recv_pairs(Pad* const* pads, int rank, int world, int par,
                                      uint8_t* const* rptr, const int64_t* rbytes, uint32_t sig_base,
                                      uint32_t epoch, uint64_t tmo, int64_t ll_max, int b, int G) {
  for (int k = 1; k < world; ++k) {
    const int i = (rank - k + world) % world;
    const int64_t B = rbytes[i];
    if (B > ll_max) continue;
    const int64_t nu = (B + 7) / 8;
    const int e = ll_recv(ll_slot(pads[rank], par, i), rptr[i], B, nu * b / G, nu * (b + 1) / G,
                          b == 0, ll_pair_sig(sig_base, B), epoch, pads[rank], tmo);
    if (e) return e;
  }
  return 0;
}

}  // namespace mcrdl
