// Low-latency (LL) protocol for small messages: all_reduce one-shot and the
// exchange engine (a2a(v), allgatherv, gatherv, bcast, barrier).
//
// Each 16-byte store to a peer carries 8 payload bytes interleaved with the
// op's epoch: {d0, epoch, d1, epoch}. Each 8-byte half is written and read
// single-copy-atomically, so the receiver polls the payload words themselves
// until both flag words equal the epoch — no release fence, no separate flag
// round trip. A 16-byte header per (sender -> receiver) slot carries
// {sig, bytes, epoch}: it restates the reference's header agreement
// (collectives.py:245-285) exactly like the flag protocol.
//
// Protocol choice is PER PAIR: a pair moving <= kLLMaxPairBytes uses LL lines,
// a larger one the bulk flag protocol (exchange.cu). Both endpoints know the
// pair's byte count (sender: scount, receiver: rcount), so they always agree,
// even when the two ranks run different kernels for the rest of the op.
// LL lines live in a dedicated area of the pad (common.cuh) that bulk
// kernels never write, so stale lines always carry an older epoch.
#include <algorithm>
#include <cstring>

#include "ll.cuh"

namespace mcrdl {

// ------------------------------------------------------------ all_reduce
// CTA b owns 8-byte units [ub, ue). It LL-pushes them to every peer's slot
// `rank`, then folds units in ascending rank order (own input for slot ==
// rank) straight into `out`, loading all peers' lines of a unit before
// checking any. Bit-identical to the oracle.
template <typename T, int OP>
__device__ __forceinline__ void ar_ll_body(DevComm c, const T* in, T* out, int64_t n, uint32_t epoch, uint32_t sig) {
  constexpr int E = 8 / int(sizeof(T));  // elements per 8-byte unit
  using A = typename AccT<T>::type;
  __shared__ SComm S;
  __shared__ int s_err;
  const int par = epoch & 1, rank = c.rank, world = c.world;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t B = n * int64_t(sizeof(T));
  const int64_t nu = (B + 7) / 8;
  const int64_t ub = nu * blockIdx.x / gridDim.x, ue = nu * (blockIdx.x + 1) / gridDim.x;
  const uint8_t* src = reinterpret_cast<const uint8_t*>(in);
  if (tid == 0) s_err = 0;
  stage_comm(c, S);
  __syncthreads();
  for (int k = 1; k < world; ++k) {
    const int q = (rank + k) % world;
    ll_send(ll_slot(S.pad[q], par, rank), src, B, ub, ue, blockIdx.x == 0, sig, epoch);
  }
  if (blockIdx.x == 0 && tid < world && tid != rank) {
    uint2 h;
    int e = 0;
    if (!poll_ll(ll_slot(S.pad[rank], par, tid), epoch, S.pad[rank], c.timeout_ns, h, &e)) {
      atomicCAS(&s_err, 0, e);
    } else if (h.x != sig || h.y != uint32_t(B)) {
      // abort at once: every spinning poll (here and on peers) sees the abort word
      atomicCAS(&s_err, 0, MCRDL_ERR_ORDER_MISMATCH);
      raise_error(S.pad, world, c.err, MCRDL_ERR_ORDER_MISMATCH, epoch);
    }
  }
  volatile int* verr = &s_err;
  for (int64_t u = ub + tid; u < ue && !*verr; u += nt) {
    uint4 lines[kMaxRanks];
#pragma unroll
    for (int r = 0; r < kMaxRanks; ++r)
      if (r < world && r != rank) lines[r] = ld_ll(ll_slot(S.pad[rank], par, r) + kLLHeader + u * 16);
    A acc[E];
    bool ok = true;
#pragma unroll
    for (int r = 0; r < kMaxRanks; ++r) {
      if (r >= world) break;
      uint2 v;
      if (r == rank) {
        v = load8(src, u, B);
      } else if (ll_ready(lines[r], epoch)) {
        v = make_uint2(lines[r].x, lines[r].z);
      } else {
        int e = 0;
        if (!poll_ll(ll_slot(S.pad[rank], par, r) + kLLHeader + u * 16, epoch, S.pad[rank],
                     c.timeout_ns, v, &e)) {
          atomicCAS(&s_err, 0, e);
          ok = false;
          break;
        }
      }
      const T* ev = reinterpret_cast<const T*>(&v);
#pragma unroll
      for (int k = 0; k < E; ++k) {
        const A x = Pack<T>::to_acc(ev[k]);
        acc[k] = r == 0 ? x : apply_op<OP, A>(acc[k], x);
      }
    }
    if (!ok) break;
#pragma unroll
    for (int k = 0; k < E; ++k)
      if (u * E + k < n) out[u * E + k] = Pack<T>::from_acc(acc[k]);
  }
  __syncthreads();
  if (s_err && tid == 0) raise_error(S.pad, world, c.err, s_err, epoch);
}

template <typename T, int OP>
__global__ void __launch_bounds__(kLLThreads) k_ar_ll(DevComm c, const T* in, T* out, int64_t n, uint32_t sig) {
  const uint32_t epoch = epoch_enter(c);
  ar_ll_body<T, OP>(c, in, out, n, epoch, sig);
  epoch_exit(c, epoch);
}

template <typename T, int OP>
mcrdl_status_t launch_ar_ll(mcrdl_comm* c, const T* in, T* out, int64_t n,
                            uint32_t sig, cudaStream_t stream) {
  const int64_t nu = (n * int64_t(sizeof(T)) + 7) / 8;
  if (nu * 8 > kLLMaxPayload)
    return set_error(MCRDL_ERR_INTERNAL, "LL all_reduce above the LL slot size");
  int64_t g = (nu + kLLThreads - 1) / kLLThreads;
  g = std::max<int64_t>(1, std::min<int64_t>(g, std::min(32, 4 * c->num_sms)));
  k_ar_ll<T, OP><<<int(g), kLLThreads, 0, stream>>>(c->dc, in, out, n, sig);
  count_launch();
  MCRDL_CUDA_CHECK(cudaGetLastError());
  return MCRDL_OK;
}

#define INST_AR_LL(T, OP)                                                                       \
  template mcrdl_status_t launch_ar_ll<T, OP>(mcrdl_comm*, const T*, T*, int64_t,     \
                                              uint32_t, cudaStream_t);
#define INST_AR_LL_T(T) INST_AR_LL(T, 0) INST_AR_LL(T, 1) INST_AR_LL(T, 2) INST_AR_LL(T, 3)
INST_AR_LL_T(float)
INST_AR_LL_T(double)
INST_AR_LL_T(int32_t)
INST_AR_LL_T(int64_t)
INST_AR_LL_T(uint8_t)
INST_AR_LL_T(__nv_bfloat16)

// -------------------------------------------------------------- exchange
// All of this rank's pairs are LL pairs: G CTAs, CTA b moves units
// [nu*b/G, nu*(b+1)/G) of every pair; CTA 0 also writes / checks headers.
__device__ __forceinline__ void exchange_ll_body(DevComm c, LLArgs a, uint32_t epoch) {
  __shared__ SComm S;
  __shared__ int s_err;
  const int par = epoch & 1, rank = c.rank, world = c.world;
  const int tid = threadIdx.x, b = blockIdx.x, G = gridDim.x;
  if (tid == 0) s_err = 0;
  stage_comm(c, S);
  __syncthreads();
  for (int k = 1; k < world; ++k) {
    const int j = (rank + k) % world;
    const int64_t B = a.sbytes[j], nu = (B + 7) / 8;
    ll_send(ll_slot(S.pad[j], par, rank), a.sptr[j], B, nu * b / G, nu * (b + 1) / G, b == 0,
            ll_pair_sig(a.sig_base, B), epoch, (a.sig_base & kSigCodecBit) != 0);
  }
  if (a.sptr[rank] != a.rptr[rank]) {  // local segment
    int64_t lo, hi;
    byte_share(a.sbytes[rank], b, G, lo, hi);
    block_copy<2>(a.rptr[rank] + lo, a.sptr[rank] + lo, hi - lo);
  }
  // Receive: headers checked by one thread per peer in parallel; this CTA's
  // units of every peer flattened into one index space, so each thread issues
  // its line loads for all peers before polling any (one L2 round trip
  // instead of one per peer).
  __shared__ int64_t s_u0[kMaxRanks], s_cnt[kMaxRanks];
  if (tid < world) {
    const int64_t nu = tid == rank ? 0 : (a.rbytes[tid] + 7) / 8;
    s_u0[tid] = nu * b / G;
    s_cnt[tid] = nu * (b + 1) / G - nu * b / G;
  }
  if (b == 0 && tid < world && tid != rank) {
    uint2 h;
    int e = 0;
    const uint32_t sig = ll_pair_sig(a.sig_base, a.rbytes[tid]);
    if (!poll_ll(ll_slot(S.pad[rank], par, tid), epoch, S.pad[rank], c.timeout_ns, h, &e)) {
      atomicCAS(&s_err, 0, e);
    } else if (h.x != sig || h.y != uint32_t(a.rbytes[tid])) {
      const int code = h.x != sig ? ll_header_error(h.x, sig) : MCRDL_ERR_ORDER_MISMATCH;
      atomicCAS(&s_err, 0, code);
      raise_error(S.pad, world, c.err, code, epoch);
    }
  }
  __syncthreads();
  int64_t total = 0;
  for (int r = 0; r < world; ++r) total += s_cnt[r];
  constexpr int D = 4;
  volatile int* verr = &s_err;
  for (int64_t base = tid; base < total && !*verr; base += int64_t(D) * blockDim.x) {
    uint4 v[D];
    int pi[D];
    int64_t ui[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      int64_t idx = base + int64_t(d) * blockDim.x;
      pi[d] = -1;
      if (idx >= total) continue;
      int r = 0;
      while (idx >= s_cnt[r]) idx -= s_cnt[r++];
      pi[d] = r;
      ui[d] = s_u0[r] + idx;
      v[d] = ld_ll(ll_slot(S.pad[rank], par, r) + kLLHeader + ui[d] * 16);
    }
#pragma unroll
    for (int d = 0; d < D; ++d) {
      if (pi[d] < 0) continue;
      const int r = pi[d];
      uint2 w;
      if (ll_ready(v[d], epoch)) {
        w = make_uint2(v[d].x, v[d].z);
      } else {
        int e = 0;
        if (!poll_ll(ll_slot(S.pad[rank], par, r) + kLLHeader + ui[d] * 16, epoch, S.pad[rank],
                     c.timeout_ns, w, &e)) {
          atomicCAS(&s_err, 0, e);
          break;
        }
      }
      store8(a.rptr[r], ui[d], a.rbytes[r], w);
    }
  }
  __syncthreads();
  if (s_err && tid == 0) raise_error(S.pad, world, c.err, s_err, epoch);
}

__global__ void __launch_bounds__(kLLThreads) k_exchange_ll(DevComm c, LLArgs a) {
  const uint32_t epoch = epoch_enter(c);
  exchange_ll_body(c, a, epoch);
  epoch_exit(c, epoch);
}

// Returns true when every pair of this rank is an LL pair (the LL kernel
// then takes the whole op; peers may still run k_exchange for their bulk
// pairs with other ranks).
int64_t exchange_ll_max() {
  // Per-pair LL limit (both ends of a pair decide from its byte count and this
  // value, identical on every rank). MCRDL_LL_PAIR_BYTES overrides.
  static const int64_t v = std::min<int64_t>(env_int("MCRDL_LL_PAIR_BYTES", kLLMaxPairBytes),
                                             kLLMaxPayload);
  return v;
}

bool try_exchange_ll(mcrdl_comm* c, const ExchangeSpec& sp, int64_t ll_max, cudaStream_t stream,
                     mcrdl_status_t* st) {
  int64_t mx = 0;
  for (int r = 0; r < c->world; ++r) {
    if (r == c->rank) continue;
    mx = std::max(mx, std::max(sp.sbytes[r], sp.rbytes[r]));
  }
  if (sp.d_counts != nullptr || mx > ll_max) return false;
  LLArgs a;
  memset(&a, 0, sizeof(a));
  for (int r = 0; r < c->world; ++r) {
    a.sptr[r] = sp.sptr[r];
    a.sbytes[r] = sp.sbytes[r];
    a.rptr[r] = sp.rptr[r];
    a.rbytes[r] = sp.rbytes[r];
  }
  a.sig_base = sp.sig_base;
  // CTAs: one per kLLThreads * upt units of the widest pair (MCRDL_LL_X_UPT
  // units per thread, default 1); a function of this rank's own bytes only
  // (the LL line protocol needs no grid agreement)
  // (1 measured best at p = 4: 32 / 256 KiB all_to_allv 14.3 / 14.2 us vs
  // 14.8 / 15.7 with 2, profiles/r2_ll_upt_log_p4.csv)
  static const int64_t upt = std::max<int64_t>(1, env_int("MCRDL_LL_X_UPT", 1));
  int64_t g = (mx / 8 + kLLThreads * upt - 1) / (kLLThreads * upt);
  g = std::max<int64_t>(g, (sp.sbytes[c->rank] + (256 << 10) - 1) >> 18);
  g = std::max<int64_t>(1, std::min<int64_t>(g, std::min(64, 4 * c->num_sms)));
  k_exchange_ll<<<int(g), kLLThreads, 0, stream>>>(c->dc, a);
  count_launch();
  cudaError_t e = cudaGetLastError();
  *st = e == cudaSuccess ? MCRDL_OK
                         : set_error(MCRDL_ERR_CUDA, "k_exchange_ll: %s", cudaGetErrorString(e));
  return true;
}

}  // namespace mcrdl
