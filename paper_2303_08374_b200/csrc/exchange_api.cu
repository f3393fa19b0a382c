// Public C-ABI entry points of the exchange engine (exchange.cu): each maps a
// reference collective onto per-peer (pointer, bytes) spans.
#include <string.h>

#include <algorithm>

#include "internal.h"

namespace mcrdl {

static bool check_counts(const int64_t* counts, const int64_t* displs, int world, const char* what) {
  for (int r = 0; r < world; ++r) {
    if (counts[r] < 0 || displs[r] < 0) {
      set_error(MCRDL_ERR_VALIDATION, "%s: counts and displacements must be >= 0", what);
      return false;
    }
  }
  return true;
}

// Strip the payload-codec flag from `algo` (MCRDL_CODEC_TRUNC16); the codec
// applies to f32 payloads only (CompressionConfig.active_for,
// middleware.py:86-95: other dtypes bypass silently).
static int split_codec(mcrdl_algo_t* algo, mcrdl_dtype_t dtype) {
  const int f = int(*algo);
  *algo = mcrdl_algo_t(f & 0xFF);
  return ((f & MCRDL_CODEC_TRUNC16) != 0 && dtype == MCRDL_F32) ? 1 : 0;
}

// Pair sizes where storing straight into symmetric outputs beats the staged
// exchange (measured, profiles/symmx_perf_r1.log: +5-13 % for 4-128 MiB
// pairs; below, LL / staged latency wins; above, -2-3 %). Agreed by all ranks.
static bool symm_x_window(int64_t pair_bytes) {
  return pair_bytes > (int64_t(4) << 20) && pair_bytes <= (int64_t(128) << 20);
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
  const int codec = split_codec(&algo, dtype);
  if (c == nullptr) return set_error(MCRDL_ERR_NOT_INITIALIZED, "communicator is NULL");
  const int es = elem_size(dtype);
  if (es == 0) return set_error(MCRDL_ERR_VALIDATION, "unknown dtype %d", int(dtype));
  if (!check_counts(scounts, sdispls, c->world, "scounts") ||
      !check_counts(rcounts, rdispls, c->world, "rcounts"))
    return MCRDL_ERR_VALIDATION;
  // Sender and receiver CTAs run concurrently, so an aliased input could be
  // overwritten before it is sent: the caller snapshots it (the reference
  // does the same, collectives.py:662-663).
  if (in == out && in != nullptr && c->world > 1)
    return set_error(MCRDL_ERR_VALIDATION, "in-place all_to_allv: pass a snapshot of the input");
  ExchangeSpec s = empty_spec(es, op_sig(kKindA2AV, dtype, 0, -1, 0, seq));
  s.codec = codec;
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
  const int codec = split_codec(&algo, dtype);
  if (c == nullptr) return set_error(MCRDL_ERR_NOT_INITIALIZED, "communicator is NULL");
  const int es = elem_size(dtype);
  if (es == 0) return set_error(MCRDL_ERR_VALIDATION, "unknown dtype %d", int(dtype));
  if (d_counts == nullptr) return set_error(MCRDL_ERR_VALIDATION, "NULL device count array");
  ExchangeSpec s = empty_spec(es, op_sig(kKindA2AV, dtype, 0, -1, 0, seq));
  s.codec = codec;
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
  const int codec = split_codec(&algo, dtype);
  if (c == nullptr) return set_error(MCRDL_ERR_NOT_INITIALIZED, "communicator is NULL");
  const int es = elem_size(dtype);
  if (es == 0) return set_error(MCRDL_ERR_VALIDATION, "unknown dtype %d", int(dtype));
  if (count % uint64_t(c->world) != 0)
    return set_error(MCRDL_ERR_VALIDATION, "count %llu not divisible by %d",
                     (unsigned long long)count, c->world);
  if (in == out && c->world > 1 && count > 0)
    return set_error(MCRDL_ERR_VALIDATION, "in-place all_to_all_single: pass a snapshot of the input");
  const int64_t m = int64_t(count) / c->world;
  if (!codec && symm_x_window(m * es)) {  // symmetric output: zero-copy direct write
    int64_t so[kMaxRanks], ro[kMaxRanks], b[kMaxRanks];
    for (int q = 0; q < c->world; ++q) {
      so[q] = int64_t(q) * m * es;
      ro[q] = int64_t(c->rank) * m * es;
      b[q] = m * es;
    }
    mcrdl_status_t st;
    if (try_exchange_symm(c, in, out, uint64_t(count) * es, so, ro, b, m * es,
                          op_sig(kKindA2ASingle, dtype, 1, -1, uint64_t(m), seq),
                          reinterpret_cast<cudaStream_t>(stream), &st))
      return st;
  }
  ExchangeSpec s = empty_spec(es, op_sig(kKindA2ASingle, dtype, 0, -1, uint64_t(m), seq));
  s.codec = codec;
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
  const int codec = split_codec(&algo, dtype);
  if (c == nullptr) return set_error(MCRDL_ERR_NOT_INITIALIZED, "communicator is NULL");
  const int es = elem_size(dtype);
  if (es == 0) return set_error(MCRDL_ERR_VALIDATION, "unknown dtype %d", int(dtype));
  ExchangeSpec s = empty_spec(es, op_sig(kKindA2AList, dtype, 0, -1, 0, seq));
  s.codec = codec;
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
  const int codec = split_codec(&algo, dtype);
  if (c == nullptr) return set_error(MCRDL_ERR_NOT_INITIALIZED, "communicator is NULL");
  const int es = elem_size(dtype);
  if (es == 0) return set_error(MCRDL_ERR_VALIDATION, "unknown dtype %d", int(dtype));
  if (!check_counts(rcounts, displs, c->world, "rcounts")) return MCRDL_ERR_VALIDATION;
  {  // symmetric output: every rank stores its block straight into every output
    int64_t mx = 0, end = 0;
    for (int r = 0; r < c->world; ++r) {
      mx = std::max<int64_t>(mx, rcounts[r] * es);
      end = std::max<int64_t>(end, (displs[r] + rcounts[r]) * es);
    }
    if (!codec && symm_x_window(mx)) {
      int64_t so[kMaxRanks], ro[kMaxRanks], b[kMaxRanks];
      for (int q = 0; q < c->world; ++q) {
        so[q] = 0;
        ro[q] = displs[c->rank] * es;
        b[q] = rcounts[c->rank] * es;
      }
      // Direct writes place rank q's block at ITS displs[q] in every output:
      // every rank must pass the same rcounts and displs (fold them into the
      // signature so a disagreement raises ORDER_MISMATCH instead of
      // scattering blocks to the wrong place).
      uint32_t sig = op_sig(kKindAllGatherv, dtype, 1, -1, 0, seq);
      for (int r = 0; r < c->world; ++r)
        sig = mix32(mix32(sig, uint64_t(rcounts[r])), uint64_t(displs[r]));
      sig &= ~kSigCodecBit;
      mcrdl_status_t st;
      if (try_exchange_symm(c, in, out, uint64_t(end), so, ro, b, mx, sig,
                            reinterpret_cast<cudaStream_t>(stream), &st))
        return st;
    }
  }
  ExchangeSpec s = empty_spec(es, op_sig(kKindAllGatherv, dtype, 0, -1, 0, seq));
  s.codec = codec;
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
  const int codec = split_codec(&algo, dtype);
  if (c == nullptr) return set_error(MCRDL_ERR_NOT_INITIALIZED, "communicator is NULL");
  const int es = elem_size(dtype);
  if (es == 0) return set_error(MCRDL_ERR_VALIDATION, "unknown dtype %d", int(dtype));
  if (root < 0 || root >= c->world)
    return set_error(MCRDL_ERR_VALIDATION, "root %d outside world %d", root, c->world);
  if (!check_counts(rcounts, displs, c->world, "rcounts")) return MCRDL_ERR_VALIDATION;
  if (c->rank == root && out == nullptr && rcounts[root] > 0)
    return set_error(MCRDL_ERR_VALIDATION, "root must supply the output buffer");
  ExchangeSpec s = empty_spec(es, op_sig(kKindGatherv, dtype, 0, root, 0, seq));
  s.codec = codec;
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

// Device-resident rcounts / displs (runtime.py:542-569 with tensors on the
// GPU): the exchange kernel reads them itself, no host round trip.
static mcrdl_status_t gather_dev(mcrdl_comm* c, int layout, int kind, const void* in,
                                 uint64_t in_count, void* out, uint64_t out_count,
                                 const int64_t* d_rcounts, const int64_t* d_displs, int root,
                                 mcrdl_dtype_t dtype, mcrdl_algo_t algo, uint64_t seq,
                                 void* stream) {
  const int codec = split_codec(&algo, dtype);
  if (c == nullptr) return set_error(MCRDL_ERR_NOT_INITIALIZED, "communicator is NULL");
  const int es = elem_size(dtype);
  if (es == 0) return set_error(MCRDL_ERR_VALIDATION, "unknown dtype %d", int(dtype));
  if (d_rcounts == nullptr || d_displs == nullptr)
    return set_error(MCRDL_ERR_VALIDATION, "NULL device count array");
  if (root < 0 || root >= c->world)
    return set_error(MCRDL_ERR_VALIDATION, "root %d outside world %d", root, c->world);
  ExchangeSpec s = empty_spec(es, op_sig(kind, dtype, 2, layout == kDevGatherv ? root : -1, 0, seq));
  s.codec = codec;
  s.d_counts = d_rcounts;
  s.d_displs = d_displs;
  s.d_layout = layout;
  s.d_root = root;
  s.in_base = reinterpret_cast<const uint8_t*>(in);
  s.out_base = reinterpret_cast<uint8_t*>(out);
  s.in_count = int64_t(in_count);
  s.out_count = out == nullptr ? 0 : int64_t(out_count);
  return launch_exchange(c, s, -1, reinterpret_cast<cudaStream_t>(stream));
}

mcrdl_status_t mcrdl_all_gatherv_dev(mcrdl_comm* c, const void* in, uint64_t in_count, void* out,
                                     uint64_t out_count, const int64_t* d_rcounts,
                                     const int64_t* d_displs, mcrdl_dtype_t dtype,
                                     mcrdl_algo_t algo, uint64_t seq, void* stream) {
  return gather_dev(c, kDevAllGatherv, kKindAllGatherv, in, in_count, out, out_count, d_rcounts,
                    d_displs, 0, dtype, algo, seq, stream);
}

mcrdl_status_t mcrdl_gatherv_dev(mcrdl_comm* c, const void* in, uint64_t in_count,
                                 void* out_or_null, uint64_t out_count, const int64_t* d_rcounts,
                                 const int64_t* d_displs, int root, mcrdl_dtype_t dtype,
                                 mcrdl_algo_t algo, uint64_t seq, void* stream) {
  // (an empty root output may be NULL: the device bounds check then rejects
  // any nonzero count)
  if (c != nullptr && c->rank == root && out_or_null == nullptr && out_count > 0)
    return set_error(MCRDL_ERR_VALIDATION, "root must supply the output buffer");
  return gather_dev(c, kDevGatherv, kKindGatherv, in, in_count, out_or_null, out_count, d_rcounts,
                    d_displs, root, dtype, algo, seq, stream);
}

mcrdl_status_t mcrdl_bcast(mcrdl_comm* c, void* buf, uint64_t count, mcrdl_dtype_t dtype, int root,
                           mcrdl_algo_t algo, uint64_t seq, void* stream) {
  const int codec = split_codec(&algo, dtype);
  if (c == nullptr) return set_error(MCRDL_ERR_NOT_INITIALIZED, "communicator is NULL");
  const int es = elem_size(dtype);
  if (es == 0) return set_error(MCRDL_ERR_VALIDATION, "unknown dtype %d", int(dtype));
  if (root < 0 || root >= c->world)
    return set_error(MCRDL_ERR_VALIDATION, "root %d outside world %d", root, c->world);
  if (c->world == 1) return MCRDL_OK;
  const int64_t nb = int64_t(count) * es;
  // NVLS (switch multicast): root egress S instead of (p-1)·S. AUTO takes it
  // above 32 MiB / (p-1) (measured crossover 4-16 MiB at p=4,
  // profiles/bcast_r1_p4.csv). The choice uses only values every rank agrees
  // on (the kernel copes with unaligned buffers and partial packs).
  const bool nv_ok = c->nvls.ok && nb > 0 && !codec;  // the multicast path moves raw bytes
  if (algo == MCRDL_ALGO_AUTO) algo = tuned_algo(c, MCRDL_TUNE_BCAST, uint64_t(nb));
  if (nv_ok && (algo == MCRDL_ALGO_NVLS ||
                (algo == MCRDL_ALGO_AUTO && c->world >= 3 &&
                 nb >= (int64_t(32) << 20) / (c->world - 1)))) {
    c->last_algo[MCRDL_TUNE_BCAST] = MCRDL_ALGO_NVLS;
    return launch_bcast_nvls(c, reinterpret_cast<uint8_t*>(buf), nb, root, int(dtype), count, seq,
                             reinterpret_cast<cudaStream_t>(stream));
  }
  if (algo == MCRDL_ALGO_CHAIN && !codec) {
    c->last_algo[MCRDL_TUNE_BCAST] = MCRDL_ALGO_CHAIN;
    return launch_bcast_chain(c, reinterpret_cast<uint8_t*>(buf), nb, root, int(dtype), count, seq,
                              reinterpret_cast<cudaStream_t>(stream));
  }
  c->last_algo[MCRDL_TUNE_BCAST] = MCRDL_ALGO_DIRECT_WRITE;
  ExchangeSpec s = empty_spec(es, op_sig(kKindBcast, dtype, 0, root, count, seq));
  s.codec = codec;
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
