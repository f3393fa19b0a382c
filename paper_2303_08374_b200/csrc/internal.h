// Host-side communicator state and helpers shared by the launch files.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdarg>
#include <cstdint>
#include <map>
#include <string>
#include <utility>
#include <vector>

#include "../../include/mcrdl_nvl.h"
#include "common.cuh"

namespace mcrdl {

// One peer-mapped VMM region (the base pad+workspace or a user symmetric alloc).
struct Region {
  uint64_t bytes = 0;  // mapped size (granularity-rounded)
  CUmemGenericAllocationHandle local_handle = 0;
  CUmemGenericAllocationHandle handles[kMaxRanks] = {};
  CUdeviceptr ptr[kMaxRanks] = {};  // rank r's region mapped here
  // user symmetric allocations only: NVSwitch multicast view of the region
  // (every rank's physical copy bound to one multicast object), else 0
  CUmemGenericAllocationHandle mc_handle = 0;
  CUdeviceptr mc_ptr = 0;
  bool mc_bound = false;
};

// NVSwitch multicast (NVLS) buffer: one physical allocation per rank bound
// to a multicast object; uc_ptr is this rank's own (unicast) mapping, mc_ptr
// the multicast mapping whose loads reduce across ranks in the switch
// (multimem.ld_reduce) and whose stores land on every rank (multimem.st).
struct Nvls {
  bool ok = false;
  CUmemGenericAllocationHandle mc_handle = 0;
  CUmemGenericAllocationHandle mem_handle = 0;
  CUdeviceptr mc_ptr = 0;
  CUdeviceptr uc_ptr = 0;
  uint64_t bytes = 0;  // two halves (epoch parity)
  bool bound = false;
};

}  // namespace mcrdl

struct mcrdl_comm {
  int rank = 0;
  int world = 1;
  int device = 0;
  // SM budget every launch is sized from (grids stay <= 2 CTAs per budgeted
  // SM). The device's SM count, divided between the ranks that share this
  // GPU (co-located ranks: their spinning grids must all be resident at once),
  // capped by MCRDL_MAX_SMS (leave SMs to overlapped compute), and agreed by
  // every rank (min) because launch geometry must match across ranks.
  int num_sms = 0;
  int ranks_per_device = 1;  // max ranks sharing one physical GPU in this comm
  // The comm's own non-blocking stream, created on first request: the host
  // layer's lane for async posts (mcrdl_comm_stream). One per comm, never
  // pooled, so two communicators (e.g. co-located ranks) never share one.
  cudaStream_t aux = nullptr;
  cudaStream_t xfer[2] = {nullptr, nullptr};  // H2D / D2H staging (pipelined host posts)
  int fd_tag = 0;                              // fd-exchange round counter
  std::map<std::pair<int, int>, int> fd_stash; // (tag, rank) -> early fd
  mcrdl_allgather_fn allgather = nullptr;
  void* ag_ctx = nullptr;
  uint64_t jobid = 0;
  int listen_fd = -1;
  uint64_t gran = 0;
  mcrdl::Region base;                 // [pad | workspace]
  std::vector<mcrdl::Region> symm;    // user symmetric allocations
  mcrdl::Nvls nvls;
  int* err_host = nullptr;            // cudaHostAllocMapped
  int* err_dev = nullptr;
  uint64_t timeout_ns = 30ull * 1000000000ull;
  uint64_t ws_bytes = 0;
  mcrdl::DevComm dc{};
  int sticky = MCRDL_OK;              // poisoned after a device error
  // Ops of one order chain must run in issue order on the device (flag
  // epochs / p2p stream counters / the shared exit counter). Ops may be
  // issued on different streams: when the stream changes, the new stream
  // waits for the previous one (event, no host sync). Chains: collectives,
  // sends, receives — they use disjoint pad words, so a recv may run
  // concurrently with a send or a collective on another stream.
  struct Chain {
    cudaEvent_t ev = nullptr;
    cudaStream_t last = nullptr;
    bool have = false;
  } chain[3];
  uint64_t* trace_host = nullptr;  // trace builds: kMaxBlocks x kTraceSlots stamps
  uint64_t* oplog_host = nullptr;  // kOpLogSlots x {tag0, t0, tag1, t1} (mapped)
  uint64_t log_seq = 0;            // last log id handed to a launch
  // tuning rows per MCRDL_TUNE_* kind: (max_bytes ascending, algorithm)
  std::vector<std::pair<uint64_t, int>> tune[MCRDL_TUNE_KINDS];
  int last_algo[MCRDL_TUNE_KINDS] = {0, 0};
};

namespace mcrdl {

// Thread-local last-error message + return code.
mcrdl_status_t set_error(mcrdl_status_t code, const char* fmt, ...);
void count_launch();

#define MCRDL_CUDA_CHECK(expr)                                                        \
  do {                                                                                \
    cudaError_t e_ = (expr);                                                          \
    if (e_ != cudaSuccess)                                                            \
      return ::mcrdl::set_error(MCRDL_ERR_CUDA, "%s failed: %s (%s:%d)", #expr,      \
                                cudaGetErrorString(e_), __FILE__, __LINE__);          \
  } while (0)

// Validates the comm and orders `stream` after the comm's previous op. The
// op epoch itself lives on the device (Pad::dev_epoch, common.cuh), so a
// launch carries no per-op host state and can be replayed from a CUDA graph.
enum : int { kChainCollective = 0, kChainSend = 1, kChainRecv = 2 };

// The user symmetric allocation holding [p, p + bytes) (nullptr if none);
// *off = p - region base. Every rank maps every rank's copy at ptr[r].
const Region* find_symm(const mcrdl_comm* c, const void* p, uint64_t bytes, uint64_t* off);
mcrdl_status_t begin_op(mcrdl_comm* comm, cudaStream_t stream, int chain = kChainCollective);

// Tuning-table algorithm for `bytes` of op `kind`, or AUTO if no rows.
inline mcrdl_algo_t tuned_algo(const mcrdl_comm* c, int kind, uint64_t bytes) {
  const auto& rows = c->tune[kind];
  if (rows.empty()) return MCRDL_ALGO_AUTO;
  for (const auto& r : rows)
    if (bytes <= r.first) return mcrdl_algo_t(r.second);
  return mcrdl_algo_t(rows.back().second);
}

inline int64_t env_int(const char* name, int64_t dflt) {
  const char* e = getenv(name);
  return (e && *e) ? int64_t(strtoll(e, nullptr, 10)) : dflt;
}

inline int elem_size(mcrdl_dtype_t dt) {
  switch (dt) {
    case MCRDL_F32: return 4;
    case MCRDL_F64: return 8;
    case MCRDL_I32: return 4;
    case MCRDL_I64: return 8;
    case MCRDL_U8: return 1;
    case MCRDL_BF16: return 2;
  }
  return 0;
}

inline uint32_t op_sig(int kind, int dtype, int op, int root, uint64_t count, uint64_t seq) {
  uint32_t h = 2166136261u;
  h = mix32(h, uint64_t(kind));
  h = mix32(h, uint64_t(dtype));
  h = mix32(h, uint64_t(op));
  h = mix32(h, uint64_t(int64_t(root)));
  h = mix32(h, count);
  h = mix32(h, seq);
  return h & ~kSigCodecBit;  // bit 19 of the flag signature is the codec flag
}

// Kind tags folded into signatures (CommOpKind order, core.py:89-104).
enum KindTag : int {
  kKindBcast = 2,
  kKindReduce = 3,
  kKindAllReduce = 4,
  kKindGatherv = 6,
  kKindAllGatherv = 10,
  kKindA2ASingle = 12,
  kKindA2AList = 13,
  kKindA2AV = 14,
  kKindReduceScatter = 11,
  kKindBarrier = 99,
};

// Exchange engine entry (exchange.cu): per-peer send/recv byte spans.
struct ExchangeSpec {
  int codec;  // 1: trunc16 on peer pairs (f32 only)
  const uint8_t* sptr[kMaxRanks];
  int64_t sbytes[kMaxRanks];
  uint8_t* rptr[kMaxRanks];
  int64_t rbytes[kMaxRanks];
  const int64_t* d_counts;  // optional device counts (elements), see d_layout
  const int64_t* d_displs;  // gather layouts: device displacements (elements)
  int d_layout;             // kDevA2AV / kDevAllGatherv / kDevGatherv
  int d_root;               // kDevGatherv: the root
  const uint8_t* in_base;
  uint8_t* out_base;
  int64_t in_count;  // element capacities for device-count bounds checks
  int64_t out_count;
  int esize;
  uint32_t sig_base;
};
// Device-resident count layouts the exchange kernel decodes itself:
//   kDevA2AV:       d_counts = [scounts | sdispls | rcounts | rdispls] (4p)
//   kDevAllGatherv: d_counts = rcounts (p), d_displs = displs (p)
//   kDevGatherv:    as all_gatherv, only pairs with d_root carry data
enum : int { kDevA2AV = 0, kDevAllGatherv = 1, kDevGatherv = 2 };
mcrdl_status_t launch_exchange(mcrdl_comm* comm, const ExchangeSpec& spec, int64_t total_hint,
                               cudaStream_t stream);

// LL protocol (ll.cu) for small messages.
constexpr int64_t kLLMaxPairBytes = 256 << 10;  // measured: tools/ll_ab.sh, profiles/ll_ab_r1_p{2,4}.log      // exchange: every pair <= this
// Last bytes of each NVLS half: multicast flag words (bcast), zeroed at init.
constexpr int64_t kNvlsFlagBytes = 64 << 10;
mcrdl_status_t launch_bcast_chain(mcrdl_comm* c, uint8_t* buf, int64_t nbytes, int root,
                                  int dtype, uint64_t count, uint64_t seq, cudaStream_t stream);
mcrdl_status_t launch_bcast_nvls(mcrdl_comm* c, uint8_t* buf, int64_t nbytes, int root, int dtype,
                                 uint64_t count, uint64_t seq, cudaStream_t stream);
// all_reduce one-shot message <= this takes LL lines; above, the bulk one-shot.
// 128 KiB measured (profiles/r2_ll_threshold_p{2,4}.csv): at 256 KiB the bulk
// one-shot beats LL (p = 4: 14.0 vs 17.2 us, p = 2: 11.4 vs 11.9), at 128 KiB
// LL still wins (13.4 vs 13.8, 9.8 vs 10.8).
constexpr int64_t kLLMaxAllReduceBytes = 128 << 10;
int64_t exchange_ll_max();
bool try_exchange_symm(mcrdl_comm* c, const void* in, void* out, uint64_t out_bytes,
                       const int64_t* send_off, const int64_t* recv_off, const int64_t* bytes,
                       int64_t grid_bytes, uint32_t sig, cudaStream_t stream, mcrdl_status_t* st);
bool try_exchange_ll(mcrdl_comm* c, const ExchangeSpec& sp, int64_t ll_max, cudaStream_t stream,
                     mcrdl_status_t* st);
template <typename T, int OP>
mcrdl_status_t launch_ar_ll(mcrdl_comm* c, const T* in, T* out, int64_t n,
                            uint32_t sig, cudaStream_t stream);

}  // namespace mcrdl
