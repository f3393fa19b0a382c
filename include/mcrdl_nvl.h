/*
 * mcrdl_nvl.h — C ABI of the B200-native NVLink/NVSwitch collective backend.
 *
 * This is the drop-in boundary below the MCR-DL Python API. In the reference
 * (pure Python, /root/reference/pkg/src/mcrdl) the seam it replaces is
 *
 *   BackendInstance.execute(request)            runtime.py:238-277
 *     -> run_collective(transport, rank, p, req, algorithm, ...)
 *                                                collectives.py:769-789
 *        -> _agree_header  (order/count check)   collectives.py:245-285
 *        -> _IMPLS[(kind, algorithm)](...)       collectives.py:736-766
 *   Runtime._build_transport(config)             runtime.py:359-383
 *
 * Every entry point is plain C: raw device pointers, element counts, enum
 * codes and a cudaStream_t passed as void*. No torch types cross the ABI.
 * Every function returns an mcrdl_status_t; the thread-local message for the
 * last failure is available from mcrdl_last_error(). Status codes map 1:1 to
 * the reference error kinds (errors.py:11-117), see mcrdl_status_kind().
 *
 * Concurrency contract (mirrors the reference's per-backend single-in-flight
 * lane, runtime.py:117-119): one host thread at a time per communicator;
 * calls are asynchronous w.r.t. the host and ordered on the given stream.
 * Every rank must issue the same sequence of collective calls on a
 * communicator (the reference's posting-order contract); a
 * divergence is detected on the device and reported as
 * MCRDL_ERR_ORDER_MISMATCH by mcrdl_comm_status().
 */
#ifndef MCRDL_NVL_H_
#define MCRDL_NVL_H_

#include <stddef.h>
#include <stdint.h>
#include <sys/types.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MCRDL_NVL_ABI_VERSION 1
#define MCRDL_MAX_RANKS 8

typedef int mcrdl_status_t;

/* Status codes. The string kinds match errors.py `kind` attributes. */
enum {
  MCRDL_OK = 0,
  MCRDL_ERR_VALIDATION = 1,        /* "validation"            errors.py:17 */
  MCRDL_ERR_ORDER_MISMATCH = 2,    /* "order_mismatch"        errors.py:37 */
  MCRDL_ERR_TIMEOUT = 3,           /* "timeout"               errors.py:42 */
  MCRDL_ERR_UNSUPPORTED = 4,       /* "unsupported_operation" errors.py:95 */
  MCRDL_ERR_PEER_DISCONNECTED = 5, /* "peer_disconnected"     errors.py:58 */
  MCRDL_ERR_CUDA = 6,              /* "comm_error" (device/driver failure) */
  MCRDL_ERR_BOOTSTRAP = 7,         /* "bootstrap_timeout"     errors.py:46 */
  MCRDL_ERR_LENGTH_MISMATCH = 8,   /* "length_mismatch"       errors.py:62 */
  MCRDL_ERR_NOT_INITIALIZED = 9,   /* "not_initialized"       errors.py:83 */
  MCRDL_ERR_INTERNAL = 10,         /* "comm_error"                          */
  MCRDL_ERR_CODEC_MISMATCH = 11    /* "codec_mismatch"        errors.py:106 */
};

/* Element types: the reference DType (core.py:23-28) plus bf16. */
typedef enum {
  MCRDL_F32 = 0,
  MCRDL_F64 = 1,
  MCRDL_I32 = 2,
  MCRDL_I64 = 3,
  MCRDL_U8 = 4,
  MCRDL_BF16 = 5
} mcrdl_dtype_t;

/* Reduce ops: core.py:53-79 (C-style integer wrap, IEEE floats). */
typedef enum { MCRDL_SUM = 0, MCRDL_PROD = 1, MCRDL_MIN = 2, MCRDL_MAX = 3 } mcrdl_redop_t;

/* Algorithms inside the single NVLink backend. These extend the reference's
 * ALGORITHMS registry (collectives.py:36-52) and are what the tuning table's
 * optional "algorithm" key names. MCRDL_ALGO_AUTO lets the library pick by
 * message size (used when no tuning table is loaded). */
typedef enum {
  MCRDL_ALGO_AUTO = 0,
  MCRDL_ALGO_ONE_SHOT = 1,     /* all_reduce: push to all, local ascending fold   */
  MCRDL_ALGO_TWO_SHOT = 2,     /* all_reduce: RS by push + fold, AG by push      */
  MCRDL_ALGO_NVLS = 3,         /* all_reduce / bcast through NVSwitch multicast  */
  MCRDL_ALGO_DIRECT_WRITE = 4, /* a2a(v), allgatherv, gatherv, bcast: push      */
  MCRDL_ALGO_CHAIN = 5         /* bcast: pipelined chain root -> root+1 -> ...   */
} mcrdl_algo_t;

/* Payload codec flag, OR-ed into the `algo` argument of the movement
 * collectives (all_to_all*, all_gatherv, gatherv, bcast): Trunc16Codec
 * (middleware.py:43-75) fused into the exchange kernel — senders keep the top
 * 16 bits of every f32 (sign, exponent, 7 mantissa bits) and push 2 bytes per
 * element over NVLink, receivers widen with zero fill; a rank's own segment
 * is copied exactly (it never crosses the transport). Ignored for non-f32
 * payloads (CompressionConfig.active_for, middleware.py:86-95). Ranks that
 * disagree on the codec fail with MCRDL_ERR_CODEC_MISMATCH
 * (collectives.py:226-228, 284). */
#define MCRDL_CODEC_TRUNC16 0x100

/* Bootstrap all-gather supplied by the host runtime (the reference's star
 * bootstrap, transport.py:279-376, or a torch TCPStore). Must gather
 * `nbytes` from every rank into recv[rank * nbytes]. Return 0 on success. */
typedef int (*mcrdl_allgather_fn)(void* ctx, const void* send, void* recv, size_t nbytes);

typedef struct mcrdl_comm mcrdl_comm;

typedef struct {
  int rank;
  int world;
  int device;
  int num_sms;               /* SM budget launches are sized from (device SMs,
                                split between co-located ranks, MCRDL_MAX_SMS) */
  int nvls_supported;        /* NVSwitch multicast object usable */
  int ranks_per_device;      /* >1: ranks share a GPU (co-located test mode) */
  uint64_t workspace_bytes;  /* symmetric workspace per rank (two halves) */
  uint64_t max_oneshot_bytes;/* largest all_reduce the one-shot path takes */
  uint64_t max_twoshot_chunk;/* per-launch all_reduce chunk for two-shot   */
} mcrdl_caps_t;

/* -------------------------------------------------------------- lifecycle */
/* Reference: Runtime.init -> _build_transport (runtime.py:336-383). Collective
 * over all ranks: allocates the symmetric workspace + signal pad with cuMem
 * VMM, exchanges POSIX-fd handles over a unix socket, maps every peer over
 * NVLink and (when available) builds an NVLS multicast object. */
mcrdl_status_t mcrdl_comm_init(mcrdl_comm** comm, int rank, int world, int cuda_device,
                               mcrdl_allgather_fn allgather, void* ctx,
                               uint64_t workspace_bytes, double timeout_secs);
/* Reference: BackendInstance.finalize (runtime.py:279-290). */
mcrdl_status_t mcrdl_comm_destroy(mcrdl_comm* comm);
mcrdl_status_t mcrdl_comm_caps(const mcrdl_comm* comm, mcrdl_caps_t* caps);
/* The communicator's own non-blocking CUDA streams (created at init,
 * destroyed with the comm): which = 0 the host layer's progress lane for async
 * posts (reference: the per-backend lane thread, runtime.py:117-126), 1 / 2 the
 * H2D / D2H staging streams of pipelined host-buffer posts. Never shared
 * between communicators; they stay valid after mcrdl_comm_destroy (until
 * process exit), since callers may still hold stream-ordered references. */
mcrdl_status_t mcrdl_comm_stream(mcrdl_comm* comm, int which, void** stream);

/* Tuning table -> MCRDL_ALGO_AUTO (reference: TuningTable.lookup + the
 * runtime's table load, dispatch.py:135-150, runtime.py:330-332; the paper's
 * "mix-and-match" reinterpreted as per-op, per-size algorithm choice). For op
 * kind `kind` (MCRDL_TUNE_ALL_REDUCE / MCRDL_TUNE_BCAST) install n rows
 * (max_bytes ascending, algo): AUTO takes the first row with message bytes
 * <= max_bytes, else the last row. n = 0 restores the built-in crossovers.
 * Every rank must install the same rows (the algorithm is folded into the
 * flag signature: a disagreement raises ORDER_MISMATCH). */
enum { MCRDL_TUNE_ALL_REDUCE = 0, MCRDL_TUNE_BCAST = 1, MCRDL_TUNE_KINDS = 2 };
mcrdl_status_t mcrdl_comm_set_tuning(mcrdl_comm* comm, int kind, int n, const uint64_t* max_bytes,
                                     const int* algos);
/* Algorithm (mcrdl_algo_t) the last all_reduce / bcast launch of this
 * communicator ran (its AUTO resolution), for logs and tests. */
int mcrdl_comm_last_algo(const mcrdl_comm* comm, int kind);
/* Latched device error (order mismatch / timeout) of every op issued so far,
 * read without a device sync: call after the stream work completed
 * (WorkHandle.wait / Runtime.synchronize, core.py:312-319, runtime.py:470-494).
 * Returns MCRDL_OK or the first error, and keeps it latched (the communicator
 * is poisoned after a device-detected error). */
mcrdl_status_t mcrdl_comm_status(mcrdl_comm* comm);

/* Device-timed op log (CommLog durations: the reference appends one record
 * per completed op, runtime.py:209-230, middleware.py:100-124). Every kernel
 * launch stamps %globaltimer at entry and exit into a ring in device memory —
 * no stream commands, no host sync — and every 64th launch mirrors the last 64
 * entries to a host-mapped copy. mcrdl_comm_log_id returns the id of the last
 * launch issued (an op that launched kernels first..last); mcrdl_comm_op_time
 * sets *ns to end(last) - start(first) from the host copy, -1 while not
 * (yet) mirrored, -2 when the 4096-entry ring moved past it;
 * mcrdl_comm_log_flush mirrors the whole ring now (host-synchronous: call it
 * once the communicator's work has completed). Launches inside a CUDA-graph
 * capture are not logged. */
mcrdl_status_t mcrdl_comm_log_flush(mcrdl_comm* comm);
uint64_t mcrdl_comm_log_id(const mcrdl_comm* comm);
mcrdl_status_t mcrdl_comm_op_time(const mcrdl_comm* comm, uint64_t first, uint64_t last,
                                  int64_t* ns);

/* Symmetric allocation (collective, same size on every rank). The returned
 * local pointer is peer-mapped, so ops whose output lies in it can be written
 * zero-copy by peers. */
mcrdl_status_t mcrdl_symm_alloc(mcrdl_comm* comm, uint64_t bytes, void** local_ptr);
mcrdl_status_t mcrdl_symm_free(mcrdl_comm* comm, void* local_ptr);

/* Symmetric memory pool (csrc/pool.cu): one collective symmetric arena per
 * pool, sub-allocated first-fit by torch's pluggable-allocator hooks
 * (torch.cuda.MemPool over mcrdl_pool_malloc / mcrdl_pool_free), so ordinary
 * framework tensors allocated inside it take the zero-copy paths (k_ar_symm,
 * k_x_symm) whenever every rank allocates in the same order. mcrdl_pool_create
 * is collective; mcrdl_pool_activate selects the calling thread's pool for
 * mcrdl_pool_malloc (NULL: none -> malloc returns NULL). */
typedef struct mcrdl_pool mcrdl_pool;
mcrdl_status_t mcrdl_pool_create(mcrdl_comm* comm, uint64_t bytes, mcrdl_pool** pool);
mcrdl_status_t mcrdl_pool_activate(mcrdl_pool* pool);
mcrdl_status_t mcrdl_pool_stats(mcrdl_pool* pool, uint64_t* base, uint64_t* bytes, uint64_t* in_use);
mcrdl_status_t mcrdl_pool_destroy(mcrdl_pool* pool);
void* mcrdl_pool_malloc(ssize_t size, int device, void* stream);
void mcrdl_pool_free(void* ptr, size_t size, int device, void* stream);

/* ------------------------------------------------------------ collectives */
/* `seq` is the reference's per-backend request seq (runtime.py:147-149); it
 * is folded with the op signature into every device flag so ranks that
 * posted different operations fail with ORDER_MISMATCH (collectives.py:215-285). */

/* all_reduce (runtime.py:510-517; oracle reference.py:23-25). `in` may equal
 * `out`. one_shot/two_shot fold ranks in ascending order: bit-identical to
 * the sequential oracle for every dtype/op. */
mcrdl_status_t mcrdl_all_reduce(mcrdl_comm* comm, const void* in, void* out, uint64_t count,
                                mcrdl_dtype_t dtype, mcrdl_redop_t op, mcrdl_algo_t algo,
                                uint64_t seq, void* stream);

/* reduce (runtime.py:519-526; oracle reference.py:27-33): the two-shot
 * pipeline in root mode — every rank's reduced segment goes to the root only
 * (ascending fold, bit-exact). `out` is written on the root only and may be
 * NULL elsewhere. */
mcrdl_status_t mcrdl_reduce(mcrdl_comm* comm, const void* in, void* out, uint64_t count,
                            mcrdl_dtype_t dtype, mcrdl_redop_t op, int root, mcrdl_algo_t algo,
                            uint64_t seq, void* stream);

/* reduce_scatter (runtime.py:590-597; collectives.py:609-645; oracle
 * reference.py:79-83): in holds world*recvcount elements, rank r receives the
 * ascending-fold reduction of segment r. Needs 16-byte aligned buffers and
 * recvcount*esize % 16 == 0 within one workspace half, else
 * MCRDL_ERR_UNSUPPORTED (compose all_reduce + slice). */
mcrdl_status_t mcrdl_reduce_scatter(mcrdl_comm* comm, const void* in, void* out, uint64_t recvcount,
                                    mcrdl_dtype_t dtype, mcrdl_redop_t op, mcrdl_algo_t algo,
                                    uint64_t seq, void* stream);

/* all_to_allv (runtime.py:616-626; collectives.py:648-733). Counts and
 * displacements are in ELEMENTS. Host-array form: four arrays of `world`
 * int64 values on the host (passed by value into the kernel; no H2D copy). */
mcrdl_status_t mcrdl_all_to_allv(mcrdl_comm* comm, const void* in, void* out,
                                 const int64_t* scounts, const int64_t* sdispls,
                                 const int64_t* rcounts, const int64_t* rdispls,
                                 mcrdl_dtype_t dtype, mcrdl_algo_t algo, uint64_t seq,
                                 void* stream);
/* Device-resident form: d_counts points to 4*world int64 in device memory laid
 * out [scounts | sdispls | rcounts | rdispls]; the kernel reads them itself,
 * so counts produced on the GPU (MoE routing) need no host round trip.
 * in_count/out_count (elements) bound every segment; a violation is latched
 * as MCRDL_ERR_VALIDATION on the device. */
mcrdl_status_t mcrdl_all_to_allv_dev(mcrdl_comm* comm, const void* in, uint64_t in_count,
                                     void* out, uint64_t out_count, const int64_t* d_counts,
                                     mcrdl_dtype_t dtype, mcrdl_algo_t algo, uint64_t seq,
                                     void* stream);
/* all_to_all_single (runtime.py:599-605): count = total elements per rank. */
mcrdl_status_t mcrdl_all_to_all_single(mcrdl_comm* comm, const void* in, void* out,
                                       uint64_t count, mcrdl_dtype_t dtype, mcrdl_algo_t algo,
                                       uint64_t seq, void* stream);
/* all_to_all list form (runtime.py:607-614): world input and output block
 * pointers, counts in elements (host arrays). */
mcrdl_status_t mcrdl_all_to_all_ptrs(mcrdl_comm* comm, const void* const* in_ptrs,
                                     const int64_t* in_counts, void* const* out_ptrs,
                                     const int64_t* out_counts, mcrdl_dtype_t dtype,
                                     mcrdl_algo_t algo, uint64_t seq, void* stream);
/* all_gatherv (runtime.py:542-550; collectives.py:446-512). in holds
 * rcounts[rank] elements; out receives segment j at displs[j]. */
mcrdl_status_t mcrdl_all_gatherv(mcrdl_comm* comm, const void* in, void* out,
                                 const int64_t* rcounts, const int64_t* displs,
                                 mcrdl_dtype_t dtype, mcrdl_algo_t algo, uint64_t seq,
                                 void* stream);
/* gatherv (runtime.py:561-569; collectives.py:515-525). out may be NULL on
 * non-root ranks (core.py:513-527). */
mcrdl_status_t mcrdl_gatherv(mcrdl_comm* comm, const void* in, void* out_or_null,
                             const int64_t* rcounts, const int64_t* displs, int root,
                             mcrdl_dtype_t dtype, mcrdl_algo_t algo, uint64_t seq, void* stream);
/* Device-resident forms of all_gatherv / gatherv (runtime.py:542-569 with
 * rcounts / displs already on the GPU): d_rcounts and d_displs point to world
 * int64 each in device memory; the exchange kernel reads them itself (no host
 * round trip). in_count / out_count (elements) bound every segment; a
 * violation is latched as MCRDL_ERR_VALIDATION on the device. gatherv: out may
 * be NULL (out_count ignored) on non-root ranks. */
mcrdl_status_t mcrdl_all_gatherv_dev(mcrdl_comm* comm, const void* in, uint64_t in_count,
                                     void* out, uint64_t out_count, const int64_t* d_rcounts,
                                     const int64_t* d_displs, mcrdl_dtype_t dtype,
                                     mcrdl_algo_t algo, uint64_t seq, void* stream);
mcrdl_status_t mcrdl_gatherv_dev(mcrdl_comm* comm, const void* in, uint64_t in_count,
                                 void* out_or_null, uint64_t out_count, const int64_t* d_rcounts,
                                 const int64_t* d_displs, int root, mcrdl_dtype_t dtype,
                                 mcrdl_algo_t algo, uint64_t seq, void* stream);
/* bcast in place (runtime.py:528-532; collectives.py:418-443). */
mcrdl_status_t mcrdl_bcast(mcrdl_comm* comm, void* buf, uint64_t count, mcrdl_dtype_t dtype,
                           int root, mcrdl_algo_t algo, uint64_t seq, void* stream);
/* 0-byte collective used as a barrier by the tuner (tuner.py:151-159). */
mcrdl_status_t mcrdl_barrier(mcrdl_comm* comm, uint64_t seq, void* stream);
/* Point-to-point (Runtime.send / Runtime.recv, runtime.py:498-508, executed by
 * BackendInstance.execute, runtime.py:244-262). Only the two endpoints take
 * part; no collective sequence number is consumed. Messages are matched in
 * post order per (sender, receiver) pair. send is eager: messages <= 256 KiB
 * (LL path) up to 64 outstanding, larger ones up to 256 queued messages and
 * the per-sender mailbox (MCRDL_P2P_BYTES, default 32 MiB); beyond that it
 * streams larger messages through it (the matching recv must then be in
 * flight: post it first, on another stream). Sends, receives and collectives
 * are ordered only within their own kind, so a recv may overlap a send. A byte-count
 * difference latches MCRDL_ERR_LENGTH_MISMATCH on the receiver (runtime.py:
 * 256-260). peer == own rank is allowed. */
mcrdl_status_t mcrdl_send(mcrdl_comm* comm, const void* buf, uint64_t bytes, int peer, void* stream);
mcrdl_status_t mcrdl_recv(mcrdl_comm* comm, void* buf, uint64_t bytes, int peer, void* stream);

/* ----------------------------------------------------------------- fusion */
/* Tensor fusion (middleware.py:222-359). Segment tables are device arrays of
 * n entries: source/destination pointers, byte sizes and byte offsets into
 * the packed buffer. */
mcrdl_status_t mcrdl_fusion_pack(const void* const* d_src_ptrs, const int64_t* d_nbytes,
                                 const int64_t* d_offsets, int n, void* dst, void* stream);
mcrdl_status_t mcrdl_fusion_unpack(const void* src, void* const* d_dst_ptrs,
                                   const int64_t* d_nbytes, const int64_t* d_offsets, int n,
                                   void* stream);
/* pack -> all_reduce -> unpack in ONE launch: member i reads d_in_ptrs[i] and
 * writes d_out_ptrs[i] (may alias), d_counts[i] elements at element offset
 * d_offsets[i] of the virtual packed buffer (each offset a multiple of
 * 16 bytes, ascending, non-overlapping); total_count = packed length. */
mcrdl_status_t mcrdl_all_reduce_fused(mcrdl_comm* comm, const void* const* d_in_ptrs,
                                      void* const* d_out_ptrs, const int64_t* d_counts,
                                      const int64_t* d_offsets, int n,
                                      uint64_t total_count, mcrdl_dtype_t dtype,
                                      mcrdl_redop_t op, mcrdl_algo_t algo, uint64_t seq,
                                      void* stream);

/* ------------------------------------------------------------------ misc */
const char* mcrdl_last_error(void);
const char* mcrdl_status_kind(mcrdl_status_t status);
int mcrdl_abi_version(void);
/* Number of kernels this library launched since load (evidence counter). */
uint64_t mcrdl_launch_count(void);
/* Developer timeline: host-mapped [512 CTAs x slots] %globaltimer stamps of
 * the last ops (NULL unless the library was built with `build.py --trace`). */
mcrdl_status_t mcrdl_debug_trace(mcrdl_comm* comm, uint64_t** host_ptr, uint64_t* slots_per_cta);

#ifdef __cplusplus
}
#endif
#endif /* MCRDL_NVL_H_ */
