// Point-to-point send/recv over NVLink (reference: Runtime.send/recv,
// runtime.py:498-508, executed by BackendInstance.execute, runtime.py:244-262).
//
// Reference semantics restated:
//  * send is eager: the payload is queued on the transport and the sender
//    moves on (transport.send, transport.py:175);
//  * recv blocks for the next payload frame from `peer`; a byte count that
//    differs from the posted buffer raises LengthMismatch (runtime.py:256-260);
//  * no header agreement and no collective sequence number: only the two
//    endpoints take part.
//
// Device design. Every rank owns, after its collective workspace, one mailbox
// per sender: a ring of K = mbox_bytes / 64 KiB chunk slots. A message of B
// bytes is ceil(B / 64 KiB) chunks numbered on a per-(src, dst) stream that
// never resets (device-resident counters in the local pad, so no host state
// changes between messages and launches replay from CUDA graphs):
//  * sender CTA b moves chunks b, b+G, ...: waits until dst freed the slot
//    (p2p_free >= g - K + 1), pushes the chunk into dst's mailbox over NVLink,
//    publishes p2p_full[src][slot] = g + 1 in dst's pad (release);
//  * receiver CTA b waits p2p_full >= g + 1, copies the slot into the user
//    buffer, publishes p2p_free[dst][slot] = g + 1 in the sender's pad;
//  * a per-message header {msg + 1, bytes} (256-deep ring, acked by the
//    receiver) carries the byte count for the LengthMismatch check.
// Up to 256 messages / the mailbox capacity per pair complete without the
// receiver (eager, like the reference); larger ones stream through the ring and need the
// matching recv to be in flight (rendezvous) — post the recv on another stream
// or before the send when a rank both sends and receives large messages.
#include <algorithm>

#include "ll.cuh"

namespace mcrdl {

namespace {

constexpr int kP2PThreads = 512;

__device__ __forceinline__ uint8_t* mailbox(const DevComm& c, uint8_t* ws_owner, int sender) {
  return ws_owner + 2 * c.half_bytes + int64_t(sender) * c.mbox_bytes;
}

// LL ring of `sender` in the mailbox area of the rank owning `ws_owner`
// (after the bulk mailboxes).
__device__ __forceinline__ uint8_t* ll_box(const DevComm& c, uint8_t* ws_owner, int sender) {
  return ws_owner + 2 * c.half_bytes + int64_t(c.world) * c.mbox_bytes +
         int64_t(sender) * kP2PLLSenderBytes;
}

// Receiver side: wait for message `msg` from `peer` on EITHER path and report
// which one the sender took (a byte-count disagreement can make the two ends
// choose different paths: that is a LengthMismatch, not a hang).
static __device__ __noinline__ int p2p_wait_header(const DevComm& c, const Pad* me, int peer,
                                                   const uint8_t* ll_hdr, uint64_t msg,
                                                   bool* via_ll, uint64_t* bytes) {
  const uint64_t* h = me->p2p_hdr[peer][msg % kP2PHdr];
  const uint32_t tag = uint32_t(msg + 1);
  uint64_t start = 0;
  for (int spins = 0;; ++spins) {
    if (ld_acquire_sys(&h[0]) >= msg + 1) {
      if (ld_relaxed_sys(&h[0]) != msg + 1) return MCRDL_ERR_ORDER_MISMATCH;  // lapped
      *via_ll = false;
      *bytes = ld_relaxed_sys(&h[1]);
      return MCRDL_OK;
    }
    const uint4 v = ld_ll(ll_hdr);
    if (ll_ready(v, tag)) {
      *via_ll = true;
      *bytes = uint64_t(v.x) | (uint64_t(v.z) << 32);
      return MCRDL_OK;
    }
    if (spins >= 32) {
      spins = 0;
      if (const uint64_t pz = ld_relaxed_sys(&me->poison)) return int(pz);
      const uint64_t now = globaltimer_ns();
      if (start == 0) start = now;
      else if (now - start > c.timeout_ns) return MCRDL_ERR_TIMEOUT;
    }
  }
}

__device__ __forceinline__ bool last_cta(const DevComm& c, int dir);

// ------------------------------------------------------------ LL messages
// One CTA. Sender: wait until the receiver matched message msg - kP2PLLSlots
// (p2p_hdr_ack counts every message, LL or bulk), then write the payload as
// {d0, tag, d1, tag} lines and the header line {bytes, tag} — no fences, no
// flags. Receiver: poll the header line, then the data lines themselves.
__global__ void __launch_bounds__(kP2PThreads)
    k_send_ll(DevComm c, uint8_t* peer_ws, const uint8_t* buf, int64_t bytes, int peer) {
  __shared__ uint64_t s_msg;
  __shared__ int s_err;
  Pad* me = c.self;
  oplog_start(c);
  if (threadIdx.x == 0) {
    const uint64_t msg = *reinterpret_cast<volatile uint64_t*>(&me->p2p_tx_msgs[peer]);
    s_msg = msg;
    s_err = msg >= uint64_t(kP2PLLSlots)
                ? wait_geq(&me->p2p_hdr_ack[peer], me, c.timeout_ns, msg + 1 - kP2PLLSlots)
                : MCRDL_OK;
  }
  __syncthreads();
  const uint64_t msg = s_msg;
  if (s_err) {
    if (threadIdx.x == 0) raise_error(const_cast<Pad* const*>(c.pad), c.world, c.err, s_err, 0);
  } else {
    uint8_t* slot = ll_box(c, peer_ws, c.rank) + int64_t(msg % kP2PLLSlots) * kP2PLLSlotBytes;
    const uint32_t tag = uint32_t(msg + 1);
    const int64_t nu = (bytes + 7) / 8;
    const int64_t u0 = nu * blockIdx.x / gridDim.x, u1 = nu * (blockIdx.x + 1) / gridDim.x;
    for (int64_t u = u0 + threadIdx.x; u < u1; u += blockDim.x) {
      const uint2 v = load8(buf, u, bytes);
      st_ll(slot + 16 + u * 16, v.x, v.y, tag);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0)
      st_ll(slot, uint32_t(bytes), uint32_t(uint64_t(bytes) >> 32), tag);
  }
  if (last_cta(c, 0)) {
    me->p2p_tx_msgs[peer] = msg + 1;
    oplog_end(c);
  }
}

__global__ void __launch_bounds__(kP2PThreads)
    k_recv_ll(DevComm c, Pad* peer_pad, uint8_t* my_ws, uint8_t* buf, int64_t bytes, int peer) {
  __shared__ uint64_t s_msg;
  __shared__ int s_err;
  Pad* me = c.self;
  oplog_start(c);
  const uint8_t* base = ll_box(c, my_ws, peer);
  if (threadIdx.x == 0) {
    const uint64_t msg = *reinterpret_cast<volatile uint64_t*>(&me->p2p_rx_msgs[peer]);
    s_msg = msg;
    int e = MCRDL_OK;
    if (blockIdx.x == 0) {  // CTA 0 matches the header; the others poll data lines
      bool via_ll = false;
      uint64_t sent = 0;
      e = p2p_wait_header(c, me, peer, base + int64_t(msg % kP2PLLSlots) * kP2PLLSlotBytes, msg,
                          &via_ll, &sent);
      if (e == MCRDL_OK && (!via_ll || sent != uint64_t(bytes))) e = MCRDL_ERR_LENGTH_MISMATCH;
      if (e) raise_error(const_cast<Pad* const*>(c.pad), c.world, c.err, e, 0);
    }
    s_err = e;
  }
  __syncthreads();
  const uint64_t msg = s_msg;
  const uint8_t* slot = base + int64_t(msg % kP2PLLSlots) * kP2PLLSlotBytes;
  const uint32_t tag = uint32_t(msg + 1);
  const int64_t nu = (bytes + 7) / 8;
  const int64_t u0 = nu * blockIdx.x / gridDim.x, u1 = nu * (blockIdx.x + 1) / gridDim.x;
  volatile int* verr = &s_err;
  for (int64_t u = u0 + threadIdx.x; u < u1 && !*verr; u += blockDim.x) {
    uint2 d;
    const uint4 v = ld_ll(slot + 16 + u * 16);
    if (ll_ready(v, tag)) {
      d = make_uint2(v.x, v.z);
    } else {
      int e = 0;
      if (!poll_ll(slot + 16 + u * 16, tag, me, c.timeout_ns, d, &e)) {
        atomicCAS(&s_err, 0, e);
        break;
      }
    }
    store8(buf, u, bytes, d);
  }
  __syncthreads();
  if (s_err && threadIdx.x == 0 && blockIdx.x != 0)
    raise_error(const_cast<Pad* const*>(c.pad), c.world, c.err, s_err, 0);
  if (last_cta(c, 1)) {
    publish(&peer_pad->p2p_hdr_ack[c.rank], msg + 1);  // slot consumed
    me->p2p_rx_msgs[peer] = msg + 1;
    oplog_end(c);
  }
}

// Last CTA of the launch advances the local stream counters. Sends and
// receives have their own exit counters (and order chains, begin_op): a recv
// may run concurrently with a send or a collective on another stream.
__device__ __forceinline__ bool last_cta(const DevComm& c, int dir) {
  __syncthreads();
  if (gridDim.x == 1) return threadIdx.x == 0;  // single CTA: no exit counter
  bool last = false;
  if (threadIdx.x == 0) {
    __threadfence();
    const uint32_t prev = atomicAdd(&c.self->p2p_done[dir], 1u);
    if (prev == gridDim.x - 1) {
      *reinterpret_cast<volatile uint32_t*>(&c.self->p2p_done[dir]) = 0u;
      last = true;
    }
  }
  return last;
}

__global__ void __launch_bounds__(kP2PThreads)
    k_send(DevComm c, Pad* peer_pad, uint8_t* peer_ws, const uint8_t* buf, int64_t bytes, int peer,
           int K, int64_t chunk) {
  __shared__ uint64_t s_base, s_msg;
  __shared__ int s_err;
  Pad* me = c.self;
  oplog_start(c);
  if (threadIdx.x == 0) {
    s_base = *reinterpret_cast<volatile uint64_t*>(&me->p2p_tx_chunks[peer]);
    s_msg = *reinterpret_cast<volatile uint64_t*>(&me->p2p_tx_msgs[peer]);
    s_err = 0;
  }
  __syncthreads();
  const uint64_t base = s_base, msg = s_msg;
  const int64_t nch = (bytes + chunk - 1) / chunk;  // chunk <= slot size
  const int rank = c.rank;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    // header slot msg % H is free once the receiver matched message msg - H
    int e = msg >= uint64_t(kP2PHdr)
                ? wait_geq(&me->p2p_hdr_ack[peer], me, c.timeout_ns, msg + 1 - kP2PHdr)
                : MCRDL_OK;
    if (e == MCRDL_OK) {
      uint64_t* h = peer_pad->p2p_hdr[rank][msg % kP2PHdr];
      st_relaxed_sys(&h[1], uint64_t(bytes));
      st_release_sys(&h[0], msg + 1);
    } else {
      s_err = e;
    }
  }
  if (blockIdx.x == 0) __syncthreads();  // every thread of the CTA sees s_err
  uint8_t* box = mailbox(c, peer_ws, rank);
  // (s_err is read only right after a barrier: all threads of a CTA agree)
  for (int64_t k = blockIdx.x; k < nch; k += gridDim.x) {
    const uint64_t g = base + uint64_t(k);
    const int slot = int(g % uint64_t(K));
    if (threadIdx.x == 0 && g >= uint64_t(K)) {
      int e = wait_geq(&me->p2p_free[peer][slot], me, c.timeout_ns, g + 1 - K);
      if (e) s_err = e;
    }
    __syncthreads();
    if (s_err) break;
    const int64_t off = k * chunk;
    block_copy<8>(box + int64_t(slot) * kP2PChunk, buf + off, min(chunk, bytes - off));
    __syncthreads();
    if (threadIdx.x == 0) publish(&peer_pad->p2p_full[rank][slot], g + 1);
  }
  __syncthreads();
  if (s_err && threadIdx.x == 0) raise_error(const_cast<Pad* const*>(c.pad), c.world, c.err, s_err, 0);
  if (last_cta(c, 0)) {
    me->p2p_tx_chunks[peer] = base + uint64_t(nch);
    me->p2p_tx_msgs[peer] = msg + 1;
    __threadfence();
    oplog_end(c);
  }
}

__global__ void __launch_bounds__(kP2PThreads)
    k_recv(DevComm c, Pad* peer_pad, const uint8_t* my_ws, uint8_t* buf, int64_t bytes, int peer,
           int K, int64_t chunk) {
  __shared__ uint64_t s_base, s_msg;
  __shared__ int s_err;
  Pad* me = c.self;
  oplog_start(c);
  if (threadIdx.x == 0) {
    s_base = *reinterpret_cast<volatile uint64_t*>(&me->p2p_rx_chunks[peer]);
    s_msg = *reinterpret_cast<volatile uint64_t*>(&me->p2p_rx_msgs[peer]);
    s_err = 0;
  }
  __syncthreads();
  const uint64_t base = s_base, msg = s_msg;
  const int64_t nch = (bytes + chunk - 1) / chunk;  // chunk <= slot size
  const int rank = c.rank;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    bool via_ll = false;
    uint64_t sent = 0;
    int e = p2p_wait_header(c, me, peer,
                            ll_box(c, const_cast<uint8_t*>(my_ws), peer) +
                                int64_t(msg % kP2PLLSlots) * kP2PLLSlotBytes,
                            msg, &via_ll, &sent);
    if (e == MCRDL_OK) {
      if (via_ll || sent != uint64_t(bytes)) e = MCRDL_ERR_LENGTH_MISMATCH;
      else publish(&peer_pad->p2p_hdr_ack[rank], msg + 1);
    }
    s_err = e;
  }
  // the header check must pass before any chunk is consumed: a short sender
  // would otherwise leave chunks of its next message in our slots
  if (blockIdx.x == 0) __syncthreads();
  const uint8_t* box = mailbox(c, const_cast<uint8_t*>(my_ws), peer);
  for (int64_t k = blockIdx.x; k < nch; k += gridDim.x) {
    const uint64_t g = base + uint64_t(k);
    const int slot = int(g % uint64_t(K));
    if (threadIdx.x == 0) {
      int e = wait_geq(&me->p2p_full[peer][slot], me, c.timeout_ns, g + 1);
      if (e) s_err = e;
    }
    __syncthreads();
    if (s_err) break;
    const int64_t off = k * chunk;
    block_copy<8>(buf + off, box + int64_t(slot) * kP2PChunk, min(chunk, bytes - off));
    __syncthreads();
    if (threadIdx.x == 0) publish(&peer_pad->p2p_free[rank][slot], g + 1);
  }
  __syncthreads();
  if (s_err && threadIdx.x == 0) raise_error(const_cast<Pad* const*>(c.pad), c.world, c.err, s_err, 0);
  if (last_cta(c, 1)) {
    me->p2p_rx_chunks[peer] = base + uint64_t(nch);
    me->p2p_rx_msgs[peer] = msg + 1;
    __threadfence();
    oplog_end(c);
  }
}

mcrdl_status_t p2p_launch(mcrdl_comm* c, void* buf, uint64_t bytes, int peer, bool is_send,
                          void* stream_) {
  if (c == nullptr) return set_error(MCRDL_ERR_NOT_INITIALIZED, "communicator is NULL");
  if (peer < 0 || peer >= c->world)
    return set_error(MCRDL_ERR_VALIDATION, "peer %d outside world %d", peer, c->world);
  if (bytes > 0 && buf == nullptr) return set_error(MCRDL_ERR_VALIDATION, "NULL buffer");
  if (c->dc.mbox_bytes < kP2PChunk)
    return set_error(MCRDL_ERR_UNSUPPORTED, "point-to-point mailboxes disabled (MCRDL_P2P_BYTES=0)");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  mcrdl_status_t st = begin_op(c, stream, is_send ? kChainSend : kChainRecv);
  if (st != MCRDL_OK) return st;
  const int K = int(c->dc.mbox_bytes / kP2PChunk);
  // Chunk = one 64 KiB slot. (Smaller chunks to spread medium messages over
  // more CTAs measured slower: 256 KiB ping-pong 43 vs 37 us with 4 KiB chunks;
  // the per-chunk flag round trips dominate.)
  const int64_t chunk = kP2PChunk;
  const int64_t nch = (int64_t(bytes) + chunk - 1) / chunk;
  // one CTA per chunk in flight, at most the ring depth and one per SM
  int G = int(std::min<int64_t>(std::max<int64_t>(nch, 1), std::min(K, c->num_sms)));
  if (G < 1) G = 1;
  Pad* peer_pad = c->dc.pad[peer];
  if (bytes <= uint64_t(kP2PLLMax)) {  // small: LL lines, 8 KiB of payload per CTA
    const int gl = int(std::min<uint64_t>(std::max<uint64_t>(1, (bytes + kP2PLLCtaBytes - 1) / kP2PLLCtaBytes),
                                          uint64_t(2 * c->num_sms)));
    if (is_send)
      k_send_ll<<<gl, kP2PThreads, 0, stream>>>(c->dc, c->dc.ws[peer],
                                                static_cast<const uint8_t*>(buf), int64_t(bytes),
                                                peer);
    else
      k_recv_ll<<<gl, kP2PThreads, 0, stream>>>(c->dc, peer_pad, c->dc.ws[c->rank],
                                                static_cast<uint8_t*>(buf), int64_t(bytes), peer);
    count_launch();
    MCRDL_CUDA_CHECK(cudaGetLastError());
    return MCRDL_OK;
  }
  if (is_send) {
    k_send<<<G, kP2PThreads, 0, stream>>>(c->dc, peer_pad, c->dc.ws[peer],
                                          static_cast<const uint8_t*>(buf), int64_t(bytes), peer, K,
                                          chunk);
  } else {
    k_recv<<<G, kP2PThreads, 0, stream>>>(c->dc, peer_pad, c->dc.ws[c->rank], static_cast<uint8_t*>(buf),
                                          int64_t(bytes), peer, K, chunk);
  }
  count_launch();
  MCRDL_CUDA_CHECK(cudaGetLastError());
  return MCRDL_OK;
}

}  // namespace

}  // namespace mcrdl

using namespace mcrdl;

extern "C" mcrdl_status_t mcrdl_send(mcrdl_comm* comm, const void* buf, uint64_t bytes, int peer,
                                     void* stream) {
  return p2p_launch(comm, const_cast<void*>(buf), bytes, peer, true, stream);
}

extern "C" mcrdl_status_t mcrdl_recv(mcrdl_comm* comm, void* buf, uint64_t bytes, int peer,
                                     void* stream) {
  return p2p_launch(comm, buf, bytes, peer, false, stream);
}
