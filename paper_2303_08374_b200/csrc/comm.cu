// Communicator lifecycle: symmetric VMM workspace, POSIX-fd handle exchange
// over an abstract unix socket, peer mapping over NVLink, status/error plumbing.
//
// Reference counterpart: Runtime.init -> _build_transport (runtime.py:336-383)
// and the TCP star bootstrap (transport.py:279-376). Here the host control
// plane (the caller's allgather callback) carries only a job id and a barrier;
// memory handles travel as file descriptors (SCM_RIGHTS) between the ranks'
// processes, and every byte of payload afterwards moves GPU->GPU over NVLink.
#include <cudaTypedefs.h>
#include <errno.h>
#include <poll.h>
#include <stdio.h>
#include <string.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <time.h>
#include <unistd.h>

#include <chrono>
#include <map>
#include <mutex>
#include <random>
#include <thread>

#include "internal.h"

namespace mcrdl {

// ------------------------------------------------------------ error state
static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};

mcrdl_status_t set_error(mcrdl_status_t code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// ------------------------------------------------------------ driver API
// Resolved through the runtime (cudaGetDriverEntryPoint) so this library has
// no link-time dependency on libcuda and loads on hosts without a driver.
struct Driver {
  PFN_cuMemCreate memCreate = nullptr;
  PFN_cuMemRelease memRelease = nullptr;
  PFN_cuMemMap memMap = nullptr;
  PFN_cuMemUnmap memUnmap = nullptr;
  PFN_cuMemSetAccess memSetAccess = nullptr;
  PFN_cuMemAddressReserve addrReserve = nullptr;
  PFN_cuMemAddressFree addrFree = nullptr;
  PFN_cuMemExportToShareableHandle exportHandle = nullptr;
  PFN_cuMemImportFromShareableHandle importHandle = nullptr;
  PFN_cuMemGetAllocationGranularity granularity = nullptr;
  PFN_cuMulticastCreate mcCreate = nullptr;
  PFN_cuMulticastAddDevice mcAddDevice = nullptr;
  PFN_cuMulticastBindMem mcBindMem = nullptr;
  PFN_cuMulticastUnbind mcUnbind = nullptr;
  PFN_cuMulticastGetGranularity mcGranularity = nullptr;
  PFN_cuDeviceGetAttribute devAttr = nullptr;
  PFN_cuGetErrorString errorString = nullptr;
  bool loaded = false;
};
static Driver g_drv;
static std::mutex g_drv_mu;

template <typename F>
static bool resolve(const char* name, F* out) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || fn == nullptr)
    return false;
  *out = reinterpret_cast<F>(fn);
  return true;
}

static mcrdl_status_t load_driver() {
  std::lock_guard<std::mutex> lk(g_drv_mu);
  if (g_drv.loaded) return MCRDL_OK;
  bool ok = resolve("cuMemCreate", &g_drv.memCreate) && resolve("cuMemRelease", &g_drv.memRelease) &&
            resolve("cuMemMap", &g_drv.memMap) && resolve("cuMemUnmap", &g_drv.memUnmap) &&
            resolve("cuMemSetAccess", &g_drv.memSetAccess) &&
            resolve("cuMemAddressReserve", &g_drv.addrReserve) &&
            resolve("cuMemAddressFree", &g_drv.addrFree) &&
            resolve("cuMemExportToShareableHandle", &g_drv.exportHandle) &&
            resolve("cuMemImportFromShareableHandle", &g_drv.importHandle) &&
            resolve("cuMemGetAllocationGranularity", &g_drv.granularity) &&
            resolve("cuGetErrorString", &g_drv.errorString);
  if (!ok) return set_error(MCRDL_ERR_CUDA, "cannot resolve CUDA driver VMM entry points (no driver?)");
  // Multicast is optional (NVLS).
  resolve("cuMulticastCreate", &g_drv.mcCreate);
  resolve("cuMulticastAddDevice", &g_drv.mcAddDevice);
  resolve("cuMulticastBindMem", &g_drv.mcBindMem);
  resolve("cuMulticastUnbind", &g_drv.mcUnbind);
  resolve("cuMulticastGetGranularity", &g_drv.mcGranularity);
  resolve("cuDeviceGetAttribute", &g_drv.devAttr);
  g_drv.loaded = true;
  return MCRDL_OK;
}

static const char* cu_str(CUresult r) {
  const char* s = nullptr;
  if (g_drv.errorString) g_drv.errorString(r, &s);
  return s ? s : "unknown CUDA driver error";
}

#define CU_CHECK(expr)                                                                  \
  do {                                                                                  \
    CUresult r_ = (expr);                                                               \
    if (r_ != CUDA_SUCCESS)                                                             \
      return set_error(MCRDL_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, cu_str(r_),     \
                       __FILE__, __LINE__);                                             \
  } while (0)

// ------------------------------------------------------------ bootstrap
// Setup memsets (pads, symmetric allocations, NVLS flag words) run on the
// legacy default stream and are waited for on it alone: it does not wait for
// non-blocking streams, so a co-located peer rank's spinning kernel never
// stalls a setup, and no stream is created per communicator.
static const cudaStream_t kSetupStream = nullptr;

static mcrdl_status_t host_allgather(mcrdl_comm* c, const void* send, void* recv, size_t n) {
  if (c->world == 1) {
    memcpy(recv, send, n);
    return MCRDL_OK;
  }
  if (c->allgather(c->ag_ctx, send, recv, n) != 0)
    return set_error(MCRDL_ERR_BOOTSTRAP, "bootstrap allgather callback failed");
  return MCRDL_OK;
}

static mcrdl_status_t host_barrier(mcrdl_comm* c) {
  int x = c->rank, all[kMaxRanks];
  return host_allgather(c, &x, all, sizeof(int));
}

// --------------------------------------------- fd passing (unix sockets)
struct FdMsg {
  uint32_t magic;
  int32_t rank;
  int32_t tag;
  int32_t pad;
};
static constexpr uint32_t kFdMagic = 0x4D434644u;  // "MCFD"

static socklen_t sock_name(sockaddr_un* a, uint64_t jobid, int rank) {
  memset(a, 0, sizeof(*a));
  a->sun_family = AF_UNIX;
  // Abstract namespace: leading NUL, no filesystem entry.
  int n = snprintf(a->sun_path + 1, sizeof(a->sun_path) - 1, "mcrdl-nvl-%016llx-%d",
                   (unsigned long long)jobid, rank);
  return socklen_t(offsetof(sockaddr_un, sun_path) + 1 + n);
}

// Messages that arrived early for a later exchange tag live in the comm
// (c->fd_stash: (tag, rank) -> fd) and tags count per comm (c->fd_tag): several
// communicators of one process (ranks sharing a GPU as threads, or several
// backends) must not consume each other's tags.

static mcrdl_status_t send_fd(uint64_t jobid, int to, int from, int tag, int fd, double timeout_s) {
  sockaddr_un addr;
  socklen_t len = sock_name(&addr, jobid, to);
  auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    int s = socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
    if (s < 0) return set_error(MCRDL_ERR_BOOTSTRAP, "socket(): %s", strerror(errno));
    if (connect(s, reinterpret_cast<sockaddr*>(&addr), len) == 0) {
      FdMsg m{kFdMagic, from, tag, 0};
      iovec iov{&m, sizeof(m)};
      char cbuf[CMSG_SPACE(sizeof(int))];
      memset(cbuf, 0, sizeof(cbuf));
      msghdr msg{};
      msg.msg_iov = &iov;
      msg.msg_iovlen = 1;
      msg.msg_control = cbuf;
      msg.msg_controllen = sizeof(cbuf);
      cmsghdr* cm = CMSG_FIRSTHDR(&msg);
      cm->cmsg_level = SOL_SOCKET;
      cm->cmsg_type = SCM_RIGHTS;
      cm->cmsg_len = CMSG_LEN(sizeof(int));
      memcpy(CMSG_DATA(cm), &fd, sizeof(int));
      ssize_t w = sendmsg(s, &msg, 0);
      close(s);
      if (w != ssize_t(sizeof(m)))
        return set_error(MCRDL_ERR_PEER_DISCONNECTED, "sendmsg to rank %d: %s", to, strerror(errno));
      return MCRDL_OK;
    }
    close(s);
    double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (el > timeout_s)
      return set_error(MCRDL_ERR_BOOTSTRAP, "connect to rank %d socket timed out: %s", to,
                       strerror(errno));
    std::this_thread::sleep_for(std::chrono::milliseconds(2));
  }
}

static mcrdl_status_t recv_one_fd(int listen_fd, double timeout_s, FdMsg* m, int* fd) {
  pollfd p{listen_fd, POLLIN, 0};
  int pr = poll(&p, 1, int(timeout_s * 1000));
  if (pr <= 0) return set_error(MCRDL_ERR_BOOTSTRAP, "timed out waiting for a peer fd");
  int s = accept4(listen_fd, nullptr, nullptr, SOCK_CLOEXEC);
  if (s < 0) return set_error(MCRDL_ERR_BOOTSTRAP, "accept(): %s", strerror(errno));
  iovec iov{m, sizeof(*m)};
  char cbuf[CMSG_SPACE(sizeof(int))];
  msghdr msg{};
  msg.msg_iov = &iov;
  msg.msg_iovlen = 1;
  msg.msg_control = cbuf;
  msg.msg_controllen = sizeof(cbuf);
  ssize_t r = recvmsg(s, &msg, MSG_WAITALL);
  close(s);
  cmsghdr* cm = CMSG_FIRSTHDR(&msg);
  if (r != ssize_t(sizeof(*m)) || m->magic != kFdMagic || cm == nullptr ||
      cm->cmsg_type != SCM_RIGHTS)
    return set_error(MCRDL_ERR_PEER_DISCONNECTED, "malformed fd message from a peer");
  memcpy(fd, CMSG_DATA(cm), sizeof(int));
  return MCRDL_OK;
}

// Every rank sends `my_fd` to every peer and collects one fd per peer.
static mcrdl_status_t exchange_fds(mcrdl_comm* c, int my_fd, int peer_fds[kMaxRanks]) {
  const int tag = ++c->fd_tag;
  const double tmo = double(c->timeout_ns) * 1e-9 + 30.0;
  for (int r = 0; r < c->world; ++r) peer_fds[r] = -1;
  peer_fds[c->rank] = my_fd;
  for (int k = 1; k < c->world; ++k) {
    int to = (c->rank + k) % c->world;
    mcrdl_status_t st = send_fd(c->jobid, to, c->rank, tag, my_fd, tmo);
    if (st != MCRDL_OK) return st;
  }
  int have = 0;
  for (int r = 0; r < c->world; ++r) {
    auto it = c->fd_stash.find({tag, r});
    if (it != c->fd_stash.end()) {
      peer_fds[r] = it->second;
      c->fd_stash.erase(it);
      ++have;
    }
  }
  while (have < c->world - 1) {
    FdMsg m;
    int fd = -1;
    mcrdl_status_t st = recv_one_fd(c->listen_fd, tmo, &m, &fd);
    if (st != MCRDL_OK) return st;
    if (m.tag == tag && m.rank >= 0 && m.rank < c->world && peer_fds[m.rank] < 0) {
      peer_fds[m.rank] = fd;
      ++have;
    } else {
      c->fd_stash[{m.tag, m.rank}] = fd;
    }
  }
  return MCRDL_OK;
}

// ------------------------------------------------------------ regions
static CUmemAllocationProp alloc_prop(int dev) {
  CUmemAllocationProp prop{};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = dev;
  prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  return prop;
}

static mcrdl_status_t map_handle(mcrdl_comm* c, CUmemGenericAllocationHandle h, uint64_t bytes,
                                 CUdeviceptr* out) {
  CUdeviceptr va = 0;
  CU_CHECK(g_drv.addrReserve(&va, bytes, c->gran, 0, 0));
  CU_CHECK(g_drv.memMap(va, bytes, 0, h, 0));
  CUmemAccessDesc d{};
  d.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  d.location.id = c->device;
  d.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CU_CHECK(g_drv.memSetAccess(va, bytes, &d, 1));
  *out = va;
  return MCRDL_OK;
}

static void unmap_region(mcrdl_comm* c, Region& rg) {
  if (rg.mc_ptr) {
    g_drv.memUnmap(rg.mc_ptr, rg.bytes);
    g_drv.addrFree(rg.mc_ptr, rg.bytes);
    rg.mc_ptr = 0;
  }
  if (rg.mc_bound && g_drv.mcUnbind) g_drv.mcUnbind(rg.mc_handle, c->device, 0, rg.bytes);
  rg.mc_bound = false;
  if (rg.mc_handle) {
    g_drv.memRelease(rg.mc_handle);
    rg.mc_handle = 0;
  }
  for (int r = 0; r < c->world; ++r) {
    if (rg.ptr[r]) {
      g_drv.memUnmap(rg.ptr[r], rg.bytes);
      g_drv.addrFree(rg.ptr[r], rg.bytes);
      rg.ptr[r] = 0;
    }
    if (rg.handles[r]) {
      g_drv.memRelease(rg.handles[r]);
      rg.handles[r] = 0;
    }
  }
  rg.local_handle = 0;
}

// Collective: allocate `bytes` on this GPU, export it, import every peer's
// allocation and map all of them here.
static mcrdl_status_t alloc_region(mcrdl_comm* c, uint64_t bytes, Region* rg) {
  bytes = (bytes + c->gran - 1) / c->gran * c->gran;
  rg->bytes = bytes;
  CUmemAllocationProp prop = alloc_prop(c->device);
  CUmemGenericAllocationHandle h = 0;
  CU_CHECK(g_drv.memCreate(&h, bytes, &prop, 0));
  rg->local_handle = h;
  rg->handles[c->rank] = h;
  int my_fd = -1;
  CU_CHECK(g_drv.exportHandle(&my_fd, h, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
  int fds[kMaxRanks];
  mcrdl_status_t st = exchange_fds(c, my_fd, fds);
  if (st != MCRDL_OK) {
    close(my_fd);
    return st;
  }
  for (int r = 0; r < c->world; ++r) {
    if (r == c->rank) continue;
    CUresult res = g_drv.importHandle(&rg->handles[r], reinterpret_cast<void*>(uintptr_t(fds[r])),
                                      CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
    close(fds[r]);
    if (res != CUDA_SUCCESS)
      return set_error(MCRDL_ERR_CUDA, "cuMemImportFromShareableHandle(rank %d): %s", r, cu_str(res));
  }
  close(my_fd);
  for (int r = 0; r < c->world; ++r) {
    st = map_handle(c, rg->handles[r], bytes, &rg->ptr[r]);
    if (st != MCRDL_OK) return st;
  }
  return MCRDL_OK;
}

// Rank 0 hands one fd to every peer (the multicast object handle).
static mcrdl_status_t bcast_fd(mcrdl_comm* c, int fd, int* out_fd) {
  const int tag = ++c->fd_tag;
  const double tmo = double(c->timeout_ns) * 1e-9 + 30.0;
  if (c->rank == 0) {
    for (int r = 1; r < c->world; ++r) {
      mcrdl_status_t st = send_fd(c->jobid, r, 0, tag, fd, tmo);
      if (st != MCRDL_OK) return st;
    }
    *out_fd = fd;
    return MCRDL_OK;
  }
  {
    auto it = c->fd_stash.find({tag, 0});
    if (it != c->fd_stash.end()) {
      *out_fd = it->second;
      c->fd_stash.erase(it);
      return MCRDL_OK;
    }
  }
  for (;;) {
    FdMsg m;
    int got = -1;
    mcrdl_status_t st = recv_one_fd(c->listen_fd, tmo, &m, &got);
    if (st != MCRDL_OK) return st;
    if (m.tag == tag && m.rank == 0) {
      *out_fd = got;
      return MCRDL_OK;
    }
    c->fd_stash[{m.tag, m.rank}] = got;
  }
}

// Collective: build the NVLS multicast buffer. Every rank reports whether
// its part succeeded and NVLS is enabled only if all did (so ranks never
// disagree on the algorithm). Failure is not an error: the communicator
// simply has no NVLS (caps.nvls_supported = 0).
// Collective: bind every rank's physical copy of `rg` to one new multicast
// object and map its multicast view (rg->mc_ptr). Failure to create or bind
// is not an error: the region then stays P2P-only (mc_ptr == 0), agreed by
// all ranks.
static mcrdl_status_t bind_multicast(mcrdl_comm* c, Region* rg) {
  CUmulticastObjectProp mp{};
  mp.numDevices = unsigned(c->world);
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  mp.size = rg->bytes;
  int ok = 1, oks[kMaxRanks];
  int fd = -1, rfd = -1;
  mcrdl_status_t st;
  if (c->rank == 0 &&
      (g_drv.mcCreate(&rg->mc_handle, &mp) != CUDA_SUCCESS ||
       g_drv.exportHandle(&fd, rg->mc_handle, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0) !=
           CUDA_SUCCESS))
    ok = 0;
  if ((st = host_allgather(c, &ok, oks, sizeof(int))) != MCRDL_OK) return st;
  if (!oks[0]) return MCRDL_OK;
  if ((st = bcast_fd(c, fd, &rfd)) != MCRDL_OK) return st;
  if (c->rank != 0) {
    if (g_drv.importHandle(&rg->mc_handle, reinterpret_cast<void*>(uintptr_t(rfd)),
                           CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR) != CUDA_SUCCESS)
      ok = 0;
    close(rfd);
  } else {
    close(fd);
  }
  if (ok && g_drv.mcAddDevice(rg->mc_handle, c->device) != CUDA_SUCCESS) ok = 0;
  if ((st = host_allgather(c, &ok, oks, sizeof(int))) != MCRDL_OK) return st;
  for (int r = 0; r < c->world; ++r) ok &= oks[r];
  if (ok && g_drv.mcBindMem(rg->mc_handle, 0, rg->local_handle, 0, rg->bytes, 0) != CUDA_SUCCESS)
    ok = 0;
  rg->mc_bound = ok != 0;
  if (ok && map_handle(c, rg->mc_handle, rg->bytes, &rg->mc_ptr) != MCRDL_OK) ok = 0;
  if ((st = host_allgather(c, &ok, oks, sizeof(int))) != MCRDL_OK) return st;
  for (int r = 0; r < c->world; ++r) ok &= oks[r];
  if (!ok && rg->mc_ptr) {  // some rank failed: every rank drops the view
    g_drv.memUnmap(rg->mc_ptr, rg->bytes);
    g_drv.addrFree(rg->mc_ptr, rg->bytes);
    rg->mc_ptr = 0;
  }
  return MCRDL_OK;
}

const Region* find_symm(const mcrdl_comm* c, const void* p, uint64_t bytes, uint64_t* off) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  for (const Region& rg : c->symm) {
    const uintptr_t base = uintptr_t(rg.ptr[c->rank]);
    if (a >= base && a + bytes <= base + rg.bytes) {
      *off = a - base;
      return &rg;
    }
  }
  return nullptr;
}

static mcrdl_status_t setup_nvls(mcrdl_comm* c, uint64_t bytes) {
  Nvls& nv = c->nvls;
  int ok = 1;
  int attr = 0;
  if (c->world < 2 || !g_drv.mcCreate || !g_drv.mcAddDevice || !g_drv.mcBindMem ||
      !g_drv.mcGranularity || !g_drv.devAttr)
    ok = 0;
  if (ok && (g_drv.devAttr(&attr, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, c->device) != CUDA_SUCCESS ||
             attr == 0))
    ok = 0;
  CUmulticastObjectProp mp{};
  size_t mg = 0;
  if (ok) {
    mp.numDevices = unsigned(c->world);
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    mp.size = bytes;
    if (g_drv.mcGranularity(&mg, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS) ok = 0;
  }
  // Agree on attempting it at all.
  int oks[kMaxRanks];
  mcrdl_status_t st = host_allgather(c, &ok, oks, sizeof(int));
  if (st != MCRDL_OK) return st;
  for (int r = 0; r < c->world; ++r) ok &= oks[r];
  if (!ok) return MCRDL_OK;
  size_t gran = std::max<size_t>(mg, c->gran);
  bytes = (bytes + 2 * gran - 1) / (2 * gran) * (2 * gran);
  mp.size = bytes;
  nv.bytes = bytes;
  int fd = -1, rfd = -1;
  if (c->rank == 0) {
    if (g_drv.mcCreate(&nv.mc_handle, &mp) != CUDA_SUCCESS ||
        g_drv.exportHandle(&fd, nv.mc_handle, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0) !=
            CUDA_SUCCESS)
      ok = 0;
  }
  if ((st = host_allgather(c, &ok, oks, sizeof(int))) != MCRDL_OK) return st;
  if (!oks[0]) return MCRDL_OK;
  if ((st = bcast_fd(c, fd, &rfd)) != MCRDL_OK) return st;
  if (c->rank != 0) {
    if (g_drv.importHandle(&nv.mc_handle, reinterpret_cast<void*>(uintptr_t(rfd)),
                           CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR) != CUDA_SUCCESS)
      ok = 0;
    close(rfd);
  } else {
    close(fd);
  }
  if (ok && g_drv.mcAddDevice(nv.mc_handle, c->device) != CUDA_SUCCESS) ok = 0;
  // Every device must join before any rank binds memory.
  if ((st = host_allgather(c, &ok, oks, sizeof(int))) != MCRDL_OK) return st;
  for (int r = 0; r < c->world; ++r) ok &= oks[r];
  if (ok) {
    CUmemAllocationProp prop = alloc_prop(c->device);
    if (g_drv.memCreate(&nv.mem_handle, bytes, &prop, 0) != CUDA_SUCCESS) ok = 0;
    if (ok && g_drv.mcBindMem(nv.mc_handle, 0, nv.mem_handle, 0, bytes, 0) != CUDA_SUCCESS) ok = 0;
    nv.bound = ok;
    if (ok && map_handle(c, nv.mc_handle, bytes, &nv.mc_ptr) != MCRDL_OK) ok = 0;
    if (ok && map_handle(c, nv.mem_handle, bytes, &nv.uc_ptr) != MCRDL_OK) ok = 0;
  }
  if (ok) {  // multicast flag words at the end of each half start at 0
    for (int h = 0; h < 2; ++h)
      if (cudaMemsetAsync(reinterpret_cast<uint8_t*>(nv.uc_ptr) + (h + 1) * (bytes / 2) -
                              kNvlsFlagBytes,
                          0, kNvlsFlagBytes, kSetupStream) != cudaSuccess)
        ok = 0;
    if (cudaStreamSynchronize(kSetupStream) != cudaSuccess) ok = 0;
  }
  if ((st = host_allgather(c, &ok, oks, sizeof(int))) != MCRDL_OK) return st;
  for (int r = 0; r < c->world; ++r) ok &= oks[r];
  nv.ok = ok != 0;
  return MCRDL_OK;
}

static void teardown_nvls(mcrdl_comm* c) {
  Nvls& nv = c->nvls;
  if (nv.mc_ptr) {
    g_drv.memUnmap(nv.mc_ptr, nv.bytes);
    g_drv.addrFree(nv.mc_ptr, nv.bytes);
  }
  if (nv.uc_ptr) {
    g_drv.memUnmap(nv.uc_ptr, nv.bytes);
    g_drv.addrFree(nv.uc_ptr, nv.bytes);
  }
  if (nv.bound && g_drv.mcUnbind) g_drv.mcUnbind(nv.mc_handle, c->device, 0, nv.bytes);
  if (nv.mem_handle) g_drv.memRelease(nv.mem_handle);
  if (nv.mc_handle) g_drv.memRelease(nv.mc_handle);
  nv = Nvls{};
}

mcrdl_status_t begin_op(mcrdl_comm* comm, cudaStream_t stream, int chain) {
  if (comm == nullptr) return set_error(MCRDL_ERR_NOT_INITIALIZED, "communicator is NULL");
  if (comm->sticky != MCRDL_OK)
    return set_error(comm->sticky, "communicator poisoned by an earlier device error (%s)",
                     mcrdl_status_kind(comm->sticky));
  if (comm->err_host && *reinterpret_cast<volatile int*>(comm->err_host) != 0) {
    comm->sticky = *comm->err_host;
    return set_error(comm->sticky, "communicator poisoned by an earlier device error (%s)",
                     mcrdl_status_kind(comm->sticky));
  }
  // Log id of the launch that follows (0 inside a CUDA-graph capture: replays
  // must not stamp stale ids into the ring).
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  MCRDL_CUDA_CHECK(cudaStreamIsCapturing(stream, &cap));
  static const int64_t log_on = env_int("MCRDL_LOG", 1);
  comm->dc.log_id = (log_on && cap == cudaStreamCaptureStatusNone) ? ++comm->log_seq : 0;
  auto& ch = comm->chain[chain];
  if (ch.have && ch.last != stream) {
    // A stream being captured into a CUDA graph cannot wait on work outside
    // the capture; capture starts from a synchronized device
    // (torch.cuda.graph does this), and replays are ordered by the caller
    // like any other op of the communicator.
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    MCRDL_CUDA_CHECK(cudaStreamIsCapturing(stream, &cs));
    if (cs == cudaStreamCaptureStatusNone) {
      MCRDL_CUDA_CHECK(cudaEventRecord(ch.ev, ch.last));
      MCRDL_CUDA_CHECK(cudaStreamWaitEvent(stream, ch.ev, 0));
    }
  }
  ch.last = stream;
  ch.have = true;
  return MCRDL_OK;
}

}  // namespace mcrdl

using namespace mcrdl;

extern "C" {

const char* mcrdl_last_error(void) { return g_last_error.c_str(); }

int mcrdl_abi_version(void) { return MCRDL_NVL_ABI_VERSION; }

uint64_t mcrdl_launch_count(void) { return g_launches.load(); }

const char* mcrdl_status_kind(mcrdl_status_t s) {
  switch (s) {
    case MCRDL_OK: return "ok";
    case MCRDL_ERR_VALIDATION: return "validation";
    case MCRDL_ERR_ORDER_MISMATCH: return "order_mismatch";
    case MCRDL_ERR_TIMEOUT: return "timeout";
    case MCRDL_ERR_UNSUPPORTED: return "unsupported_operation";
    case MCRDL_ERR_PEER_DISCONNECTED: return "peer_disconnected";
    case MCRDL_ERR_CUDA: return "comm_error";
    case MCRDL_ERR_BOOTSTRAP: return "bootstrap_timeout";
    case MCRDL_ERR_LENGTH_MISMATCH: return "length_mismatch";
    case MCRDL_ERR_NOT_INITIALIZED: return "not_initialized";
    case MCRDL_ERR_CODEC_MISMATCH: return "codec_mismatch";
    default: return "comm_error";
  }
}

mcrdl_status_t mcrdl_comm_init(mcrdl_comm** out, int rank, int world, int cuda_device,
                               mcrdl_allgather_fn allgather, void* ctx, uint64_t workspace_bytes,
                               double timeout_secs) {
  if (out == nullptr) return set_error(MCRDL_ERR_VALIDATION, "comm out-pointer is NULL");
  *out = nullptr;
  if (world < 1 || world > kMaxRanks)
    return set_error(MCRDL_ERR_VALIDATION, "world size %d outside [1, %d]", world, kMaxRanks);
  if (rank < 0 || rank >= world)
    return set_error(MCRDL_ERR_VALIDATION, "rank %d outside world %d", rank, world);
  if (world > 1 && allgather == nullptr)
    return set_error(MCRDL_ERR_VALIDATION, "world > 1 needs a bootstrap allgather callback");
  mcrdl_status_t st = load_driver();
  if (st != MCRDL_OK) return st;
  MCRDL_CUDA_CHECK(cudaSetDevice(cuda_device));
  MCRDL_CUDA_CHECK(cudaFree(nullptr));  // make the primary context current

  auto* c = new mcrdl_comm();
  c->rank = rank;
  c->world = world;
  c->device = cuda_device;
  c->allgather = allgather;
  c->ag_ctx = ctx;
  if (timeout_secs > 0) c->timeout_ns = uint64_t(timeout_secs * 1e9);
  int dev_sms = 0;
  cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, cuda_device);
  auto fail = [&](mcrdl_status_t s) {
    mcrdl_comm_destroy(c);
    return s;
  };

  // Job id from rank 0 (fresh random per init) names the sockets; the device
  // UUIDs tell which ranks share a GPU.
  struct Hello {
    uint64_t id;
    unsigned char uuid[16];
    int32_t sms;
    int32_t pad;
  } mine{}, all[kMaxRanks];
  std::random_device rd;
  mine.id = (uint64_t(rd()) << 32) ^ rd() ^ uint64_t(getpid());
  {
    cudaDeviceProp prop;
    MCRDL_CUDA_CHECK(cudaGetDeviceProperties(&prop, cuda_device));
    memcpy(mine.uuid, prop.uuid.bytes, 16);
  }
  // MCRDL_MAX_SMS: SM budget for this rank's collectives (the rest stays free
  // for overlapped compute); co-located ranks split the device between them.
  mine.sms = dev_sms;
  if (const int64_t cap = env_int("MCRDL_MAX_SMS", 0); cap > 0 && cap < mine.sms) mine.sms = int32_t(cap);
  if ((st = host_allgather(c, &mine, all, sizeof(Hello))) != MCRDL_OK) return fail(st);
  c->jobid = all[0].id;
  int budget = mine.sms;
  for (int q = 0; q < world; ++q) {
    int same = 0;
    for (int k = 0; k < world; ++k) same += memcmp(all[q].uuid, all[k].uuid, 16) == 0;
    c->ranks_per_device = std::max(c->ranks_per_device, same);
    budget = std::min<int>(budget, all[q].sms);
  }
  // Co-located ranks: every rank's grids must be resident at once, or a
  // spinning grid would wait for a peer grid that cannot be scheduled. Grids
  // are sized at up to 2 CTAs (512 threads, <= 64 regs) per budgeted SM, up
  // to two chains (send + recv, or a collective and a recv) are in flight per
  // rank, and transient kernels of the host framework share the SMs: a
  // quarter of the device per rank-share (measured: p = 4 send/recv rings
  // stall with 18 SMs per rank, pass with 8).
  if (c->ranks_per_device > 1) budget = std::min(budget, dev_sms / (4 * c->ranks_per_device));
  c->num_sms = std::max(1, budget);
  if (c->ranks_per_device > 1) {
    // Lazy kernel loading waits for the context to idle: a co-located rank's
    // first launch of a kernel would wait on a peer kernel spinning for it.
    PFN_cuModuleGetLoadingMode getmode = nullptr;
    CUmoduleLoadingMode mode = CU_MODULE_EAGER_LOADING;
    if (resolve("cuModuleGetLoadingMode", &getmode) && getmode(&mode) == CUDA_SUCCESS &&
        mode != CU_MODULE_EAGER_LOADING && rank == 0)
      fprintf(stderr, "[mcrdl] warning: %d ranks share a GPU under lazy module loading; set "
                      "CUDA_MODULE_LOADING=EAGER or first launches can stall until the timeout\n",
              c->ranks_per_device);
  }

  if (world > 1) {
    c->listen_fd = socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
    sockaddr_un addr;
    socklen_t len = sock_name(&addr, c->jobid, rank);
    if (c->listen_fd < 0 || bind(c->listen_fd, reinterpret_cast<sockaddr*>(&addr), len) != 0 ||
        listen(c->listen_fd, 128) != 0)
      return fail(set_error(MCRDL_ERR_BOOTSTRAP, "unix socket setup failed: %s", strerror(errno)));
  }
  if ((st = host_barrier(c)) != MCRDL_OK) return fail(st);

  CUmemAllocationProp prop = alloc_prop(cuda_device);
  size_t g = 0;
  CUresult r = g_drv.granularity(&g, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
  if (r != CUDA_SUCCESS)
    return fail(set_error(MCRDL_ERR_CUDA, "cuMemGetAllocationGranularity: %s", cu_str(r)));
  c->gran = g < (2u << 20) ? (2u << 20) : g;

  if (workspace_bytes == 0) workspace_bytes = uint64_t(1) << 30;
  workspace_bytes = (workspace_bytes + 2 * c->gran - 1) / (2 * c->gran) * (2 * c->gran);
  c->ws_bytes = workspace_bytes;
  // Point-to-point mailboxes after the workspace: one ring per sender
  // (MCRDL_P2P_BYTES per sender, multiple of 64 KiB, <= 32 MiB; 0 disables).
  int64_t mbox = int64_t(env_int("MCRDL_P2P_BYTES", int64_t(kP2PSlots) * kP2PChunk));
  mbox = std::min<int64_t>(mbox, int64_t(kP2PSlots) * kP2PChunk) / kP2PChunk * kP2PChunk;
  if (mbox < 0) mbox = 0;
  const uint64_t p2p_bytes =
      (uint64_t(mbox) + (mbox > 0 ? uint64_t(kP2PLLSenderBytes) : 0)) * uint64_t(world);
  if ((st = alloc_region(c, kPadBytes + workspace_bytes + p2p_bytes, &c->base)) != MCRDL_OK)
    return fail(st);
  // Setup memsets run on the comm's private stream and are waited for on
  // that stream only: a device-wide sync could wait on spinning kernels of
  // co-located ranks whose peers have not launched yet.
  MCRDL_CUDA_CHECK(cudaMemsetAsync(reinterpret_cast<void*>(c->base.ptr[rank]), 0, kPadBytes, kSetupStream));
  MCRDL_CUDA_CHECK(cudaStreamSynchronize(kSetupStream));

  // NVLS buffer: twice the workspace by default (2 GiB halves for the default
  // 2 GiB workspace), so a 1 GiB all_reduce is ONE k_ar_nvls launch: measured
  // p = 4, 1 GiB 592 -> 667 GB/s f32 (665 bf16) against two 512 MiB launches
  // (profiles/r2_nvls_buffer_p4.log). MCRDL_NVLS_BYTES overrides, 0 disables.
  uint64_t nvls_bytes = 2 * workspace_bytes;
  if (const char* e = getenv("MCRDL_NVLS_BYTES")) nvls_bytes = strtoull(e, nullptr, 10);
  // A multicast object spans distinct GPUs: none for co-located ranks (agreed:
  // every rank computed ranks_per_device from the same UUID table).
  if (c->ranks_per_device > 1) nvls_bytes = 0;
  if (nvls_bytes > 0 && (st = setup_nvls(c, nvls_bytes)) != MCRDL_OK) return fail(st);

  MCRDL_CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&c->err_host), sizeof(int),
                                 cudaHostAllocMapped | cudaHostAllocPortable));
  *c->err_host = 0;
  MCRDL_CUDA_CHECK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->err_dev), c->err_host, 0));
  for (auto& ch : c->chain) MCRDL_CUDA_CHECK(cudaEventCreateWithFlags(&ch.ev, cudaEventDisableTiming));
  {
    const size_t lb = size_t(kOpLogSlots) * 2 * sizeof(uint64_t);
    MCRDL_CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&c->oplog_host), lb, cudaHostAllocMapped));
    memset(c->oplog_host, 0, lb);
    MCRDL_CUDA_CHECK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->dc.oplog), c->oplog_host, 0));
  }
#ifdef MCRDL_TRACE
  {
    const size_t tb = size_t(kMaxBlocks) * kTraceSlots * sizeof(uint64_t);
    MCRDL_CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&c->trace_host), tb, cudaHostAllocMapped));
    memset(c->trace_host, 0, tb);
    MCRDL_CUDA_CHECK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->dc.trace), c->trace_host, 0));
  }
#endif

  c->dc.rank = rank;
  c->dc.world = world;
  c->dc.err = c->err_dev;
  c->dc.timeout_ns = c->timeout_ns;
  c->dc.half_bytes = int64_t(workspace_bytes / 2);
  c->dc.mbox_bytes = mbox;
  c->dc.self = reinterpret_cast<Pad*>(c->base.ptr[rank]);
  for (int q = 0; q < world; ++q) {
    c->dc.pad[q] = reinterpret_cast<Pad*>(c->base.ptr[q]);
    c->dc.ws[q] = reinterpret_cast<uint8_t*>(c->base.ptr[q]) + kPadBytes;
  }
  // Nobody may signal into a pad before its owner zeroed it.
  if ((st = host_barrier(c)) != MCRDL_OK) return fail(st);
  if (env_int("MCRDL_DEBUG", 0))
    fprintf(stderr, "[mcrdl] comm %p rank %d/%d dev %d sms %d co-located %d pad %p nvls %d\n",
            (void*)c, rank, world, cuda_device, c->num_sms, c->ranks_per_device,
            (void*)c->base.ptr[rank], int(c->nvls.ok));
  *out = c;
  return MCRDL_OK;
}

mcrdl_status_t mcrdl_comm_destroy(mcrdl_comm* c) {
  if (c == nullptr) return MCRDL_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (auto& rg : c->symm) unmap_region(c, rg);
  c->symm.clear();
  unmap_region(c, c->base);
  teardown_nvls(c);
  if (c->err_host) cudaFreeHost(c->err_host);
  for (auto& ch : c->chain)
    if (ch.ev) cudaEventDestroy(ch.ev);
  if (c->trace_host) cudaFreeHost(c->trace_host);
  if (c->oplog_host) cudaFreeHost(c->oplog_host);
  // The comm's streams are NOT destroyed: host frameworks keep stream-ordered
  // references (e.g. torch's caching allocator records events on a lane
  // stream when a tensor used there is freed, possibly after finalize). A
  // handful of streams per communicator live until process exit.
  for (auto& kv : c->fd_stash) close(kv.second);
  if (c->listen_fd >= 0) close(c->listen_fd);
  delete c;
  return MCRDL_OK;
}

mcrdl_status_t mcrdl_debug_trace(mcrdl_comm* c, uint64_t** host_ptr, uint64_t* slots_per_cta) {
  if (c == nullptr || host_ptr == nullptr) return set_error(MCRDL_ERR_VALIDATION, "NULL argument");
  *host_ptr = c->trace_host;  // NULL unless built with --trace
  if (slots_per_cta) *slots_per_cta = kTraceSlots;
  return MCRDL_OK;
}

uint64_t mcrdl_comm_log_id(const mcrdl_comm* c) { return c ? c->log_seq : 0; }

}  // extern "C"

namespace mcrdl {
__global__ void k_oplog_flush(const Pad* pad, uint64_t* host) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < kOpLogSlots * 2; i += gridDim.x * blockDim.x)
    host[i] = reinterpret_cast<const volatile uint64_t*>(pad->oplog)[i];
}
}  // namespace mcrdl

extern "C" {

mcrdl_status_t mcrdl_comm_log_flush(mcrdl_comm* c) {
  if (c == nullptr) return set_error(MCRDL_ERR_NOT_INITIALIZED, "communicator is NULL");
  if (c->oplog_host == nullptr || c->log_seq == 0) return MCRDL_OK;
  void* s = nullptr;
  mcrdl_status_t st = mcrdl_comm_stream(c, 0, &s);
  if (st != MCRDL_OK) return st;
  k_oplog_flush<<<16, 512, 0, reinterpret_cast<cudaStream_t>(s)>>>(c->dc.self, c->dc.oplog);
  MCRDL_CUDA_CHECK(cudaGetLastError());
  MCRDL_CUDA_CHECK(cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(s)));
  return MCRDL_OK;
}

mcrdl_status_t mcrdl_comm_op_time(const mcrdl_comm* c, uint64_t first, uint64_t last, int64_t* ns) {
  if (c == nullptr || ns == nullptr) return set_error(MCRDL_ERR_VALIDATION, "NULL argument");
  *ns = -1;
  if (first == 0 || last < first || c->oplog_host == nullptr) return MCRDL_OK;
  if (c->log_seq - first >= uint64_t(kOpLogSlots)) {  // ring wrapped past it
    *ns = -2;
    return MCRDL_OK;
  }
  const uint64_t a = c->oplog_host[(first % kOpLogSlots) * 2];
  const uint64_t b = c->oplog_host[(last % kOpLogSlots) * 2 + 1];
  if ((a >> 48) != (first & 0xFFFF) || (b >> 48) != (last & 0xFFFF)) return MCRDL_OK;  // pending
  const uint64_t t0 = a & 0xFFFFFFFFFFFFull, t1 = b & 0xFFFFFFFFFFFFull;
  *ns = t1 >= t0 ? int64_t(t1 - t0) : int64_t(t1 + (1ull << 48) - t0);
  return MCRDL_OK;
}

mcrdl_status_t mcrdl_comm_caps(const mcrdl_comm* c, mcrdl_caps_t* caps) {
  if (c == nullptr || caps == nullptr) return set_error(MCRDL_ERR_VALIDATION, "NULL argument");
  memset(caps, 0, sizeof(*caps));
  caps->rank = c->rank;
  caps->world = c->world;
  caps->device = c->device;
  caps->num_sms = c->num_sms;
  caps->nvls_supported = c->nvls.ok ? 1 : 0;
  caps->ranks_per_device = c->ranks_per_device;
  caps->workspace_bytes = c->ws_bytes;
  caps->max_oneshot_bytes = uint64_t(c->dc.half_bytes) / uint64_t(c->world) / 256 * 256;
  caps->max_twoshot_chunk = uint64_t(c->dc.half_bytes) / 2 / 256 * 256;
  return MCRDL_OK;
}

mcrdl_status_t mcrdl_comm_stream(mcrdl_comm* c, int which, void** stream) {
  if (c == nullptr || stream == nullptr) return set_error(MCRDL_ERR_VALIDATION, "NULL argument");
  if (which < 0 || which > 2) return set_error(MCRDL_ERR_VALIDATION, "stream index %d", which);
  // created on first request: a communicator that never posts async work
  // adds no stream (co-located ranks share the device's hardware queues)
  cudaStream_t& s = which == 0 ? c->aux : c->xfer[which - 1];
  if (s == nullptr) {
    MCRDL_CUDA_CHECK(cudaSetDevice(c->device));
    MCRDL_CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  }
  *stream = reinterpret_cast<void*>(s);
  return MCRDL_OK;
}

mcrdl_status_t mcrdl_comm_set_tuning(mcrdl_comm* c, int kind, int n, const uint64_t* max_bytes,
                                     const int* algos) {
  if (c == nullptr) return set_error(MCRDL_ERR_NOT_INITIALIZED, "communicator is NULL");
  if (kind < 0 || kind >= MCRDL_TUNE_KINDS) return set_error(MCRDL_ERR_VALIDATION, "tuning kind %d", kind);
  if (n < 0 || n > 64 || (n > 0 && (max_bytes == nullptr || algos == nullptr)))
    return set_error(MCRDL_ERR_VALIDATION, "tuning rows: n = %d", n);
  std::vector<std::pair<uint64_t, int>> rows;
  for (int i = 0; i < n; ++i) {
    if (algos[i] < MCRDL_ALGO_AUTO || algos[i] > MCRDL_ALGO_CHAIN)
      return set_error(MCRDL_ERR_VALIDATION, "tuning row %d: algorithm %d", i, algos[i]);
    if (i > 0 && max_bytes[i] <= max_bytes[i - 1])
      return set_error(MCRDL_ERR_VALIDATION, "tuning rows: max_bytes must strictly increase");
    rows.emplace_back(max_bytes[i], algos[i]);
  }
  c->tune[kind] = std::move(rows);
  return MCRDL_OK;
}

int mcrdl_comm_last_algo(const mcrdl_comm* c, int kind) {
  if (c == nullptr || kind < 0 || kind >= MCRDL_TUNE_KINDS) return -1;
  return c->last_algo[kind];
}

mcrdl_status_t mcrdl_comm_status(mcrdl_comm* c) {
  if (c == nullptr) return set_error(MCRDL_ERR_NOT_INITIALIZED, "communicator is NULL");
  int e = *reinterpret_cast<volatile int*>(c->err_host);
  if (e != 0 && c->sticky == MCRDL_OK) c->sticky = e;
  if (c->sticky != MCRDL_OK)
    return set_error(c->sticky, "device reported %s", mcrdl_status_kind(c->sticky));
  return MCRDL_OK;
}

mcrdl_status_t mcrdl_symm_alloc(mcrdl_comm* c, uint64_t bytes, void** local_ptr) {
  if (c == nullptr || local_ptr == nullptr) return set_error(MCRDL_ERR_VALIDATION, "NULL argument");
  if (bytes == 0) bytes = 1;
  // With NVLS, size the region for a multicast binding (minimum granularity).
  size_t mg = 0;
  if (c->nvls.ok) {
    CUmulticastObjectProp mp{};
    mp.numDevices = unsigned(c->world);
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    mp.size = bytes;
    static const int64_t rec = env_int("MCRDL_SYMM_MC_RECOMMENDED", 0);
    if (g_drv.mcGranularity(&mp.size, &mp,
                            rec ? CU_MULTICAST_GRANULARITY_RECOMMENDED
                                : CU_MULTICAST_GRANULARITY_MINIMUM) == CUDA_SUCCESS)
      mg = mp.size;
    if (mg > 0) bytes = (bytes + mg - 1) / mg * mg;
  }
  Region rg;
  mcrdl_status_t st = alloc_region(c, bytes, &rg);
  if (st != MCRDL_OK) {
    unmap_region(c, rg);
    return st;
  }
  MCRDL_CUDA_CHECK(cudaMemsetAsync(reinterpret_cast<void*>(rg.ptr[c->rank]), 0, rg.bytes, kSetupStream));
  if (c->nvls.ok && mg > 0 && (st = bind_multicast(c, &rg)) != MCRDL_OK) {
    unmap_region(c, rg);
    return st;
  }
  MCRDL_CUDA_CHECK(cudaStreamSynchronize(kSetupStream));
  c->symm.push_back(rg);
  *local_ptr = reinterpret_cast<void*>(rg.ptr[c->rank]);
  return MCRDL_OK;
}

mcrdl_status_t mcrdl_symm_free(mcrdl_comm* c, void* local_ptr) {
  if (c == nullptr) return set_error(MCRDL_ERR_VALIDATION, "NULL communicator");
  for (size_t i = 0; i < c->symm.size(); ++i) {
    if (reinterpret_cast<void*>(c->symm[i].ptr[c->rank]) == local_ptr) {
      cudaDeviceSynchronize();
      unmap_region(c, c->symm[i]);
      c->symm.erase(c->symm.begin() + i);
      return MCRDL_OK;
    }
  }
  return set_error(MCRDL_ERR_VALIDATION, "pointer is not a symmetric allocation of this comm");
}

}  // extern "C"
