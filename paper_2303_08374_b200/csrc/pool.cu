// Symmetric memory pool: ordinary torch tensors on the zero-copy paths.
//
// One collective mcrdl_symm_alloc arena per pool (peer-mapped, bound to the
// NVSwitch multicast object when NVLS exists); a first-fit sub-allocator hands
// out pieces of it through torch's pluggable-allocator hooks
// (torch.cuda.MemPool + CUDAPluggableAllocator -> mcrdl_pool_malloc/free).
// A tensor allocated inside the pool has the same offset in the arena on
// every rank whenever the ranks allocate in the same order (SPMD), so
// all_reduce on it takes the zero-copy symmetric kernels (k_ar_symm: NVLS
// multimem or peer loads, no workspace staging) and exchanges into it store
// straight into the peers' outputs (k_x_symm). Offsets are folded into the
// flag signature: ranks whose pool layouts diverged fail with ORDER_MISMATCH.
//
// Reference counterpart: none (the reference has no device memory); this is
// the B200 answer to "ordinary tensors get the zero-copy path".
#include <map>
#include <mutex>
#include <vector>

#include "internal.h"

struct mcrdl_pool {
  mcrdl_comm* comm = nullptr;
  uint8_t* base = nullptr;
  uint64_t bytes = 0;
  std::map<uint64_t, uint64_t> free_list;  // offset -> bytes (coalesced)
  std::map<uint64_t, uint64_t> used;       // offset -> bytes
  uint64_t in_use = 0;
  std::mutex mu;
};

namespace mcrdl {
namespace {
constexpr uint64_t kPoolAlign = 512;
thread_local mcrdl_pool* t_active = nullptr;  // the calling thread's rank's pool
std::mutex g_pools_mu;
std::vector<mcrdl_pool*> g_pools;

mcrdl_pool* owner_of(const void* p) {
  std::lock_guard<std::mutex> lk(g_pools_mu);
  const uint8_t* q = static_cast<const uint8_t*>(p);
  for (mcrdl_pool* pool : g_pools)
    if (q >= pool->base && q < pool->base + pool->bytes) return pool;
  return nullptr;
}
}  // namespace
}  // namespace mcrdl

using namespace mcrdl;

extern "C" {

mcrdl_status_t mcrdl_pool_create(mcrdl_comm* c, uint64_t bytes, mcrdl_pool** out) {
  if (c == nullptr || out == nullptr) return set_error(MCRDL_ERR_VALIDATION, "NULL argument");
  *out = nullptr;
  bytes = (bytes + kPoolAlign - 1) / kPoolAlign * kPoolAlign;
  void* base = nullptr;
  mcrdl_status_t st = mcrdl_symm_alloc(c, bytes, &base);  // collective
  if (st != MCRDL_OK) return st;
  auto* p = new mcrdl_pool();
  p->comm = c;
  p->base = static_cast<uint8_t*>(base);
  p->bytes = bytes;
  p->free_list[0] = bytes;
  {
    std::lock_guard<std::mutex> lk(g_pools_mu);
    g_pools.push_back(p);
  }
  *out = p;
  return MCRDL_OK;
}

mcrdl_status_t mcrdl_pool_activate(mcrdl_pool* p) {
  t_active = p;  // NULL deactivates
  return MCRDL_OK;
}

mcrdl_status_t mcrdl_pool_stats(mcrdl_pool* p, uint64_t* base, uint64_t* bytes, uint64_t* in_use) {
  if (p == nullptr) return set_error(MCRDL_ERR_VALIDATION, "NULL pool");
  std::lock_guard<std::mutex> lk(p->mu);
  if (base) *base = reinterpret_cast<uint64_t>(p->base);
  if (bytes) *bytes = p->bytes;
  if (in_use) *in_use = p->in_use;
  return MCRDL_OK;
}

mcrdl_status_t mcrdl_pool_destroy(mcrdl_pool* p) {
  if (p == nullptr) return MCRDL_OK;
  {
    std::lock_guard<std::mutex> lk(g_pools_mu);
    for (size_t i = 0; i < g_pools.size(); ++i)
      if (g_pools[i] == p) g_pools.erase(g_pools.begin() + i), i = g_pools.size();
  }
  if (t_active == p) t_active = nullptr;
  mcrdl_status_t st = mcrdl_symm_free(p->comm, p->base);
  delete p;
  return st;
}

// torch.cuda.memory.CUDAPluggableAllocator hooks. Allocation comes from the
// calling thread's active pool (NULL -> torch reports out of memory).
void* mcrdl_pool_malloc(ssize_t size, int device, void* stream) {
  (void)device;
  (void)stream;
  mcrdl_pool* p = t_active;
  if (p == nullptr || size <= 0) return nullptr;
  const uint64_t want = (uint64_t(size) + kPoolAlign - 1) / kPoolAlign * kPoolAlign;
  std::lock_guard<std::mutex> lk(p->mu);
  for (auto it = p->free_list.begin(); it != p->free_list.end(); ++it) {
    if (it->second < want) continue;
    const uint64_t off = it->first, len = it->second;
    p->free_list.erase(it);
    if (len > want) p->free_list[off + want] = len - want;
    p->used[off] = want;
    p->in_use += want;
    return p->base + off;
  }
  return nullptr;
}

void mcrdl_pool_free(void* ptr, size_t size, int device, void* stream) {
  (void)size;
  (void)device;
  (void)stream;
  mcrdl_pool* p = owner_of(ptr);
  if (p == nullptr) return;
  std::lock_guard<std::mutex> lk(p->mu);
  const uint64_t off = uint64_t(static_cast<uint8_t*>(ptr) - p->base);
  auto u = p->used.find(off);
  if (u == p->used.end()) return;
  uint64_t start = off, len = u->second;
  p->in_use -= len;
  p->used.erase(u);
  auto next = p->free_list.lower_bound(start);
  if (next != p->free_list.end() && next->first == start + len) {  // merge right
    len += next->second;
    next = p->free_list.erase(next);
  }
  if (next != p->free_list.begin()) {  // merge left
    auto prev = std::prev(next);
    if (prev->first + prev->second == start) {
      start = prev->first;
      len += prev->second;
      p->free_list.erase(prev);
    }
  }
  p->free_list[start] = len;
}

}  // extern "C"
