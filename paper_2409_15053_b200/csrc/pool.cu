// pool.cu — caching allocator behind DevBuf and the pinned staging buffers.
//
// A solve allocates the same few large blocks every time (the Lanczos basis: 2.7 GB on the
// PARSEC-shaped config, 24 GB on the 100^3 Laplacian; the recovery blocks V, AV; small
// coefficient scratch).  cudaMalloc/cudaFree of such blocks cost tens to hundreds of
// milliseconds per solve (measured: up to 0.4 s of a 0.7 s solve, and worse while
// nvidia-smi polls the driver), so freed blocks are kept per device and handed out again.
// Reuse is safe without synchronisation because every context issues its work on one
// stream and blocks are returned only after the work that uses them has been enqueued.
// When the driver runs out of memory the cache is emptied and the allocation retried.

#include <map>
#include <mutex>
#include <unordered_map>

#include "flz_internal.hpp"

namespace flz {

namespace {

struct Pool {
  std::mutex mu;
  // cached free blocks per device, by size
  std::map<int, std::multimap<size_t, void*>> free_blocks;
  std::unordered_map<void*, std::pair<int, size_t>> live;  // ptr -> (device, size)
  std::multimap<size_t, void*> free_pinned;
  std::unordered_map<void*, size_t> live_pinned;
  size_t cached_bytes = 0;
  size_t cached_pinned = 0;
};

Pool& pool() {
  static Pool* p = new Pool;  // leaked on purpose: no CUDA calls during static destruction
  return *p;
}

size_t round_size(size_t bytes) {
  const size_t g = bytes >= (size_t(1) << 20) ? (size_t(2) << 20) : 512;
  return (bytes + g - 1) / g * g;
}

void trim_locked(Pool& P) {
  for (auto& dev : P.free_blocks) {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(dev.first);
    for (auto& b : dev.second) cudaFree(b.second);
    dev.second.clear();
    cudaSetDevice(cur);
  }
  P.cached_bytes = 0;
}

}  // namespace

void* pool_alloc(size_t bytes) {
  if (bytes == 0) return nullptr;
  Pool& P = pool();
  const size_t want = round_size(bytes);
  int dev = 0;
  FLZ_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(P.mu);
  auto& fb = P.free_blocks[dev];
  auto it = fb.lower_bound(want);
  if (it != fb.end() && it->first <= want + want / 4) {  // at most 25 % slack
    void* p = it->second;
    P.live[p] = {dev, it->first};
    P.cached_bytes -= it->first;
    fb.erase(it);
    return p;
  }
  void* p = nullptr;
  cudaError_t err = cudaMalloc(&p, want);
  if (err == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    trim_locked(P);
    err = cudaMalloc(&p, want);
  }
  if (err != cudaSuccess)
    throw ApiError(FLZ_ECUDA, std::string("cudaMalloc(") + std::to_string(want) +
                                  " bytes): " + cudaGetErrorString(err));
  P.live[p] = {dev, want};
  return p;
}

void pool_free(void* p) {
  if (!p) return;
  Pool& P = pool();
  std::lock_guard<std::mutex> lock(P.mu);
  auto it = P.live.find(p);
  if (it == P.live.end()) {  // not ours
    cudaFree(p);
    return;
  }
  P.free_blocks[it->second.first].emplace(it->second.second, p);
  P.cached_bytes += it->second.second;
  P.live.erase(it);
}

void pool_trim() {
  Pool& P = pool();
  std::lock_guard<std::mutex> lock(P.mu);
  trim_locked(P);
}

size_t pool_cached_bytes() {
  Pool& P = pool();
  std::lock_guard<std::mutex> lock(P.mu);
  return P.cached_bytes;
}

void* pinned_alloc(size_t bytes) {
  if (bytes == 0) return nullptr;
  Pool& P = pool();
  const size_t want = round_size(bytes);
  std::lock_guard<std::mutex> lock(P.mu);
  auto it = P.free_pinned.lower_bound(want);
  if (it != P.free_pinned.end() && it->first <= 2 * want) {
    void* p = it->second;
    P.live_pinned[p] = it->first;
    P.cached_pinned -= it->first;
    P.free_pinned.erase(it);
    return p;
  }
  void* p = nullptr;
  FLZ_CUDA(cudaMallocHost(&p, want));
  P.live_pinned[p] = want;
  return p;
}

void pinned_free(void* p) {
  if (!p) return;
  Pool& P = pool();
  std::lock_guard<std::mutex> lock(P.mu);
  auto it = P.live_pinned.find(p);
  if (it == P.live_pinned.end()) {
    cudaFreeHost(p);
    return;
  }
  // eigenvector blocks of consecutive solves are reused; the cache of page-locked memory is
  // capped so that it cannot pin the host down
  constexpr size_t kPinnedCacheCap = size_t(4) << 30;
  if (P.cached_pinned + it->second > kPinnedCacheCap) {
    cudaFreeHost(p);
  } else {
    P.free_pinned.emplace(it->second, p);
    P.cached_pinned += it->second;
  }
  P.live_pinned.erase(it);
}

}  // namespace flz
