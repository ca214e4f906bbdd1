// devpool.cu -- see devpool.h.
#include "devpool.h"

#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <unordered_map>
#include <vector>

namespace ssqa_engine {
namespace {

struct Block {
  int device;
  size_t bytes;  // size class actually allocated
};

struct Pool {
  std::mutex mu;
  // (device, size class) -> cached blocks
  std::map<std::pair<int, size_t>, std::vector<void*>> free_blocks;
  std::unordered_map<void*, Block> live;
  std::map<int, size_t> cached, in_use;
};

Pool& pool() {
  static Pool* p = new Pool();  // never destroyed: frees may run during exit
  return *p;
}

// Size classes: 512 B granules up to 1 MiB, 2 MiB granules above (the
// driver's large-page size), so repeated batches of one shape hit exactly.
size_t size_class(size_t bytes) {
  if (bytes == 0) bytes = 1;
  if (bytes <= (size_t(1) << 20)) return (bytes + 511) / 512 * 512;
  const size_t g = size_t(2) << 20;
  return (bytes + g - 1) / g * g;
}

size_t release_locked(Pool& P, int device) {
  size_t freed = 0;
  int cur = -1;
  cudaGetDevice(&cur);
  for (auto it = P.free_blocks.begin(); it != P.free_blocks.end();) {
    if (device >= 0 && it->first.first != device) {
      ++it;
      continue;
    }
    cudaSetDevice(it->first.first);
    for (void* b : it->second) {
      cudaFree(b);
      freed += it->first.second;
      P.cached[it->first.first] -= it->first.second;
    }
    it = P.free_blocks.erase(it);
  }
  if (cur >= 0) cudaSetDevice(cur);
  return freed;
}

}  // namespace

int pool_malloc(void** p, size_t bytes) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return int(e);
  const size_t cls = size_class(bytes);
  Pool& P = pool();
  std::lock_guard<std::mutex> lk(P.mu);
  auto it = P.free_blocks.find({dev, cls});
  if (it != P.free_blocks.end() && !it->second.empty()) {
    *p = it->second.back();
    it->second.pop_back();
    P.cached[dev] -= cls;
    P.in_use[dev] += cls;
    P.live[*p] = Block{dev, cls};
    return int(cudaSuccess);
  }
  e = cudaMalloc(p, cls);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();  // clear the sticky-free error state of this call
    release_locked(P, dev);
    e = cudaMalloc(p, cls);
  }
  if (e != cudaSuccess) {
    *p = nullptr;
    return int(e);
  }
  P.in_use[dev] += cls;
  P.live[*p] = Block{dev, cls};
  return int(cudaSuccess);
}

void pool_free(void* p) {
  if (!p) return;
  Pool& P = pool();
  std::lock_guard<std::mutex> lk(P.mu);
  auto it = P.live.find(p);
  if (it == P.live.end()) {  // not ours: plain free
    cudaFree(p);
    return;
  }
  const Block b = it->second;
  P.live.erase(it);
  P.in_use[b.device] -= b.bytes;
  P.cached[b.device] += b.bytes;
  P.free_blocks[{b.device, b.bytes}].push_back(p);
}

size_t pool_trim(int device) {
  Pool& P = pool();
  std::lock_guard<std::mutex> lk(P.mu);
  return release_locked(P, device);
}

void pool_stats(int device, size_t* cached, size_t* in_use) {
  Pool& P = pool();
  std::lock_guard<std::mutex> lk(P.mu);
  if (cached) *cached = P.cached.count(device) ? P.cached[device] : 0;
  if (in_use) *in_use = P.in_use.count(device) ? P.in_use[device] : 0;
}

}  // namespace ssqa_engine

extern "C" {

long long ssqa_pool_trim(int device) { return (long long)ssqa_engine::pool_trim(device); }

int ssqa_pool_stats(int device, long long* cached_bytes, long long* in_use_bytes) {
  size_t c = 0, u = 0;
  ssqa_engine::pool_stats(device, &c, &u);
  if (cached_bytes) *cached_bytes = (long long)c;
  if (in_use_bytes) *in_use_bytes = (long long)u;
  return 0;
}

}  // extern "C"
