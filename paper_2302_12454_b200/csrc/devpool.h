// devpool.h -- process-wide caching allocator for the engine's device buffers.
//
// A public ssqa_run_batch call (the drop-in for the reference's ssqa_run /
// run_trials, annealer.cpp:474-487, bench.cpp:359-432) creates and destroys a
// problem and a batch every time: at C3 that is ~450 MB of device state.
// cudaMalloc / cudaFree of such blocks cost milliseconds and, at times,
// hundreds of milliseconds (cudaFree waits for the device and unmaps), so
// freed blocks are kept per (device, size class) and handed to the next
// request of the same class.  Every free happens after the owner's stream has
// been synchronised (batch/problem destroy, scratch buffers), so a cached
// block is never still in use by a kernel when it is handed out again.
// On cudaErrorMemoryAllocation the cache of that device is released and the
// allocation retried once; ssqa_pool_trim() releases it on request.
#pragma once

#include <cuda_runtime_api.h>

#include <cstddef>

namespace ssqa_engine {

// cudaMalloc semantics (on the current device); returns cudaSuccess or the error.
int pool_malloc(void** p, size_t bytes);
// Returns a block from pool_malloc to the cache (nullptr is a no-op).
void pool_free(void* p);
// Releases every cached block of `device` (-1: all devices); returns bytes freed.
size_t pool_trim(int device);
// Bytes cached (free, not handed out) and bytes handed out on `device`.
void pool_stats(int device, size_t* cached, size_t* in_use);

template <class T>
inline cudaError_t pmalloc(T** p, size_t bytes) {
  return cudaError_t(pool_malloc(reinterpret_cast<void**>(p), bytes));
}

}  // namespace ssqa_engine
