// Stream-ordered device allocation with an exact-size cache for large blocks
// (declared in gh_internal.cuh; see the comment there).
//
// Small blocks go straight to the default memory pool. A freed block of
// kCacheMin bytes or more is parked under its size with an event recorded on
// the freeing stream; the next request of exactly that size (on any stream of
// the same device) takes it after making its stream wait on the event, so
// reuse stays stream-ordered. The end-to-end solve allocates the same sizes
// in the same order call after call, so after the first call every large
// request is a cache hit and the pool never has to map new memory mid-solve.

#include <cstdio>
#include <cstdlib>
#include <list>
#include <mutex>

#include "gh_internal.cuh"

namespace gh {

namespace {

constexpr size_t kCacheMin = size_t(1) << 20;  // smaller blocks: the pool directly
constexpr size_t kCacheMax = size_t(2) << 30;  // larger ones too: a cache holding them kept the
                                               // pool from reusing that memory for other sizes
                                               // (config 5: every call ran out of memory once)

struct Block {
  void* p;
  size_t bytes;
  int device;
  cudaEvent_t ready;  // recorded on the freeing stream
};

struct Cache {
  std::mutex mu;
  std::list<Block> blocks;    // oldest first
  size_t bytes[64] = {};      // cached bytes per device
  size_t limit[64] = {};      // an eighth of the device memory, set on first use
  std::vector<cudaEvent_t> spare_events;
};

Cache& cache() {
  static Cache* c = new Cache();  // never destroyed: frees may run during static destruction
  return *c;
}

cudaEvent_t take_event(Cache& c) {
  if (!c.spare_events.empty()) {
    cudaEvent_t e = c.spare_events.back();
    c.spare_events.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  GH_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return e;
}

// Give a cached block back to the pool on stream s (of the block's device),
// ordered after its last use.
void release_block(Cache& c, const Block& b, cudaStream_t s) {
  cudaStreamWaitEvent(s, b.ready, 0);
  cudaFreeAsync(b.p, s);
  c.spare_events.push_back(b.ready);
  c.bytes[b.device] -= b.bytes;
}

}  // namespace

void* dev_alloc(size_t bytes, cudaStream_t s) {
  int dev = 0;
  GH_CUDA(cudaGetDevice(&dev));
  Cache& c = cache();
  if (bytes >= kCacheMin && bytes <= kCacheMax && dev >= 0 && dev < 64) {
    std::lock_guard<std::mutex> lock(c.mu);
    for (auto it = c.blocks.begin(); it != c.blocks.end(); ++it) {
      if (it->bytes != bytes || it->device != dev) continue;
      void* p = it->p;
      GH_CUDA(cudaStreamWaitEvent(s, it->ready, 0));
      c.spare_events.push_back(it->ready);
      c.bytes[dev] -= bytes;
      c.blocks.erase(it);
      return p;
    }
  }
  void* p = nullptr;
  cudaError_t e = cudaMallocAsync(&p, bytes, s);
  if (e == cudaErrorMemoryAllocation && getenv("GH_ALLOC_TRACE"))
    fprintf(stderr, "[gh_alloc] %zu B: pool allocation failed, flushing the cache\n", bytes);
  if (e == cudaErrorMemoryAllocation) {  // hand the cached blocks back to the pool and retry
    (void)cudaGetLastError();
    dev_cache_flush();
    e = cudaMallocAsync(&p, bytes, s);
  }
  if (e == cudaErrorMemoryAllocation) {
    // the pool's free blocks are too fragmented for this request: let it return
    // what it holds unused to the driver (slow: the memory is mapped again), retry
    (void)cudaGetLastError();
    cudaMemPool_t pool;
    if (cudaDeviceSynchronize() == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess)
      cudaMemPoolTrimTo(pool, 0);
    (void)cudaGetLastError();
    e = cudaMallocAsync(&p, bytes, s);
  }
  GH_CUDA(e);
  return p;
}

void dev_free(void* p, size_t bytes, cudaStream_t s) {
  if (!p) return;
  // the block's own device (a handle may be destroyed with another device current)
  cudaPointerAttributes attr{};
  if (bytes < kCacheMin || bytes > kCacheMax || cudaPointerGetAttributes(&attr, p) != cudaSuccess || attr.device < 0 ||
      attr.device >= 64) {
    (void)cudaGetLastError();
    cudaFreeAsync(p, s);
    return;
  }
  const int dev = attr.device;
  Cache& c = cache();
  std::lock_guard<std::mutex> lock(c.mu);
  if (!c.limit[dev]) {
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) total_b = 0;
    c.limit[dev] = total_b / 8;
  }
  cudaEvent_t ev = nullptr;
  try {
    ev = take_event(c);
  } catch (...) {
    cudaFreeAsync(p, s);
    return;
  }
  if (cudaEventRecord(ev, s) != cudaSuccess) {
    c.spare_events.push_back(ev);
    cudaFreeAsync(p, s);
    return;
  }
  c.blocks.push_back(Block{p, bytes, dev, ev});
  c.bytes[dev] += bytes;
  // oldest blocks of this device back to the pool past the limit
  for (auto it = c.blocks.begin(); c.bytes[dev] > c.limit[dev] && it != c.blocks.end();) {
    if (it->device != dev) {
      ++it;
      continue;
    }
    release_block(c, *it, s);
    it = c.blocks.erase(it);
  }
}

void dev_cache_flush() {
  Cache& c = cache();
  std::lock_guard<std::mutex> lock(c.mu);
  for (const Block& b : c.blocks) {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(b.device);
    cudaEventSynchronize(b.ready);
    cudaFree(b.p);
    cudaSetDevice(cur);
    c.spare_events.push_back(b.ready);
    c.bytes[b.device] -= b.bytes;
  }
  c.blocks.clear();
}

}  // namespace gh
