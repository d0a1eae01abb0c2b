// Pooled memory arena for fab storage and exchange staging (device HBM,
// pinned host, or plain host memory for host-only tests).
//
// Replaces the reference's Arena (/root/reference/pkg/src/miniamr_core/
// arena.py:87-163): slabs reserved up front (or grown lazily by at least
// 1 MiB), aligned blocks bump-allocated from the newest slab, freed blocks
// kept on LIFO free lists segregated by (padded size, alignment) so repeated
// temporaries never reach cudaMalloc; in_use counts alignment padding.  The
// "system" kind makes one allocation per request (SystemArena,
// arena.py:166-197).  Stream-ordered reuse (the AsyncArena of arena.py:
// 201-334 on a GPU): ghx_arena_free_after records an event on each stream
// whose queued work may still touch the block and parks the block until
// every event has completed; parked blocks are recycled by the next
// alloc/free/poll that finds their events done (cudaFreeAsync-style
// semantics, no host wait).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include "ghx_internal.h"

using ghx::set_error;

namespace {

constexpr size_t kGrowUnit = size_t(1) << 20;

struct Blk {
  char *ptr;
  size_t padded, align;
  char *raw;  // system kind: the allocation to release
};

int sys_alloc(int memory, int device, size_t bytes, void **out) {
  *out = nullptr;
  if (memory == GHX_ARENA_HOST) {
    *out = std::malloc(bytes);
    if (!*out) {
      set_error("ghx_arena: host allocation failed");
      return GHX_ENOMEM;
    }
    return GHX_OK;
  }
  int prev = 0;
  cudaGetDevice(&prev);
  if (memory == GHX_ARENA_DEVICE && prev != device) cudaSetDevice(device);
  cudaError_t e = memory == GHX_ARENA_DEVICE ? cudaMalloc(out, bytes) : cudaHostAlloc(out, bytes, cudaHostAllocMapped);
  if (memory == GHX_ARENA_DEVICE && prev != device) cudaSetDevice(prev);
  if (e != cudaSuccess) {
    set_error(std::string("ghx_arena: ") + cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? GHX_ENOMEM : GHX_ECUDA;
  }
  return GHX_OK;
}

void sys_free(int memory, void *p) {
  if (!p) return;
  if (memory == GHX_ARENA_HOST)
    std::free(p);
  else if (memory == GHX_ARENA_DEVICE)
    cudaFree(p);
  else
    cudaFreeHost(p);
}

}  // namespace

struct ghx_arena {
  int kind = GHX_ARENA_POOLED;
  int memory = GHX_ARENA_DEVICE;
  int device = 0;
  std::mutex mu;
  struct Slab {
    char *base;
    size_t cap, cursor;
  };
  std::vector<Slab> slabs;
  std::map<std::pair<size_t, size_t>, std::vector<Blk>> free_lists;
  std::unordered_map<char *, Blk> live;
  struct Parked {
    Blk b;
    std::vector<cudaEvent_t> events;
  };
  std::vector<Parked> parked;  // freed, waiting for stream work to finish
  int64_t reserved = 0, in_use = 0, alloc_calls = 0, slab_growths = 0;
};

namespace {

int carve(ghx_arena *a, size_t padded, size_t align, Blk *out) {
  auto aligned = [&](const ghx_arena::Slab &s) {
    const uintptr_t addr = reinterpret_cast<uintptr_t>(s.base) + s.cursor;
    return s.cursor + ((align - addr % align) % align);
  };
  if (!a->slabs.empty()) {
    ghx_arena::Slab &s = a->slabs.back();
    const size_t start = aligned(s);
    if (start + padded <= s.cap) {
      s.cursor = start + padded;
      *out = Blk{s.base + start, padded, align, nullptr};
      return GHX_OK;
    }
  }
  const size_t growth = std::max(padded + align, kGrowUnit);
  void *p = nullptr;
  if (int rc = sys_alloc(a->memory, a->device, growth, &p)) return rc;
  a->slabs.push_back({static_cast<char *>(p), growth, 0});
  a->reserved += (int64_t)growth;
  a->slab_growths += 1;
  ghx_arena::Slab &s = a->slabs.back();
  const size_t start = aligned(s);
  s.cursor = start + padded;
  *out = Blk{s.base + start, padded, align, nullptr};
  return GHX_OK;
}

void release(ghx_arena *a, const Blk &b) {
  a->in_use -= (int64_t)b.padded;
  if (a->kind == GHX_ARENA_SYSTEM) {
    a->reserved -= (int64_t)b.padded;
    sys_free(a->memory, b.raw);
  } else {
    a->free_lists[{b.padded, b.align}].push_back(b);
  }
}

// Recycle every parked block whose events have all completed (caller holds
// a->mu).  Returns the number still parked.
int64_t drain(ghx_arena *a) {
  size_t keep = 0;
  for (size_t i = 0; i < a->parked.size(); ++i) {
    ghx_arena::Parked &p = a->parked[i];
    bool done = true;
    for (cudaEvent_t e : p.events) {
      const cudaError_t q = cudaEventQuery(e);
      if (q == cudaErrorNotReady) {
        done = false;
        break;
      }
      if (q != cudaSuccess) cudaGetLastError();  // a failed event cannot be waited on: treat as done
    }
    if (done) {
      for (cudaEvent_t e : p.events) cudaEventDestroy(e);
      release(a, p.b);
    } else {
      if (keep != i) a->parked[keep] = std::move(p);
      ++keep;
    }
  }
  a->parked.resize(keep);
  return (int64_t)keep;
}

}  // namespace

extern "C" {

int ghx_arena_create(int32_t kind, int32_t memory, int32_t device, size_t capacity_bytes, ghx_arena **out) {
  if (!out || (kind != GHX_ARENA_POOLED && kind != GHX_ARENA_SYSTEM) ||
      (memory != GHX_ARENA_DEVICE && memory != GHX_ARENA_PINNED && memory != GHX_ARENA_HOST)) {
    set_error("ghx_arena_create: bad arguments");
    return GHX_EINVAL;
  }
  ghx_arena *a = new (std::nothrow) ghx_arena();
  if (!a) {
    set_error("ghx_arena_create: out of memory");
    return GHX_ENOMEM;
  }
  a->kind = kind;
  a->memory = memory;
  a->device = device;
  if (kind == GHX_ARENA_POOLED && capacity_bytes > 0) {
    void *p = nullptr;
    if (int rc = sys_alloc(memory, device, capacity_bytes, &p)) {
      delete a;
      return rc;
    }
    a->slabs.push_back({static_cast<char *>(p), capacity_bytes, 0});
    a->reserved = (int64_t)capacity_bytes;
  }
  *out = a;
  return GHX_OK;
}

int ghx_arena_alloc(ghx_arena *a, size_t nbytes, size_t align, void **out) {
  if (!a || !out || align == 0 || (align & (align - 1)) != 0) {
    set_error("ghx_arena_alloc: alignment must be a power of two");
    return GHX_EINVAL;
  }
  *out = nullptr;
  if (nbytes == 0) return GHX_OK;  // the null block
  const size_t padded = (nbytes + align - 1) / align * align;
  std::lock_guard<std::mutex> lk(a->mu);
  if (!a->parked.empty()) drain(a);
  a->alloc_calls += 1;
  Blk b{};
  if (a->kind == GHX_ARENA_SYSTEM) {
    const size_t total = padded + align;
    void *p = nullptr;
    if (int rc = sys_alloc(a->memory, a->device, total, &p)) return rc;
    char *raw = static_cast<char *>(p);
    const uintptr_t addr = reinterpret_cast<uintptr_t>(raw);
    b = Blk{raw + (align - addr % align) % align, total, align, raw};
    a->reserved += (int64_t)total;
  } else {
    auto it = a->free_lists.find({padded, align});
    if (it != a->free_lists.end() && !it->second.empty()) {
      b = it->second.back();  // LIFO reuse per size class
      it->second.pop_back();
    } else if (int rc = carve(a, padded, align, &b)) {
      return rc;
    }
  }
  a->in_use += (int64_t)b.padded;
  a->live[b.ptr] = b;
  *out = b.ptr;
  return GHX_OK;
}

int ghx_arena_free(ghx_arena *a, void *ptr) {
  if (!a) {
    set_error("ghx_arena_free: null arena");
    return GHX_EINVAL;
  }
  if (!ptr) return GHX_OK;
  std::lock_guard<std::mutex> lk(a->mu);
  auto it = a->live.find(static_cast<char *>(ptr));
  if (it == a->live.end()) {
    set_error("ghx_arena_free: double free (or foreign pointer) of an arena block");
    return GHX_EOVERLAP;
  }
  const Blk b = it->second;
  a->live.erase(it);
  release(a, b);
  if (!a->parked.empty()) drain(a);
  return GHX_OK;
}

int ghx_arena_free_after(ghx_arena *a, void *ptr, void *const *streams, int32_t nstreams) {
  if (!a || nstreams < 0 || (nstreams && !streams)) {
    set_error("ghx_arena_free_after: bad arguments");
    return GHX_EINVAL;
  }
  if (!ptr) return GHX_OK;
  std::lock_guard<std::mutex> lk(a->mu);
  auto it = a->live.find(static_cast<char *>(ptr));
  if (it == a->live.end()) {
    set_error("ghx_arena_free_after: double free (or foreign pointer) of an arena block");
    return GHX_EOVERLAP;
  }
  ghx_arena::Parked p{it->second, {}};
  for (int32_t i = 0; i < nstreams; ++i) {
    cudaStream_t st = static_cast<cudaStream_t>(streams[i]);
    int dev = 0, prev = 0;
    cudaGetDevice(&prev);
    if (cudaStreamGetDevice(st, &dev) != cudaSuccess) {
      cudaGetLastError();
      dev = prev;
    }
    if (dev != prev) cudaSetDevice(dev);
    cudaEvent_t e = nullptr;
    cudaError_t rc = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    if (rc == cudaSuccess) rc = cudaEventRecord(e, st);
    if (dev != prev) cudaSetDevice(prev);
    if (rc != cudaSuccess) {
      if (e) cudaEventDestroy(e);
      for (cudaEvent_t x : p.events) cudaEventDestroy(x);
      set_error(std::string("ghx_arena_free_after: ") + cudaGetErrorString(rc));
      return GHX_ECUDA;
    }
    p.events.push_back(e);
  }
  a->live.erase(it);
  if (p.events.empty())
    release(a, p.b);
  else
    a->parked.push_back(std::move(p));
  drain(a);
  return GHX_OK;
}

int ghx_arena_poll(ghx_arena *a, int64_t *parked) {
  if (!a) {
    set_error("ghx_arena_poll: null arena");
    return GHX_EINVAL;
  }
  std::lock_guard<std::mutex> lk(a->mu);
  const int64_t n = drain(a);
  if (parked) *parked = n;
  return GHX_OK;
}

int ghx_arena_block_size(const ghx_arena *a, const void *ptr, size_t *padded) {
  if (!a || !ptr || !padded) {
    set_error("ghx_arena_block_size: bad arguments");
    return GHX_EINVAL;
  }
  ghx_arena *m = const_cast<ghx_arena *>(a);
  std::lock_guard<std::mutex> lk(m->mu);
  auto it = m->live.find(const_cast<char *>(static_cast<const char *>(ptr)));
  if (it == m->live.end()) {
    set_error("ghx_arena_block_size: not a live block");
    return GHX_EINVAL;
  }
  *padded = it->second.padded;
  return GHX_OK;
}

int ghx_arena_stats(const ghx_arena *a, int64_t out[4]) {
  if (!a || !out) {
    set_error("ghx_arena_stats: bad arguments");
    return GHX_EINVAL;
  }
  ghx_arena *m = const_cast<ghx_arena *>(a);
  std::lock_guard<std::mutex> lk(m->mu);
  out[0] = m->reserved;
  out[1] = m->in_use;
  out[2] = m->alloc_calls;
  out[3] = m->slab_growths;
  return GHX_OK;
}

void ghx_arena_destroy(ghx_arena *a) {
  if (!a) return;
  for (auto &p : a->parked) {  // the slabs go away: let the queued work finish first
    for (cudaEvent_t e : p.events) {
      cudaEventSynchronize(e);
      cudaEventDestroy(e);
    }
    if (p.b.raw) sys_free(a->memory, p.b.raw);
  }
  for (auto &kv : a->live)
    if (kv.second.raw) sys_free(a->memory, kv.second.raw);
  for (auto &s : a->slabs) sys_free(a->memory, s.base);
  delete a;
}

}  // extern "C"
