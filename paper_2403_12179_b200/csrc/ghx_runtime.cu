// Device memory, CUDA-IPC, cross-rank device barrier and the synthetic
// input generator.  Fab storage is owned by the Python layer through these
// calls (one slab per MultiFab per device), so the fused exchange kernel
// can address local fabs, peer-mapped fabs and IPC-mapped fabs uniformly.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>

#include "ghx_internal.h"

using ghx::set_error;

namespace {

int fail(cudaError_t e, const char *what) {
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  // consume a non-sticky error (e.g. cudaErrorAlreadyMapped from an IPC open
  // the caller retries) so a later cudaGetLastError() does not report it
  // again for an unrelated, successful call
  (void)cudaGetLastError();
  return GHX_ECUDA;
}

struct Guard {
  int prev = -1;
  explicit Guard(int dev) {
    cudaGetDevice(&prev);
    if (dev >= 0 && dev != prev) cudaSetDevice(dev);
  }
  ~Guard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

__global__ void memset_u64_kernel(uint64_t *p, uint64_t v, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = v;
}

struct FlagPtrs {
  uint64_t *p[64];
};

__device__ unsigned int g_barrier_timeouts = 0;

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Spins at most timeout_ns: a peer that never arrives (crashed rank) makes
// the barrier give up and count a timeout instead of hanging the GPU.
__global__ void barrier_kernel(FlagPtrs flags, int rank, int nranks, uint64_t epoch, uint64_t timeout_ns) {
  const int peer = threadIdx.x;
  if (peer >= nranks) return;
  // make every earlier write of this stream visible system-wide, then signal
  __threadfence_system();
  uint64_t *remote = flags.p[peer] + rank;
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(remote), "l"(epoch) : "memory");
  const uint64_t *mine = flags.p[rank] + peer;
  const uint64_t t0 = globaltimer_ns();
  uint64_t v = 0;
  for (uint32_t it = 0;; ++it) {
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory");
    if (v >= epoch) break;
    if ((it & 1023) == 1023 && globaltimer_ns() - t0 > timeout_ns) {
      atomicAdd(&g_barrier_timeouts, 1u);
      break;
    }
    __nanosleep(64);
  }
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct FillArgs {
  int64_t flo[3], fn[3];  // fab storage lo, extents
  int64_t vlo[3], vhi[3];
  int64_t dlo[3], dn[3];  // hash domain lo, extents
  int64_t ncomp;
  uint64_t seed;
  int32_t wrap;           // 0: hash on the valid box; else bit d = periodic axis d, hash wherever the
                          // periodically wrapped cell lies in the domain
};

__device__ __forceinline__ int64_t wrap_axis(int64_t g, int64_t lo, int64_t n) {
  int64_t r = (g - lo) % n;
  return (r < 0 ? r + n : r) + lo;
}

template <class T>
__global__ void fill_hash_kernel(T *fab, FillArgs a) {
  const int64_t plane = a.fn[0] * a.fn[1];
  const int64_t vol = plane * a.fn[2];
  const int64_t total = vol * a.ncomp;
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < total;
       n += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = n / vol;
    int64_t r = n - c * vol;
    const int64_t k = r / plane;
    r -= k * plane;
    const int64_t j = r / a.fn[0];
    const int64_t i = r - j * a.fn[0];
    int64_t gi = i + a.flo[0], gj = j + a.flo[1], gk = k + a.flo[2];
    bool valid;
    if (a.wrap) {
      if (a.wrap & 1) gi = wrap_axis(gi, a.dlo[0], a.dn[0]);
      if (a.wrap & 2) gj = wrap_axis(gj, a.dlo[1], a.dn[1]);
      if (a.wrap & 4) gk = wrap_axis(gk, a.dlo[2], a.dn[2]);
      valid = gi >= a.dlo[0] && gi < a.dlo[0] + a.dn[0] && gj >= a.dlo[1] && gj < a.dlo[1] + a.dn[1] &&
              gk >= a.dlo[2] && gk < a.dlo[2] + a.dn[2];
    } else {
      valid = gi >= a.vlo[0] && gi <= a.vhi[0] && gj >= a.vlo[1] && gj <= a.vhi[1] && gk >= a.vlo[2] &&
              gk <= a.vhi[2];
    }
    if (sizeof(T) == 8) {
      uint64_t bits = 0x7FF40000DEADBEEFull;
      if (valid) {
        const int64_t lin = ((c * a.dn[2] + (gk - a.dlo[2])) * a.dn[1] + (gj - a.dlo[1])) * a.dn[0] + (gi - a.dlo[0]);
        const uint64_t h = splitmix64(a.seed ^ (uint64_t)lin);
        const double v = (double)(h >> 11) * 0x1.0p-53;
        bits = (uint64_t)__double_as_longlong(v);
      }
      reinterpret_cast<uint64_t *>(fab)[n] = bits;
    } else {
      uint32_t bits = 0x7F80DEADu;
      if (valid) {
        const int64_t lin = ((c * a.dn[2] + (gk - a.dlo[2])) * a.dn[1] + (gj - a.dlo[1])) * a.dn[0] + (gi - a.dlo[0]);
        const uint64_t h = splitmix64(a.seed ^ (uint64_t)lin);
        const float v = (float)(h >> 40) * 0x1.0p-24f;
        bits = (uint32_t)__float_as_uint(v);
      }
      reinterpret_cast<uint32_t *>(fab)[n] = bits;
    }
  }
}

int grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  return g < 1 ? 1 : (int)g;
}

}  // namespace

extern "C" {

int ghx_device_alloc(int32_t device, size_t bytes, void **out) {
  if (!out) {
    set_error("ghx_device_alloc: null out");
    return GHX_EINVAL;
  }
  Guard g(device);
  cudaError_t e = cudaMalloc(out, bytes ? bytes : 256);
  if (e != cudaSuccess) return fail(e, "ghx_device_alloc");
  return GHX_OK;
}

int ghx_device_free(void *ptr) {
  if (!ptr) return GHX_OK;
  cudaPointerAttributes at;
  int dev = -1;
  if (cudaPointerGetAttributes(&at, ptr) == cudaSuccess) dev = at.device;
  Guard g(dev);
  cudaError_t e = cudaFree(ptr);
  if (e != cudaSuccess) return fail(e, "ghx_device_free");
  return GHX_OK;
}

int ghx_host_alloc(size_t bytes, void **out) {
  if (!out) {
    set_error("ghx_host_alloc: null out");
    return GHX_EINVAL;
  }
  cudaError_t e = cudaHostAlloc(out, bytes ? bytes : 256, cudaHostAllocMapped | cudaHostAllocPortable);
  if (e != cudaSuccess) return fail(e, "ghx_host_alloc");
  return GHX_OK;
}

int ghx_host_free(void *ptr) {
  if (!ptr) return GHX_OK;
  cudaError_t e = cudaFreeHost(ptr);
  if (e != cudaSuccess) return fail(e, "ghx_host_free");
  return GHX_OK;
}

int ghx_memset_u64(void *ptr, uint64_t value, size_t count, void *stream) {
  if (!ptr && count) {
    set_error("ghx_memset_u64: null pointer");
    return GHX_EINVAL;
  }
  if (!count) return GHX_OK;
  cudaPointerAttributes at;
  int dev = -1;
  if (cudaPointerGetAttributes(&at, ptr) == cudaSuccess && at.type == cudaMemoryTypeDevice) dev = at.device;
  Guard g(dev);
  memset_u64_kernel<<<grid_for((int64_t)count), 256, 0, (cudaStream_t)stream>>>((uint64_t *)ptr, value, count);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(e, "ghx_memset_u64");
  return GHX_OK;
}

int ghx_enable_peer_access(int32_t device, int32_t peer) {
  if (device == peer) return GHX_OK;
  int can = 0;
  cudaError_t e = cudaDeviceCanAccessPeer(&can, device, peer);
  if (e != cudaSuccess) return fail(e, "ghx_enable_peer_access");
  if (!can) {
    set_error("ghx_enable_peer_access: no P2P path between devices " + std::to_string(device) + " and " +
              std::to_string(peer));
    return GHX_EINVAL;
  }
  Guard g(device);
  e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return GHX_OK;
  }
  if (e != cudaSuccess) return fail(e, "ghx_enable_peer_access");
  return GHX_OK;
}

int ghx_ipc_get_handle(void *ptr, uint8_t handle[64]) {
  if (!ptr || !handle) {
    set_error("ghx_ipc_get_handle: bad arguments");
    return GHX_EINVAL;
  }
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, ptr);
  if (e != cudaSuccess) return fail(e, "ghx_ipc_get_handle");
  static_assert(sizeof(h) == 64, "ipc handle size");
  std::memcpy(handle, &h, 64);
  return GHX_OK;
}

int ghx_alloc_offset(const void *ptr, uint64_t *offset) {
  // byte offset of ptr inside its cudaMalloc allocation (a CUDA-IPC handle
  // maps the whole allocation, so peers add this offset to the opened base)
  if (!ptr || !offset) {
    set_error("ghx_alloc_offset: bad arguments");
    return GHX_EINVAL;
  }
  using GetRange = int (*)(unsigned long long *, size_t *, unsigned long long);
  static GetRange fn = [] {
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<GetRange>(f);
  }();
  if (!fn) {
    set_error("ghx_alloc_offset: cuMemGetAddressRange unavailable");
    return GHX_ECUDA;
  }
  unsigned long long base = 0;
  size_t size = 0;
  if (fn(&base, &size, (unsigned long long)reinterpret_cast<uintptr_t>(ptr)) != 0) {
    set_error("ghx_alloc_offset: not a device allocation");
    return GHX_EINVAL;
  }
  *offset = (uint64_t)(reinterpret_cast<uintptr_t>(ptr) - base);
  return GHX_OK;
}

int ghx_ipc_open_handle(int32_t device, const uint8_t handle[64], void **out) {
  if (!handle || !out) {
    set_error("ghx_ipc_open_handle: bad arguments");
    return GHX_EINVAL;
  }
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  Guard g(device);
  cudaError_t e = cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return fail(e, "ghx_ipc_open_handle");
  return GHX_OK;
}

int ghx_ipc_close_handle(void *ptr) {
  if (!ptr) return GHX_OK;
  cudaError_t e = cudaIpcCloseMemHandle(ptr);
  if (e != cudaSuccess) return fail(e, "ghx_ipc_close_handle");
  return GHX_OK;
}

int ghx_stream_sync(void *stream) {
  cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) return fail(e, "ghx_stream_sync");
  return GHX_OK;
}

int ghx_signal_barrier(uint64_t *const *flag_ptrs, int32_t rank, int32_t nranks, uint64_t epoch, void *stream) {
  if (!flag_ptrs || nranks < 1 || nranks > 64 || rank < 0 || rank >= nranks) {
    set_error("ghx_signal_barrier: bad arguments (nranks <= 64)");
    return GHX_EINVAL;
  }
  FlagPtrs f;
  std::memset(&f, 0, sizeof(f));
  for (int i = 0; i < nranks; ++i) {
    if (!flag_ptrs[i]) {
      set_error("ghx_signal_barrier: null flag pointer");
      return GHX_EINVAL;
    }
    f.p[i] = flag_ptrs[i];
  }
  static const uint64_t timeout_ns = [] {
    const char *v = std::getenv("GHX_BARRIER_TIMEOUT_S");
    const double sec = v ? std::atof(v) : 30.0;
    return (uint64_t)(sec * 1e9);
  }();
  barrier_kernel<<<1, 64, 0, (cudaStream_t)stream>>>(f, rank, nranks, epoch, timeout_ns);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(e, "ghx_signal_barrier");
  return GHX_OK;
}

static int fill_hash(void *fab, const int64_t fab_box[6], int32_t ncomp, const int64_t valid_box[6],
                     const int64_t domain_box[6], uint64_t seed, int32_t elem_bytes, int32_t wrap, void *stream) {
  if (!fab || !fab_box || !valid_box || !domain_box || ncomp < 1 || (elem_bytes != 4 && elem_bytes != 8)) {
    set_error("ghx_fill_hash: bad arguments");
    return GHX_EINVAL;
  }
  FillArgs a;
  for (int d = 0; d < 3; ++d) {
    a.flo[d] = fab_box[d];
    a.fn[d] = fab_box[3 + d] - fab_box[d] + 1;
    a.vlo[d] = valid_box[d];
    a.vhi[d] = valid_box[3 + d];
    a.dlo[d] = domain_box[d];
    a.dn[d] = domain_box[3 + d] - domain_box[d] + 1;
  }
  a.ncomp = ncomp;
  a.seed = seed;
  a.wrap = wrap;
  const int64_t total = a.fn[0] * a.fn[1] * a.fn[2] * ncomp;
  cudaPointerAttributes at;
  int dev = -1;
  if (cudaPointerGetAttributes(&at, fab) == cudaSuccess && at.type == cudaMemoryTypeDevice) dev = at.device;
  Guard g(dev);
  if (elem_bytes == 8)
    fill_hash_kernel<double><<<grid_for(total), 256, 0, (cudaStream_t)stream>>>((double *)fab, a);
  else
    fill_hash_kernel<float><<<grid_for(total), 256, 0, (cudaStream_t)stream>>>((float *)fab, a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(e, "ghx_fill_hash");
  return GHX_OK;
}

int64_t ghx_barrier_timeouts(void) {
  unsigned int v = 0;
  if (cudaMemcpyFromSymbol(&v, g_barrier_timeouts, sizeof(v)) != cudaSuccess) return -1;
  const int64_t k = ghx::sync_timeouts();
  return k < 0 ? -1 : (int64_t)v + k;
}

int ghx_fill_hash(void *fab, const int64_t fab_box[6], int32_t ncomp, const int64_t valid_box[6],
                  const int64_t domain_box[6], uint64_t seed, int32_t elem_bytes, void *stream) {
  return fill_hash(fab, fab_box, ncomp, valid_box, domain_box, seed, elem_bytes, 0, stream);
}

int ghx_fill_hash_wrapped(void *fab, const int64_t fab_box[6], int32_t ncomp, const int64_t domain_box[6],
                          const int32_t periodic[3], uint64_t seed, int32_t elem_bytes, void *stream) {
  if (!periodic) {
    set_error("ghx_fill_hash_wrapped: null periodic");
    return GHX_EINVAL;
  }
  const int32_t wrap = 8 | (periodic[0] ? 1 : 0) | (periodic[1] ? 2 : 0) | (periodic[2] ? 4 : 0);
  return fill_hash(fab, fab_box, ncomp, domain_box, domain_box, seed, elem_bytes, wrap, stream);
}

}  // extern "C"

// ------------------------------------------------------------ index copy

namespace {

// One thread per (cell, component): rows = {src byte address, dst byte
// address, src component stride, dst component stride} per cell; raw words.
template <class W>
__global__ void index_copy_kernel(const int64_t *__restrict__ rows, int64_t n, int ncomp) {
  const int64_t total = n * ncomp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t cell = i % n, c = i / n;
    const int64_t *r = rows + 4 * cell;
    const W v = *reinterpret_cast<const W *>(r[0] + c * r[2]);
    *reinterpret_cast<W *>(r[1] + c * r[3]) = v;
  }
}

}  // namespace

extern "C" int ghx_index_copy(const int64_t *d_rows, int64_t ncells, int32_t ncomp, int32_t elem_bytes,
                              void *stream) {
  if ((ncells && !d_rows) || ncells < 0 || ncomp < 1 || (elem_bytes != 4 && elem_bytes != 8)) {
    set_error("ghx_index_copy: bad arguments");
    return GHX_EINVAL;
  }
  if (ncells == 0) return GHX_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (ncells * ncomp + 255) / 256;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * 8));
  if (elem_bytes == 8)
    index_copy_kernel<uint64_t><<<blocks, 256, 0, st>>>(d_rows, ncells, ncomp);
  else
    index_copy_kernel<uint32_t><<<blocks, 256, 0, st>>>(d_rows, ncells, ncomp);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(e, "ghx_index_copy");
  return GHX_OK;
}
