// Microbenchmark (not product code): how fast can a B200 move isolated
// 32-byte sectors that sit at a 1056-byte stride (the x-face ghost pattern of
// a 132-wide float64 fab row)?  Compares LSU loads/stores of several widths
// and cache flavours with TMA box copies (L2 promotion none / 128B).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sector_probe sector_probe.cu
//   ./sector_probe
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdio>
#include <vector>
#include <cstring>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return 1;                                                                     \
    }                                                                               \
  } while (0)

constexpr int64_t ROW = 1056;  // bytes per fab row (132 doubles)

__global__ void rd_sector(const char *buf, int64_t nrows, int64_t off, unsigned long long *sink, int mode) {
  uint32_t acc = 0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
    const char *p = buf + r * ROW + off;
    uint32_t w[8];
    if (mode == 0)
      asm volatile("ld.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
                   : "l"(p));
    else if (mode == 1)
      asm volatile("ld.global.cg.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
                   : "l"(p));
    else if (mode == 2)
      asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
                   : "l"(p));
    else {  // 16-byte load of the sector's first half
      asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]) : "l"(p));
      w[4] = w[5] = w[6] = w[7] = 0;
    }
    acc ^= w[0] ^ w[1] ^ w[2] ^ w[3] ^ w[4] ^ w[5] ^ w[6] ^ w[7];
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

__global__ void rw_sector(char *buf, int64_t nrows, int64_t off) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
    char *p = buf + r * ROW + off;
    uint32_t w[8];
    asm volatile("ld.global.cg.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
                 : "l"(p));
    w[0] += 1;
    asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(w[0]), "r"(w[1]), "r"(w[2]),
                 "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
                 : "memory");
  }
}

__global__ void wr_sector(char *buf, int64_t nrows, int64_t off, int mode) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
    char *p = buf + r * ROW + off;
    const uint32_t v = (uint32_t)r;
    if (mode == 0)
      asm volatile("st.global.v8.u32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p), "r"(v) : "memory");
    else if (mode == 1)
      asm volatile("st.global.wt.v8.u32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p), "r"(v) : "memory");
    else if (mode == 2)
      asm volatile("st.global.cs.v8.u32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p), "r"(v) : "memory");
    else if (mode == 3)
      asm volatile("st.global.v4.u32 [%0], {%1,%1,%1,%1};" ::"l"(p), "r"(v) : "memory");
    else if (mode == 4) {  // full 128-byte line (8 x 16B from 8 consecutive... one lane writes 4 x 32B)
      char *q = buf + r * 128;
      for (int i = 0; i < 4; ++i)
        asm volatile("st.global.v8.u32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(q + 32 * i), "r"(v) : "memory");
    } else if (mode == 5)
      asm volatile("st.global.L1::no_allocate.v8.u32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p), "r"(v) : "memory");
  }
}

__global__ void copy_dense(const uint4 *a, uint4 *b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

// TMA: 2-D tensor (inner: 132 doubles per row, outer: rows); box = 4 x BOXR
template <int BOXR>
__global__ void tma_rd(const __grid_constant__ CUtensorMap map, int64_t nboxes, int x0, unsigned long long *sink,
                       int write_back) {
  __shared__ alignas(128) double tile[BOXR * 4];
  __shared__ alignas(8) uint64_t bar;
  const uint32_t sbar = (uint32_t)__cvta_generic_to_shared(&bar);
  const uint32_t stile = (uint32_t)__cvta_generic_to_shared(tile);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(sbar));
    asm volatile("fence.proxy.async.shared::cta;");
  }
  __syncthreads();
  uint32_t phase = 0;
  double acc = 0;
  for (int64_t b = blockIdx.x; b < nboxes; b += gridDim.x) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(sbar), "r"(BOXR * 32));
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              stile),
          "l"(&map), "r"(x0), "r"((int)(b * BOXR)), "r"(sbar)
          : "memory");
    }
    // wait
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(sbar), "r"(phase));
    }
    phase ^= 1;
    acc += tile[threadIdx.x % (BOXR * 4)];
    if (write_back && threadIdx.x == 0) {
      asm volatile("fence.proxy.async.shared::cta;");
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&map), "r"(x0),
                   "r"((int)(b * BOXR)), "r"(stile)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;");
      asm volatile("cp.async.bulk.wait_group.read 0;");
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;");
  if (acc == 1234.5) atomicAdd(sink, 1ull);
}

int main() {
  const int64_t nrows = (8ll << 30) / ROW;  // ~8 GiB
  char *buf, *buf2;
  unsigned long long *sink;
  CK(cudaMalloc(&buf, nrows * ROW));
  CK(cudaMalloc(&buf2, nrows * ROW));
  CK(cudaMalloc(&sink, 8));
  CK(cudaMemset(buf, 1, nrows * ROW));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto timeit = [&](auto fn, int reps) {
    fn();
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) fn();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / reps;
  };
  const double sectors = (double)nrows;
  {
    size_t g = 0;
    cudaDeviceGetLimit(&g, cudaLimitMaxL2FetchGranularity);
    printf("default cudaLimitMaxL2FetchGranularity = %zu\n", g);
    for (size_t want : {32, 64, 128}) {
      cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, want);
      cudaDeviceGetLimit(&g, cudaLimitMaxL2FetchGranularity);
      float ms = timeit([&] { rd_sector<<<sms * 16, 256>>>(buf, nrows, 0, sink, 1); }, 5);
      printf("L2 fetch granularity set %zu (%s) -> %zu: isolated sector read %.3f ms %.1f GB/s useful\n", want,
             cudaGetErrorString(e), g, ms, sectors * 32 / ms / 1e6);
    }
  }
  const char *names[] = {"ld.v8 (default)", "ld.cg.v8", "ld.nc.na.v8", "ld.v4 (16B)"};
  for (int mode = 0; mode < 4; ++mode)
    for (int occ : {8, 16, 32}) {
      float ms = timeit([&] { rd_sector<<<sms * occ, 256>>>(buf, nrows, 0, sink, mode); }, 5);
      printf("read isolated sector  %-16s blocks/SM=%2d: %.3f ms  %.1f GB/s useful(32B)  %.1f Gsector/s\n",
             names[mode], occ, ms, sectors * 32 / ms / 1e6, sectors / ms / 1e6);
    }
  {
    float ms = timeit([&] { rd_sector<<<sms * 16, 256>>>(buf, nrows, 1024, sink, 1); }, 5);
    printf("read isolated sector  ld.cg.v8 off=1024: %.3f ms  %.1f GB/s\n", ms, sectors * 32 / ms / 1e6);
  }
  {
    float ms = timeit([&] { rw_sector<<<sms * 16, 256>>>(buf, nrows, 0); }, 5);
    printf("read+write sector     ld.cg/st.v8:       %.3f ms  %.1f GB/s useful(64B/row)\n", ms,
           sectors * 64 / ms / 1e6);
  }
  {
    const int64_t n = nrows * ROW / 16;
    float ms = timeit([&] { copy_dense<<<sms * 8, 256>>>((const uint4 *)buf, (uint4 *)buf2, n); }, 5);
    printf("dense copy:                               %.3f ms  %.1f GB/s (r+w)\n", ms, 2.0 * n * 16 / ms / 1e6);
  }
  // pinned host memory (zero-copy over PCIe)
  {
    const int64_t hrows = (1ll << 30) / ROW;  // 1 GiB
    char *h;
    CK(cudaHostAlloc(&h, hrows * ROW, cudaHostAllocMapped));
    memset(h, 1, hrows * ROW);
    char *hd;
    CK(cudaHostGetDevicePointer(&hd, h, 0));
    for (int64_t off : {0, 1024}) {
      float ms = timeit([&] { rd_sector<<<sms * 16, 256>>>(hd, hrows, off, sink, 1); }, 3);
      printf("HOST read isolated 32B sector off=%ld: %.3f ms  %.2f GB/s useful\n", (long)off, ms, hrows * 32.0 / ms / 1e6);
    }
    {
      float ms = timeit([&] { rd_sector<<<sms * 16, 256>>>(hd, hrows, 0, sink, 3); }, 3);
      printf("HOST read isolated 16B: %.3f ms  %.2f GB/s useful\n", ms, hrows * 16.0 / ms / 1e6);
    }
    {
      float ms = timeit([&] { rw_sector<<<sms * 16, 256>>>(hd, hrows, 0); }, 3);
      printf("HOST read+write isolated 32B sector: %.3f ms  %.2f GB/s useful (64B/row)\n", ms, hrows * 64.0 / ms / 1e6);
    }
    const char *wn[] = {"st.v8", "st.wt.v8", "st.cs.v8", "st.v4 (16B)", "full 128B lines (contiguous)", "st.na.v8"};
    for (int m = 0; m < 6; ++m) {
      const int64_t rows = m == 4 ? (hrows * ROW / 128) : hrows;
      float ms = timeit([&] { wr_sector<<<sms * 16, 256>>>(hd, rows, 0, m); }, 3);
      const double useful = m == 4 ? 128.0 : (m == 3 ? 16.0 : 32.0);
      printf("HOST write isolated %-28s: %.3f ms  %.2f GB/s useful  %.3f G writes/s\n", wn[m], ms,
             rows * useful / ms / 1e6, rows / ms / 1e6);
    }
    {
      const int64_t n = hrows * ROW / 16;
      float ms = timeit([&] { copy_dense<<<sms * 8, 256>>>((const uint4 *)hd, (uint4 *)buf2, n); }, 3);
      printf("HOST->DEV dense read: %.3f ms  %.2f GB/s\n", ms, n * 16.0 / ms / 1e6);
      ms = timeit([&] { copy_dense<<<sms * 8, 256>>>((const uint4 *)buf2, (uint4 *)hd, n); }, 3);
      printf("DEV->HOST dense write: %.3f ms  %.2f GB/s\n", ms, n * 16.0 / ms / 1e6);
      ms = timeit([&] { cudaMemcpyAsync(buf2, h, n * 16, cudaMemcpyHostToDevice); }, 3);
      printf("cudaMemcpy H2D: %.3f ms  %.2f GB/s\n", ms, n * 16.0 / ms / 1e6);
    }
    cudaFreeHost(h);
  }
  // TMA
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q));
  for (int prom = 0; prom < 2; ++prom)
    for (int wb = 0; wb < 2; ++wb) {
      CUtensorMap map;
      cuuint64_t dims[2] = {132, (cuuint64_t)nrows};
      cuuint64_t strides[1] = {ROW};
      cuuint32_t box[2] = {4, 256};
      cuuint32_t es[2] = {1, 1};
      CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, buf, dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                       prom ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) {
        printf("encode failed %d\n", (int)r);
        continue;
      }
      const int64_t nboxes = nrows / 256;
      for (int occ : {8, 16}) {
        float ms = timeit([&] { tma_rd<256><<<sms * occ, 128>>>(map, nboxes, 0, sink, wb); }, 5);
        printf("TMA box 4x256 promo=%s %s blocks/SM=%d: %.3f ms  %.1f GB/s useful\n", prom ? "128B" : "none",
               wb ? "read+write" : "read", occ, ms, nboxes * 256.0 * 32 * (wb ? 2 : 1) / ms / 1e6);
      }
    }
  CK(cudaGetLastError());
  return 0;
}
