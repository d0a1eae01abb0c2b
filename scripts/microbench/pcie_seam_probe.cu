// Microbenchmark (not product code): the FillBoundary e2e access patterns on
// pinned, mapped host memory at the C3 row pitch (1,056 B), over an 8 GiB
// buffer like C3's 9.4 GB of host fabs.  Which costs add, which overlap?
//   seam rd      read every row seam (64 B at the row end, 2 lanes x 32 B)
//   seam wr      write every row seam
//   seam rmw     read the seam, then write it back (what the x exchange needs)
//   seam rd||wr  half the warps read seams of one half of the buffer while
//                the other half write seams of the other half
//   row rd / wr  whole 1,024-B rows (face rows), 32 lanes x 32 B
//   row copy     read a row, write it 1 GiB further (the face exchange)
//   row rd||wr   readers and writers on disjoint halves at the same time
// Each at several grid sizes (the host executors run 8 CTAs).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pcie_seam_probe pcie_seam_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define CK(x)                                                                             \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess) {                                                              \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);     \
      return 1;                                                                           \
    }                                                                                     \
  } while (0)

constexpr int64_t kPitch = 1056;

__device__ __forceinline__ void ld32(const char *p, uint32_t (&w)[8]) {
  asm volatile("ld.global.cg.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
               : "l"(p));
}
__device__ __forceinline__ void st32(char *p, const uint32_t (&w)[8]) {
  asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(w[0]), "r"(w[1]), "r"(w[2]),
               "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
               : "memory");
}

// MODE 0 read, 1 write, 2 read+write same place, 3 half read / half write
// (by warp parity, disjoint buffer halves), 4 copy (read at p, write at p + half)
// ROW: false = 64-B seam at the row end (2 lanes), true = 1,024-B row (32 lanes)
template <int MODE, bool ROW>
__global__ void probe(char *buf, int64_t nrows, unsigned *sink) {
  constexpr int LPS = ROW ? 32 : 2;
  const int64_t lane_g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  const int64_t half = nrows / 2;
  uint32_t acc = 0;
  const int warp = (int)(lane_g >> 5);
  const bool writer = MODE == 1 || (MODE == 3 && (warp & 1));
  const int64_t limit = (MODE == 3 || MODE == 4) ? half : nrows;
  // MODE 3: readers take even warps, writers odd warps; each covers its half
  const int64_t t0 = MODE == 3 ? ((int64_t)(warp >> 1) * 32 + (lane_g & 31)) : lane_g;
  const int64_t step = MODE == 3 ? nthr / 2 : nthr;
  for (int64_t t = t0; t < limit * LPS; t += step) {
    const int64_t r = t / LPS;
    const int part = (int)(t % LPS);
    char *p = buf + (MODE == 3 && writer ? half : 0) * kPitch + r * kPitch + (ROW ? 0 : 1024 - 32) + part * 32;
    uint32_t w[8];
    if (MODE == 0 || MODE == 2 || MODE == 4 || (MODE == 3 && !writer)) {
      ld32(p, w);
      acc ^= w[0] ^ w[7];
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) w[i] = (uint32_t)r;
    }
    if (MODE == 1 || MODE == 2 || (MODE == 3 && writer)) st32(p, w);
    if (MODE == 4) st32(p + half * kPitch, w);
  }
  if (acc == 0x9e3779b9u) atomicAdd(sink, 1u);
}

template <int MODE, bool ROW>
void run(const char *name, char *buf, int64_t nrows, unsigned *sink, int blocks) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int it = 0; it < 3; ++it) {
    cudaEventRecord(e0);
    probe<MODE, ROW><<<blocks, 256>>>(buf, nrows, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (it > 0 && ms < best) best = ms;
  }
  const int64_t n = (MODE == 3 || MODE == 4) ? nrows / 2 : nrows;
  const double per = (MODE == 2 || MODE == 4) ? 2.0 : 1.0;  // requests per row
  const double bytes = ROW ? 1024.0 : 64.0;
  const double reqs = (MODE == 3 ? 2.0 * n : n * per);
  printf("  %-12s blocks %5d  %9.3f ms  %6.3f G req/s  %6.2f GB/s moved\n", name, blocks, best,
         reqs / (best * 1e-3) * 1e-9, reqs * bytes / (best * 1e-3) * 1e-9);
}

int main() {
  const int64_t bytes = 8ll << 30;
  const int64_t nrows = bytes / kPitch - 1;
  char *h, *d;
  unsigned *sink;
  CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  CK(cudaHostGetDevicePointer((void **)&d, h, 0));
  CK(cudaMalloc(&sink, 4));
  for (int64_t i = 0; i < bytes; i += 4096) h[i] = 1;
  printf("pinned mapped host, pitch %lld, %lld rows over %lld GiB\n", (long long)kPitch, (long long)nrows,
         (long long)(bytes >> 30));
  for (int blocks : {8, 32, 148, 1184}) {
    run<0, false>("seam rd", d, nrows, sink, blocks);
    run<1, false>("seam wr", d, nrows, sink, blocks);
    run<2, false>("seam rmw", d, nrows, sink, blocks);
    run<3, false>("seam rd||wr", d, nrows, sink, blocks);
  }
  const int64_t frows = nrows / 8;  // face rows: 1 GiB worth
  for (int blocks : {8, 32, 148}) {
    run<0, true>("row rd", d, frows, sink, blocks);
    run<1, true>("row wr", d, frows, sink, blocks);
    run<4, true>("row copy", d, frows, sink, blocks);
    run<3, true>("row rd||wr", d, frows, sink, blocks);
  }
  return 0;
}
