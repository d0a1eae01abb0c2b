// Microbenchmark (not product code): cost of the x-face "row seam" pattern.
// A float64 fab row of nx cells is ROW = 8*nx bytes; with 2 ghosts the end of
// row r and the start of row r+1 form one 64-byte chunk
//   [hi valid | hi ghost][lo ghost | lo valid]   (32-byte aligned)
// that FillBoundary reads half of and rewrites half of.  Variants:
//   rd16x2     read the two 16-byte valid halves only
//   rd64       read the 64-byte chunk
//   rdline     read every 128-byte line the chunk touches
//   wr64       write the 64-byte chunk (2 full sectors)
//   wrline     write every touched line whole
//   swap       read 2x16 B, write 2x32 B            (the v3 sector swap)
//   rmw64      read 64 B, write 64 B
//   rmwline    read the touched lines, write them back whole
// Usage: seam_probe [row_bytes=544] [unroll]
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess) {                                                                   \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);          \
      return 1;                                                                                \
    }                                                                                          \
  } while (0)

struct V8 {
  uint32_t w[8];
};
__device__ __forceinline__ V8 ld32(const char *p) {
  V8 r;
  asm volatile("ld.global.cg.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]), "=r"(r.w[6]),
                 "=r"(r.w[7])
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ld16(const char *p) {
  uint4 r;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void st32(char *p, const V8 &v) {
  asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v.w[0]), "r"(v.w[1]), "r"(v.w[2]),
               "r"(v.w[3]), "r"(v.w[4]), "r"(v.w[5]), "r"(v.w[6]), "r"(v.w[7])
               : "memory");
}

// one thread per seam, U seams in flight per thread (grid-stride over groups)
template <int MODE, int U>
__global__ void __launch_bounds__(256) seam_kernel(char *buf, int64_t nseams, int64_t row, unsigned *sink) {
  uint32_t acc = 0;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  for (int64_t s0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s0 < nseams; s0 += nthr * U) {
    V8 a[U], b[U], c[U], d[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t s = s0 + u * nthr;
      if (s >= nseams) continue;
      char *p = buf + (s + 1) * row - 32;  // 64-byte chunk start
      if (MODE == 0 || MODE == 5) {        // rd16x2 / swap
        uint4 x = ld16(p), y = ld16(p + 48);
        a[u].w[0] = x.x; a[u].w[1] = x.y; a[u].w[2] = x.z; a[u].w[3] = x.w;
        a[u].w[4] = y.x; a[u].w[5] = y.y; a[u].w[6] = y.z; a[u].w[7] = y.w;
      } else if (MODE == 1 || MODE == 6) {  // rd64 / rmw64
        a[u] = ld32(p);
        b[u] = ld32(p + 32);
      } else if (MODE == 2 || MODE == 7) {  // rdline / rmwline: 128-byte line of the chunk start
        char *l = (char *)((uintptr_t)p & ~(uintptr_t)127);
        a[u] = ld32(l);
        b[u] = ld32(l + 32);
        c[u] = ld32(l + 64);
        d[u] = ld32(l + 96);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t s = s0 + u * nthr;
      if (s >= nseams) continue;
      char *p = buf + (s + 1) * row - 32;
      if (MODE <= 2) {
        acc ^= a[u].w[0] ^ a[u].w[7];
        if (MODE >= 1) acc ^= b[u].w[3];
        if (MODE == 2) acc ^= c[u].w[1] ^ d[u].w[2];
      } else if (MODE == 3) {  // wr64
        V8 v;
        for (int i = 0; i < 8; ++i) v.w[i] = (uint32_t)s;
        st32(p, v);
        st32(p + 32, v);
      } else if (MODE == 4) {  // wrline
        V8 v;
        for (int i = 0; i < 8; ++i) v.w[i] = (uint32_t)s;
        char *l = (char *)((uintptr_t)p & ~(uintptr_t)127);
        st32(l, v); st32(l + 32, v); st32(l + 64, v); st32(l + 96, v);
      } else if (MODE == 5) {  // swap: write both sectors whole
        st32(p, a[u]);
        st32(p + 32, a[u]);
      } else if (MODE == 6) {
        st32(p, b[u]);
        st32(p + 32, a[u]);
      } else if (MODE == 7) {
        char *l = (char *)((uintptr_t)p & ~(uintptr_t)127);
        st32(l, a[u]); st32(l + 32, b[u]); st32(l + 64, c[u]); st32(l + 96, d[u]);
      }
    }
  }
  if (acc == 0x9e3779b9u) atomicAdd(sink, 1u);
}

__global__ void flush_kernel(uint4 *f, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    f[i] = make_uint4((uint32_t)i, 0, 0, 0);
}

template <int MODE, int U>
float run(char *buf, int64_t nseams, int64_t row, unsigned *sink, uint4 *fl, int64_t fln, int blocks) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int it = 0; it < 6; ++it) {
    flush_kernel<<<148 * 8, 256>>>(fl, fln);
    cudaEventRecord(e0);
    seam_kernel<MODE, U><<<blocks, 256>>>(buf, nseams, row, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (it > 0 && ms < best) best = ms;
  }
  return best;
}

int main(int argc, char **argv) {
  const int64_t row = argc > 1 ? atoll(argv[1]) : 544;
  const int64_t bytes = 4ll << 30;
  const int64_t nseams = bytes / row - 2;
  char *buf;
  unsigned *sink;
  uint4 *fl;
  const int64_t fln = (512ll << 20) / 16;
  CK(cudaMalloc(&buf, bytes));
  CK(cudaMalloc(&sink, 4));
  CK(cudaMalloc(&fl, fln * 16));
  CK(cudaMemset(buf, 1, bytes));
  const char *names[] = {"rd16x2", "rd64", "rdline", "wr64", "wrline", "swap", "rmw64", "rmwline"};
  // useful bytes per seam: the FillBoundary algorithmic bytes (32 read + 32 written)
  for (int occ : {4, 8}) {
    const int blocks = 148 * occ;
    printf("row=%lld seams=%lld blocks=%d\n", (long long)row, (long long)nseams, blocks);
    for (int m = 0; m < 8; ++m) {
      float ms1 = 0, ms4 = 0;
#define CASE(M)                                                  \
  case M:                                                        \
    ms1 = run<M, 1>(buf, nseams, row, sink, fl, fln, blocks);    \
    ms4 = run<M, 4>(buf, nseams, row, sink, fl, fln, blocks);    \
    break;
      switch (m) { CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) }
      const double g1 = nseams * 1e-9 / (ms1 * 1e-3), g4 = nseams * 1e-9 / (ms4 * 1e-3);
      printf("  %-8s U=1 %8.3f ms %6.2f Gseam/s (%7.1f GB/s alg) | U=4 %8.3f ms %6.2f Gseam/s (%7.1f GB/s alg)\n",
             names[m], ms1, g1, g1 * 64, ms4, g4, g4 * 64);
    }
  }
  CK(cudaGetLastError());
  return 0;
}
