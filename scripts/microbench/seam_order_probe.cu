// Microbenchmark (not product code): does the ORDER in which the x-face row
// seams are visited change their HBM cost?  C3 geometry in device memory
// (64 fabs x 1,056 (z, comp) planes x 132 rows of 1,056 B = 9.4 GB); every
// seam is read (64 B) and written back (64 B), the x exchange's minimum.
//   O0 row order       consecutive threads -> consecutive rows of one plane
//   O1 plane order     consecutive threads -> the same row of consecutive planes (139 KB apart)
//   O2 fab order       consecutive threads -> the same row of different fabs (147 MB apart)
//   O3 scattered       a multiplicative permutation of all seams
//   O4 row pairs       one thread = two consecutive rows (two seams 1,056 B apart)
// L2 flushed (1 GiB write) before every launch.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o seam_order_probe seam_order_probe.cu
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

constexpr int64_t kPitch = 1056, kRows = 132, kPlane = kPitch * kRows, kPlanes = 132 * 8;
constexpr int64_t kFab = kPlane * kPlanes;
constexpr int64_t kFabs = 64, kSeams = kFabs * kPlanes * 128;

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

template <int ORDER>
__device__ __forceinline__ char *seam_of(char *buf, int64_t s) {
  int64_t fab, plane, row;
  if (ORDER == 0 || ORDER == 4) {
    row = s % 128;
    plane = (s / 128) % kPlanes;
    fab = s / (128 * kPlanes);
  } else if (ORDER == 1) {
    plane = s % kPlanes;
    row = (s / kPlanes) % 128;
    fab = s / (128 * kPlanes);
  } else if (ORDER == 2) {
    fab = s % kFabs;
    row = (s / kFabs) % 128;
    plane = s / (kFabs * 128);
  } else {
    const int64_t q = (int64_t)(((unsigned __int128)s * 2654435761ull) % (uint64_t)kSeams);
    row = q % 128;
    plane = (q / 128) % kPlanes;
    fab = q / (128 * kPlanes);
  }
  return buf + fab * kFab + plane * kPlane + (row + 2) * kPitch - 32;
}

// lane pair = one 64-B seam chunk (32 B per lane), U chunks in flight per pair
template <int ORDER, int U>
__global__ void seam_rmw(char *buf) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t npairs = ((int64_t)gridDim.x * blockDim.x) >> 1;
  const int side = (int)(t & 1);
  const int64_t pair = t >> 1;
  const int64_t per = ORDER == 4 ? 2 : 1;
  for (int64_t s0 = pair * per; s0 < kSeams; s0 += npairs * U) {
    uint32_t w[U][8];
    char *p[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t s = ORDER == 4 ? s0 + (u & 1) + (u >> 1) * npairs * 2 : s0 + u * npairs;
      p[u] = s < kSeams ? seam_of<ORDER>(buf, s) + side * 32 : nullptr;
      if (p[u]) ld32(p[u], w[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (p[u]) {
        w[u][0] += 1;
        st32(p[u], w[u]);
      }
  }
}

__global__ void flush(uint4 *f, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    f[i] = make_uint4((uint32_t)i, 0, 0, 0);
}

template <int ORDER, int U>
void run(const char *name, char *buf, uint4 *fl, int64_t fln, int blocks) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int it = 0; it < 4; ++it) {
    flush<<<148 * 8, 256>>>(fl, fln);
    cudaEventRecord(e0);
    seam_rmw<ORDER, U><<<blocks, 256>>>(buf);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (it > 0 && ms < best) best = ms;
  }
  printf("  %-12s U=%d blocks %5d  %8.3f ms  %6.2f G seams/s\n", name, U, blocks, best, kSeams / (best * 1e-3) * 1e-9);
}

int main() {
  char *buf;
  uint4 *fl;
  const int64_t fln = (1ll << 30) / 16;
  CK(cudaMalloc(&buf, kFab * kFabs));
  CK(cudaMalloc(&fl, fln * 16));
  CK(cudaMemset(buf, 0, kFab * kFabs));
  printf("device: %lld seams (C3 x faces), pitch %lld\n", (long long)kSeams, (long long)kPitch);
  for (int blocks : {296, 1184}) {
    run<0, 2>("row order", buf, fl, fln, blocks);
    run<1, 2>("plane order", buf, fl, fln, blocks);
    run<2, 2>("fab order", buf, fl, fln, blocks);
    run<3, 2>("scattered", buf, fl, fln, blocks);
    run<4, 2>("row pairs", buf, fl, fln, blocks);
    run<0, 4>("row order", buf, fl, fln, blocks);
    run<4, 4>("row pairs", buf, fl, fln, blocks);
  }
  return 0;
}
