// Microbenchmark (not product code): do the x-face row seams (one 64-B
// read + write per seam, latency/DRAM-service bound) and the y/z face rows
// (1-KB streaming copies) overlap in HBM when they run at the SAME time on
// different warps?  C3 geometry in device memory: 64 fabs x 1,056 (z, comp)
// planes x 132 rows of 1,056 B (9.4 GB), 8.65 M seams; face rows: 0.5 M
// 1,024-B rows copied between two other 0.55 GB regions.
//   S   seams alone (every warp)            R   rows alone (every warp)
//   S+R one kernel, half the warps on seams and half on rows (warp
//       specialised: warp w takes seams if w is even), then each side steals
//       the other's remaining work when it runs out
//   S|R two kernels on two streams at once (1 CTA/SM each)
// L2 flushed before every launch.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o seam_row_overlap_probe seam_row_overlap_probe.cu
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
constexpr int64_t kFab = kPlane * kPlanes, kFabs = 64;
constexpr int64_t kSeams = kFabs * kPlanes * 128;
constexpr int64_t kFaceRows = 1 << 19, kRowBytes = 1024;

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

// seam unit u (16 seams of one plane, lane pair = seam, 32 B per lane)
__device__ __forceinline__ void seam_unit(char *buf, int64_t u, int lane) {
  const int64_t s = u * 16 + (lane >> 1);
  if (s >= kSeams) return;
  const int64_t row = s % 128, plane = (s / 128) % kPlanes, fab = s / (128 * kPlanes);
  char *p = buf + fab * kFab + plane * kPlane + (row + 2) * kPitch - 32 + (lane & 1) * 32;
  uint32_t w[8];
  ld32(p, w);
  w[0] += 1;
  st32(p, w);
}

// row unit u (4 face rows of 1 KB: 32 B per lane per row, rows at the C3 pitch)
__device__ __forceinline__ void row_unit(const char *src, char *dst, int64_t u, int lane) {
  uint32_t w[4][8];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int64_t r = u * 4 + k;
    if (r < kFaceRows) ld32(src + r * kPitch + lane * 32, w[k]);
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int64_t r = u * 4 + k;
    if (r < kFaceRows) st32(dst + r * kPitch + lane * 32, w[k]);
  }
}

constexpr int64_t kSeamUnits = (kSeams + 15) / 16, kRowUnits = (kFaceRows + 3) / 4;

// MODE 0 seams only, 1 rows only, 2 warp-specialised both (with stealing)
template <int MODE>
__global__ void __launch_bounds__(256, 2) work(char *buf, const char *src, char *dst, unsigned long long *ctr) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const bool seams_first = MODE == 0 || (MODE == 2 && (warp & 1) == 0);
  for (int side = 0; side < (MODE == 2 ? 2 : 1); ++side) {
    const bool do_seams = side == 0 ? seams_first : !seams_first;
    const int64_t n = do_seams ? kSeamUnits : kRowUnits;
    unsigned long long *c = ctr + (do_seams ? 0 : 1);
    while (true) {
      unsigned long long u = 0;
      if (lane == 0) u = atomicAdd(c, 8ull);
      u = __shfl_sync(0xffffffffu, u, 0);
      if ((int64_t)u >= n) break;
      for (int k = 0; k < 8 && (int64_t)(u + k) < n; ++k) {
        if (do_seams)
          seam_unit(buf, u + k, lane);
        else
          row_unit(src, dst, u + k, lane);
      }
    }
  }
}

__global__ void flush(uint4 *f, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    f[i] = make_uint4((uint32_t)i, 0, 0, 0);
}

int main() {
  char *buf, *src, *dst;
  uint4 *fl;
  unsigned long long *ctr;
  const int64_t fln = (1ll << 29) / 16;
  CK(cudaMalloc(&buf, kFab * kFabs));
  CK(cudaMalloc(&src, kFaceRows * kPitch));
  CK(cudaMalloc(&dst, kFaceRows * kPitch));
  CK(cudaMalloc(&fl, fln * 16));
  CK(cudaMalloc(&ctr, 4 * sizeof(unsigned long long)));
  CK(cudaMemset(buf, 0, kFab * kFabs));
  CK(cudaMemset(src, 1, kFaceRows * kPitch));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timed = [&](const char *name, int mode) {
    float best = 1e30f;
    for (int it = 0; it < 5; ++it) {
      cudaMemset(ctr, 0, 4 * sizeof(unsigned long long));
      flush<<<sms * 8, 256>>>(fl, fln);
      cudaDeviceSynchronize();
      cudaEventRecord(e0, 0);
      if (mode == 0) work<0><<<sms * 2, 256>>>(buf, src, dst, ctr);
      if (mode == 1) work<1><<<sms * 2, 256>>>(buf, src, dst, ctr);
      if (mode == 2) work<2><<<sms * 2, 256>>>(buf, src, dst, ctr);
      if (mode == 3) {  // two kernels at once, one CTA per SM each
        cudaStreamWaitEvent(s1, e0, 0);
        cudaStreamWaitEvent(s2, e0, 0);
        work<0><<<sms, 256, 0, s1>>>(buf, src, dst, ctr);
        work<1><<<sms, 256, 0, s2>>>(buf, src, dst, ctr + 2);
        cudaEvent_t j1, j2;
        cudaEventCreate(&j1);
        cudaEventCreate(&j2);
        cudaEventRecord(j1, s1);
        cudaEventRecord(j2, s2);
        cudaStreamWaitEvent(0, j1, 0);
        cudaStreamWaitEvent(0, j2, 0);
      }
      cudaEventRecord(e1, 0);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (it > 0 && ms < best) best = ms;
    }
    printf("  %-34s %8.3f ms\n", name, best);
  };
  printf("C3 geometry: %lld seams (64-B rmw), %lld face rows of %lld B copied\n", (long long)kSeams,
         (long long)kFaceRows, (long long)kRowBytes);
  timed("S   seams alone", 0);
  timed("R   rows alone", 1);
  timed("S+R warp-specialised, one kernel", 2);
  timed("S|R two kernels, two streams", 3);
  return 0;
}
