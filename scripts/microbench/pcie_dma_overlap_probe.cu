// Microbenchmark (not product code): can the copy engines move face rows
// over PCIe while the SMs run the request-bound x-seam traffic?  C3-like:
// 8 M row seams (64-B read + 64-B write each, the tile walk's pattern in
// address order) of an 8 GiB pinned buffer, and 0.5 M 1,056-B face rows
// moved host -> device and device -> host with cudaMemcpy2DAsync on two
// other streams (the two directions of a device-staged face exchange).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pcie_dma_overlap_probe pcie_dma_overlap_probe.cu
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

__global__ void seams(char *buf, int64_t nseams) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = t; i < nseams * 2; i += nthr) {
    char *p = buf + (i >> 1) * kPitch + 1024 + (i & 1) * 32;
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

int main() {
  const int64_t seam_bytes = 8ll << 30, nseams = seam_bytes / kPitch - 1;
  const int64_t nrows = 1 << 19, row = 1056, face_bytes = nrows * kPitch;
  char *h, *d, *hf_src, *hf_dst, *df;
  CK(cudaHostAlloc(&h, seam_bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  CK(cudaHostGetDevicePointer((void **)&d, h, 0));
  CK(cudaHostAlloc(&hf_src, face_bytes, cudaHostAllocPortable));
  CK(cudaHostAlloc(&hf_dst, face_bytes, cudaHostAllocPortable));
  CK(cudaMalloc(&df, face_bytes));
  for (int64_t i = 0; i < seam_bytes; i += 4096) h[i] = 1;
  for (int64_t i = 0; i < face_bytes; i += 4096) hf_src[i] = hf_dst[i] = 1;
  cudaStream_t s0, s1, s2;
  CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timed = [&](const char *name, bool do_seams, bool do_h2d, bool do_d2h) {
    float best = 1e30f;
    for (int it = 0; it < 3; ++it) {
      cudaDeviceSynchronize();
      cudaEventRecord(a, 0);
      cudaStreamWaitEvent(s0, a, 0);
      cudaStreamWaitEvent(s1, a, 0);
      cudaStreamWaitEvent(s2, a, 0);
      if (do_seams) seams<<<8, 256, 0, s0>>>(d, nseams);
      // rows of 1,024 B at the C3 pitch (source rows -> device staging, staging -> destination rows)
      if (do_h2d) cudaMemcpy2DAsync(df, row, hf_src, kPitch, 1024, nrows, cudaMemcpyHostToDevice, s1);
      if (do_d2h) cudaMemcpy2DAsync(hf_dst, kPitch, df, row, 1024, nrows, cudaMemcpyDeviceToHost, s2);
      cudaDeviceSynchronize();
      cudaEventRecord(b, 0);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (it > 0 && ms < best) best = ms;
    }
    printf("  %-26s %8.3f ms\n", name, best);
  };
  printf("seams %lld (64-B rmw, 8 CTAs), face rows %lld x 1024 B each way\n", (long long)nseams, (long long)nrows);
  timed("seams alone", true, false, false);
  timed("rows H2D alone", false, true, false);
  timed("rows D2H alone", false, false, true);
  timed("rows H2D + D2H", false, true, true);
  timed("seams + rows H2D + D2H", true, true, true);
  return 0;
}
