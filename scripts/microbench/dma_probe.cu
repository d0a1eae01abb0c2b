// Microbenchmark (not product code): copy-engine (DMA) rate for strided 2-D
// copies between pinned host memory and HBM -- the x-face seam chunks of a
// C2 fab (64 B every 544 B) and face slabs -- to judge a staged e2e path.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dma_probe dma_probe.cu
#include <cuda_runtime.h>

#include <cstdio>

int main() {
  const size_t pitch = 544, bytes = size_t(1) << 30, rows = bytes / pitch;
  char *h, *d;
  cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
  cudaMalloc(&d, bytes);
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (size_t w : {16, 32, 64, 128, 256, 544}) {
    for (int dir = 0; dir < 2; ++dir) {
      float best = 1e9f;
      for (int it = 0; it < 3; ++it) {
        cudaEventRecord(a, s1);
        if (dir == 0)
          cudaMemcpy2DAsync(d, pitch, h, pitch, w, rows, cudaMemcpyHostToDevice, s1);
        else
          cudaMemcpy2DAsync(h, pitch, d, pitch, w, rows, cudaMemcpyDeviceToHost, s1);
        cudaEventRecord(b, s1);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      printf("2-D %s width %4zu B pitch %zu: %8.3f ms  %6.2f GB/s useful  %6.3f G rows/s\n", dir ? "D2H" : "H2D", w,
             pitch, best, rows * w / (best * 1e-3) / 1e9, rows / (best * 1e-3) / 1e9);
    }
  }
  // both directions at once (separate copy engines)
  for (size_t w : {64}) {
    cudaEventRecord(a, s1);
    cudaStreamWaitEvent(s2, a, 0);
    cudaMemcpy2DAsync(d, pitch, h, pitch, w, rows / 2, cudaMemcpyHostToDevice, s1);
    cudaMemcpy2DAsync(h + bytes / 2, pitch, d + bytes / 2, pitch, w, rows / 2, cudaMemcpyDeviceToHost, s2);
    cudaEvent_t c;
    cudaEventCreate(&c);
    cudaEventRecord(c, s2);
    cudaStreamWaitEvent(s1, c, 0);
    cudaEventRecord(b, s1);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("2-D H2D + D2H concurrently, width %zu: %8.3f ms for %zu rows each way (%6.2f GB/s useful per direction)\n",
           w, ms, rows / 2, rows / 2 * w / (ms * 1e-3) / 1e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
