// Microbenchmark (not product code): isolated accesses to pinned, mapped host
// memory from a B200 kernel, at the 544-byte row stride of a C2 fab.  How
// does the access rate depend on the access size (16/32/64/128 B per seam)
// and on how the bytes are split over lanes?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pcie_probe pcie_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <sys/mman.h>

#define CK(x)                                                                             \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess) {                                                              \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);     \
      return 1;                                                                           \
    }                                                                                     \
  } while (0)

// LPS lanes cooperate on one access of BYTES bytes (each lane BYTES/LPS, 16 or 32 B)
__device__ int64_t g_perm_mul = 1;  // 1: sequential seams; large odd: scattered order

template <int BYTES, int LPS, bool WRITE, int PF = 0>
__global__ void probe(char *buf, int64_t n, int64_t stride, unsigned *sink) {
  const int64_t pm = g_perm_mul;
  constexpr int PER = BYTES / LPS;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  uint32_t acc = 0;
  for (int64_t t = tid; t < n * LPS; t += nthr) {
    const int64_t s = (int64_t)(((unsigned __int128)(t / LPS) * (uint64_t)pm) % (uint64_t)n);
    const int part = (int)(t % LPS);
    char *p = buf + s * stride + part * PER;
    if (WRITE) {
      if (PER >= 32)
        for (int i = 0; i < PER; i += 32)
          asm volatile("st.global.v8.u32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p + i), "r"((uint32_t)s) : "memory");
      else
        asm volatile("st.global.v4.u32 [%0], {%1,%1,%1,%1};" ::"l"(p), "r"((uint32_t)s) : "memory");
    } else {
      if (PER >= 32) {
        for (int i = 0; i < PER; i += 32) {
          uint32_t w[8];
          if (PF == 0) asm volatile("ld.global.cg.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                       : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
                       : "l"(p + i));
          else if (PF == 1) asm volatile("ld.global.cg.L2::64B.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                       : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
                       : "l"(p + i));
          else asm volatile("ld.global.cg.L2::128B.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                       : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
                       : "l"(p + i));
          acc ^= w[0] ^ w[7];
        }
      } else {
        uint4 v;
        if (PF == 0) asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
        else if (PF == 1) asm volatile("ld.global.cg.L2::64B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
        else asm volatile("ld.global.cg.L2::128B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
        acc ^= v.x ^ v.w;
      }
    }
  }
  if (acc == 0x9e3779b9u) atomicAdd(sink, 1u);
}

template <int BYTES, int LPS, bool WRITE, int PF = 0>
void run(const char *name, char *buf, int64_t n, int64_t stride, unsigned *sink) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int it = 0; it < 4; ++it) {
    cudaEventRecord(e0);
    probe<BYTES, LPS, WRITE, PF><<<148 * 8, 256>>>(buf, n, stride, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (it > 0 && ms < best) best = ms;
  }
  printf("  %-28s %8.3f ms  %6.3f G acc/s  %6.2f GB/s useful\n", name, best, n / (best * 1e-3) * 1e-9,
         n * (double)BYTES / (best * 1e-3) * 1e-9);
}

int main(int argc, char **argv) {
  const int64_t stride = 544;
  const bool wc = argc > 1 && argv[1][0] == 'w';
  const bool huge = argc > 1 && argv[1][0] == 'h';
  const int64_t bytes = 1ll << 30;
  const int64_t n = bytes / stride - 1;
  char *h, *d;
  unsigned *sink;
  if (huge) {  // 2 MiB-aligned anonymous memory with transparent huge pages, then registered
    h = (char *)mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (h == MAP_FAILED) { printf("mmap failed\n"); return 1; }
    printf("madvise(MADV_HUGEPAGE) rc=%d\n", madvise(h, bytes, MADV_HUGEPAGE));
    for (int64_t i = 0; i < bytes; i += 4096) h[i] = 1;
    CK(cudaHostRegister(h, bytes, cudaHostRegisterMapped));
  } else {
    CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped | (wc ? cudaHostAllocWriteCombined : 0)));
  }
  CK(cudaHostGetDevicePointer((void **)&d, h, 0));
  CK(cudaMalloc(&sink, 4));
  for (int64_t i = 0; i < bytes; i += 4096) h[i] = 1;
  printf("%s pinned mapped host, stride", wc ? "write-combined" : huge ? "THP-registered" : "cached");
  printf(" %lld, %lld accesses\n", (long long)stride, (long long)n);
  run<16, 1, false>("read 16B", d, n, stride, sink);
  run<32, 1, false>("read 32B", d, n, stride, sink);
  run<64, 1, false>("read 64B (1 lane 2x32)", d, n, stride, sink);
  run<64, 2, false>("read 64B (2 lanes x32)", d, n, stride, sink);
  run<128, 4, false>("read 128B (4 lanes x32)", d, n, stride, sink);
  run<256, 8, false>("read 256B (8 lanes x32)", d, n, stride, sink);
  run<16, 1, false, 1>("read 16B L2::64B", d, n, stride, sink);
  run<16, 1, false, 2>("read 16B L2::128B", d, n, stride, sink);
  run<32, 1, false, 1>("read 32B L2::64B", d, n, stride, sink);
  run<32, 1, false, 2>("read 32B L2::128B", d, n, stride, sink);
  run<64, 2, false, 1>("read 64B (2x32) L2::64B", d, n, stride, sink);
  run<64, 2, false, 2>("read 64B (2x32) L2::128B", d, n, stride, sink);
  run<128, 4, false, 2>("read 128B (4x32) L2::128B", d, n, stride, sink);
  run<16, 1, true>("write 16B", d, n, stride, sink);
  run<32, 1, true>("write 32B", d, n, stride, sink);
  run<64, 1, true>("write 64B (1 lane 2x32)", d, n, stride, sink);
  run<64, 2, true>("write 64B (2 lanes x32)", d, n, stride, sink);
  run<128, 4, true>("write 128B (4 lanes x32)", d, n, stride, sink);
  run<256, 8, true>("write 256B (8 lanes x32)", d, n, stride, sink);
  run<512, 16, true>("write 512B (16 lanes x32)", d, n, stride, sink);
  run<512, 16, false>("read 512B (16 lanes x32)", d, n, stride, sink);
  int64_t pm = 1000003;  // coprime with n: a scattered permutation of the seams
  cudaMemcpyToSymbol(g_perm_mul, &pm, sizeof(pm));
  printf("scattered order (seam i -> i * %lld mod n)\n", (long long)pm);
  run<32, 1, false>("read 32B", d, n, stride, sink);
  run<64, 2, false>("read 64B (2 lanes x32)", d, n, stride, sink);
  run<32, 1, true>("write 32B", d, n, stride, sink);
  run<64, 2, true>("write 64B (2 lanes x32)", d, n, stride, sink);
  run<512, 16, false>("read 512B (16 lanes x32)", d, n, stride, sink);
  CK(cudaGetLastError());
  return 0;
}
