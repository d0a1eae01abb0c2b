// Microbenchmark (not product code): the x-seam walk of the host-memory
// FillBoundary (ring tasks) on pinned, mapped host memory.  Every lane pair
// reads a 64-B row seam and writes it back (one read + one write request,
// the x exchange's minimum), walking 16 consecutive rows; what differs is
// which seams the 16 lane pairs of a warp cover at once:
//   ring      4 fabs (147 MB apart) x 4 z-planes (139 KB apart): the current
//             ring task (16 different host pages per warp instruction)
//   rowsegs   4 fabs x 4 consecutive 16-row segments of ONE plane
//   onefab    one fab: 16 consecutive 16-row segments (256 contiguous rows)
//   flat      one seam per lane pair in address order (pcie_probe's rmw)
//   tile      4 fabs x 4 CONSECUTIVE rows per instruction, stepping 4 rows
//   tile-pf / ring-pf  the same with the next step's seam loaded one step ahead
// Geometry of C3: 64 fabs x 8 comps x 132 planes x 132 rows of 1,056 B
// (9.4 GB); the walk covers the 128 valid rows of every plane.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pcie_ring_probe pcie_ring_probe.cu
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
constexpr int64_t kFab = kPlane * kPlanes;  // 147 MB
constexpr int kFabs = 64, kLine = 4;        // x-lines of 4 fabs
constexpr int kSeg = 16;                    // rows per lane-pair walk

__device__ __forceinline__ void rmw(char *p) {
  uint32_t w[8];
  asm volatile("ld.global.cg.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
               : "l"(p));
  w[0] += 1;
  asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(w[0]), "r"(w[1]), "r"(w[2]),
               "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
               : "memory");
}

// seam chunk of (fab, plane, row): last 32 B of the row and first 32 B of the next
__device__ __forceinline__ char *seam(char *buf, int64_t fab, int64_t plane, int64_t row, int side) {
  return buf + fab * kFab + plane * kPlane + row * kPitch + 1024 + side * 32;
}

__device__ __forceinline__ void ld(const char *p, uint32_t (&w)[8]) {
  asm volatile("ld.global.cg.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
               : "l"(p));
}
__device__ __forceinline__ void st(char *p, const uint32_t (&w)[8]) {
  asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(w[0]), "r"(w[1]), "r"(w[2]),
               "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
               : "memory");
}

// MODE 3: tile walk (4 fabs x rows s, s+4, ...: one instruction = 4 consecutive rows of 4 fabs)
// MODE 4: MODE 3 with a one-step-ahead load;  MODE 5: ring layout with a one-step-ahead load
// MODE 6: MODE 4 writing only the 32 ghost bytes [16, 48) of the seam (a
//         16-B store per lane, the two adjacent) instead of the whole 64 B
// MODE 7: MODE 4 writing nothing (reads only, same walk)
template <int MODE>
__global__ void tile_walk(char *buf, int64_t units) {
  const int lane = threadIdx.x & 31, pair = lane >> 1, side = lane & 1;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  constexpr int64_t segs = 128 / kSeg;
  for (int64_t u = warp; u < units; u += nwarps) {
    int64_t fab, plane, row0, dr;
    if (MODE == 5) {
      const int64_t seg = u % segs, g = (u / segs) % (kPlanes / 4), line = u / (segs * (kPlanes / 4));
      fab = line * kLine + pair % kLine;
      plane = g * 4 + pair / kLine;
      row0 = 2 + seg * kSeg;
      dr = 1;
    } else {  // unit = (line, plane, group of 64 rows): pair (j, s) takes rows s, s+4, ...
      const int64_t half = u % 2, pl = (u / 2) % kPlanes, line = u / (2 * kPlanes);
      fab = line * kLine + pair % kLine;
      plane = pl;
      row0 = 2 + half * 64 + pair / kLine;
      dr = 4;
    }
    if (MODE == 3) {
      for (int r = 0; r < kSeg; ++r) rmw(seam(buf, fab, plane, row0 + r * dr, side));
    } else {
      uint32_t cur[8], nxt[8];
      ld(seam(buf, fab, plane, row0, side), cur);
      for (int r = 0; r < kSeg; ++r) {
        if (r + 1 < kSeg) ld(seam(buf, fab, plane, row0 + (r + 1) * dr, side), nxt);
        cur[0] += 1;
        if (MODE == 6) {
          char *q = seam(buf, fab, plane, row0 + r * dr, side) + (side ? 0 : 16);
          asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(q), "r"(cur[0]), "r"(cur[1]), "r"(cur[2]),
                       "r"(cur[3]) : "memory");
        } else if (MODE != 7) {
          st(seam(buf, fab, plane, row0 + r * dr, side), cur);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) cur[i] = nxt[i];
      }
    }
  }
}

// MODE 8: line walk -- one warp instruction = 16 consecutive rows of ONE
// fab; the warp visits the k = 4 fabs of its x-line in turn for the same
// 16 rows (the next fab's chunk loaded before this one's write), then the
// next 16 rows: the seam exchange across the x-line would keep all k
// chunks of a row block in registers.
__global__ void line_walk(char *buf, int64_t units) {
  const int lane = threadIdx.x & 31, pair = lane >> 1, side = lane & 1;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // unit = (line, plane, 64-row half): 4 blocks of 16 rows x 4 fabs
  for (int64_t u = warp; u < units; u += nwarps) {
    const int64_t half = u % 2, pl = (u / 2) % kPlanes, line = u / (2 * kPlanes);
    uint32_t cur[8], nxt[8];
    int64_t row = 2 + half * 64 + pair;
    ld(seam(buf, line * kLine, pl, row, side), cur);
    for (int s = 0; s < 16; ++s) {  // s = (row block b, fab j)
      const int b = s / kLine, j = s % kLine;
      if (s + 1 < 16) {
        const int b2 = (s + 1) / kLine, j2 = (s + 1) % kLine;
        ld(seam(buf, line * kLine + j2, pl, 2 + half * 64 + b2 * 16 + pair, side), nxt);
      }
      cur[0] += 1;
      st(seam(buf, line * kLine + j, pl, 2 + half * 64 + b * 16 + pair, side), cur);
#pragma unroll
      for (int i = 0; i < 8; ++i) cur[i] = nxt[i];
    }
  }
}

template <int MODE>
__global__ void walk(char *buf, int64_t units) {
  const int lane = threadIdx.x & 31, pair = lane >> 1, side = lane & 1;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  constexpr int64_t segs = 128 / kSeg;  // 8 segments of the 128 valid rows
  for (int64_t u = warp; u < units; u += nwarps) {
    int64_t fab, plane, row0;
    if (MODE == 0) {  // unit = (line, plane group of 4, segment)
      const int64_t seg = u % segs, g = (u / segs) % (kPlanes / 4), line = u / (segs * (kPlanes / 4));
      fab = line * kLine + pair % kLine;
      plane = g * 4 + pair / kLine;
      row0 = 2 + seg * kSeg;
    } else if (MODE == 1) {  // unit = (line, plane, half): 4 fabs x 4 segments of one plane
      const int64_t half = u % 2, pl = (u / 2) % kPlanes, line = u / (2 * kPlanes);
      fab = line * kLine + pair % kLine;
      plane = pl;
      row0 = 2 + (half * 4 + pair / kLine) * kSeg;
    } else {  // MODE 2: unit = (fab, plane pair): 16 segments over 2 consecutive planes
      const int64_t pp = u % (kPlanes / 2), f = u / (kPlanes / 2);
      fab = f;
      plane = pp * 2 + pair / 8;
      row0 = 2 + (pair % 8) * kSeg;
    }
    for (int r = 0; r < kSeg; ++r) rmw(seam(buf, fab, plane, row0 + r, side));
  }
}

__global__ void flat(char *buf, int64_t nseams) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = t; i < nseams * 2; i += nthr) {
    const int64_t s = i >> 1;
    const int64_t fab = s / (kPlanes * 128), rem = s % (kPlanes * 128);
    rmw(seam(buf, fab, rem / 128, 2 + rem % 128, (int)(i & 1)));
  }
}

// seam rmw (flat order) over the first `nseams` seams by the warps with
// (warp % 2 == 0) when WHICH & 1, and 1,024-B row copies (face rows) over a
// separate 2 GB region by the odd warps when WHICH & 2: do the
// request-bound seams and the bandwidth-bound rows overlap on PCIe?
template <int WHICH>
__global__ void mix(char *buf, int64_t nseams, char *rows, int64_t nrows) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 6;  // warps per class
  const int64_t w = warp >> 1;
  if ((warp & 1) == 0) {
    if (!(WHICH & 1)) return;
    for (int64_t i = w * 32 + lane; i < nseams * 2; i += nw * 32) {
      const int64_t s = i >> 1;
      const int64_t fab = s / (kPlanes * 128), rem = s % (kPlanes * 128);
      rmw(seam(buf, fab, rem / 128, 2 + rem % 128, (int)(i & 1)));
    }
  } else {
    if (!(WHICH & 2)) return;
    const int64_t half = nrows / 2;
    for (int64_t r = w; r < half; r += nw) {
      uint32_t v[8];
      ld(rows + r * kPitch + lane * 32, v);
      st(rows + (r + half) * kPitch + lane * 32, v);
    }
  }
}

template <int WHICH>
void run_mix(const char *name, char *buf, int64_t nseams, char *rows, int64_t nrows, int blocks) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int it = 0; it < 3; ++it) {
    cudaEventRecord(e0);
    mix<WHICH><<<blocks, 256>>>(buf, nseams, rows, nrows);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (it > 0 && ms < best) best = ms;
  }
  printf("  %-12s blocks %4d  %8.3f ms\n", name, blocks, best);
}

template <int MODE>
void run(const char *name, char *buf, int blocks) {
  const int64_t nseams = (int64_t)kFabs * kPlanes * 128;
  const int64_t units = nseams / 16 / kSeg;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int it = 0; it < 3; ++it) {
    cudaEventRecord(e0);
    if (MODE < 3)
      walk<MODE><<<blocks, 256>>>(buf, units);
    else if (MODE == 9)
      flat<<<blocks, 256>>>(buf, nseams);
    else if (MODE == 8)
      line_walk<<<blocks, 256>>>(buf, units);
    else
      tile_walk<MODE><<<blocks, 256>>>(buf, units);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (it > 0 && ms < best) best = ms;
  }
  printf("  %-8s blocks %4d  %8.3f ms  %6.3f ns/seam  %6.3f G req/s\n", name, blocks, best, best * 1e6 / nseams,
         2.0 * nseams / (best * 1e-3) * 1e-9);
}

int main() {
  const int64_t bytes = kFab * kFabs;
  char *h, *d;
  CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  CK(cudaHostGetDevicePointer((void **)&d, h, 0));
  for (int64_t i = 0; i < bytes; i += 4096) h[i] = 1;
  printf("pinned mapped host: %d fabs x %lld planes x %lld rows of %lld B (%.2f GB), %lld seams\n", kFabs,
         (long long)kPlanes, (long long)kRows, (long long)kPitch, bytes / 1e9, (long long)kFabs * kPlanes * 128);
  {
    // 4.3 M seams (half of C3's x seams) next to 0.5 M face-row copies (~C3's y/z rows)
    const int64_t ns = (int64_t)kFabs / 2 * kPlanes * 128, nr = 1 << 20;
    char *rows = d + kFab * (kFabs / 2);
    for (int blocks : {16, 32, 64}) {
      run_mix<1>("seams only", d, ns, rows, nr, blocks);
      run_mix<2>("rows only", d, ns, rows, nr, blocks);
      run_mix<3>("seams+rows", d, ns, rows, nr, blocks);
    }
  }
  for (int blocks : {8, 16, 32}) {
    run<0>("ring", d, blocks);
    run<1>("rowsegs", d, blocks);
    run<2>("onefab", d, blocks);
    run<9>("flat", d, blocks);
    run<3>("tile", d, blocks);
    run<4>("tile-pf", d, blocks);
    run<5>("ring-pf", d, blocks);
    run<6>("tile-pf-w32", d, blocks);
    run<8>("linewalk", d, blocks);
    run<7>("tile-pf-rd", d, blocks);
  }
  return 0;
}
