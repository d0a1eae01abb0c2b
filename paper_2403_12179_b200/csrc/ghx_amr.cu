// Coarse/fine level transfers for sm_100a: the two local kernels that
// fill_patch and average_down run around the exchange engine.
//
//   ghx_interp        interp_box (reference amr.py:269-314): fine cells of a
//                     region from their coarse parents, piecewise constant
//                     or with unlimited centred slopes (LINEAR);
//   ghx_average_down  the per-fab restriction of average_down
//                     (amr.py:251-264): each coarse cell becomes the mean of
//                     its ratio^D children; the ParallelCopy that follows is
//                     the exchange engine (ghx_exec.cu).
//
// Both are one launch over every job (fab) of a call and HBM-bound: the fine
// side is streamed once (written by interp, read by average_down), the
// coarse side once per fine-parent row (it stays in L1/L2 between the r
// fine rows that share it).  Arithmetic replays numpy's operation order with
// explicit round-to-nearest intrinsics (no FMA contraction), so results are
// bit-identical to the reference for float64 and float32 storage.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <string>
#include <vector>

#include "ghx_internal.h"

using ghx::set_error;

namespace {

constexpr int kAmrThreads = 256;

struct Geo3 {
  int64_t lo[3], n[3];  // storage box lo, extents
};

struct DevInterpJob {
  uint64_t crse, fine;
  Geo3 c, f;
  int64_t rlo[3], rn[3];  // fine region lo, extents
  int64_t start;          // first flat cell of this job in the launch
};

struct DevAvgJob {
  uint64_t fine, crse;
  Geo3 f, c;
  int64_t rlo[3], rn[3];  // coarse region lo, extents
  int64_t start;
};

__device__ __forceinline__ int64_t floordiv(int64_t a, int64_t b) {
  const int64_t q = a / b;
  return (q * b > a) ? q - 1 : q;
}

template <class J>
__device__ __forceinline__ int find_job(const J *jobs, int njobs, int64_t i) {
  int lo = 0, hi = njobs - 1;
  while (lo < hi) {  // last job with start <= i
    const int mid = (lo + hi + 1) >> 1;
    if (jobs[mid].start <= i)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }

// One thread per fine cell of the launch (x fastest: coalesced fine stores),
// all components.  LINEAR, per axis d < spacedim in order (amr.py:302-313):
//   slope = 0.5 * (c[p+e_d] - c[p-e_d])          (storage type T)
//   off   = ((f mod r) + 0.5) / r - 0.5          (float64)
//   v     = T(double(v) + double(slope) * off)   (numpy's float64 loop for
//                                                 v += slope * off)
template <class T, bool LINEAR>
__global__ void __launch_bounds__(kAmrThreads) interp_kernel(const DevInterpJob *__restrict__ jobs, int njobs,
                                                             int64_t total, int ncomp, int r0, int r1, int r2,
                                                             int spacedim) {
  const int r[3] = {r0, r1, r2};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const DevInterpJob &J = jobs[find_job(jobs, njobs, i)];
    int64_t q = i - J.start;
    int64_t fidx[3];
    fidx[0] = J.rlo[0] + q % J.rn[0];
    q /= J.rn[0];
    fidx[1] = J.rlo[1] + q % J.rn[1];
    fidx[2] = J.rlo[2] + q / J.rn[1];
    int64_t pl[3];
    double off[3];
    for (int d = 0; d < 3; ++d) {
      const int64_t p = floordiv(fidx[d], r[d]);
      pl[d] = p - J.c.lo[d];
      const int64_t m = fidx[d] - p * r[d];
      off[d] = __dsub_rn(__ddiv_rn(__dadd_rn((double)m, 0.5), (double)r[d]), 0.5);
    }
    const int64_t csy = J.c.n[0], csz = J.c.n[0] * J.c.n[1], csc = csz * J.c.n[2];
    const int64_t fsc = J.f.n[0] * J.f.n[1] * J.f.n[2];
    const int64_t co = pl[0] + pl[1] * csy + pl[2] * csz;
    const int64_t fo = (fidx[0] - J.f.lo[0]) + (fidx[1] - J.f.lo[1]) * J.f.n[0] +
                       (fidx[2] - J.f.lo[2]) * J.f.n[0] * J.f.n[1];
    const T *crse = reinterpret_cast<const T *>(J.crse);
    T *fine = reinterpret_cast<T *>(J.fine);
    const int64_t step[3] = {1, csy, csz};
    for (int c = 0; c < ncomp; ++c) {
      const T *cc = crse + co + c * csc;
      T v = __ldg(cc);
      if (LINEAR) {
        for (int d = 0; d < spacedim; ++d) {
          const T slope = mul_rn(T(0.5), sub_rn(__ldg(cc + step[d]), __ldg(cc - step[d])));
          v = T(__dadd_rn((double)v, __dmul_rn((double)slope, off[d])));
        }
      }
      fine[fo + c * fsc] = v;
    }
  }
}

// One thread per coarse cell: acc = child(0,0,0), then += children in
// (oz, oy, ox) loop order, then acc / ratio^D (amr.py:254-264).
template <class T>
__global__ void __launch_bounds__(kAmrThreads) avgdown_kernel(const DevAvgJob *__restrict__ jobs, int njobs,
                                                              int64_t total, int ncomp, int r0, int r1, int r2,
                                                              T rpow) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const DevAvgJob &J = jobs[find_job(jobs, njobs, i)];
    int64_t q = i - J.start;
    int64_t cidx[3];
    cidx[0] = J.rlo[0] + q % J.rn[0];
    q /= J.rn[0];
    cidx[1] = J.rlo[1] + q % J.rn[1];
    cidx[2] = J.rlo[2] + q / J.rn[1];
    const int64_t fsy = J.f.n[0], fsz = J.f.n[0] * J.f.n[1], fsc = fsz * J.f.n[2];
    const int64_t csc = J.c.n[0] * J.c.n[1] * J.c.n[2];
    const int64_t fo = (cidx[0] * r0 - J.f.lo[0]) + (cidx[1] * r1 - J.f.lo[1]) * fsy + (cidx[2] * r2 - J.f.lo[2]) * fsz;
    const int64_t co = (cidx[0] - J.c.lo[0]) + (cidx[1] - J.c.lo[1]) * J.c.n[0] +
                       (cidx[2] - J.c.lo[2]) * J.c.n[0] * J.c.n[1];
    const T *fine = reinterpret_cast<const T *>(J.fine);
    T *crse = reinterpret_cast<T *>(J.crse);
    for (int c = 0; c < ncomp; ++c) {
      const T *f = fine + fo + c * fsc;
      T acc = T(0);
      bool first = true;
      for (int oz = 0; oz < r2; ++oz)
        for (int oy = 0; oy < r1; ++oy)
          for (int ox = 0; ox < r0; ++ox) {
            const T v = __ldg(f + ox + oy * fsy + oz * fsz);
            acc = first ? v : add_rn(acc, v);
            first = false;
          }
      crse[co + c * csc] = div_rn(acc, rpow);
    }
  }
}

Geo3 geo(const int64_t *b) {
  Geo3 g;
  for (int d = 0; d < 3; ++d) {
    g.lo[d] = b[d];
    g.n[d] = b[3 + d] - b[d] + 1;
  }
  return g;
}

bool inside(const int64_t *outer, const int64_t *lo, const int64_t *hi) {
  for (int d = 0; d < 3; ++d)
    if (lo[d] < outer[d] || hi[d] > outer[3 + d]) return false;
  return true;
}

int cuda_fail(cudaError_t e, const char *what) {
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return GHX_ECUDA;
}

int64_t floordiv_h(int64_t a, int64_t b) {
  const int64_t q = a / b;
  return (q * b > a) ? q - 1 : q;
}

// stream-ordered upload of a job table, launch, free
template <class J, class Launch>
int run_jobs(const std::vector<J> &jobs, int64_t total, void *stream, const char *what, Launch launch) {
  if (total == 0) return GHX_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  J *dj = nullptr;
  const size_t bytes = jobs.size() * sizeof(J);
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(&dj), bytes, st);
  if (e != cudaSuccess) return cuda_fail(e, what);
  e = cudaMemcpyAsync(dj, jobs.data(), bytes, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) {
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (total + kAmrThreads - 1) / kAmrThreads;
    const int blocks = (int)std::min<int64_t>(want, (int64_t)sms * 8);
    launch(dj, blocks, st);
    e = cudaGetLastError();
  }
  cudaError_t e2 = cudaFreeAsync(dj, st);
  if (e != cudaSuccess) return cuda_fail(e, what);
  if (e2 != cudaSuccess) return cuda_fail(e2, what);
  return GHX_OK;
}

std::atomic<int64_t> g_amr_launches{0};

}  // namespace

extern "C" {

int64_t ghx_amr_launch_count(void) { return g_amr_launches.load(); }

int ghx_interp(const ghx_interp_job *jobs, int64_t njobs, int32_t ncomp, const int32_t ratio[3], int32_t spacedim,
               int32_t scheme, int32_t elem_bytes, void *stream) {
  if ((njobs && !jobs) || njobs < 0 || njobs > (1 << 30) || ncomp < 1 || !ratio || spacedim < 1 || spacedim > 3 ||
      (scheme != GHX_INTERP_PC && scheme != GHX_INTERP_LINEAR) || (elem_bytes != 4 && elem_bytes != 8)) {
    set_error("ghx_interp: bad arguments");
    return GHX_EINVAL;
  }
  for (int d = 0; d < 3; ++d)
    if (ratio[d] < 1 || (d >= spacedim && ratio[d] != 1)) {
      set_error("ghx_interp: ratio must be >= 1 (1 on axes >= spacedim)");
      return GHX_EINVAL;
    }
  std::vector<DevInterpJob> dj;
  dj.reserve(njobs);
  int64_t total = 0;
  for (int64_t j = 0; j < njobs; ++j) {
    const ghx_interp_job &J = jobs[j];
    const int64_t *R = J.region;
    if (R[3] < R[0] || R[4] < R[1] || R[5] < R[2]) continue;  // empty region: nothing to do
    if (!inside(J.fine_box, R, R + 3)) {
      set_error("ghx_interp: job " + std::to_string(j) + ": fine_region must lie inside the fine fab");
      return GHX_EINVAL;
    }
    int64_t need_lo[3], need_hi[3];
    for (int d = 0; d < 3; ++d) {
      const int64_t g = (scheme == GHX_INTERP_LINEAR && d < spacedim) ? 1 : 0;
      need_lo[d] = floordiv_h(R[d], ratio[d]) - g;
      need_hi[d] = floordiv_h(R[3 + d], ratio[d]) + g;
    }
    if (!inside(J.crse_box, need_lo, need_hi)) {
      set_error("ghx_interp: job " + std::to_string(j) + ": insufficient coarse data");
      return GHX_EINVAL;
    }
    if (!J.crse || !J.fine) {
      set_error("ghx_interp: null fab pointer");
      return GHX_EINVAL;
    }
    DevInterpJob d;
    std::memset(&d, 0, sizeof(d));
    d.crse = reinterpret_cast<uint64_t>(J.crse);
    d.fine = reinterpret_cast<uint64_t>(J.fine);
    d.c = geo(J.crse_box);
    d.f = geo(J.fine_box);
    for (int a = 0; a < 3; ++a) {
      d.rlo[a] = R[a];
      d.rn[a] = R[3 + a] - R[a] + 1;
    }
    d.start = total;
    total += d.rn[0] * d.rn[1] * d.rn[2];
    dj.push_back(d);
  }
  const int nj = (int)dj.size();
  const int r0 = ratio[0], r1 = ratio[1], r2 = ratio[2];
  int rc = run_jobs(dj, total, stream, "ghx_interp", [&](const DevInterpJob *p, int blocks, cudaStream_t st) {
    const bool lin = scheme == GHX_INTERP_LINEAR;
    if (elem_bytes == 8) {
      if (lin)
        interp_kernel<double, true><<<blocks, kAmrThreads, 0, st>>>(p, nj, total, ncomp, r0, r1, r2, spacedim);
      else
        interp_kernel<double, false><<<blocks, kAmrThreads, 0, st>>>(p, nj, total, ncomp, r0, r1, r2, spacedim);
    } else {
      if (lin)
        interp_kernel<float, true><<<blocks, kAmrThreads, 0, st>>>(p, nj, total, ncomp, r0, r1, r2, spacedim);
      else
        interp_kernel<float, false><<<blocks, kAmrThreads, 0, st>>>(p, nj, total, ncomp, r0, r1, r2, spacedim);
    }
  });
  if (rc == GHX_OK && total) g_amr_launches.fetch_add(1);
  return rc;
}

int ghx_average_down(const ghx_avgdown_job *jobs, int64_t njobs, int32_t ncomp, const int32_t ratio[3],
                     int32_t spacedim, int32_t elem_bytes, void *stream) {
  if ((njobs && !jobs) || njobs < 0 || njobs > (1 << 30) || ncomp < 1 || !ratio || spacedim < 1 || spacedim > 3 ||
      (elem_bytes != 4 && elem_bytes != 8)) {
    set_error("ghx_average_down: bad arguments");
    return GHX_EINVAL;
  }
  int64_t rpow = 1;
  for (int d = 0; d < 3; ++d) {
    if (ratio[d] < 1 || (d >= spacedim && ratio[d] != 1)) {
      set_error("ghx_average_down: ratio must be >= 1 (1 on axes >= spacedim)");
      return GHX_EINVAL;
    }
    rpow *= ratio[d];
  }
  std::vector<DevAvgJob> dj;
  dj.reserve(njobs);
  int64_t total = 0;
  for (int64_t j = 0; j < njobs; ++j) {
    const ghx_avgdown_job &J = jobs[j];
    const int64_t *R = J.region;
    if (R[3] < R[0] || R[4] < R[1] || R[5] < R[2]) continue;
    int64_t flo[3], fhi[3];
    for (int d = 0; d < 3; ++d) {
      flo[d] = R[d] * ratio[d];
      fhi[d] = R[3 + d] * ratio[d] + ratio[d] - 1;
    }
    if (!inside(J.crse_box, R, R + 3) || !inside(J.fine_box, flo, fhi)) {
      set_error("ghx_average_down: job " + std::to_string(j) + ": region outside the fine or coarse fab");
      return GHX_EINVAL;
    }
    if (!J.crse || !J.fine) {
      set_error("ghx_average_down: null fab pointer");
      return GHX_EINVAL;
    }
    DevAvgJob d;
    std::memset(&d, 0, sizeof(d));
    d.fine = reinterpret_cast<uint64_t>(J.fine);
    d.crse = reinterpret_cast<uint64_t>(J.crse);
    d.f = geo(J.fine_box);
    d.c = geo(J.crse_box);
    for (int a = 0; a < 3; ++a) {
      d.rlo[a] = R[a];
      d.rn[a] = R[3 + a] - R[a] + 1;
    }
    d.start = total;
    total += d.rn[0] * d.rn[1] * d.rn[2];
    dj.push_back(d);
  }
  const int nj = (int)dj.size();
  const int r0 = ratio[0], r1 = ratio[1], r2 = ratio[2];
  int rc = run_jobs(dj, total, stream, "ghx_average_down", [&](const DevAvgJob *p, int blocks, cudaStream_t st) {
    if (elem_bytes == 8)
      avgdown_kernel<double><<<blocks, kAmrThreads, 0, st>>>(p, nj, total, ncomp, r0, r1, r2, (double)rpow);
    else
      avgdown_kernel<float><<<blocks, kAmrThreads, 0, st>>>(p, nj, total, ncomp, r0, r1, r2, (float)rpow);
  });
  if (rc == GHX_OK && total) g_amr_launches.fetch_add(1);
  return rc;
}

}  // extern "C"
