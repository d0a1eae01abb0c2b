// Coarse/fine level transfers for sm_100a: the two local kernels that
// fill_patch and average_down run around the exchange engine, plus the heat
// step's stencil (the consumer the exchange overlaps with).
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
#include <cstdlib>
#include <atomic>
#include <cstring>
#include <string>
#include <vector>

#include "ghx_internal.h"

using ghx::set_error;

namespace {

constexpr int kAmrThreads = 256;
#ifndef GHX_INTERP_MINB
#define GHX_INTERP_MINB 5
#endif
#ifndef GHX_INTERP_COMPS
#define GHX_INTERP_COMPS 2
#endif
constexpr int kInterpComps = GHX_INTERP_COMPS;  // interp: components whose loads are batched

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

__device__ __forceinline__ int32_t floordiv32(int32_t a, int32_t b) {
  const int32_t q = a / b;
  return (q * b > a) ? q - 1 : q;
}

__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }

// One thread per fine cell: blocks take kAmrThreads consecutive cells of one
// job (x fastest: coalesced fine stores), all components.  LINEAR, per axis d < spacedim in order (amr.py:302-313):
//   slope = 0.5 * (c[p+e_d] - c[p-e_d])          (storage type T)
//   off   = ((f mod r) + 0.5) / r - 0.5          (float64)
//   v     = T(double(v) + double(slope) * off)   (numpy's float64 loop for
//                                                 v += slope * off)
template <class T, bool LINEAR>
__global__ void __launch_bounds__(kAmrThreads, GHX_INTERP_MINB) interp_kernel(const DevInterpJob *__restrict__ jobs,
                                                             const int4 *__restrict__ btasks, int ncomp, int r0,
                                                             int r1, int r2, int spacedim) {
  const int r[3] = {r0, r1, r2};
  const int4 bt = btasks[blockIdx.x];  // {job, first cell, cells}: one job per block
  const DevInterpJob &J = jobs[bt.x];
  for (int k = threadIdx.x; k < bt.z; k += kAmrThreads) {
    // 32-bit index math inside a job (jobs are < 2^31 cells, host-checked)
    const uint32_t q = (uint32_t)(bt.y + k), nx = (uint32_t)J.rn[0], ny = (uint32_t)J.rn[1];
    const uint32_t t = q / nx;
    int32_t fidx[3];
    fidx[0] = (int32_t)J.rlo[0] + (int32_t)(q - t * nx);
    fidx[1] = (int32_t)J.rlo[1] + (int32_t)(t % ny);
    fidx[2] = (int32_t)J.rlo[2] + (int32_t)(t / ny);
    int64_t pl[3];
    double off[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const int32_t p = floordiv32(fidx[d], r[d]);
      pl[d] = (int64_t)p - J.c.lo[d];
      const int32_t m = fidx[d] - p * r[d];
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
    // components in groups of kInterpComps: every coarse value of a group is
    // requested before any arithmetic (up to 7 * kInterpComps loads in flight)
    for (int c0 = 0; c0 < ncomp; c0 += kInterpComps) {
      T v[kInterpComps], up[kInterpComps][3], dn[kInterpComps][3];
#pragma unroll
      for (int i = 0; i < kInterpComps; ++i) {
        if (c0 + i >= ncomp) break;
        const T *cc = crse + co + (c0 + i) * csc;
        v[i] = __ldg(cc);
        if (LINEAR) {
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            up[i][d] = d < spacedim ? __ldg(cc + step[d]) : T(0);
            dn[i][d] = d < spacedim ? __ldg(cc - step[d]) : T(0);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < kInterpComps; ++i) {
        if (c0 + i >= ncomp) break;
        T w = v[i];
        if (LINEAR) {
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            if (d >= spacedim) break;
            const T slope = mul_rn(T(0.5), sub_rn(up[i][d], dn[i][d]));
            w = T(__dadd_rn((double)w, __dmul_rn((double)slope, off[d])));
          }
        }
        fine[fo + (c0 + i) * fsc] = w;
      }
    }
  }
}

// One thread per coarse cell: acc = child(0,0,0), then += children in
// (oz, oy, ox) loop order, then acc / ratio^D (amr.py:254-264).
template <class T, bool R222>
__global__ void __launch_bounds__(kAmrThreads, 4) avgdown_kernel(const DevAvgJob *__restrict__ jobs,
                                                              const int4 *__restrict__ btasks, int ncomp, int r0,
                                                              int r1, int r2, T rpow) {
  const int4 bt = btasks[blockIdx.x];
  const DevAvgJob &J = jobs[bt.x];
  for (int k = threadIdx.x; k < bt.z; k += kAmrThreads) {
    const uint32_t q = (uint32_t)(bt.y + k), nx = (uint32_t)J.rn[0], ny = (uint32_t)J.rn[1];
    const uint32_t t = q / nx;
    int64_t cidx[3];
    cidx[0] = J.rlo[0] + (int64_t)(q - t * nx);
    cidx[1] = J.rlo[1] + (int64_t)(t % ny);
    cidx[2] = J.rlo[2] + (int64_t)(t / ny);
    const int64_t fsy = J.f.n[0], fsz = J.f.n[0] * J.f.n[1], fsc = fsz * J.f.n[2];
    const int64_t csc = J.c.n[0] * J.c.n[1] * J.c.n[2];
    const int64_t fo = (cidx[0] * r0 - J.f.lo[0]) + (cidx[1] * r1 - J.f.lo[1]) * fsy + (cidx[2] * r2 - J.f.lo[2]) * fsz;
    const int64_t co = (cidx[0] - J.c.lo[0]) + (cidx[1] - J.c.lo[1]) * J.c.n[0] +
                       (cidx[2] - J.c.lo[2]) * J.c.n[0] * J.c.n[1];
    const T *fine = reinterpret_cast<const T *>(J.fine);
    T *crse = reinterpret_cast<T *>(J.crse);
    if (R222) {  // ratio 2 in 3-D: all eight children loaded before the ordered sum
      for (int c = 0; c < ncomp; ++c) {
        const T *f = fine + fo + c * fsc;
        T v[8];
#pragma unroll
        for (int o = 0; o < 8; ++o) v[o] = __ldg(f + (o & 1) + ((o >> 1) & 1) * fsy + (o >> 2) * fsz);
        T acc = v[0];
#pragma unroll
        for (int o = 1; o < 8; ++o) acc = add_rn(acc, v[o]);  // (oz, oy, ox) order, ox fastest
        crse[co + c * csc] = div_rn(acc, rpow);
      }
    } else {
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
}

// One heat-equation step (reference heat.py:172-189, comp 0):
//   acc = u;  acc += c_d * ((u[+e_d] - 2*u) + u[-e_d])   for d < DIM
// in numpy's order, storage type T throughout (coefficients rounded to T).
// 2.5-D blocking: a block is a TX x (256 / TX) (x, y) tile of one job that
// marches kAdvZ planes in z, carrying u[z-1], u[z], u[z+1] in registers, so
// each source value comes from HBM once (x/y neighbours hit L1).  TX = 64
// (longer contiguous runs per plane) when the regions are wide enough to
// keep the lanes busy, else 32.
#ifndef GHX_ADV_MINB
#define GHX_ADV_MINB 4
#endif
#ifndef GHX_ADV_PF
#define GHX_ADV_PF 2
#endif
#ifndef GHX_ADV_Z
#define GHX_ADV_Z 32
#endif
constexpr int kAdvZ = GHX_ADV_Z, kAdvPF = GHX_ADV_PF;

template <class T, int DIM, int TX>
__global__ void __launch_bounds__(kAmrThreads, GHX_ADV_MINB) advance_kernel(const DevAvgJob *__restrict__ jobs,
                                                                 const int4 *__restrict__ btasks, T c0, T c1, T c2) {
  const int4 bt = btasks[blockIdx.x];  // {job, x0 | y0 << 16, z0, nz}
  const DevAvgJob &J = jobs[bt.x];
  const int tx = threadIdx.x & (TX - 1), ty = threadIdx.x / TX;
  const int64_t xr = (bt.y & 0xffff) + tx, yr = (bt.y >> 16) + ty;
  if (xr >= J.rn[0] || yr >= J.rn[1]) return;
  const int64_t x = J.rlo[0] + xr, y = J.rlo[1] + yr, z = J.rlo[2] + bt.z;
  const int64_t usy = J.f.n[0], usz = J.f.n[0] * J.f.n[1];
  const int64_t osy = J.c.n[0], osz = J.c.n[0] * J.c.n[1];
  const T *u = reinterpret_cast<const T *>(J.fine) + (x - J.f.lo[0]) + (y - J.f.lo[1]) * usy + (z - J.f.lo[2]) * usz;
  T *o = reinterpret_cast<T *>(J.crse) + (x - J.c.lo[0]) + (y - J.c.lo[1]) * osy + (z - J.c.lo[2]) * osz;
  // register queue of the next kAdvPF planes: plane z+kAdvPF is requested
  // kAdvPF - 1 steps before it is used (more DRAM loads in flight per thread)
  T um = DIM >= 3 ? __ldg(u - usz) : T(0);
  T uc = __ldg(u);
  T q[kAdvPF];
#pragma unroll
  for (int a = 0; a < kAdvPF; ++a) q[a] = (DIM >= 3 && a < bt.w) ? __ldg(u + (a + 1) * usz) : T(0);
#pragma unroll 4
  for (int k = 0; k < bt.w; ++k) {
    const T up = q[0];
#pragma unroll
    for (int a = 0; a + 1 < kAdvPF; ++a) q[a] = q[a + 1];
    q[kAdvPF - 1] = (DIM >= 3 && k + kAdvPF < bt.w) ? __ldg(u + (kAdvPF + 1) * usz) : T(0);
    const T two_u = mul_rn(T(2), uc);
    T acc = uc;
    acc = add_rn(acc, mul_rn(c0, add_rn(sub_rn(__ldg(u + 1), two_u), __ldg(u - 1))));
    if (DIM >= 2) acc = add_rn(acc, mul_rn(c1, add_rn(sub_rn(__ldg(u + usy), two_u), __ldg(u - usy))));
    if (DIM >= 3) acc = add_rn(acc, mul_rn(c2, add_rn(sub_rn(up, two_u), um)));
    *o = acc;
    um = uc;
    uc = up;
    u += usz;
    o += osz;
  }
}

// The same stencil, one thread per cell of a flat cell list (block tasks of
// kAmrThreads * 4 cells of one job): for the thin one-cell shells of the
// overlapped heat step, where 32 x 8 tiles would idle most lanes.
template <class T, int DIM>
__global__ void __launch_bounds__(kAmrThreads, 4) advance_flat_kernel(const DevAvgJob *__restrict__ jobs,
                                                                      const int4 *__restrict__ btasks, T c0, T c1,
                                                                      T c2) {
  const int4 bt = btasks[blockIdx.x];
  const DevAvgJob &J = jobs[bt.x];
  for (int k = threadIdx.x; k < bt.z; k += kAmrThreads) {
    const uint32_t q = (uint32_t)(bt.y + k), nx = (uint32_t)J.rn[0], ny = (uint32_t)J.rn[1];
    const uint32_t t = q / nx;
    const int64_t x = J.rlo[0] + (int64_t)(q - t * nx), y = J.rlo[1] + (int64_t)(t % ny),
                  z = J.rlo[2] + (int64_t)(t / ny);
    const int64_t usy = J.f.n[0], usz = J.f.n[0] * J.f.n[1];
    const T *u = reinterpret_cast<const T *>(J.fine) + (x - J.f.lo[0]) + (y - J.f.lo[1]) * usy +
                 (z - J.f.lo[2]) * usz;
    T *o = reinterpret_cast<T *>(J.crse) + (x - J.c.lo[0]) + (y - J.c.lo[1]) * J.c.n[0] +
           (z - J.c.lo[2]) * J.c.n[0] * J.c.n[1];
    const T uc = __ldg(u);
    const T two_u = mul_rn(T(2), uc);
    T acc = uc;
    acc = add_rn(acc, mul_rn(c0, add_rn(sub_rn(__ldg(u + 1), two_u), __ldg(u - 1))));
    if (DIM >= 2) acc = add_rn(acc, mul_rn(c1, add_rn(sub_rn(__ldg(u + usy), two_u), __ldg(u - usy))));
    if (DIM >= 3) acc = add_rn(acc, mul_rn(c2, add_rn(sub_rn(__ldg(u + usz), two_u), __ldg(u - usz))));
    *o = acc;
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
  // consume a non-sticky error (e.g. cudaErrorAlreadyMapped from an IPC open
  // the caller retries) so a later cudaGetLastError() does not report it
  // again for an unrelated, successful call
  (void)cudaGetLastError();
  return GHX_ECUDA;
}

int64_t floordiv_h(int64_t a, int64_t b) {
  const int64_t q = a / b;
  return (q * b > a) ? q - 1 : q;
}

std::atomic<int64_t> g_amr_launches{0};

}  // namespace

// A prepared transfer: the device job table of one interp / average_down
// call pattern (fill_patch and average_down cache one per plan), so a call
// is a single kernel launch with no host-side table work.
struct ghx_xfer {
  int kind = 0;  // 0 interp, 1 average_down, 2 stencil (tiles), 3 stencil (flat cells)
  int device = 0;
  void *djobs = nullptr;
  int4 *dtasks = nullptr;  // one block per task: {job, ...}
  int ntasks = 0;
  int njobs = 0;
  int64_t total = 0;
  int ncomp = 1, r[3] = {1, 1, 1}, spacedim = 3, scheme = 0, elem_bytes = 8;
  int64_t rpow = 1;
  double coef[3] = {0, 0, 0};  // advance: dt * diffusivity / dx_d^2
  int blocks = 0;
  int tile_x = 32;  // advance: x extent of a block tile (32 or 64)
};

namespace {

constexpr int kCellsPerBlock = kAmrThreads * 4;

// Block tasks: interp blocks take kAmrThreads consecutive cells of one job
// (one per thread), average_down blocks kCellsPerBlock; the stencil takes
// TX x (256 / TX) x kAdvZ tiles of one job.
template <class J>
std::vector<int4> block_tasks(ghx_xfer *x, const std::vector<J> &jobs) {
  std::vector<int4> t;
  if (x->kind == 2) {  // 64-wide tiles when they waste <= 1/4 of the lanes over the launch
    int64_t cells = 0, lanes64 = 0;
    for (const J &d : jobs) {
      cells += d.rn[0] * d.rn[1] * d.rn[2];
      lanes64 += (d.rn[0] + 63) / 64 * 64 * d.rn[1] * d.rn[2];
    }
    x->tile_x = (cells > 0 && 4 * cells >= 3 * lanes64) ? 64 : 32;
  }
  const int tx = x->tile_x, ty = kAmrThreads / tx;
  for (size_t j = 0; j < jobs.size(); ++j) {
    const J &d = jobs[j];
    if (x->kind == 2) {
      for (int64_t z0 = 0; z0 < d.rn[2]; z0 += kAdvZ)
        for (int64_t y0 = 0; y0 < d.rn[1]; y0 += ty)
          for (int64_t x0 = 0; x0 < d.rn[0]; x0 += tx)
            t.push_back(make_int4((int)j, (int)(x0 | (y0 << 16)), (int)z0, (int)std::min<int64_t>(kAdvZ, d.rn[2] - z0)));
    } else {
      const int64_t cells = d.rn[0] * d.rn[1] * d.rn[2];
      const int64_t per = x->kind == 0 ? kAmrThreads : kCellsPerBlock;  // interp: one cell per thread
      for (int64_t c0 = 0; c0 < cells; c0 += per)
        t.push_back(make_int4((int)j, (int)c0, (int)std::min<int64_t>(per, cells - c0), 0));
    }
  }
  return t;
}

template <class J>
int xfer_upload(ghx_xfer *x, const std::vector<J> &jobs, const char *what) {
  x->njobs = (int)jobs.size();
  if (jobs.empty()) return GHX_OK;
  for (const J &d : jobs)
    if (x->kind == 2 && (d.rn[0] >= 65536 || d.rn[1] >= 32768)) {
      set_error(std::string(what) + ": stencil region extent too large (x < 65536, y < 32768)");
      return GHX_EINVAL;
    }
  const std::vector<int4> tasks = block_tasks(x, jobs);
  x->ntasks = (int)tasks.size();
  x->blocks = x->ntasks;
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != x->device) cudaSetDevice(x->device);
  cudaError_t e = cudaMalloc(&x->djobs, jobs.size() * sizeof(J));
  if (e == cudaSuccess) e = cudaMemcpy(x->djobs, jobs.data(), jobs.size() * sizeof(J), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&x->dtasks, tasks.size() * sizeof(int4));
  if (e == cudaSuccess) e = cudaMemcpy(x->dtasks, tasks.data(), tasks.size() * sizeof(int4), cudaMemcpyHostToDevice);
  if (prev != x->device) cudaSetDevice(prev);
  if (e != cudaSuccess) return cuda_fail(e, what);
  return GHX_OK;
}

int xfer_launch(const ghx_xfer *x, cudaStream_t st) {
  if (x->total == 0 || x->ntasks == 0) return GHX_OK;
  if (x->kind == 0) {
    const DevInterpJob *p = static_cast<const DevInterpJob *>(x->djobs);
    const bool lin = x->scheme == GHX_INTERP_LINEAR;
    const int g = x->blocks;
    if (x->elem_bytes == 8) {
      if (lin)
        interp_kernel<double, true><<<g, kAmrThreads, 0, st>>>(p, x->dtasks, x->ncomp, x->r[0], x->r[1],
                                                                       x->r[2], x->spacedim);
      else
        interp_kernel<double, false><<<g, kAmrThreads, 0, st>>>(p, x->dtasks, x->ncomp, x->r[0], x->r[1],
                                                                        x->r[2], x->spacedim);
    } else {
      if (lin)
        interp_kernel<float, true><<<g, kAmrThreads, 0, st>>>(p, x->dtasks, x->ncomp, x->r[0], x->r[1],
                                                                      x->r[2], x->spacedim);
      else
        interp_kernel<float, false><<<g, kAmrThreads, 0, st>>>(p, x->dtasks, x->ncomp, x->r[0], x->r[1],
                                                                       x->r[2], x->spacedim);
    }
  } else if (x->kind == 2 || x->kind == 3) {
    const DevAvgJob *p = static_cast<const DevAvgJob *>(x->djobs);
    const double *c = x->coef;
#define GHX_ADV(T, D)                                                                                        \
  if (x->kind == 2 && x->tile_x == 64)                                                                       \
    advance_kernel<T, D, 64><<<x->blocks, kAmrThreads, 0, st>>>(p, x->dtasks, (T)c[0], (T)c[1], (T)c[2]);    \
  else if (x->kind == 2)                                                                                     \
    advance_kernel<T, D, 32><<<x->blocks, kAmrThreads, 0, st>>>(p, x->dtasks, (T)c[0], (T)c[1], (T)c[2]);    \
  else                                                                                                       \
    advance_flat_kernel<T, D><<<x->blocks, kAmrThreads, 0, st>>>(p, x->dtasks, (T)c[0], (T)c[1], (T)c[2])
    if (x->elem_bytes == 8) {
      if (x->spacedim == 1) GHX_ADV(double, 1);
      else if (x->spacedim == 2) GHX_ADV(double, 2);
      else GHX_ADV(double, 3);
    } else {
      if (x->spacedim == 1) GHX_ADV(float, 1);
      else if (x->spacedim == 2) GHX_ADV(float, 2);
      else GHX_ADV(float, 3);
    }
#undef GHX_ADV
  } else {
    const DevAvgJob *p = static_cast<const DevAvgJob *>(x->djobs);
    const bool r222 = x->r[0] == 2 && x->r[1] == 2 && x->r[2] == 2;
    if (x->elem_bytes == 8)
      (r222 ? avgdown_kernel<double, true> : avgdown_kernel<double, false>)<<<x->blocks, kAmrThreads, 0, st>>>(
          p, x->dtasks, x->ncomp, x->r[0], x->r[1], x->r[2], (double)x->rpow);
    else
      (r222 ? avgdown_kernel<float, true> : avgdown_kernel<float, false>)<<<x->blocks, kAmrThreads, 0, st>>>(
          p, x->dtasks, x->ncomp, x->r[0], x->r[1], x->r[2], (float)x->rpow);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "ghx_xfer_run: launch");
  g_amr_launches.fetch_add(1);
  return GHX_OK;
}

bool check_common(int64_t njobs, const void *jobs, int32_t ncomp, const int32_t *ratio, int32_t spacedim,
                  int32_t elem_bytes, const char *what) {
  if ((njobs && !jobs) || njobs < 0 || njobs > (1 << 30) || ncomp < 1 || !ratio || spacedim < 1 || spacedim > 3 ||
      (elem_bytes != 4 && elem_bytes != 8)) {
    set_error(std::string(what) + ": bad arguments");
    return false;
  }
  for (int d = 0; d < 3; ++d)
    if (ratio[d] < 1 || (d >= spacedim && ratio[d] != 1)) {
      set_error(std::string(what) + ": ratio must be >= 1 (1 on axes >= spacedim)");
      return false;
    }
  return true;
}

}  // namespace

extern "C" {

int64_t ghx_amr_launch_count(void) { return g_amr_launches.load(); }

int ghx_interp_prepare(const ghx_interp_job *jobs, int64_t njobs, int32_t ncomp, const int32_t ratio[3],
                       int32_t spacedim, int32_t scheme, int32_t elem_bytes, int32_t device, ghx_xfer **out) {
  if (!out || !check_common(njobs, jobs, ncomp, ratio, spacedim, elem_bytes, "ghx_interp") ||
      (scheme != GHX_INTERP_PC && scheme != GHX_INTERP_LINEAR)) {
    if (out && scheme != GHX_INTERP_PC && scheme != GHX_INTERP_LINEAR) set_error("ghx_interp: unknown scheme");
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
    if (d.rn[0] * d.rn[1] * d.rn[2] >= (1ll << 31) || std::abs(R[0]) >= (1ll << 30) || std::abs(R[3]) >= (1ll << 30) ||
        std::abs(R[1]) >= (1ll << 30) || std::abs(R[4]) >= (1ll << 30) || std::abs(R[2]) >= (1ll << 30) ||
        std::abs(R[5]) >= (1ll << 30)) {
      set_error("ghx_interp: job " + std::to_string(j) + ": region too large (>= 2^31 cells or |index| >= 2^30)");
      return GHX_EINVAL;
    }
    total += d.rn[0] * d.rn[1] * d.rn[2];
    dj.push_back(d);
  }
  ghx_xfer *x = new (std::nothrow) ghx_xfer();
  if (!x) {
    set_error("ghx_interp: out of memory");
    return GHX_ENOMEM;
  }
  x->kind = 0;
  x->device = device;
  x->total = total;
  x->ncomp = ncomp;
  for (int d = 0; d < 3; ++d) x->r[d] = ratio[d];
  x->spacedim = spacedim;
  x->scheme = scheme;
  x->elem_bytes = elem_bytes;
  if (int rc = xfer_upload(x, dj, "ghx_interp_prepare")) {
    delete x;
    return rc;
  }
  *out = x;
  return GHX_OK;
}

int ghx_average_down_prepare(const ghx_avgdown_job *jobs, int64_t njobs, int32_t ncomp, const int32_t ratio[3],
                             int32_t spacedim, int32_t elem_bytes, int32_t device, ghx_xfer **out) {
  if (!out || !check_common(njobs, jobs, ncomp, ratio, spacedim, elem_bytes, "ghx_average_down"))
    return GHX_EINVAL;
  int64_t rpow = 1;
  for (int d = 0; d < 3; ++d) rpow *= ratio[d];
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
    if (d.rn[0] * d.rn[1] * d.rn[2] >= (1ll << 31)) {
      set_error("ghx_average_down: job " + std::to_string(j) + ": region too large (>= 2^31 cells)");
      return GHX_EINVAL;
    }
    total += d.rn[0] * d.rn[1] * d.rn[2];
    dj.push_back(d);
  }
  ghx_xfer *x = new (std::nothrow) ghx_xfer();
  if (!x) {
    set_error("ghx_average_down: out of memory");
    return GHX_ENOMEM;
  }
  x->kind = 1;
  x->device = device;
  x->total = total;
  x->ncomp = ncomp;
  for (int d = 0; d < 3; ++d) x->r[d] = ratio[d];
  x->spacedim = spacedim;
  x->elem_bytes = elem_bytes;
  x->rpow = rpow;
  if (int rc = xfer_upload(x, dj, "ghx_average_down_prepare")) {
    delete x;
    return rc;
  }
  *out = x;
  return GHX_OK;
}

int ghx_advance_prepare(const ghx_stencil_job *jobs, int64_t njobs, const double coef[3], int32_t spacedim,
                        int32_t elem_bytes, int32_t layout, int32_t device, ghx_xfer **out) {
  if (layout != GHX_ADVANCE_TILES && layout != GHX_ADVANCE_CELLS) {
    set_error("ghx_advance: layout must be GHX_ADVANCE_TILES or GHX_ADVANCE_CELLS");
    return GHX_EINVAL;
  }
  const int32_t one[3] = {1, 1, 1};
  if (!out || !coef || !check_common(njobs, jobs, 1, one, spacedim, elem_bytes, "ghx_advance")) return GHX_EINVAL;
  std::vector<DevAvgJob> dj;
  dj.reserve(njobs);
  int64_t total = 0;
  for (int64_t j = 0; j < njobs; ++j) {
    const ghx_stencil_job &J = jobs[j];
    const int64_t *R = J.region;
    if (R[3] < R[0] || R[4] < R[1] || R[5] < R[2]) continue;
    int64_t glo[3], ghi[3];  // the stencil reads one cell around the region on axes < spacedim
    for (int d = 0; d < 3; ++d) {
      glo[d] = R[d] - (d < spacedim ? 1 : 0);
      ghi[d] = R[3 + d] + (d < spacedim ? 1 : 0);
    }
    if (!inside(J.src_box, glo, ghi) || !inside(J.dst_box, R, R + 3)) {
      set_error("ghx_advance: job " + std::to_string(j) + ": region (grown by 1) outside the source or "
                "destination fab");
      return GHX_EINVAL;
    }
    if (!J.src || !J.dst) {
      set_error("ghx_advance: null fab pointer");
      return GHX_EINVAL;
    }
    DevAvgJob d;
    std::memset(&d, 0, sizeof(d));
    d.fine = reinterpret_cast<uint64_t>(J.src);
    d.crse = reinterpret_cast<uint64_t>(J.dst);
    d.f = geo(J.src_box);
    d.c = geo(J.dst_box);
    for (int a = 0; a < 3; ++a) {
      d.rlo[a] = R[a];
      d.rn[a] = R[3 + a] - R[a] + 1;
    }
    d.start = total;
    if (d.rn[0] * d.rn[1] * d.rn[2] >= (1ll << 31)) {
      set_error("ghx_advance: job " + std::to_string(j) + ": region too large (>= 2^31 cells)");
      return GHX_EINVAL;
    }
    total += d.rn[0] * d.rn[1] * d.rn[2];
    dj.push_back(d);
  }
  ghx_xfer *x = new (std::nothrow) ghx_xfer();
  if (!x) {
    set_error("ghx_advance: out of memory");
    return GHX_ENOMEM;
  }
  x->kind = layout == GHX_ADVANCE_TILES ? 2 : 3;
  x->device = device;
  x->total = total;
  x->spacedim = spacedim;
  x->elem_bytes = elem_bytes;
  for (int d = 0; d < 3; ++d) x->coef[d] = coef[d];
  if (int rc = xfer_upload(x, dj, "ghx_advance_prepare")) {
    delete x;
    return rc;
  }
  *out = x;
  return GHX_OK;
}

int ghx_xfer_run(ghx_xfer *x, void *stream) {
  if (!x) {
    set_error("ghx_xfer_run: null handle");
    return GHX_EINVAL;
  }
  return xfer_launch(x, static_cast<cudaStream_t>(stream));
}

int64_t ghx_xfer_cells(const ghx_xfer *x) { return x ? x->total : 0; }

void ghx_xfer_free(ghx_xfer *x) {
  if (!x) return;
  if (x->djobs) {
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != x->device) cudaSetDevice(x->device);
    cudaFree(x->djobs);  // synchronising: no launch of this handle is in flight afterwards
    if (x->dtasks) cudaFree(x->dtasks);
    if (prev != x->device) cudaSetDevice(prev);
  }
  delete x;
}

int ghx_interp(const ghx_interp_job *jobs, int64_t njobs, int32_t ncomp, const int32_t ratio[3], int32_t spacedim,
               int32_t scheme, int32_t elem_bytes, void *stream) {
  int dev = 0;
  cudaGetDevice(&dev);
  ghx_xfer *x = nullptr;
  if (int rc = ghx_interp_prepare(jobs, njobs, ncomp, ratio, spacedim, scheme, elem_bytes, dev, &x)) return rc;
  const int rc = ghx_xfer_run(x, stream);
  ghx_xfer_free(x);
  return rc;
}

int ghx_average_down(const ghx_avgdown_job *jobs, int64_t njobs, int32_t ncomp, const int32_t ratio[3],
                     int32_t spacedim, int32_t elem_bytes, void *stream) {
  int dev = 0;
  cudaGetDevice(&dev);
  ghx_xfer *x = nullptr;
  if (int rc = ghx_average_down_prepare(jobs, njobs, ncomp, ratio, spacedim, elem_bytes, dev, &x)) return rc;
  const int rc = ghx_xfer_run(x, stream);
  ghx_xfer_free(x);
  return rc;
}

}  // extern "C"
