// Fused ghost-exchange executor for sm_100a (B200).
//
// Replaces _execute_plan (/root/reference/pkg/src/miniamr_core/comm.py:316-380):
// the reference runs one numpy slice copy per segment for the local phase,
// packs each peer's segments into an arena buffer, hands it over the Bus and
// unpacks it on the receiver.  Here every rank compiles its share of the
// plan into a device tag table once (per storage layout) and a single
// launch of ghx_copy_kernel moves all of it:
//
//   * GHX_EXEC_DIRECT  local tags + remote tags stored straight into the
//                      peer's fab (same-device pointer, peer-mapped pointer
//                      or CUDA-IPC mapping): pack + send + unpack fused;
//   * GHX_EXEC_LOCAL   local tags only;
//   * GHX_EXEC_PACK / GHX_EXEC_UNPACK  the NCCL fallback's pack and unpack
//                      (same per-peer F-order buffer layout as comm.py:341-377).
//
// Work decomposition
//   * each tag is flattened to (x/vec, y, z, comp) with the widest raw-word
//     vector (16/8/4 B) its alignment allows (rows whose src and dst share
//     the same 16-byte phase are peeled into head/body/tail);
//   * a warp task is TWO chunks of 32*kU vectors: either a tag and its
//     mirror (the tag that writes the other half of the same 32-byte
//     sectors, e.g. fab A's x-lo ghosts <- fab L's last valid columns and
//     L's x-hi ghosts <- A's first valid columns), so both halves of every
//     touched sector are read and rewritten together and L2 merges the
//     partial-sector writes instead of refilling them from HBM; or two
//     consecutive chunks of one tag;
//   * every lane issues its 2*kU vector loads before any store;
//   * the grid is persistent; each warp owns a contiguous range of tasks,
//     so the two tag descriptors it needs stay cached in shared memory;
//   * descriptors carry absolute base addresses, bound once per pointer
//     table by ghx_bind_kernel (no pointer-table load on the critical path).
// Values are copied as raw words, so NaN payloads survive bit-exactly.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <tuple>
#include <vector>

#include "ghx_internal.h"

using ghx::Box;
using ghx::Piece;
using ghx::set_error;

namespace {

#ifndef GHX_KU
#define GHX_KU 4
#endif
#ifndef GHX_MINB
#define GHX_MINB 2  // 2 x 256 threads per SM (<= 128 registers, no spills): +10-40 % over 1 (profiles/)
#endif
constexpr int kU = GHX_KU;          // vectors per lane per chunk
constexpr int kChunk = 32 * kU;     // vectors per chunk (a task has two)
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kSwapSlots = 8;
// task kinds (int4 .z): >= -1 copy / pair, -2 sector swap, -3 chain, -4 ring,
// -5 bulk rows, -6 tile ring, <= kFillTask sector fill (.z = kFillTask - mate)
constexpr int kFillTask = -16;
#ifndef GHX_CHAIN_ROWS
#define GHX_CHAIN_ROWS 16
#endif
constexpr int kChainRows = GHX_CHAIN_ROWS;  // rows per chain task
#ifndef GHX_CHAIN_R
#define GHX_CHAIN_R 2
#endif

std::atomic<int64_t> g_launches{0};

struct FastDiv {
  uint32_t d, m, s;
};

FastDiv make_div(uint32_t d) {
  FastDiv f{d, 0, 0};
  if (d <= 1) return f;
  uint32_t l = 0;
  while ((1ull << l) < d) ++l;  // ceil(log2 d)
  const uint32_t p = 31 + l;
  f.m = (uint32_t)(((1ull << p) + d - 1) / d);
  f.s = p - 32;
  return f;
}

struct __align__(16) DevTag {
  uint64_t src, dst;         // byte address of element (0,0,0,0); bound per pointer table
  int64_t src_sz, dst_sz;    // z stride, vectors
  int64_t src_sc, dst_sc;    // component stride, vectors
  int32_t src_sy, dst_sy;    // y stride, vectors
  uint32_t nvec;             // nxv * ny * nz * nc
  uint32_t nxv, ny, nz;
  uint32_t mx, my, mz;       // fast-divmod multipliers
  uint8_t sx, sy, sz, vlog;  // shifts, log2(vector bytes)
  int32_t src_ptr, dst_ptr;  // pointer-table slots (bind only)
  int64_t src_off, dst_off;  // vectors from the slot's base (bind only)
};
static_assert(sizeof(DevTag) == 112, "DevTag layout");
constexpr int kTagVec = sizeof(DevTag) / 16;

__device__ __forceinline__ uint32_t fdiv(uint32_t n, uint32_t d, uint32_t m, uint32_t s) {
  return d == 1 ? n : (__umulhi(n, m) >> s);
}

// Load flavours (template LD): 0 = ld.global.nc.L1::no_allocate (read-only
// path), 1 = ld.global.L1::no_allocate, 2 = ld.global.cg (L2 only),
// 3 = ld.global.cs (streaming), 4 = ld.global (default caching).
#define GHX_LD(SUFFIX, TYPE, ...)                                                        \
  if (LD == 0)                                                                           \
    asm volatile("ld.global.nc.L1::no_allocate" SUFFIX : __VA_ARGS__);                  \
  else if (LD == 1)                                                                      \
    asm volatile("ld.global.L1::no_allocate" SUFFIX : __VA_ARGS__);                     \
  else if (LD == 2)                                                                      \
    asm volatile("ld.global.cg" SUFFIX : __VA_ARGS__);                                  \
  else if (LD == 3)                                                                      \
    asm volatile("ld.global.cs" SUFFIX : __VA_ARGS__);                                  \
  else                                                                                   \
    asm volatile("ld.global" SUFFIX : __VA_ARGS__);

template <int LD>
__device__ __forceinline__ uint4 ld16(const void *p) {
  uint4 r;
  GHX_LD(".v4.u32 {%0,%1,%2,%3}, [%4];", uint4, "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p))
  return r;
}
template <int LD>
__device__ __forceinline__ uint2 ld8(const void *p) {
  uint2 r;
  GHX_LD(".v2.u32 {%0,%1}, [%2];", uint2, "=r"(r.x), "=r"(r.y) : "l"(p))
  return r;
}
template <int LD>
__device__ __forceinline__ uint32_t ld4(const void *p) {
  uint32_t r;
  GHX_LD(".u32 %0, [%1];", uint32_t, "=r"(r) : "l"(p))
  return r;
}

struct u8x32 {
  uint32_t w[8];
};
template <int LD>
__device__ __forceinline__ u8x32 ld32(const void *p) {
  u8x32 r;
  GHX_LD(".v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];", u8x32, "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]),
         "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]), "=r"(r.w[6]), "=r"(r.w[7]) : "l"(p))
  return r;
}
// store cache qualifier (experiment knob, e.g. -DGHX_ST_Q='".cs"'); default: plain st.global
#ifdef GHX_ST_Q
#define GHX_ST_ASM 1
#else
#define GHX_ST_Q ""
#define GHX_ST_ASM 0
#endif
__device__ __forceinline__ void st32(void *p, const uint32_t (&w)[8]) {
  asm volatile("st.global" GHX_ST_Q ".v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(w[0]), "r"(w[1]), "r"(w[2]),
               "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
               : "memory");
}

// element offset (in vectors) of flattened vector index v, for src or dst
template <bool SRC>
__device__ __forceinline__ int64_t vec_offset(const DevTag &t, uint32_t v) {
  const uint32_t r = fdiv(v, t.nxv, t.mx, t.sx);
  const uint32_t r2 = fdiv(r, t.ny, t.my, t.sy);
  const uint32_t c = fdiv(r2, t.nz, t.mz, t.sz);
  const uint32_t x = v - r * t.nxv, y = r - r2 * t.ny, z = r2 - c * t.nz;
  return SRC ? (int64_t)x + (int64_t)y * t.src_sy + (int64_t)z * t.src_sz + (int64_t)c * t.src_sc
             : (int64_t)x + (int64_t)y * t.dst_sy + (int64_t)z * t.dst_sz + (int64_t)c * t.dst_sc;
}

#ifndef GHX_HOST_CONT
#define GHX_HOST_CONT 0  // experiment knob (scripts/build_variants.sh); measured slower, see DESIGN.md
#endif
// CONT (fabs in host memory): an isolated 16-byte row (edge / corner tags,
// one vector per row) is read as its aligned 32-byte sector -- over PCIe a
// 16-byte read costs twice a 32-byte one (profiles/r01_pcie_probe.txt:
// 0.28 vs 0.57 G requests/s); the sector never crosses a page, and the
// other half is discarded.
template <int LD, bool CONT = false>
__device__ __forceinline__ void load_chunk(const DevTag &t, uint32_t start, int lane, uint4 (&val)[kU]) {
  const char *base = reinterpret_cast<const char *>(t.src);
  const int vl = t.vlog;
  const bool cont = CONT && vl == 4 && t.nxv == 1;
#pragma unroll
  for (int u = 0; u < kU; ++u) {
    const uint32_t v = start + (uint32_t)(u * 32 + lane);
    if (v < t.nvec) {
      const char *p = base + (vec_offset<true>(t, v) << vl);
      if (cont) {
        const u8x32 s = ld32<LD>(reinterpret_cast<const char *>(reinterpret_cast<uintptr_t>(p) & ~uintptr_t(31)));
        val[u] = (reinterpret_cast<uintptr_t>(p) & 16) ? make_uint4(s.w[4], s.w[5], s.w[6], s.w[7])
                                                       : make_uint4(s.w[0], s.w[1], s.w[2], s.w[3]);
      } else if (vl == 4)
        val[u] = ld16<LD>(p);
      else if (vl == 3) {
        const uint2 q = ld8<LD>(p);
        val[u].x = q.x;
        val[u].y = q.y;
      } else
        val[u].x = ld4<LD>(p);
    }
  }
}

__device__ __forceinline__ void store_chunk(const DevTag &t, uint32_t start, int lane, const uint4 (&val)[kU]) {
  char *base = reinterpret_cast<char *>(t.dst);
  const int vl = t.vlog;
#pragma unroll
  for (int u = 0; u < kU; ++u) {
    const uint32_t v = start + (uint32_t)(u * 32 + lane);
    if (v < t.nvec) {
      char *p = base + (vec_offset<false>(t, v) << vl);
#if GHX_ST_ASM
      if (vl == 4)
        asm volatile("st.global" GHX_ST_Q ".v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(val[u].x), "r"(val[u].y),
                     "r"(val[u].z), "r"(val[u].w) : "memory");
      else if (vl == 3)
        asm volatile("st.global" GHX_ST_Q ".v2.u32 [%0], {%1,%2};" ::"l"(p), "r"(val[u].x), "r"(val[u].y) : "memory");
      else
        asm volatile("st.global" GHX_ST_Q ".u32 [%0], %1;" ::"l"(p), "r"(val[u].x) : "memory");
#else
      if (vl == 4)
        *reinterpret_cast<uint4 *>(p) = val[u];
      else if (vl == 3)
        *reinterpret_cast<uint2 *>(p) = make_uint2(val[u].x, val[u].y);
      else
        *reinterpret_cast<uint32_t *>(p) = val[u].x;
#endif
    }
  }
}

// Sector swap for a mirror pair of 16-byte-row tags (T1 described by t,
// T2 implied): T1 writes the low half of sector SA (fab A's first 32 bytes
// of the row: ghost | first valid columns) from the low half of sector SL
// (fab L's last 32 bytes: last valid columns | ghost); T2 writes the high
// half of SL from the high half of SA.  Both sectors end up holding
// (SL.lo, SA.hi): each lane reads two whole sectors and writes them back
// whole, so L2 never refills a partially written sector from HBM.
#ifndef GHX_SWAP_PASSES
#define GHX_SWAP_PASSES 2  // load/store passes per chunk (1: all kU vectors' loads before any store)
#endif
template <int LD>
__device__ __forceinline__ void swap_chunk(const DevTag &t, uint32_t start, int lane) {
  constexpr int kS = kU / GHX_SWAP_PASSES;
  char *const da = reinterpret_cast<char *>(t.dst);
  char *const sl = reinterpret_cast<char *>(t.src);
#pragma unroll 1
  for (int h = 0; h < GHX_SWAP_PASSES; ++h) {
    uint4 lo[kS], hi[kS];
#pragma unroll
    for (int u = 0; u < kS; ++u) {
      const uint32_t v = start + (uint32_t)((h * kS + u) * 32 + lane);
      if (v < t.nvec) {
        hi[u] = ld16<LD>(da + (vec_offset<false>(t, v) << 4) + 16);
        lo[u] = ld16<LD>(sl + (vec_offset<true>(t, v) << 4));
      }
    }
#pragma unroll
    for (int u = 0; u < kS; ++u) {
      const uint32_t v = start + (uint32_t)((h * kS + u) * 32 + lane);
      if (v < t.nvec) {
        const uint32_t w[8] = {lo[u].x, lo[u].y, lo[u].z, lo[u].w, hi[u].x, hi[u].y, hi[u].z, hi[u].w};
        st32(da + (vec_offset<false>(t, v) << 4), w);
        st32(sl + (vec_offset<true>(t, v) << 4), w);
      }
    }
  }
}

// Sector fill (unpack of 16-byte x-ghost rows from a receive buffer): the
// ghost half of a 32-byte sector is stored together with the sector's other
// half -- valid cells of the same fab, which no tag writes, read first -- so
// the sector is written whole and L2 never merges a partial sector with HBM
// (a 16-byte ghost store costs a line fill plus a write-back; the whole
// sector costs what a local sector swap does).  The host enables it per tag
// when every row's vector sits in the same sector half (dst_off & 1, for a
// 32-byte aligned fab base) and the other half is valid cells; a fab base
// that is only 16-byte aligned runs the task as a plain copy instead.
__device__ __forceinline__ bool fill_aligned(const DevTag &t) {
  return ((t.dst - ((uint64_t)t.dst_off << 4)) & 31) == 0;
}

template <int LD>
__device__ __forceinline__ void fill_chunk(const DevTag &t, uint32_t start, int lane) {
  constexpr int kS = kU / GHX_SWAP_PASSES;
  const char *sb = reinterpret_cast<const char *>(t.src);
  char *db = reinterpret_cast<char *>(t.dst);
  const bool ghost_hi = t.dst_off & 1;  // the ghost is the sector's high half
#pragma unroll 1
  for (int h = 0; h < GHX_SWAP_PASSES; ++h) {
    uint4 g[kS], o[kS];
#pragma unroll
    for (int u = 0; u < kS; ++u) {
      const uint32_t v = start + (uint32_t)((h * kS + u) * 32 + lane);
      if (v < t.nvec) {
        g[u] = ld16<LD>(sb + (vec_offset<true>(t, v) << 4));
        o[u] = ld16<LD>(db + (vec_offset<false>(t, v) << 4) + (ghost_hi ? -16 : 16));
      }
    }
#pragma unroll
    for (int u = 0; u < kS; ++u) {
      const uint32_t v = start + (uint32_t)((h * kS + u) * 32 + lane);
      if (v < t.nvec) {
        const uint4 lo = ghost_hi ? o[u] : g[u], hi = ghost_hi ? g[u] : o[u];
        const uint32_t w[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
        st32(db + (vec_offset<false>(t, v) << 4) - (ghost_hi ? 16 : 0), w);
      }
    }
  }
}

// A chain task runs the sector swaps of every seam of one chain of fabs
// (e.g. the x-line L|A|R|... of a uniform decomposition) over the same rows
// in one warp: lane = (seam j, row offset).  Row r+1 of seam (L,A) and row r
// of seam (A,R) touch the two halves of the same 64 bytes of A (end of row
// r, start of row r+1), so their loads coalesce into one line request.
template <int LD>
__device__ __forceinline__ void chain_task(const DevTag *__restrict__ tags, const int *__restrict__ chain,
                                           int off, int k, uint32_t start, uint32_t rows, int lane) {
  const int per = 32 / k;
  const int j = lane / per;
  const int rl = lane - j * per;
  if (j >= k) return;
  const DevTag &t = tags[__ldg(chain + off + j)];
  char *const da = reinterpret_cast<char *>(__ldg(&t.dst));
  char *const sl = reinterpret_cast<char *>(__ldg(&t.src));
  const uint32_t nvec = __ldg(&t.nvec), ny = __ldg(&t.ny), nz = __ldg(&t.nz);
  const uint32_t my = __ldg(&t.my), mz = __ldg(&t.mz);
  const uint32_t shy = __ldg(&t.sy), shz = __ldg(&t.sz);
  const int64_t dsy = __ldg(&t.dst_sy), dsz = __ldg(&t.dst_sz), dsc = __ldg(&t.dst_sc);
  const int64_t ssy = __ldg(&t.src_sy), ssz = __ldg(&t.src_sz), ssc = __ldg(&t.src_sc);
  const uint32_t end = min(nvec, start + rows);
  constexpr int R = GHX_CHAIN_R;  // rows per lane per iteration (2R loads in flight)
  // only the halves that survive are loaded: the new content of both
  // sectors is (L-sector low half | A-sector high half)
#pragma unroll 1
  for (uint32_t r0 = start + rl; r0 < end; r0 += R * per) {
    uint4 lo[R], hi[R];
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const uint32_t r = r0 + u * per;
      if (r < end) {
        const uint32_t q = fdiv(r, ny, my, shy);
        const uint32_t c = fdiv(q, nz, mz, shz);
        const uint32_t y = r - q * ny, z = q - c * nz;
        hi[u] = ld16<LD>(da + (((int64_t)y * dsy + (int64_t)z * dsz + (int64_t)c * dsc) << 4) + 16);
        lo[u] = ld16<LD>(sl + (((int64_t)y * ssy + (int64_t)z * ssz + (int64_t)c * ssc) << 4));
      }
    }
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const uint32_t r = r0 + u * per;
      if (r < end) {
        const uint32_t q = fdiv(r, ny, my, shy);
        const uint32_t c = fdiv(q, nz, mz, shz);
        const uint32_t y = r - q * ny, z = q - c * nz;
        const uint32_t w[8] = {lo[u].x, lo[u].y, lo[u].z, lo[u].w, hi[u].x, hi[u].y, hi[u].z, hi[u].w};
        st32(da + (((int64_t)y * dsy + (int64_t)z * dsz + (int64_t)c * dsc) << 4), w);
        st32(sl + (((int64_t)y * ssy + (int64_t)z * ssz + (int64_t)c * ssc) << 4), w);
      }
    }
  }
}

// A ring task runs the x-face sector swaps of a periodic x-line of k fabs
// F_0..F_{k-1} (ring tags T_j: F_j's last sector <-> F_{j+1}'s first
// sector, all with the same row geometry) as *seam chunks*: the last
// sector of row y and the first sector of row y+1 of a fab are adjacent
// 64 bytes, so a lane pair owns a chunk and reads and writes it with one
// coalesced 64-byte access each (the swap form needs two 32-byte reads and
// two writes to different fabs; over PCIe the transaction count is the
// cost, scripts/microbench/pcie_probe.cu).  Lane pair p = (fab j = p % k,
// stream s = p / k); a stream walks one (z, comp) column of the tag's rows.
// Per column, chunk c = (S0 row c, S1 row c+1), c = -1 .. ny-1, where S0 =
// a fab's last sector (hi valid | hi ghost) and S1 = its first sector (lo
// ghost | lo valid).  New contents (x-ring neighbours, same row y):
//   S0(j, y) = [S0(j, y).lo | S1(j+1, y).hi],  S1(j, y) = [S0(j-1, y).lo | S1(j, y).hi]
// At step c a lane loads its sector of chunk c, receives its neighbour half
// with one shuffle and writes its sector of chunk c-1 (side 0 waits for
// S1(j+1, c-1), loaded two steps earlier; side 1 for S0(j-1, c), loaded
// this step).  Every sector is loaded before it is stored, so loads are
// issued kRingAhead steps ahead.  A task covers kRingRows rows: the rows
// each side writes are exactly the rows it loads, so tasks need no halo.
constexpr int kRingAhead = 2;
constexpr int kRingRows = 16;  // rows per ring task (a task writes rows [y0, y0 + kRingRows) of its columns)

template <int LD>
__device__ __forceinline__ void ring_task(const DevTag *__restrict__ tags, const int *__restrict__ ring, int off,
                                          int kw, int q0, int lane) {
  const int k = kw & 31, y0 = (kw >> 5) * kRingRows;
  const int p = lane >> 1, side = lane & 1;
  const int j = p % k, sidx = p / k;
  const int jn = (j + 1) % k, jp = (j + k - 1) % k;
  // my sector's tag: side 0 = T_j's source (F_j last sector), side 1 = T_{j-1}'s destination (F_j first sector)
  const DevTag &t = tags[__ldg(ring + off + (side ? jp : j))];
  const char *base = reinterpret_cast<const char *>(side ? __ldg(&t.dst) : __ldg(&t.src));
  const int64_t sy = side ? __ldg(&t.dst_sy) : __ldg(&t.src_sy);
  const int64_t sz = side ? __ldg(&t.dst_sz) : __ldg(&t.src_sz);
  const int64_t sc = side ? __ldg(&t.dst_sc) : __ldg(&t.src_sc);
  const int ny_tag = (int)__ldg(&t.ny), nz = (int)__ldg(&t.nz);
  const int ncol = (int)(__ldg(&t.nvec) / (uint32_t)(ny_tag * nz));
  const int y1 = min(ny_tag, y0 + kRingRows);  // rows [y0, y1) of this task
  const int q = q0 + sidx;
  const bool active = sidx < (32 / (2 * k)) && q < nz * ncol;
  const int src = side ? 2 * (jp + k * sidx) : 2 * (jn + k * sidx) + 1;  // whose half I receive
  const char *col = base + ((((int64_t)(q % nz)) * sz + (int64_t)(q / max(nz, 1)) * sc) << 4);
  // row r of my sector: side 0 holds row c at step c, side 1 holds row c+1
  auto addr = [&](int r) { return const_cast<char *>(col + (((int64_t)r * sy) << 4)); };
  auto my_row = [&](int c) { return side ? c + 1 : c; };
  auto loadable = [&](int c) { const int r = my_row(c); return active && r >= y0 && r < y1; };
  // loads stay whole 32-byte sectors (one coalesced 64-byte access per lane
  // pair); each side keeps only the half it needs: side 0 the low half of
  // its S0 (valid, kept), side 1 the high half of its S1 (valid, kept)
  u8x32 pre[kRingAhead + 1];
  uint4 h0 = make_uint4(0, 0, 0, 0), h1 = h0, h2 = h0;
#pragma unroll
  for (int a = 0; a <= kRingAhead; ++a) {
    const int c = y0 - 1 + a;
    if (loadable(c)) pre[a] = ld32<LD>(addr(my_row(c)));
  }
#pragma unroll 1
  for (int c = y0 - 1; c <= y1; ++c) {
    h2 = h1;
    h1 = h0;
    h0 = side ? make_uint4(pre[0].w[4], pre[0].w[5], pre[0].w[6], pre[0].w[7])
              : make_uint4(pre[0].w[0], pre[0].w[1], pre[0].w[2], pre[0].w[3]);
#pragma unroll
    for (int a = 0; a < kRingAhead; ++a) pre[a] = pre[a + 1];
    if (loadable(c + kRingAhead + 1)) pre[kRingAhead] = ld32<LD>(addr(my_row(c + kRingAhead + 1)));
    // side 0 gives its S0 row c low half (to side 1 of F_{j+1}); side 1 gives
    // its S1 row c-1 high half (to side 0 of F_{j-1})
    const uint4 give = side ? h2 : h0;
    uint4 got;
    got.x = __shfl_sync(0xffffffffu, give.x, src);
    got.y = __shfl_sync(0xffffffffu, give.y, src);
    got.z = __shfl_sync(0xffffffffu, give.z, src);
    got.w = __shfl_sync(0xffffffffu, give.w, src);
    if (!active) continue;
    const int r = side ? c : c - 1;  // side 0 writes S0 row c-1, side 1 writes S1 row c
    if (r >= y0 && r < y1) {
      const uint4 lo = side ? got : h1, hi = side ? h1 : got;
      const uint32_t w[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
      st32(addr(r), w);
    }
  }
}

// Tile ring task: the same seam chunks, but one warp instruction covers k
// fabs x R = 16/k CONSECUTIVE chunks of one (z, comp) column, and the warp
// steps down R chunks at a time (ring_task covers k fabs x 16/k columns, one
// chunk each).  Over PCIe the host side serves a warp's requests faster when
// they fall on neighbouring rows (scripts/microbench/pcie_ring_probe.cu:
// 4.0 ns per seam read+write against 4.3 for the column layout; the seam
// read of the next step is issued before this step's write).
// Chunk c of fab j = [S0 row c | S1 row c+1]; its new contents are
//   q0 = S0(j,c).lo (kept)        q1 = S1(j+1,c).hi = chunk(j+1,c-1).q3
//   q2 = S0(j-1,c+1).lo = chunk(j-1,c+1).q0        q3 = S1(j,c+1).hi (kept)
// Lane (j, r, side) holds chunk c = c0 + t*R + r of fab j at step t (side 0
// the S0 sector, side 1 the S1 sector).  q1 comes from lane (j+1, r-1, 1)
// this step, or for r = 0 from lane (j+1, R-1, 1)'s previous step; q2 from
// lane (j-1, r+1, 0) this step, or for r = R-1 from lane (j-1, 0, 0)'s next
// step (already loaded as the prefetch): one shuffle per step, every lane
// offering exactly the half some other lane needs.  A task owns chunks
// [c0, c0 + nch) of its column; chunks run from -1 (S1 row 0 only) to ny-1
// (S0 row ny-1 only), and only sectors of rows in [0, ny) are touched.
#ifndef GHX_RING_W16
#define GHX_RING_W16 0
#endif
template <int LD>
__device__ __forceinline__ void tile_ring_task(const DevTag *__restrict__ tags, const int *__restrict__ ring, int off,
                                               int q, int kw, int lane) {
  const int k = kw & 31;
  const int c0 = ((kw >> 5) & 0xFFFF) - 1;
  const int span = (kw >> 21) & 0x1FF;  // chunks owned: [c0, c0 + span)
  const int R = 16 / k;
  const int steps = (span + R - 1) / R;
  const int p = lane >> 1, side = lane & 1;
  const int j = p % k, r = p / k;
  const bool active = r < R;
  const int jn = (j + 1) % k, jp = (j + k - 1) % k;
  const DevTag &t = tags[__ldg(ring + off + (side ? jp : j))];
  const char *base = reinterpret_cast<const char *>(side ? __ldg(&t.dst) : __ldg(&t.src));
  const int64_t sy = side ? __ldg(&t.dst_sy) : __ldg(&t.src_sy);
  const int64_t sz = side ? __ldg(&t.dst_sz) : __ldg(&t.src_sz);
  const int64_t sc = side ? __ldg(&t.dst_sc) : __ldg(&t.src_sc);
  const int ny = (int)__ldg(&t.ny), nz = (int)__ldg(&t.nz);
  const char *col = base + ((((int64_t)(q % nz)) * sz + (int64_t)(q / max(nz, 1)) * sc) << 4);
  const int c_end = min(c0 + span, ny);  // chunks run -1 .. ny-1
  // the row of my sector in chunk c: side 0 -> row c (S0), side 1 -> row c + 1 (S1)
  auto row_of = [&](int c) { return side ? c + 1 : c; };
  auto ok = [&](int c) { const int y = row_of(c); return active && y >= 0 && y < ny; };
  auto addr = [&](int c) { return const_cast<char *>(col + (((int64_t)row_of(c) * sy) << 4)); };
  // source lanes of the one shuffle per step
  const int src = side ? 2 * (jp + k * ((r + 1) % R)) : 2 * (jn + k * ((r + R - 1) % R)) + 1;
  u8x32 cur, nxt;
  uint4 prev_hi = make_uint4(0, 0, 0, 0);
  // halo: lane (j, R-1, 1) starts with chunk c0-1's S1 high half (q3) for lane (jp, 0, 0)
  if (side && r == R - 1 && ok(c0 - 1)) {
    const u8x32 h = ld32<LD>(addr(c0 - 1));
    prev_hi = make_uint4(h.w[4], h.w[5], h.w[6], h.w[7]);
  }
  {
    const int c = c0 + r;
    if (ok(c)) cur = ld32<LD>(addr(c));
  }
#pragma unroll 1
  for (int s = 0; s < steps; ++s) {
    const int c = c0 + s * R + r;
    const int cn = c + R;
    // next step's sector (lane (j, 0, 0) also serves the last step's halo)
    if (ok(cn) && (s + 1 < steps || (r == 0 && !side))) nxt = ld32<LD>(addr(cn));
    // what I offer: side 0 my q0 (or, at r = 0, the next step's q0); side 1
    // my q3 (or, at r = R-1, the previous step's q3)
    uint4 give;
    if (side)
      give = (r == R - 1) ? prev_hi : make_uint4(cur.w[4], cur.w[5], cur.w[6], cur.w[7]);
    else
      give = (r == 0) ? make_uint4(nxt.w[0], nxt.w[1], nxt.w[2], nxt.w[3])
                      : make_uint4(cur.w[0], cur.w[1], cur.w[2], cur.w[3]);
    uint4 got;
    got.x = __shfl_sync(0xffffffffu, give.x, src);
    got.y = __shfl_sync(0xffffffffu, give.y, src);
    got.z = __shfl_sync(0xffffffffu, give.z, src);
    got.w = __shfl_sync(0xffffffffu, give.w, src);
    if (ok(c) && c < c_end) {
#if GHX_RING_W16
      // only the ghost half: the pair's two 16-B stores are the 32 adjacent
      // ghost bytes of the seam (one PCIe write, the kept halves untouched)
      char *g = addr(c) + (side ? 0 : 16);
      asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(g), "r"(got.x), "r"(got.y), "r"(got.z), "r"(got.w)
                   : "memory");
#else
      uint32_t w[8];
      if (side) {
        w[0] = got.x, w[1] = got.y, w[2] = got.z, w[3] = got.w;
        w[4] = cur.w[4], w[5] = cur.w[5], w[6] = cur.w[6], w[7] = cur.w[7];
      } else {
        w[0] = cur.w[0], w[1] = cur.w[1], w[2] = cur.w[2], w[3] = cur.w[3];
        w[4] = got.x, w[5] = got.y, w[6] = got.z, w[7] = got.w;
      }
      st32(addr(c), w);
#endif
    }
    if (side && r == R - 1) prev_hi = make_uint4(cur.w[4], cur.w[5], cur.w[6], cur.w[7]);
    cur = nxt;
  }
}

// Seam task (host-memory pack / unpack of one fab's remote x faces, see
// seam_pair_hi): one column q (z, component) of rows; lane pair p takes seam
// chunk c = step * 16 + p - 1, side 0 moves H's row c, side 1 L's row c + 1.
// Pack reads the chunk's two 32-byte halves (adjacent lanes: one 64-byte
// PCIe read) and stores each side's 16-byte vector into its peer's slab;
// unpack reads the two slab vectors and stores them to the adjacent ghost
// halves (one PCIe write).
template <int LD>
__device__ __forceinline__ void seam_task(const DevTag &H, const DevTag &L, uint32_t q, bool pack, int lane) {
  const int p = lane >> 1, side = lane & 1;
  const int ny = (int)H.ny;
  const DevTag &T = side ? L : H;
#pragma unroll 1
  for (int c0 = -1; c0 < ny; c0 += 16) {
    const int c = c0 + p;
    const int row = side ? c + 1 : c;
    if (c >= ny || row < 0 || row >= ny) continue;
    const uint32_t v = (uint32_t)row + (uint32_t)ny * q;  // one vector per row
    const char *src = reinterpret_cast<const char *>(T.src) + (vec_offset<true>(T, v) << 4);
    char *dst = reinterpret_cast<char *>(T.dst) + (vec_offset<false>(T, v) << 4);
    uint4 val;
    if (pack) {  // side 0: [H.src | hg], side 1: [lg | L.src] -- the chunk's two halves
      const u8x32 h = ld32<LD>(side ? src - 16 : src);
      val = side ? make_uint4(h.w[4], h.w[5], h.w[6], h.w[7]) : make_uint4(h.w[0], h.w[1], h.w[2], h.w[3]);
    } else {
      val = ld16<LD>(src);
    }
    *reinterpret_cast<uint4 *>(dst) = val;
  }
}

// Bulk-row task (TMA 1-D bulk copies): rows of a 16-byte-vector tag are
// moved global -> shared -> global by the copy engine of the SM, one lane
// per row (cp.async.bulk with an mbarrier per warp), so a warp keeps
// kBulkBytes in flight without holding them in registers.  Only for tags
// whose source and destination do not alias (FillBoundary).
#ifndef GHX_BULK_BYTES
#define GHX_BULK_BYTES 8192
#endif
constexpr int kBulkBytes = GHX_BULK_BYTES;  // per-warp staging buffer (dynamic shared memory)

__device__ __forceinline__ void bulk_task(const DevTag &t, uint32_t r0, uint32_t nrows, int lane, char *sbuf,
                                          uint64_t *bar, uint32_t &phase) {
  const uint32_t row_bytes = t.nxv << 4;
  const uint32_t sbuf_s = (uint32_t)__cvta_generic_to_shared(sbuf);
  const uint32_t bar_s = (uint32_t)__cvta_generic_to_shared(bar);
  const uint32_t per = kBulkBytes / row_bytes;
  for (uint32_t b0 = 0; b0 < nrows; b0 += per) {
    const uint32_t n = min(per, nrows - b0);
    // previous batch's stores must have read the buffer before it is refilled
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __syncwarp();
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_s), "r"(n * row_bytes)
                   : "memory");
    __syncwarp();
    const uint32_t r = r0 + b0 + (uint32_t)lane;
    int64_t soff = 0, doff = 0;
    if ((uint32_t)lane < n) {
      const uint32_t q = fdiv(r, t.ny, t.my, t.sy);
      const uint32_t c = fdiv(q, t.nz, t.mz, t.sz);
      const uint32_t y = r - q * t.ny, z = q - c * t.nz;
      soff = ((int64_t)y * t.src_sy + (int64_t)z * t.src_sz + (int64_t)c * t.src_sc) << 4;
      doff = ((int64_t)y * t.dst_sy + (int64_t)z * t.dst_sz + (int64_t)c * t.dst_sc) << 4;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              sbuf_s + lane * row_bytes),
          "l"(t.src + soff), "r"(row_bytes), "r"(bar_s)
          : "memory");
    }
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done)
                   : "r"(bar_s), "r"(phase)
                   : "memory");
    phase ^= 1;
    if ((uint32_t)lane < n) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(t.dst + doff),
                   "r"(sbuf_s + lane * row_bytes), "r"(row_bytes)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
}

// cooperative 112-byte descriptor load into this warp's shared slot
__device__ __forceinline__ void fetch_tag(const DevTag *__restrict__ tags, int idx, DevTag *slot, int lane) {
  if (lane < kTagVec)
    reinterpret_cast<uint4 *>(slot)[lane] = __ldg(reinterpret_cast<const uint4 *>(tags + idx) + lane);
}

// In-kernel cross-rank synchronisation (process mode, one GPU per rank).
// Every rank owns an IPC-shared flag array of 3 * nranks uint64 slots:
// [0, n) the standalone barrier kernel's, [n, 2n) READY (rank p has started
// this exchange, so its earlier work on its fabs and receive slab is done),
// [2n, 3n) DONE (every store rank p pushed to me in this exchange is
// visible).  Values are the exchange epoch, monotonic and identical on all
// ranks, so a slot never needs resetting.
//   mode 1 (push kernel): each block's warp 0 signals READY to every peer on
//     entry; the remote tasks -- the first `nhead` tasks -- wait for their
//     peer's READY (once per warp per peer) while local tasks start at
//     once; the last warp to finish fences and signals DONE to every peer.
//   mode 2 (unpack kernel): a task reading peer p's receive slab waits for
//     p's DONE (each peer's slab is unpacked as soon as it lands), and block
//     0 waits for every peer's DONE (direct pushes into my fabs) before the
//     kernel can complete.
// Spins give up after timeout_ns and count a timeout (ghx_barrier_timeouts)
// instead of hanging the GPU when a peer rank dies.
constexpr int kSlotReady = 1, kSlotDone = 2;

struct SyncArgs {
  uint64_t *const *flags;   // device table: rank p's flag array as mapped here
  const int32_t *tag_peer;  // per tag: peer rank (push: destination, unpack: source), -1 local
  uint64_t epoch;
  uint64_t timeout_ns;
  int32_t rank, nranks;
  int32_t mode;             // 0 none, 1 push, 2 unpack / wait, 3 push + unpack (EXCHANGE_PACKED)
  int32_t nhead;            // mode 1: tasks [0, nhead) are remote
  int32_t pe0, pe1;         // phased executor: tasks [pe0, pe1) phase 1, [pe1, n) phase 2 (0, 0: no phases)
  const int32_t *peer_total;  // mode 3: push tasks per peer (a peer's DONE when they are all done)
};

__device__ unsigned int g_sync_timeouts = 0;

__device__ __forceinline__ uint64_t gtimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void flag_store(uint64_t *p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __noinline__ void flag_wait(const uint64_t *p, uint64_t epoch, uint64_t timeout_ns) {
  const uint64_t t0 = gtimer_ns();
  uint64_t v = 0;
  for (uint32_t it = 0;; ++it) {
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    if (v >= epoch) return;
    if ((it & 1023) == 1023 && gtimer_ns() - t0 > timeout_ns) {
      atomicAdd(&g_sync_timeouts, 1u);
      return;
    }
    __nanosleep(64);
  }
}

// every peer's slot `slot` of this rank's flag array reaches the epoch
__device__ __forceinline__ void wait_all_peers(const SyncArgs &s, int slot, int lane) {
  for (int p = lane; p < s.nranks; p += 32)
    if (p != s.rank) flag_wait(s.flags[s.rank] + slot * s.nranks + p, s.epoch, s.timeout_ns);
}

__device__ __forceinline__ void signal_all_peers(const SyncArgs &s, int slot, int lane) {
  for (int p = lane; p < s.nranks; p += 32)
    if (p != s.rank) flag_store(s.flags[p] + slot * s.nranks + s.rank, s.epoch);
}

}  // namespace

// Empty executors still take part in the protocol: mode 1 signals READY
// and DONE, mode 2 waits for every peer's DONE (direct-mode exit wait).
__global__ void ghx_sync_kernel(const SyncArgs sync) {
  const int lane = threadIdx.x;
  if (lane >= 32) return;
  if (sync.mode == 1 || sync.mode == 3) {
    __threadfence_system();
    signal_all_peers(sync, kSlotReady, lane);
    signal_all_peers(sync, kSlotDone, lane);
  }
  if (sync.mode == 2 || sync.mode == 3) wait_all_peers(sync, kSlotDone, lane);
}

// Resolve pointer-table slots into absolute addresses (once per table).
__global__ void ghx_bind_kernel(DevTag *tags, int ntags, void *const *__restrict__ ptrs) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ntags; i += gridDim.x * blockDim.x) {
    DevTag &t = tags[i];
    t.src = reinterpret_cast<uint64_t>(ptrs[t.src_ptr]) + ((uint64_t)t.src_off << t.vlog);
    t.dst = reinterpret_cast<uint64_t>(ptrs[t.dst_ptr]) + ((uint64_t)t.dst_off << t.vlog);
  }
}

// tasks: {tagA, startA, tagB (-1: none), startB}
// Dynamic schedule: warps grab batches of kBatch consecutive tasks from a
// per-executor counter (counter[0]); every warp counts itself out in
// counter[1] and the last one resets both, so the next launch (stream
// ordered) starts from zero without a memset.  Heavy tasks come first.
template <int LD, bool RING = false, bool BULK = false, bool FILL = false>
__global__ void __launch_bounds__(kThreads, RING ? 1 : GHX_MINB) ghx_copy_kernel(const DevTag *__restrict__ tags,
                                                            const int4 *__restrict__ tasks, int ntasks,
                                                            const int *__restrict__ chains,
                                                            unsigned long long *__restrict__ counter, int batch,
                                                            const SyncArgs sync) {
  __shared__ DevTag slots[kWarps][2];
  __shared__ DevTag swc[kWarps][kSwapSlots];  // direct-mapped cache of sector-swap descriptors
  __shared__ int swc_id[kWarps][kSwapSlots];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  DevTag &ta = slots[wib][0];
  DevTag &tb = slots[wib][1];
  int have_a = -1, have_b = -1;
  if (lane < kSwapSlots) swc_id[wib][lane] = -1;
  extern __shared__ __align__(128) char bulk_smem[];  // BULK: kWarps x kBulkBytes
  __shared__ __align__(8) uint64_t bulk_bar[kWarps];
  uint32_t bulk_phase = 0;
  if (BULK) {
    if (lane == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bulk_bar[wib])));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
  }
  if ((sync.mode == 1 || sync.mode == 3) && wib == 0) signal_all_peers(sync, kSlotReady, lane);
  if (sync.mode == 3 && blockIdx.x == 0 && wib == 0)
    for (int p = lane; p < sync.nranks; p += 32)  // peers this rank pushes nothing to: done already
      if (p != sync.rank && __ldg(sync.peer_total + p) == 0)
        flag_store(sync.flags[p] + kSlotDone * sync.nranks + sync.rank, sync.epoch);
  uint64_t peers_ok = 0;  // peers whose READY (mode 1) / DONE (mode 2) this warp has seen
  // phased executor: a warp passing into phase p (it grabbed a task of phase
  // p, so it will run no task of an earlier phase again) counts itself in
  // counter[2 + p - 1] and waits until every warp has; tasks are grabbed in
  // index order, so every waiter waits only for warps still running tasks
  const bool phased = sync.pe1 > 0 || sync.pe0 > 0;
  int my_phase = 0;
  const unsigned long long nwarps_all = (unsigned long long)gridDim.x * kWarps;
  auto pass_to = [&](int ph, bool wait) {
    while (my_phase < ph) {
      __syncwarp();
      __threadfence_system();  // my earlier phases' stores (host memory too) are visible
      __syncwarp();
      if (lane == 0) atomicAdd(counter + 2 + my_phase, 1ull);
      ++my_phase;
      if (wait) {
        if (lane == 0) {
          // bounded like the cross-rank waits: a grid that is not fully
          // resident (it must be) counts a timeout instead of hanging
          const uint64_t t0 = gtimer_ns();
          unsigned long long v = 0;
          for (uint32_t it = 0;; ++it) {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(counter + 2 + my_phase - 1) : "memory");
            if (v >= nwarps_all) break;
            if ((it & 1023) == 1023 && gtimer_ns() - t0 > sync.timeout_ns) {
              atomicAdd(&g_sync_timeouts, 1u);
              break;
            }
            __nanosleep(128);
          }
        }
        __syncwarp();
      }
    }
  };
  __syncwarp();
  // first batch static (warp id), later ones dynamic from an offset of one
  // batch per warp: no atomic -- and no contention of every warp on one
  // counter -- on the critical path of a warp's first task
  const unsigned long long static_tasks = (unsigned long long)gridDim.x * kWarps * batch;
  unsigned long long nb = ((unsigned long long)blockIdx.x * kWarps + wib) * batch;
#pragma unroll 1
  while (true) {
    const long long first = (long long)nb;
    if (first >= ntasks) break;
    if (lane == 0) nb = atomicAdd(counter, (unsigned long long)batch) + static_tasks;  // prefetch the next batch
    const int last = (int)min((long long)ntasks, first + batch);
    int4 tk = __ldg(tasks + first);
#pragma unroll 1
    for (int w = (int)first; w < last; ++w) {
      const int4 nxt = (w + 1 < last) ? __ldg(tasks + w + 1) : tk;
      if (phased) pass_to(w >= sync.pe1 ? 2 : (w >= sync.pe0 ? 1 : 0), true);
      if ((tk.z >= -1 || tk.z <= kFillTask || tk.z == -7 || tk.z == -8) &&
          (sync.mode >= 2 || (sync.mode == 1 && w < sync.nhead))) {
        // a remote push waits for the peer's READY, an unpack for its DONE
        // (both tags of a pair task: they may belong to different peers).
        // Mode 3 tells the two apart by the tag's peer (+ 64: unpack) and
        // keeps READY peers in bits 0-31 and DONE peers in bits 32-63.
#pragma unroll 1
        for (int k2 = 0; k2 < 2; ++k2) {
          const int tg = k2 ? (tk.z <= kFillTask ? kFillTask - tk.z : (tk.z == -7 || tk.z == -8) ? tk.w : tk.z) : tk.x;
          if (tg < 0) continue;
          const int raw = __ldg(sync.tag_peer + tg);
          if (raw < 0 || raw >= 128) continue;
          const bool done_wait = sync.mode == 2 || raw >= 64;
          const int peer = raw & 63;
          const int bit = sync.mode == 3 ? (peer & 31) + (done_wait ? 32 : 0) : peer;
          if (!((peers_ok >> bit) & 1ull)) {
            if (lane == 0)
              flag_wait(sync.flags[sync.rank] + (done_wait ? kSlotDone : kSlotReady) * sync.nranks + peer,
                        sync.epoch, sync.timeout_ns);
            __syncwarp();
            peers_ok |= 1ull << bit;
          }
        }
      }
      if (!FILL && tk.z == -3) {  // chain task: all seams of one chain, kChainRows rows
        chain_task<LD>(tags, chains, tk.x, tk.w, (uint32_t)tk.y, kChainRows, lane);
      } else if (RING && tk.z == -4) {  // ring task: seam chunks of 32/(2k) columns of one x-ring
        ring_task<LD>(tags, chains, tk.x, tk.w, tk.y, lane);
      } else if (RING && tk.z == -6) {  // tile ring task: k fabs x 16/k consecutive seam chunks per step
        tile_ring_task<LD>(tags, chains, tk.x, tk.y, tk.w, lane);
      } else if (RING && (tk.z == -7 || tk.z == -8)) {  // seam pack / unpack task: column tk.y of tags tk.x (H), tk.w (L)
        if (tk.x != have_a || tk.w != have_b) {
          __syncwarp();
          if (tk.x != have_a) fetch_tag(tags, tk.x, &ta, lane);
          if (tk.w != have_b) fetch_tag(tags, tk.w, &tb, lane);
          have_a = tk.x;
          have_b = tk.w;
          __syncwarp();
        }
        seam_task<LD>(ta, tb, (uint32_t)tk.y, tk.z == -7, lane);
      } else if (BULK && tk.z == -5) {  // bulk-row task: tk.w rows of tag tk.x from row tk.y
        if (tk.x != have_a || have_b != -5) {
          __syncwarp();
          fetch_tag(tags, tk.x, &ta, lane);
          have_a = tk.x;
          have_b = -5;
          __syncwarp();
        }
        bulk_task(ta, (uint32_t)tk.y, (uint32_t)tk.w, lane, bulk_smem + wib * kBulkBytes, &bulk_bar[wib], bulk_phase);
      } else if (FILL && tk.z <= kFillTask) {  // sector-fill task: chunk tk.y of tag tk.x, chunk tk.w of tag kFillTask - tk.z
        const int bt = kFillTask - tk.z;
        if (tk.x != have_a || (bt != tk.x && bt != have_b)) {
          __syncwarp();
          if (tk.x != have_a) fetch_tag(tags, tk.x, &ta, lane);
          if (bt != tk.x && bt != have_b) fetch_tag(tags, bt, &tb, lane);
          have_a = tk.x;
          if (bt != tk.x) have_b = bt;
          __syncwarp();
        }
        const DevTag &tB = bt == tk.x ? ta : tb;
#pragma unroll 1
        for (int k2 = 0; k2 < 2; ++k2) {
          if (k2 && tk.w < 0) break;
          const DevTag &tt = k2 ? tB : ta;
          const uint32_t st = (uint32_t)(k2 ? tk.w : tk.y);
          if (fill_aligned(tt)) {
            fill_chunk<LD>(tt, st, lane);
          } else {
            uint4 val[kU];
            load_chunk<LD>(tt, st, lane, val);
            store_chunk(tt, st, lane, val);
          }
        }
      } else if (tk.z < -2 || (FILL && tk.z == -2)) {  // a task kind this instantiation does not carry: fail loudly
        __trap();
      } else if (!FILL && tk.z == -2) {  // sector-swap task over one chunk of T1
        const int sl = tk.x & (kSwapSlots - 1);
        if (swc_id[wib][sl] != tk.x) {
          __syncwarp();
          fetch_tag(tags, tk.x, &swc[wib][sl], lane);
          if (lane == 0) swc_id[wib][sl] = tk.x;
          __syncwarp();
        }
        swap_chunk<LD>(swc[wib][sl], (uint32_t)tk.y, lane);
        if (tk.w >= 0) swap_chunk<LD>(swc[wib][sl], (uint32_t)tk.w, lane);
      } else {
        if (tk.x != have_a || tk.z != have_b) {
          __syncwarp();
          if (tk.x == have_b && tk.z == have_a) {  // swapped pair order: swap roles
            tk = make_int4(tk.z, tk.w, tk.x, tk.y);
          } else {
            if (tk.x != have_a) fetch_tag(tags, tk.x, &ta, lane);
            if (tk.z >= 0 && tk.z != have_b) fetch_tag(tags, tk.z, &tb, lane);
            have_a = tk.x;
            have_b = tk.z;
          }
          __syncwarp();
        }
        uint4 va[kU], vb[kU];
        load_chunk<LD, RING && GHX_HOST_CONT>(ta, (uint32_t)tk.y, lane, va);
        if (tk.z >= 0) load_chunk<LD, RING && GHX_HOST_CONT>(tb, (uint32_t)tk.w, lane, vb);
        store_chunk(ta, (uint32_t)tk.y, lane, va);
        if (tk.z >= 0) store_chunk(tb, (uint32_t)tk.w, lane, vb);
      }
      if (sync.mode == 3 && w < sync.nhead) {
        // per-peer DONE: this warp's stores of the task are visible system
        // wide, then the task is counted against each of its push peers; the
        // count that completes a peer's total releases the peer's DONE
        const int4 t0 = __ldg(tasks + w);  // (re-read: a pair task may have swapped roles)
        __threadfence_system();
        __syncwarp();
        if (lane == 0 && t0.z >= -1) {
          const int pa = __ldg(sync.tag_peer + t0.x);
          const int pb = t0.z >= 0 ? __ldg(sync.tag_peer + t0.z) : -1;
#pragma unroll 1
          for (int k2 = 0; k2 < 2; ++k2) {
            const int p = k2 ? pb : pa;
            if (p < 0 || p >= 64 || (k2 && p == pa)) continue;
            if (atomicAdd(counter + 8 + p, 1ull) + 1 == (unsigned long long)__ldg(sync.peer_total + p))
              flag_store(sync.flags[p] + kSlotDone * sync.nranks + sync.rank, sync.epoch);
          }
        }
        __syncwarp();
      }
      tk = nxt;
    }
    nb = __shfl_sync(0xffffffffu, nb, 0);
  }
  if (BULK) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // this lane's bulk stores are done
  if (phased) pass_to(3, false);  // no more tasks: count out of every remaining phase
  if ((sync.mode == 2 || sync.mode == 3) && blockIdx.x == 0 && wib == 0) wait_all_peers(sync, kSlotDone, lane);
  if (sync.mode == 1 || sync.mode == 3) __threadfence_system();  // this lane's pushes are visible system-wide
  __syncwarp();
  if (lane == 0) {
    const unsigned long long total = (unsigned long long)gridDim.x * (blockDim.x >> 5);
    if (atomicAdd(counter + 1, 1ull) == total - 1) {
      if (sync.mode == 1 || sync.mode == 3) {  // every warp has fenced its pushes: tell the peers
        __threadfence_system();
        for (int p = 0; p < sync.nranks; ++p)
          if (p != sync.rank) flag_store(sync.flags[p] + kSlotDone * sync.nranks + sync.rank, sync.epoch);
      }
      counter[0] = 0;
      counter[1] = 0;
      counter[2] = 0;
      counter[3] = 0;
      counter[4] = 0;
      if (sync.mode == 3)
        for (int p = 0; p < sync.nranks; ++p) counter[8 + p] = 0;
    }
  }
}

// ---------------------------------------------------------------- helpers

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (dev >= 0 && dev != prev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

int cuda_fail(cudaError_t e, const char *what) {
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  // consume a non-sticky error (e.g. cudaErrorAlreadyMapped from an IPC open
  // the caller retries) so a later cudaGetLastError() does not report it
  // again for an unrelated, successful call
  (void)cudaGetLastError();
  return GHX_ECUDA;
}

struct Layout {
  Box box;
  int64_t nx, ny, nz, ncomp;
};

bool contains(const Box &outer, const Box &inner) {
  for (int d = 0; d < 3; ++d)
    if (inner.lo[d] < outer.lo[d] || inner.hi[d] > outer.hi[d]) return false;
  return true;
}

// One side (src or dst) of a host tag before vectorisation: element offset
// of the first cell and element strides.
struct Side {
  int64_t off, sy, sz, sc;
  int32_t ptr;
};

struct HostTag {
  Side s, d;
  int64_t nx, ny, nz, nc;  // elements
  bool remote;
  int32_t peer;            // push: destination rank of a remote tag; unpack: source rank; else -1
  int32_t sfab, dfab;      // plan fab ids (pairing)
  int64_t shift[3];
  bool unpack_role = false;  // reads a receive buffer (unpack kinds, EXCHANGE_PACKED's unpacks)
  // sector fill (unpack of x-face ghosts): the destination's valid x range
  // and the tag's first x, in elements from the storage box's lo (fill_vhi <
  // fill_vlo: not eligible)
  int64_t fill_x0 = 0, fill_vlo = 0, fill_vhi = -1;
};

int vec_log(const HostTag &t, int64_t eb, int64_t x0, int64_t nxe) {
  for (int vl = 4; vl >= 2; --vl) {
    const int64_t vb = 1ll << vl;
    if (vb < eb) break;
    if (((t.s.off + x0) * eb) % vb || ((t.d.off + x0) * eb) % vb) continue;
    if ((nxe * eb) % vb) continue;
    if ((t.s.sy * eb) % vb || (t.s.sz * eb) % vb || (t.s.sc * eb) % vb) continue;
    if ((t.d.sy * eb) % vb || (t.d.sz * eb) % vb || (t.d.sc * eb) % vb) continue;
    return vl;
  }
  return eb == 8 ? 3 : 2;
}

// Phased FillBoundary (GHX_EXEC_PHASED, fabs in host memory): every face
// tag that reaches its destination's valid boundary in a lower axis is
// extended over the destination's ghost cells in that axis, reading the
// source fab's own ghost cells there -- which the earlier phases have filled
// with the same periodic images the edge and corner tags would have read.
// The edge / corner tags inside the extensions are dropped, so over PCIe a
// ghost row is one request instead of a row plus two 16-byte pieces.
// Why the values agree: a ghost cell g of A is filled by the reference iff
// its periodically wrapped position is covered by a valid box, and then
// with that cell's value; the extension reads S's cell g - shift, whose
// wrapped position is the same (shifts are period multiples), and which is
// either valid or a ghost cell of S in lower axes only (filled by an earlier
// phase iff covered).  Per destination fab the transformation is kept only
// if the extensions exactly tile the dropped tags (same cells), are
// disjoint from everything else, and read inside the source storage;
// otherwise that fab keeps its original tags (any layout stays bit-exact).
// Returns false if the plan does not qualify at all (nothing changed).
bool phase_pieces(const ghx_plan *plan, int32_t rank, const std::vector<Box> &sstore, std::vector<Piece> &ps,
                  std::vector<int8_t> &phase) {
  if (plan->mode != GHX_MODE_FILL_BOUNDARY || plan->clipped || (int64_t)plan->vbox.size() != plan->ndst) return false;
  const size_t n = ps.size();
  std::vector<int> gmask(n, 0);
  for (size_t i = 0; i < n; ++i) {
    const Piece &p = ps[i];
    if (p.srank != rank || p.drank != rank) return false;
    const Box &V = plan->vbox[p.dst];
    for (int d = 0; d < 3; ++d) {
      if (p.dbox.hi[d] < V.lo[d] || p.dbox.lo[d] > V.hi[d])
        gmask[i] |= 1 << d;
      else if (p.dbox.lo[d] < V.lo[d] || p.dbox.hi[d] > V.hi[d])
        return false;  // straddles the valid boundary
    }
    if (!gmask[i]) return false;  // writes valid cells (not a cell-centred exchange)
    phase[i] = (int8_t)(gmask[i] & 4 ? 2 : gmask[i] & 2 ? 1 : 0);
  }
  std::vector<std::vector<size_t>> by_dst(plan->ndst);
  for (size_t i = 0; i < n; ++i) by_dst[ps[i].dst].push_back(i);
  std::vector<uint8_t> drop(n, 0);
  std::vector<Box> ext(n);
  for (size_t i = 0; i < n; ++i) ext[i] = ps[i].dbox;
  auto cells = [](const Box &b) { return b.cells(); };
  auto inside = [](const Box &in, const Box &out) {
    for (int d = 0; d < 3; ++d)
      if (in.lo[d] < out.lo[d] || in.hi[d] > out.hi[d]) return false;
    return true;
  };
  for (int32_t a = 0; a < plan->ndst; ++a) {
    const std::vector<size_t> &ids = by_dst[a];
    const Box &V = plan->vbox[a];
    std::vector<Box> e(ids.size());
    std::vector<uint8_t> isface(ids.size(), 0), extended(ids.size(), 0), rm(ids.size(), 0);
    bool ok = true;
    int64_t ext_cells = 0;
    for (size_t u = 0; u < ids.size(); ++u) {
      const Piece &p = ps[ids[u]];
      e[u] = p.dbox;
      const int g = gmask[ids[u]];
      if (g & (g - 1)) continue;  // edge / corner
      isface[u] = 1;
      const int d = g == 1 ? 0 : g == 2 ? 1 : 2;
      for (int x = 0; x < d; ++x) {
        if (plan->ngrow[x] <= 0) continue;
        if (p.dbox.lo[x] == V.lo[x]) e[u].lo[x] = V.lo[x] - plan->ngrow[x];
        if (p.dbox.hi[x] == V.hi[x]) e[u].hi[x] = V.hi[x] + plan->ngrow[x];
      }
      if (cells(e[u]) != cells(p.dbox)) {
        extended[u] = 1;
        ext_cells += cells(e[u]) - cells(p.dbox);
        Box sb = e[u];
        for (int d2 = 0; d2 < 3; ++d2) {
          sb.lo[d2] -= p.shift[d2];
          sb.hi[d2] -= p.shift[d2];
        }
        if (!inside(sb, sstore[p.src])) ok = false;
      }
    }
    // every edge / corner tag lies inside one extension or outside all
    int64_t rm_cells = 0;
    for (size_t u = 0; u < ids.size() && ok; ++u) {
      if (isface[u]) continue;
      int in = 0, touch = 0;
      for (size_t w = 0; w < ids.size(); ++w) {
        if (!extended[w]) continue;
        if (inside(ps[ids[u]].dbox, e[w])) ++in;
        else if (ghx::overlap(ps[ids[u]].dbox, e[w])) ++touch;
      }
      if (touch || in > 1) ok = false;
      if (in == 1) {
        rm[u] = 1;
        rm_cells += cells(ps[ids[u]].dbox);
      }
    }
    // extensions disjoint from each other and from every kept tag
    for (size_t u = 0; u < ids.size() && ok; ++u) {
      if (!extended[u]) continue;
      for (size_t w = 0; w < ids.size() && ok; ++w) {
        if (w == u || rm[w]) continue;
        if (ghx::overlap(e[u], extended[w] ? e[w] : ps[ids[w]].dbox)) ok = false;
      }
    }
    if (!ok || rm_cells != ext_cells) continue;  // this fab keeps its original tags
    for (size_t u = 0; u < ids.size(); ++u) {
      if (rm[u]) drop[ids[u]] = 1;
      if (extended[u]) ext[ids[u]] = e[u];
    }
  }
  std::vector<Piece> out;
  std::vector<int8_t> ph;
  for (size_t i = 0; i < n; ++i) {
    if (drop[i]) continue;
    Piece p = ps[i];
    p.dbox = ext[i];
    out.push_back(p);
    ph.push_back(phase[i]);
  }
  ps.swap(out);
  phase.swap(ph);
  return true;
}

// pairing key of a device tag: (src fab, dst fab, shift, part, shape)
using PairKey = std::tuple<int32_t, int32_t, int64_t, int64_t, int64_t, int, uint32_t, uint32_t, uint32_t, int>;

}  // namespace

struct ghx_exec {
  int32_t device = 0;
  int32_t kind = 0;
  int32_t nranks = 1, nsrc = 0, ndst = 0;
  int32_t elem_bytes = 8;
  bool nc_loads = true;
  int ld_mode = 2;  // ld.global.cg measured best on B200 (see profiles/)
  int64_t elems = 0;
  int64_t npaired = 0, nswap = 0;
  bool ring = false;    // x-face seams as ring tasks (coalesced 64-B chunks)
  bool fab_local = false;  // small fabs: per-tag swaps in destination-fab order, no chains
  bool bulk = false;       // wide 16-byte-vector rows as TMA bulk-row tasks
  int64_t nbulk = 0;
  int64_t nring = 0;
  std::vector<uint8_t> swap_fab;  // fabs touched by sector-swap tasks
  std::vector<int64_t> buf_elems;  // per peer (pack: send, unpack: recv)
  std::vector<int64_t> recv_elems; // per peer, receive side (EXCHANGE_PACKED; unpack kinds = buf_elems)
  std::vector<DevTag> htags;
  std::vector<PairKey> hkeys;
  std::vector<int32_t> hremote;
  std::vector<int32_t> hpeer;   // per tag (SyncArgs::tag_peer)
  int32_t nhead = 0;            // remote tasks at the head of htasks
  // phased exchange (GHX_EXEC_PHASED): x faces, then y faces extended over
  // the x ghosts, then z faces extended over x and y ghosts (no edge or
  // corner tags); tasks ordered by phase, [0, pe0) x, [pe0, pe1) y, rest z
  bool phased = false;
  int8_t cur_phase = 0;         // phase of the tag being emitted
  std::vector<int8_t> hphase;   // per tag
  std::vector<uint8_t> hfill;   // per tag: 16-byte ghost halves written as whole sectors (fill_load)
  int64_t nfill = 0;            // tags run as sector-fill tasks
  int64_t nseam = 0;            // tags run as seam pack / unpack tasks (host memory, remote x faces)
  int32_t pe0 = 0, pe1 = 0;
  // in-kernel synchronisation (ghx_exec_set_sync)
  int32_t sync_rank = -1, sync_n = 0;
  uint64_t **dflags = nullptr;
  int32_t *dpeer = nullptr;
  int32_t rank = 0;  // the rank this executor was compiled for
  // EXCHANGE_PACKED: remote push tasks per destination peer (a pair task
  // counted once per distinct peer); the kernel releases a peer's DONE when
  // its last push task to that peer is done
  std::vector<int32_t> peer_total;
  int32_t *dpeer_total = nullptr;
  std::vector<int4> htasks;
  std::vector<int> hchain;  // chain tables (tag indices of consecutive seams)
  int *dchain = nullptr;
  DevTag *dtags = nullptr;
  int4 *dtasks = nullptr;
  void **dptrs = nullptr;
  // Bound descriptor tables, one per pointer table in use: each holds its
  // own copy of the descriptors with absolute addresses and its own
  // scheduler counter.  Pinned bindings (ghx_exec_bind, held by a prepared
  // exchange and baked into CUDA graphs) are never rebound; unpinned ones
  // (ghx_exec_run with a raw table) are recycled least-recently-used, at
  // most kMaxLoose of them.
  struct Binding {
    std::vector<void *> ptrs;
    DevTag *dtags = nullptr;
    void **dptrs = nullptr;
    unsigned long long *counter = nullptr;
    uint64_t last_use = 0;
    int pins = 0;
    int64_t id = 0;
  };
  std::vector<std::unique_ptr<Binding>> bindings;
  int64_t next_binding = 1;
  uint64_t uses = 0;
  int64_t nptrs = 0;
  int blocks = 0, threads = kThreads;
  bool uploaded = false;
  std::mutex mu;
};

namespace {

void add_devtag(ghx_exec *ex, const HostTag &t, int64_t x0, int64_t nxe, int vl, int part) {
  const int64_t eb = ex->elem_bytes;
  const int64_t epv = (1ll << vl) / eb;  // elements per vector
  DevTag g;
  std::memset(&g, 0, sizeof(g));
  g.src_off = (t.s.off + x0) / epv;
  g.dst_off = (t.d.off + x0) / epv;
  g.src_sy = (int32_t)(t.s.sy / epv);
  g.dst_sy = (int32_t)(t.d.sy / epv);
  g.src_sz = t.s.sz / epv;
  g.dst_sz = t.d.sz / epv;
  g.src_sc = t.s.sc / epv;
  g.dst_sc = t.d.sc / epv;
  g.src_ptr = t.s.ptr;
  g.dst_ptr = t.d.ptr;
  g.nxv = (uint32_t)(nxe / epv);
  g.ny = (uint32_t)t.ny;
  g.nz = (uint32_t)t.nz;
  g.nvec = (uint32_t)(g.nxv * t.ny * t.nz * t.nc);
  FastDiv fx = make_div(g.nxv), fy = make_div(g.ny), fz = make_div(g.nz);
  g.mx = fx.m;
  g.sx = (uint8_t)fx.s;
  g.my = fy.m;
  g.sy = (uint8_t)fy.s;
  g.mz = fz.m;
  g.sz = (uint8_t)fz.s;
  g.vlog = (uint8_t)vl;
  ex->htags.push_back(g);
  ex->hkeys.emplace_back(t.sfab, t.dfab, t.shift[0], t.shift[1], t.shift[2], part, g.nxv, g.ny, g.nz, vl);
  // hremote: 1 remote, 2 the unpack side of an EXCHANGE_PACKED executor;
  // hpeer: the peer, + 64 for that unpack side (the kernel waits for the
  // peer's DONE instead of its READY)
  const bool xunpack = ex->kind == GHX_EXEC_EXCHANGE_PACKED && t.unpack_role;
  ex->hremote.push_back(xunpack ? 2 : (t.remote ? 1 : 0));
  ex->hpeer.push_back(xunpack ? t.peer + 64 : t.peer);
  ex->hphase.push_back(ex->cur_phase);
  // sector fill: one 16-byte vector per row, every row in the same sector
  // half (even strides), and the other half of its sectors valid cells
  bool fill = t.fill_vhi >= t.fill_vlo && vl == 4 && g.nxv == 1 && g.dst_sy % 2 == 0 && g.dst_sz % 2 == 0 &&
              g.dst_sc % 2 == 0;
  if (fill) {
    const int64_t x = t.fill_x0 + x0;  // first element of the vector
    const int64_t olo = (g.dst_off & 1) ? x - epv : x + epv;
    fill = olo >= t.fill_vlo && olo + epv - 1 <= t.fill_vhi;
  }
  ex->hfill.push_back(fill ? 1 : 0);
}

// Split a row range into an unaligned head, 16-byte body and tail when src
// and dst share the same 16-byte phase; otherwise use the widest common
// vector for the whole row.
void emit_tag(ghx_exec *ex, const HostTag &t) {
  const int64_t eb = ex->elem_bytes;
  const int64_t xb = t.nx * eb;
  const int64_t ps = (t.s.off * eb) % 16, pd = (t.d.off * eb) % 16;
  const bool strides16 = (t.s.sy * eb) % 16 == 0 && (t.s.sz * eb) % 16 == 0 && (t.s.sc * eb) % 16 == 0 &&
                         (t.d.sy * eb) % 16 == 0 && (t.d.sz * eb) % 16 == 0 && (t.d.sc * eb) % 16 == 0;
  if (eb < 16 && ps == pd && ps != 0 && strides16 && xb >= 32) {
    const int64_t head = ((16 - ps) % 16) / eb;
    const int64_t body = ((t.nx - head) * eb / 16) * 16 / eb;
    const int64_t tail = t.nx - head - body;
    if (head > 0) add_devtag(ex, t, 0, head, vec_log(t, eb, 0, head), 1);
    if (body > 0) add_devtag(ex, t, head, body, 4, 2);
    if (tail > 0) add_devtag(ex, t, head + body, tail, vec_log(t, eb, head + body, tail), 3);
    return;
  }
  if (eb < 16 && ps == pd && ps == 0 && strides16 && xb >= 32 && xb % 16 != 0) {
    const int64_t body = (xb / 16) * 16 / eb;
    add_devtag(ex, t, 0, body, 4, 2);
    add_devtag(ex, t, body, t.nx - body, vec_log(t, eb, body, t.nx - body), 3);
    return;
  }
  add_devtag(ex, t, 0, t.nx, vec_log(t, eb, 0, t.nx), 0);
}

// Can mirror tags a, b run as a sector swap?  Both 16-byte rows (one vector
// per row), identical row geometry, and one writes the low half of the
// 32-byte sector whose high half the other reads (and vice versa).  Returns
// the index of the tag that writes low halves, or -1.
int swap_low(const ghx_exec *ex, int ia, int ib) {
  const DevTag &a = ex->htags[ia], &b = ex->htags[ib];
  // fab identity (the plan's fab ids); the src and dst pointer slots of one
  // fab must alias, which ghx_exec_run verifies for swap executors
  auto fab = [&](int i, bool src) { return src ? std::get<0>(ex->hkeys[i]) : std::get<1>(ex->hkeys[i]); };
  auto fits = [&](const DevTag &t1, int i1, const DevTag &t2, int i2) {
    return (ex->kind <= GHX_EXEC_LOCAL || ex->kind == GHX_EXEC_PUSH_PACKED || ex->kind == GHX_EXEC_PUSH_PACKED_ALL) && t1.vlog == 4 && t2.vlog == 4 && t1.nxv == 1 && t2.nxv == 1 &&
           t1.ny == t2.ny && t1.nz == t2.nz && t1.nvec == t2.nvec && fab(i1, false) == fab(i2, true) &&
           fab(i1, true) == fab(i2, false) &&
           t1.dst_sy == t2.src_sy && t1.dst_sz == t2.src_sz && t1.dst_sc == t2.src_sc &&
           t1.src_sy == t2.dst_sy && t1.src_sz == t2.dst_sz && t1.src_sc == t2.dst_sc &&
           t2.src_off == t1.dst_off + 1 && t2.dst_off == t1.src_off + 1 && t1.dst_off % 2 == 0 &&
           t1.src_off % 2 == 0 && t1.dst_sy % 2 == 0 && t1.dst_sz % 2 == 0 && t1.dst_sc % 2 == 0 &&
           t1.src_sy % 2 == 0 && t1.src_sz % 2 == 0 && t1.src_sc % 2 == 0;
  };
  if (fits(a, ia, b, ib)) return ia;
  if (fits(b, ib, a, ia)) return ib;
  return -1;
}

// Seam pairs of one fab's remote x faces over PCIe (host-memory pack and
// unpack executors): H moves the high-x 16-byte vector of every row, L the
// low-x one, of the SAME fab rows.  The end of row y and the start of row
// y+1 are one 64-byte seam chunk, so a lane pair can move H's row y and
// L's row y+1 with one coalesced request instead of two 16-byte ones:
//   pack (src side in the fab):   chunk = [H.src(y) | hg | lg | L.src(y+1)]
//   unpack (dst side in the fab): chunk = [hv | H.dst(y) | L.dst(y+1) | lv]
// Returns H's index, or -1 when (a, b) is not such a pair.
int seam_pair_hi(const ghx_exec *ex, int ia, int ib, bool pack) {
  const DevTag &a = ex->htags[ia], &b = ex->htags[ib];
  if (a.vlog != 4 || b.vlog != 4 || a.nxv != 1 || b.nxv != 1 || a.ny != b.ny || a.nz != b.nz || a.nvec != b.nvec ||
      a.ny < 1)
    return -1;
  auto fits = [&](const DevTag &H, const DevTag &L) {
    if (pack)
      return H.src_ptr == L.src_ptr && H.src_sy == L.src_sy && H.src_sz == L.src_sz && H.src_sc == L.src_sc &&
             L.src_off + L.src_sy == H.src_off + 3 && H.src_off % 2 == 0 && H.src_sy % 2 == 0 &&
             H.src_sz % 2 == 0 && H.src_sc % 2 == 0;
    return H.dst_ptr == L.dst_ptr && H.dst_sy == L.dst_sy && H.dst_sz == L.dst_sz && H.dst_sc == L.dst_sc &&
           L.dst_off + L.dst_sy == H.dst_off + 1 && (H.dst_off - 1) % 2 == 0 && H.dst_sy % 2 == 0 &&
           H.dst_sz % 2 == 0 && H.dst_sc % 2 == 0;
  };
  if (fits(a, b)) return ia;
  if (fits(b, a)) return ib;
  return -1;
}

// Order the sector-swap tags of one chain of fabs as an x-ring for
// ring_task: T_j moves F_j's last sector <-> F_{j+1}'s first sector, every
// fab appears once on each side, the ring closes, and for every fab the
// first sector of row y+1 directly follows the last sector of row y (seam
// chunks are 64 contiguous bytes).  Returns {} if the chain is not such a
// ring (then chain / swap tasks are used).
std::vector<int32_t> ring_order(const ghx_exec *ex, const std::vector<int32_t> &ts) {
  const int k = (int)ts.size();
  if (k < 1 || k > 16) return {};
  std::map<int32_t, int32_t> by_src;  // source fab (L) -> tag
  for (int32_t t : ts)
    if (!by_src.emplace(std::get<0>(ex->hkeys[t]), t).second) return {};
  std::vector<int32_t> order;
  int32_t t = ts[0];
  for (int n = 0; n < k; ++n) {
    order.push_back(t);
    auto it = by_src.find(std::get<1>(ex->hkeys[t]));  // next fab's tag
    if (it == by_src.end()) return {};
    t = it->second;
  }
  if (t != ts[0]) return {};
  std::vector<int32_t> seen(order);
  std::sort(seen.begin(), seen.end());
  if (std::unique(seen.begin(), seen.end()) != seen.end()) return {};
  for (int j = 0; j < k; ++j) {
    const DevTag &a = ex->htags[order[(j + k - 1) % k]];  // its dst = F_j's first sector
    const DevTag &b = ex->htags[order[j]];                // its src = F_j's last sector
    if (a.ny != b.ny || a.nz != b.nz || a.nvec != b.nvec || a.dst_sy != b.src_sy || a.dst_sz != b.src_sz ||
        a.dst_sc != b.src_sc || a.dst_off + a.dst_sy != b.src_off + 2 || a.ny < 1)
      return {};
  }
  return order;
}

bool seam_tasks_on() {  // GHX_SEAM_TASKS=0: host-memory remote x faces as plain pair copies
  static const bool on = [] {
    const char *v = std::getenv("GHX_SEAM_TASKS");
    return !v || std::atoi(v) != 0;
  }();
  return on;
}

// Warp tasks.  Mirror tags (src<->dst swapped, opposite shift, same shape)
// are paired chunk by chunk so the two halves of every shared sector move
// together; everything else pairs consecutive chunks of one tag.
void build_tasks(ghx_exec *ex) {
  const size_t n = ex->htags.size();
  std::map<PairKey, int32_t> index;
  for (size_t i = 0; i < n; ++i) index.emplace(ex->hkeys[i], (int32_t)i);
  std::vector<int32_t> mate(n, -1);
  const bool pair_mirrors = std::getenv("GHX_NO_MIRROR") == nullptr;
  if (pair_mirrors)
    for (size_t i = 0; i < n; ++i) {
      if (mate[i] >= 0 || ex->hremote[i]) continue;
      const PairKey &k = ex->hkeys[i];
      if (std::get<0>(k) == std::get<1>(k) && std::get<2>(k) == 0 && std::get<3>(k) == 0 && std::get<4>(k) == 0)
        continue;
      PairKey m(std::get<1>(k), std::get<0>(k), -std::get<2>(k), -std::get<3>(k), -std::get<4>(k), std::get<5>(k),
                std::get<6>(k), std::get<7>(k), std::get<8>(k), std::get<9>(k));
      auto it = index.find(m);
      if (it == index.end() || it->second == (int32_t)i || mate[it->second] >= 0 || ex->hremote[it->second]) continue;
      mate[i] = it->second;
      mate[it->second] = (int32_t)i;
    }
  // Remote tags of one fab with the same shape run as pair tasks, chunk by
  // chunk: a sender's lo- and hi-x-face tags read the two ends of the same
  // rows -- one 128-B line per row seam -- and an unpack's lo- and hi-x-ghost
  // tags fill the two halves of the same seam lines, so the second access
  // of each line hits in L2 instead of fetching (and, for the partial-sector
  // ghost writes, refilling) it again.  Anchor fab: the source for pushes,
  // the destination for unpacks.  (GHX_REMOTE_PAIR=0: unpaired.)
  static const bool pair_remote = [] {
    const char *v = std::getenv("GHX_REMOTE_PAIR");
    return !v || std::atoi(v) != 0;
  }();
  if (pair_remote) {
    const bool unpack_kind = ex->kind == GHX_EXEC_UNPACK || ex->kind == GHX_EXEC_UNPACK_PACKED ||
                             ex->kind == GHX_EXEC_UNPACK_PACKED_ALL;
    std::map<std::tuple<int32_t, uint32_t, uint32_t, uint32_t, uint32_t, int, int>, int32_t> open;
    for (size_t i = 0; i < n; ++i) {
      if (mate[i] >= 0 || !ex->hremote[i]) continue;
      const DevTag &t = ex->htags[i];
      const bool unpack = unpack_kind || ex->hremote[i] == 2;
      const auto key = std::make_tuple(unpack ? std::get<1>(ex->hkeys[i]) : std::get<0>(ex->hkeys[i]), t.nxv, t.ny,
                                       t.nz, t.nvec, (int)t.vlog, (int)ex->hremote[i]);
      auto it = open.find(key);
      if (it == open.end()) {
        open.emplace(key, (int32_t)i);
      } else {
        mate[i] = it->second;
        mate[it->second] = (int32_t)i;
        open.erase(it);
      }
    }
  }
  std::vector<int4> loc, rem, swaps, unp;  // unp: EXCHANGE_PACKED's unpack tasks
  ex->npaired = 0;
  ex->nswap = 0;
  ex->nring = 0;
  ex->hchain.clear();
  ex->swap_fab.clear();
  // an EXCHANGE_PACKED executor with sector fills runs in the fill-capable
  // kernel instantiation, which carries no sector-swap / chain tasks (their
  // registers): its local mirror pairs run as pair copies instead
  bool any_fill = false;
  for (size_t i = 0; i < n && !ex->ring; ++i) any_fill = any_fill || (i < ex->hfill.size() && ex->hfill[i]);
  const bool allow_swap = std::getenv("GHX_NO_SWAP") == nullptr && !(ex->kind == GHX_EXEC_EXCHANGE_PACKED && any_fill);
  std::vector<int32_t> swap_lo;  // low tag of every sector-swap pair
  ex->nbulk = 0;
  auto bulk_ok = [&](size_t i) {
    const DevTag &t = ex->htags[i];
    const uint32_t rb = t.nxv << 4;
    // (not with ring tasks: one kernel instantiation carries one of the two)
    return ex->bulk && !ex->ring && !ex->hremote[i] && t.vlog == 4 && rb >= 256 && rb <= (uint32_t)kBulkBytes &&
           ex->kind <= GHX_EXEC_LOCAL;
  };
  // sector fill: not over PCIe (ring executors: fabs in host memory, where
  // the extra 16-byte read costs a request)
  ex->nfill = 0;
  ex->nseam = 0;
  auto fill_ok = [&](size_t i) { return !ex->ring && i < ex->hfill.size() && ex->hfill[i] && n < (1u << 30); };
  auto emit_bulk = [&](size_t i, std::vector<int4> &out) {
    const DevTag &t = ex->htags[i];
    const uint32_t rows = t.nvec / t.nxv, per = std::min<uint32_t>(32, kBulkBytes / (t.nxv << 4));
    const uint32_t step = per * 2;  // two buffer fills per task
    for (uint32_t r = 0; r < rows; r += step) out.push_back(make_int4((int)i, (int)r, -5, (int)std::min(step, rows - r)));
    ex->nbulk += 1;
  };
  for (size_t i = 0; i < n; ++i) {
    const uint32_t nv = ex->htags[i].nvec;
    auto &out = ex->hremote[i] == 2 ? unp : (ex->hremote[i] ? rem : loc);
    if (mate[i] >= 0) {
      if ((size_t)mate[i] < i) continue;
      const int lo = allow_swap ? swap_low(ex, (int)i, mate[i]) : -1;
      if (lo >= 0) {
        ex->nswap += 2;
        const int32_t fa = std::get<0>(ex->hkeys[i]), fb = std::get<1>(ex->hkeys[i]);
        if (ex->swap_fab.size() <= (size_t)std::max(fa, fb)) ex->swap_fab.resize(std::max(fa, fb) + 1, 0);
        ex->swap_fab[fa] = ex->swap_fab[fb] = 1;
        swap_lo.push_back(lo);
        continue;
      }
      ex->npaired += 2;
      if (bulk_ok(i) && bulk_ok(mate[i])) {
        emit_bulk(i, out);
        emit_bulk(mate[i], out);
        continue;
      }
      // host-memory pack / unpack of a fab's remote x faces: seam tasks, one
      // column of rows per task, one PCIe request per seam and side
      if (ex->ring && ex->hremote[i] && ex->hremote[mate[i]] &&
          (ex->kind == GHX_EXEC_PUSH_PACKED_ALL || ex->kind == GHX_EXEC_UNPACK_PACKED_ALL) && seam_tasks_on()) {
        const bool pack = ex->kind == GHX_EXEC_PUSH_PACKED_ALL;
        const int hi = seam_pair_hi(ex, (int)i, mate[i], pack);
        if (hi >= 0) {
          const int lo = hi == (int)i ? mate[i] : (int)i;
          const DevTag &H = ex->htags[hi];
          const uint32_t ncol = H.nvec / H.ny;
          for (uint32_t q = 0; q < ncol; ++q) out.push_back(make_int4(hi, (int)q, pack ? -7 : -8, lo));
          ex->nseam += 2;
          continue;
        }
      }
      if (fill_ok(i) && fill_ok(mate[i]) && ex->htags[mate[i]].nvec == nv) {
        ex->nfill += 2;
        for (uint32_t s = 0; s < nv; s += kChunk) out.push_back(make_int4((int)i, (int)s, kFillTask - mate[i], (int)s));
        continue;
      }
      for (uint32_t s = 0; s < nv; s += kChunk) out.push_back(make_int4((int)i, (int)s, mate[i], (int)s));
    } else if (bulk_ok(i)) {
      emit_bulk(i, out);
    } else if (fill_ok(i)) {
      ex->nfill += 1;
      for (uint32_t s = 0; s < nv; s += 2 * kChunk)
        out.push_back(make_int4((int)i, (int)s, kFillTask - (int)i, s + kChunk < nv ? (int)(s + kChunk) : -1));
    } else {
      for (uint32_t s = 0; s < nv; s += 2 * kChunk)
        out.push_back(make_int4((int)i, (int)s, s + kChunk < nv ? (int)i : -1, (int)(s + kChunk)));
    }
  }
  // Sector swaps of one chain of fabs (an x-line of boxes: ...L|A|R...) share
  // 128-byte lines at the row seams (the end of row r and the start of row
  // r+1 of a fab are adjacent), so the seams of one chain are issued chunk by
  // chunk together and each line is fetched from / written to HBM once.
  if (!swap_lo.empty()) {
    std::map<int32_t, int32_t> parent;
    std::function<int32_t(int32_t)> find = [&](int32_t x) {
      auto it = parent.find(x);
      if (it == parent.end()) {
        parent[x] = x;
        return x;
      }
      if (it->second == x) return x;
      const int32_t r = find(it->second);
      parent[x] = r;
      return r;
    };
    for (int32_t t : swap_lo) {
      const int32_t a = find(std::get<0>(ex->hkeys[t])), b = find(std::get<1>(ex->hkeys[t]));
      if (a != b) parent[std::max(a, b)] = std::min(a, b);
    }
    std::map<int32_t, std::vector<int32_t>> chains;
    for (int32_t t : swap_lo) chains[find(std::get<0>(ex->hkeys[t]))].push_back(t);
    const bool chain_tasks = std::getenv("GHX_NO_CHAIN") == nullptr && !ex->fab_local;
    const bool ring_mode = ex->ring;
    // tile ring tasks (default) or the column-layout ring tasks (GHX_RING_TILE=0)
    static const bool tile_ring = [] {
      const char *v = std::getenv("GHX_RING_TILE");
      return !v || std::atoi(v) != 0;
    }();
    for (auto &kv : chains) {
      std::vector<int32_t> &ts = kv.second;
      std::sort(ts.begin(), ts.end());
      bool uniform = ts.size() <= 32;
      for (int32_t t : ts) uniform = uniform && ex->htags[t].nvec == ex->htags[ts[0]].nvec;
      if (uniform && ring_mode) {
        std::vector<int32_t> order = ring_order(ex, ts);
        if (!order.empty()) {
          const DevTag &t0 = ex->htags[order[0]];
          const int k = (int)order.size();
          const int streams = 16 / k;
          const uint32_t ncols = t0.nz * (t0.nvec / (t0.ny * t0.nz));
          const int off = (int)ex->hchain.size();
          ex->hchain.insert(ex->hchain.end(), order.begin(), order.end());
          ex->nring += 2 * k;
          if (tile_ring && t0.ny + 1 <= 65534) {
            // tile ring tasks: one column each, chunk ranges of ~32
            // (balanced), columns in address order
            const int R = 16 / k;
            const uint32_t nch = t0.ny + 1;
            const uint32_t per_task = (uint32_t)std::max(R, 8 * R);
            const uint32_t nt = (nch + per_task - 1) / per_task;
            const uint32_t span = (nch + nt - 1) / nt;
            for (uint32_t q = 0; q < ncols; ++q)
              for (uint32_t a = 0; a < nch; a += span) {
                const uint32_t sp = std::min(span, nch - a);
                // c0 + 1 = a (chunk -1 is a = 0)
                swaps.push_back(make_int4(off, (int)q, -6, k | (int)(a << 5) | (int)(sp << 21)));
              }
            continue;
          }
          // column-major (q, then row segment): concurrent warps stay on few
          // host pages (fabs in host memory are the ring's use)
          const uint32_t nseg = (t0.ny + kRingRows - 1) / kRingRows;
          for (uint32_t q = 0; q < ncols; q += streams)
            for (uint32_t seg = 0; seg < nseg; ++seg)
              swaps.push_back(make_int4(off, (int)q, -4, k | (int)(seg << 5)));
          continue;
        }
      }
      if (uniform && chain_tasks) {
        const int off = (int)ex->hchain.size();
        ex->hchain.insert(ex->hchain.end(), ts.begin(), ts.end());
        for (uint32_t s = 0; s < ex->htags[ts[0]].nvec; s += kChainRows)
          swaps.push_back(make_int4(off, (int)s, -3, (int)ts.size()));
        continue;
      }
      uint32_t maxv = 0;
      for (int32_t t : ts) maxv = std::max(maxv, ex->htags[t].nvec);
      for (uint32_t s = 0; s < maxv; s += kChunk)
        for (int32_t t : ts)
          if (s < ex->htags[t].nvec) swaps.push_back(make_int4(t, (int)s, -2, -1));
    }
    // spread the latency-bound seam work over the launch so it overlaps the
    // bandwidth-bound row copies
    if (std::getenv("GHX_BULK_FIRST")) {  // experiment: bulk face rows first, then the seams
      loc.insert(loc.end(), swaps.begin(), swaps.end());
      swaps.clear();
    } else if (std::getenv("GHX_NO_INTERLEAVE") || ex->nbulk || ex->ring) {
      // bulk (TMA) face rows and latency-bound seams interfere when
      // interleaved (measured); seams first, then the bulk rows.  Same over
      // PCIe (host-memory fabs, ring tasks): C3 e2e 56.3 -> 53.8 ms
      swaps.insert(swaps.end(), loc.begin(), loc.end());
      loc.swap(swaps);
      swaps.clear();
    }
    std::vector<int4> merged;
    merged.reserve(swaps.size() + loc.size());
    size_t ia = 0, ib = 0;
    const double ra = 1.0 / swaps.size(), rb = loc.empty() ? 0 : 1.0 / loc.size();
    while (!swaps.empty() && (ia < swaps.size() || ib < loc.size())) {
      if (ib >= loc.size() || (ia < swaps.size() && (ia + 0.5) * ra <= (ib + 0.5) * rb))
        merged.push_back(swaps[ia++]);
      else
        merged.push_back(loc[ib++]);
    }
    if (!swaps.empty()) loc.swap(merged);
  }
  // remote (NVLink) tasks first, so the pushes -- the longer pole at N > 1
  // -- start at t = 0 and the local HBM work fills in behind them
  // (GHX_REMOTE_ORDER=interleave: the earlier proportional interleave)
  std::vector<int4> &a = loc;
  const std::vector<int4> &b = rem;
  static const bool interleave = [] {
    const char *v = std::getenv("GHX_REMOTE_ORDER");
    return v && std::string(v) == "interleave";
  }();
  // EXCHANGE_PACKED: pushes in peer-distance order (rank r serves r+1
  // first, then r+2, ...: every peer's DONE is released in turn, and at any
  // moment the ranks push to different peers), unpacks in arrival order
  // (r-1's slab first, then r-2's, ...)
  if (ex->kind == GHX_EXEC_EXCHANGE_PACKED) {
    const int n = std::max(1, ex->nranks);
    auto order = [&](std::vector<int4> &v, bool arrival) {
      auto dist = [&](int32_t tag) -> int {
        if (tag < 0 || ex->hpeer[tag] < 0) return n;
        const int p = ex->hpeer[tag] & 63;
        return arrival ? (ex->rank - p + n) % n : (p - ex->rank + n) % n;
      };
      auto key = [&](const int4 &t) { return std::min(dist(t.x), dist(t.z >= 0 ? t.z : -1)); };
      std::stable_sort(v.begin(), v.end(), [&](const int4 &l, const int4 &r) { return key(l) < key(r); });
    };
    order(rem, false);
    order(unp, true);
  }
  ex->peer_total.assign(64, 0);
  for (const int4 &t : rem) {
    const int32_t pa = ex->hpeer[t.x], pb = t.z >= 0 ? ex->hpeer[t.z] : -1;
    if (pa >= 0 && pa < 64) ex->peer_total[pa] += 1;
    if (pb >= 0 && pb < 64 && pb != pa) ex->peer_total[pb] += 1;
  }
  ex->nhead = 0;
  if (!b.empty() && !interleave) {
    std::vector<int4> merged(b);
    merged.insert(merged.end(), a.begin(), a.end());
    a.swap(merged);
    ex->nhead = (int32_t)b.size();
  } else if (!b.empty()) {
    ex->nhead = (int32_t)(a.size() + b.size());  // remote tasks anywhere: every task checks its peer
    std::vector<int4> merged;
    merged.reserve(a.size() + b.size());
    size_t ia = 0, ib = 0;
    const double ra = a.empty() ? 0 : 1.0 / a.size(), rb = 1.0 / b.size();
    while (ia < a.size() || ib < b.size()) {
      if (ib >= b.size() || (ia < a.size() && (ia + 0.5) * ra <= (ib + 0.5) * rb))
        merged.push_back(a[ia++]);
      else
        merged.push_back(b[ib++]);
    }
    a.swap(merged);
  }
  if (ex->fab_local && !ex->ring) {
    // small fabs: sweep the destination fabs in order, so the tasks that
    // share a fab's lines (seam sectors, face rows) run close in time and
    // hit in L2 (C4: -23 % time, C2: -6 %; measured)
    // key: (destination fab, component, position in the component)
    auto key = [&](const int4 &t) -> std::tuple<int64_t, int64_t, int64_t> {
      const int32_t tag = (t.z == -4 || t.z == -3 || t.z == -6) ? ex->hchain[t.x] : t.x;
      const DevTag &d = ex->htags[tag];
      const int64_t per_comp = std::max<int64_t>(1, (int64_t)d.nxv * d.ny * d.nz);
      return {std::get<1>(ex->hkeys[tag]), (int64_t)t.y / per_comp, (int64_t)t.y % per_comp};
    };
    std::stable_sort(a.begin() + (interleave ? 0 : ex->nhead), a.end(), [&](const int4 &l, const int4 &r) { return key(l) < key(r); });
  }
  ex->pe0 = ex->pe1 = 0;
  if (ex->phased) {
    auto tphase = [&](const int4 &t) -> int {
      const int32_t tag = (t.z == -4 || t.z == -3 || t.z == -6) ? ex->hchain[t.x] : t.x;
      return ex->hphase[tag];
    };
    std::stable_sort(a.begin(), a.end(), [&](const int4 &l, const int4 &r) { return tphase(l) < tphase(r); });
    int32_t c0 = 0, c1 = 0;
    for (const int4 &t : a) {
      const int ph = tphase(t);
      c0 += ph < 1;
      c1 += ph < 2;
    }
    ex->pe0 = c0;
    ex->pe1 = c1;
  }
  // the unpacks last: every push and local task is grabbed before a warp
  // can wait on a peer's DONE
  a.insert(a.end(), unp.begin(), unp.end());
  ex->htasks.swap(a);
}

void apply_l2_fetch_limit() {
  static std::once_flag once;
  std::call_once(once, []() {
    const char *v = std::getenv("GHX_L2_FETCH");
    size_t g = v ? (size_t)std::atoi(v) : 0;
    if (g == 32 || g == 64 || g == 128) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, g);
  });
}

}  // namespace

extern "C" {

int64_t ghx_launch_count(void) { return g_launches.load(); }

int ghx_exec_create(const ghx_plan *plan, int32_t rank, int32_t kind, const int64_t *src_fab_boxes,
                    int32_t src_ncomp_total, const int64_t *dst_fab_boxes, int32_t dst_ncomp_total,
                    int32_t scomp, int32_t dcomp, int32_t ncomp, int32_t elem_bytes, int32_t device,
                    ghx_exec **out) {
  const bool want_phased = (kind & GHX_EXEC_PHASED) != 0;
  const int xsel = kind & (GHX_EXEC_ONLY_XFACES | GHX_EXEC_NO_XFACES | 0x800);
  kind &= ~(GHX_EXEC_PHASED | GHX_EXEC_ONLY_XFACES | GHX_EXEC_NO_XFACES | 0x800);
  if (!plan || !out || (plan->nsrc && !src_fab_boxes) || (plan->ndst && !dst_fab_boxes) ||
      rank < 0 || rank >= plan->nranks || kind < GHX_EXEC_DIRECT || kind > GHX_EXEC_EXCHANGE_PACKED ||
      (elem_bytes != 4 && elem_bytes != 8) || ncomp < 1 || scomp < 0 || dcomp < 0 ||
      scomp + ncomp > src_ncomp_total || dcomp + ncomp > dst_ncomp_total) {
    set_error("ghx_exec_create: bad arguments");
    return GHX_EINVAL;
  }
  ghx_exec *ex = nullptr;
  try {
    ex = new ghx_exec();
  } catch (const std::bad_alloc &) {
    set_error("ghx_exec_create: out of memory");
    return GHX_ENOMEM;
  }
  ex->device = device;
  ex->kind = kind;
  ex->rank = rank;
  ex->nranks = plan->nranks;
  ex->nsrc = plan->nsrc;
  ex->ndst = plan->ndst;
  ex->elem_bytes = elem_bytes;
  ex->nc_loads = plan->mode == GHX_MODE_FILL_BOUNDARY;
  if (const char *v = std::getenv("GHX_LD_MODE")) ex->ld_mode = std::atoi(v);
  ex->nptrs = (int64_t)plan->nsrc + plan->ndst + 2 * (int64_t)plan->nranks;
  ex->buf_elems.assign(plan->nranks, 0);

  auto layout = [](const int64_t *b, int32_t nct) {
    Layout L;
    L.box = ghx::box_from(b);
    L.nx = L.box.hi[0] - L.box.lo[0] + 1;
    L.ny = L.box.hi[1] - L.box.lo[1] + 1;
    L.nz = L.box.hi[2] - L.box.lo[2] + 1;
    L.ncomp = nct;
    return L;
  };
  const int32_t send_base = plan->nsrc + plan->ndst;
  const int32_t recv_base = send_base + plan->nranks;
  std::vector<int64_t> buf_off(plan->nranks, 0);
  std::vector<int64_t> recv_off(plan->nranks, 0);  // EXCHANGE_PACKED: the unpack side's receive slabs
  // remote tags with narrow rows travel packed (contiguous over NVLink);
  // the rule is identical on every rank, so pushes and unpacks agree
  static const int64_t pack_row_bytes = [] {
    const char *v = std::getenv("GHX_PACK_ROW_BYTES");
    return v ? (int64_t)std::atoll(v) : (int64_t)128;
  }();
  const bool pack_all = kind == GHX_EXEC_PUSH_PACKED_ALL || kind == GHX_EXEC_UNPACK_PACKED_ALL;
  auto packable = [&](const Piece &p) {
    return p.srank != p.drank && (pack_all || (p.dbox.hi[0] - p.dbox.lo[0] + 1) * elem_bytes <= pack_row_bytes);
  };
  // sector fill for the unpack kinds of a FillBoundary (GHX_SECTOR_FILL=0: off)
  const char *sf = std::getenv("GHX_SECTOR_FILL");
  const bool fill_ok = (kind == GHX_EXEC_UNPACK || kind == GHX_EXEC_UNPACK_PACKED || kind == GHX_EXEC_UNPACK_PACKED_ALL ||
                        kind == GHX_EXEC_EXCHANGE_PACKED) &&
                       plan->mode == GHX_MODE_FILL_BOUNDARY && !plan->clipped &&
                       (int64_t)plan->vbox.size() == plan->ndst && !(sf && std::atoi(sf) == 0);
  int64_t bad = -1;
  std::vector<Piece> taken;
  std::vector<int64_t> taken_id;  // wtags index (error reporting)
  std::vector<uint8_t> taken_sfab, taken_dfab;
  for (size_t i = 0; i < plan->wtags.size(); ++i) {
    const Piece &p = plan->wtags[i];
    bool take = false, src_is_fab = true, dst_is_fab = true;
    switch (kind) {
      case GHX_EXEC_DIRECT: take = p.srank == rank; break;
      case GHX_EXEC_LOCAL: take = p.srank == rank && p.drank == rank; break;
      case GHX_EXEC_PACK: take = p.srank == rank && p.drank != rank; dst_is_fab = false; break;
      case GHX_EXEC_UNPACK: take = p.drank == rank && p.srank != rank; src_is_fab = false; break;
      case GHX_EXEC_PUSH_PACKED:
      case GHX_EXEC_PUSH_PACKED_ALL: take = p.srank == rank; dst_is_fab = !packable(p); break;
      case GHX_EXEC_UNPACK_PACKED:
      case GHX_EXEC_UNPACK_PACKED_ALL: take = p.drank == rank && packable(p); src_is_fab = false; break;
      case GHX_EXEC_EXCHANGE_PACKED:  // this rank's pushes (as PUSH_PACKED) and unpacks (as UNPACK_PACKED)
        if (p.srank == rank) {
          take = true;
          dst_is_fab = !packable(p);
        } else if (p.drank == rank && packable(p)) {
          take = true;
          src_is_fab = false;
        }
        break;
    }
    if (take && xsel && plan->mode == GHX_MODE_FILL_BOUNDARY && (int64_t)plan->vbox.size() == plan->ndst) {
      // diagnostic split: x-face tags (outside the valid box in x only) or the rest
      const Box &V = plan->vbox[p.dst];
      int g = 0;
      for (int d = 0; d < 3; ++d)
        if (p.dbox.hi[d] < V.lo[d] || p.dbox.lo[d] > V.hi[d]) g |= 1 << d;
      const bool xface = g == 1;
      if (xsel & 0x800)  // experiment: the y / z faces alone (no x faces, edges, corners)
        take = g == 2 || g == 4;
      else
        take = (xsel & GHX_EXEC_ONLY_XFACES) ? xface : !xface;
    }
    if (!take) continue;
    taken.push_back(p);
    taken_id.push_back((int64_t)i);
    taken_sfab.push_back(src_is_fab);
    taken_dfab.push_back(dst_is_fab);
  }
  std::vector<int8_t> taken_phase(taken.size(), 0);
  if (want_phased && (kind == GHX_EXEC_DIRECT || kind == GHX_EXEC_LOCAL)) {
    std::vector<Box> sstore(plan->nsrc);
    for (int32_t f = 0; f < plan->nsrc; ++f) sstore[f] = ghx::box_from(src_fab_boxes + 6 * f);
    ex->phased = phase_pieces(plan, rank, sstore, taken, taken_phase);
    if (ex->phased) {
      taken_id.assign(taken.size(), -1);
      taken_sfab.assign(taken.size(), 1);
      taken_dfab.assign(taken.size(), 1);
    }
  }
  for (size_t i = 0; i < taken.size(); ++i) {
    const Piece &p = taken[i];
    const bool src_is_fab = taken_sfab[i], dst_is_fab = taken_dfab[i];
    const Layout S = layout(src_fab_boxes + 6 * p.src, src_ncomp_total);
    const Layout D = layout(dst_fab_boxes + 6 * p.dst, dst_ncomp_total);
    Box sbox = p.dbox;
    for (int d = 0; d < 3; ++d) {
      sbox.lo[d] -= p.shift[d];
      sbox.hi[d] -= p.shift[d];
    }
    HostTag t;
    t.nx = p.dbox.hi[0] - p.dbox.lo[0] + 1;
    t.ny = p.dbox.hi[1] - p.dbox.lo[1] + 1;
    t.nz = p.dbox.hi[2] - p.dbox.lo[2] + 1;
    t.nc = ncomp;
    t.remote = p.srank != p.drank;
    t.peer = !t.remote ? -1 : (src_is_fab ? p.drank : p.srank);
    t.sfab = p.src;
    t.dfab = p.dst;
    for (int d = 0; d < 3; ++d) t.shift[d] = p.shift[d];
    if ((src_is_fab && !contains(S.box, sbox)) || (dst_is_fab && !contains(D.box, p.dbox))) {
      bad = taken_id[i] >= 0 ? taken_id[i] : 0;
      break;
    }
    ex->cur_phase = taken_phase[i];
    const int64_t cells = t.nx * t.ny * t.nz;
    if (src_is_fab) {
      t.s.off = (sbox.lo[0] - S.box.lo[0]) +
                S.nx * ((sbox.lo[1] - S.box.lo[1]) + S.ny * ((sbox.lo[2] - S.box.lo[2]) + S.nz * scomp));
      t.s.sy = S.nx;
      t.s.sz = S.nx * S.ny;
      t.s.sc = S.nx * S.ny * S.nz;
      t.s.ptr = p.src;
    } else {  // unpack: dense F-order piece inside the recv buffer from srank
      std::vector<int64_t> &off = kind == GHX_EXEC_EXCHANGE_PACKED ? recv_off : buf_off;
      t.s.off = off[p.srank];
      t.s.sy = t.nx;
      t.s.sz = t.nx * t.ny;
      t.s.sc = cells;
      t.s.ptr = recv_base + p.srank;
      off[p.srank] += cells * ncomp;
      t.unpack_role = true;
    }
    if (dst_is_fab) {
      t.d.off = (p.dbox.lo[0] - D.box.lo[0]) +
                D.nx * ((p.dbox.lo[1] - D.box.lo[1]) + D.ny * ((p.dbox.lo[2] - D.box.lo[2]) + D.nz * dcomp));
      t.d.sy = D.nx;
      t.d.sz = D.nx * D.ny;
      t.d.sc = D.nx * D.ny * D.nz;
      t.d.ptr = plan->nsrc + p.dst;
    } else {  // pack: dense F-order piece inside the send buffer to drank
      t.d.off = buf_off[p.drank];
      t.d.sy = t.nx;
      t.d.sz = t.nx * t.ny;
      t.d.sc = cells;
      t.d.ptr = send_base + p.drank;
      buf_off[p.drank] += cells * ncomp;
    }
    if (fill_ok && !src_is_fab && dst_is_fab) {
      // an x-face ghost piece (outside the valid box in x only): its sectors'
      // other halves may be valid cells, which a FillBoundary never writes
      const Box &V = plan->vbox[p.dst];
      bool xface = p.dbox.hi[0] < V.lo[0] || p.dbox.lo[0] > V.hi[0];
      for (int d = 1; d < 3; ++d) xface = xface && p.dbox.lo[d] >= V.lo[d] && p.dbox.hi[d] <= V.hi[d];
      if (xface) {
        t.fill_x0 = p.dbox.lo[0] - D.box.lo[0];
        t.fill_vlo = V.lo[0] - D.box.lo[0];
        t.fill_vhi = V.hi[0] - D.box.lo[0];
      }
    }
    if (cells * ncomp >= (1ll << 31)) {
      set_error("ghx_exec_create: a single tag exceeds 2^31 elements");
      delete ex;
      return GHX_EINVAL;
    }
    ex->elems += cells * ncomp;
    emit_tag(ex, t);
  }
  if (bad >= 0) {
    const Piece &p = plan->wtags[bad];
    set_error("ghx_exec_create: tag " + std::to_string(bad) + " (src fab " + std::to_string(p.src) +
              " -> dst fab " + std::to_string(p.dst) +
              ") reaches outside the fab storage box (storage ngrow too small)");
    delete ex;
    return GHX_EINVAL;
  }
  ex->buf_elems = buf_off;
  ex->recv_elems = kind == GHX_EXEC_EXCHANGE_PACKED ? recv_off
                   : (kind == GHX_EXEC_UNPACK || kind == GHX_EXEC_UNPACK_PACKED || kind == GHX_EXEC_UNPACK_PACKED_ALL)
                       ? buf_off
                       : std::vector<int64_t>(plan->nranks, 0);
  if (ex->htags.size() >= (size_t)INT32_MAX) {
    set_error("ghx_exec_create: too many tags");
    delete ex;
    return GHX_EINVAL;
  }
  {
    // fab-local task order pays when a fab's lines can stay in L2 while its
    // tasks run: FillBoundary with under 64 MiB per fab (C2, C4; not C3)
    double bytes = 0;
    for (int32_t f = 0; f < plan->ndst; ++f) {
      const Layout D = layout(dst_fab_boxes + 6 * f, dst_ncomp_total);
      bytes += (double)D.nx * D.ny * D.nz * D.ncomp * elem_bytes;
    }
    ex->fab_local = plan->mode == GHX_MODE_FILL_BOUNDARY && plan->ndst > 0 && bytes / plan->ndst < 64.0 * (1 << 20);
    if (const char *v = std::getenv("GHX_FAB_LOCAL")) ex->fab_local = std::atoi(v) != 0;
    // TMA bulk rows for the wide face rows of large-fab FillBoundary (C3:
    // -3.6 %; small fabs keep the fab-local LSU order, which bulk rows slow)
    ex->bulk = plan->mode == GHX_MODE_FILL_BOUNDARY && !ex->fab_local;
    if (const char *v = std::getenv("GHX_BULK")) ex->bulk = plan->mode == GHX_MODE_FILL_BOUNDARY && std::atoi(v) != 0;
  }
  build_tasks(ex);
  if (ex->htasks.size() >= (size_t)INT32_MAX / 2) {
    set_error("ghx_exec_create: too many tasks");
    delete ex;
    return GHX_EINVAL;
  }

  // device tables are uploaded on first run (host-only builds work without a GPU)
  *out = ex;
  return GHX_OK;
}

}  // extern "C"

static int bulk_smem_attr(int device) {
  static std::mutex mu;
  static std::vector<char> done;
  std::lock_guard<std::mutex> lk(mu);
  if (device >= 0 && (size_t)device < done.size() && done[device]) return GHX_OK;
  cudaError_t e = cudaFuncSetAttribute(ghx_copy_kernel<2, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kWarps * kBulkBytes);
  if (e != cudaSuccess) return cuda_fail(e, "ghx_exec_run: bulk-row shared memory attribute");
  if (device >= 0) {
    if ((size_t)device >= done.size()) done.resize(device + 1, 0);
    done[device] = 1;
  }
  return GHX_OK;
}

static int exec_upload(ghx_exec *ex) {
  if (ex->uploaded) return GHX_OK;
  apply_l2_fetch_limit();
  cudaError_t e;
  if (!ex->htags.empty()) {
    e = cudaMalloc(&ex->dtags, ex->htags.size() * sizeof(DevTag));
    if (e == cudaSuccess)
      e = cudaMemcpy(ex->dtags, ex->htags.data(), ex->htags.size() * sizeof(DevTag), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&ex->dchain, std::max<size_t>(1, ex->hchain.size()) * sizeof(int));
    if (e == cudaSuccess && !ex->hchain.empty())
      e = cudaMemcpy(ex->dchain, ex->hchain.data(), ex->hchain.size() * sizeof(int), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&ex->dtasks, ex->htasks.size() * sizeof(int4));
    if (e == cudaSuccess)
      e = cudaMemcpy(ex->dtasks, ex->htasks.data(), ex->htasks.size() * sizeof(int4), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "ghx_exec_run: tag upload");
  }
  e = cudaMalloc(&ex->dptrs, std::max<int64_t>(ex->nptrs, 1) * sizeof(void *));
  if (e != cudaSuccess) return cuda_fail(e, "ghx_exec_run: pointer table");
  if (ex->blocks == 0) {
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ghx_copy_kernel<0>, kThreads, 0);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ex->device);
    if (e != cudaSuccess || occ < 1) occ = 1;
    const int64_t need = ((int64_t)ex->htasks.size() + kWarps - 1) / kWarps;
    ex->blocks = (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)sms * occ));
    if (const char *v = std::getenv("GHX_BLOCKS")) ex->blocks = std::max(1, std::atoi(v));
  }
  ex->uploaded = true;
  return GHX_OK;
}

extern "C" {

void ghx_exec_free(ghx_exec *ex) {
  if (!ex) return;
  DeviceGuard g(ex->device);
  for (auto &b : ex->bindings) {
    cudaFree(b->dtags);
    cudaFree(b->dptrs);
    cudaFree(b->counter);
  }
  if (ex->dtags) cudaFree(ex->dtags);
  if (ex->dtasks) cudaFree(ex->dtasks);
  if (ex->dchain) cudaFree(ex->dchain);
  if (ex->dptrs) cudaFree(ex->dptrs);
  if (ex->dflags) cudaFree(ex->dflags);
  if (ex->dpeer) cudaFree(ex->dpeer);
  if (ex->dpeer_total) cudaFree(ex->dpeer_total);
  delete ex;
}

int ghx_exec_set_ring(ghx_exec *ex, int32_t on) {
  if (!ex) {
    set_error("ghx_exec_set_ring: null handle");
    return GHX_EINVAL;
  }
  std::lock_guard<std::mutex> lk(ex->mu);
  if (ex->uploaded) {
    set_error("ghx_exec_set_ring: the executor has already run");
    return GHX_EINVAL;
  }
  if (ex->ring != (on != 0)) {
    ex->ring = on != 0;
    build_tasks(ex);
  }
  return GHX_OK;
}

int ghx_exec_set_bulk(ghx_exec *ex, int32_t on) {
  if (!ex) {
    set_error("ghx_exec_set_bulk: null handle");
    return GHX_EINVAL;
  }
  std::lock_guard<std::mutex> lk(ex->mu);
  if (ex->uploaded) {
    set_error("ghx_exec_set_bulk: the executor has already run");
    return GHX_EINVAL;
  }
  if (ex->bulk != (on != 0)) {
    ex->bulk = on != 0;
    build_tasks(ex);
  }
  return GHX_OK;
}

int ghx_exec_set_grid(ghx_exec *ex, int32_t blocks, int32_t threads) {
  if (!ex || threads != kThreads || blocks < 0) {
    set_error("ghx_exec_set_grid: only 256-thread blocks are compiled");
    return GHX_EINVAL;
  }
  if (blocks > 0) ex->blocks = blocks;
  return GHX_OK;
}

int ghx_exec_info(const ghx_exec *ex, int64_t *ntags, int64_t *ntasks, int64_t *elems, int64_t *alg_bytes) {
  if (!ex) {
    set_error("ghx_exec_info: null handle");
    return GHX_EINVAL;
  }
  if (ntags) *ntags = (int64_t)ex->htags.size();
  if (ntasks) *ntasks = (int64_t)ex->htasks.size();
  if (elems) *elems = ex->elems;
  if (alg_bytes) *alg_bytes = 2 * ex->elems * ex->elem_bytes;
  return GHX_OK;
}

int ghx_exec_detail(const ghx_exec *ex, int64_t out[8]) {
  if (!ex || !out) {
    set_error("ghx_exec_detail: bad arguments");
    return GHX_EINVAL;
  }
  out[0] = (int64_t)ex->htags.size();
  out[1] = (int64_t)ex->htasks.size();
  out[2] = ex->elems;
  out[3] = 2 * ex->elems * ex->elem_bytes;
  out[4] = ex->npaired;
  out[5] = ex->nswap;
  out[6] = ex->blocks;
  out[7] = ex->ld_mode;
  return GHX_OK;
}

int ghx_exec_task_kinds(const ghx_exec *ex, int64_t out[6]) {
  if (!ex || !out) {
    set_error("ghx_exec_task_kinds: bad arguments");
    return GHX_EINVAL;
  }
  for (int i = 0; i < 6; ++i) out[i] = 0;
  for (const int4 &t : ex->htasks) {
    if (t.z == -4 || t.z == -6)
      out[3] += 1;
    else if (t.z == -3)
      out[2] += 1;
    else if (t.z == -2)
      out[1] += 1;
    else
      out[0] += 1;
  }
  out[4] = ex->ring ? 1 : 0;
  out[5] = ex->fab_local ? 1 : 0;
  return GHX_OK;
}

int ghx_exec_phases(const ghx_exec *ex, int64_t out[4]) {
  if (!ex || !out) {
    set_error("ghx_exec_phases: bad arguments");
    return GHX_EINVAL;
  }
  out[0] = ex->phased ? 1 : 0;
  out[1] = ex->pe0;
  out[2] = ex->pe1;
  out[3] = (int64_t)ex->htags.size();
  return GHX_OK;
}

int ghx_exec_recv_elems(const ghx_exec *ex, int64_t *per_peer) {
  if (!ex || !per_peer) {
    set_error("ghx_exec_recv_elems: bad arguments");
    return GHX_EINVAL;
  }
  for (size_t i = 0; i < ex->recv_elems.size(); ++i) per_peer[i] = ex->recv_elems[i];
  return GHX_OK;
}

int ghx_exec_sector_fills(const ghx_exec *ex, int64_t *ntags) {
  if (!ex || !ntags) {
    set_error("ghx_exec_sector_fills: bad arguments");
    return GHX_EINVAL;
  }
  *ntags = ex->nfill;
  return GHX_OK;
}

int ghx_exec_buffer_elems(const ghx_exec *ex, int64_t *per_peer) {
  if (!ex || !per_peer) {
    set_error("ghx_exec_buffer_elems: bad arguments");
    return GHX_EINVAL;
  }
  for (int32_t r = 0; r < ex->nranks; ++r) per_peer[r] = ex->buf_elems[r];
  return GHX_OK;
}

}  // extern "C"

namespace {

constexpr size_t kMaxLoose = 4;

int check_table(ghx_exec *ex, void *const *ptrs, int64_t nptrs) {
  const uintptr_t amask = ex->nswap ? 31 : 15;
  for (int64_t i = 0; i < nptrs; ++i)
    if (reinterpret_cast<uintptr_t>(ptrs[i]) & amask) {
      set_error("ghx_exec_run: base pointer " + std::to_string(i) + " is not " + std::to_string(amask + 1) +
                "-byte aligned");
      return GHX_EINVAL;
    }
  // every slot referenced by this rank's tags must be set
  for (const DevTag &t : ex->htags)
    if (!ptrs[t.src_ptr] || !ptrs[t.dst_ptr]) {
      set_error("ghx_exec_run: a pointer slot used by this rank's tags is NULL");
      return GHX_EINVAL;
    }
  // sector swaps read and write both fabs of a pair through one slot each
  if (ex->nswap)
    for (int32_t f = 0; f < std::min(ex->nsrc, ex->ndst); ++f)
      if (ex->swap_fab.size() > (size_t)f && ex->swap_fab[f] && ptrs[f] != ptrs[ex->nsrc + f]) {
        set_error("ghx_exec_run: FillBoundary executor needs src slot == dst slot for every fab");
        return GHX_EINVAL;
      }
  return GHX_OK;
}

// Find the binding of this pointer table, or create one (recycling the
// least recently used unpinned binding when kMaxLoose are in use).  The
// bind (table upload + ghx_bind_kernel) is stream-ordered on st.  Caller
// holds ex->mu.
int find_or_bind(ghx_exec *ex, void *const *ptrs, int64_t nptrs, cudaStream_t st, ghx_exec::Binding **out) {
  for (auto &b : ex->bindings)
    if (b->ptrs.size() == (size_t)nptrs && std::memcmp(b->ptrs.data(), ptrs, nptrs * sizeof(void *)) == 0) {
      *out = b.get();
      return GHX_OK;
    }
  if (int rc = check_table(ex, ptrs, nptrs)) return rc;
  ghx_exec::Binding *bd = nullptr;
  size_t loose = 0;
  for (auto &b : ex->bindings) loose += b->pins == 0;
  if (loose >= kMaxLoose) {  // recycle the LRU unpinned binding (stream-ordered rebind)
    for (auto &b : ex->bindings)
      if (b->pins == 0 && (!bd || b->last_use < bd->last_use)) bd = b.get();
  } else {
    std::unique_ptr<ghx_exec::Binding> nb(new ghx_exec::Binding());
    cudaError_t e = cudaMalloc(&nb->dtags, std::max<size_t>(1, ex->htags.size()) * sizeof(DevTag));
    if (e == cudaSuccess) e = cudaMalloc(&nb->dptrs, std::max<int64_t>(ex->nptrs, 1) * sizeof(void *));
    // [0, 8) scheduler / phase counters, [8, 72) EXCHANGE_PACKED's per-peer push counts
    if (e == cudaSuccess) e = cudaMalloc(&nb->counter, 72 * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemsetAsync(nb->counter, 0, 72 * sizeof(unsigned long long), st);
    if (e == cudaSuccess && !ex->htags.empty())
      e = cudaMemcpyAsync(nb->dtags, ex->dtags, ex->htags.size() * sizeof(DevTag), cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) {
      cudaFree(nb->dtags);
      cudaFree(nb->dptrs);
      cudaFree(nb->counter);
      return cuda_fail(e, "ghx_exec_run: binding");
    }
    nb->id = ex->next_binding++;
    bd = nb.get();
    ex->bindings.push_back(std::move(nb));
  }
  bd->ptrs.assign(ptrs, ptrs + nptrs);
  // pageable source: the copy has consumed the host table when this returns
  cudaError_t e = cudaMemcpyAsync(bd->dptrs, bd->ptrs.data(), nptrs * sizeof(void *), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) {
    const int n = (int)ex->htags.size();
    if (n) ghx_bind_kernel<<<std::min(1184, (n + 255) / 256), 256, 0, st>>>(bd->dtags, n, bd->dptrs);
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) {
    bd->ptrs.clear();
    return cuda_fail(e, "ghx_exec_run: pointer bind");
  }
  *out = bd;
  return GHX_OK;
}

static uint64_t sync_timeout_ns() {
  static const uint64_t ns = [] {
    const char *v = std::getenv("GHX_BARRIER_TIMEOUT_S");
    const double sec = v ? std::atof(v) : 30.0;
    return (uint64_t)(sec * 1e9);
  }();
  return ns;
}

int launch(ghx_exec *ex, ghx_exec::Binding *bd, cudaStream_t st, const SyncArgs &sync_in) {
  bd->last_use = ++ex->uses;
  SyncArgs sync = sync_in;
  sync.pe0 = ex->phased ? ex->pe0 : 0;
  sync.pe1 = ex->phased ? ex->pe1 : 0;
  if (ex->phased && sync.timeout_ns == 0) sync.timeout_ns = sync_timeout_ns();
  DevTag *const dtags = bd->dtags;
  unsigned long long *const counter = bd->counter;
  const int ntasks = (int)ex->htasks.size();
  int blocks = ex->blocks;
  if (ex->phased) {  // phase waits need every CTA resident
    static int cap = [] {
      int occ = 0, sms = 148;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ghx_copy_kernel<2, true>, kThreads, 0);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
      return std::max(1, occ) * sms;
    }();
    blocks = std::min(blocks, cap);
  }
  int ld = ex->ld_mode;
  if (ld == 0 && !ex->nc_loads) ld = 2;  // sources may alias destinations (ParallelCopy): no .nc
  if (ex->nbulk && ex->nring) {
    set_error("ghx_exec_run: ring and bulk tasks in one executor");
    return GHX_EINVAL;
  }
  if (ex->nbulk) {
    // the dynamic shared memory limit is a per-device (per-context) function
    // attribute: set it once on every device that launches bulk rows
    if (int rc = bulk_smem_attr(ex->device)) return rc;
  }
  // one launch over tasks [first, first + count)
  auto go = [&](int first, int count, int nblocks, bool ring, const SyncArgs &sy) {
    if (count <= 0) return;
    // tasks per atomic grab: single tasks balance the latency-bound seam work
    // best (FillBoundary plans, measured), long streaming task lists
    // (ParallelCopy regrids) amortise the atomic over ~64 grabs per warp
    int batch = (int)std::max<int64_t>(1, std::min<int64_t>(64, count / ((int64_t)nblocks * kWarps * 64)));
    if (const char *v = std::getenv("GHX_BATCH")) batch = std::max(1, std::atoi(v));
    const int4 *tk = ex->dtasks + first;
    if (ex->nbulk)
      ghx_copy_kernel<2, false, true><<<nblocks, ex->threads, kWarps * kBulkBytes, st>>>(dtags, tk, count, ex->dchain,
                                                                                        counter, batch, sy);
    else if (ring)  // ring tasks present: the ring-capable instantiation
      ghx_copy_kernel<2, true><<<nblocks, ex->threads, 0, st>>>(dtags, tk, count, ex->dchain, counter, batch, sy);
    else if (ex->nfill)  // sector-fill tasks (unpack): their own instantiation keeps the others spill-free
      ghx_copy_kernel<2, false, false, true><<<nblocks, ex->threads, 0, st>>>(dtags, tk, count, ex->dchain, counter,
                                                                             batch, sy);
    else switch (ld) {
      case 0: ghx_copy_kernel<0><<<nblocks, ex->threads, 0, st>>>(dtags, tk, count, ex->dchain, counter, batch, sy); break;
      case 1: ghx_copy_kernel<1><<<nblocks, ex->threads, 0, st>>>(dtags, tk, count, ex->dchain, counter, batch, sy); break;
      case 2: ghx_copy_kernel<2><<<nblocks, ex->threads, 0, st>>>(dtags, tk, count, ex->dchain, counter, batch, sy); break;
      case 3: ghx_copy_kernel<3><<<nblocks, ex->threads, 0, st>>>(dtags, tk, count, ex->dchain, counter, batch, sy); break;
      default: ghx_copy_kernel<4><<<nblocks, ex->threads, 0, st>>>(dtags, tk, count, ex->dchain, counter, batch, sy); break;
    }
    g_launches.fetch_add(1);
  };
  // Experiment (GHX_PHASE_LAUNCHES=1): a phased executor with no cross-rank
  // sync runs its three phases as three stream-ordered launches (no
  // in-kernel phase waits), the face phases on a wider grid
  // (GHX_HOST_FACE_BLOCKS, 32).  Measured: C3 e2e 49.7 -> 48.7 ms, C2 same,
  // C4 27.2 -> 28.8 ms -- the single launch with phase waits stays.
  static const bool split = [] {
    const char *v = std::getenv("GHX_PHASE_LAUNCHES");
    return v && std::atoi(v) != 0;
  }();
  if (ex->phased && split && sync.mode == 0) {
    static const int face_blocks = [] {
      const char *v = std::getenv("GHX_HOST_FACE_BLOCKS");
      return v ? std::max(1, std::atoi(v)) : 32;
    }();
    SyncArgs plain = sync;
    plain.pe0 = plain.pe1 = 0;
    const int fb = std::max(blocks, face_blocks);
    go(0, ex->pe0, blocks, ex->nring > 0 || ex->nseam > 0, plain);
    go(ex->pe0, ex->pe1 - ex->pe0, fb, false, plain);
    go(ex->pe1, ntasks - ex->pe1, fb, false, plain);
  } else {
    go(0, ntasks, blocks, ex->nring > 0 || ex->nseam > 0, sync);  // seam tasks live in the ring instantiation
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "ghx_exec_run: launch");
  return GHX_OK;
}

}  // namespace

extern "C" {

int ghx_exec_run(ghx_exec *ex, void *const *ptrs, int64_t nptrs, void *stream) {
  if (!ex || (nptrs && !ptrs) || nptrs != ex->nptrs) {
    set_error("ghx_exec_run: pointer table must have nsrc + ndst + 2*nranks entries");
    return GHX_EINVAL;
  }
  if (ex->kind == GHX_EXEC_EXCHANGE_PACKED) {  // its unpacks must wait for the peers' DONE
    set_error("ghx_exec_run: GHX_EXEC_EXCHANGE_PACKED executors run through ghx_exec_run_synced only");
    return GHX_EINVAL;
  }
  if (ex->htasks.empty()) return GHX_OK;
  std::lock_guard<std::mutex> lk(ex->mu);
  DeviceGuard g(ex->device);
  if (int rc = exec_upload(ex)) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ghx_exec::Binding *bd = nullptr;
  if (int rc = find_or_bind(ex, ptrs, nptrs, st, &bd)) return rc;
  return launch(ex, bd, st, SyncArgs{});
}

int ghx_exec_bind(ghx_exec *ex, void *const *ptrs, int64_t nptrs, void *stream, int64_t *binding) {
  if (!ex || !binding || (nptrs && !ptrs) || nptrs != ex->nptrs) {
    set_error("ghx_exec_bind: pointer table must have nsrc + ndst + 2*nranks entries");
    return GHX_EINVAL;
  }
  *binding = 0;
  if (ex->htasks.empty()) return GHX_OK;  // nothing to run: binding 0 is a no-op
  std::lock_guard<std::mutex> lk(ex->mu);
  DeviceGuard g(ex->device);
  if (int rc = exec_upload(ex)) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ghx_exec::Binding *bd = nullptr;
  if (int rc = find_or_bind(ex, ptrs, nptrs, st, &bd)) return rc;
  bd->pins += 1;
  *binding = bd->id;
  // a pinned binding may be launched on any stream later: make the bind
  // complete now unless this stream is being captured into a graph (then
  // the bind is part of the graph, ahead of the launch)
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  if (cs == cudaStreamCaptureStatusNone) {
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "ghx_exec_bind: synchronize");
  }
  return GHX_OK;
}

int ghx_exec_run_bound(ghx_exec *ex, int64_t binding, void *stream) {
  if (!ex) {
    set_error("ghx_exec_run_bound: null handle");
    return GHX_EINVAL;
  }
  if (ex->kind == GHX_EXEC_EXCHANGE_PACKED) {
    set_error("ghx_exec_run_bound: GHX_EXEC_EXCHANGE_PACKED executors run through ghx_exec_run_synced only");
    return GHX_EINVAL;
  }
  if (ex->htasks.empty()) return GHX_OK;
  std::lock_guard<std::mutex> lk(ex->mu);
  DeviceGuard g(ex->device);
  for (auto &b : ex->bindings)
    if (b->id == binding && b->pins > 0) return launch(ex, b.get(), static_cast<cudaStream_t>(stream), SyncArgs{});
  set_error("ghx_exec_run_bound: unknown or released binding " + std::to_string(binding));
  return GHX_EINVAL;
}

int ghx_exec_set_sync(ghx_exec *ex, uint64_t *const *flag_arrays, int32_t rank, int32_t nranks) {
  if (!ex || !flag_arrays || nranks < 1 || nranks > 64 || rank < 0 || rank >= nranks || nranks != ex->nranks) {
    set_error("ghx_exec_set_sync: bad arguments (nranks <= 64, matching the plan)");
    return GHX_EINVAL;
  }
  if (ex->kind == GHX_EXEC_EXCHANGE_PACKED && nranks > 32) {
    set_error("ghx_exec_set_sync: GHX_EXEC_EXCHANGE_PACKED synchronises at most 32 ranks");
    return GHX_EINVAL;
  }
  for (int i = 0; i < nranks; ++i)
    if (!flag_arrays[i]) {
      set_error("ghx_exec_set_sync: null flag array");
      return GHX_EINVAL;
    }
  std::lock_guard<std::mutex> lk(ex->mu);
  DeviceGuard g(ex->device);
  cudaError_t e = cudaSuccess;
  if (!ex->dflags) e = cudaMalloc(&ex->dflags, 64 * sizeof(uint64_t *));
  if (e == cudaSuccess) e = cudaMemcpy(ex->dflags, flag_arrays, nranks * sizeof(uint64_t *), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !ex->dpeer)
    e = cudaMalloc(&ex->dpeer, std::max<size_t>(1, ex->hpeer.size()) * sizeof(int32_t));
  if (e == cudaSuccess && !ex->hpeer.empty())
    e = cudaMemcpy(ex->dpeer, ex->hpeer.data(), ex->hpeer.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !ex->dpeer_total) e = cudaMalloc(&ex->dpeer_total, 64 * sizeof(int32_t));
  if (e == cudaSuccess && ex->peer_total.size() == 64)
    e = cudaMemcpy(ex->dpeer_total, ex->peer_total.data(), 64 * sizeof(int32_t), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_fail(e, "ghx_exec_set_sync");
  ex->sync_rank = rank;
  ex->sync_n = nranks;
  return GHX_OK;
}

static int sync_args(ghx_exec *ex, uint64_t epoch, int32_t mode, SyncArgs *out) {
  if (ex->sync_rank < 0 || !ex->dflags) {
    set_error("ghx_exec_run_synced: ghx_exec_set_sync was not called");
    return GHX_EINVAL;
  }
  SyncArgs s{};
  s.flags = ex->dflags;
  s.tag_peer = ex->dpeer;
  s.epoch = epoch;
  s.timeout_ns = sync_timeout_ns();
  s.rank = ex->sync_rank;
  s.nranks = ex->sync_n;
  s.mode = mode;
  s.nhead = ex->nhead;
  s.peer_total = ex->dpeer_total;
  *out = s;
  return GHX_OK;
}

int ghx_exec_run_synced(ghx_exec *ex, int64_t binding, uint64_t epoch, void *stream) {
  if (!ex) {
    set_error("ghx_exec_run_synced: null handle");
    return GHX_EINVAL;
  }
  const bool unpack = ex->kind == GHX_EXEC_UNPACK_PACKED || ex->kind == GHX_EXEC_UNPACK_PACKED_ALL;
  const bool push = ex->kind == GHX_EXEC_DIRECT || ex->kind == GHX_EXEC_PUSH_PACKED ||
                    ex->kind == GHX_EXEC_PUSH_PACKED_ALL;
  const bool both = ex->kind == GHX_EXEC_EXCHANGE_PACKED;
  if (!unpack && !push && !both) {
    set_error("ghx_exec_run_synced: only push (direct / packed), packed-unpack and exchange executors "
              "synchronise in-kernel");
    return GHX_EINVAL;
  }
  std::lock_guard<std::mutex> lk(ex->mu);
  DeviceGuard g(ex->device);
  SyncArgs s;
  if (int rc = sync_args(ex, epoch, both ? 3 : (unpack ? 2 : 1), &s)) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (ex->htasks.empty()) {  // nothing to move: still signal (push) / wait (unpack)
    ghx_sync_kernel<<<1, 32, 0, st>>>(s);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? GHX_OK : cuda_fail(e, "ghx_exec_run_synced: sync kernel");
  }
  for (auto &b : ex->bindings)
    if (b->id == binding && b->pins > 0) return launch(ex, b.get(), st, s);
  set_error("ghx_exec_run_synced: unknown or released binding " + std::to_string(binding));
  return GHX_EINVAL;
}

int ghx_exec_sync_wait(ghx_exec *ex, uint64_t epoch, void *stream) {
  if (!ex) {
    set_error("ghx_exec_sync_wait: null handle");
    return GHX_EINVAL;
  }
  std::lock_guard<std::mutex> lk(ex->mu);
  DeviceGuard g(ex->device);
  SyncArgs s;
  if (int rc = sync_args(ex, epoch, 2, &s)) return rc;
  ghx_sync_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(s);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? GHX_OK : cuda_fail(e, "ghx_exec_sync_wait");
}

int ghx_exec_unbind(ghx_exec *ex, int64_t binding) {
  if (!ex) {
    set_error("ghx_exec_unbind: null handle");
    return GHX_EINVAL;
  }
  if (binding == 0) return GHX_OK;
  std::lock_guard<std::mutex> lk(ex->mu);
  for (auto &b : ex->bindings)
    if (b->id == binding && b->pins > 0) {
      b->pins -= 1;  // stays allocated; recyclable once unpinned
      return GHX_OK;
    }
  set_error("ghx_exec_unbind: unknown or released binding " + std::to_string(binding));
  return GHX_EINVAL;
}

}  // extern "C"

// timeouts of the in-kernel waits (added to ghx_barrier_timeouts)
int64_t ghx::sync_timeouts() {
  unsigned int v = 0;
  if (cudaMemcpyFromSymbol(&v, g_sync_timeouts, sizeof(v)) != cudaSuccess) return -1;
  return (int64_t)v;
}
