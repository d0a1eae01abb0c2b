// Copy-plan builder: box-intersection tags for FillBoundary and
// ParallelCopy, binned instead of the reference's all-pairs loop.
//
// Semantics follow /root/reference/pkg/src/miniamr_core/comm.py:
//   _shift_candidates    comm.py:250-266  (periodic k ranges per axis)
//   _build_copy_segments comm.py:269-286  (intersect + box_diff pieces)
//   CommPlan             comm.py:218-237  (sort key + rank-pair grouping)
//   box_diff             index_space.py:297-320 (axis order, lo then hi)
// The set of (dst, src, shift) triples is exactly the set of lattice
// shifts s for which src + s meets the dst target, so any exact spatial
// search reproduces the reference's segments; after sorting by the unique
// key (dst_fab, dst_lo, src_fab, shift) the order is identical too.
#include <algorithm>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "ghx_internal.h"

namespace ghx {

static thread_local std::string g_err;
void set_error(const std::string &msg) { g_err = msg; }

static inline int64_t floor_div(int64_t a, int64_t b) {
  int64_t q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
  return q;
}
static inline int64_t ceil_div(int64_t a, int64_t b) { return -floor_div(-a, b); }

// Uniform-grid bin index over a box list (CSR: bin -> box ids).
struct BinIndex {
  int64_t org[3] = {0, 0, 0}, bsz[3] = {1, 1, 1}, nb[3] = {1, 1, 1};
  Box bb{};
  bool any = false;
  std::vector<int64_t> start;
  std::vector<int32_t> ids;

  void range(const Box &b, int64_t lo[3], int64_t hi[3]) const {
    for (int d = 0; d < 3; ++d) {
      int64_t l = b.lo[d] < bb.lo[d] ? bb.lo[d] : b.lo[d];
      int64_t h = b.hi[d] > bb.hi[d] ? bb.hi[d] : b.hi[d];
      lo[d] = (l - org[d]) / bsz[d];
      hi[d] = (h - org[d]) / bsz[d];
    }
  }

  void build(const std::vector<Box> &boxes) {
    const int64_t n = (int64_t)boxes.size();
    any = false;
    for (const Box &b : boxes) {
      if (b.empty()) continue;
      if (!any) {
        bb = b;
        any = true;
        for (int d = 0; d < 3; ++d) bsz[d] = b.hi[d] - b.lo[d] + 1;
        continue;
      }
      for (int d = 0; d < 3; ++d) {
        bb.lo[d] = std::min(bb.lo[d], b.lo[d]);
        bb.hi[d] = std::max(bb.hi[d], b.hi[d]);
        bsz[d] = std::max(bsz[d], b.hi[d] - b.lo[d] + 1);
      }
    }
    if (!any) return;
    for (int d = 0; d < 3; ++d) org[d] = bb.lo[d];
    auto nbins = [&]() {
      int64_t t = 1;
      for (int d = 0; d < 3; ++d) {
        nb[d] = (bb.hi[d] - bb.lo[d]) / bsz[d] + 1;
        t *= nb[d];
      }
      return t;
    };
    while (nbins() > 8 * n + 64) {
      int dm = 0;
      for (int d = 1; d < 3; ++d)
        if (nb[d] > nb[dm]) dm = d;
      bsz[dm] *= 2;
    }
    const int64_t total = nb[0] * nb[1] * nb[2];
    start.assign(total + 1, 0);
    int64_t lo[3], hi[3];
    for (const Box &b : boxes) {
      if (b.empty()) continue;
      range(b, lo, hi);
      for (int64_t z = lo[2]; z <= hi[2]; ++z)
        for (int64_t y = lo[1]; y <= hi[1]; ++y)
          for (int64_t x = lo[0]; x <= hi[0]; ++x) ++start[(z * nb[1] + y) * nb[0] + x + 1];
    }
    for (int64_t i = 0; i < total; ++i) start[i + 1] += start[i];
    ids.assign(start[total], 0);
    std::vector<int64_t> fill(start.begin(), start.end() - 1);
    for (int64_t i = 0; i < n; ++i) {
      const Box &b = boxes[i];
      if (b.empty()) continue;
      range(b, lo, hi);
      for (int64_t z = lo[2]; z <= hi[2]; ++z)
        for (int64_t y = lo[1]; y <= hi[1]; ++y)
          for (int64_t x = lo[0]; x <= hi[0]; ++x) ids[fill[(z * nb[1] + y) * nb[0] + x]++] = (int32_t)i;
    }
  }

  // f(id) for every box registered in a bin that q touches (duplicates
  // possible when a box spans several bins).
  template <class F>
  void query(const Box &q, F &&f) const {
    if (!any || q.empty() || !overlap(q, bb)) return;
    int64_t lo[3], hi[3];
    range(q, lo, hi);
    for (int64_t z = lo[2]; z <= hi[2]; ++z)
      for (int64_t y = lo[1]; y <= hi[1]; ++y)
        for (int64_t x = lo[0]; x <= hi[0]; ++x) {
          const int64_t bin = (z * nb[1] + y) * nb[0] + x;
          for (int64_t k = start[bin]; k < start[bin + 1]; ++k) f(ids[k]);
        }
  }
};

// a \ b as disjoint pieces, same decomposition as index_space.box_diff.
static void box_diff(const Box &a, const Box &b, std::vector<Box> &out) {
  out.clear();
  if (a.empty()) return;
  if (!overlap(a, b)) {
    out.push_back(a);
    return;
  }
  Box is = meet(a, b);
  Box rem = a;
  for (int d = 0; d < 3; ++d) {
    if (rem.lo[d] < is.lo[d]) {
      Box p = rem;
      p.hi[d] = is.lo[d] - 1;
      out.push_back(p);
    }
    if (rem.hi[d] > is.hi[d]) {
      Box p = rem;
      p.lo[d] = is.hi[d] + 1;
      out.push_back(p);
    }
    rem.lo[d] = is.lo[d];
    rem.hi[d] = is.hi[d];
  }
}

static bool seg_less(const Piece &a, const Piece &b) {
  if (a.dst != b.dst) return a.dst < b.dst;
  for (int d = 0; d < 3; ++d)
    if (a.dbox.lo[d] != b.dbox.lo[d]) return a.dbox.lo[d] < b.dbox.lo[d];
  if (a.src != b.src) return a.src < b.src;
  for (int d = 0; d < 3; ++d)
    if (a.shift[d] != b.shift[d]) return a.shift[d] < b.shift[d];
  return false;
}

static void build_pieces(const std::vector<Box> &targets, const std::vector<Box> *valids,
                         const std::vector<Box> &srcs, const int32_t *periodic,
                         const int64_t *period, std::vector<Piece> &out) {
  BinIndex idx;
  idx.build(srcs);
  if (!idx.any) return;
  std::vector<int64_t> mark(srcs.size(), -1);
  int64_t stamp = 0;
  std::vector<Box> parts;
  const int32_t nd = (int32_t)targets.size();
  for (int32_t dj = 0; dj < nd; ++dj) {
    const Box &t = targets[dj];
    if (t.empty()) continue;
    int64_t kmin[3] = {0, 0, 0}, kmax[3] = {0, 0, 0};
    for (int d = 0; d < 3; ++d) {
      if (periodic && periodic[d]) {
        kmin[d] = ceil_div(t.lo[d] - idx.bb.hi[d], period[d]);
        kmax[d] = floor_div(t.hi[d] - idx.bb.lo[d], period[d]);
      }
    }
    for (int64_t k2 = kmin[2]; k2 <= kmax[2]; ++k2)
      for (int64_t k1 = kmin[1]; k1 <= kmax[1]; ++k1)
        for (int64_t k0 = kmin[0]; k0 <= kmax[0]; ++k0) {
          const int64_t s[3] = {periodic ? k0 * period[0] : 0, periodic ? k1 * period[1] : 0,
                                periodic ? k2 * period[2] : 0};
          Box q = t;
          for (int d = 0; d < 3; ++d) {
            q.lo[d] -= s[d];
            q.hi[d] -= s[d];
          }
          ++stamp;
          const bool zero = s[0] == 0 && s[1] == 0 && s[2] == 0;
          idx.query(q, [&](int32_t si) {
            if (mark[si] == stamp) return;
            mark[si] = stamp;
            if (!overlap(srcs[si], q)) return;
            if (valids && si == dj && zero) return;
            Box reg = meet(q, srcs[si]);
            for (int d = 0; d < 3; ++d) {
              reg.lo[d] += s[d];
              reg.hi[d] += s[d];
            }
            Piece pc;
            pc.src = si;
            pc.dst = dj;
            pc.srank = pc.drank = 0;
            for (int d = 0; d < 3; ++d) pc.shift[d] = s[d];
            if (valids) {
              box_diff(reg, (*valids)[dj], parts);
              for (const Box &p : parts) {
                pc.dbox = p;
                out.push_back(pc);
              }
            } else {
              pc.dbox = reg;
              out.push_back(pc);
            }
          });
        }
  }
}

// Last writer wins (reference order on the receiving rank: local segments
// in plan order, then each peer's message in ascending peer order,
// comm.py:328-378): clip earlier writers so destinations become disjoint.
static bool clip_writes(const std::vector<Piece> &segs, int32_t ndst, std::vector<Piece> &out) {
  out.clear();
  bool clipped = false;
  std::vector<std::vector<int64_t>> by_dst(ndst);
  for (int64_t i = 0; i < (int64_t)segs.size(); ++i) by_dst[segs[i].dst].push_back(i);
  std::vector<Box> cur, nxt, parts;
  for (int32_t dj = 0; dj < ndst; ++dj) {
    std::vector<int64_t> &ids = by_dst[dj];
    if (ids.empty()) continue;
    // quick overlap test: sweep on x
    std::vector<int64_t> ord(ids);
    std::sort(ord.begin(), ord.end(),
              [&](int64_t a, int64_t b) { return segs[a].dbox.lo[0] < segs[b].dbox.lo[0]; });
    bool any = false;
    for (size_t a = 0; a < ord.size() && !any; ++a)
      for (size_t b = a + 1; b < ord.size(); ++b) {
        if (segs[ord[b]].dbox.lo[0] > segs[ord[a]].dbox.hi[0]) break;
        if (overlap(segs[ord[a]].dbox, segs[ord[b]].dbox)) {
          any = true;
          break;
        }
      }
    if (!any) {
      for (int64_t i : ids) out.push_back(segs[i]);
      continue;
    }
    clipped = true;
    const int32_t drank = segs[ids[0]].drank;
    std::vector<int64_t> worder(ids);
    std::stable_sort(worder.begin(), worder.end(), [&](int64_t a, int64_t b) {
      const int32_t ka = segs[a].srank == drank ? -1 : segs[a].srank;
      const int32_t kb = segs[b].srank == drank ? -1 : segs[b].srank;
      if (ka != kb) return ka < kb;
      return a < b;
    });
    std::vector<Box> claimed;
    std::vector<Piece> kept;
    for (auto it = worder.rbegin(); it != worder.rend(); ++it) {
      const Piece &sg = segs[*it];
      cur.assign(1, sg.dbox);
      for (const Box &c : claimed) {
        nxt.clear();
        for (const Box &b : cur) {
          box_diff(b, c, parts);
          nxt.insert(nxt.end(), parts.begin(), parts.end());
        }
        cur.swap(nxt);
        if (cur.empty()) break;
      }
      for (const Box &b : cur) {
        Piece p = sg;
        p.dbox = b;
        kept.push_back(p);
      }
      claimed.push_back(sg.dbox);
    }
    std::sort(kept.begin(), kept.end(), seg_less);
    out.insert(out.end(), kept.begin(), kept.end());
  }
  return clipped;
}

static int finish_plan(ghx_plan *p, std::vector<Piece> &pieces, const int32_t *src_rank,
                       const int32_t *dst_rank) {
  std::sort(pieces.begin(), pieces.end(), seg_less);
  for (Piece &pc : pieces) {
    pc.srank = src_rank[pc.src];
    pc.drank = dst_rank[pc.dst];
  }
  p->segs.swap(pieces);
  p->clipped = clip_writes(p->segs, p->ndst, p->wtags);
  return GHX_OK;
}

static bool check_ranks(const int32_t *r, int64_t n, int32_t nranks) {
  for (int64_t i = 0; i < n; ++i)
    if (r[i] < 0 || r[i] >= nranks) return false;
  return true;
}

}  // namespace ghx

using namespace ghx;

extern "C" {

const char *ghx_last_error(void) { return g_err.c_str(); }
int ghx_version(void) { return 1; }

int ghx_boxes_disjoint(int64_t nboxes, const int64_t *boxes, int64_t *oa, int64_t *ob) {
  if (nboxes < 0 || (nboxes > 0 && !boxes) || !oa || !ob) {
    set_error("ghx_boxes_disjoint: bad arguments");
    return GHX_EINVAL;
  }
  std::vector<Box> bs(nboxes);
  for (int64_t i = 0; i < nboxes; ++i) bs[i] = box_from(boxes + 6 * i);
  BinIndex idx;
  idx.build(bs);
  int64_t ba = -1, bb = -1;
  for (int64_t i = 0; i < nboxes; ++i) {
    if (ba >= 0 && i > ba) break;
    idx.query(bs[i], [&](int32_t j) {
      if (j <= i || !overlap(bs[i], bs[j])) return;
      if (ba < 0 || i < ba || (i == ba && j < bb)) {
        ba = i;
        bb = j;
      }
    });
  }
  *oa = ba;
  *ob = bb;
  return GHX_OK;
}

int ghx_plan_build_fill_boundary(int64_t nboxes, const int64_t *boxes, const int64_t ngrow[3],
                                 const int32_t periodic[3], const int64_t period[3],
                                 const int32_t *rank_of, int32_t nranks, ghx_plan **out) {
  if (!out || nboxes < 0 || nboxes > INT32_MAX || (nboxes && (!boxes || !rank_of)) || !ngrow ||
      !periodic || !period || nranks < 1) {
    set_error("ghx_plan_build_fill_boundary: bad arguments");
    return GHX_EINVAL;
  }
  for (int d = 0; d < 3; ++d)
    if (periodic[d] && period[d] < 1) {
      set_error("ghx_plan_build_fill_boundary: period must be >= 1 on periodic axes");
      return GHX_EINVAL;
    }
  if (!check_ranks(rank_of, nboxes, nranks)) {
    set_error("ghx_plan_build_fill_boundary: rank id out of range");
    return GHX_EINVAL;
  }
  try {
    ghx_plan *p = new ghx_plan();
    p->mode = GHX_MODE_FILL_BOUNDARY;
    p->nranks = nranks;
    p->nsrc = p->ndst = (int32_t)nboxes;
    std::vector<Box> valid(nboxes), tgt(nboxes);
    for (int64_t i = 0; i < nboxes; ++i) {
      valid[i] = box_from(boxes + 6 * i);
      tgt[i] = valid[i];
      if (!valid[i].empty())
        for (int d = 0; d < 3; ++d) {
          tgt[i].lo[d] -= ngrow[d];
          tgt[i].hi[d] += ngrow[d];
        }
    }
    std::vector<Piece> pieces;
    build_pieces(tgt, &valid, valid, periodic, period, pieces);
    finish_plan(p, pieces, rank_of, rank_of);
    p->vbox = valid;
    for (int d = 0; d < 3; ++d) p->ngrow[d] = ngrow[d];
    *out = p;
    return GHX_OK;
  } catch (const std::bad_alloc &) {
    set_error("ghx_plan_build_fill_boundary: out of memory");
    return GHX_ENOMEM;
  }
}

int ghx_plan_build_parallel_copy(int64_t ndst, const int64_t *dst_boxes, const int64_t ngrow_dst[3],
                                 int64_t nsrc, const int64_t *src_boxes, const int64_t ngrow_src[3],
                                 const int32_t *periodic, const int64_t period[3],
                                 const int32_t *src_rank, const int32_t *dst_rank, int32_t nranks,
                                 ghx_plan **out) {
  if (!out || ndst < 0 || nsrc < 0 || ndst > INT32_MAX || nsrc > INT32_MAX ||
      (ndst && (!dst_boxes || !dst_rank)) || (nsrc && (!src_boxes || !src_rank)) || !ngrow_dst ||
      !ngrow_src || (periodic && !period) || nranks < 1) {
    set_error("ghx_plan_build_parallel_copy: bad arguments");
    return GHX_EINVAL;
  }
  if (periodic)
    for (int d = 0; d < 3; ++d)
      if (periodic[d] && period[d] < 1) {
        set_error("ghx_plan_build_parallel_copy: period must be >= 1 on periodic axes");
        return GHX_EINVAL;
      }
  if (!check_ranks(src_rank, nsrc, nranks) || !check_ranks(dst_rank, ndst, nranks)) {
    set_error("ghx_plan_build_parallel_copy: rank id out of range");
    return GHX_EINVAL;
  }
  try {
    ghx_plan *p = new ghx_plan();
    p->mode = GHX_MODE_PARALLEL_COPY;
    p->nranks = nranks;
    p->nsrc = (int32_t)nsrc;
    p->ndst = (int32_t)ndst;
    std::vector<Box> tgt(ndst), src(nsrc);
    for (int64_t i = 0; i < ndst; ++i) {
      tgt[i] = box_from(dst_boxes + 6 * i);
      if (!tgt[i].empty())
        for (int d = 0; d < 3; ++d) {
          tgt[i].lo[d] -= ngrow_dst[d];
          tgt[i].hi[d] += ngrow_dst[d];
        }
    }
    for (int64_t i = 0; i < nsrc; ++i) {
      src[i] = box_from(src_boxes + 6 * i);
      if (!src[i].empty())
        for (int d = 0; d < 3; ++d) {
          src[i].lo[d] -= ngrow_src[d];
          src[i].hi[d] += ngrow_src[d];
        }
    }
    std::vector<Piece> pieces;
    build_pieces(tgt, nullptr, src, periodic, period, pieces);
    finish_plan(p, pieces, src_rank, dst_rank);
    *out = p;
    return GHX_OK;
  } catch (const std::bad_alloc &) {
    set_error("ghx_plan_build_parallel_copy: out of memory");
    return GHX_ENOMEM;
  }
}

void ghx_plan_free(ghx_plan *plan) { delete plan; }

int64_t ghx_plan_num_segments(const ghx_plan *plan) { return plan ? (int64_t)plan->segs.size() : -1; }
int64_t ghx_plan_num_write_tags(const ghx_plan *plan) {
  return plan ? (int64_t)plan->wtags.size() : -1;
}

int ghx_plan_get_segments(const ghx_plan *plan, int64_t *rows) {
  if (!plan || (!rows && !plan->segs.empty())) {
    set_error("ghx_plan_get_segments: bad arguments");
    return GHX_EINVAL;
  }
  int64_t *r = rows;
  for (const Piece &pc : plan->segs) {
    r[0] = pc.src;
    r[1] = pc.dst;
    for (int d = 0; d < 3; ++d) {
      r[2 + d] = pc.dbox.lo[d];
      r[5 + d] = pc.dbox.hi[d];
      r[8 + d] = pc.shift[d];
    }
    r[11] = pc.srank;
    r[12] = pc.drank;
    r += 13;
  }
  return GHX_OK;
}

int ghx_plan_pair_cells(const ghx_plan *plan, int64_t *out) {
  if (!plan || !out) {
    set_error("ghx_plan_pair_cells: bad arguments");
    return GHX_EINVAL;
  }
  const int64_t n = plan->nranks;
  std::memset(out, 0, sizeof(int64_t) * n * n);
  for (const Piece &pc : plan->segs) out[pc.srank * n + pc.drank] += pc.dbox.cells();
  return GHX_OK;
}

}  // extern "C"
