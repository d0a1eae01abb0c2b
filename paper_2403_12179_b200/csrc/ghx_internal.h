// Internal declarations shared by the plan builder (host C++) and the
// executor (CUDA).  Not part of the C ABI.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "ghostx.h"

namespace ghx {

struct Box {
  int64_t lo[3];
  int64_t hi[3];
  bool empty() const { return hi[0] < lo[0] || hi[1] < lo[1] || hi[2] < lo[2]; }
  int64_t cells() const {
    if (empty()) return 0;
    return (hi[0] - lo[0] + 1) * (hi[1] - lo[1] + 1) * (hi[2] - lo[2] + 1);
  }
};

inline Box box_from(const int64_t *p) {
  Box b;
  for (int d = 0; d < 3; ++d) {
    b.lo[d] = p[d];
    b.hi[d] = p[3 + d];
  }
  return b;
}

inline bool overlap(const Box &a, const Box &b) {
  for (int d = 0; d < 3; ++d)
    if (a.lo[d] > b.hi[d] || b.lo[d] > a.hi[d]) return false;
  return true;
}

inline Box meet(const Box &a, const Box &b) {
  Box r;
  for (int d = 0; d < 3; ++d) {
    r.lo[d] = a.lo[d] > b.lo[d] ? a.lo[d] : b.lo[d];
    r.hi[d] = a.hi[d] < b.hi[d] ? a.hi[d] : b.hi[d];
  }
  return r;
}

// One copy piece: dst cells `dbox` of dst fab `dst` receive src fab `src`
// cells `dbox - shift`.
struct Piece {
  int32_t src, dst;
  int32_t srank, drank;
  Box dbox;
  int64_t shift[3];
};

}  // namespace ghx

struct ghx_plan {
  int32_t mode = 0;
  int32_t nranks = 1;
  int32_t nsrc = 0, ndst = 0;
  std::vector<ghx::Piece> segs;   // reference segments, CommPlan order
  std::vector<ghx::Piece> wtags;  // disjoint write tags (last writer wins)
  bool clipped = false;            // some destinations overlapped (wtags != segs)
  // FillBoundary: the valid boxes and ghost widths the plan was built for
  std::vector<ghx::Box> vbox;
  int64_t ngrow[3] = {0, 0, 0};
};

namespace ghx {
void set_error(const std::string &msg);
int64_t sync_timeouts();  // ghx_exec.cu: in-kernel READY/DONE waits that gave up
}
