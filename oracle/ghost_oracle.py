"""CPU ORACLE (test infrastructure only) for the FillBoundary / ParallelCopy path.

This module is the checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product path
(``paper_2403_12179_b200``) never imports it and fails loudly when its CUDA
library is missing.

It restates, in numpy, the reference algorithm of
``/root/reference/pkg/src/miniamr_core/comm.py`` (the "reference" below):

* ``shift_ranges``       <- ``_shift_candidates``        comm.py:250-266
* ``box_diff``           <- ``box_diff``                  index_space.py:297-320
* ``build_segments``     <- ``_build_copy_segments``      comm.py:269-286
* ``OraclePlan``         <- ``CommPlan`` sort + split      comm.py:218-247
* ``plan_fill_boundary`` <- ``plan_build_fill_boundary``  comm.py:289-309
* ``plan_parallel_copy`` <- ``parallel_copy`` plan part   comm.py:413-424
* ``execute``            <- ``_execute_plan``             comm.py:316-380
  (local fused copy, then one packed F-order message per ordered rank pair,
  unpacked on the receiver in ascending peer order)

Parity pinning: ``tests/golden/make_golden.py`` runs the reference itself on
identical inputs and stores plans / fab contents / message stats under
``tests/golden/``; ``tests/test_oracle_golden.py`` checks this module against
every fixture plus the reference's own known-answer tests
(tests/test_comm.py:168-223 in the reference).

Conventions: boxes are int64 arrays ``[lo0, lo1, lo2, hi0, hi1, hi2]`` padded
to three axes (lo 0 / hi 0 on unused axes, core/mesh.py:31-40); a segment row
is ``[src_fab, dst_fab, dlo0, dlo1, dlo2, dhi0, dhi1, dhi2, s0, s1, s2]`` with
``src_box = dst_box - shift``.  Fab storage is F-order ``(nx, ny, nz, ncomp)``
over the grown box (core/mesh.py:38-58).
"""

from __future__ import annotations

import itertools
import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

SEG_COLS = 11


def _empty(b) -> bool:
    return bool(np.any(b[3:] < b[:3]))


def box_diff(a, b):
    """a minus b as disjoint boxes, axis by axis (index_space.py:297-320)."""
    if _empty(a):
        return []
    lo = np.maximum(a[:3], b[:3])
    hi = np.minimum(a[3:], b[3:])
    if np.any(hi < lo):
        return [a.copy()]
    out = []
    rem = a.copy()
    for d in range(3):
        if rem[d] < lo[d]:
            p = rem.copy()
            p[3 + d] = lo[d] - 1
            out.append(p)
        if rem[3 + d] > hi[d]:
            p = rem.copy()
            p[d] = hi[d] + 1
            out.append(p)
        rem[d] = lo[d]
        rem[3 + d] = hi[d]
    return out


def shift_ranges(src, tgt, periodic, period):
    """Per-axis k ranges of periodic images of ``src`` that can meet ``tgt``
    (comm.py:250-266).  ``src`` is (n, 6); returns kmin, kmax as (n, 3).
    ``periodic is None`` means "no geometry": only the zero shift."""
    n = src.shape[0]
    kmin = np.zeros((n, 3), np.int64)
    kmax = np.zeros((n, 3), np.int64)
    for d in range(3):
        if periodic is None or not periodic[d]:
            # only k = 0; mark the axis empty when the boxes cannot meet (the
            # reference finds the same pairs through its intersect() test)
            miss = (src[:, d] > tgt[3 + d]) | (src[:, 3 + d] < tgt[d])
            kmin[miss, d] = 1
            continue
        p = int(period[d])
        # ceil((t.lo - s.hi)/p) and floor((t.hi - s.lo)/p), exact integer math
        kmin[:, d] = -((src[:, 3 + d] - tgt[d]) // p)
        kmax[:, d] = (tgt[3 + d] - src[:, d]) // p
    return kmin, kmax


def build_segments(dst_targets, dst_valids, srcs, periodic, period, exclude_valid):
    """Every (dst, src, shift) overlap, cut by box_diff against the dst valid
    box for FillBoundary (comm.py:269-286).  Brute force over all src boxes
    per dst box, vectorised with numpy (the reference loops in Python)."""
    dst_targets = np.asarray(dst_targets, np.int64).reshape(-1, 6)
    srcs = np.asarray(srcs, np.int64).reshape(-1, 6)
    rows = []
    for dj in range(dst_targets.shape[0]):
        t = dst_targets[dj]
        if _empty(t):
            continue
        kmin, kmax = shift_ranges(srcs, t, periodic, period)
        ok = np.all(kmin <= kmax, axis=1)
        for si in np.nonzero(ok)[0]:
            ranges = [range(int(kmin[si, d]), int(kmax[si, d]) + 1) for d in range(3)]
            for ks in itertools.product(*ranges):
                s = np.array([ks[d] * (int(period[d]) if periodic is not None else 0)
                              for d in range(3)], np.int64)
                if exclude_valid and si == dj and not s.any():
                    continue
                lo = np.maximum(t[:3], srcs[si, :3] + s)
                hi = np.minimum(t[3:], srcs[si, 3:] + s)
                if np.any(hi < lo):
                    continue
                region = np.concatenate([lo, hi])
                parts = box_diff(region, dst_valids[dj]) if exclude_valid else [region]
                for p in parts:
                    rows.append(np.concatenate([[si, dj], p, s]))
    if not rows:
        return np.zeros((0, SEG_COLS), np.int64)
    return np.asarray(rows, np.int64)


def sort_segments(segs):
    """Sort key (dst_fab, dst_box.lo, src_fab, shift) as in comm.py:224-227."""
    if segs.shape[0] == 0:
        return segs
    keys = (segs[:, 10], segs[:, 9], segs[:, 8], segs[:, 0],
            segs[:, 4], segs[:, 3], segs[:, 2], segs[:, 1])
    return segs[np.lexsort(keys)]


class OraclePlan:
    """Sorted segments split into per-rank local lists and per-ordered-pair
    message lists (comm.py:221-237)."""

    def __init__(self, segs, src_ranks, dst_ranks, nranks):
        self.segments = sort_segments(np.asarray(segs, np.int64).reshape(-1, SEG_COLS))
        self.nranks = nranks
        src_ranks = np.asarray(src_ranks, np.int64)
        dst_ranks = np.asarray(dst_ranks, np.int64)
        self.local_by_rank = {}
        self.pair_segments = {}
        for row in self.segments:
            sr = int(src_ranks[row[0]])
            dr = int(dst_ranks[row[1]])
            if sr == dr:
                self.local_by_rank.setdefault(sr, []).append(row)
            else:
                self.pair_segments.setdefault((sr, dr), []).append(row)
        self.local_by_rank = {k: np.asarray(v) for k, v in self.local_by_rank.items()}
        self.pair_segments = {k: np.asarray(v) for k, v in sorted(self.pair_segments.items())}

    @property
    def num_segments(self):
        return int(self.segments.shape[0])


def grow_boxes(boxes, ngrow):
    b = np.asarray(boxes, np.int64).reshape(-1, 6).copy()
    g = np.asarray(ngrow, np.int64)
    b[:, :3] -= g
    b[:, 3:] += g
    return b


def pad_boxes(boxes, dim):
    """(n, 2*dim) lo/hi -> padded (n, 6)."""
    b = np.asarray(boxes, np.int64).reshape(-1, 2 * dim)
    out = np.zeros((b.shape[0], 6), np.int64)
    out[:, :dim] = b[:, :dim]
    out[:, 3:3 + dim] = b[:, dim:]
    return out


def pad_vec(v, dim, fill=0):
    out = [fill] * 3
    for d in range(dim):
        out[d] = int(v[d])
    return out


def plan_fill_boundary(valid_boxes, ngrow, periodic, period, rank_of, nranks):
    """plan_build_fill_boundary (comm.py:289-309) minus caching/validation.
    Boxes and vectors are already padded to 3 axes (unused: ngrow 0,
    periodic False)."""
    valid = np.asarray(valid_boxes, np.int64).reshape(-1, 6)
    targets = grow_boxes(valid, ngrow)
    segs = build_segments(targets, valid, valid, periodic, period, exclude_valid=True)
    return OraclePlan(segs, rank_of, rank_of, nranks)


def plan_parallel_copy(dst_boxes, src_boxes, ngrow_dst, ngrow_src, periodic, period,
                       src_rank_of, dst_rank_of, nranks):
    """parallel_copy plan (comm.py:413-424); ``periodic=None`` when no geom."""
    tgt = grow_boxes(dst_boxes, ngrow_dst)
    src = grow_boxes(src_boxes, ngrow_src)
    segs = build_segments(tgt, tgt, src, periodic, period, exclude_valid=False)
    return OraclePlan(segs, src_rank_of, dst_rank_of, nranks)


# ----------------------------------------------------------------- execution

def _slices(fab_lo, lo, hi):
    return tuple(slice(int(lo[d] - fab_lo[d]), int(hi[d] - fab_lo[d] + 1)) for d in range(3))


def _src_box(row):
    return row[2:5] - row[8:11], row[5:8] - row[8:11]


class _Pool:
    """fused_segments-style launcher: contiguous chunks over a thread pool
    (core/kernels.py:124-132, :280-297)."""

    def __init__(self, workers):
        self.workers = max(1, int(workers))
        self._pool = ThreadPoolExecutor(self.workers) if self.workers > 1 else None

    def run(self, n, fn):
        if n == 0:
            return
        if self._pool is None:
            for i in range(n):
                fn(i)
            return
        base, rem = divmod(n, self.workers)
        bounds = []
        s = 0
        for w in range(self.workers):
            e = s + base + (1 if w < rem else 0)
            bounds.append((s, e))
            s = e

        def chunk(b):
            for i in range(b[0], b[1]):
                fn(i)
        list(self._pool.map(chunk, bounds))

    def close(self):
        if self._pool is not None:
            self._pool.shutdown()


def execute(plan, src_fabs, src_lo, dst_fabs, dst_lo, scomp, dcomp, ncomp,
            workers=1, pool=None, ranks=None):
    """Run ``plan`` for every simulated rank (comm.py:316-380).

    ``src_fabs`` / ``dst_fabs`` map fab id -> ndarray (nx, ny, nz, nc) in
    F-order; ``src_lo`` / ``dst_lo`` map fab id -> storage-box lo (3,).
    Returns ``{(src_rank, dst_rank): (messages, bytes)}`` message stats.
    ``ranks`` restricts execution to those destination ranks."""
    own = pool is None
    pool = pool or _Pool(workers)
    stats = {}
    try:
        ssl = slice(scomp, scomp + ncomp)
        dsl = slice(dcomp, dcomp + ncomp)
        for r in sorted(plan.local_by_rank):
            if ranks is not None and r not in ranks:
                continue
            segs = plan.local_by_rank[r]

            def copy_local(n, segs=segs):
                row = segs[n]
                s_lo, s_hi = _src_box(row)
                si, dj = int(row[0]), int(row[1])
                dst_fabs[dj][_slices(dst_lo[dj], row[2:5], row[5:8]) + (dsl,)] = \
                    src_fabs[si][_slices(src_lo[si], s_lo, s_hi) + (ssl,)]
            pool.run(len(segs), copy_local)
        for (sr, dr), segs in plan.pair_segments.items():
            if ranks is not None and dr not in ranks:
                continue
            itemsize = next(iter(src_fabs.values())).dtype.itemsize
            cells = (segs[:, 5:8] - segs[:, 2:5] + 1).prod(axis=1)
            offs = np.concatenate([[0], np.cumsum(cells * ncomp)])
            buf = np.empty(int(offs[-1]), next(iter(src_fabs.values())).dtype)

            def pack(n, segs=segs, offs=offs, buf=buf):
                row = segs[n]
                s_lo, s_hi = _src_box(row)
                si = int(row[0])
                vals = src_fabs[si][_slices(src_lo[si], s_lo, s_hi) + (ssl,)]
                buf[offs[n]:offs[n + 1]] = vals.ravel(order="F")
            pool.run(len(segs), pack)
            st = stats.setdefault((sr, dr), [0, 0])
            st[0] += 1
            st[1] += buf.nbytes

            def unpack(n, segs=segs, offs=offs, buf=buf):
                row = segs[n]
                dj = int(row[1])
                sl = _slices(dst_lo[dj], row[2:5], row[5:8]) + (dsl,)
                shape = dst_fabs[dj][sl].shape
                dst_fabs[dj][sl] = buf[offs[n]:offs[n + 1]].reshape(shape, order="F")
            pool.run(len(segs), unpack)
    finally:
        if own:
            pool.close()
    return {k: tuple(v) for k, v in stats.items()}


def ghost_bytes(plan, ncomp, itemsize):
    """Total cells x ncomp x itemsize moved by the plan (local + remote)."""
    s = plan.segments
    if s.shape[0] == 0:
        return 0
    return int((s[:, 5:8] - s[:, 2:5] + 1).prod(axis=1).sum()) * ncomp * itemsize


def index_copy(dst_boxes, dst_fabs, dst_lo, src_boxes, src_fabs, src_lo, mapping_fn, region=None):
    """index_mapped_copy (comm.py:465-560): dst(cell) = src(mapping(cell)) over
    the dst valid cells (intersected with region), the first src valid box in
    order owning each mapped point; all components.  Boxes padded (n, 6)."""
    src_boxes = np.asarray(src_boxes, np.int64).reshape(-1, 6)
    for dj, db in enumerate(np.asarray(dst_boxes, np.int64).reshape(-1, 6)):
        w = db.copy()
        if region is not None:
            w = np.concatenate([np.maximum(db[:3], region[:3]), np.minimum(db[3:], region[3:])])
        if np.any(w[3:] < w[:3]):
            continue
        ex = w[3:] - w[:3] + 1
        flat = np.arange(int(np.prod(ex)), dtype=np.int64)
        di, dy, dk = flat % ex[0] + w[0], (flat // ex[0]) % ex[1] + w[1], flat // (ex[0] * ex[1]) + w[2]
        mi, mj, mk = (np.asarray(v, np.int64) for v in mapping_fn(di, dy, dk))
        owner = np.full(di.size, -1, np.int64)
        for si, sb in enumerate(src_boxes):
            m = ((mi >= sb[0]) & (mi <= sb[3]) & (mj >= sb[1]) & (mj <= sb[4]) & (mk >= sb[2]) & (mk <= sb[5])
                 & (owner < 0))
            owner[m] = si
        if (owner < 0).any():
            raise ValueError("mapping leaves cells outside src coverage")
        dl = dst_lo[dj]
        for si in np.unique(owner):
            m = owner == si
            sl = src_lo[int(si)]
            dst_fabs[dj][di[m] - dl[0], dy[m] - dl[1], dk[m] - dl[2], :] = \
                src_fabs[int(si)][mi[m] - sl[0], mj[m] - sl[1], mk[m] - sl[2], :]
