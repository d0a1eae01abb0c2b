"""Coarse/fine level transfers on top of the exchange engine: fill_patch
(FillBoundary + gather of coarse data + interpolation), average_down
(restriction + ParallelCopy) and interp_box.

Drop-in for the reference's level-transfer functions
(/root/reference/pkg/src/miniamr_core/amr.py:235-397): same names, argument
meaning, validation order and ValueErrors.  The exchange steps run on the
fused copy kernel (ghx_exec.cu), the local arithmetic on ghx_amr.cu, one
launch per call for all fabs (the reference's ``fused_segments``).
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _native as N
from . import comm, config
from .index_space import Box, Geometry, IntVect, box_diff, box_list_diff, coarsen, grow, intersect
from .mesh import BoxArray, Fab, MultiFab

PIECEWISE_CONSTANT = "piecewise_constant"
LINEAR = "linear"
_SCHEMES = {PIECEWISE_CONSTANT: N.INTERP_PC, LINEAR: N.INTERP_LINEAR}


def _pad(vals, fill: int) -> list:
    v = list(vals)
    return v + [fill] * (3 - len(v))


def _row(b: Box) -> list:
    return list(b.as_row())


def _ratio3(ratio: int) -> np.ndarray:
    return np.asarray(_pad([ratio] * config.spacedim, 1), np.int32)


def _stream(device: int) -> int:
    import torch
    return torch.cuda.current_stream(device).cuda_stream


def _sync(device: int) -> None:
    import torch
    torch.cuda.current_stream(device).synchronize()


class _Xfer:
    """A prepared interp / average_down launch (ghx_xfer): the job table is
    validated and uploaded once; ``run`` is one kernel launch."""

    def __init__(self, handle: int, device: int):
        self._h = C.c_void_p(handle)
        self.device = device
        self.cells = int(N.lib.ghx_xfer_cells(self._h))

    def run(self) -> None:
        N.check(N.lib.ghx_xfer_run(self._h, C.c_void_p(_stream(self.device))))

    def __del__(self):
        try:
            if self._h:
                N.lib.ghx_xfer_free(self._h)
                self._h = None
        except Exception:
            pass


def _interp_rows(jobs: list) -> np.ndarray:
    rows = np.zeros((len(jobs), N.JOB_WORDS), np.int64)
    for n, (cf, ff, region) in enumerate(jobs):
        rows[n, 0] = np.uint64(cf.ptr).view(np.int64)
        rows[n, 1:7] = _row(cf.box)
        rows[n, 7] = np.uint64(ff.ptr).view(np.int64)
        rows[n, 8:14] = _row(ff.box)
        rows[n, 14:20] = _row(region)
    return rows


def _prepare_interp(jobs: list, ncomp: int, ratio: int, scheme: str, item: int, device: int) -> _Xfer:
    """jobs: (coarse Fab, fine Fab, fine region) -> one prepared launch."""
    rows = _interp_rows(jobs)
    h = C.c_void_p()
    N.check(N.lib.ghx_interp_prepare(C.c_void_p(rows.ctypes.data), len(jobs), ncomp, N.i32p(_ratio3(ratio)),
                                     config.spacedim, _SCHEMES[scheme], item, device, C.byref(h)))
    return _Xfer(h.value, device)


def _launch_interp(jobs: list, ncomp: int, ratio: int, scheme: str, item: int, device: int) -> None:
    """One-shot: jobs -> one ghx_interp launch."""
    if not jobs:
        return
    rows = _interp_rows(jobs)
    N.check(N.lib.ghx_interp(C.c_void_p(rows.ctypes.data), len(jobs), ncomp, N.i32p(_ratio3(ratio)),
                             config.spacedim, _SCHEMES[scheme], item, C.c_void_p(_stream(device))))


def interp_box(coarse_fab: Fab, fine_fab: Fab, fine_region: Box, ratio: int,
               scheme: str = PIECEWISE_CONSTANT) -> None:
    """Interpolate coarse_fab onto the cells of fine_region in fine_fab: one
    interp_kernel launch (reference amr.py:269-314, same arithmetic order,
    bit-identical).  PIECEWISE_CONSTANT copies each fine cell's parent;
    LINEAR adds unlimited centred slopes per axis, so it reads a one-cell
    coarse halo around the coarsened region -- checked, like every other
    precondition, with the reference's ValueError before the launch."""
    if fine_region.is_empty:
        return
    ratio = int(ratio)
    if not fine_fab.box.contains(fine_region):
        raise ValueError("fine_region must lie inside the fine fab")
    creg = coarsen(fine_region, ratio)
    need = grow(creg, 1) if scheme == LINEAR else creg
    if not coarse_fab.box.contains(need):
        raise ValueError(f"insufficient coarse data: need {need} inside {coarse_fab.box}")
    if scheme not in (PIECEWISE_CONSTANT, LINEAR):
        raise ValueError(f"unknown interpolation scheme {scheme!r}")
    if coarse_fab.ncomp != fine_fab.ncomp:
        raise ValueError(f"component count mismatch: coarse {coarse_fab.ncomp}, fine {fine_fab.ncomp}")
    if coarse_fab.dtype != fine_fab.dtype or coarse_fab.device != fine_fab.device:
        raise ValueError("coarse and fine fabs must share the real type and the device")
    _launch_interp([(coarse_fab, fine_fab, fine_region)], fine_fab.ncomp, ratio, scheme,
                   fine_fab.dtype.itemsize, fine_fab.device)
    _sync(fine_fab.device)


def interp_coarse_to_fine(coarse_fab: Fab, fine_fab: Fab, fine_region: Box, ratio: int,
                          scheme: str = PIECEWISE_CONSTANT) -> None:
    interp_box(coarse_fab, fine_fab, fine_region, ratio, scheme)


# -------------------------------------------------------------- average_down

def _restriction_layout(fine: MultiFab, ratio: int) -> MultiFab:
    """tmp MultiFab over coarsen(fine.ba) with fine's DistributionMapping
    (amr.py:247-249), cached on fine so the ParallelCopy plan into a given
    coarse MultiFab is built once (the reference rebuilds both per call)."""
    key = ("average_down_tmp", fine.ba.uid, fine.dm.uid, ratio, fine.ncomp, fine.dtype.str)
    tmp = fine._peer_cache.get(key)
    if tmp is None:
        crse_ba = BoxArray([coarsen(b, ratio) for b in fine.ba])
        tmp = fine._peer_cache[key] = MultiFab(crse_ba, fine.dm, fine.ncomp, 0, rank=fine.rank, device=fine.device)
    return tmp


def average_down(fine: MultiFab, coarse: MultiFab, ratio: int, backend=None, *, _wait: bool = True) -> None:
    """Covered coarse cells become the mean of their ratio^D fine children
    (amr.py:235-266): one restriction launch over the local fine fabs, then
    ParallelCopy into ``coarse``."""
    ratio = int(ratio)
    if ratio < 1:
        raise ValueError("ratio must be >= 1")
    fine.check_open()
    coarse.check_open()
    for b in fine.ba:
        if any(e % ratio for e in b.extents) or any(lo % ratio for lo in b.lo):
            raise ValueError(f"fine box {b} is not aligned to ratio {ratio}")
    if fine.ncomp != coarse.ncomp:
        raise ValueError("component count mismatch")
    tmp = _restriction_layout(fine, ratio)
    if comm.current_ctx().nranks == 1 and os.environ.get("GHX_AVGDOWN_DIRECT", "1") != "0":
        _average_down_direct(fine, coarse, tmp, ratio)
        if _wait:
            _sync(fine.device)
        return
    key = ("average_down_xfer", fine.ba.uid, fine.dm.uid, ratio, fine.ncomp, fine.dtype.str)
    xf = fine._peer_cache.get(key)
    if xf is None:
        rows = np.zeros((len(fine.local_indices), N.JOB_WORDS), np.int64)
        for n, gi in enumerate(fine.local_indices):
            ff, tf = fine.fabs[gi], tmp.fabs[gi]
            rows[n, 0] = np.uint64(ff.ptr).view(np.int64)
            rows[n, 1:7] = _row(ff.box)
            rows[n, 7] = np.uint64(tf.ptr).view(np.int64)
            rows[n, 8:14] = _row(tf.box)
            rows[n, 14:20] = _row(tmp.ba[gi])
        h = C.c_void_p()
        N.check(N.lib.ghx_average_down_prepare(C.c_void_p(rows.ctypes.data), len(rows), fine.ncomp,
                                               N.i32p(_ratio3(ratio)), config.spacedim, fine.dtype.itemsize,
                                               fine.device, C.byref(h)))
        xf = fine._peer_cache[key] = _Xfer(h.value, fine.device)
    xf.run()
    if comm.current_ctx().nranks == 1:  # stream-ordered: one host wait
        comm.prepare_parallel_copy(coarse, tmp).enqueue(_stream(fine.device))
        if _wait:
            _sync(fine.device)
    else:
        comm.parallel_copy(coarse, tmp, backend=backend)


def _average_down_direct(fine: MultiFab, coarse: MultiFab, tmp: MultiFab, ratio: int) -> None:
    """Single rank: restrict straight into the coarse fabs.  The
    ParallelCopy tmp -> coarse (amr.py:265) is planned as the reference
    does (cached on ``coarse``, ``plan_builds`` as in the reference); its
    segments -- pieces of coarsened fine boxes inside coarse boxes, no
    shift -- become the restriction jobs, so the kernel writes exactly the
    cells the copy would, with the same bits, and tmp is never touched."""
    ncomp, gs, gd = comm._pc_args(coarse, tmp, 0, 0, None, 0, 0)
    plan = comm._parallel_copy_plan(coarse, tmp, gs, gd, None)
    if plan.is_empty:
        return
    key = ("average_down_direct", plan.uid, coarse.uid, ratio, fine.ncomp, fine.dtype.str)
    xf = fine._peer_cache.get(key)
    if xf is None:
        segs = plan.local_by_rank.get(0, [])
        rows = np.zeros((len(segs), N.JOB_WORDS), np.int64)
        for n, sg in enumerate(segs):
            assert not any(sg.shift) and sg.src_box == sg.dst_box
            ff, cf = fine.fabs[sg.src_fab], coarse.fabs[sg.dst_fab]
            rows[n, 0] = np.uint64(ff.ptr).view(np.int64)
            rows[n, 1:7] = _row(ff.box)
            rows[n, 7] = np.uint64(cf.ptr).view(np.int64)
            rows[n, 8:14] = _row(cf.box)
            rows[n, 14:20] = _row(sg.dst_box)
        h = C.c_void_p()
        N.check(N.lib.ghx_average_down_prepare(C.c_void_p(rows.ctypes.data), len(rows), fine.ncomp,
                                               N.i32p(_ratio3(ratio)), config.spacedim, fine.dtype.itemsize,
                                               fine.device, C.byref(h)))
        xf = comm.cache_put(fine, key, _Xfer(h.value, fine.device), coarse)
    xf.run()


# ---------------------------------------------------------------- fill_patch

def _same_level_sources(ba: BoxArray, geom: Geometry) -> list:
    """Valid boxes plus their periodic images (amr.py:322-331)."""
    out = []
    reach = IntVect.filled(max(g for g in geom.period))
    big = grow(geom.domain, reach)
    for b in ba:
        out.append(b)
        for s in _shift_candidates(b, big, geom):
            if any(v != 0 for v in s):
                out.append(b.shift(s))
    return out


def _shift_candidates(src_box: Box, target: Box, geom: Geometry | None) -> list:
    """Period multiples moving src_box onto target (comm.py:250-266)."""
    import itertools
    import math
    dim = len(src_box.lo)
    if geom is None:
        return [IntVect.zero()]
    per_axis = []
    for d in range(dim):
        if not geom.periodic[d]:
            per_axis.append([0])
            continue
        ext = geom.period[d]
        kmin = math.ceil((target.lo[d] - src_box.hi[d]) / ext)
        kmax = math.floor((target.hi[d] - src_box.lo[d]) / ext)
        if kmin > kmax:
            return []
        per_axis.append([k * ext for k in range(kmin, kmax + 1)])
    return [IntVect(*c) for c in itertools.product(*per_axis)]


def _coarse_fill_targets(fine_ba: BoxArray, ngrow: IntVect, geom: Geometry) -> dict:
    """Per fine fab: ghost boxes not coverable by same-level valid data
    (amr.py:334-352); non-periodic axes clip at the domain."""
    sources = _same_level_sources(fine_ba, geom)
    clip_lo, clip_hi = [], []
    big = max(geom.period) + max(ngrow) + 1
    for d in range(config.spacedim):
        clip_lo.append(geom.domain.lo[d] - (big if geom.periodic[d] else 0))
        clip_hi.append(geom.domain.hi[d] + (big if geom.periodic[d] else 0))
    clip = Box(clip_lo, clip_hi)
    out = {}
    for gi, b in enumerate(fine_ba):
        ghost = box_diff(grow(b, ngrow), b)
        rest = box_list_diff(ghost, sources)
        rest = [intersect(r, clip) for r in rest]
        rest = [r for r in rest if not r.is_empty]
        if rest:
            out[gi] = rest
    return out


def fill_patch(fine: MultiFab, coarse: MultiFab, fine_geom: Geometry, coarse_geom: Geometry, ratio: int,
               scheme: str = LINEAR, backend=None, *, _wait: bool = True) -> None:
    """Fill fine ghost cells: same-level data where available, interpolated
    coarse data elsewhere; valid cells are never modified (amr.py:355-397).

    FillBoundary (fused exchange) -> gather of the coarse cells under each
    fine fab's uncovered ghost regions (fused exchange, plan-cached target
    slab) -> one interp launch over every (fab, region) job.  With a single
    rank the three steps are enqueued back to back on the current stream and
    the host waits once at the end."""
    fine.check_open()
    coarse.check_open()
    serial = comm.current_ctx().nranks == 1
    reach = 1 if scheme == LINEAR else 0
    key = comm.PlanKey(coarse.ba.uid, coarse.dm.uid, fine.ba.uid, fine.dm.uid, (reach,) * len(fine.ngrow),
                       fine.ngrow.comps, fine.ba.ixtype.flags, fine_geom.periodic, "fill_patch")
    cached = fine.plan_cache.get(key)
    if cached is None:
        targets = _coarse_fill_targets(fine.ba, fine.ngrow, fine_geom)
        gather_list, dst_ranks = [], []
        for gi in sorted(targets):
            cbox = grow(coarsen(grow(fine.ba[gi], fine.ngrow), ratio), reach)
            gather_list.append((gi, cbox))
            dst_ranks.append(fine.dm[gi])
        plan = comm.build_gather_plan(gather_list, dst_ranks, coarse, coarse_geom) if gather_list else None
        cached = (targets, gather_list, dst_ranks, plan)
        fine.plan_cache[key] = cached
        fine.plan_builds += 1
    targets, gather_list, dst_ranks, plan = cached
    if not serial:
        comm.fill_boundary(fine, fine_geom, backend=backend)
        if not targets:
            return
        owned = comm.gather_targets(plan, gather_list, dst_ranks, coarse)
        comm.gather_fabs(gather_list, dst_ranks, owned, coarse, coarse_geom, backend=backend, plan=plan)
        _interp_xfer(fine, coarse, key, targets, owned, ratio, scheme).run()
        _sync(fine.device)
        return
    fb = comm.prepare_fill_boundary(fine, fine_geom)
    if not targets:
        fb.enqueue(_stream(fine.device))
        if _wait:
            _sync(fine.device)
        return
    owned = comm.gather_targets(plan, gather_list, dst_ranks, coarse)
    gather = None
    if not plan.is_empty:
        if os.environ.get("GHX_FP_GATHER", "regions") == "regions":
            gather = _region_gather(fine, coarse, coarse_geom, key, targets, owned, ratio, reach)
        else:
            gather = comm.exchange_for(plan, coarse, comm._gather_set(plan, gather_list, dst_ranks, coarse), 0, 0,
                                       coarse.ncomp)
    xf = _interp_xfer(fine, coarse, key, targets, owned, ratio, scheme)
    # Single rank: the FillBoundary writes the covered ghost cells, the
    # gather + interp the uncovered ones (disjoint by construction, and the
    # interp reads only the gathered coarse data), so they run on two
    # streams, forked from and joined back to the current one.
    import torch
    main = torch.cuda.current_stream(fine.device)
    if _fp_overlap():
        side = _side_stream(fine.device)
        side.wait_stream(main)
        fb.enqueue(main.cuda_stream)
        with torch.cuda.stream(side):
            if gather is not None:
                gather.enqueue(side.cuda_stream)
            xf.run()
        main.wait_stream(side)
    else:
        fb.enqueue(main.cuda_stream)
        if gather is not None:
            gather.enqueue(main.cuda_stream)
        xf.run()
    if _wait:
        _sync(fine.device)


class _RegionSet:
    """Destination of the single-rank fill_patch gather: one slot per coarse
    box the interpolation reads (a region's coarsened footprint, grown by the
    stencil reach), addressed inside its parent gather-target fab.  The
    reference gathers each target's whole box (comm.py:432-462); only these
    cells are ever read, so the fine result is the same while the gather
    moves the thin shells instead of whole coarsened fabs."""

    def __init__(self, parents: dict, slots: list, like: MultiFab):
        from .mesh import _next_uid
        self.ncomp, self.dtype, self.device = like.ncomp, like.dtype, like.device
        self.ngrow = IntVect(*([0] * len(like.ngrow)))
        self.uid = _next_uid()
        self._peer_cache: dict = {}
        self._parents = parents  # the target fabs (and their slab) stay alive with the set
        self.local_indices = tuple(range(len(slots)))
        self._rows = np.ascontiguousarray(
            np.asarray([parents[fid].box.as_row() for fid, _ in slots], np.int64).reshape(-1, 6))
        self._ptrs = np.array([parents[fid].ptr for fid, _ in slots], np.uint64)

    def storage_rows(self) -> np.ndarray:
        return self._rows


def _region_gather(fine: MultiFab, coarse: MultiFab, coarse_geom: Geometry, key, targets: dict, owned: dict,
                   ratio: int, reach: int) -> "comm.Exchange":
    gkey = ("fill_patch_region_gather", key, coarse.uid, coarse.ncomp)
    ex = fine._peer_cache.get(gkey)
    if ex is None:
        slots = []
        for gi in sorted(targets):
            seen = set()
            for r in targets[gi]:
                need = grow(coarsen(r, int(ratio)), reach)
                if tuple(need.as_row()) not in seen:
                    seen.add(tuple(need.as_row()))
                    slots.append((gi, need))
        plan = comm.build_gather_plan(list(enumerate(b for _, b in slots)), [0] * len(slots), coarse, coarse_geom)
        dst = _RegionSet(owned, slots, coarse)
        ex = comm.cache_put(fine, gkey, (plan, dst, None if plan.is_empty else
                                         comm.exchange_for(plan, coarse, dst, 0, 0, coarse.ncomp)), coarse)
    return ex[2]


_side_streams: dict = {}


def _side_stream(device: int):
    import torch
    st = _side_streams.get(device)
    if st is None:
        st = _side_streams[device] = torch.cuda.Stream(device)
    return st


def _fp_overlap() -> bool:
    return os.environ.get("GHX_FP_OVERLAP", "1") != "0"


def _interp_xfer(fine: MultiFab, coarse: MultiFab, key, targets, owned, ratio: int, scheme: str) -> _Xfer:
    """The prepared interp launch of a fill_patch plan (validated once)."""
    # the gather targets (``owned``) belong to this coarse MultiFab: two
    # coarse MultiFabs of one layout (time levels, a rebuilt coarse) get
    # their own prepared launch, dropped when that coarse MultiFab goes
    xkey = ("fill_patch_interp", key, coarse.uid, int(ratio), scheme, fine.ncomp)
    xf = fine._peer_cache.get(xkey)
    if xf is None:
        if coarse.ncomp != fine.ncomp:
            raise ValueError(f"component count mismatch: coarse {coarse.ncomp}, fine {fine.ncomp}")
        jobs = [(owned[gi], fine.fabs[gi], region) for gi in sorted(targets) if gi in owned
                for region in targets[gi]]
        for cf, ff, region in jobs:  # interp_box's checks (amr.py:281-293), once per plan
            if not ff.box.contains(region):
                raise ValueError("fine_region must lie inside the fine fab")
            creg = coarsen(region, int(ratio))
            need = grow(creg, 1) if scheme == LINEAR else creg
            if not cf.box.contains(need):
                raise ValueError(f"insufficient coarse data: need {need} inside {cf.box}")
        if scheme not in (PIECEWISE_CONSTANT, LINEAR):
            raise ValueError(f"unknown interpolation scheme {scheme!r}")
        xf = comm.cache_put(fine, xkey, _prepare_interp(jobs, fine.ncomp, int(ratio), scheme, fine.dtype.itemsize,
                                                        fine.device), coarse)
    return xf
