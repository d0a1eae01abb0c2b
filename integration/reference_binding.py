"""The reference-side binding a maintainer would add to miniamr_core
(INTEGRATION.md section 2), as runnable code: the reference's OWN MultiFab,
Fab and Geometry objects, its numpy fab arrays allocated from pinned,
mapped host memory, and the exchange done by libghostx.so through the
plain C ABI (ctypes, pointers and sizes only -- no torch, no
paper_2403_12179_b200 Python layer).

    from miniamr_core import mesh, comm
    from integration.reference_binding import PinnedArena, fill_boundary_native
    mf = mesh.MultiFab(ba, dm, ncomp, ngrow, geom, arena=PinnedArena())
    fill_boundary_native(mf, geom)        # instead of comm.fill_boundary(mf, geom)

The arena duck-types the reference's (arena.py:87-163: ``alloc(nbytes,
align)`` returning a block with ``as_array(dtype, count)`` / ``free()``),
so Fab (mesh.py:43-86) allocates its storage in memory the GPU kernel can
address directly (UVA: the host pointer is the device pointer).

Under the reference's ``runtime_spawn`` (rank threads, comm.py:143-180)
the same calls are collective, like the reference's: every rank runs its
share of the plan (the tags whose source fab it owns) as one launch that
writes its neighbours' ghost cells directly -- all fabs are pinned host
memory of one process -- between an entry barrier (no rank writes a
peer's ghost cells before the peer has entered the call) and the
reference's trailing barrier; one Bus message per ordered rank pair with
the pair's payload bytes keeps ``Bus.message_stats`` the reference's
(comm.py:356-357).
"""

from __future__ import annotations

import ctypes as C
import importlib
import os
import threading
import weakref

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.environ.get("GHX_LIB") or os.path.join(os.path.dirname(_HERE), "paper_2403_12179_b200", "_lib",
                                                       "libghostx.so")
_lib = None

P, I32, I64 = C.c_void_p, C.c_int32, C.c_int64
GHX_EXEC_DIRECT, GHX_EXEC_PHASED = 0, 0x100  # include/ghostx.h
PI64, PI32 = C.POINTER(C.c_int64), C.POINTER(C.c_int32)


def lib():
    """Load libghostx.so and declare the entry points this binding uses."""
    global _lib
    if _lib is None:
        L = C.CDLL(_LIB_PATH)
        L.ghx_last_error.restype = C.c_char_p
        L.ghx_host_alloc.argtypes = [C.c_size_t, C.POINTER(P)]
        L.ghx_host_free.argtypes = [P]
        L.ghx_plan_build_fill_boundary.argtypes = [I64, PI64, PI64, PI32, PI64, PI32, I32, C.POINTER(P)]
        L.ghx_plan_free.argtypes = [P]
        L.ghx_plan_free.restype = None
        L.ghx_exec_create.argtypes = [P, I32, I32, PI64, I32, PI64, I32, I32, I32, I32, I32, I32, C.POINTER(P)]
        L.ghx_exec_free.argtypes = [P]
        L.ghx_exec_free.restype = None
        L.ghx_exec_run.argtypes = [P, C.POINTER(P), I64, P]
        L.ghx_stream_sync.argtypes = [P]
        L.ghx_interp.argtypes = [P, I64, I32, PI32, I32, I32, I32, P]
        L.ghx_average_down.argtypes = [P, I64, I32, PI32, I32, I32, P]
        L.ghx_plan_build_parallel_copy.argtypes = [I64, PI64, PI64, I64, PI64, PI64, PI32, PI64, PI32, PI32, I32,
                                                   C.POINTER(P)]
        L.ghx_plan_num_segments.argtypes = [P]
        L.ghx_plan_num_segments.restype = I64
        L.ghx_plan_pair_cells.argtypes = [P, PI64]
        L.ghx_exec_set_ring.argtypes = [P, I32]
        L.ghx_exec_set_grid.argtypes = [P, I32, I32]
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc:
        msg = lib().ghx_last_error().decode()
        raise (ValueError if rc == 1 else RuntimeError)(msg)


# ------------------------------------------------------------------ arena

class _PinnedBlock:
    __slots__ = ("arena", "chunk", "ptr", "nbytes", "freed")

    def __init__(self, arena, chunk, ptr: int, nbytes: int):
        self.arena, self.chunk, self.ptr, self.nbytes, self.freed = arena, chunk, ptr, nbytes, False

    @property
    def is_null(self) -> bool:
        return self.ptr == 0

    @property
    def address(self) -> int:
        return self.ptr

    def as_array(self, dtype, count: int) -> np.ndarray:
        if self.is_null:
            return np.empty(0, dtype=dtype)
        raw = (C.c_uint8 * (np.dtype(dtype).itemsize * count)).from_address(self.ptr)
        return np.frombuffer(raw, dtype=dtype, count=count)

    def free(self) -> None:
        if not self.freed and self.chunk is not None:
            self.arena._release(self.chunk)
        self.freed = True


class _Chunk:
    __slots__ = ("base", "size", "top", "live")

    def __init__(self, base: int, size: int):
        self.base, self.size, self.top, self.live = base, size, 0, 0


class PinnedArena:
    """A reference-compatible arena whose blocks are pinned, mapped host
    memory (ghx_host_alloc): numpy sees ordinary arrays, the GPU the same
    addresses.  Blocks are cut from large pinned chunks (bump allocation;
    a chunk is returned when its last block is freed; chunks start at 256
    MiB and double up to 4 GiB): a MultiFab's fabs then sit side by side in
    few allocations, which the GPU reaches over PCIe faster than one
    allocation per fab (C3 FillBoundary through this binding: 54.7 ms with a
    pinned allocation per fab, 49.8-50.7 with these growing chunks, 2 GiB
    chunks or one slab; scripts/binding_e2e_probe.py,
    profiles/r02_binding_arena_probe.txt)."""

    FIRST, LAST = 1 << 28, 1 << 32

    def __init__(self, chunk_bytes: int | None = None):
        self.chunk_bytes = int(chunk_bytes) if chunk_bytes else None  # fixed chunk size, else growing
        self._next = self.FIRST
        self._cur = None
        self._lock = threading.Lock()  # rank threads may share one arena

    def alloc(self, nbytes: int, align: int = 256) -> _PinnedBlock:
        if nbytes == 0:
            return _PinnedBlock(self, None, 0, 0)
        with self._lock:
            return self._alloc(int(nbytes), max(int(align), 256))

    def _alloc(self, nbytes: int, align: int) -> _PinnedBlock:
        c = self._cur
        if c is not None:
            off = -(-c.top // align) * align
            if off + nbytes > c.size:
                c = None
        if c is None:
            step = self.chunk_bytes or self._next
            if not self.chunk_bytes:
                self._next = min(2 * self._next, self.LAST)
            size = max(step, -(-int(nbytes) // 4096) * 4096)
            p = P()
            _check(lib().ghx_host_alloc(size, C.byref(p)))  # cudaHostAlloc: page aligned
            c = self._cur = _Chunk(p.value, size)
            off = 0
        c.top = off + int(nbytes)
        c.live += 1
        return _PinnedBlock(self, c, c.base + off, nbytes)

    def _release(self, c: _Chunk) -> None:
        with self._lock:
            c.live -= 1
            if c.live:
                return
            if c is self._cur:
                self._cur = None
        lib().ghx_host_free(P(c.base))

    def free(self, block: _PinnedBlock) -> None:
        block.free()


# ---------------------------------------------------------------- helpers

def _rows(boxes, grow=(0, 0, 0)) -> np.ndarray:
    """Boxes -> int64[n, 6] rows (lo0 lo1 lo2 hi0 hi1 hi2), padded to 3-D."""
    out = np.zeros((len(boxes), 6), np.int64)
    for i, b in enumerate(boxes):
        d = len(b.lo)
        out[i, :d] = [v - grow[k] for k, v in enumerate(b.lo)]
        out[i, 3:3 + d] = [v + grow[k] for k, v in enumerate(b.hi)]
    return out


def _p64(a: np.ndarray):
    return a.ctypes.data_as(PI64)


def _p32(a: np.ndarray):
    return a.ctypes.data_as(PI32)


def _ctx_of(mf):
    """The reference's current rank context (``comm.current_ctx()`` of the
    package the MultiFab comes from)."""
    pkg = type(mf).__module__.rsplit(".", 1)[0]
    return importlib.import_module(pkg + ".comm").current_ctx()


def _allgather_addrs(ctx, local: dict) -> dict:
    """Every rank's {fab index: address}.  Rank threads share the process, so
    the addresses meet in a registry on the reference's Bus between two
    barriers -- no messages, the Bus statistics stay the reference's.  The
    n-th call on every rank uses slot n (collectives run in the same order
    on all ranks)."""
    if ctx.nranks == 1:
        return dict(local)
    reg = ctx.bus.__dict__.setdefault("_ghostx_addrs", {})
    seq = getattr(ctx, "_ghostx_seq", 0)
    ctx._ghostx_seq = seq + 1
    slot = reg.setdefault(seq, {})  # atomic for a dict under the GIL
    slot[ctx.rank] = dict(local)
    ctx.barrier()
    out = {}
    for part in slot.values():
        out.update(part)
    ctx.barrier()  # every rank has read the slot
    if ctx.rank == 0:
        reg.pop(seq, None)
    return out


def _addrs(mf) -> dict:
    return {i: fab.data.__array_interface__["data"][0] for i, fab in mf.fabs.items()}


class _Side:
    """One side of an exchange: the fabs' storage boxes (int64[n, 6]), their
    component count, this rank's {fab id: address} and the rank count."""

    def __init__(self, rows, ncomp, addrs, nranks, item=None):
        self.rows, self.ncomp, self.addrs, self.nranks, self.item = rows, int(ncomp), addrs, int(nranks), item


def _side_of(mf, grow) -> _Side:
    fab = next(iter(mf.fabs.values()), None)
    return _Side(_rows(list(mf.ba), grow=grow), mf.ncomp, _addrs(mf), mf.dm.nranks,
                 fab.data.dtype.itemsize if fab is not None else None)


class _Prepared:
    """A built plan + this rank's executor + its pointer table (the reference
    caches its plan per PlanKey, comm.py:299-308; this caches all three).
    ``plan`` is built by ``build_plan()``; the executor runs the tags whose
    source fab this rank owns (GHX_EXEC_DIRECT), writing local and peer
    destination fabs."""

    def __init__(self, ctx, build_plan, src: _Side, dst: _Side, scomp, dcomp, ncomp, phased=False):
        L = lib()
        self.plan = P()
        _check(build_plan(C.byref(self.plan)))
        self.ex = P()
        self.nseg = L.ghx_plan_num_segments(self.plan)
        nranks = max(src.nranks, dst.nranks)
        rank = ctx.rank
        item = dst.item or src.item or 8  # a rank without fabs runs no tags
        # the reference's fabs are numpy arrays, i.e. host memory (pinned and
        # mapped): the exchange crosses PCIe, where requests, not bytes,
        # cost -- the phased FillBoundary (faces extended over the lower-axis
        # ghosts, no edge/corner requests), seam-chunk ring tasks and a small
        # grid (include/ghostx.h)
        kind = GHX_EXEC_DIRECT | (GHX_EXEC_PHASED if phased else 0)
        _check(L.ghx_exec_create(self.plan, rank, kind, _p64(src.rows), src.ncomp, _p64(dst.rows), dst.ncomp, scomp,
                                 dcomp, ncomp, item, 0, C.byref(self.ex)))
        _check(L.ghx_exec_set_ring(self.ex, 1))
        _check(L.ghx_exec_set_grid(self.ex, 6, 256))
        ns, nd = len(src.rows), len(dst.rows)
        self.table = np.zeros(ns + nd + 2 * nranks, np.uint64)  # [src fabs][dst fabs][send][recv]
        for i, a in src.addrs.items():
            self.table[i] = a
        for i, a in _allgather_addrs(ctx, dst.addrs).items():
            self.table[ns + i] = a
        # Bus accounting per call: one message per ordered pair, the pair's
        # payload bytes (the reference's pack buffers, comm.py:343-357)
        pc = np.zeros(nranks * nranks, np.int64)
        _check(L.ghx_plan_pair_cells(self.plan, _p64(pc)))
        pc = pc.reshape(nranks, nranks) * ncomp * item
        self.sends = [(d, int(pc[rank, d])) for d in range(nranks) if d != rank and pc[rank, d]]
        self.recvs = [s for s in range(nranks) if s != rank and pc[s, rank]]

    def run(self, ctx) -> None:
        if self.nseg == 0:  # the reference returns before its barrier (comm.py:390-391)
            return
        L = lib()
        multi = ctx.nranks > 1
        if multi:
            ctx.barrier()  # every rank is in the call: its ghost cells may be written
        t = self.table
        _check(L.ghx_exec_run(self.ex, t.ctypes.data_as(C.POINTER(P)), len(t), None))
        _check(L.ghx_stream_sync(None))
        if multi:
            for d, nbytes in self.sends:
                ctx.send(d, None, nbytes=nbytes)
            for s in self.recvs:
                ctx.recv(s)
            ctx.barrier()

    def __del__(self):
        try:
            lib().ghx_exec_free(self.ex)
            lib().ghx_plan_free(self.plan)
        except Exception:  # noqa: BLE001
            pass


def fill_boundary_native(mf, geom=None) -> None:
    """Drop-in body for the reference's comm.fill_boundary (comm.py:383-394):
    the plan and executor are built once per MultiFab and geometry, every
    call is one kernel launch plus a stream synchronize (the reference API
    is synchronous); collective under ``runtime_spawn``, where every rank
    must build its MultiFabs at the same program points (SPMD, as the
    reference's programs do: the first call per MultiFab is a collective
    setup).  The fabs must live in device or pinned-mapped memory
    (``PinnedArena``)."""
    geom = geom or mf.geom
    key = ("ghostx", tuple(bool(v) for v in geom.periodic), tuple(geom.period))  # cf. PlanKey, comm.py:296-299
    ctx = _ctx_of(mf)
    prep = mf.plan_cache.get(key)
    if prep is None:
        L = lib()
        d = len(mf.ngrow)
        ng = np.array(list(mf.ngrow) + [0] * (3 - d), np.int64)
        per = np.array([int(v) for v in geom.periodic] + [0] * (3 - d), np.int32)
        period = np.array(list(geom.period) + [1] * (3 - d), np.int64)
        rows = _rows(list(mf.ba))
        ranks = np.asarray(mf.dm.rank_of, np.int32)

        def build(out):
            return L.ghx_plan_build_fill_boundary(len(rows), _p64(rows), _p64(ng), _p32(per), _p64(period),
                                                  _p32(ranks), mf.dm.nranks, out)
        side = _side_of(mf, tuple(int(v) for v in ng))
        prep = mf.plan_cache[key] = _Prepared(ctx, build, side, side, 0, 0, mf.ncomp, phased=True)
        mf.plan_builds += 1  # the reference counts its plan builds (comm.py:308)
    prep.run(ctx)


def parallel_copy_native(dst, src, scomp=0, dcomp=0, ncomp=None, ngrow_src=0, ngrow_dst=0, geom=None) -> None:
    """Drop-in body for the reference's comm.parallel_copy (comm.py:397-429)
    (the reference's argument checks omitted): a ParallelCopy plan between
    the two layouts, cached on ``dst`` per (source layout, ghost widths,
    geometry), one launch per call; collective under ``runtime_spawn``."""
    ncomp = ncomp if ncomp is not None else min(src.ncomp - scomp, dst.ncomp - dcomp)
    ctx = _ctx_of(dst)
    key = ("ghostx_pc", id(src), int(ngrow_src), int(ngrow_dst), id(geom), scomp, dcomp, ncomp)
    prep = dst.plan_cache.get(key)
    if prep is None or prep.src() is not src:  # (a new source at a recycled id: rebuild)
        L = lib()
        d = len(dst.ngrow)
        gs = np.array([int(ngrow_src)] * d + [0] * (3 - d), np.int64)
        gd = np.array([int(ngrow_dst)] * d + [0] * (3 - d), np.int64)
        drows, srows = _rows(list(dst.ba)), _rows(list(src.ba))
        if geom is not None:
            per = np.array([int(v) for v in geom.periodic] + [0] * (3 - d), np.int32)
            period = np.array(list(geom.period) + [1] * (3 - d), np.int64)
        else:
            per, period = None, np.ones(3, np.int64)
        sr, dr = np.asarray(src.dm.rank_of, np.int32), np.asarray(dst.dm.rank_of, np.int32)
        nranks = max(src.dm.nranks, dst.dm.nranks)

        def build(out):
            return L.ghx_plan_build_parallel_copy(len(drows), _p64(drows), _p64(gd), len(srows), _p64(srows),
                                                  _p64(gs), None if per is None else _p32(per), _p64(period),
                                                  _p32(sr), _p32(dr), nranks, out)
        sg = tuple(int(v) for v in src.ngrow) + (0,) * (3 - d)
        dg = tuple(int(v) for v in dst.ngrow) + (0,) * (3 - d)
        prep = dst.plan_cache[key] = _Prepared(ctx, build, _side_of(src, sg), _side_of(dst, dg), scomp, dcomp, ncomp)
        prep.src = weakref.ref(src)
        dst.plan_builds += 1  # (comm.py:424)
    prep.run(ctx)


def _ref_module(obj, name):
    """A module of the reference package ``obj`` comes from."""
    return importlib.import_module(type(obj).__module__.rsplit(".", 1)[0] + "." + name)


class _FillPatch:
    """fill_patch's cached coarse side for one (fine, coarse) pair: the
    reference's own coarse-fill targets (amr.py:320-352, host planning), a
    ParallelCopy-shaped gather plan from the coarse valid cells (periodic
    images included) into pinned target fabs (comm.py:432-443), and one
    interp job per (owned target, region)."""

    def __init__(self, ctx, fine, coarse, fine_geom, coarse_geom, ratio, scheme):
        ramr, rix, rmesh = (_ref_module(fine, m) for m in ("amr", "index_space", "mesh"))
        L = lib()
        self.coarse = weakref.ref(coarse)
        reach = 1 if scheme == ramr.LINEAR else 0
        targets = ramr._coarse_fill_targets(fine.ba, fine.ngrow, fine_geom)
        gather = [(gi, rix.grow(rix.coarsen(rix.grow(fine.ba[gi], fine.ngrow), ratio), reach))
                  for gi in sorted(targets)]
        self.gather, self.jobs = None, None
        if not gather:
            return
        me = ctx.rank
        dst_ranks = np.asarray([fine.dm[gi] for gi, _ in gather], np.int32)
        arena = fine.arena if isinstance(fine.arena, PinnedArena) else PinnedArena()
        # this rank's target fabs, kept across calls (the reference allocates
        # them per call, amr.py:385-386); plan positions address them
        self.owned = {pos: rmesh.Fab(cbox, fine.ncomp, arena) for pos, (gi, cbox) in enumerate(gather)
                      if dst_ranks[pos] == me}
        d = len(fine.ngrow)
        drows = _rows([b for _, b in gather])
        srows = _rows(list(coarse.ba))
        zero = np.zeros(3, np.int64)
        per = np.array([int(v) for v in coarse_geom.periodic] + [0] * (3 - d), np.int32)
        period = np.array(list(coarse_geom.period) + [1] * (3 - d), np.int64)
        sr = np.asarray(coarse.dm.rank_of, np.int32)
        nranks = max(coarse.dm.nranks, int(dst_ranks.max()) + 1)

        def build(out):
            return L.ghx_plan_build_parallel_copy(len(drows), _p64(drows), _p64(zero), len(srows), _p64(srows),
                                                  _p64(zero), _p32(per), _p64(period), _p32(sr), _p32(dst_ranks),
                                                  nranks, out)
        cg = tuple(int(v) for v in coarse.ngrow) + (0,) * (3 - d)
        item = next(iter(fine.fabs.values())).data.dtype.itemsize if fine.fabs else None
        tside = _Side(drows, fine.ncomp, {pos: f.data.__array_interface__["data"][0] for pos, f in self.owned.items()},
                      nranks, item)
        self.gather = _Prepared(ctx, build, _side_of(coarse, cg), tside, 0, 0, coarse.ncomp)
        # interp jobs (ghx_interp_job: 20 int64 words each), fine fabs in order
        rows = []
        pos_of = {gi: pos for pos, (gi, _) in enumerate(gather)}
        fg = tuple(int(v) for v in fine.ngrow) + (0,) * (3 - d)
        for gi in sorted(targets):
            pos = pos_of[gi]
            if pos not in self.owned:
                continue
            crse = self.owned[pos]
            for region in targets[gi]:
                rows.append([crse.data.__array_interface__["data"][0], *_rows([gather[pos][1]])[0],
                             fine.fabs[gi].data.__array_interface__["data"][0], *_rows([fine.ba[gi]], grow=fg)[0],
                             *_rows([region])[0]])
        self.jobs = np.ascontiguousarray(np.asarray(rows, np.int64).reshape(-1, 20))
        self.ratio = np.array([int(ratio)] * d + [1] * (3 - d), np.int32)
        self.dim, self.scheme = d, 1 if scheme == ramr.LINEAR else 0
        self.ncomp, self.item = fine.ncomp, item or 8

    def run(self, ctx) -> None:
        if self.gather is None:
            return
        self.gather.run(ctx)  # collective, ends with the reference's barrier
        if len(self.jobs):
            L = lib()
            _check(L.ghx_interp(P(self.jobs.ctypes.data), len(self.jobs), self.ncomp, _p32(self.ratio), self.dim,
                                self.scheme, self.item, None))
            _check(L.ghx_stream_sync(None))


def fill_patch_native(fine, coarse, fine_geom, coarse_geom, ratio: int, scheme: str = "linear") -> None:
    """Drop-in body for the reference's amr.fill_patch (amr.py:355-397): the
    fine FillBoundary, the gather of coarse data into target fabs and every
    interpolation job in one launch; the coarse-side plan is built once per
    (fine, coarse) pair.  Collective under ``runtime_spawn`` (SPMD)."""
    ratio = int(ratio)
    fill_boundary_native(fine, fine_geom)
    ctx = _ctx_of(fine)
    key = ("ghostx_fp", id(coarse), tuple(coarse_geom.period), ratio, scheme)
    prep = fine.plan_cache.get(key)
    if prep is None or prep.coarse() is not coarse:
        prep = fine.plan_cache[key] = _FillPatch(ctx, fine, coarse, fine_geom, coarse_geom, ratio, scheme)
        fine.plan_builds += 1  # (amr.py:380)
    prep.run(ctx)


class _AverageDown:
    """average_down's cached tmp MultiFab (the coarsened fine layout, pinned)
    and its restriction jobs (ghx_avgdown_job: 20 int64 words each)."""

    def __init__(self, fine, coarse, ratio):
        rix, rmesh, rconfig = (_ref_module(fine, m) for m in ("index_space", "mesh", "config"))
        self.coarse = weakref.ref(coarse)
        arena = fine.arena if isinstance(fine.arena, PinnedArena) else PinnedArena()
        self.tmp = rmesh.MultiFab(rmesh.BoxArray([rix.coarsen(b, ratio) for b in fine.ba]), fine.dm, fine.ncomp, 0,
                                  arena=arena)
        d = len(fine.ngrow)
        fg = tuple(int(v) for v in fine.ngrow) + (0,) * (3 - d)
        rows = []
        for gi in fine.local_indices:
            cb = self.tmp.ba[gi]
            rows.append([fine.fabs[gi].data.__array_interface__["data"][0], *_rows([fine.ba[gi]], grow=fg)[0],
                         self.tmp.fabs[gi].data.__array_interface__["data"][0], *_rows([cb])[0], *_rows([cb])[0]])
        self.jobs = np.ascontiguousarray(np.asarray(rows, np.int64).reshape(-1, 20))
        self.ratio = np.array([int(ratio)] * d + [1] * (3 - d), np.int32)
        self.dim, self.ncomp = d, fine.ncomp
        self.item = next(iter(fine.fabs.values())).data.dtype.itemsize if fine.fabs else 8
        if rconfig.spacedim != d:
            raise ValueError(f"MultiFab has {d} axes, the reference is configured for {rconfig.spacedim}")

    def run(self) -> None:
        if len(self.jobs):
            L = lib()
            _check(L.ghx_average_down(P(self.jobs.ctypes.data), len(self.jobs), self.ncomp, _p32(self.ratio),
                                      self.dim, self.item, None))
            _check(L.ghx_stream_sync(None))


def average_down_native(fine, coarse, ratio: int) -> None:
    """Drop-in body for the reference's amr.average_down (amr.py:235-266):
    the restriction of every local fine fab into a tmp MultiFab on the
    coarsened fine layout (one launch), then parallel_copy_native(coarse,
    tmp); the tmp MultiFab and the jobs are kept per (fine, coarse) pair.
    Collective under ``runtime_spawn`` (SPMD)."""
    ratio = int(ratio)
    if ratio < 1:
        raise ValueError("ratio must be >= 1")
    for b in fine.ba:
        if any(e % ratio for e in b.extents) or any(v % ratio for v in b.lo):
            raise ValueError(f"fine box {b} is not aligned to ratio {ratio}")
    if fine.ncomp != coarse.ncomp:
        raise ValueError("component count mismatch")
    key = ("ghostx_ad", id(coarse), ratio)
    prep = fine.plan_cache.get(key)
    if prep is None or prep.coarse() is not coarse:
        prep = fine.plan_cache[key] = _AverageDown(fine, coarse, ratio)
    prep.run()
    parallel_copy_native(coarse, prep.tmp)


def interp_box_native(coarse_fab, fine_fab, fine_region, ratio: int, scheme: str = "pc") -> None:
    """Drop-in body for the reference's amr.interp_box (amr.py:269-314) on
    pinned fabs: one ghx_interp job (20 int64 words)."""
    job = np.zeros((1, 20), np.int64)
    job[0, 0] = coarse_fab.data.__array_interface__["data"][0]
    job[0, 1:7] = _rows([coarse_fab.box])[0]
    job[0, 7] = fine_fab.data.__array_interface__["data"][0]
    job[0, 8:14] = _rows([fine_fab.box])[0]
    job[0, 14:20] = _rows([fine_region])[0]
    d = len(fine_region.lo)
    r3 = np.array([int(ratio)] * d + [1] * (3 - d), np.int32)
    L = lib()
    _check(L.ghx_interp(P(job.ctypes.data), 1, fine_fab.ncomp, _p32(r3), d, 1 if scheme == "linear" else 0,
                        fine_fab.data.dtype.itemsize, None))
    _check(L.ghx_stream_sync(None))
