"""FillBoundary / ParallelCopy: cached plans, one fused launch per call.

Drop-in for the hot path of the reference's ``miniamr_core.comm``
(/root/reference/pkg/src/miniamr_core/comm.py):

====================================  =========================================
reference (comm.py)                   here
====================================  =========================================
Bus / RankContext / runtime_spawn     same semantics (ranks are threads, one
  :35-180                             per GPU round-robin); plus a process
                                      context when torch.distributed is up
PlanKey / CopySegment / CommPlan      same fields; segments come from the
  :189-247                            native binned builder (ghx_plan_*)
plan_build_fill_boundary :289-309     same validation order, per-MultiFab
                                      cache and ``plan_builds`` counter
_execute_plan :316-380                ghx_exec_run: ONE fused sm_100a launch
                                      moves local tags and pushes remote tags
                                      straight into the peer's fabs
                                      (NCCL send/recv only as a fallback)
fill_boundary :383-394                same contract, synchronous
parallel_copy :397-429                same contract, synchronous
====================================  =========================================

Message accounting keeps the reference's contract (tests/test_comm.py:182,
:236, :356): per call at most one "message" per ordered rank pair, bytes =
cells * ncomp * itemsize of the reference segments for that pair.
"""

from __future__ import annotations

import contextlib
import ctypes as C
import itertools
import os
import sys
import threading
import weakref
from collections import deque
from dataclasses import dataclass

import numpy as np

from . import _native as N
from . import config
from .index_space import Box, Geometry, IntVect, grow
from .mesh import MultiFab, Slab

SUM, MIN, MAX = "sum", "min", "max"
_COMBINE = {SUM: lambda a, b: a + b, MIN: min, MAX: max}


class RankFailure(RuntimeError):
    """A thread rank of ``runtime_spawn`` raised; ``rank`` is the root cause,
    ``cause`` its exception (reference comm.py:28-32 semantics)."""

    def __init__(self, rank: int, cause: BaseException):
        super().__init__(f"rank {rank} failed: {cause!r}")
        self.rank, self.cause = rank, cause


# --------------------------------------------------------------- rank runtime

class _Mailbox:
    """One ordered rank pair's FIFO: a deque plus an event a blocked
    receiver sleeps on (set while messages are queued or the run aborts)."""

    __slots__ = ("items", "ready")

    def __init__(self):
        self.items: deque = deque()
        self.ready = threading.Event()


class Bus:
    """In-process transport of the thread ranks (reference comm.py:35-87
    semantics): FIFO per ordered pair, exactly-once delivery, per-pair
    (messages, bytes) counters, one reusable barrier, an abort that wakes
    every blocked receiver and breaks the barrier when a rank fails.  Device
    exchanges move no payload through it -- they only ``account`` the
    message the reference would have sent."""

    def __init__(self, nranks: int):
        self.nranks = nranks
        self._box = [[_Mailbox() for _ in range(nranks)] for _ in range(nranks)]  # [src][dst]
        self._counts = np.zeros((nranks, nranks, 2), np.int64)  # messages, bytes
        self._lock = threading.Lock()
        self.barrier = threading.Barrier(nranks) if nranks > 1 else None
        self._slots: list = [None] * nranks  # allgather exchange area
        self._failed: int | None = None

    def account(self, src: int, dst: int, nbytes: int) -> None:
        with self._lock:
            self._counts[src, dst, 0] += 1
            self._counts[src, dst, 1] += int(nbytes)

    def send(self, src: int, dst: int, payload, nbytes: int) -> None:
        box = self._box[src][dst]
        box.items.append(payload)  # deque appends are atomic
        self.account(src, dst, nbytes)
        box.ready.set()

    def recv(self, src: int, dst: int):
        box = self._box[src][dst]  # one receiving thread per mailbox
        while True:
            if box.items:
                return box.items.popleft()
            if self._failed is not None:
                raise RuntimeError(f"recv aborted: rank {self._failed} failed")
            box.ready.clear()
            if not box.items:  # a send between the check and the clear is seen here
                box.ready.wait(timeout=0.1)

    def fail(self, rank: int) -> None:
        with self._lock:
            if self._failed is None:  # the first failure is the root cause
                self._failed = rank
        for row in self._box:
            for box in row:
                box.ready.set()
        if self.barrier is not None:
            self.barrier.abort()

    @property
    def message_stats(self) -> dict:
        return {k: list(v) for k, v in self.stats_snapshot().items()}

    def stats_snapshot(self) -> dict:
        with self._lock:
            c = self._counts.copy()
        n = self.nranks
        return {(s_, d_): (int(c[s_, d_, 0]), int(c[s_, d_, 1])) for s_ in range(n) for d_ in range(n)}

    def format_stats(self) -> str:
        active = [f"  {s_}->{d_}: {m} messages, {b} bytes"
                  for (s_, d_), (m, b) in sorted(self.stats_snapshot().items()) if m]
        return "comm message stats (src->dst: messages, bytes):\n" + "\n".join(active or ["  (no messages)"])


def _cuda_devices() -> int:
    try:
        import torch
        return torch.cuda.device_count() if torch.cuda.is_available() else 0
    except Exception:
        return 0


class RankContext:
    """Per-rank handle: rank id, device, shared bus."""

    kind = "thread"

    def __init__(self, rank: int, nranks: int, bus: Bus, device: int | None = None):
        self.rank = rank
        self.nranks = nranks
        self.bus = bus
        self._device = device

    @property
    def device(self) -> int:
        if self._device is not None:
            return self._device
        if _cuda_devices():
            import torch
            return torch.cuda.current_device()
        return 0

    def send(self, dst: int, payload, nbytes: int = 0) -> None:
        self.bus.send(self.rank, dst, payload, nbytes)

    def recv(self, src: int):
        return self.bus.recv(src, self.rank)

    def barrier(self) -> None:
        if self.bus.barrier is not None:
            self.bus.barrier.wait()

    def allgather(self, obj) -> list:
        if self.nranks == 1:
            return [obj]
        self.bus._slots[self.rank] = obj
        self.barrier()
        out = list(self.bus._slots)
        self.barrier()
        return out

    def allreduce(self, ops, values) -> tuple:
        ops = tuple(ops)
        values = tuple(float(v) for v in values)
        if len(ops) != len(values):
            raise ValueError("allreduce needs one value per op")
        if self.nranks == 1:
            return values
        slots = self.allgather((ops, values))
        if any(s[0] != ops for s in slots):
            raise ValueError("mismatched reduction op lists across ranks")
        out = list(slots[0][1])
        for _, vals in slots[1:]:
            out = [_COMBINE[op](a, b) for op, a, b in zip(ops, out, vals)]
        return tuple(out)


class ProcessContext:
    """One process per GPU under torch.distributed (torchrun): rank = the
    process group rank, device = LOCAL_RANK.  Bus statistics record the
    messages this process sends."""

    kind = "process"

    def __init__(self):
        import torch
        import torch.distributed as dist
        self._dist = dist
        self.rank = dist.get_rank()
        self.nranks = dist.get_world_size()
        self.bus = Bus(self.nranks) if self.nranks == 1 else _LocalBus(self.nranks)
        ndev = _cuda_devices()
        local = int(os.environ.get("LOCAL_RANK", self.rank))
        self.device = (local % ndev) if ndev else 0
        self.backend = dist.get_backend()

    def barrier(self) -> None:
        if self.nranks > 1:
            self._dist.barrier()

    def allgather(self, obj) -> list:
        if self.nranks == 1:
            return [obj]
        out = [None] * self.nranks
        self._dist.all_gather_object(out, obj)
        return out

    def allreduce(self, ops, values) -> tuple:
        ops = tuple(ops)
        values = tuple(float(v) for v in values)
        slots = self.allgather((ops, values))
        if any(s[0] != ops for s in slots):
            raise ValueError("mismatched reduction op lists across ranks")
        out = list(slots[0][1])
        for _, vals in slots[1:]:
            out = [_COMBINE[op](a, b) for op, a, b in zip(ops, out, vals)]
        return tuple(out)

    def send(self, dst, payload, nbytes=0):
        raise NotImplementedError("object send/recv is only available between thread ranks")

    recv = send


class _LocalBus(Bus):
    """Process mode: only this process's message counters (no mailboxes in
    use, the collectives go through torch.distributed)."""

    def __init__(self, nranks):
        super().__init__(nranks)
        self.barrier = None


_tls = threading.local()
_serial_ctx = RankContext(0, 1, Bus(1))
_process_ctx: ProcessContext | None = None


def current_ctx():
    ctx = getattr(_tls, "ctx", None)
    if ctx is not None:
        return ctx
    global _process_ctx
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            if _process_ctx is None or _process_ctx.nranks != dist.get_world_size():
                _process_ctx = ProcessContext()
            return _process_ctx
    except Exception:
        pass
    return _serial_ctx


def current_rank() -> int:
    return current_ctx().rank


@contextlib.contextmanager
def _rank_scope(ctx):
    """Make ``ctx`` the calling thread's current rank for the block."""
    prev = getattr(_tls, "ctx", None)
    _tls.ctx = ctx
    try:
        yield ctx
    finally:
        _tls.ctx = prev


def runtime_spawn(nranks: int, program) -> list:
    """Run program(ctx) once per logical rank, each on its own thread with
    its own GPU (rank r -> device r % device_count), and return the per-rank
    results.  A rank that raises aborts the others' blocking calls (bus
    abort) and the run raises RankFailure naming the root-cause rank
    (reference comm.py:143-180 semantics)."""
    if nranks < 1:
        raise ValueError("nranks must be >= 1")
    bus = Bus(nranks)
    ndev = _cuda_devices()
    ctxs = [RankContext(r, nranks, bus, (r % ndev) if ndev else 0) for r in range(nranks)]
    if nranks == 1:
        with _rank_scope(ctxs[0]):
            return [program(ctxs[0])]
    outcome: list = [None] * nranks  # (ok, value or exception)

    def body(ctx) -> None:
        with _rank_scope(ctx):
            try:
                if ndev:
                    import torch
                    torch.cuda.set_device(ctx.device)
                outcome[ctx.rank] = (True, program(ctx))
            except BaseException as exc:  # noqa: BLE001 - reported with its rank below
                outcome[ctx.rank] = (False, exc)
                bus.fail(ctx.rank)

    workers = [threading.Thread(target=body, args=(c,), name=f"rank{c.rank}") for c in ctxs]
    for w in workers:
        w.start()
    for w in workers:
        w.join()
    failed = {r: o[1] for r, o in enumerate(outcome) if not o[0]}
    if failed:
        root = bus._failed if bus._failed in failed else min(failed)
        raise RankFailure(root, failed[root]) from failed[root]
    return [o[1] for o in outcome]


def global_reduce(ops, values, ctx=None) -> tuple:
    ctx = ctx or current_ctx()
    return ctx.allreduce(ops, values)


# ---------------------------------------------------------------------- plans

@dataclass(frozen=True)
class PlanKey:
    src_ba: int
    src_dm: int
    dst_ba: int
    dst_dm: int
    ngrow_src: tuple
    ngrow_dst: tuple
    ixtype: tuple
    periodic: tuple
    op: str


@dataclass(frozen=True)
class CopySegment:
    src_fab: int
    dst_fab: int
    src_box: Box
    dst_box: Box
    shift: tuple

    @property
    def cells(self) -> int:
        return self.dst_box.num_pts


_plan_uid = itertools.count(1)
_plan_lock = threading.Lock()
# process-wide cache of native plans so per-rank MultiFabs sharing a layout
# build once; per-MultiFab ``plan_cache`` / ``plan_builds`` still follow the
# reference exactly
_global_plans: "weakref.WeakValueDictionary" = weakref.WeakValueDictionary()


class CommPlan:
    """Cached copy schedule: sorted segments grouped into per-rank local
    lists and per-ordered-pair message lists (comm.py:218-247)."""

    def __init__(self, handle: int, nranks: int, dim: int, ixtype):
        self.uid = next(_plan_uid)
        self._h = C.c_void_p(handle)
        self.nranks = nranks
        self._dim = dim
        self._ixtype = ixtype
        self.num_segments = int(N.lib.ghx_plan_num_segments(self._h))
        self.num_write_tags = int(N.lib.ghx_plan_num_write_tags(self._h))
        pc = np.zeros(nranks * nranks, np.int64)
        N.check(N.lib.ghx_plan_pair_cells(self._h, N.i64p(pc)))
        self.pair_cells = pc.reshape(nranks, nranks)
        self._rows = None
        self._groups = None
        self._execs: dict = {}
        self._lock = threading.Lock()

    @property
    def is_empty(self) -> bool:
        return self.num_segments == 0

    def rows(self) -> np.ndarray:
        """(num_segments, 13) int64: src dst dlo(3) dhi(3) shift(3) srank drank."""
        if self._rows is None:
            r = np.zeros((self.num_segments, 13), np.int64)
            if self.num_segments:
                N.check(N.lib.ghx_plan_get_segments(self._h, N.i64p(r)))
            self._rows = r
        return self._rows

    def _build_groups(self):
        from .index_space import IntVect as IV
        d = self._dim
        local, pairs = {}, {}
        for row in self.rows():
            lo = IV(*row[2:2 + d])
            hi = IV(*row[5:5 + d])
            s = tuple(int(v) for v in row[8:8 + d])
            dst = Box(lo, hi, self._ixtype)
            seg = CopySegment(int(row[0]), int(row[1]), dst.shift(tuple(-v for v in s)), dst, s)
            sr, dr = int(row[11]), int(row[12])
            if sr == dr:
                local.setdefault(sr, []).append(seg)
            else:
                pairs.setdefault((sr, dr), []).append(seg)
        self._groups = (local, pairs)

    @property
    def local_by_rank(self) -> dict:
        if self._groups is None:
            self._build_groups()
        return self._groups[0]

    @property
    def pair_segments(self) -> dict:
        if self._groups is None:
            self._build_groups()
        return self._groups[1]

    def sends_from(self, rank: int) -> dict:
        return {d: segs for (s, d), segs in sorted(self.pair_segments.items()) if s == rank}

    def recvs_to(self, rank: int) -> dict:
        return {s: segs for (s, d), segs in sorted(self.pair_segments.items()) if d == rank}

    def executor(self, rank, kind, src_mf, dst_mf, scomp, dcomp, ncomp) -> "Executor":
        # fabs in pinned host memory: seam-chunk (ring) tasks, fewer and larger PCIe transactions
        host = getattr(dst_mf, "memory", "device") == "pinned" or getattr(src_mf, "memory", "device") == "pinned"
        ring = {"1": True, "0": False}.get(os.environ.get("GHX_RING", ""), host)
        # distinct source and destination storage: no byte is read after being
        # written in one run, so wide rows may go through TMA bulk copies
        bulk = src_mf is not dst_mf and not host and os.environ.get("GHX_PC_BULK", "1") == "1"
        # fabs in host memory: the phased exchange (faces extended over the
        # lower-axis ghosts, no edge / corner tags: fewer PCIe requests);
        # GHX_PHASED=1 / 0 forces it on / off (device fabs: parity testing)
        phased = kind in (N.EXEC_DIRECT, N.EXEC_LOCAL) and src_mf is dst_mf and \
            {"1": True, "0": False}.get(os.environ.get("GHX_PHASED", ""), host)
        key = (rank, kind, src_mf.ngrow.comps, src_mf.ncomp, dst_mf.ngrow.comps, dst_mf.ncomp,
               scomp, dcomp, ncomp, dst_mf.dtype.itemsize, dst_mf.device, ring, host, bulk, phased)
        with self._lock:
            ex = self._execs.get(key)
            if ex is None:
                ex = Executor(self, rank, kind | (N.EXEC_PHASED if phased else 0), src_mf.storage_rows(),
                              src_mf.ncomp, dst_mf.storage_rows(), dst_mf.ncomp, scomp, dcomp, ncomp,
                              dst_mf.dtype.itemsize, dst_mf.device, ring, host, bulk)
                self._execs[key] = ex
        return ex

    def __del__(self):
        try:
            self._execs.clear()
            if self._h:
                N.lib.ghx_plan_free(self._h)
                self._h = None
        except Exception:
            pass


class Executor:
    """One rank's compiled share of a plan for one storage layout (a device
    tag table; ``run`` is one launch of the fused copy kernel)."""

    def __init__(self, plan, rank, kind, src_rows, src_nc, dst_rows, dst_nc, scomp, dcomp, ncomp, item, device,
                 ring=False, host=False, bulk=False):
        h = C.c_void_p()
        N.check(N.lib.ghx_exec_create(plan._h, rank, kind, N.i64p(src_rows), src_nc, N.i64p(dst_rows), dst_nc,
                                      scomp, dcomp, ncomp, item, device, C.byref(h)))
        self._h = h
        if ring:
            N.check(N.lib.ghx_exec_set_ring(h, 1))
        if bulk:
            N.check(N.lib.ghx_exec_set_bulk(h, 1))
        if host:
            # fabs in host memory: the PCIe / IOMMU path saturates with few
            # concurrent warps and degrades with many (scattered 32-64 B
            # requests); 6 CTAs measured best with the phased exchange and
            # tile-ring seams (C3 e2e 49.4 -> 47.9 ms, C4 28.0 -> 26.8; C2
            # 5.76 -> 5.87; 4, 5, 7, 10, 12, 16 slower)
            N.check(N.lib.ghx_exec_set_grid(h, int(os.environ.get("GHX_HOST_BLOCKS", "6")), 256))
        self.plan = plan
        self.device = device
        self.nsrc = len(src_rows)
        self.ndst = len(dst_rows)
        self.nranks = plan.nranks
        self.nptrs = self.nsrc + self.ndst + 2 * self.nranks
        a, b, c, d = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        N.check(N.lib.ghx_exec_info(h, C.byref(a), C.byref(b), C.byref(c), C.byref(d)))
        self.ntags, self.ntasks, self.elems, self.alg_bytes = a.value, b.value, c.value, d.value
        be = np.zeros(self.nranks, np.int64)
        N.check(N.lib.ghx_exec_buffer_elems(h, N.i64p(be)))
        self.buffer_elems = be
        re_ = np.zeros(self.nranks, np.int64)
        N.check(N.lib.ghx_exec_recv_elems(h, N.i64p(re_)))
        self.recv_elems = re_
        det = np.zeros(8, np.int64)
        N.check(N.lib.ghx_exec_detail(h, N.i64p(det)))
        self.detail = dict(zip(("tags", "tasks", "elems", "alg_bytes", "mirror_tags", "swap_tags", "blocks",
                                "ld_mode"), (int(v) for v in det)))
        kinds = np.zeros(6, np.int64)
        N.check(N.lib.ghx_exec_task_kinds(h, N.i64p(kinds)))
        self.detail.update(zip(("copy_tasks", "swap_tasks", "chain_tasks", "ring_tasks", "ring_mode", "fab_local"),
                               (int(v) for v in kinds)))
        ph = np.zeros(4, np.int64)
        N.check(N.lib.ghx_exec_phases(h, N.i64p(ph)))
        self.detail["phased"] = int(ph[0])
        sf = C.c_int64()
        N.check(N.lib.ghx_exec_sector_fills(h, C.byref(sf)))
        self.detail["sector_fill_tags"] = sf.value

    def run(self, table: np.ndarray, stream: int) -> None:
        """One launch with a raw pointer table (bound on the fly; an
        unpinned binding may be recycled later)."""
        assert table.dtype == np.uint64 and table.size == self.nptrs
        N.check(N.lib.ghx_exec_run(self._h, table.ctypes.data_as(C.POINTER(C.c_void_p)), self.nptrs,
                                   C.c_void_p(stream)))

    def bind(self, table: np.ndarray, stream: int | None = None) -> "Binding":
        """Pin ``table`` (ghx_exec_bind): launches of the returned binding
        skip all host table work and stay valid inside CUDA graphs."""
        assert table.dtype == np.uint64 and table.size == self.nptrs
        if stream is None:
            stream = _stream(self.device).cuda_stream
        bid = C.c_int64()
        N.check(N.lib.ghx_exec_bind(self._h, table.ctypes.data_as(C.POINTER(C.c_void_p)), self.nptrs,
                                    C.c_void_p(stream), C.byref(bid)))
        return Binding(self, bid.value)

    def set_grid(self, blocks: int) -> None:
        N.check(N.lib.ghx_exec_set_grid(self._h, int(blocks), 256))

    def set_sync(self, flag_table: np.ndarray, rank: int, nranks: int) -> None:
        """In-kernel READY / DONE synchronisation over the ranks' IPC flag
        arrays (ghx_exec_set_sync)."""
        assert flag_table.dtype == np.uint64 and flag_table.size == nranks
        N.check(N.lib.ghx_exec_set_sync(self._h, flag_table.ctypes.data_as(C.POINTER(C.c_void_p)), rank, nranks))

    def sync_wait(self, epoch: int, stream: int) -> None:
        N.check(N.lib.ghx_exec_sync_wait(self._h, C.c_uint64(epoch), C.c_void_p(stream)))

    def __del__(self):
        try:
            if self._h:
                N.lib.ghx_exec_free(self._h)
                self._h = None
        except Exception:
            pass


class Binding:
    """A pinned pointer table of an Executor (released with the object)."""

    __slots__ = ("ex", "id", "__weakref__")

    def __init__(self, ex: Executor, bid: int):
        self.ex, self.id = ex, bid

    def run(self, stream: int) -> None:
        N.check(N.lib.ghx_exec_run_bound(self.ex._h, self.id, C.c_void_p(stream)))

    def run_synced(self, stream: int, epoch: int) -> None:
        N.check(N.lib.ghx_exec_run_synced(self.ex._h, self.id, C.c_uint64(epoch), C.c_void_p(stream)))

    def __del__(self):
        # the executor's live handle, never a cached copy: when a GC cycle
        # holds both objects, Python may finalize the executor first
        # (ghx_exec_free releases every binding with it)
        try:
            h = self.ex._h
            if self.id and h:
                N.lib.ghx_exec_unbind(h, self.id)
            self.id = 0
        except Exception:
            pass


def _native_plan(gkey, build) -> int:
    with _plan_lock:
        plan = _global_plans.get(gkey)
    if plan is not None:
        return plan
    plan = build()
    with _plan_lock:
        return _global_plans.setdefault(gkey, plan)


def plan_build_fill_boundary(mf: MultiFab, geom: Geometry | None = None) -> CommPlan:
    """Ghost-exchange plan for mf, cached on the MultiFab by PlanKey
    (reference comm.py:289-309: same checks, same order)."""
    geom = geom or mf.geom
    if geom is None:
        raise ValueError("fill_boundary needs a Geometry (periodicity)")
    if mf.ba.ixtype.is_mixed:
        raise ValueError("ghost exchange supports cell or fully-nodal index types only")
    key = PlanKey(mf.ba.uid, mf.dm.uid, mf.ba.uid, mf.dm.uid, (0,) * len(mf.ngrow), mf.ngrow.comps,
                  mf.ba.ixtype.flags, geom.periodic, "fill_boundary")
    plan = mf.plan_cache.get(key)
    if plan is not None:
        return plan
    if max(mf.ngrow) > mf.ba.minimal_extent():
        raise ValueError("ngrow larger than the smallest box extent is not supported")
    per = np.zeros(3, np.int32)
    per[:len(geom.periodic)] = geom.periodic
    period = np.ones(3, np.int64)
    period[:len(geom.period)] = geom.period
    ng = np.zeros(3, np.int64)
    ng[:len(mf.ngrow)] = mf.ngrow.comps
    ranks = mf.dm.array()

    def build():
        h = C.c_void_p()
        N.check(N.lib.ghx_plan_build_fill_boundary(len(mf.ba), N.i64p(mf.ba.rows()), N.i64p(ng), N.i32p(per),
                                                   N.i64p(period), N.i32p(ranks), mf.dm.nranks, C.byref(h)))
        return CommPlan(h.value, mf.dm.nranks, len(mf.ngrow), mf.ba.ixtype)

    plan = _native_plan((key, tuple(period)), build)
    mf.plan_cache[key] = plan
    mf.plan_builds += 1
    return plan


def _parallel_copy_plan(dst: MultiFab, src: MultiFab, gs: IntVect, gd: IntVect, geom) -> CommPlan:
    key = PlanKey(src.ba.uid, src.dm.uid, dst.ba.uid, dst.dm.uid, gs.comps, gd.comps, dst.ba.ixtype.flags,
                  geom.periodic if geom else (False,) * len(gs), "parallel_copy")
    plan = dst.plan_cache.get(key)
    if plan is not None:
        return plan
    nranks = max(src.dm.nranks, dst.dm.nranks)
    gsa = np.zeros(3, np.int64)
    gsa[:len(gs)] = gs.comps
    gda = np.zeros(3, np.int64)
    gda[:len(gd)] = gd.comps
    per = period = None
    if geom is not None:
        per = np.zeros(3, np.int32)
        per[:len(geom.periodic)] = geom.periodic
        period = np.ones(3, np.int64)
        period[:len(geom.period)] = geom.period

    def build():
        h = C.c_void_p()
        N.check(N.lib.ghx_plan_build_parallel_copy(
            len(dst.ba), N.i64p(dst.ba.rows()), N.i64p(gda), len(src.ba), N.i64p(src.ba.rows()), N.i64p(gsa),
            N.i32p(per) if per is not None else None, N.i64p(period) if period is not None else None,
            N.i32p(src.dm.array()), N.i32p(dst.dm.array()), nranks, C.byref(h)))
        return CommPlan(h.value, nranks, len(gs), dst.ba.ixtype)

    plan = _native_plan((key, None if period is None else tuple(period)), build)
    dst.plan_cache[key] = plan
    dst.plan_builds += 1
    return plan


# ------------------------------------------------------------------ execution

TRANSPORTS = ("p2p", "nccl")


def _transport(ctx=None) -> str:
    """The cross-process transport: GHX_TRANSPORT when set, else the
    CUDA-IPC push when every rank can map every peer's memory (probed once
    per process context, collectively), else the NCCL fallback."""
    t = os.environ.get("GHX_TRANSPORT")
    if t is None:
        return "p2p" if ctx is None or _ipc_capable(ctx) else "nccl"
    if t not in TRANSPORTS:
        raise ValueError(f"GHX_TRANSPORT must be one of {TRANSPORTS}, got {t!r}")
    return t


def _ipc_open(device: int, handle: bytes) -> int:
    """Map a peer's CUDA-IPC allocation.  If CUDA says the memory is already
    mapped, a stale mapping of a freed allocation at the same address is
    still held by objects awaiting the cyclic GC in this process (an
    Exchange and its MultiFab reference each other): collect, which closes
    those mappings through their finalizers, and retry once."""
    p = C.c_void_p()
    rc = N.lib.ghx_ipc_open_handle(device, (C.c_uint8 * 64).from_buffer_copy(handle), C.byref(p))
    if rc != 0 and "already mapped" in N.lib.ghx_last_error().decode():
        import gc
        gc.collect()
        rc = N.lib.ghx_ipc_open_handle(device, (C.c_uint8 * 64).from_buffer_copy(handle), C.byref(p))
    N.check(rc)
    return p.value


def _ipc_capable(ctx) -> bool:
    """Collective probe (cached on the context): every rank exports a small
    device allocation and maps every peer's; the IPC push is used only if
    all of them succeed on every rank (a box or container without CUDA IPC
    between the processes falls back to NCCL instead of failing)."""
    cap = getattr(ctx, "_ipc_ok", None)
    if cap is not None:
        return cap
    ok, h, probe = True, (C.c_uint8 * 64)(), None
    try:
        probe = Slab(256, ctx.device)
        N.check(N.lib.ghx_ipc_get_handle(C.c_void_p(probe.ptr), h))
        hb = bytes(h)
    except Exception:  # noqa: BLE001
        ok, hb = False, None
    handles = ctx.allgather(hb)
    for r, other in enumerate(handles):
        if r == ctx.rank or not ok:
            continue
        if other is None:
            ok = False
            break
        try:
            if os.environ.get("GHX_TEST_NO_IPC"):  # tests: a box without CUDA IPC between processes
                raise N.GhostxError("CUDA IPC disabled (GHX_TEST_NO_IPC)")
            N.lib.ghx_ipc_close_handle(C.c_void_p(_ipc_open(ctx.device, other)))
        except Exception:  # noqa: BLE001
            ok = False
    cap = all(ctx.allgather(ok))
    ctx.barrier()  # no rank frees its probe while a peer still maps it
    del probe
    if not cap and ctx.rank == 0:
        sys.stderr.write("[paper_2403_12179_b200] CUDA IPC between the ranks is unavailable: "
                         "cross-process exchanges use the NCCL transport\n")
    ctx._ipc_ok = cap
    return cap


def _host_resident(mf) -> bool:
    return getattr(mf, "memory", "device") == "pinned"


@contextlib.contextmanager
def torch_stream(stream: int, device: int):
    """Make the raw CUDA stream ``stream`` torch's current stream (torch's
    collectives and copies order against the current stream).  Handle 0 is
    the legacy default stream, which torch knows as its default stream:
    ``torch.cuda.ExternalStream(0)`` is NOT that stream (it syncs nothing
    launched on 0), so 0 must map to ``torch.cuda.default_stream``."""
    import torch
    dev = torch.device("cuda", device)
    cur = torch.cuda.current_stream(dev)
    if cur.cuda_stream == stream:
        ts = cur
    elif stream == 0:
        ts = torch.cuda.default_stream(dev)
    else:
        ts = torch.cuda.ExternalStream(stream, device=dev)
    with torch.cuda.stream(ts):
        yield ts


def _stream(device: int):
    import torch
    return torch.cuda.current_stream(device)


def _table(ex: Executor, src_mf: MultiFab, dst_parts, bufs=None) -> np.ndarray:
    """Pointer table [src fabs][dst fabs][send bufs][recv bufs]."""
    t = np.zeros(ex.nptrs, np.uint64)
    if src_mf.local_indices:
        t[np.asarray(src_mf.local_indices, np.int64)] = src_mf._ptrs
    for idx, ptrs in dst_parts:
        if len(idx):
            t[ex.nsrc + np.asarray(idx, np.int64)] = ptrs
    if bufs is not None:
        t[ex.nsrc + ex.ndst:] = bufs
    return t


_peer_enabled: set = set()


class _ProcessSync:
    """IPC-shared flag array per rank for the device-side barrier kernel."""

    def __init__(self, ctx):
        self.ctx = ctx
        n = ctx.nranks
        # 3 * n slots: [0, n) barrier kernel, [n, 2n) READY, [2n, 3n) DONE
        # (the in-kernel protocol of ghx_exec_run_synced)
        self.slab = Slab(8 * 3 * n, ctx.device)
        N.check(N.lib.ghx_memset_u64(C.c_void_p(self.slab.ptr), 0, 3 * n, None))
        import torch
        torch.cuda.synchronize(ctx.device)
        h = (C.c_uint8 * 64)()
        N.check(N.lib.ghx_ipc_get_handle(C.c_void_p(self.slab.ptr), h))
        handles = ctx.allgather(bytes(h))
        self.ptrs = []
        self._opened = []
        for r, hb in enumerate(handles):
            if r == ctx.rank:
                self.ptrs.append(self.slab.ptr)
                continue
            pv = _ipc_open(ctx.device, hb)
            self.ptrs.append(pv)
            self._opened.append(pv)
        self.table = np.asarray(self.ptrs, np.uint64)
        self.epoch = 0

    def next_epoch(self) -> int:
        self.epoch += 1
        return self.epoch

    def barrier(self, stream: int) -> None:
        self.epoch += 1
        N.check(N.lib.ghx_signal_barrier(self.table.ctypes.data_as(C.POINTER(C.c_void_p)), self.ctx.rank,
                                         self.ctx.nranks, C.c_uint64(self.epoch), C.c_void_p(stream)))


_psync: dict = {}


def _process_sync(ctx) -> _ProcessSync:
    key = (ctx.nranks, ctx.device)
    s = _psync.get(key)
    if s is None:
        s = _psync[key] = _ProcessSync(ctx)
    return s


def _sync_mode(ctx) -> str:
    """'device' (flag barrier kernels, no host round trip) when every rank
    owns its own GPU; 'host' when ranks share a device (they cannot spin-wait
    on each other) or GHX_SYNC=host."""
    m = os.environ.get("GHX_SYNC")
    if m in ("host", "device"):
        return m
    devs = getattr(ctx, "_devs", None)
    if devs is None:
        devs = ctx._devs = ctx.allgather((os.uname().nodename, ctx.device))
    return "device" if len(set(devs)) == len(devs) else "host"


def _ipc_peers(ctx, mf: MultiFab):
    """(indices, pointers) of every rank's fabs of ``mf``'s layout, mapped
    into this process with CUDA IPC (cached on the MultiFab)."""
    cache = mf._peer_cache.get("ipc")
    if cache is not None:
        return cache
    h = (C.c_uint8 * 64)()
    have = mf._slab is not None
    base = 0
    if have:
        N.check(N.lib.ghx_ipc_get_handle(C.c_void_p(mf._slab.ptr), h))
        # the handle maps the whole allocation (an arena slab may hold this
        # MultiFab's storage at an offset)
        o = C.c_uint64()
        N.check(N.lib.ghx_alloc_offset(C.c_void_p(mf._slab.ptr), C.byref(o)))
        base = mf._slab.ptr - o.value
    offs = [int(p) - base for p in mf._ptrs] if have else []
    infos = ctx.allgather((ctx.rank, bytes(h) if have else None, mf.local_indices, offs))
    parts, opened = [], []
    for (r, hb, idx, off) in infos:
        if r == ctx.rank:
            parts.append((mf.local_indices, mf._ptrs))
            continue
        if hb is None:
            continue
        pv = _ipc_open(mf.device, hb)
        opened.append(pv)
        parts.append((idx, np.asarray([pv + o for o in off], np.uint64)))
    mf._peer_cache["ipc"] = parts
    weakref.finalize(mf, _close_ipc, list(opened))
    return parts


def _close_ipc(ptrs):
    for p in ptrs:
        try:
            N.lib.ghx_ipc_close_handle(C.c_void_p(p))
        except Exception:
            pass


class Exchange:
    """A prepared FillBoundary / ParallelCopy for this rank: the compiled
    executor(s), the pointer table and the synchronisation it needs.

    ``enqueue(stream)`` puts the whole exchange on a CUDA stream without a
    host round trip (serial; process mode with device barriers; NCCL
    fallback) -- the FillBoundary_nowait analogue.  ``run()`` is the
    synchronous reference contract (data in place, messages accounted)."""

    def __init__(self, plan: CommPlan, src_mf: MultiFab, dst_mf: MultiFab, scomp: int, dcomp: int,
                 ncomp: int, ctx):
        if src_mf.dtype != dst_mf.dtype:
            raise ValueError("source and destination MultiFabs must share the real type")
        # a cached exchange lives on dst and must not keep a distinct source
        # alive (exchange_for evicts it when the source is collected)
        self._src = src_mf if src_mf is dst_mf else weakref.ref(src_mf)
        self.plan, self.dst, self.ctx = plan, dst_mf, ctx
        self.scomp, self.dcomp, self.ncomp = scomp, dcomp, ncomp
        self.item = dst_mf.dtype.itemsize
        self.device = dst_mf.device
        me = ctx.rank
        self.mode = "serial" if ctx.nranks == 1 else ctx.kind
        self.transport = "p2p"
        host = _host_resident(src_mf) or _host_resident(dst_mf)
        if self.mode == "process":
            self.transport = _transport(ctx)
            self.sync = _sync_mode(ctx) if self.transport == "p2p" else "stream"
        else:
            self.sync = "host" if self.mode == "thread" else "none"
        self.remote = "direct"
        self.unp = None
        self.one_kernel = False
        if self.transport == "nccl":
            self._init_nccl()
        elif self.mode == "process" and host:
            # fabs in pinned host memory cannot be CUDA-IPC mapped by the
            # peers: every remote tag is packed by the sender's kernel (reading
            # its host fabs over PCIe) straight into the peer's IPC-mapped
            # DEVICE receive slab; the receiver unpacks into its host fabs
            self.remote = "packed_all"
            self._init_packed(all_remote=True)
        elif self.mode == "process" and os.environ.get("GHX_REMOTE", "packed") == "packed":
            self.remote = "packed"
            self._init_packed()
        else:
            self.ex = plan.executor(me, N.EXEC_DIRECT, src_mf, dst_mf, scomp, dcomp, ncomp)
            if self.mode == "serial":
                self.table = _table(self.ex, src_mf, [(dst_mf.local_indices, dst_mf._ptrs)])
            elif self.mode == "process":
                self.table = _table(self.ex, src_mf, _ipc_peers(ctx, dst_mf))
                if self.sync == "device":
                    self.psync = _process_sync(ctx)
            else:
                self.table = None  # thread ranks: gathered per call
        self._thread_bindings: dict = {}
        self._pin()
        self._init_fused_sync()
        ex0 = getattr(self, "ex", None)
        self._phased = bool(ex0 is not None and ex0.detail.get("phased"))
        row = plan.pair_cells[me]
        self.messages = [(me, d, int(row[d]) * ncomp * self.item) for d in range(plan.nranks)
                         if d != me and row[d] > 0]
        # bytes moved by this rank's launch (local + pushed), read + write
        self.local_cells = int(row[me])
        self.remote_cells = int(sum(row[d] for d in range(plan.nranks) if d != me))
        self.ghost_bytes = int(plan.pair_cells.sum()) * ncomp * self.item  # whole job, counted once

    def _bind_thread(self, gen, infos, stream: int) -> "Binding":
        for (_, d, _, _) in infos:
            if d != self.device and (self.device, d) not in _peer_enabled:
                N.check(N.lib.ghx_enable_peer_access(self.device, d))
                _peer_enabled.add((self.device, d))
        table = _table(self.ex, self.src, [(idx, ptrs) for (_, _, idx, ptrs) in infos])
        if len(self._thread_bindings) >= 4:  # bounded: drop the oldest generation
            self._thread_bindings.pop(next(iter(self._thread_bindings)))
        b = self._thread_bindings[gen] = self.ex.bind(table, stream)
        return b

    def _init_fused_sync(self) -> None:
        """Device-sync process mode: the copy kernel itself waits for each
        destination peer's READY and signals DONE; the unpack (or a DONE
        wait) closes the exchange -- no standalone barrier kernels
        (GHX_FUSED_SYNC=0 restores barrier -> push -> barrier -> unpack)."""
        self.fused = (self.mode == "process" and self.sync == "device" and self.transport == "p2p"
                      and os.environ.get("GHX_FUSED_SYNC", "1") != "0")
        if not self.fused:
            return
        ps = self.psync
        self.ex.set_sync(ps.table, self.ctx.rank, self.ctx.nranks)
        if self.unp is not None:
            self.unp.set_sync(ps.table, self.ctx.rank, self.ctx.nranks)

    def _pin(self) -> None:
        """Pin every pointer table this exchange launches with (once)."""
        if self.transport == "nccl":
            self.b_pack = self.pack.bind(self.t_pack)
            self.b_local = self.local.bind(self.t_local)
            self.b_unpack = self.unpack.bind(self.t_unpack)
            return
        if self.table is not None:
            self.b_ex = self.ex.bind(self.table)
        if self.unp is not None:
            self.b_unp = self.unp.bind(self.t_unp)

    @property
    def src(self) -> MultiFab:
        s = self._src if not isinstance(self._src, weakref.ref) else self._src()
        if s is None:
            raise RuntimeError("the source MultiFab of this exchange has been released")
        return s

    # -- packed push (process mode) ---------------------------------------
    def _init_packed(self, all_remote=False):
        """Narrow-row remote tags (every remote tag with ``all_remote``) are
        packed by the sending kernel straight into the receiver's
        CUDA-IPC-mapped receive slab (contiguous NVLink stores); the receiver
        unpacks locally after the exit barrier.  Wide rows, and all local
        tags, are stored directly into the fabs."""
        plan, src_mf, dst_mf, ctx, me = self.plan, self.src, self.dst, self.ctx, self.ctx.rank
        a = (self.scomp, self.dcomp, self.ncomp)
        # with the in-kernel device sync, pushes and unpacks run as ONE
        # executor and launch (GHX_EXEC_EXCHANGE_PACKED): each peer's DONE is
        # released when this rank's pushes to it are done, and the slabs that
        # land early are unpacked while later pushes are in flight
        # (GHX_ONE_KERNEL=0: push kernel, then unpack kernel)
        self.one_kernel = (not all_remote and self.sync == "device" and plan.nranks <= 32
                           and os.environ.get("GHX_FUSED_SYNC", "1") != "0"
                           and os.environ.get("GHX_ONE_KERNEL", "1") != "0")
        if self.one_kernel:
            self.ex = plan.executor(me, N.EXEC_EXCHANGE_PACKED, src_mf, dst_mf, *a)
            self.unp = None
            recv_el = self.ex.recv_elems
        else:
            kp, ku = ((N.EXEC_PUSH_PACKED_ALL, N.EXEC_UNPACK_PACKED_ALL) if all_remote
                      else (N.EXEC_PUSH_PACKED, N.EXEC_UNPACK_PACKED))
            self.ex = plan.executor(me, kp, src_mf, dst_mf, *a)
            self.unp = plan.executor(me, ku, src_mf, dst_mf, *a)
            recv_el = self.unp.buffer_elems
        item, n = self.item, plan.nranks
        offs, total = [], 0
        for r in range(n):
            offs.append(total)
            total += -(-int(recv_el[r]) * item // 256) * 256
        self._recv = Slab(max(256, total), dst_mf.device)
        h = (C.c_uint8 * 64)()
        N.check(N.lib.ghx_ipc_get_handle(C.c_void_p(self._recv.ptr), h))
        infos = ctx.allgather((me, bytes(h), offs, self.ex.buffer_elems.tolist(), recv_el.tolist()))
        for (s_, _, _, send_el, _) in infos:
            for (d_, _, _, _, rcv) in infos:
                if s_ != d_ and send_el[d_] != rcv[s_]:
                    raise RuntimeError(f"packed-push buffer mismatch {s_}->{d_}: {send_el[d_]} vs {rcv[s_]}")
        send = np.zeros(n, np.uint64)
        self._opened = []
        for (r, hb, roffs, _, _) in infos:
            if r == me or self.ex.buffer_elems[r] == 0:
                continue
            pv = _ipc_open(dst_mf.device, hb)
            self._opened.append(pv)
            send[r] = pv + roffs[me]
        recv = np.asarray([self._recv.ptr + o for o in offs], np.uint64)
        bufs = np.concatenate([send, recv])
        # with every remote tag packed, only this rank's own fabs are addressed
        parts = [(dst_mf.local_indices, dst_mf._ptrs)] if all_remote else _ipc_peers(ctx, dst_mf)
        self.table = _table(self.ex, src_mf, parts, bufs)
        if self.unp is not None:
            self.t_unp = _table(self.unp, src_mf, [(dst_mf.local_indices, dst_mf._ptrs)], bufs)
        weakref.finalize(self, _close_ipc, list(self._opened))
        if self.sync == "device":
            self.psync = _process_sync(ctx)

    # -- NCCL fallback ---------------------------------------------------
    def _init_nccl(self):
        plan, src_mf, dst_mf, me = self.plan, self.src, self.dst, self.ctx.rank
        a = (self.scomp, self.dcomp, self.ncomp)
        self.pack = plan.executor(me, N.EXEC_PACK, src_mf, dst_mf, *a)
        self.unpack = plan.executor(me, N.EXEC_UNPACK, src_mf, dst_mf, *a)
        self.local = plan.executor(me, N.EXEC_LOCAL, src_mf, dst_mf, *a)
        item, n = self.item, plan.nranks
        send_el, recv_el = self.pack.buffer_elems, self.unpack.buffer_elems
        self._slabs = (Slab(max(256, int(send_el.sum()) * item + 256 * n), dst_mf.device),
                       Slab(max(256, int(recv_el.sum()) * item + 256 * n), dst_mf.device))
        ts, tr = (sl.tensor(dst_mf.dtype) for sl in self._slabs)
        sbufs, rbufs = np.zeros(n, np.uint64), np.zeros(n, np.uint64)
        self.send_t, self.recv_t = {}, {}
        off_s = off_r = 0
        for r in range(n):
            if send_el[r]:
                sbufs[r] = self._slabs[0].ptr + off_s * item
                self.send_t[r] = ts[off_s:off_s + int(send_el[r])]
                off_s += -(-int(send_el[r]) * item // 256) * 256 // item
            if recv_el[r]:
                rbufs[r] = self._slabs[1].ptr + off_r * item
                self.recv_t[r] = tr[off_r:off_r + int(recv_el[r])]
                off_r += -(-int(recv_el[r]) * item // 256) * 256 // item
        bufs = np.concatenate([sbufs, rbufs])
        own = [(dst_mf.local_indices, dst_mf._ptrs)]
        self.t_pack = _table(self.pack, src_mf, own, bufs)
        self.t_unpack = _table(self.unpack, src_mf, own, bufs)
        self.t_local = _table(self.local, src_mf, own, bufs)

    def _enqueue_nccl(self, stream: int) -> None:
        # torch.distributed orders NCCL work (and gloo's host staging) against
        # torch's CURRENT stream: make ``stream`` current for the whole
        # sequence so the sends follow the pack and the unpack follows the
        # receives on the caller's stream
        with torch_stream(stream, self.device) as ts:
            self._enqueue_nccl_current(stream, ts)

    def _enqueue_nccl_current(self, stream: int, ts) -> None:
        import torch
        import torch.distributed as dist
        self.b_pack.run(stream)
        if dist.get_backend() != "nccl":
            # host-staged message passing (gloo): test path for ranks sharing a GPU
            ts.synchronize()
            send = {r: t.cpu() for r, t in self.send_t.items()}
            recv = {r: torch.empty(t.shape, dtype=t.dtype) for r, t in self.recv_t.items()}
            ops = [dist.P2POp(dist.isend, t, r) for r, t in sorted(send.items())]
            ops += [dist.P2POp(dist.irecv, t, r) for r, t in sorted(recv.items())]
            for q in (dist.batch_isend_irecv(ops) if ops else []):
                q.wait()
            for r, t in recv.items():
                self.recv_t[r].copy_(t)
            self.b_local.run(stream)
            self.b_unpack.run(stream)
            return
        ops = [dist.P2POp(dist.isend, t, r) for r, t in sorted(self.send_t.items())]
        ops += [dist.P2POp(dist.irecv, t, r) for r, t in sorted(self.recv_t.items())]
        reqs = dist.batch_isend_irecv(ops) if ops else []
        self.b_local.run(stream)
        for q in reqs:
            q.wait()  # NCCL: the current stream waits, the host does not
        self.b_unpack.run(stream)

    # -- launching ---------------------------------------------------------
    @property
    def launches_per_call(self) -> int:
        if self.transport == "nccl":
            return 3
        return 2 if self.remote in ("packed", "packed_all") and not self.one_kernel else 1

    def enqueue(self, stream: int, marks=None) -> None:
        """Put the exchange on ``stream``.  ``marks`` (diagnostics): three
        callables run between the launches of a device-synced process-mode
        exchange (e.g. CUDA event records on ``stream``) -- before the push
        kernel, after it, after the unpack / DONE wait."""
        if self.transport == "nccl":
            self._enqueue_nccl(stream)
        elif self.mode == "serial":
            self.b_ex.run(stream)
        elif self.mode == "process" and self.sync == "device" and self.fused:
            e = self.psync.next_epoch()
            if marks:
                marks[0]()
            self.b_ex.run_synced(stream, e)  # pushes wait per peer for READY, then signal DONE
            if marks:
                marks[1]()
            if self.unp is not None:
                self.b_unp.run_synced(stream, e)  # each peer's slab unpacked once its DONE lands
            elif not self.one_kernel:
                self.ex.sync_wait(e, stream)  # every push into my fabs has landed
            # (one kernel: its unpack tasks waited for each source's DONE and
            # its CTA 0 for every peer's before the launch completes)
            if marks:
                marks[2]()
        elif self.mode == "process" and self.sync == "device":
            self.psync.barrier(stream)  # peers finished earlier work on their fabs
            self.b_ex.run(stream)
            self.psync.barrier(stream)  # every push into my fabs has landed
            if self.unp is not None:
                self.b_unp.run(stream)
        else:
            raise RuntimeError(f"{self.mode} ranks with host synchronisation cannot enqueue; use run()")

    def run(self) -> None:
        stream = _stream(self.device)
        ctx = self.ctx
        if self.mode == "thread":
            stream.synchronize()  # my earlier work on my fabs is done
            # the peers' destination MultiFabs of this call (one object per
            # rank); their fab pointers are fixed for a MultiFab's life, so the
            # bound pointer table is cached per tuple of MultiFab uids
            infos = ctx.allgather((self.dst.uid, self.dst.device, self.dst.local_indices, self.dst._ptrs))
            gen = tuple(i[0] for i in infos)
            b = self._thread_bindings.get(gen)
            if b is None:
                b = self._bind_thread(gen, infos, stream.cuda_stream)
            b.run(stream.cuda_stream)
            stream.synchronize()
        elif self.mode == "process" and self.sync == "host":
            stream.synchronize()
            ctx.barrier()
            self.b_ex.run(stream.cuda_stream)
            stream.synchronize()
            ctx.barrier()
            if self.unp is not None:
                self.b_unp.run(stream.cuda_stream)
                stream.synchronize()
        else:
            self.enqueue(stream.cuda_stream)
            stream.synchronize()
            if (self.mode == "process" and self.sync == "device") or self._phased:
                check_barriers()  # in-kernel waits are bounded: a timeout means an incomplete result
        for (s, d, nbytes) in self.messages:
            ctx.bus.account(s, d, nbytes)


_barrier_timeouts_seen = 0


def check_barriers() -> None:
    """Raise if a device barrier timed out (a peer rank never arrived)."""
    global _barrier_timeouts_seen
    n = int(N.lib.ghx_barrier_timeouts())
    if n > _barrier_timeouts_seen:
        _barrier_timeouts_seen = n
        raise N.GhostxError("device barrier timed out: a peer rank did not arrive "
                            "(GHX_BARRIER_TIMEOUT_S); the exchange result is incomplete")


def exchange_for(plan: CommPlan, src_mf: MultiFab, dst_mf: MultiFab, scomp: int, dcomp: int, ncomp: int,
                 ctx=None) -> Exchange:
    for m in (src_mf, dst_mf):
        if hasattr(m, "check_open"):
            m.check_open()
    ctx = ctx or current_ctx()
    key = ("xchg", plan.uid, src_mf.uid, scomp, dcomp, ncomp, ctx.kind, ctx.nranks,
           _transport(ctx) if ctx.kind == "process" else None)
    ex = dst_mf._peer_cache.get(key)
    if ex is None:
        ex = cache_put(dst_mf, key, Exchange(plan, src_mf, dst_mf, scomp, dcomp, ncomp, ctx), src_mf)
    return ex


def cache_put(owner, key, value, *deps):
    """``owner._peer_cache[key] = value``, dropped again when any of ``deps``
    (other MultiFabs the entry was built for) is garbage-collected, so a
    long-lived MultiFab does not accumulate executors, device tables or
    staging slabs for partners that no longer exist."""
    owner._peer_cache[key] = value
    oref = weakref.ref(owner)
    for d in deps:
        if d is not None and d is not owner:
            weakref.finalize(d, _cache_drop, oref, key)
    return value


def _cache_drop(oref, key) -> None:
    o = oref()
    if o is not None:
        o._peer_cache.pop(key, None)


def _execute_plan(plan: CommPlan, src_mf: MultiFab, dst_mf: MultiFab, scomp: int, dcomp: int,
                  ncomp: int, ctx, backend=None) -> None:
    """Run ``plan`` for this rank (reference comm.py:316-380) on the current
    torch stream of the MultiFab's device; returns when the data is in
    place (the reference API is synchronous).  ``backend`` is accepted for
    signature compatibility only: there is one execution path, the fused
    CUDA kernel; a reference-style backend object (kernels.Backend) gets
    this call's device launches added to its ``launch_counter``."""
    ex = exchange_for(plan, src_mf, dst_mf, scomp, dcomp, ncomp, ctx)
    ex.run()
    if backend is not None and hasattr(backend, "launch_counter"):
        bump = getattr(backend, "_bump", None)
        if bump is not None:
            bump(ex.launches_per_call)
        else:
            backend.launch_counter += ex.launches_per_call


def prepare_fill_boundary(mf: MultiFab, geom: Geometry | None = None) -> Exchange:
    """Plan + compile the FillBoundary of ``mf`` once; the returned
    Exchange can be enqueued on a stream repeatedly (FillBoundary_nowait)."""
    plan = plan_build_fill_boundary(mf, geom)
    return exchange_for(plan, mf, mf, 0, 0, mf.ncomp)


def prepare_parallel_copy(dst: MultiFab, src: MultiFab, scomp: int = 0, dcomp: int = 0, ncomp=None,
                          ngrow_src=0, ngrow_dst=0, geom: Geometry | None = None) -> Exchange:
    ncomp, gs, gd = _pc_args(dst, src, scomp, dcomp, ncomp, ngrow_src, ngrow_dst)
    plan = _parallel_copy_plan(dst, src, gs, gd, geom)
    return exchange_for(plan, src, dst, scomp, dcomp, ncomp)


# --------------------------------------------------------------- public entry

def _raw_stream_fn():
    import torch
    f = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    return f if f is not None else (lambda dev: torch.cuda.current_stream(dev).cuda_stream)


_raw_stream = None


def _dist_initialized() -> bool:
    d = sys.modules.get("torch.distributed")
    return d is not None and d.is_available() and d.is_initialized()


def _plan_key_of(mf: MultiFab, plan) -> object:
    for k, v in mf.plan_cache.items():
        if v is plan:
            return k
    return None


def _fill_boundary_serial_fast(mf: MultiFab, geom, backend) -> bool:
    """Repeat call of a single-rank FillBoundary: one bound launch and one
    stream synchronize, no plan lookup or Python object churn (the first
    call took the full path and left ``mf._fb_fast``).  False = take the
    full path."""
    fast = getattr(mf, "_fb_fast", None)
    if fast is None or backend is not None or geom is not fast[0]:
        return False
    if getattr(_tls, "ctx", None) is not None or _dist_initialized() or mf.plan_cache.get(fast[2]) is not fast[3]:
        return False
    h, bid, dev = fast[1].ex._h, fast[1].id, mf.device
    if not h:
        return False
    st = _raw_stream(dev)
    rc = N.lib.ghx_exec_run_bound(h, bid, C.c_void_p(st))
    if rc == 0:
        rc = N.lib.ghx_stream_sync(C.c_void_p(st))
    N.check(rc)
    if fast[4]:
        check_barriers()
    return True


def fill_boundary(mf: MultiFab, geom: Geometry | None = None, backend=None) -> None:
    """Fill every coverable ghost cell of ``mf`` from (periodically shifted)
    valid data.  Collective over ranks; at most one message per ordered rank
    pair; physical-boundary ghosts with no source and all valid cells are
    left untouched (reference comm.py:383-394)."""
    if _fill_boundary_serial_fast(mf, geom, backend):
        return
    plan = plan_build_fill_boundary(mf, geom)
    if plan.is_empty:
        return
    ctx = current_ctx()
    _execute_plan(plan, mf, mf, 0, 0, mf.ncomp, ctx, backend)
    ctx.barrier()
    if ctx is _serial_ctx:
        ex = exchange_for(plan, mf, mf, 0, 0, mf.ncomp, ctx)
        if ex.mode == "serial" and ex.transport == "p2p" and getattr(ex, "b_ex", None) is not None:
            global _raw_stream
            if _raw_stream is None:
                _raw_stream = _raw_stream_fn()
            # the geometry object this plan was built for (None = mf.geom)
            mf._fb_fast = (geom, ex.b_ex, _plan_key_of(mf, plan), plan, ex._phased)


def _pc_args(dst, src, scomp, dcomp, ncomp, ngrow_src, ngrow_dst):
    if src.ba.ixtype != dst.ba.ixtype:
        raise ValueError("parallel_copy requires matching index types")
    ncomp = ncomp if ncomp is not None else min(src.ncomp - scomp, dst.ncomp - dcomp)
    if scomp < 0 or scomp + ncomp > src.ncomp or dcomp < 0 or dcomp + ncomp > dst.ncomp or ncomp < 1:
        raise ValueError(f"component range out of bounds: scomp={scomp} dcomp={dcomp} ncomp={ncomp}")
    gs = ngrow_src if isinstance(ngrow_src, IntVect) else IntVect.filled(ngrow_src)
    gd = ngrow_dst if isinstance(ngrow_dst, IntVect) else IntVect.filled(ngrow_dst)
    return ncomp, gs, gd


def parallel_copy(dst: MultiFab, src: MultiFab, scomp: int = 0, dcomp: int = 0, ncomp: int | None = None,
                  ngrow_src=0, ngrow_dst=0, geom: Geometry | None = None, backend=None) -> None:
    """Copy src's (grown) valid data into every overlapping cell of dst's
    (grown) boxes; periodic images only with ``geom`` (comm.py:397-429)."""
    ncomp, gs, gd = _pc_args(dst, src, scomp, dcomp, ncomp, ngrow_src, ngrow_dst)
    plan = _parallel_copy_plan(dst, src, gs, gd, geom)
    if plan.is_empty:
        return
    ctx = current_ctx()
    _execute_plan(plan, src, dst, scomp, dcomp, ncomp, ctx, backend)
    ctx.barrier()


# ------------------------------------------------------------------ gathers

class _FabSet:
    """The private destination fabs of a gather (comm.py:432-462), laid out
    like a MultiFab for the exchange engine: position p of the global
    dst_fabs list is dst slot p; this rank's positions live in one slab (so
    process-mode peers can map it with CUDA IPC)."""

    def __init__(self, boxes: list, ranks: list, ncomp: int, dtype, device: int, rank: int, dim: int):
        from .mesh import _ALIGN, Slab, Fab, _next_uid
        self.ncomp = int(ncomp)
        self.dtype = dtype
        self.device = int(device)
        self.ngrow = IntVect(*([0] * dim))
        self.uid = _next_uid()
        self._peer_cache: dict = {}
        self._rows = np.ascontiguousarray(np.asarray([b.as_row() for b in boxes], np.int64).reshape(-1, 6))
        self.local_indices = tuple(p for p, r in enumerate(ranks) if r == rank)
        item = np.dtype(dtype).itemsize
        offs, total = {}, 0
        for p in self.local_indices:
            offs[p] = total // item
            total += -(-boxes[p].num_pts * self.ncomp * item // _ALIGN) * _ALIGN
        self._slab = Slab(max(total, 256), self.device) if self.local_indices else None
        if self._slab is not None and config.debug:  # fresh fabs are poisoned, like Fab()
            N.check(N.lib.ghx_memset_u64(C.c_void_p(self._slab.ptr), config.poison_word64(item),
                                         -(-total // 8), None))
        self.fabs = {p: Fab(boxes[p], self.ncomp, _slab=self._slab, _offset=offs[p]) for p in self.local_indices}
        self._ptrs = np.array([self.fabs[p].ptr for p in self.local_indices], np.uint64)

    def storage_rows(self) -> np.ndarray:
        return self._rows


def build_gather_plan(dst_fabs: list, dst_ranks: list, src: MultiFab, geom: Geometry | None = None) -> CommPlan:
    """Plan a collective gather of src valid data into private target fabs
    (reference comm.py:432-443): every (fab_id, box) of ``dst_fabs`` (the
    same list on every rank; boxes may overlap) receives the overlapping
    valid cells of src, periodic images included when ``geom`` is given."""
    boxes = [b for _, b in dst_fabs]
    nranks = max(src.dm.nranks, max(dst_ranks, default=0) + 1)
    if not boxes:
        h = C.c_void_p()
        rows = np.zeros((0, 6), np.int64)
        N.check(N.lib.ghx_plan_build_parallel_copy(0, N.i64p(rows), N.i64p(np.zeros(3, np.int64)), len(src.ba),
                                                   N.i64p(src.ba.rows()), N.i64p(np.zeros(3, np.int64)), None, None,
                                                   N.i32p(src.dm.array()), N.i32p(np.zeros(0, np.int32)), nranks,
                                                   C.byref(h)))
        return CommPlan(h.value, nranks, len(src.ngrow), src.ba.ixtype)
    rows = np.ascontiguousarray(np.asarray([b.as_row() for b in boxes], np.int64))
    per = period = None
    if geom is not None:
        per = np.zeros(3, np.int32)
        per[:len(geom.periodic)] = geom.periodic
        period = np.ones(3, np.int64)
        period[:len(geom.period)] = geom.period
    zero = np.zeros(3, np.int64)
    h = C.c_void_p()
    N.check(N.lib.ghx_plan_build_parallel_copy(
        len(boxes), N.i64p(rows), N.i64p(zero), len(src.ba), N.i64p(src.ba.rows()), N.i64p(zero.copy()),
        N.i32p(per) if per is not None else None, N.i64p(period) if period is not None else None,
        N.i32p(src.dm.array()), N.i32p(np.asarray(dst_ranks, np.int32)), nranks, C.byref(h)))
    return CommPlan(h.value, nranks, len(src.ngrow), src.ba.ixtype)


def _drop_plan_entry(pref, key) -> None:
    p = pref()
    if p is not None:
        p._execs.pop(key, None)


def _gather_set(plan: CommPlan, dst_fabs: list, dst_ranks: list, src: MultiFab) -> _FabSet:
    ctx = current_ctx()
    key = ("gather_set", src.uid, ctx.rank, src.ncomp)
    fs = plan._execs.get(key)
    if fs is None:
        fs = plan._execs[key] = _FabSet([b for _, b in dst_fabs], list(dst_ranks), src.ncomp, src.dtype,
                                        src.device, ctx.rank, len(src.ngrow))
        # the target slab goes with its source; the finalizer holds the plan
        # only weakly, so a plan built per call (gather_fabs(plan=None)) and its
        # slab are freed when the caller drops it
        weakref.finalize(src, _drop_plan_entry, weakref.ref(plan), key)
    return fs


def gather_fabs(dst_fabs: list, dst_ranks: list, owned: dict, src: MultiFab, geom: Geometry | None = None,
                backend=None, plan: CommPlan | None = None) -> None:
    """Collective gather of src valid data into caller-private fabs
    (reference comm.py:446-462).  ``owned`` maps this rank's fab ids to
    destination Fabs over exactly their dst_fabs boxes.  The exchange lands
    in a plan-cached device slab (one fused launch, peers write it directly
    in process mode), then each owned Fab receives its target region with
    one device copy; pass the plan's own fabs (``gather_targets``) to skip
    that copy."""
    if plan is None:
        plan = build_gather_plan(dst_fabs, dst_ranks, src, geom)
    if plan.is_empty:
        return
    fs = _gather_set(plan, dst_fabs, dst_ranks, src)
    ctx = current_ctx()
    _execute_plan(plan, src, fs, 0, 0, src.ncomp, ctx, backend)
    pos_of = {fid: pos for pos, (fid, _) in enumerate(dst_fabs)}
    for fid, fab in owned.items():
        mine = fs.fabs.get(pos_of[fid])
        if mine is None:
            raise ValueError(f"gather_fabs: fab {fid} is not a target of rank {ctx.rank}")
        if fab.data is not mine.data:
            if fab.box != mine.box or fab.ncomp != mine.ncomp:
                raise ValueError(f"gather_fabs: owned fab {fid} does not match its target box {mine.box}")
            fab.data.copy_(mine.data)
    ctx.barrier()


def gather_targets(plan: CommPlan, dst_fabs: list, dst_ranks: list, src: MultiFab) -> dict:
    """This rank's plan-cached gather destination fabs, by fab id (fill_patch
    gathers straight into them)."""
    fs = _gather_set(plan, dst_fabs, dst_ranks, src)
    return {fid: fs.fabs[pos] for pos, (fid, _) in enumerate(dst_fabs) if pos in fs.fabs}



# ---------------------------------------------------------- index-mapped copy

def _box_cells(box: Box):
    """Global (i, j, k) int64 arrays of the box's cells in F order, padded to
    3-D (kernels.py:159-171)."""
    from .mesh import _pad3
    ex, ey, ez = _pad3(box.extents, 1)
    lo = _pad3(box.lo, 0)
    flat = np.arange(ex * ey * ez, dtype=np.int64)
    return flat % ex + lo[0], (flat // ex) % ey + lo[1], flat // (ex * ey) + lo[2]


def index_mapped_copy(dst: MultiFab, src: MultiFab, mapping_fn, region: Box | None = None, backend=None) -> None:
    """dst(cell) = src(mapping_fn(cell)) over dst's valid cells (reference
    comm.py:465-560).  ``mapping_fn`` takes (i, j, k) int64 arrays and returns
    the mapped (i, j, k); every mapped point must lie in a src valid box
    (the first one in BoxArray order wins), else ValueError.  The mapping is
    evaluated on the host, redundantly on every rank (it is user Python);
    each rank then pushes the cells it owns the sources of -- local and
    remote destinations alike -- with one gather/scatter launch, and the
    per-ordered-pair message accounting follows the reference."""
    import torch
    from .index_space import intersect
    from .mesh import _pad3
    if src.ba.ixtype != dst.ba.ixtype:
        raise ValueError("index_mapped_copy requires matching index types")
    if src.ncomp != dst.ncomp:
        raise ValueError("index_mapped_copy requires matching component counts")
    if src.dtype != dst.dtype:
        raise ValueError("index_mapped_copy requires matching real types")
    ctx = current_ctx()
    me = ctx.rank
    slo = np.asarray([_pad3(b.lo, 0) for b in src.ba], np.int64).reshape(-1, 3)
    shi = np.asarray([_pad3(b.hi, 0) for b in src.ba], np.int64).reshape(-1, 3)
    jobs = []  # (src fab, dst fab, mapped coords, dst coords) with src rank == me
    pair_cells: dict = {}
    for dj, dbox in enumerate(dst.ba):
        work = dbox if region is None else intersect(dbox, region)
        if work.is_empty:
            continue
        di, dy, dk = _box_cells(work)
        mi, mj, mk = (np.asarray(v, dtype=np.int64) for v in mapping_fn(di, dy, dk))
        owner = np.full(di.size, -1, np.int64)
        for si in range(len(src.ba)):
            m = ((mi >= slo[si, 0]) & (mi <= shi[si, 0]) & (mj >= slo[si, 1]) & (mj <= shi[si, 1])
                 & (mk >= slo[si, 2]) & (mk <= shi[si, 2]) & (owner < 0))
            owner[m] = si
        if (owner < 0).any():
            raise ValueError(f"mapping leaves {int((owner < 0).sum())} cells of dst fab {dj} outside src coverage")
        dr = dst.dm[dj]
        for si in np.unique(owner):
            sr = src.dm[int(si)]
            m = owner == si
            pair_cells[(sr, dr)] = pair_cells.get((sr, dr), 0) + int(m.sum())
            if sr == me:
                jobs.append((int(si), dj, (mi[m], mj[m], mk[m]), (di[m], dy[m], dk[m])))
    # destination pointers of every rank's fabs
    if ctx.nranks == 1:
        dptr = dict(zip(dst.local_indices, (int(p) for p in dst._ptrs)))
    elif ctx.kind == "process":
        dptr = {}
        for idx, ptrs in _ipc_peers(ctx, dst):
            dptr.update(zip(idx, (int(p) for p in ptrs)))
    else:
        torch.cuda.current_stream(dst.device).synchronize()  # peers may still work on their fabs
        dptr = {}
        for (_, d, idx, ptrs) in ctx.allgather((me, dst.device, dst.local_indices, dst._ptrs)):
            if d != dst.device and (dst.device, d) not in _peer_enabled:
                N.check(N.lib.ghx_enable_peer_access(dst.device, d))
                _peer_enabled.add((dst.device, d))
            dptr.update(zip(idx, (int(p) for p in ptrs)))
    if ctx.kind == "process" and ctx.nranks > 1:
        torch.cuda.current_stream(dst.device).synchronize()
        ctx.barrier()  # peers finished earlier work on the fabs this rank writes
    item = dst.dtype.itemsize
    rows = []
    for si, dj, (mi, mj, mk), (di, dy, dk) in jobs:
        sf = src.fabs[si]
        sb_lo, sn = _pad3(sf.box.lo, 0), _pad3(sf.box.extents, 1)
        db = grow(dst.ba[dj], dst.ngrow)
        db_lo, dn = _pad3(db.lo, 0), _pad3(db.extents, 1)
        soff = (mi - sb_lo[0]) + sn[0] * ((mj - sb_lo[1]) + sn[1] * (mk - sb_lo[2]))
        doff = (di - db_lo[0]) + dn[0] * ((dy - db_lo[1]) + dn[1] * (dk - db_lo[2]))
        r = np.empty((soff.size, 4), np.int64)
        r[:, 0] = np.uint64(sf.ptr).view(np.int64) + soff * item
        r[:, 1] = np.uint64(dptr[dj]).view(np.int64) + doff * item
        r[:, 2] = sn[0] * sn[1] * sn[2] * item
        r[:, 3] = dn[0] * dn[1] * dn[2] * item
        rows.append(r)
    stream = torch.cuda.current_stream(src.device)
    if rows:
        table = torch.from_numpy(np.ascontiguousarray(np.concatenate(rows))).to(f"cuda:{src.device}")
        N.check(N.lib.ghx_index_copy(C.c_void_p(table.data_ptr()), table.shape[0], src.ncomp, item,
                                     C.c_void_p(stream.cuda_stream)))
    stream.synchronize()
    for (sr, dr), cells in sorted(pair_cells.items()):
        if sr == me and dr != me:
            ctx.bus.account(sr, dr, cells * src.ncomp * item)
    ctx.barrier()
