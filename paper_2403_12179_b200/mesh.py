"""Fab / BoxArray / DistributionMapping / MultiFab with fab storage in HBM.

Drop-in for the reference's ``miniamr_core.mesh`` (core/mesh.py:38-325) on
the exchange path.  Differences that follow from living on a B200:

* storage is one device slab per MultiFab (``ghx_device_alloc``), carved
  into 256-byte aligned fabs; each ``Fab.data`` is a zero-copy torch CUDA
  tensor of shape (nx, ny, nz, ncomp) with F-order strides (1, nx, nx*ny,
  nx*ny*nz) -- the same layout law as core/mesh.py:38-58 and
  tests/test_mesh.py:67-80, offset (i-lo0) + ex0*((j-lo1) + ex1*((k-lo2) +
  ex2*c));
* ``memory="pinned"`` puts the slab in mapped, page-locked host memory: the
  same exchange kernel then runs over PCIe on host-resident fabs (used for
  the end-to-end host-buffer measurement);
* ``BoxArray`` disjointness is checked by the native binned sweep instead
  of the O(n^2) pair loop (core/mesh.py:203-205, 126 s at 4,096 boxes).
"""

from __future__ import annotations

import ctypes as C
import itertools
import math
import threading
from typing import Iterable, Iterator, Sequence

import numpy as np

from . import _native as N
from . import config
from .index_space import Box, Geometry, IndexType, IntVect, grow

_uid_lock = threading.Lock()
_uid_iter = itertools.count(1)


def _next_uid() -> int:
    with _uid_lock:
        return next(_uid_iter)


def _pad3(vals: Sequence[int], fill: int) -> tuple:
    v = tuple(int(x) for x in vals)
    return v + (fill,) * (3 - len(v))


def storage_shape(box: Box, ncomp: int) -> tuple:
    """(nx, ny, nz, ncomp), trailing spatial axes of extent 1 below 3-D."""
    return _pad3(box.extents, 1) + (int(ncomp),)


def _torch():
    import torch
    return torch


def _torch_dtype(dt: np.dtype):
    torch = _torch()
    return torch.float64 if np.dtype(dt).itemsize == 8 else torch.float32


def _native_arena(arena):
    """An arena from paper_2403_12179_b200.arena (pooled storage), or None:
    anything else passed as ``arena=`` (the reference's CPU arenas) keeps the
    one-allocation-per-MultiFab default."""
    from . import arena as _arena_mod
    if isinstance(arena, (_arena_mod.Arena, _arena_mod.AsyncArena)):
        return arena
    return None


def _current_device() -> int:
    from . import comm
    return comm.current_ctx().device


class Slab:
    """One native allocation (device HBM or pinned host), freed on GC."""

    def __init__(self, nbytes: int, device: int, memory: str = "device", arena=None):
        if memory not in ("device", "pinned"):
            raise ValueError(f"memory must be 'device' or 'pinned', got {memory!r}")
        self._block = None
        if arena is not None:  # pooled storage (arena.py); 256-B aligned blocks
            if getattr(arena, "memory", None) != memory:
                raise ValueError(f"arena holds {getattr(arena, 'memory', '?')} memory, the MultiFab needs {memory}")
            if memory == "device" and arena.device != int(device):
                raise ValueError(f"arena is on device {arena.device}, the MultiFab on device {device}")
            self._block = arena.alloc(-(-int(nbytes) // 256) * 256, 256)
            self.ptr = self._block.address
        else:
            p = C.c_void_p()
            if memory == "device":
                N.check(N.lib.ghx_device_alloc(int(device), -(-int(nbytes) // 256) * 256, C.byref(p)))
            else:
                N.check(N.lib.ghx_host_alloc(-(-int(nbytes) // 256) * 256, C.byref(p)))
            self.ptr = int(p.value)
        self.nbytes = int(nbytes)
        self.device = int(device)
        self.memory = memory

    @property
    def __cuda_array_interface__(self):
        return {"shape": (self.nbytes,), "typestr": "|u1", "data": (self.ptr, False),
                "version": 3, "strides": None}

    @property
    def __array_interface__(self):
        if self.memory != "pinned":
            raise AttributeError("device slab has no host array interface")
        return {"shape": (self.nbytes,), "typestr": "|u1", "data": (self.ptr, False), "version": 3}

    def tensor(self, dtype):
        """1-D torch tensor over the whole slab (keeps the slab alive)."""
        torch = _torch()
        if self.memory == "device":
            t = torch.as_tensor(self, device=f"cuda:{self.device}")
        else:
            t = torch.from_numpy(np.asarray(self))
        return t.view(_torch_dtype(dtype))

    def __del__(self):
        try:
            if self._block is not None:
                self._block.free()
                self._block = None
                self.ptr = 0
            elif self.ptr:
                (N.lib.ghx_device_free if self.memory == "device" else N.lib.ghx_host_free)(C.c_void_p(self.ptr))
                self.ptr = 0
        except Exception:
            pass


class Fab:
    """Multi-component real array over a Box, F-order, on the device."""

    def __init__(self, box: Box, ncomp: int, arena=None, *, device: int | None = None,
                 memory: str = "device", _slab=None, _offset: int = 0):
        if box.is_empty:
            raise ValueError("cannot create a Fab over an empty box")
        if ncomp < 1:
            raise ValueError(f"ncomp must be >= 1, got {ncomp}")
        self.box = box
        self.ncomp = int(ncomp)
        self.dtype = config.real_dtype
        shape = storage_shape(box, ncomp)
        count = math.prod(shape)
        if _slab is None:
            dev = _current_device() if device is None else int(device)
            _slab = Slab(count * self.dtype.itemsize, dev, memory, arena=_native_arena(arena))
            _offset = 0
            if config.debug:
                N.check(N.lib.ghx_memset_u64(C.c_void_p(_slab.ptr), config.poison_word64(self.dtype.itemsize),
                                             -(-count * self.dtype.itemsize // 8), None))
        self._slab = _slab
        self.device = _slab.device
        self.memory = _slab.memory
        flat = _slab.tensor(self.dtype)
        nx, ny, nz, nc = shape
        self.data = flat.as_strided(shape, (1, nx, nx * ny, nx * ny * nz), _offset)
        self.ptr = _slab.ptr + _offset * self.dtype.itemsize
        self.nbytes = count * self.dtype.itemsize

    @property
    def lo3(self) -> tuple:
        return _pad3(self.box.lo, 0)

    def raw(self):
        """Flat storage in layout order (zero-copy)."""
        return self.data.as_strided((self.data.numel(),), (1,))

    def view(self, writable: bool = True) -> "FabView":
        return FabView(self.data, self.lo3, self.ncomp, writable)

    def setval(self, value: float, region: Box | None = None, comp_range=None) -> None:
        fab_setval(self, value, region, comp_range)

    def release(self) -> None:
        self.data = None
        self._slab = None


def fab_create(box: Box, ncomp: int, arena=None) -> Fab:
    return Fab(box, ncomp, arena)


def _components(spec, ncomp: int) -> slice:
    """None -> all, int c -> [c, c+1), (a, b) -> [a, b); ValueError outside."""
    if spec is None:
        lo, hi = 0, ncomp
    elif isinstance(spec, (int, np.integer)):
        lo, hi = int(spec), int(spec) + 1
        if hi > ncomp or lo < 0:
            raise ValueError(f"component {spec} does not exist (ncomp={ncomp})")
    else:
        lo, hi = (int(v) for v in spec)
        if lo < 0 or hi < lo or hi > ncomp:
            raise ValueError(f"component range {tuple(spec)} not within [0, {ncomp}]")
    return slice(lo, hi)


def _region_slices(fab_box: Box, region: Box) -> tuple:
    """Zero-based (x, y, z) slices of ``region`` inside a fab over ``fab_box``."""
    base = _pad3(fab_box.lo, 0)
    lo, hi = _pad3(region.lo, 0), _pad3(region.hi, 0)
    return tuple(slice(l - o, h - o + 1) for o, l, h in zip(base, lo, hi))


def fab_setval(f: Fab, value: float, region: Box | None = None, comp_range=None) -> None:
    """Assign ``value`` to region x comps of the fab (whole fab by default)."""
    target = f.box if region is None else region
    if target.is_empty:
        return
    if not f.box.contains(target):
        raise ValueError(f"setval: {target} lies outside the fab box {f.box}")
    f.data[_region_slices(f.box, target) + (_components(comp_range, f.ncomp),)] = value


class FabView:
    """Global-index accessor of a fab: view[i, j, k], view[i, j, k, c] or
    spacedim-arity indices; ints give a Python float, integer arrays give a
    tensor (fancy indexing, evaluated on the fab's device)."""

    __slots__ = ("_a", "lo3", "ncomp", "writable")

    def __init__(self, data, lo3: tuple, ncomp: int, writable: bool):
        self._a, self.lo3, self.ncomp, self.writable = data, lo3, ncomp, writable

    @property
    def array(self):
        return self._a

    def _resolve(self, key):
        key = key if isinstance(key, tuple) else (key,)
        if len(key) == 4:
            pos, comp = key[:3], key[3]
        elif len(key) == 3 or len(key) == config.spacedim:
            pos, comp = tuple(key) + (0,) * (3 - len(key)), 0
        else:
            raise IndexError(f"FabView takes (i, j, k[, c]) or {config.spacedim} indices, got {len(key)}")
        scalar = isinstance(comp, (int, np.integer))
        loc = []
        for axis, (g, base) in enumerate(zip(pos, self.lo3)):
            if isinstance(g, (int, np.integer)):
                z = int(g) - base
                if not 0 <= z < self._a.shape[axis]:
                    raise IndexError(f"index {g} outside the fab on axis {axis}")
                loc.append(z)
            else:
                scalar = False
                z = np.asarray(g) - base
                # debug builds check vector indices too (reference mesh.py:172-174);
                # otherwise negative offsets wrap like numpy/torch fancy indexing
                if config.debug and z.size and (int(z.min()) < 0 or int(z.max()) >= self._a.shape[axis]):
                    raise IndexError(f"vector index outside the fab on axis {axis}")
                loc.append(_torch().as_tensor(z, device=self._a.device))
        return tuple(loc) + (comp,), scalar

    def __getitem__(self, key):
        loc, scalar = self._resolve(key)
        out = self._a[loc]
        return out.item() if scalar else out

    def __setitem__(self, key, value):
        if not self.writable:
            raise ValueError("this FabView is read-only")
        loc, _ = self._resolve(key)
        if isinstance(value, np.ndarray):
            value = _torch().as_tensor(value, device=self._a.device, dtype=self._a.dtype)
        self._a[loc] = value


class BoxArray:
    """Pairwise-disjoint valid boxes (one centering), in a fixed order.  The
    disjointness check is the native binned sweep ``ghx_boxes_disjoint``."""

    def __init__(self, boxes: Iterable[Box], ixtype=None):
        self.boxes = tuple(boxes)
        self.uid = _next_uid()
        self._grown = {}
        if not self.boxes:
            self.ixtype = IndexType.cell() if ixtype is None else ixtype
            self._rows = np.zeros((0, 6), np.int64)
            self._dim = config.spacedim
            return
        self.ixtype = self.boxes[0].ixtype
        if any(b.is_empty for b in self.boxes):
            raise ValueError("BoxArray: empty boxes are not allowed")
        if any(b.ixtype != self.ixtype for b in self.boxes):
            raise ValueError("BoxArray: all boxes need the same index type")
        self._rows = np.ascontiguousarray(np.array([b.as_row() for b in self.boxes], dtype=np.int64))
        self._dim = len(self.boxes[0].lo)
        first, second = C.c_int64(), C.c_int64()
        N.check(N.lib.ghx_boxes_disjoint(len(self.boxes), N.i64p(self._rows), C.byref(first), C.byref(second)))
        if first.value >= 0:
            raise ValueError(f"BoxArray: valid regions must be disjoint, but {self.boxes[first.value]} "
                             f"overlaps {self.boxes[second.value]}")

    def __len__(self) -> int:
        return len(self.boxes)

    def __getitem__(self, i: int) -> Box:
        return self.boxes[i]

    def __iter__(self) -> Iterator[Box]:
        return iter(self.boxes)

    def minimal_extent(self) -> int:
        d = self._dim
        return int((self._rows[:, 3:3 + d] - self._rows[:, :d]).min()) + 1

    def rows(self, ngrow=None) -> np.ndarray:
        """(n, 6) int64 [lo0 lo1 lo2 hi0 hi1 hi2] rows, optionally grown."""
        if ngrow is None:
            return self._rows
        g = _pad3(ngrow, 0)
        if g not in self._grown:
            grown = self._rows.copy()
            grown[:, :3] -= g
            grown[:, 3:] += g
            self._grown[g] = np.ascontiguousarray(grown)
        return self._grown[g]


def decompose(domain: Box, max_grid_size) -> BoxArray:
    """Cut ``domain`` into boxes no longer than max_grid_size per axis;
    box k = ix + nbx*(iy + nby*iz) (x fastest), like core/mesh.py:223-235."""
    dim = len(domain.lo)
    sizes = [max_grid_size] * dim if isinstance(max_grid_size, int) else [int(v) for v in max_grid_size]
    spans = []
    for d in range(dim):
        cuts = range(domain.lo[d], domain.hi[d] + 1, sizes[d])
        spans.append([(c, min(c + sizes[d], domain.hi[d] + 1) - 1) for c in cuts])
    out = []
    for combo in itertools.product(*spans[::-1]):
        combo = combo[::-1]
        out.append(Box(tuple(c[0] for c in combo), tuple(c[1] for c in combo), domain.ixtype))
    return BoxArray(out)


class DistributionMapping:
    """Owner rank of every BoxArray entry."""

    def __init__(self, rank_of: Iterable[int], nranks: int | None = None):
        owners = tuple(int(r) for r in rank_of)
        self.rank_of = owners
        self.nranks = int(nranks) if nranks is not None else (1 + max(owners) if owners else 1)
        if owners and (min(owners) < 0 or max(owners) >= self.nranks):
            raise ValueError(f"DistributionMapping: ranks must be in [0, {self.nranks})")
        self.uid = _next_uid()
        self._arr = np.ascontiguousarray(np.asarray(owners, dtype=np.int32))

    @staticmethod
    def round_robin(nboxes: int, nranks: int) -> "DistributionMapping":
        return DistributionMapping([k % nranks for k in range(nboxes)], nranks)

    def __len__(self) -> int:
        return len(self.rank_of)

    def __getitem__(self, i: int) -> int:
        return self.rank_of[i]

    def array(self) -> np.ndarray:
        return self._arr


_ALIGN = 256


class MultiFab:
    """BoxArray + DistributionMapping + ghost width + one device slab."""

    def __init__(self, ba: BoxArray, dm: DistributionMapping, ncomp: int, ngrow,
                 geom: Geometry | None = None, arena=None, rank: int | None = None,
                 device: int | None = None, memory: str = "device"):
        if len(ba) == 0:
            raise ValueError("MultiFab needs a non-empty BoxArray")
        if len(dm) != len(ba):
            raise ValueError(f"distribution mapping length {len(dm)} != boxarray length {len(ba)}")
        from . import comm
        self.ba = ba
        self.dm = dm
        self.ncomp = int(ncomp)
        if self.ncomp < 1:
            raise ValueError(f"ncomp must be >= 1, got {ncomp}")
        self.ngrow = ngrow if isinstance(ngrow, IntVect) else IntVect.filled(ngrow)
        if any(g < 0 for g in self.ngrow):
            raise ValueError("ngrow components must be >= 0")
        self.geom = geom
        self.arena = arena
        self.dtype = config.real_dtype
        ctx = comm.current_ctx()
        self.rank = ctx.rank if rank is None else int(rank)
        self.device = ctx.device if device is None else int(device)
        self.memory = memory
        self.local_indices = tuple(i for i, r in enumerate(dm.rank_of) if r == self.rank)
        self.uid = _next_uid()
        self.plan_cache: dict = {}
        self.plan_builds = 0
        self._peer_cache: dict = {}
        self._fb_fast = None  # comm.fill_boundary's single-rank repeat-call entry
        self._alloc()

    def _alloc(self) -> None:
        item = self.dtype.itemsize
        rows = self.ba.rows(self.ngrow)
        offs = {}
        total = 0
        for i in self.local_indices:
            r = rows[i]
            count = int(np.prod(r[3:] - r[:3] + 1)) * self.ncomp
            offs[i] = total // item
            total += -(-count * item // _ALIGN) * _ALIGN
        self._offsets = offs
        self.fabs = {}
        self._slab = None
        if not self.local_indices:
            self._ptrs = np.zeros(0, np.uint64)
            return
        self._slab = Slab(total, self.device, self.memory, arena=_native_arena(self.arena))
        if config.debug:
            N.check(N.lib.ghx_memset_u64(C.c_void_p(self._slab.ptr), config.poison_word64(item),
                                         total // 8, None))
        for i in self.local_indices:
            self.fabs[i] = Fab(grow(self.ba[i], self.ngrow), self.ncomp, _slab=self._slab, _offset=offs[i])
        self._ptrs = np.array([self.fabs[i].ptr for i in self.local_indices], np.uint64)

    # -- reference surface (core/mesh.py:285-320)
    def valid_box(self, i: int) -> Box:
        return self.ba[i]

    def grown_box(self, i: int) -> Box:
        return grow(self.ba[i], self.ngrow)

    def fab(self, i: int) -> Fab:
        if i not in self.fabs:
            raise KeyError(f"fab {i} is not owned by rank {self.rank}")
        return self.fabs[i]

    def view(self, i: int) -> FabView:
        return self.fab(i).view(writable=True)

    def const_view(self, i: int) -> FabView:
        return self.fab(i).view(writable=False)

    def arrays(self) -> list:
        return [self.view(i) for i in self.local_indices]

    def const_arrays(self) -> list:
        return [self.const_view(i) for i in self.local_indices]

    def local_boxes(self, grown: bool = False) -> list:
        return [self.grown_box(i) if grown else self.ba[i] for i in self.local_indices]

    def setval(self, value: float, comp_range=None, grown: bool = True) -> None:
        for i in self.local_indices:
            self.fabs[i].setval(value, self.grown_box(i) if grown else self.ba[i], comp_range)

    def close(self) -> None:
        for f in self.fabs.values():
            f.release()
        self.fabs = {}
        self._slab = None
        self._ptrs = np.zeros(0, np.uint64)
        self._peer_cache = {}  # cached executors hold device pointers into the released storage
        self._fb_fast = None
        self._closed = True

    def check_open(self) -> None:
        """Raise ValueError if close() released this MultiFab's storage (the
        reference fails on its emptied ``fabs``; here cached device tables
        would otherwise point at freed memory)."""
        if getattr(self, "_closed", False):
            raise ValueError("MultiFab has been closed")

    # -- exchange entry points named by the north star
    def fill_boundary(self, geom: Geometry | None = None, backend=None) -> None:
        from . import comm
        comm.fill_boundary(self, geom, backend)

    def parallel_copy(self, src: "MultiFab", scomp: int = 0, dcomp: int = 0, ncomp=None,
                      ngrow_src=0, ngrow_dst=0, geom: Geometry | None = None, backend=None) -> None:
        from . import comm
        comm.parallel_copy(self, src, scomp, dcomp, ncomp, ngrow_src, ngrow_dst, geom, backend)

    # -- synthetic data (bench / parity tests)
    def fill_hash(self, seed: int, domain, stream=None) -> None:
        """Valid cells <- splitmix64 counter hash over ``domain`` (a Box or
        a padded [lo0 lo1 lo2 hi0 hi1 hi2] row; formula in oracle/inputs.py),
        other cells <- sNaN poison."""
        row = domain.as_row() if isinstance(domain, Box) else list(domain)
        dom = np.ascontiguousarray(np.asarray(row, np.int64))
        st = None if stream is None else C.c_void_p(stream)
        for i in self.local_indices:
            f = self.fabs[i]
            fb = np.ascontiguousarray(np.asarray(f.box.as_row(), np.int64))
            vb = np.ascontiguousarray(np.asarray(self.ba[i].as_row(), np.int64))
            N.check(N.lib.ghx_fill_hash(C.c_void_p(f.ptr), N.i64p(fb), self.ncomp, N.i64p(vb), N.i64p(dom),
                                        C.c_uint64(int(seed)), self.dtype.itemsize, st))

    def storage_rows(self) -> np.ndarray:
        return self.ba.rows(self.ngrow)


def multifab_define(ba: BoxArray, dm: DistributionMapping, ncomp: int, ngrow,
                    geom: Geometry | None = None, arena=None, **kw) -> MultiFab:
    return MultiFab(ba, dm, ncomp, ngrow, geom, arena, **kw)


def fab_view(mf: MultiFab, fab_index: int) -> FabView:
    return mf.view(fab_index)


def const_fab_view(mf: MultiFab, fab_index: int) -> FabView:
    return mf.const_view(fab_index)
