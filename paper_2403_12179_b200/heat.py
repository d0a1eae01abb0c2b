"""Heat-equation step loop on the exchange engine: the reference demo's
per-step body (/root/reference/pkg/src/miniamr_core/heat.py:264-273) and its
explicit stencil ``_advance_level`` (heat.py:172-189), the end-to-end
consumer of FillBoundary / fill_patch / average_down.

B200 design: the stencil is a 2.5-D blocked kernel (32 x 8 tiles marching in
z, each source value read from HBM once).  Optionally (``overlap=True``) the
stencil of the cells that do not read ghost data (each valid box shrunk by
one cell) runs on a side stream while the ghost exchange (FillBoundary,
fill_patch) runs on the main stream; only the one-cell shell next to the
ghosts waits for the exchange.  Results are bit-identical to the
reference (same per-cell operation order, no FMA contraction), whatever the
overlap.  Out of scope: the demo driver around the loop (AmrMesh, regrid,
tagging, the Gaussian oracle, integrals, plotfiles).
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _native as N
from . import comm, config
from .amr import LINEAR, _Xfer, average_down, fill_patch
from .index_space import Box, Geometry, box_diff, grow
from .mesh import MultiFab


def _coefs(dt: float, diffusivity: float, geom: Geometry) -> np.ndarray:
    c = np.zeros(3, np.float64)
    for d in range(config.spacedim):
        c[d] = dt * diffusivity / geom.cell_size[d] ** 2  # heat.py:174, Python float64
    return c


def _shrink(b: Box) -> Box:
    return grow(b, -1)


def _prepare(u: MultiFab, w: MultiFab, coef: np.ndarray, part: str) -> _Xfer:
    """Prepared stencil launch over every local valid box ('all'), their
    interiors shrunk by one cell ('interior') or the remaining shells."""
    jobs = []
    for gi in u.local_indices:
        vb = u.ba[gi]
        if part == "all":
            regions = [vb]
        else:
            inner = _shrink(vb)
            if part == "interior":
                regions = [] if inner.is_empty else [inner]
            else:
                regions = [vb] if inner.is_empty else box_diff(vb, inner)
        for r in regions:
            jobs.append((u.fabs[gi], w.fabs[gi], r))
    rows = np.zeros((len(jobs), N.JOB_WORDS), np.int64)
    for n, (uf, wf, r) in enumerate(jobs):
        rows[n, 0] = np.uint64(uf.ptr).view(np.int64)
        rows[n, 1:7] = uf.box.as_row()
        rows[n, 7] = np.uint64(wf.ptr).view(np.int64)
        rows[n, 8:14] = wf.box.as_row()
        rows[n, 14:20] = r.as_row()
    h = C.c_void_p()
    N.check(N.lib.ghx_advance_prepare(C.c_void_p(rows.ctypes.data), len(jobs),
                                      coef.ctypes.data_as(C.POINTER(C.c_double)), config.spacedim,
                                      u.dtype.itemsize, N.ADVANCE_CELLS if part == "shell" else N.ADVANCE_TILES,
                                      u.device, C.byref(h)))
    return _Xfer(h.value, u.device)


def _stencil(u: MultiFab, w: MultiFab, dt: float, diffusivity: float, geom: Geometry, part: str) -> _Xfer:
    u.check_open()
    w.check_open()
    if u.ba is not w.ba and list(u.ba) != list(w.ba):
        raise ValueError("advance_level: u and unew must share the BoxArray")
    if min(u.ngrow) < 1 and part != "interior":
        raise ValueError("advance_level needs one ghost cell")
    coef = _coefs(dt, diffusivity, geom)
    key = ("advance", part, w.uid, tuple(coef.tolist()))
    xf = u._peer_cache.get(key)
    if xf is None:
        xf = comm.cache_put(u, key, _prepare(u, w, coef, part), w)
    return xf


def advance_level(u: MultiFab, unew: MultiFab, dt: float, diffusivity: float, geom: Geometry,
                  backend=None) -> None:
    """unew = u + dt * diffusivity * Laplacian(u) on every valid cell (comp
    0), u's ghosts already filled (heat.py:172-189); one launch."""
    _stencil(u, unew, dt, diffusivity, geom, "all").run()
    _sync(u.device)


def _sync(device: int) -> None:
    import torch
    torch.cuda.current_stream(device).synchronize()


_side_streams: dict = {}


def _side_stream(device: int):
    import torch
    s = _side_streams.get(device)
    if s is None:
        s = _side_streams[device] = torch.cuda.Stream(device=device)
    return s


def _enqueue_step(levels: list, geoms: list, dt: float, diffusivity: float, ref_ratio: int) -> list:
    """Single rank: the whole loop body enqueued on the current stream, no
    host wait (also what HeatLoop captures into a CUDA graph)."""
    import torch
    dev = levels[0][0].device
    main = torch.cuda.current_stream(dev)
    if len(levels) > 1 and os.environ.get("GHX_LEVEL_OVERLAP", "1") != "0":
        # The coarse chain (FillBoundary, stencil into unew) and the fine one
        # (fill_patch -- its gather reads coarse VALID cells only, which
        # neither coarse kernel writes -- then the fine stencil) are
        # independent; average_down writes coarse unew, so it joins both.
        lvl = _level_stream(dev)
        lvl.wait_stream(main)
        comm.prepare_fill_boundary(levels[0][0], geoms[0]).enqueue(main.cuda_stream)
        _stencil(levels[0][0], levels[0][1], dt, diffusivity, geoms[0], "all").run()
        with torch.cuda.stream(lvl):
            fill_patch(levels[1][0], levels[0][0], geoms[1], geoms[0], ref_ratio, LINEAR, _wait=False)
            _stencil(levels[1][0], levels[1][1], dt, diffusivity, geoms[1], "all").run()
        main.wait_stream(lvl)
        average_down(levels[1][1], levels[0][1], ref_ratio, _wait=False)
        return [(w, u) for (u, w) in levels]
    comm.prepare_fill_boundary(levels[0][0], geoms[0]).enqueue(main.cuda_stream)
    if len(levels) > 1:
        fill_patch(levels[1][0], levels[0][0], geoms[1], geoms[0], ref_ratio, LINEAR, _wait=False)
    for lv, (u, w) in enumerate(levels):
        _stencil(u, w, dt, diffusivity, geoms[lv], "all").run()
    if len(levels) > 1:
        average_down(levels[1][1], levels[0][1], ref_ratio, _wait=False)
    return [(w, u) for (u, w) in levels]


_level_streams: dict = {}


def _level_stream(device: int):
    import torch
    st = _level_streams.get(device)
    if st is None:
        st = _level_streams[device] = torch.cuda.Stream(device)
    return st


def heat_step(levels: list, geoms: list, dt: float, diffusivity: float, ref_ratio: int = 2, backend=None,
              overlap: bool = False) -> list:
    """One step of the reference loop (heat.py:264-273) on ``levels`` =
    [(u, unew)] per level (1 or 2 levels): FillBoundary of the coarse
    solution, fill_patch of the fine one (LINEAR), the stencil on every
    level, average_down of the new fine solution, then the (u, unew) swap,
    which is returned.  With ``overlap`` the interior stencils run on a side
    stream during the exchanges.  Measured on one B200 (bench_amr.py --op
    heat): off by default -- with the exchange local, both phases are
    HBM-bound and the split adds a launch and a one-cell shell pass whose
    x-faces are isolated seams again (0.103 vs 0.122 ms); it is
    meant for exchanges whose latency is remote (NVLink / host memory)."""
    import torch
    if not 1 <= len(levels) <= 2:
        raise ValueError("heat_step supports one or two levels")
    dev = levels[0][0].device
    main = torch.cuda.current_stream(dev)
    if not overlap and comm.current_ctx().nranks == 1:
        out = _enqueue_step(levels, geoms, dt, diffusivity, ref_ratio)
        main.synchronize()
        return out
    if overlap:
        side = _side_stream(dev)
        ready = torch.cuda.Event()
        ready.record(main)
        side.wait_event(ready)
        with torch.cuda.stream(side):
            for lv, (u, w) in enumerate(levels):
                _stencil(u, w, dt, diffusivity, geoms[lv], "interior").run()
        done = torch.cuda.Event()
        done.record(side)
    if comm.current_ctx().nranks == 1:  # stream-ordered, no host wait before the stencil
        comm.prepare_fill_boundary(levels[0][0], geoms[0]).enqueue(main.cuda_stream)
    else:
        comm.fill_boundary(levels[0][0], geoms[0], backend=backend)
    if len(levels) > 1:
        fill_patch(levels[1][0], levels[0][0], geoms[1], geoms[0], ref_ratio, LINEAR, backend=backend)
    for lv, (u, w) in enumerate(levels):
        _stencil(u, w, dt, diffusivity, geoms[lv], "shell" if overlap else "all").run()
    if overlap:
        main.wait_event(done)
    if len(levels) > 1:
        average_down(levels[1][1], levels[0][1], ref_ratio, backend)
    main.synchronize()
    return [(w, u) for (u, w) in levels]


class HeatLoop:
    """The heat loop with each step's launches replayed from a CUDA graph
    (single rank; launch-bound multi-level steps become one graph launch).

    Steps 1-2 run eagerly (they build the plans, executors, prepared
    transfers and bind pointer tables for both (u, unew) parities); from
    step 3 on each parity's step is captured once and replayed.  Results are
    identical to ``heat_step`` (same kernels, same order).  With more than
    one rank it falls back to ``heat_step``."""

    def __init__(self, levels: list, geoms: list, dt: float, diffusivity: float, ref_ratio: int = 2,
                 graphs: bool = True):
        self.levels, self.geoms = list(levels), list(geoms)
        self.dt, self.diffusivity, self.ref_ratio = dt, diffusivity, ref_ratio
        self.graphs = graphs and comm.current_ctx().nranks == 1
        self.nsteps = 0
        self._graph = {}
        self._after = {}

    def step(self) -> list:
        import torch
        if not self.graphs or self.nsteps < 2:
            self.levels = heat_step(self.levels, self.geoms, self.dt, self.diffusivity, self.ref_ratio)
        else:
            p = self.nsteps % 2
            g = self._graph.get(p)
            if g is None:
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    self._after[p] = _enqueue_step(self.levels, self.geoms, self.dt, self.diffusivity,
                                                   self.ref_ratio)
                self._graph[p] = g
            g.replay()
            self.levels = self._after[p]
            torch.cuda.current_stream(self.levels[0][0].device).synchronize()
        self.nsteps += 1
        return self.levels

