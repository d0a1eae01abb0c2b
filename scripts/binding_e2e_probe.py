"""Probe: C3 FillBoundary through integration/reference_binding on the
reference's MultiFab in pinned memory -- per-fab pinned blocks, one pinned
slab cut into the fabs, or PinnedArena's 2 GiB chunks (the arena choice),
each timed alone:  python scripts/binding_e2e_probe.py blocks|slab|chunks [none|cpu|gpu]"""
import os
import statistics
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import bench  # noqa: E402

ref, _ = bench.import_reference()
from miniamr_core import config as rconfig  # noqa: E402
from miniamr_core.index_space import Box as RBox, Geometry as RGeometry  # noqa: E402
from miniamr_core.mesh import DistributionMapping as RDM, MultiFab as RMF, decompose as rdecompose  # noqa: E402
from integration import reference_binding as RB  # noqa: E402
import ctypes as C  # noqa: E402


class SlabArena:
    """One pinned slab, bump-allocated."""

    def __init__(self, nbytes):
        p = C.c_void_p()
        RB._check(RB.lib().ghx_host_alloc(int(nbytes), C.byref(p)))
        self.base, self.off, self.n = p.value, 0, nbytes

    def alloc(self, nbytes, align=256):
        self.off = (self.off + 4095) // 4096 * 4096
        b = RB._PinnedBlock(self, None, self.base + self.off, nbytes)
        b.freed = True  # the slab owns the memory
        self.off += nbytes
        assert self.off <= self.n
        return b

    def free(self, block):
        pass


def run(arena, steps=10, fill="cpu"):
    rconfig.set_spacedim(3)
    dom = RBox((0, 0, 0), (511, 511, 511))
    geom = RGeometry(dom, (0.0,) * 3, (1.0,) * 3, (True,) * 3)
    ba = rdecompose(dom, 128)
    mf = RMF(ba, RDM.round_robin(len(ba), 1), 8, 2, geom, arena=arena)
    if fill == "cpu":
        for i in mf.local_indices:
            mf.fabs[i].data[...] = 1.0
    elif fill == "gpu":  # the device writes every fab word (mapped memory)
        L = RB.lib()
        L.ghx_memset_u64.argtypes = [C.c_void_p, C.c_uint64, C.c_int64, C.c_void_p]
        for i in mf.local_indices:
            a = mf.fabs[i].data
            RB._check(L.ghx_memset_u64(a.__array_interface__["data"][0], 0x3FF0000000000000, a.size, None))
        RB._check(L.ghx_stream_sync(None))
    RB.fill_boundary_native(mf, geom)
    ts = []
    for _ in range(steps):
        a = time.perf_counter()
        RB.fill_boundary_native(mf, geom)
        ts.append(time.perf_counter() - a)
    return statistics.median(ts) * 1e3


if os.environ.get("PROBE_TORCH"):  # let torch create the CUDA context first
    import torch
    torch.zeros(1, device="cuda")
which = sys.argv[1] if len(sys.argv) > 1 else "blocks"
fill = sys.argv[2] if len(sys.argv) > 2 else "cpu"
if which == "blocks":
    print("per-fab pinned blocks, %s fill: %.2f ms" % (fill, run(RB.PinnedArena(chunk_bytes=1), fill=fill)))
elif which == "chunks":
    print("PinnedArena (growing chunks), %s fill: %.2f ms" % (fill, run(RB.PinnedArena(), fill=fill)))
elif which == "chunks2g":
    print("PinnedArena (2 GiB chunks), %s fill: %.2f ms" % (fill, run(RB.PinnedArena(1 << 31), fill=fill)))
else:
    print("one pinned slab, %s fill:       %.2f ms" % (fill, run(SlabArena(64 * 132 ** 3 * 8 * 8 + 64 * 4096), fill=fill)))
