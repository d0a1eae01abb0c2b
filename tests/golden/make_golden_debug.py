"""Generate the debug-mode golden fixtures by running the REFERENCE itself.

Build container only (needs /root/reference):

    cd /tmp && PYTHONDONTWRITEBYTECODE=1 python /root/repo/tests/golden/make_golden_debug.py

With ``config.set_debug(True)`` the reference fills every fresh fab with
``config.POISON_REAL`` (reference config.py:21, mesh.py:59-60).  For float32
storage that is numpy's float64 -> float32 narrowing of the signalling NaN,
so uncoverable ghost cells end up holding those exact bits after an
exchange.  Each case here creates the MultiFabs in debug mode, writes hash
values into the VALID cells only (ghosts keep the reference's poison), runs
``fill_boundary`` / ``parallel_copy`` (serial backend) under
``runtime_spawn`` and records every fab's raw bits plus the Bus message
stats.  A non-periodic axis (or a ParallelCopy with ``ngrow_dst > 0``)
leaves some ghosts uncovered, which is what pins the poison.

Outputs: tests/golden/golden_debug.json and tests/golden/golden_debug.npz.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.environ.get("MINIAMR_REF", "/root/reference/pkg/src"))

from miniamr_core import comm, config  # noqa: E402
from miniamr_core.index_space import Box, Geometry  # noqa: E402
from miniamr_core.kernels import Backend  # noqa: E402
from miniamr_core.mesh import BoxArray, DistributionMapping, MultiFab  # noqa: E402

from oracle import inputs  # noqa: E402

CASES: list[dict] = []
ARRAYS: dict[str, np.ndarray] = {}


def pad3(v, fill=0):
    v = list(int(x) for x in v)
    return v + [fill] * (3 - len(v))


def fill_valid(fab, valid_box, dlo, dhi, seed=inputs.SEED):
    """Hash values into the valid cells; every other cell keeps its bits."""
    lo, hi = pad3(valid_box.lo), pad3(valid_box.hi)
    flo = pad3(fab.box.lo)
    tmp = inputs.make_fab(lo, hi, fab.ncomp, fab.data.dtype, lo, hi, dlo, dhi, seed)
    sl = tuple(slice(lo[d] - flo[d], hi[d] - flo[d] + 1) for d in range(3))
    fab.data[sl] = tmp


def stats_delta(a, b):
    out = [[s, d, b[(s, d)][0] - a[(s, d)][0], b[(s, d)][1] - a[(s, d)][1]]
           for (s, d) in sorted(b) if b[(s, d)] != a[(s, d)]]
    return np.asarray(out, np.int64).reshape(-1, 4)


def fb_case(name, dim, ext, boxes, rank_of, nranks, ngrow, periodic, ncomp, dtype):
    config.set_spacedim(dim)
    config.set_real_dtype(dtype)
    config.set_debug(True)
    ba = BoxArray([Box(l, h) for l, h in boxes])
    dm = DistributionMapping(rank_of, nranks)
    geom = Geometry(Box([0] * dim, [e - 1 for e in ext]), [0.0] * dim, [1.0] * dim, periodic)
    dlo, dhi = [0, 0, 0], pad3([e - 1 for e in ext])

    def program(ctx):
        mf = MultiFab(ba, dm, ncomp, ngrow, geom)
        fresh = {gi: inputs.bits(mf.fabs[gi].data).copy(order="F") for gi in mf.local_indices}
        for gi in mf.local_indices:
            fill_valid(mf.fabs[gi], ba[gi], dlo, dhi)
        ctx.barrier()
        s0 = ctx.bus.stats_snapshot()
        ctx.barrier()
        comm.fill_boundary(mf, geom, backend=Backend("serial"))
        ctx.barrier()
        s1 = ctx.bus.stats_snapshot()
        ctx.barrier()
        return ({gi: inputs.bits(mf.fabs[gi].data).copy(order="F") for gi in mf.local_indices},
                stats_delta(s0, s1), fresh)

    res = comm.runtime_spawn(nranks, program)
    for out, _, fresh in res:
        for gi, a in out.items():
            ARRAYS[f"{name}/fab{gi}"] = a
        for gi, a in fresh.items():
            ARRAYS[f"{name}/fresh{gi}"] = a
    ARRAYS[f"{name}/stats"] = res[0][1]
    CASES.append(dict(name=name, kind="fill_boundary", dim=dim, ext=pad3(ext, 1),
                      boxes=[pad3(l) + pad3(h) for l, h in boxes], rank_of=list(rank_of), nranks=nranks,
                      ngrow=pad3([ngrow] * dim), periodic=[bool(p) for p in periodic] + [False] * (3 - dim),
                      ncomp=ncomp, dtype=np.dtype(dtype).name))


def pc_case(name, dim, ext, src_boxes, dst_boxes, src_rank, dst_rank, nranks, ncomp, ngrow_dst, dtype):
    config.set_spacedim(dim)
    config.set_real_dtype(dtype)
    config.set_debug(True)
    sba = BoxArray([Box(l, h) for l, h in src_boxes])
    dba = BoxArray([Box(l, h) for l, h in dst_boxes])
    sdm, ddm = DistributionMapping(src_rank, nranks), DistributionMapping(dst_rank, nranks)
    dlo, dhi = [0, 0, 0], pad3([e - 1 for e in ext])

    def program(ctx):
        src = MultiFab(sba, sdm, ncomp, 0)
        dst = MultiFab(dba, ddm, ncomp, ngrow_dst)
        for gi in src.local_indices:
            fill_valid(src.fabs[gi], sba[gi], dlo, dhi)
        ctx.barrier()
        s0 = ctx.bus.stats_snapshot()
        ctx.barrier()
        comm.parallel_copy(dst, src, ngrow_dst=ngrow_dst, backend=Backend("serial"))
        ctx.barrier()
        s1 = ctx.bus.stats_snapshot()
        ctx.barrier()
        return {gi: inputs.bits(dst.fabs[gi].data).copy(order="F") for gi in dst.local_indices}, stats_delta(s0, s1)

    res = comm.runtime_spawn(nranks, program)
    for out, _ in res:
        for gi, a in out.items():
            ARRAYS[f"{name}/fab{gi}"] = a
    ARRAYS[f"{name}/stats"] = res[0][1]
    CASES.append(dict(name=name, kind="parallel_copy", dim=dim, ext=pad3(ext, 1),
                      src_boxes=[pad3(l) + pad3(h) for l, h in src_boxes],
                      dst_boxes=[pad3(l) + pad3(h) for l, h in dst_boxes], src_rank=list(src_rank),
                      dst_rank=list(dst_rank), nranks=nranks, ncomp=ncomp, ngrow_dst=pad3([ngrow_dst] * dim),
                      dtype=np.dtype(dtype).name))


def main():
    f32, f64 = np.float32, np.float64
    b3 = [([x, y, z], [x + 3, y + 3, z + 3]) for z in (0, 4) for y in (0, 4) for x in (0, 4)]
    b2 = [([x, y], [x + 4, y + 3]) for y in (0, 4) for x in (0, 5)]
    b1 = [([0], [3]), ([4], [9]), ([10], [13])]
    for dt in (f32, f64):
        t = np.dtype(dt).name
        # 3-D, z not periodic: the z-lo / z-hi ghost layers have no source
        fb_case(f"dbg_fb3_{t}_r1", 3, [8, 8, 8], b3, [0] * 8, 1, 2, [True, True, False], 2, dt)
        fb_case(f"dbg_fb3_{t}_r2", 3, [8, 8, 8], b3, [i % 2 for i in range(8)], 2, 1, [True, False, True], 1, dt)
        # 2-D, nothing periodic
        fb_case(f"dbg_fb2_{t}_r2", 2, [10, 8], b2, [0, 1, 1, 0], 2, 2, [False, False], 3, dt)
        # 1-D, not periodic: the two outer ghost layers keep the poison
        fb_case(f"dbg_fb1_{t}_r1", 1, [14], b1, [0, 0, 0], 1, 2, [False], 1, dt)
        # ParallelCopy into grown dst boxes: ghosts outside the source cover keep the poison
        src = [([0, 0, 0], [5, 7, 7]), ([6, 0, 0], [7, 7, 7])]
        pc_case(f"dbg_pc3_{t}_r2", 3, [8, 8, 8], src, b3, [0, 1], [i % 2 for i in range(8)], 2, 2, 1, dt)
    config.set_debug(False)
    config.set_spacedim(3)
    config.set_real_dtype(f64)
    with open(os.path.join(HERE, "golden_debug.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden_debug.py",
                   "reference": "miniamr_core (pkg/src) from /root/reference, config.debug=True",
                   "poison32_bits": int(np.asarray([config.POISON_REAL]).astype(np.float32).view(np.uint32)[0]),
                   "cases": CASES}, f, indent=1)
    np.savez_compressed(os.path.join(HERE, "golden_debug.npz"), **ARRAYS)
    print(f"wrote {len(CASES)} debug cases, {len(ARRAYS)} arrays")


if __name__ == "__main__":
    main()
