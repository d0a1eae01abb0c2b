"""Generate golden fixtures for the coarse/fine level transfers by running the
REFERENCE implementation itself (build container only: needs /root/reference).

    cd /tmp && PYTHONDONTWRITEBYTECODE=1 python /root/repo/tests/golden/make_golden_amr.py

Cases (miniamr_core.amr, serial backend, runtime_spawn ranks):

* ``interp``       interp_box(coarse_fab, fine_fab, region, ratio, scheme) on a
                   hash-filled coarse fab; the fine fab starts poisoned;
* ``average_down`` average_down(fine, coarse, ratio) with hash-filled fine
                   valid cells and hash-filled coarse valid cells;
* ``fill_patch``   fill_patch(fine, coarse, fgeom, cgeom, ratio, scheme) with
                   hash-filled valid cells and poisoned fine ghosts.

Non-periodic LINEAR cases are avoided: their slopes at the domain edge read
coarse cells no rank ever writes (uninitialised arena memory in the
reference).  Every fab's raw bits after the call are stored.

Outputs: tests/golden/golden_amr.json and tests/golden/golden_amr.npz.
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

from miniamr_core import amr, comm, config  # noqa: E402
from miniamr_core.index_space import Box, Geometry, coarsen, refine  # noqa: E402
from miniamr_core.kernels import Backend  # noqa: E402
from miniamr_core.mesh import BoxArray, DistributionMapping, Fab, MultiFab, decompose  # noqa: E402

from oracle import inputs  # noqa: E402

CASES: list = []
ARRAYS: dict = {}
SEED_C = inputs.SEED + 1  # coarse-level hash seed (fine level uses inputs.SEED)


def pad3(v, fill=0):
    v = [int(x) for x in v]
    return v + [fill] * (3 - len(v))


def box6(b):
    return pad3(b.lo) + pad3(b.hi)


def fill(fab, valid, domain, seed):
    inputs.fill_fab(fab.data, pad3(fab.box.lo), pad3(valid.lo), pad3(valid.hi), pad3(domain.lo), pad3(domain.hi),
                    seed)


def set_cfg(dim, dtype):
    config.set_spacedim(dim)
    config.set_real_dtype(dtype)


def reset_cfg():
    config.set_spacedim(3)
    config.set_real_dtype(np.float64)


# ---------------------------------------------------------------- interp_box

def run_interp(name, dim, cbox, fbox, region, ratio, scheme, ncomp, dtype):
    set_cfg(dim, dtype)
    cb, fb, rg = Box(*cbox), Box(*fbox), Box(*region)  # noqa
    cf = Fab(cb, ncomp)
    fill(cf, cb, cb, SEED_C)
    ff = Fab(fb, ncomp)
    inputs.bits(ff.data)[...] = inputs.POISON64 if ff.data.dtype.itemsize == 8 else inputs.POISON32
    amr.interp_box(cf, ff, rg, ratio, scheme)
    ARRAYS[f"{name}/fine"] = inputs.bits(ff.data).copy(order="F")
    CASES.append(dict(name=name, kind="interp", dim=dim, crse_box=box6(cb), fine_box=box6(fb), region=box6(rg),
                      ratio=ratio, scheme=scheme, ncomp=ncomp, dtype=np.dtype(dtype).name, seed=SEED_C))
    reset_cfg()


def gen_interp(rng, n):
    for t in range(n):
        dim = [1, 2, 3][t % 3]
        ratio = [2, 3, 4][(t // 3) % 3]
        scheme = amr.LINEAR if t % 2 else amr.PIECEWISE_CONSTANT
        dtype = np.float32 if t % 5 == 4 else np.float64
        ncomp = int(rng.integers(1, 4))
        flo = [int(rng.integers(-9, 9)) for _ in range(dim)]
        fext = [int(rng.integers(3, 14)) for _ in range(dim)]
        fhi = [l + e - 1 for l, e in zip(flo, fext)]
        rlo = [int(rng.integers(l, h + 1)) for l, h in zip(flo, fhi)]
        rhi = [int(rng.integers(a, h + 1)) for a, h in zip(rlo, fhi)]
        g = 1 if scheme == amr.LINEAR else 0
        clo = [(a // ratio) - g - int(rng.integers(0, 2)) for a in rlo]
        chi = [(b // ratio) + g + int(rng.integers(0, 2)) for b in rhi]
        run_interp(f"interp_{t:02d}", dim, (clo, chi), (flo, fhi), (rlo, rhi), ratio, scheme, ncomp, dtype)


# -------------------------------------------------------------- average_down

def aligned_boxes(rng, dim, fext, ratio, nbox):
    """Disjoint ratio-aligned fine boxes inside [0, fext)."""
    out = []
    tries = 0
    while len(out) < nbox and tries < 200:
        tries += 1
        lo = [int(rng.integers(0, fext[d] // ratio)) * ratio for d in range(dim)]
        ext = [int(rng.integers(1, 4)) * ratio for _ in range(dim)]
        hi = [min(l + e, fext[d]) - 1 for d, (l, e) in enumerate(zip(lo, ext))]
        if any(h < l for l, h in zip(lo, hi)) or any((h - l + 1) % ratio for l, h in zip(lo, hi)):
            continue
        b = Box(lo, hi)
        if any(b.intersects(o) for o in out):
            continue
        out.append(b)
    out.sort(key=lambda b: tuple(b.lo))
    return out


def run_avgdown(name, dim, cext, cmgs, fine_boxes, ratio, nranks, ncomp, fngrow, cngrow, dtype):
    set_cfg(dim, dtype)
    cdom = Box([0] * dim, [e - 1 for e in cext])
    fdom = refine(cdom, ratio)
    cba = decompose(cdom, cmgs)
    cdm = DistributionMapping([i % nranks for i in range(len(cba))], nranks)
    fba = BoxArray(fine_boxes)
    fdm = DistributionMapping([(i + 1) % nranks for i in range(len(fba))], nranks)
    geom = Geometry(cdom, [0.0] * dim, [1.0] * dim, [True] * dim)

    def program(ctx):
        coarse = MultiFab(cba, cdm, ncomp, cngrow, geom)
        fine = MultiFab(fba, fdm, ncomp, fngrow, geom.refined(ratio))
        for gi in coarse.local_indices:
            fill(coarse.fabs[gi], cba[gi], cdom, SEED_C)
        for gi in fine.local_indices:
            fill(fine.fabs[gi], fba[gi], fdom, inputs.SEED)
        ctx.barrier()
        amr.average_down(fine, coarse, ratio, Backend("serial"))
        return {gi: inputs.bits(coarse.fabs[gi].data).copy(order="F") for gi in coarse.local_indices}

    res = comm.runtime_spawn(nranks, program)
    for out in res:
        for gi, a in out.items():
            ARRAYS[f"{name}/crse{gi}"] = a
    CASES.append(dict(name=name, kind="average_down", dim=dim, cext=pad3(cext, 1), cmgs=cmgs,
                      fine_boxes=[box6(b) for b in fine_boxes], ratio=ratio, nranks=nranks, ncomp=ncomp,
                      fngrow=fngrow, cngrow=cngrow, dtype=np.dtype(dtype).name,
                      crse_boxes=[box6(b) for b in cba], crse_rank=list(cdm.rank_of),
                      fine_rank=list(fdm.rank_of)))
    reset_cfg()


def gen_avgdown(rng, n):
    for t in range(n):
        dim = [1, 2, 3][t % 3]
        ratio = [2, 4, 3][(t // 3) % 3] if dim < 3 else 2
        cext = [int(rng.integers(4, 9)) for _ in range(dim)]
        fext = [e * ratio for e in cext]
        config.set_spacedim(dim)
        boxes = aligned_boxes(rng, dim, fext, ratio, int(rng.integers(1, 5)))
        if not boxes:
            continue
        run_avgdown(f"avgdown_{t:02d}", dim, cext, int(rng.integers(2, 6)), boxes, ratio, int(rng.integers(1, 3)),
                    int(rng.integers(1, 3)), int(rng.integers(0, 2)), int(rng.integers(0, 2)),
                    np.float32 if t % 4 == 3 else np.float64)


# ---------------------------------------------------------------- fill_patch

def run_fill_patch(name, dim, cext, cmgs, fine_boxes, ratio, nranks, ncomp, fngrow, periodic, scheme, dtype):
    set_cfg(dim, dtype)
    cdom = Box([0] * dim, [e - 1 for e in cext])
    cgeom = Geometry(cdom, [0.0] * dim, [1.0] * dim, periodic)
    fgeom = cgeom.refined(ratio)
    fdom = fgeom.domain
    cba = decompose(cdom, cmgs)
    cdm = DistributionMapping([i % nranks for i in range(len(cba))], nranks)
    fba = BoxArray(fine_boxes)
    fdm = DistributionMapping([(i + 1) % nranks for i in range(len(fba))], nranks)

    def program(ctx):
        coarse = MultiFab(cba, cdm, ncomp, 0, cgeom)
        fine = MultiFab(fba, fdm, ncomp, fngrow, fgeom)
        for gi in coarse.local_indices:
            fill(coarse.fabs[gi], cba[gi], cdom, SEED_C)
        for gi in fine.local_indices:
            fill(fine.fabs[gi], fba[gi], fdom, inputs.SEED)
        ctx.barrier()
        amr.fill_patch(fine, coarse, fgeom, cgeom, ratio, scheme, backend=Backend("serial"))
        amr.fill_patch(fine, coarse, fgeom, cgeom, ratio, scheme, backend=Backend("serial"))
        return ({gi: inputs.bits(fine.fabs[gi].data).copy(order="F") for gi in fine.local_indices},
                fine.plan_builds)

    res = comm.runtime_spawn(nranks, program)
    for out, _ in res:
        for gi, a in out.items():
            ARRAYS[f"{name}/fine{gi}"] = a
    CASES.append(dict(name=name, kind="fill_patch", dim=dim, cext=pad3(cext, 1), cmgs=cmgs,
                      fine_boxes=[box6(b) for b in fine_boxes], ratio=ratio, nranks=nranks, ncomp=ncomp,
                      fngrow=fngrow, periodic=list(periodic) + [False] * (3 - dim), scheme=scheme,
                      dtype=np.dtype(dtype).name, crse_boxes=[box6(b) for b in cba],
                      crse_rank=list(cdm.rank_of), fine_rank=list(fdm.rank_of),
                      plan_builds=[r[1] for r in res]))
    reset_cfg()


def gen_fill_patch(rng, n):
    for t in range(n):
        dim = 2 if t % 3 else 3
        ratio = 2 if t % 4 else 4
        cext = [int(rng.integers(6, 11)) if dim == 2 else int(rng.integers(4, 7)) for _ in range(dim)]
        fext = [e * ratio for e in cext]
        periodic = [True] * dim if t % 3 != 1 else [bool(rng.integers(0, 2)) for _ in range(dim)]
        scheme = amr.LINEAR if all(periodic) and t % 2 == 0 else amr.PIECEWISE_CONSTANT
        config.set_spacedim(dim)
        boxes = aligned_boxes(rng, dim, fext, ratio, int(rng.integers(1, 5)))
        if not boxes:
            continue
        fngrow = int(rng.integers(1, 3))
        if fngrow > min(min(b.extents) for b in boxes):
            fngrow = 1
        run_fill_patch(f"fillpatch_{t:02d}", dim, cext, int(rng.integers(3, 6)), boxes, ratio,
                       int(rng.integers(1, 3)), int(rng.integers(1, 3)), fngrow, periodic, scheme,
                       np.float32 if t % 5 == 4 else np.float64)
    # the reference's own configurations (tests/test_amr.py:226-303 shapes)
    config.set_spacedim(2)
    run_fill_patch("fillpatch_interior", 2, [16, 16], 8, [Box((8, 8), (15, 15))], 2, 1, 1, 1,
                   [True, True], amr.LINEAR, np.float64)
    config.set_spacedim(2)
    run_fill_patch("fillpatch_mixed", 2, [16, 16], 8,
                   [Box((0, 0), (15, 7)), Box((8, 8), (23, 15)), Box((16, 16), (31, 31))], 2, 2, 2, 1,
                   [True, True], amr.LINEAR, np.float64)
    config.set_spacedim(2)
    run_fill_patch("fillpatch_full", 2, [16, 16], 8, list(decompose(Box((0, 0), (31, 31)), 16)), 2, 2, 1, 1,
                   [True, True], amr.LINEAR, np.float64)


# ------------------------------------------------------------- heat step loop

def run_heat(name, dim, cext, cmgs, fine_boxes, ratio, nranks, steps, dt, diffusivity, dtype):
    """The reference demo's loop body (heat.py:264-273) for ``steps`` steps."""
    from miniamr_core.heat import _advance_level
    set_cfg(dim, dtype)
    cdom = Box([0] * dim, [e - 1 for e in cext])
    cgeom = Geometry(cdom, [0.0] * dim, [1.0] * dim, [True] * dim)
    fgeom = cgeom.refined(ratio)
    cba = decompose(cdom, cmgs)
    cdm = DistributionMapping([i % nranks for i in range(len(cba))], nranks)
    fba = BoxArray(fine_boxes) if fine_boxes else None
    fdm = DistributionMapping([(i + 1) % nranks for i in range(len(fba))], nranks) if fba else None
    geoms = [cgeom, fgeom]

    def program(ctx):
        levels = []
        for lv, (ba, dm, geom) in enumerate([(cba, cdm, cgeom)] + ([(fba, fdm, fgeom)] if fba else [])):
            u = MultiFab(ba, dm, 1, 1, geom=geom)
            w = MultiFab(ba, dm, 1, 1, geom=geom)
            for gi in u.local_indices:
                fill(u.fabs[gi], ba[gi], geom.domain, inputs.SEED + lv)
            w.setval(0.0)
            levels.append((u, w))
        ctx.barrier()
        be = Backend("serial")
        for _ in range(steps):
            comm.fill_boundary(levels[0][0], geoms[0], backend=be)
            if len(levels) > 1:
                amr.fill_patch(levels[1][0], levels[0][0], geoms[1], geoms[0], ratio, amr.LINEAR, backend=be)
            for lv, (u, w) in enumerate(levels):
                _advance_level(u, w, dt, diffusivity, geoms[lv], be)
            if len(levels) > 1:
                amr.average_down(levels[1][1], levels[0][1], ratio, be)
            levels = [(w, u) for (u, w) in levels]
        out = {}
        for lv, (u, w) in enumerate(levels):
            for gi in u.local_indices:
                out[(lv, "u", gi)] = inputs.bits(u.fabs[gi].data).copy(order="F")
                out[(lv, "w", gi)] = inputs.bits(w.fabs[gi].data).copy(order="F")
        return out

    for out in comm.runtime_spawn(nranks, program):
        for (lv, which, gi), a in out.items():
            ARRAYS[f"{name}/l{lv}{which}{gi}"] = a
    CASES.append(dict(name=name, kind="heat", dim=dim, cext=pad3(cext, 1), cmgs=cmgs,
                      fine_boxes=[box6(b) for b in (fine_boxes or [])], ratio=ratio, nranks=nranks, steps=steps,
                      dt=dt, diffusivity=diffusivity, dtype=np.dtype(dtype).name,
                      crse_boxes=[box6(b) for b in cba], crse_rank=list(cdm.rank_of),
                      fine_rank=list(fdm.rank_of) if fdm else []))
    reset_cfg()


def gen_heat(rng):
    run_heat("heat_1l_2d", 2, [16, 16], 8, None, 2, 1, 3, 1e-4, 1.0, np.float64)
    run_heat("heat_1l_3d_2r", 3, [12, 12, 12], 6, None, 2, 2, 2, 2e-5, 0.7, np.float64)
    run_heat("heat_1l_3d_f32", 3, [8, 8, 8], 4, None, 2, 1, 2, 1e-4, 1.0, np.float32)
    run_heat("heat_1l_1d", 1, [32], 8, None, 2, 2, 4, 1e-4, 1.0, np.float64)
    config.set_spacedim(2)
    run_heat("heat_2l_2d", 2, [16, 16], 8, [Box((8, 8), (23, 23))], 2, 1, 2, 2e-5, 1.0, np.float64)
    config.set_spacedim(2)
    run_heat("heat_2l_2d_2r", 2, [16, 16], 8, [Box((4, 8), (15, 23)), Box((16, 8), (27, 19))], 2, 2, 2, 2e-5,
             1.0, np.float64)
    config.set_spacedim(3)
    run_heat("heat_2l_3d", 3, [8, 8, 8], 4, [Box((4, 4, 4), (11, 11, 11))], 2, 2, 2, 1e-5, 1.0, np.float64)


# ------------------------------------------------------- index_mapped_copy

MAPPINGS = {
    "identity": lambda n: (lambda i, j, k: (i, j, k)),
    "reflect_x": lambda n: (lambda i, j, k: (n[0] - 1 - i, j, k)),
    "shift_wrap": lambda n: (lambda i, j, k: ((i + 3) % n[0], (j + 5) % n[1], k)),
    "transpose_xy": lambda n: (lambda i, j, k: (j, i, k)),
}


def run_index_copy(name, dim, ext, smgs, dmgs, nranks, ncomp, sng, dng, mapping, region, dtype):
    set_cfg(dim, dtype)
    dom = Box([0] * dim, [e - 1 for e in ext])
    sba, dba = decompose(dom, smgs), decompose(dom, dmgs)
    sdm = DistributionMapping([i % nranks for i in range(len(sba))], nranks)
    ddm = DistributionMapping([(i + 1) % nranks for i in range(len(dba))], nranks)
    fn = MAPPINGS[mapping](pad3(ext, 1))
    reg = None if region is None else Box(region[0][:dim], region[1][:dim])

    def program(ctx):
        src = MultiFab(sba, sdm, ncomp, sng)
        dst = MultiFab(dba, ddm, ncomp, dng)
        for gi in src.local_indices:
            fill(src.fabs[gi], sba[gi], dom, inputs.SEED)
        for gi in dst.local_indices:
            fill(dst.fabs[gi], dba[gi], dom, SEED_C)
        ctx.barrier()
        s0 = ctx.bus.stats_snapshot()
        ctx.barrier()  # no rank sends before every rank took its snapshot
        comm.index_mapped_copy(dst, src, fn, region=reg, backend=Backend("serial"))
        ctx.barrier()  # every rank's sends are in the Bus stats
        s1 = ctx.bus.stats_snapshot()
        stats = {f"{a}->{b}": (s1[(a, b)][0] - s0[(a, b)][0], s1[(a, b)][1] - s0[(a, b)][1])
                 for (a, b) in s1 if s1[(a, b)] != s0[(a, b)]}
        return {gi: inputs.bits(dst.fabs[gi].data).copy(order="F") for gi in dst.local_indices}, stats

    res = comm.runtime_spawn(nranks, program)
    for out, _ in res:
        for gi, a in out.items():
            ARRAYS[f"{name}/dst{gi}"] = a
    CASES.append(dict(name=name, kind="index_copy", dim=dim, ext=pad3(ext, 1), smgs=smgs, dmgs=dmgs, nranks=nranks,
                      ncomp=ncomp, sng=sng, dng=dng, mapping=mapping,
                      region=None if region is None else [pad3(region[0]), pad3(region[1])],
                      dtype=np.dtype(dtype).name, stats=res[0][1],
                      src_boxes=[box6(b) for b in sba], src_rank=list(sdm.rank_of),
                      dst_boxes=[box6(b) for b in dba], dst_rank=list(ddm.rank_of)))
    reset_cfg()


def gen_index_copy():
    run_index_copy("imc_identity_1d", 1, [16], 8, 8, 1, 1, 0, 0, "identity", None, np.float64)
    run_index_copy("imc_reflect_1d_2r", 1, [24], 8, 6, 2, 2, 0, 1, "reflect_x", None, np.float64)
    run_index_copy("imc_shift_2d", 2, [12, 10], 5, 4, 1, 2, 1, 1, "shift_wrap", None, np.float64)
    run_index_copy("imc_shift_2d_2r", 2, [12, 10], 6, 5, 2, 1, 0, 2, "shift_wrap", ([1, 2], [9, 8]), np.float32)
    run_index_copy("imc_transpose_3d_2r", 3, [8, 8, 6], 4, 3, 2, 2, 1, 0, "transpose_xy", None, np.float64)
    run_index_copy("imc_reflect_3d", 3, [10, 6, 6], 4, 5, 1, 3, 0, 0, "reflect_x", ([2, 0, 1], [8, 5, 4]),
                   np.float64)


def main():
    rng = np.random.default_rng(20261017)
    gen_interp(rng, 30)
    gen_avgdown(rng, 18)
    gen_fill_patch(rng, 18)
    gen_heat(rng)
    gen_index_copy()
    with open(os.path.join(HERE, "golden_amr.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden_amr.py", "reference": "miniamr_core (amr.py)",
                   "seed_fine": inputs.SEED, "seed_crse": SEED_C, "cases": CASES}, f, indent=0)
    np.savez_compressed(os.path.join(HERE, "golden_amr.npz"), **ARRAYS)
    print(f"{len(CASES)} cases, {len(ARRAYS)} arrays")


if __name__ == "__main__":
    main()
