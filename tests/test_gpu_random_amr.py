"""Randomised fill_patch / average_down layouts on the GPU against the oracle
replay of the reference algorithm (oracle/amr_oracle.py + ghost_oracle.py,
both pinned to reference fixtures): ratios 2 and 4, 2-D and 3-D, 1-3 ghosts,
LINEAR and piecewise constant, 1-2 thread ranks; raw bits."""

import numpy as np
import pytest

from gpu_util import bits_of, upload
from test_amr_oracle import avgdown_expected, fill_patch_expected, g3, grown, hashed, meta

pytestmark = pytest.mark.gpu


def _aligned_boxes(rng, dim, fext, ratio, nbox):
    out = []
    for _ in range(400):
        if len(out) == nbox:
            break
        lo = [int(rng.integers(0, fext[d] // ratio)) * ratio for d in range(dim)]
        ext = [int(rng.integers(1, 4)) * ratio for _ in range(dim)]
        hi = [min(l + e, fext[d]) - 1 for d, (l, e) in enumerate(zip(lo, ext))]
        if any((h - l + 1) % ratio for l, h in zip(lo, hi)):
            continue
        b = lo + hi
        if any(all(b[d] <= o[dim + d] and o[d] <= b[dim + d] for d in range(dim)) for o in out):
            continue
        out.append(b)
    out.sort()
    return [list(b[:dim]) + [0] * (3 - dim) + list(b[dim:]) + [0] * (3 - dim) for b in out]


def _case(rng, kind, seed):
    dim = 2 + seed % 2
    ratio = 4 if seed % 3 == 0 else 2
    cext = [int(rng.integers(4, 8 if dim == 3 else 12)) for _ in range(dim)]
    fext = [e * ratio for e in cext]
    boxes = _aligned_boxes(rng, dim, fext, ratio, int(rng.integers(1, 5)))
    nranks = int(rng.integers(1, 3))
    cmgs = int(rng.integers(2, 6))
    import paper_2403_12179_b200 as amr
    amr.config.set_spacedim(dim)
    cba = amr.decompose(amr.Box((0,) * dim, tuple(e - 1 for e in cext)), cmgs)
    minext = min(min(b[3 + d] - b[d] + 1 for d in range(dim)) for b in boxes)
    c = dict(kind=kind, dim=dim, ratio=ratio, cext=cext + [1] * (3 - dim), cmgs=cmgs, fine_boxes=boxes,
             nranks=nranks, ncomp=int(rng.integers(1, 3)), fngrow=int(rng.integers(1, min(3, minext) + 1)),
             cngrow=int(rng.integers(0, 2)), periodic=[True] * dim + [False] * (3 - dim),
             scheme="linear" if seed % 2 == 0 else "piecewise_constant", dtype="float64",
             crse_boxes=[list(b.as_row()) for b in cba], crse_rank=[i % nranks for i in range(len(cba))],
             fine_rank=[(i + 1) % nranks for i in range(len(boxes))])
    return c


def _run(c):
    import paper_2403_12179_b200 as amr
    from paper_2403_12179_b200 import amr as A
    dim, nc, dt, r = c["dim"], c["ncomp"], np.dtype(c["dtype"]), c["ratio"]
    amr.config.set_spacedim(dim)
    amr.config.set_real_dtype(dt)
    box = lambda b6: amr.Box(tuple(b6[:dim]), tuple(b6[3:3 + dim]))  # noqa: E731
    cdom6 = [0, 0, 0] + [e - 1 for e in c["cext"]]
    fdom6 = [0, 0, 0] + [e * (r if d < dim else 1) - 1 for d, e in enumerate(c["cext"])]
    cgeom = amr.Geometry(box(cdom6), (0.0,) * dim, (1.0,) * dim, (True,) * dim)
    fgeom = cgeom.refined(r)
    cba = amr.BoxArray([box(b) for b in c["crse_boxes"]])
    fba = amr.BoxArray([box(b) for b in c["fine_boxes"]])
    cdm = amr.DistributionMapping(c["crse_rank"], c["nranks"])
    fdm = amr.DistributionMapping(c["fine_rank"], c["nranks"])
    cng = c["cngrow"] if c["kind"] == "average_down" else 0

    def program(ctx):
        coarse = amr.MultiFab(cba, cdm, nc, cng, cgeom)
        fine = amr.MultiFab(fba, fdm, nc, c["fngrow"], fgeom)
        for gi in coarse.local_indices:
            b = np.asarray(c["crse_boxes"][gi])
            upload(coarse.fabs[gi], hashed(grown(b, g3(cng, dim)), b, np.asarray(cdom6), nc, dt, meta()["seed_crse"]))
        for gi in fine.local_indices:
            b = np.asarray(c["fine_boxes"][gi])
            upload(fine.fabs[gi], hashed(grown(b, g3(c["fngrow"], dim)), b, np.asarray(fdom6), nc, dt,
                                         meta()["seed_fine"]))
        ctx.barrier()
        if c["kind"] == "fill_patch":
            A.fill_patch(fine, coarse, fgeom, cgeom, r, c["scheme"])
            A.fill_patch(fine, coarse, fgeom, cgeom, r, c["scheme"])
            return {gi: bits_of(fine.fabs[gi]) for gi in fine.local_indices}
        A.average_down(fine, coarse, r)
        return {gi: bits_of(coarse.fabs[gi]) for gi in coarse.local_indices}

    got = {}
    for res in amr.runtime_spawn(c["nranks"], program):
        got.update(res)
    return got


@pytest.mark.parametrize("seed", range(10))
def test_random_fill_patch_matches_oracle(seed):
    c = _case(np.random.default_rng(3000 + seed), "fill_patch", seed)
    got = _run(c)
    exp = fill_patch_expected(c)
    for gi, a in exp.items():
        assert np.array_equal(got[gi], a.view(np.uint64).ravel(order="F")), gi


@pytest.mark.parametrize("seed", range(10))
def test_random_average_down_matches_oracle(seed):
    c = _case(np.random.default_rng(4000 + seed), "average_down", seed)
    got = _run(c)
    exp = avgdown_expected(c)
    for gi, a in exp.items():
        assert np.array_equal(got[gi], a.view(np.uint64).ravel(order="F")), gi
