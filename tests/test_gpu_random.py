"""Randomised FillBoundary layouts (anisotropic ghosts, odd extents, mixed
periodicity, float32/float64, device and pinned host memory, every task
variant of the fused kernel) against the CPU oracle (oracle/ghost_oracle.py,
itself pinned to the reference's golden vectors): raw bits."""

import numpy as np
import pytest

from gpu_util import bits_of
from oracle import ghost_oracle as go
from oracle import inputs

pytestmark = pytest.mark.gpu

VARIANTS = [{}, {"GHX_FAB_LOCAL": "0", "GHX_BULK": "1"}, {"GHX_FAB_LOCAL": "1"}, {"GHX_RING": "1"},
            {"GHX_PHASED": "1"}, {"GHX_PHASED": "1", "GHX_RING": "1"}]


def _layout(rng):
    ext = [int(rng.integers(6, 40)) for _ in range(3)]
    cuts = [np.unique(np.concatenate([[0], rng.integers(3, e - 2, int(rng.integers(0, 3))), [e]])) for e in ext]
    boxes = np.asarray([[x0, y0, z0, x1 - 1, y1 - 1, z1 - 1]
                        for z0, z1 in zip(cuts[2][:-1], cuts[2][1:])
                        for y0, y1 in zip(cuts[1][:-1], cuts[1][1:])
                        for x0, x1 in zip(cuts[0][:-1], cuts[0][1:])], np.int64)
    minext = int((boxes[:, 3:] - boxes[:, :3] + 1).min())  # the reference bounds max(ngrow) by it
    ng = [int(rng.integers(0, min(3, minext) + 1)) for _ in range(3)]
    per = [bool(v) for v in rng.integers(0, 2, 3)]
    return ext, boxes, ng, per


@pytest.mark.parametrize("seed", range(36))
def test_random_fill_boundary_matches_oracle(seed, monkeypatch):
    import paper_2403_12179_b200 as amr
    rng = np.random.default_rng(1000 + seed)
    ext, boxes, ng, per = _layout(rng)
    nc = int(rng.integers(1, 4))
    dt = np.float32 if seed % 5 == 4 else np.float64
    memory = "pinned" if seed % 7 == 3 else "device"
    for k, v in VARIANTS[seed % len(VARIANTS)].items():
        monkeypatch.setenv(k, v)
    amr.config.set_spacedim(3)
    amr.config.set_real_dtype(dt)
    dom = amr.Box((0, 0, 0), tuple(e - 1 for e in ext))
    geom = amr.Geometry(dom, (0.0,) * 3, (1.0,) * 3, tuple(per))
    ba = amr.BoxArray([amr.Box(tuple(b[:3]), tuple(b[3:])) for b in boxes])
    dm = amr.DistributionMapping([0] * len(ba))
    mf = amr.MultiFab(ba, dm, nc, amr.IntVect(*ng), geom, memory=memory)
    mf.fill_hash(inputs.SEED, dom)
    import torch
    torch.cuda.synchronize()
    amr.fill_boundary(mf, geom)
    # oracle
    plan = go.plan_fill_boundary(boxes, ng, per, ext, [0] * len(boxes), 1)
    fabs, lo = {}, {}
    for gi, b in enumerate(boxes):
        g = b.copy()
        g[:3] -= ng
        g[3:] += ng
        fabs[gi] = inputs.make_fab(g[:3], g[3:], nc, dt, b[:3], b[3:], [0] * 3, [e - 1 for e in ext])
        lo[gi] = g[:3]
    go.execute(plan, fabs, lo, fabs, lo, 0, 0, nc)
    for gi in range(len(boxes)):
        assert np.array_equal(bits_of(mf.fabs[gi]), inputs.bits(fabs[gi]).ravel(order="F")), f"fab {gi}"


def _cuts(rng, e, k):
    return np.unique(np.concatenate([[0], rng.integers(3, e - 2, k), [e]]))


def _boxes(cuts):
    return np.asarray([[x0, y0, z0, x1 - 1, y1 - 1, z1 - 1]
                       for z0, z1 in zip(cuts[2][:-1], cuts[2][1:])
                       for y0, y1 in zip(cuts[1][:-1], cuts[1][1:])
                       for x0, x1 in zip(cuts[0][:-1], cuts[0][1:])], np.int64)


@pytest.mark.parametrize("seed", range(12))
def test_random_parallel_copy_matches_oracle(seed, monkeypatch):
    """Distinct source / destination MultiFabs with wide rows: the TMA
    bulk-row path of ParallelCopy (and its LSU twin) against the oracle."""
    import paper_2403_12179_b200 as amr
    rng = np.random.default_rng(2000 + seed)
    if seed % 3 == 2:
        monkeypatch.setenv("GHX_PC_BULK", "0")
    ext = [int(rng.integers(40, 97)), int(rng.integers(6, 20)), int(rng.integers(6, 16))]
    sb = _boxes([_cuts(rng, e, int(rng.integers(0, 3))) for e in ext])
    db = _boxes([_cuts(rng, e, int(rng.integers(0, 3))) for e in ext])
    gs, gd = int(rng.integers(0, 2)), int(rng.integers(0, 3))
    nc_s, nc_d = int(rng.integers(1, 4)), int(rng.integers(1, 4))
    ncomp = int(rng.integers(1, min(nc_s, nc_d) + 1))
    scomp, dcomp = int(rng.integers(0, nc_s - ncomp + 1)), int(rng.integers(0, nc_d - ncomp + 1))
    dt = np.float32 if seed % 4 == 3 else np.float64
    amr.config.set_spacedim(3)
    amr.config.set_real_dtype(dt)
    dom = [0, 0, 0] + [e - 1 for e in ext]
    sba = amr.BoxArray([amr.Box(tuple(b[:3]), tuple(b[3:])) for b in sb])
    dba = amr.BoxArray([amr.Box(tuple(b[:3]), tuple(b[3:])) for b in db])
    src = amr.MultiFab(sba, amr.DistributionMapping([0] * len(sba)), nc_s, gs)
    dst = amr.MultiFab(dba, amr.DistributionMapping([0] * len(dba)), nc_d, gd)
    from gpu_util import upload
    hsrc, hdst, slo, dlo = {}, {}, {}, {}
    for gi, b in enumerate(sb):
        g = b.copy()
        g[:3] -= gs
        g[3:] += gs
        hsrc[gi] = inputs.make_fab(g[:3], g[3:], nc_s, dt, b[:3], b[3:], dom[:3], dom[3:], ghost_tag=gi)
        slo[gi] = g[:3]
        upload(src.fabs[gi], hsrc[gi])
    for gi, b in enumerate(db):
        g = b.copy()
        g[:3] -= gd
        g[3:] += gd
        hdst[gi] = inputs.make_fab(g[:3], g[3:], nc_d, dt, b[:3], b[3:], dom[:3], dom[3:], seed=inputs.SEED + 7)
        dlo[gi] = g[:3]
        upload(dst.fabs[gi], hdst[gi])
    amr.parallel_copy(dst, src, scomp, dcomp, ncomp, ngrow_src=gs, ngrow_dst=gd)
    plan = go.plan_parallel_copy(db, sb, [gd] * 3, [gs] * 3, None, None, [0] * len(sb), [0] * len(db), 1)
    go.execute(plan, hsrc, slo, hdst, dlo, scomp, dcomp, ncomp)
    for gi in range(len(db)):
        assert np.array_equal(bits_of(dst.fabs[gi]), inputs.bits(hdst[gi]).ravel(order="F")), f"fab {gi}"
