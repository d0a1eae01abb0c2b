"""Edge cases of FillBoundary on the device against the CPU oracle
(oracle/ghost_oracle.py, pinned to the reference's golden vectors): empty
plans, a single box that is its own periodic neighbour at the maximal ghost
width the reference allows (comm.py:302-303, ngrow <= minimal extent),
one-cell boxes, more ranks than boxes (ranks with no fabs), many components.
Raw bits compared."""

import numpy as np
import pytest

from gpu_util import bits_of
from oracle import ghost_oracle as go
from oracle import inputs

pytestmark = pytest.mark.gpu


def _expected(boxes, ng, per, ext, nc, dt):
    """Oracle FillBoundary over 3-D padded boxes (spacedim < 3: extent 1,
    ngrow 0, not periodic on the padded axes)."""
    plan = go.plan_fill_boundary(boxes, ng, per, ext, [0] * len(boxes), 1)
    fabs, lo = {}, {}
    for gi, b in enumerate(boxes):
        g = b.copy()
        g[:3] -= ng
        g[3:] += ng
        fabs[gi] = inputs.make_fab(g[:3], g[3:], nc, dt, b[:3], b[3:], [0] * 3, [e - 1 for e in ext])
        lo[gi] = g[:3]
    go.execute(plan, fabs, lo, fabs, lo, 0, 0, nc)
    return {gi: inputs.bits(f).ravel(order="F") for gi, f in fabs.items()}


def _setup(amr, dim, ext, boxes, dt):
    amr.config.set_spacedim(dim)
    amr.config.set_real_dtype(dt)
    dom = amr.Box((0,) * dim, tuple(e - 1 for e in ext[:dim]))
    ba = amr.BoxArray([amr.Box(tuple(b[:dim]), tuple(b[3:3 + dim])) for b in boxes])
    return dom, ba


def _pad(ext, boxes, ng, per, dim):
    ext3 = list(ext[:dim]) + [1] * (3 - dim)
    b3 = np.asarray([list(b[:dim]) + [0] * (3 - dim) + list(b[3:3 + dim]) + [0] * (3 - dim) for b in boxes],
                    np.int64)
    return ext3, b3, list(ng[:dim]) + [0] * (3 - dim), list(per[:dim]) + [False] * (3 - dim)


def test_no_tags_leaves_every_byte_untouched():
    import torch
    import paper_2403_12179_b200 as amr
    dom, ba = _setup(amr, 3, [6, 5, 4], [[0, 0, 0, 5, 4, 3]], np.float64)
    geom = amr.Geometry(dom, (0.0,) * 3, (1.0,) * 3, (False,) * 3)
    mf = amr.MultiFab(ba, amr.DistributionMapping([0]), 3, 2, geom)
    mf.fill_hash(inputs.SEED, dom)
    torch.cuda.synchronize()
    before = bits_of(mf.fabs[0]).copy()
    plan = amr.plan_build_fill_boundary(mf, geom)
    assert plan.is_empty and plan.num_segments == 0
    amr.fill_boundary(mf, geom)
    assert np.array_equal(bits_of(mf.fabs[0]), before)


@pytest.mark.parametrize("dim,ext", [(1, [5]), (2, [3, 7]), (3, [3, 4, 5])])
@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_single_box_is_its_own_periodic_neighbour_at_max_ngrow(dim, ext, dt):
    """ngrow = minimal extent: every ghost (corners too) is a periodic image
    of the box itself, some images several periods away."""
    import torch
    import paper_2403_12179_b200 as amr
    ng = [min(ext)] * dim
    box = [[0, 0, 0, *[e - 1 for e in ext] + [0] * (3 - dim)]]
    dom, ba = _setup(amr, dim, ext, box, dt)
    geom = amr.Geometry(dom, (0.0,) * dim, (1.0,) * dim, (True,) * dim)
    mf = amr.MultiFab(ba, amr.DistributionMapping([0]), 2, amr.IntVect(*ng), geom)
    mf.fill_hash(inputs.SEED, dom)
    torch.cuda.synchronize()
    amr.fill_boundary(mf, geom)
    ext3, b3, ng3, per3 = _pad(ext, box, ng, [True] * dim, dim)
    exp = _expected(b3, ng3, per3, ext3, 2, dt)
    assert np.array_equal(bits_of(mf.fabs[0]), exp[0])


@pytest.mark.parametrize("nranks", [3, 5])
def test_one_cell_boxes_with_more_ranks_than_boxes(nranks):
    """2-D, 2 x 2 one-cell boxes, ngrow 1, periodic: with 5 ranks one rank
    owns nothing and still takes part in every barrier."""
    import torch
    import paper_2403_12179_b200 as amr
    ext = [2, 2]
    boxes = [[i, j, 0, i, j, 0] for j in range(2) for i in range(2)]
    dom, ba = _setup(amr, 2, ext, boxes, np.float64)
    geom = amr.Geometry(dom, (0.0,) * 2, (1.0,) * 2, (True, True))
    dm = amr.DistributionMapping([k % nranks for k in range(len(boxes))], nranks)

    def program(ctx):
        mf = amr.MultiFab(ba, dm, 1, 1, geom)
        mf.fill_hash(inputs.SEED, dom)
        torch.cuda.synchronize()
        ctx.barrier()
        amr.fill_boundary(mf, geom)
        amr.fill_boundary(mf, geom)
        return {gi: bits_of(mf.fabs[gi]) for gi in mf.local_indices}

    got = {}
    for r in amr.runtime_spawn(nranks, program):
        got.update(r)
    assert sorted(got) == list(range(len(boxes)))
    ext3, b3, ng3, per3 = _pad(ext, boxes, [1, 1], [True, True], 2)
    exp = _expected(b3, ng3, per3, ext3, 1, np.float64)
    for gi in got:
        assert np.array_equal(got[gi], exp[gi]), f"fab {gi}"


def test_many_components_float32_anisotropic_ghosts():
    import torch
    import paper_2403_12179_b200 as amr
    ext = [12, 9, 10]
    cuts = [[0, 5, 12], [0, 4, 9], [0, 3, 10]]
    boxes = [[x0, y0, z0, x1 - 1, y1 - 1, z1 - 1]
             for z0, z1 in zip(cuts[2][:-1], cuts[2][1:])
             for y0, y1 in zip(cuts[1][:-1], cuts[1][1:])
             for x0, x1 in zip(cuts[0][:-1], cuts[0][1:])]
    ng, per, nc = [1, 3, 0], [True, True, False], 19
    dom, ba = _setup(amr, 3, ext, boxes, np.float32)
    geom = amr.Geometry(dom, (0.0,) * 3, (1.0,) * 3, tuple(per))
    mf = amr.MultiFab(ba, amr.DistributionMapping([0] * len(ba)), nc, amr.IntVect(*ng), geom)
    mf.fill_hash(inputs.SEED, dom)
    torch.cuda.synchronize()
    amr.fill_boundary(mf, geom)
    exp = _expected(np.asarray(boxes, np.int64), ng, per, ext, nc, np.float32)
    for gi in range(len(boxes)):
        assert np.array_equal(bits_of(mf.fabs[gi]), exp[gi]), f"fab {gi}"
