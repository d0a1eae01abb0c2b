"""Host-side drop-in surface on CPU: index algebra, BoxArray / DM / plan API,
rank runtime (reference tests/test_index_space.py, test_mesh.py,
test_comm.py semantics).  No device needed: MultiFabs here own no boxes on
the calling rank, so nothing is allocated."""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2403_12179_b200 as amr
from paper_2403_12179_b200 import comm, config
from paper_2403_12179_b200.index_space import (Box, Geometry, IndexType, IntVect, box_diff, coarsen, convert,
                                              empty_box, grow, intersect, num_pts, periodic_shift_images,
                                              refine)


def boxes3(max_abs=10, max_extent=8):
    lo = st.tuples(*[st.integers(-max_abs, max_abs)] * 3)
    ext = st.tuples(*[st.integers(1, max_extent)] * 3)
    return st.builds(lambda l, e: Box(l, tuple(a + b - 1 for a, b in zip(l, e))), lo, ext)


# ------------------------------------------------------------ index space

def test_intersect_and_grow_examples():
    a = Box((0, 0, 0), (3, 3, 3))
    assert intersect(a, Box((2, 2, 2), (5, 5, 5))) == Box((2, 2, 2), (3, 3, 3))
    with pytest.raises(ValueError):
        intersect(a, Box((0, 0, 0), (3, 3, 3), IndexType.node()))
    config.set_spacedim(2)
    assert grow(Box((0, 0), (7, 7)), 2) == Box((-2, -2), (9, 9))
    e = intersect(Box((0, 0), (3, 3)), Box((5, 5), (7, 7)))
    assert e == empty_box(IndexType.cell()) and e.hi == IntVect(-1, -1)
    config.set_spacedim(1)
    assert grow(Box((0,), (1,)), -1).is_empty


@given(boxes3(), boxes3(), boxes3())
@settings(max_examples=100, deadline=None)
def test_intersect_properties(a, b, c):
    ab = intersect(a, b)
    assert ab == intersect(b, a)
    assert intersect(ab, c) == intersect(a, intersect(b, c))
    if not ab.is_empty:
        assert a.contains(ab) and b.contains(ab)


@given(boxes3(), boxes3())
@settings(max_examples=100, deadline=None)
def test_box_diff_partition(a, b):
    parts = box_diff(a, b)
    assert num_pts(a) == num_pts(intersect(a, b)) + sum(num_pts(p) for p in parts)
    for n, p in enumerate(parts):
        assert a.contains(p) and intersect(p, b).is_empty
        for q in parts[n + 1:]:
            assert intersect(p, q).is_empty


def test_refine_coarsen_convert():
    b = Box((1, 2, 3), (4, 5, 6))
    assert coarsen(refine(b, 2), 2) == b
    assert convert(b, IndexType.node()).hi == IntVect(5, 6, 7)


def test_periodic_shift_images():
    config.set_spacedim(1)
    g = Geometry(Box((0,), (7,)), (0.0,), (1.0,), (True,))
    got = {(im.lo[0], im.hi[0], s[0]) for im, s in periodic_shift_images(Box((-1,), (0,)), g)}
    assert got == {(-1, 0, 0), (7, 8, 8)}
    config.set_spacedim(2)
    gp = Geometry(Box((0, 0), (7, 7)), (0, 0), (1, 1), (True, True))
    interior = Box((2, 2), (5, 5))
    im = periodic_shift_images(interior, gp)
    assert len(im) == 1 and im[0][0] == interior


def test_geometry_validation():
    with pytest.raises(ValueError):
        Geometry(Box((0, 0, 0), (3, 3, 3), IndexType.node()), (0,) * 3, (1,) * 3, (True,) * 3)
    g = Geometry(Box((0, 0, 0), (7, 3, 1)), (0,) * 3, (1,) * 3, (True,) * 3)
    assert g.period == (8, 4, 2)


# ------------------------------------------------------------------ mesh

def test_boxarray_disjointness_and_decompose_order():
    with pytest.raises(ValueError, match="disjoint"):
        amr.BoxArray([Box((0, 0, 0), (3, 3, 3)), Box((3, 0, 0), (5, 3, 3))])
    ba = amr.decompose(Box((0, 0, 0), (7, 7, 7)), 4)
    assert len(ba) == 8
    assert [b.lo.comps for b in ba][:3] == [(0, 0, 0), (4, 0, 0), (0, 4, 0)]  # x fastest
    assert ba.minimal_extent() == 4


def test_boxarray_large_is_fast():
    import time
    t0 = time.perf_counter()
    ba = amr.decompose(Box((0, 0, 0), (255, 255, 255)), 16)
    assert len(ba) == 4096
    assert time.perf_counter() - t0 < 10.0  # the reference's O(n^2) check needs ~126 s


def test_distribution_mapping():
    dm = amr.DistributionMapping.round_robin(5, 2)
    assert dm.rank_of == (0, 1, 0, 1, 0) and dm.nranks == 2
    with pytest.raises(ValueError):
        amr.DistributionMapping([0, 3], nranks=2)


def _remote_mf(ba, ncomp, ngrow, geom=None, nranks=2):
    """A MultiFab whose boxes all live on another rank (no allocation)."""
    dm = amr.DistributionMapping([1] * len(ba), nranks)
    return amr.MultiFab(ba, dm, ncomp, ngrow, geom, rank=0)


def test_multifab_validation():
    config.set_spacedim(1)
    ba = amr.BoxArray([Box((i * 4,), (i * 4 + 3,)) for i in range(4)])
    with pytest.raises(ValueError):
        amr.MultiFab(ba, amr.DistributionMapping([0]), 1, 0)
    mf = amr.MultiFab(ba, amr.DistributionMapping([1, 2, 1, 2], 3), 1, 0, rank=0)
    assert mf.local_indices == () and mf.fabs == {}
    with pytest.raises(ValueError):
        amr.MultiFab(ba, amr.DistributionMapping([1] * 4, 2), 1, -1, rank=0)


# ------------------------------------------------------------- plan API

def test_plan_1d_periodic_example_and_cache():
    """Reference tests/test_comm.py:168-177."""
    config.set_spacedim(1)
    geom = Geometry(Box((0,), (7,)), (0.0,), (1.0,), (True,))
    ba = amr.BoxArray([Box((0,), (3,)), Box((4,), (7,))])
    mf = _remote_mf(ba, 1, 1, geom)
    plan = amr.plan_build_fill_boundary(mf, geom)
    assert plan.num_segments == 4 and mf.plan_builds == 1
    again = amr.plan_build_fill_boundary(mf, geom)
    assert again is plan and mf.plan_builds == 1
    segs = plan.local_by_rank[1]
    assert [(s.src_fab, s.dst_fab, s.dst_box.lo[0], s.shift) for s in segs] == \
        [(1, 0, -1, (-8,)), (1, 0, 4, (0,)), (0, 1, 3, (0,)), (0, 1, 8, (8,))]
    assert segs[0].src_box == Box((7,), (7,))


def test_plan_ngrow_zero_empty_and_errors():
    config.set_spacedim(1)
    geom = Geometry(Box((0,), (7,)), (0.0,), (1.0,), (True,))
    ba = amr.BoxArray([Box((0,), (3,)), Box((4,), (7,))])
    assert amr.plan_build_fill_boundary(_remote_mf(ba, 1, 0, geom), geom).is_empty
    with pytest.raises(ValueError):
        amr.plan_build_fill_boundary(_remote_mf(ba, 1, 1))  # no geometry
    with pytest.raises(ValueError):
        amr.plan_build_fill_boundary(_remote_mf(ba, 1, 5, geom), geom)  # ngrow > minimal extent
    config.set_spacedim(2)
    mixed = IndexType(0, 1)
    g2 = Geometry(Box((0, 0), (7, 7)), (0, 0), (1, 1), (True, True))
    mf = _remote_mf(amr.BoxArray([Box((0, 0), (7, 7), mixed)]), 1, 1, g2)
    with pytest.raises(ValueError):
        amr.plan_build_fill_boundary(mf, g2)


def test_plan_shared_across_multifabs_counts_per_multifab():
    """tests/test_acceptance.py:157-171: plan_builds == 1 per MultiFab even
    when several per-rank MultiFabs share a BoxArray."""
    config.set_spacedim(2)
    dom = Box((0, 0), (11, 11))
    geom = Geometry(dom, (0, 0), (1, 1), (True, True))
    ba = amr.decompose(dom, 6)
    a = _remote_mf(ba, 1, 1, geom)
    b = _remote_mf(ba, 1, 1, geom)
    pa = amr.plan_build_fill_boundary(a, geom)
    pb = amr.plan_build_fill_boundary(b, geom)
    assert a.plan_builds == b.plan_builds == 1
    assert pa.num_segments == pb.num_segments


def test_plan_pairs_and_messages():
    """Aggregation layout of tests/test_comm.py:407-422: 12 active ordered
    pairs, every pair exactly one message."""
    config.set_spacedim(2)
    dom = Box((0, 0), (11, 11))
    geom = Geometry(dom, (0, 0), (1, 1), (True, True))
    ba = amr.decompose(dom, 6)
    dm = amr.DistributionMapping.round_robin(len(ba), 4)
    mf = amr.MultiFab(ba, amr.DistributionMapping(dm.rank_of, 5), 1, 1, geom, rank=4)
    plan = amr.plan_build_fill_boundary(mf, geom)
    assert len(plan.pair_segments) == 12
    assert set(plan.sends_from(0)) == {1, 2, 3}
    pc = plan.pair_cells
    assert pc[0, 1] == 12 and pc[0, 3] == 4  # 2 faces x 6 cells; 4 corners


def test_parallel_copy_argument_errors():
    config.set_spacedim(1)
    sba = amr.BoxArray([Box((0,), (3,))])
    dba = amr.BoxArray([Box((10,), (13,))])
    src = _remote_mf(sba, 2, 0)
    dst = _remote_mf(dba, 2, 0)
    with pytest.raises(ValueError):
        amr.parallel_copy(dst, src, scomp=2, ncomp=1)
    nodal = amr.BoxArray([Box((0,), (3,), IndexType.node())])
    with pytest.raises(ValueError):
        amr.parallel_copy(dst, _remote_mf(nodal, 2, 0))


# -------------------------------------------------------------- runtime

def test_runtime_spawn_single_rank():
    seen = []

    def program(ctx):
        seen.append(ctx.bus.stats_snapshot())
        return ctx.rank * 10

    assert amr.runtime_spawn(1, program) == [0]
    assert all(v == (0, 0) for v in seen[0].values())


def test_ping_pong_message_stats():
    buses = []

    def program(ctx):
        buses.append(ctx.bus)
        if ctx.rank == 0:
            ctx.send(1, b"ping", nbytes=4)
            return ctx.recv(1)
        got = ctx.recv(0)
        ctx.send(0, b"pong", nbytes=4)
        return got

    assert amr.runtime_spawn(2, program) == [b"pong", b"ping"]
    s = buses[0].stats_snapshot()
    assert s[(0, 1)] == (1, 4) and s[(1, 0)] == (1, 4)


def test_rank_failure_propagates():
    def program(ctx):
        if ctx.rank == 1:
            raise RuntimeError("boom")
        ctx.barrier()

    with pytest.raises(amr.RankFailure) as ei:
        amr.runtime_spawn(2, program)
    assert ei.value.rank == 1


def test_global_reduce():
    def program(ctx):
        v = float(ctx.rank + 1)
        return amr.global_reduce([amr.SUM, amr.MIN, amr.MAX], [v, v, v], ctx)

    assert amr.runtime_spawn(4, program) == [(10.0, 1.0, 4.0)] * 4

    def bad(ctx):
        return amr.global_reduce([amr.SUM] if ctx.rank == 0 else [amr.MIN], [1.0], ctx)

    with pytest.raises(amr.RankFailure):
        amr.runtime_spawn(2, bad)


def test_bus_accounting_format():
    bus = comm.Bus(2)
    bus.account(0, 1, 96)
    assert bus.stats_snapshot()[(0, 1)] == (1, 96)
    assert "0->1: 1 messages, 96 bytes" in bus.format_stats()
