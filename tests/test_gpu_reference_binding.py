"""The reference-side binding (integration/reference_binding.py, the stub of
INTEGRATION.md section 2) driving libghostx.so through the plain C ABI on
the REFERENCE's own objects: miniamr_core's MultiFab / Fab with their numpy
storage allocated from pinned, mapped host memory.  Its FillBoundary and
interp_box must equal the reference's own functions on twin objects bit for
bit.  Needs the reference install in baseline/_ref (skipped without it)."""

import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.environ.get("MINIAMR_REF", os.path.join(REPO, "baseline", "_ref"))


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(os.path.join(REF, "miniamr_core")):
        pytest.skip("reference install (baseline/_ref) not present")
    sys.path.insert(0, REF)
    import miniamr_core
    from miniamr_core import amr, comm, config, index_space, kernels, mesh
    # the reference's defined semantics come from its serial backend: its
    # parallel backend races on overlapping destinations (ParallelCopy with
    # source ghosts, reference a11), so the comparisons use Backend("serial")
    miniamr_core._serial = kernels.Backend("serial")
    yield miniamr_core, amr, comm, config, index_space, mesh
    sys.path.remove(REF)


def _fill(mf, seed):
    rng = np.random.default_rng(seed)
    for i in mf.local_indices:
        a = mf.fabs[i].data
        a[...] = rng.standard_normal(a.shape)


@pytest.mark.parametrize("dim,n,b,nc,ng,per", [(3, 32, 16, 2, 2, (1, 1, 1)), (3, 24, 8, 1, 1, (1, 0, 1)),
                                                (2, 40, 16, 3, 2, (1, 1)), (3, 20, (8, 12, 20), 2, 1, (0, 1, 1))])
def test_fill_boundary_through_c_abi_equals_reference(ref, dim, n, b, nc, ng, per):
    _, _, comm, config, ix, mesh = ref
    from integration.reference_binding import PinnedArena, fill_boundary_native
    config.set_spacedim(dim) if hasattr(config, "set_spacedim") else None
    dom = ix.Box((0,) * dim, (n - 1,) * dim)
    geom = ix.Geometry(dom, (0.0,) * dim, (1.0,) * dim, per)
    ba = mesh.decompose(dom, b if isinstance(b, int) else list(b[:dim]))
    dm = mesh.DistributionMapping.round_robin(len(ba), 1)
    ours = mesh.MultiFab(ba, dm, nc, ng, geom, arena=PinnedArena())
    theirs = mesh.MultiFab(ba, dm, nc, ng, geom)
    _fill(ours, 7)
    _fill(theirs, 7)
    for _ in range(2):
        fill_boundary_native(ours, geom)
        comm.fill_boundary(theirs, geom, backend=ref[0]._serial)
    for i in ours.local_indices:
        got = ours.fabs[i].data.view(np.uint64)
        exp = theirs.fabs[i].data.view(np.uint64)
        assert np.array_equal(got, exp), f"fab {i}"


@pytest.mark.parametrize("scheme", ["piecewise_constant", "linear"])
def test_interp_box_through_c_abi_equals_reference(ref, scheme):
    _, amr, _, config, ix, mesh = ref
    from integration.reference_binding import PinnedArena, interp_box_native
    config.set_spacedim(3) if hasattr(config, "set_spacedim") else None
    arena = PinnedArena()
    cbox = ix.Box((3, 2, 4), (12, 11, 13))
    fbox = ix.Box((8, 6, 10), (21, 19, 23))
    region = ix.Box((9, 7, 11), (20, 18, 22))
    rng = np.random.default_rng(3)
    c_ours, c_ref = mesh.Fab(cbox, 2, arena), mesh.Fab(cbox, 2)
    f_ours, f_ref = mesh.Fab(fbox, 2, arena), mesh.Fab(fbox, 2)
    c_ours.data[...] = c_ref.data[...] = rng.standard_normal(c_ref.data.shape)
    f_ours.data[...] = f_ref.data[...] = rng.standard_normal(f_ref.data.shape)
    interp_box_native(c_ours, f_ours, region, 2, scheme)
    amr.interp_box(c_ref, f_ref, region, 2, scheme)
    assert np.array_equal(f_ours.data.view(np.uint64), f_ref.data.view(np.uint64))


@pytest.mark.parametrize("n,sb,db,nc,gs,gd,periodic", [(32, 8, 16, 2, 0, 0, None), (24, 12, 8, 1, 1, 2, (1, 1, 1)),
                                                       (32, 16, 8, 3, 0, 1, (0, 1, 1))])
def test_parallel_copy_through_c_abi_equals_reference(ref, n, sb, db, nc, gs, gd, periodic):
    _, _, comm, config, ix, mesh = ref
    from integration.reference_binding import PinnedArena, parallel_copy_native
    config.set_spacedim(3)
    dom = ix.Box((0, 0, 0), (n - 1,) * 3)
    geom = ix.Geometry(dom, (0.0,) * 3, (1.0,) * 3, periodic) if periodic else None
    sba, dba = mesh.decompose(dom, sb), mesh.decompose(dom, db)
    sdm = mesh.DistributionMapping.round_robin(len(sba), 1)
    ddm = mesh.DistributionMapping.round_robin(len(dba), 1)
    arena = PinnedArena()
    src_o, dst_o = mesh.MultiFab(sba, sdm, nc, gs, arena=arena), mesh.MultiFab(dba, ddm, nc + 1, gd, arena=arena)
    src_r, dst_r = mesh.MultiFab(sba, sdm, nc, gs), mesh.MultiFab(dba, ddm, nc + 1, gd)
    _fill(src_o, 11)
    _fill(src_r, 11)
    _fill(dst_o, 12)
    _fill(dst_r, 12)
    parallel_copy_native(dst_o, src_o, 0, 1, nc, gs, gd, geom)
    comm.parallel_copy(dst_r, src_r, 0, 1, nc, gs, gd, geom, backend=ref[0]._serial)
    for i in dst_o.local_indices:
        assert np.array_equal(dst_o.fabs[i].data.view(np.uint64), dst_r.fabs[i].data.view(np.uint64)), f"fab {i}"


def _fill_by_fab(mf, seed):
    """Rank-independent data: fab i's values depend on (seed, i) only."""
    for i in mf.local_indices:
        a = mf.fabs[i].data
        a[...] = np.random.default_rng(seed * 1000 + i).standard_normal(a.shape)


def _spawn(comm, nranks, program):
    """runtime_spawn(program) -> (per-rank results, the Bus message stats)."""
    stats = {}

    def prog(ctx):
        out = program(ctx)
        ctx.barrier()
        if ctx.rank == 0:
            stats.update(ctx.bus.stats_snapshot())
        return out
    return comm.runtime_spawn(nranks, prog), stats


@pytest.mark.parametrize("nranks", [2, 3, 4])
@pytest.mark.parametrize("dim,n,b,nc,ng,per", [(3, 32, 16, 2, 2, (1, 1, 1)), (3, 24, 8, 1, 1, (1, 0, 1)),
                                                (2, 40, 16, 3, 2, (1, 1))])
def test_fill_boundary_rank_threads_through_c_abi_equal_reference(ref, nranks, dim, n, b, nc, ng, per):
    """The reference's runtime_spawn rank threads, each calling the binding
    collectively: ghost cells AND Bus message statistics equal the
    reference's own fill_boundary on twin MultiFabs."""
    _, _, comm, config, ix, mesh = ref
    from integration.reference_binding import PinnedArena, fill_boundary_native
    config.set_spacedim(dim) if hasattr(config, "set_spacedim") else None
    dom = ix.Box((0,) * dim, (n - 1,) * dim)
    geom = ix.Geometry(dom, (0.0,) * dim, (1.0,) * dim, per)
    ba = mesh.decompose(dom, b)
    dm = mesh.DistributionMapping.round_robin(len(ba), nranks)

    def run(native):
        def program(ctx):
            mf = mesh.MultiFab(ba, dm, nc, ng, geom, arena=PinnedArena() if native else None)
            _fill_by_fab(mf, 5)
            for _ in range(2):
                if native:
                    fill_boundary_native(mf, geom)
                else:
                    comm.fill_boundary(mf, geom, backend=ref[0]._serial)
            return {i: mf.fabs[i].data.copy() for i in mf.local_indices}
        return _spawn(comm, nranks, program)

    got, got_stats = run(True)
    exp, exp_stats = run(False)
    assert got_stats == exp_stats and any(v[0] for k, v in exp_stats.items() if k[0] != k[1])
    for r in range(nranks):
        assert got[r].keys() == exp[r].keys()
        for i in got[r]:
            assert np.array_equal(got[r][i].view(np.uint64), exp[r][i].view(np.uint64)), f"rank {r} fab {i}"


@pytest.mark.parametrize("nranks", [2, 3])
@pytest.mark.parametrize("n,sb,db,nc,gs,gd,periodic", [(32, 8, 16, 2, 0, 0, None), (24, 12, 8, 1, 1, 2, (1, 1, 1))])
def test_parallel_copy_rank_threads_through_c_abi_equal_reference(ref, nranks, n, sb, db, nc, gs, gd, periodic):
    _, _, comm, config, ix, mesh = ref
    from integration.reference_binding import PinnedArena, parallel_copy_native
    config.set_spacedim(3)
    dom = ix.Box((0, 0, 0), (n - 1,) * 3)
    geom = ix.Geometry(dom, (0.0,) * 3, (1.0,) * 3, periodic) if periodic else None
    sba, dba = mesh.decompose(dom, sb), mesh.decompose(dom, db)
    sdm = mesh.DistributionMapping.round_robin(len(sba), nranks)
    ddm = mesh.DistributionMapping.round_robin(len(dba), nranks)

    def run(native):
        def program(ctx):
            arena = PinnedArena() if native else None
            src = mesh.MultiFab(sba, sdm, nc, gs, arena=arena)
            dst = mesh.MultiFab(dba, ddm, nc + 1, gd, arena=arena)
            _fill_by_fab(src, 11)
            _fill_by_fab(dst, 12)
            for _ in range(2):
                if native:
                    parallel_copy_native(dst, src, 0, 1, nc, gs, gd, geom)
                else:
                    comm.parallel_copy(dst, src, 0, 1, nc, gs, gd, geom, backend=ref[0]._serial)
            return {i: dst.fabs[i].data.copy() for i in dst.local_indices}
        return _spawn(comm, nranks, program)

    got, got_stats = run(True)
    exp, exp_stats = run(False)
    assert got_stats == exp_stats
    for r in range(nranks):
        for i in got[r]:
            assert np.array_equal(got[r][i].view(np.uint64), exp[r][i].view(np.uint64)), f"rank {r} fab {i}"


def _levels(ix, mesh, n, b, patch_lo, patch_hi, ratio):
    dom = ix.Box((0, 0, 0), (n - 1,) * 3)
    cgeom = ix.Geometry(dom, (0.0,) * 3, (1.0,) * 3, (True, True, True))
    fgeom = cgeom.refined(ratio)
    cba = mesh.decompose(dom, b)
    fba = mesh.decompose(ix.Box((patch_lo * ratio,) * 3, ((patch_hi + 1) * ratio - 1,) * 3), b)
    return cgeom, fgeom, cba, fba


@pytest.mark.parametrize("nranks", [1, 2, 3])
@pytest.mark.parametrize("scheme", ["linear", "piecewise_constant"])
@pytest.mark.parametrize("patch", [(8, 23), (0, 11)])  # centred patch / patch on the periodic boundary
def test_fill_patch_through_c_abi_equals_reference(ref, nranks, scheme, patch):
    _, amr, comm, config, ix, mesh = ref
    from integration.reference_binding import PinnedArena, fill_patch_native
    config.set_spacedim(3)
    cgeom, fgeom, cba, fba = _levels(ix, mesh, 32, 8, patch[0], patch[1], 2)

    def run(native):
        def program(ctx):
            arena = PinnedArena() if native else None
            crse = mesh.MultiFab(cba, mesh.DistributionMapping.round_robin(len(cba), nranks), 2, 0, cgeom,
                                 arena=arena)
            fine = mesh.MultiFab(fba, mesh.DistributionMapping.round_robin(len(fba), nranks), 2, 2, fgeom,
                                 arena=arena)
            _fill_by_fab(crse, 21)
            _fill_by_fab(fine, 22)
            for _ in range(2):
                if native:
                    fill_patch_native(fine, crse, fgeom, cgeom, 2, scheme)
                else:
                    amr.fill_patch(fine, crse, fgeom, cgeom, 2, scheme, backend=ref[0]._serial)
            return {i: fine.fabs[i].data.copy() for i in fine.local_indices}, fine.plan_builds
        return _spawn(comm, nranks, program)

    got, got_stats = run(True)
    exp, exp_stats = run(False)
    assert got_stats == exp_stats
    for r in range(nranks):
        (g, gb), (e, eb) = got[r], exp[r]
        assert gb == eb  # plan builds counted like the reference (FillBoundary + fill_patch plans)
        for i in g:
            assert np.array_equal(g[i].view(np.uint64), e[i].view(np.uint64)), f"rank {r} fab {i}"


@pytest.mark.parametrize("nranks", [1, 2])
def test_average_down_through_c_abi_equals_reference(ref, nranks):
    _, amr, comm, config, ix, mesh = ref
    from integration.reference_binding import PinnedArena, average_down_native
    config.set_spacedim(3)
    cgeom, fgeom, cba, fba = _levels(ix, mesh, 32, 8, 4, 19, 2)

    def run(native):
        def program(ctx):
            arena = PinnedArena() if native else None
            crse = mesh.MultiFab(cba, mesh.DistributionMapping.round_robin(len(cba), nranks), 3, 1, cgeom,
                                 arena=arena)
            fine = mesh.MultiFab(fba, mesh.DistributionMapping.round_robin(len(fba), nranks), 3, 2, fgeom,
                                 arena=arena)
            _fill_by_fab(crse, 31)
            _fill_by_fab(fine, 32)
            for _ in range(2):
                if native:
                    average_down_native(fine, crse, 2)
                else:
                    amr.average_down(fine, crse, 2, backend=ref[0]._serial)
            return {i: crse.fabs[i].data.copy() for i in crse.local_indices}
        return _spawn(comm, nranks, program)

    got, got_stats = run(True)
    exp, exp_stats = run(False)
    assert got_stats == exp_stats
    for r in range(nranks):
        for i in got[r]:
            assert np.array_equal(got[r][i].view(np.uint64), exp[r][i].view(np.uint64)), f"rank {r} fab {i}"
