"""GPU parity: the CUDA path (C ABI -> fused sm_100a kernel) against the
reference-generated golden fixtures, the oracle, and size-independent
properties at BASELINE.json's full sizes.  Bit-exact (raw words) throughout.
"""

import numpy as np
import pytest

import golden_util as gu
from gpu_util import bits_of, device_bits, expected_wrapped, upload
from oracle import ghost_oracle as go
from oracle import inputs

pytestmark = pytest.mark.gpu


def _amr():
    import paper_2403_12179_b200 as amr
    return amr


def _boxes(amr, rows, dim, nodal):
    ixt = amr.IndexType.node() if nodal else amr.IndexType.cell()
    return [amr.Box(r[:dim], r[3:3 + dim], ixt) for r in rows]


def _domain(amr, c, key="domain"):
    d = c["dim"]
    return amr.Box(c[key][0][:d], c[key][1][:d])


# task-building variants of the fused kernel: default heuristics, x-line
# chains + TMA bulk face rows (the large-fab path), fab-local swaps
# ... and the phased exchange of host-memory fabs (faces extended over the
# lower-axis ghosts, phase waits in the kernel) on device fabs, with the
# default kernel and with the host path's tile-ring instantiation
VARIANTS = {"default": {}, "chains_bulk": {"GHX_FAB_LOCAL": "0", "GHX_BULK": "1"},
            "fab_local": {"GHX_FAB_LOCAL": "1", "GHX_BULK": "0"},
            "phased": {"GHX_PHASED": "1"}, "phased_ring": {"GHX_PHASED": "1", "GHX_RING": "1"}}


@pytest.mark.parametrize("variant", sorted(VARIANTS))
@pytest.mark.parametrize("name", gu.names("fill_boundary", store="bits"))
def test_fill_boundary_matches_reference_golden(name, variant, monkeypatch):
    for k, v in VARIANTS[variant].items():
        monkeypatch.setenv(k, v)
    amr = _amr()
    c = gu.case(name)
    d = gu.data()
    dim = c["dim"]
    amr.config.set_spacedim(dim)
    amr.config.set_real_dtype(np.dtype(c["dtype"]))
    ba = amr.BoxArray(_boxes(amr, c["boxes"], dim, c["nodal"]))
    dm = amr.DistributionMapping(c["rank_of"], c["nranks"])
    geom = amr.Geometry(_domain(amr, c), [0.0] * dim, [1.0] * dim, c["periodic"][:dim])
    hdom = list(c["hash_domain"][0]) + list(c["hash_domain"][1])  # padded 3-D row
    ng = c["ngrow"][:dim]

    def program(ctx):
        mf = amr.MultiFab(ba, dm, c["ncomp"], amr.IntVect(*ng), geom)
        mf.fill_hash(inputs.SEED, hdom)
        # the device generator equals the oracle's input generator bit-exactly
        for gi in mf.local_indices:
            f = mf.fabs[gi]
            ref = inputs.make_fab(f.lo3, gu.grown(c["boxes"][gi], c["ngrow"])[3:], c["ncomp"],
                                  np.dtype(c["dtype"]), c["boxes"][gi][:3], c["boxes"][gi][3:],
                                  c["hash_domain"][0], c["hash_domain"][1])
            assert np.array_equal(bits_of(f), inputs.bits(ref).ravel(order="F"))
        ctx.barrier()
        s0 = ctx.bus.stats_snapshot()
        ctx.barrier()
        for _ in range(c["calls"]):
            amr.fill_boundary(mf, geom)
        ctx.barrier()
        s1 = ctx.bus.stats_snapshot()
        ctx.barrier()
        out = {gi: bits_of(mf.fabs[gi]) for gi in mf.local_indices}
        stats = {k: (s1[k][0] - s0[k][0], s1[k][1] - s0[k][1]) for k in s1 if s1[k] != s0[k]}
        return out, stats, mf.plan_builds

    res = amr.runtime_spawn(c["nranks"], program)
    for out, stats, builds in res:
        assert builds == 1
        for gi, got in out.items():
            np.testing.assert_array_equal(got, d[f"{name}/fab{gi}"].ravel(order="F"), err_msg=f"fab {gi}")
    if c["nranks"] > 1:
        assert res[0][1] == gu.stats_dict(d[f"{name}/stats"])


@pytest.mark.parametrize("name", gu.names("parallel_copy"))
def test_parallel_copy_matches_reference_golden(name):
    amr = _amr()
    c = gu.case(name)
    d = gu.data()
    dim = c["dim"]
    dt = np.dtype(c["dtype"])
    amr.config.set_spacedim(dim)
    amr.config.set_real_dtype(dt)
    sba = amr.BoxArray(_boxes(amr, c["src_boxes"], dim, c["nodal"]))
    dba = amr.BoxArray(_boxes(amr, c["dst_boxes"], dim, c["nodal"]))
    sdm = amr.DistributionMapping(c["src_rank"], c["nranks"])
    ddm = amr.DistributionMapping(c["dst_rank"], c["nranks"])
    geom = None if c["periodic"] is None else amr.Geometry(_domain(amr, c), [0.0] * dim, [1.0] * dim,
                                                           c["periodic"][:dim])
    hd = c["hash_domain"]

    def program(ctx):
        src = amr.MultiFab(sba, sdm, c["src_ncomp"], amr.IntVect(*c["src_ngrow"][:dim]))
        dst = amr.MultiFab(dba, ddm, c["dst_ncomp"], amr.IntVect(*c["dst_ngrow"][:dim]))
        for gi in src.local_indices:
            g = gu.grown(c["src_boxes"][gi], c["src_ngrow"])
            b = c["src_boxes"][gi]
            upload(src.fabs[gi], inputs.make_fab(g[:3], g[3:], c["src_ncomp"], dt, b[:3], b[3:], hd[0], hd[1],
                                                 ghost_tag=gi + 1))
        for gi in dst.local_indices:
            g = gu.grown(c["dst_boxes"][gi], c["dst_ngrow"])
            b = c["dst_boxes"][gi]
            upload(dst.fabs[gi], inputs.make_fab(g[:3], g[3:], c["dst_ncomp"], dt, b[:3], b[3:], hd[0], hd[1],
                                                 seed=inputs.SEED + 1))
        ctx.barrier()
        s0 = ctx.bus.stats_snapshot()
        ctx.barrier()
        amr.parallel_copy(dst, src, scomp=c["scomp"], dcomp=c["dcomp"], ncomp=c["ncomp"],
                          ngrow_src=amr.IntVect(*c["ngrow_src"][:dim]),
                          ngrow_dst=amr.IntVect(*c["ngrow_dst"][:dim]), geom=geom)
        ctx.barrier()
        s1 = ctx.bus.stats_snapshot()
        ctx.barrier()
        out = {gi: bits_of(dst.fabs[gi]) for gi in dst.local_indices}
        stats = {k: (s1[k][0] - s0[k][0], s1[k][1] - s0[k][1]) for k in s1 if s1[k] != s0[k]}
        return out, stats

    res = amr.runtime_spawn(c["nranks"], program)
    for out, _ in res:
        for gi, got in out.items():
            np.testing.assert_array_equal(got, d[f"{name}/fab{gi}"].ravel(order="F"), err_msg=f"fab {gi}")
    if c["nranks"] > 1:
        assert res[0][1] == gu.stats_dict(d[f"{name}/stats"])


def _scale_layout(amr, n, b, G):
    amr.config.set_spacedim(3)
    dom = amr.Box((0, 0, 0), (n - 1,) * 3)
    geom = amr.Geometry(dom, (0.0,) * 3, (1.0,) * 3, (True,) * 3)
    ba = amr.decompose(dom, b)
    dm = amr.DistributionMapping.round_robin(len(ba), G)
    return dom, geom, ba, dm


@pytest.mark.parametrize("G", [1, 2])
def test_c1_matches_reference_digests(G):
    amr = _amr()
    c = gu.case(f"C1_data_x{G}")
    dom, geom, ba, dm = _scale_layout(amr, 64, 32, G)

    def program(ctx):
        mf = amr.MultiFab(ba, dm, 1, 1, geom)
        mf.fill_hash(inputs.SEED, dom)
        amr.fill_boundary(mf, geom)
        return {gi: gu.fab_digest(bits_of(mf.fabs[gi])) for gi in mf.local_indices}

    got = {}
    for r in amr.runtime_spawn(G, program):
        got.update(r)
    assert {str(k): v for k, v in got.items()} == c["fab_sha256"]


@pytest.mark.parametrize("variant", ["default", "chains_bulk", "fab_local"])
@pytest.mark.parametrize("cfg", [("C2", 256, 64, 4, 2), ("C3", 512, 128, 8, 2), ("C4", 256, 16, 4, 2)])
def test_full_size_fill_boundary_wrapped_property(cfg, variant, monkeypatch):
    """At BASELINE.json's full sizes: after FillBoundary on a fully periodic
    domain every storage cell of every fab equals the hash of its periodically
    wrapped cell (the reference acceptance oracle's global-array wrap,
    tests/test_acceptance.py:112-134), valid cells unchanged."""
    import torch
    for k, v in VARIANTS[variant].items():
        monkeypatch.setenv(k, v)
    amr = _amr()
    name, n, b, nc, ng = cfg
    dom, geom, ba, dm = _scale_layout(amr, n, b, 1)
    mf = amr.MultiFab(ba, dm, nc, ng, geom)
    mf.fill_hash(inputs.SEED, dom)
    amr.fill_boundary(mf, geom)
    amr.fill_boundary(mf, geom)  # idempotent second call, cached plan
    assert mf.plan_builds == 1
    bad = 0
    for gi in mf.local_indices:
        f = mf.fabs[gi]
        exp = expected_wrapped(f, nc, dom.as_row(), (1, 1, 1), inputs.SEED, 8)
        bad += int((device_bits(f) != exp).sum().item())
    torch.cuda.synchronize()
    assert bad == 0


def test_c2_matches_cpu_oracle():
    """Full C2 (256^3, 64^3 boxes, nc 4, ng 2): CUDA result == oracle result on
    the same inputs, every fab bit-exact."""
    amr = _amr()
    dom, geom, ba, dm = _scale_layout(amr, 256, 64, 1)
    mf = amr.MultiFab(ba, dm, 4, 2, geom)
    mf.fill_hash(inputs.SEED, dom)
    before = {gi: bits_of(mf.fabs[gi]) for gi in mf.local_indices}
    amr.fill_boundary(mf, geom)
    rows = ba.rows()
    plan = go.plan_fill_boundary(rows, [2] * 3, [True] * 3, [256] * 3, [0] * len(ba), 1)
    fabs, lo = {}, {}
    for gi in mf.local_indices:
        f = mf.fabs[gi]
        shape = tuple(f.data.shape)
        fabs[gi] = before[gi].view(np.float64).reshape(shape, order="F")
        lo[gi] = np.asarray(f.lo3)
    go.execute(plan, fabs, lo, fabs, lo, 0, 0, 4, workers=8)
    for gi in mf.local_indices:
        np.testing.assert_array_equal(bits_of(mf.fabs[gi]), fabs[gi].view(np.uint64).ravel(order="F"))


@pytest.mark.parametrize("G", [1, 8])
def test_c5_regrid_full_size(G):
    """ParallelCopy 1024^3, 64^3 -> 128^3 boxes, nc 4 (BASELINE config 5):
    every dst fab equals the hash of its own cells; with 8 thread ranks the
    message accounting matches the reference plan (14 pairs x 2.147 GB)."""
    import torch
    amr = _amr()
    amr.config.set_spacedim(3)
    n = 1024
    dom = amr.Box((0, 0, 0), (n - 1,) * 3)
    sba = amr.decompose(dom, 64)
    dba = amr.decompose(dom, 128)
    sdm = amr.DistributionMapping.round_robin(len(sba), G)
    ddm = amr.DistributionMapping.round_robin(len(dba), G)
    c = gu.case("C5")

    def program(ctx):
        src = amr.MultiFab(sba, sdm, 4, 0)
        dst = amr.MultiFab(dba, ddm, 4, 0)
        src.fill_hash(inputs.SEED, dom)
        for gi in dst.local_indices:
            dst.fabs[gi].data.fill_(-1.0)
        ctx.barrier()
        s0 = ctx.bus.stats_snapshot()
        ctx.barrier()
        amr.parallel_copy(dst, src)
        ctx.barrier()
        s1 = ctx.bus.stats_snapshot()
        bad = 0
        for gi in dst.local_indices:
            f = dst.fabs[gi]
            exp = expected_wrapped(f, 4, dom.as_row(), (0, 0, 0), inputs.SEED, 8)
            bad += int((device_bits(f) != exp).sum().item())
        torch.cuda.synchronize()
        stats = {f"{s}->{d}": s1[(s, d)][1] - s0[(s, d)][1] for (s, d) in s1
                 if s1[(s, d)][0] - s0[(s, d)][0] and s != d}
        del src, dst
        return bad, stats

    res = amr.runtime_spawn(G, program)
    assert all(r[0] == 0 for r in res)
    if G == 8:
        assert res[0][1] == c["pair_bytes"]


def test_pinned_host_multifab_fill_boundary():
    """Host-resident (pinned, mapped) fabs: the same kernel runs over PCIe."""
    amr = _amr()
    dom, geom, ba, dm = _scale_layout(amr, 64, 32, 1)
    mf = amr.MultiFab(ba, dm, 1, 1, geom, memory="pinned")
    ref = amr.MultiFab(ba, dm, 1, 1, geom)
    mf.fill_hash(inputs.SEED, dom)
    ref.fill_hash(inputs.SEED, dom)
    import torch
    torch.cuda.synchronize()
    amr.fill_boundary(mf, geom)
    amr.fill_boundary(ref, geom)
    c = gu.case("C1_data_x1")
    for gi in mf.local_indices:
        assert not mf.fabs[gi].data.is_cuda
        assert gu.fab_digest(bits_of(mf.fabs[gi])) == c["fab_sha256"][str(gi)]


@pytest.mark.parametrize("n,b,nc", [(128, 64, 2), (256, 128, 4)])
def test_pinned_host_large_and_small_fabs_wrapped_property(n, b, nc):
    """Host-resident fabs take the seam-chunk (ring) task path; with fabs
    over 64 MiB (the second case) the device path would also use x-line
    chains and TMA bulk rows -- the host executor must not mix them."""
    import torch
    amr = _amr()
    amr.config.set_spacedim(3)
    dom = amr.Box((0, 0, 0), (2 * b - 1, b - 1, b - 1)) if n == 256 else amr.Box((0, 0, 0), (n - 1,) * 3)
    geom = amr.Geometry(dom, (0.0,) * 3, (1.0,) * 3, (True,) * 3)
    ba = amr.decompose(dom, b)
    dm = amr.DistributionMapping([0] * len(ba))
    mf = amr.MultiFab(ba, dm, nc, 2, geom, memory="pinned")
    ref = amr.MultiFab(ba, dm, nc, 2, geom)  # device twin: wrapped-hash property checked on the device
    mf.fill_hash(inputs.SEED, dom)
    ref.fill_hash(inputs.SEED, dom)
    torch.cuda.synchronize()
    amr.fill_boundary(mf, geom)
    amr.fill_boundary(ref, geom)
    ex = amr.comm.prepare_fill_boundary(mf, geom).ex
    assert ex.detail["ring_tasks"] > 0 and ex.detail["ring_mode"] == 1
    bad = 0
    for gi in mf.local_indices:
        exp = expected_wrapped(ref.fabs[gi], nc, dom.as_row(), (1, 1, 1), inputs.SEED, 8)
        assert bool((device_bits(ref.fabs[gi]) == exp).all())
        got = torch.from_numpy(bits_of(mf.fabs[gi]).view(np.int64))
        bad += int((got != exp.cpu()).sum().item())
    assert bad == 0


def test_known_values_1d_and_constant_field():
    """Reference tests/test_comm.py:198-222 through the CUDA path."""
    amr = _amr()
    amr.config.set_spacedim(1)
    geom = amr.Geometry(amr.Box((0,), (7,)), (0.0,), (1.0,), (True,))
    ba = amr.BoxArray([amr.Box((0,), (3,)), amr.Box((4,), (7,))])
    mf = amr.multifab_define(ba, amr.DistributionMapping([0, 0]), 1, 1, geom)
    for gi in mf.local_indices:
        v = mf.view(gi)
        for i in range(ba[gi].lo[0], ba[gi].hi[0] + 1):
            v[i] = float(i)
    amr.fill_boundary(mf, geom)
    v0, v1 = mf.view(0), mf.view(1)
    assert (v0[-1], v0[4]) == (7.0, 4.0)
    assert (v1[3], v1[8]) == (3.0, 0.0)
    amr.config.set_spacedim(2)
    geom = amr.Geometry(amr.Box((0, 0), (7, 7)), (0, 0), (1, 1), (True, True))
    ba = amr.decompose(amr.Box((0, 0), (7, 7)), 4)
    mf = amr.multifab_define(ba, amr.DistributionMapping([0] * len(ba)), 1, 2, geom)
    mf.setval(-9999.0)
    mf.setval(3.25, grown=False)
    amr.fill_boundary(mf, geom)
    for gi in mf.local_indices:
        assert bool((mf.fabs[gi].data == 3.25).all())


def test_parallel_copy_one_to_four_ranks_message_count():
    """Reference tests/test_comm.py:278-302: exactly 3 outgoing messages."""
    amr = _amr()
    amr.config.set_spacedim(1)
    dom = amr.Box((0,), (15,))
    src_ba = amr.BoxArray([dom])
    dst_ba = amr.BoxArray([amr.Box((i * 4,), (i * 4 + 3,)) for i in range(4)])
    src_dm = amr.DistributionMapping([0], nranks=4)
    dst_dm = amr.DistributionMapping([0, 1, 2, 3])

    def program(ctx):
        src = amr.multifab_define(src_ba, src_dm, 1, 0)
        dst = amr.multifab_define(dst_ba, dst_dm, 1, 0)
        if ctx.rank == 0:
            v = src.view(0)
            v[np.arange(16), np.zeros(16, np.int64), np.zeros(16, np.int64)] = np.arange(16.0)
        dst.setval(-9999.0)
        amr.parallel_copy(dst, src)
        stats = ctx.bus.stats_snapshot()
        out = sum(1 for (s, d), (n, _) in stats.items() if s == 0 and d != 0 and n > 0)
        for gi in dst.local_indices:
            lo = dst_ba[gi].lo[0]
            assert np.array_equal(dst.fabs[gi].data[..., 0].reshape(-1).cpu().numpy(), np.arange(lo, lo + 4.0))
        return out

    assert amr.runtime_spawn(4, program)[0] == 3


@pytest.mark.parametrize("n,b,nc,ng,per,dt,memory", [
    (256, 64, 4, 2, (1, 0, 1), "f8", "device"), (256, 64, 4, 2, (0, 1, 0), "f8", "pinned"),
    (256, 16, 4, 2, (1, 1, 0), "f4", "device"), (256, 64, 3, 1, (1, 1, 1), "f4", "pinned"),
    (512, 128, 8, 2, (0, 0, 0), "f8", "device"), (128, 32, 2, 2, (1, 0, 0), "f8", "pinned")],
    ids=["C2-xz-periodic", "C2-y-periodic-pinned", "C4-f32", "f32-ng1-pinned", "C3-no-periodic",
         "x-periodic-pinned-phased"])
def test_full_size_mixed_periodicity_and_float32(n, b, nc, ng, per, dt, memory):
    """Full-size layouts with physical boundaries and float32 storage, on
    device fabs and on pinned host fabs (the phased host exchange): after
    FillBoundary every storage cell equals the hash of its periodically
    wrapped cell where that cell lies in the domain, and keeps its poison
    bits where it does not (uncoverable ghosts untouched)."""
    import torch
    amr = _amr()
    amr.config.set_spacedim(3)
    amr.config.set_real_dtype(np.dtype(dt))
    try:
        dom = amr.Box((0, 0, 0), (n - 1,) * 3)
        geom = amr.Geometry(dom, (0.0,) * 3, (1.0,) * 3, tuple(bool(p) for p in per))
        ba = amr.decompose(dom, b)
        dm = amr.DistributionMapping([0] * len(ba))
        mf = amr.MultiFab(ba, dm, nc, ng, geom, memory=memory)
        mf.fill_hash(inputs.SEED, dom)
        torch.cuda.synchronize()
        amr.fill_boundary(mf, geom)
        amr.fill_boundary(mf, geom)
        if memory == "pinned":
            assert amr.comm.prepare_fill_boundary(mf, geom).ex.detail["phased"] == 1
        item = np.dtype(dt).itemsize
        bad = 0
        for gi in mf.local_indices:
            f = mf.fabs[gi]
            exp = expected_wrapped(f, nc, dom.as_row(), per, inputs.SEED, item)
            if memory == "pinned":
                got = torch.from_numpy(bits_of(f).view(np.int64 if item == 8 else np.int32)).to(exp.device)
            else:
                got = device_bits(f)
            bad += int((got != exp).sum().item())
        assert bad == 0
    finally:
        amr.config.set_real_dtype(np.dtype("f8"))
