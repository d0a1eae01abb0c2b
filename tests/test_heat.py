"""Heat-equation step loop (reference heat.py:172-189, 264-273) against
fixtures produced by running the reference's loop body
(tests/golden/make_golden_amr.py, kind "heat"): the oracle replay on CPU and
paper_2403_12179_b200.heat.heat_step on the GPU (with and without the
interior/exchange overlap), raw bits."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import amr_oracle as ao
from oracle import ghost_oracle as go
from oracle import inputs
from test_amr_oracle import case, data, grown, hashed, meta, names, poisoned


def _g3(v, dim):
    return [v if d < dim else 0 for d in range(3)]


def _r3(r, dim):
    return [r if d < dim else 1 for d in range(3)]


def _level_setup(c):
    dim, dt = c["dim"], np.dtype(c["dtype"])
    cdom = np.asarray([0, 0, 0] + [e - 1 for e in c["cext"]], np.int64)
    levels = [dict(boxes=[np.asarray(b, np.int64) for b in c["crse_boxes"]], ranks=c["crse_rank"], dom=cdom)]
    if c["fine_boxes"]:
        rr = _r3(c["ratio"], dim)
        fdom = np.asarray([0, 0, 0] + [e * q - 1 for e, q in zip(c["cext"], rr)], np.int64)
        levels.append(dict(boxes=[np.asarray(b, np.int64) for b in c["fine_boxes"]], ranks=c["fine_rank"], dom=fdom))
    for lv, L in enumerate(levels):
        g = _g3(1, dim)
        L["u"] = {gi: hashed(grown(b, g), b, L["dom"], 1, dt, inputs.SEED + lv) for gi, b in enumerate(L["boxes"])}
        L["w"] = {gi: np.zeros(tuple(int(x) for x in (grown(b, g)[3:] - grown(b, g)[:3] + 1)) + (1,), dt, order="F")
                  for gi, b in enumerate(L["boxes"])}
        L["lo"] = {gi: grown(b, g)[:3] for gi, b in enumerate(L["boxes"])}
        # cell sizes: Geometry(domain, 0, 1) -> 1 / extent, as Python floats
        L["dx"] = [1.0 / float(L["dom"][3 + d] + 1) for d in range(dim)]
    return levels


def _fill_patch(c, fine, crse_u):
    dim, dt, r = c["dim"], np.dtype(c["dtype"]), c["ratio"]
    rr = _r3(r, dim)
    ng = _g3(1, dim)
    per = [True] * dim + [False] * (3 - dim)
    fperiod = [int(fine["dom"][3 + d] + 1) for d in range(3)]
    plan = go.plan_fill_boundary(fine["boxes"], ng, per, fperiod, fine["ranks"], c["nranks"])
    go.execute(plan, fine["u"], fine["lo"], fine["u"], fine["lo"], 0, 0, 1)
    targets = ao.fill_targets(fine["boxes"], ng, fine["dom"], per, dim)
    if not targets:
        return
    order = sorted(targets)
    cboxes = {}
    for gi in order:
        b = grown(fine["boxes"][gi], ng)
        b[:3] //= np.asarray(rr)
        b[3:] //= np.asarray(rr)
        cboxes[gi] = grown(b, _g3(1, dim))
    cperiod = [int(crse_u["dom"][3 + d] + 1) for d in range(3)]
    gplan = go.plan_parallel_copy([cboxes[g] for g in order], crse_u["boxes"], [0] * 3, [0] * 3, per, cperiod,
                                  crse_u["ranks"], [fine["ranks"][g] for g in order], c["nranks"])
    gath = {p: poisoned(cboxes[g], 1, dt) for p, g in enumerate(order)}
    go.execute(gplan, crse_u["u"], crse_u["lo"], gath, {p: cboxes[g][:3] for p, g in enumerate(order)}, 0, 0, 1)
    for p, gi in enumerate(order):
        for region in targets[gi]:
            ao.interp(gath[p], cboxes[gi], fine["u"][gi], grown(fine["boxes"][gi], ng), region, rr, True, dim)


def oracle_heat(c):
    dim = c["dim"]
    levels = _level_setup(c)
    per = [True] * dim + [False] * (3 - dim)
    for _ in range(c["steps"]):
        L0 = levels[0]
        period = [int(L0["dom"][3 + d] + 1) for d in range(3)]
        plan = go.plan_fill_boundary(L0["boxes"], _g3(1, dim), per, period, L0["ranks"], c["nranks"])
        go.execute(plan, L0["u"], L0["lo"], L0["u"], L0["lo"], 0, 0, 1)
        if len(levels) > 1:
            _fill_patch(c, levels[1], L0)
        for L in levels:
            coef = [c["dt"] * c["diffusivity"] / L["dx"][d] ** 2 for d in range(dim)] + [0.0] * (3 - dim)
            for gi, b in enumerate(L["boxes"]):
                new = ao.advance(L["u"][gi], grown(b, _g3(1, dim)), b, coef, dim)
                sl = tuple(slice(int(b[d] - L["lo"][gi][d]), int(b[3 + d] - L["lo"][gi][d]) + 1) for d in range(3))
                L["w"][gi][sl + (0,)] = new
        if len(levels) > 1:
            F, Cc = levels[1], levels[0]
            rr = _r3(c["ratio"], dim)
            tmp, tboxes = {}, []
            for gi, b in enumerate(F["boxes"]):
                tb = b.copy()
                tb[:3] //= np.asarray(rr)
                tb[3:] //= np.asarray(rr)
                tboxes.append(tb)
                tmp[gi] = ao.restrict(F["w"][gi], grown(b, _g3(1, dim)), b, rr, dim)
            plan = go.plan_parallel_copy(Cc["boxes"], tboxes, [0] * 3, [0] * 3, None, None, F["ranks"], Cc["ranks"],
                                         c["nranks"])
            go.execute(plan, tmp, {gi: b[:3] for gi, b in enumerate(tboxes)}, Cc["w"], Cc["lo"], 0, 0, 1)
        for L in levels:
            L["u"], L["w"] = L["w"], L["u"]
    return levels


@pytest.mark.parametrize("name", names("heat"))
def test_heat_oracle_matches_reference(name):
    c = case(name)
    levels = oracle_heat(c)
    for lv, L in enumerate(levels):
        for which in ("u", "w"):
            for gi, a in L[which].items():
                assert np.array_equal(inputs.bits(a), data()[f"{name}/l{lv}{which}{gi}"]), (lv, which, gi)


@pytest.mark.gpu
@pytest.mark.parametrize("overlap", [True, False])
@pytest.mark.parametrize("name", names("heat"))
def test_heat_step_bit_exact(name, overlap):
    import paper_2403_12179_b200 as amr
    from paper_2403_12179_b200 import heat as H
    from gpu_util import bits_of, upload
    c = case(name)
    dim, dt = c["dim"], np.dtype(c["dtype"])
    amr.config.set_spacedim(dim)
    amr.config.set_real_dtype(dt)
    box = lambda b6: amr.Box(tuple(b6[:dim]), tuple(b6[3:3 + dim]))  # noqa: E731
    cdom = amr.Box((0,) * dim, tuple(e - 1 for e in c["cext"][:dim]))
    cgeom = amr.Geometry(cdom, (0.0,) * dim, (1.0,) * dim, (True,) * dim)
    geoms = [cgeom, cgeom.refined(c["ratio"])]
    specs = [(amr.BoxArray([box(b) for b in c["crse_boxes"]]), amr.DistributionMapping(c["crse_rank"], c["nranks"]))]
    if c["fine_boxes"]:
        specs.append((amr.BoxArray([box(b) for b in c["fine_boxes"]]),
                      amr.DistributionMapping(c["fine_rank"], c["nranks"])))

    def program(ctx):
        levels = []
        for lv, (ba, dm) in enumerate(specs):
            u = amr.MultiFab(ba, dm, 1, 1, geoms[lv])
            w = amr.MultiFab(ba, dm, 1, 1, geoms[lv])
            dom6 = np.asarray(geoms[lv].domain.as_row(), np.int64)
            for gi in u.local_indices:
                vb = np.asarray(ba[gi].as_row(), np.int64)
                upload(u.fabs[gi], hashed(grown(vb, _g3(1, dim)), vb, dom6, 1, dt, inputs.SEED + lv))
            w.setval(0.0)
            levels.append((u, w))
        ctx.barrier()
        for _ in range(c["steps"]):
            levels = H.heat_step(levels, geoms, c["dt"], c["diffusivity"], c["ratio"], overlap=overlap)
        out = {}
        for lv, (u, w) in enumerate(levels):
            for gi in u.local_indices:
                out[(lv, "u", gi)] = bits_of(u.fabs[gi])
                out[(lv, "w", gi)] = bits_of(w.fabs[gi])
        return out

    got = {}
    for res in amr.runtime_spawn(c["nranks"], program):
        got.update(res)
    for (lv, which, gi), a in got.items():
        assert np.array_equal(a, data()[f"{name}/l{lv}{which}{gi}"].ravel(order="F")), (lv, which, gi)


@pytest.mark.gpu
def test_heat_loop_cuda_graphs_match_eager():
    """HeatLoop (steps 3+ replayed from CUDA graphs) == heat_step, bit for bit,
    on a two-level problem."""
    import paper_2403_12179_b200 as amr
    from paper_2403_12179_b200 import heat as H
    amr.config.set_spacedim(3)
    cdom = amr.Box((0, 0, 0), (15, 15, 15))
    cgeom = amr.Geometry(cdom, (0.0,) * 3, (1.0,) * 3, (True,) * 3)
    geoms = [cgeom, cgeom.refined(2)]
    cba = amr.decompose(cdom, 8)
    fba = amr.decompose(amr.Box((8, 8, 8), (23, 23, 23)), 8)

    def make():
        levels = []
        for lv, ba in enumerate((cba, fba)):
            dm = amr.DistributionMapping([0] * len(ba))
            u = amr.MultiFab(ba, dm, 1, 1, geoms[lv])
            w = amr.MultiFab(ba, dm, 1, 1, geoms[lv])
            u.fill_hash(11 + lv, geoms[lv].domain)
            w.setval(0.0)
            levels.append((u, w))
        return levels

    from gpu_util import bits_of
    eager = make()
    for _ in range(6):
        eager = H.heat_step(eager, geoms, 1e-5, 1.0, 2)
    loop = H.HeatLoop(make(), geoms, 1e-5, 1.0, 2)
    for _ in range(6):
        loop.step()
    assert len(loop._graph) == 2
    for (ue, we), (ug, wg) in zip(eager, loop.levels):
        for gi in ue.local_indices:
            assert np.array_equal(bits_of(ue.fabs[gi]), bits_of(ug.fabs[gi]))
            assert np.array_equal(bits_of(we.fabs[gi]), bits_of(wg.fabs[gi]))


@pytest.mark.gpu
def test_heat_loop_rank_invariant():
    """Reference tests/test_tools.py:215-231: the result does not depend on
    the number of ranks (1, 2, 3 thread ranks on one GPU, two levels)."""
    import paper_2403_12179_b200 as amr
    from paper_2403_12179_b200 import heat as H
    from gpu_util import bits_of
    amr.config.set_spacedim(2)
    cdom = amr.Box((0, 0), (31, 31))
    cgeom = amr.Geometry(cdom, (0.0, 0.0), (1.0, 1.0), (True, True))
    geoms = [cgeom, cgeom.refined(2)]
    cba = amr.decompose(cdom, 8)
    fba = amr.BoxArray([amr.Box((16, 16), (31, 39)), amr.Box((32, 16), (47, 31))])

    def run(nranks):
        def program(ctx):
            levels = []
            for lv, ba in enumerate((cba, fba)):
                dm = amr.DistributionMapping.round_robin(len(ba), nranks)
                u = amr.MultiFab(ba, dm, 1, 1, geoms[lv])
                w = amr.MultiFab(ba, dm, 1, 1, geoms[lv])
                u.fill_hash(5 + lv, geoms[lv].domain)
                w.setval(0.0)
                levels.append((u, w))
            ctx.barrier()
            for _ in range(3):
                levels = H.heat_step(levels, geoms, 1e-5, 1.0, 2)
            return {(lv, gi): bits_of(u.fabs[gi]) for lv, (u, _) in enumerate(levels) for gi in u.local_indices}
        out = {}
        for r in amr.runtime_spawn(nranks, program):
            out.update(r)
        return out

    base = run(1)
    for n in (2, 3):
        got = run(n)
        assert got.keys() == base.keys()
        for k in base:
            assert np.array_equal(got[k], base[k]), (n, k)


@pytest.mark.gpu
@pytest.mark.parametrize("ext,dt", [((70, 13, 40), np.float64), ((128, 9, 33), np.float32),
                                    ((20, 17, 35), np.float64), ((96, 5, 3), np.float64)])
def test_advance_tiles_match_oracle(ext, dt):
    """The stencil's tilings (64-wide tiles for wide regions, 32-wide
    otherwise; partial x / y tiles; z split into 32-plane tasks) against the
    oracle restatement of heat.py:172-189, raw bits, ghosts from the hash."""
    import paper_2403_12179_b200 as amr
    from paper_2403_12179_b200 import heat as H
    from gpu_util import bits_of, upload
    from oracle import amr_oracle as ao
    from oracle import inputs
    amr.config.set_spacedim(3)
    amr.config.set_real_dtype(dt)
    dom = amr.Box((0, 0, 0), tuple(e - 1 for e in ext))
    geom = amr.Geometry(dom, (0.0,) * 3, (1.0,) * 3, (True,) * 3)
    ba = amr.BoxArray([dom])
    dm = amr.DistributionMapping([0])
    u = amr.MultiFab(ba, dm, 1, 1, geom)
    w = amr.MultiFab(ba, dm, 1, 1, geom)
    g = [-1, -1, -1, ext[0], ext[1], ext[2]]
    host = inputs.make_fab(g[:3], g[3:], 1, dt, g[:3], g[3:], [-1] * 3, [e for e in ext])  # every cell hashed
    upload(u.fabs[0], host)
    w.setval(0.0)
    dt_, kappa = 1e-4, 1.0
    H.advance_level(u, w, dt_, kappa, geom)
    new = ao.advance(host, g, [0, 0, 0, *[e - 1 for e in ext]], H._coefs(dt_, kappa, geom), 3)
    full = np.zeros_like(host)
    full[1:-1, 1:-1, 1:-1, 0] = new
    exp = inputs.bits(full).ravel(order="F")
    assert np.array_equal(bits_of(w.fabs[0]), exp)
