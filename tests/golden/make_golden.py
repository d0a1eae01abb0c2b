"""Generate golden fixtures by running the REFERENCE implementation itself.

Run in the build container only (it needs /root/reference, which does not
exist on the GPU box):

    cd /tmp && PYTHONDONTWRITEBYTECODE=1 python /root/repo/tests/golden/make_golden.py

It imports ``miniamr_core`` from ``$MINIAMR_REF`` (default
``/root/reference/pkg/src``), builds BoxArray / DistributionMapping /
MultiFab layouts, fills valid cells with the deterministic hash inputs of
``oracle/inputs.py`` (ghosts poisoned), runs the reference
``fill_boundary`` / ``parallel_copy`` (serial backend, so "last writer
wins" is deterministic, core/comm.py:316-380) under ``runtime_spawn`` and
records, per case:

* the sorted plan segments with their (src_rank, dst_rank) group,
* per-call Bus message stats (messages, bytes) per ordered pair,
* every fab's raw bits after the call (small cases) or a sha256 per fab.

Scale cases (BASELINE.json configs C1-C5) record plan digests computed with
the reference plan builder ``_build_copy_segments`` + ``CommPlan`` directly
(SURVEY.md appendix B), plus C1 data digests.

Outputs: tests/golden/golden_cases.json and tests/golden/golden_data.npz.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.environ.get("MINIAMR_REF", "/root/reference/pkg/src"))

from miniamr_core import comm, config  # noqa: E402
from miniamr_core.index_space import Box, Geometry, IndexType  # noqa: E402
from miniamr_core.kernels import Backend  # noqa: E402
from miniamr_core.mesh import BoxArray, DistributionMapping, MultiFab, decompose  # noqa: E402

from oracle import inputs  # noqa: E402

CASES: list[dict] = []
ARRAYS: dict[str, np.ndarray] = {}


def pad3(v, fill=0):
    v = list(int(x) for x in v)
    return v + [fill] * (3 - len(v))


def box6(b):
    return pad3(b.lo) + pad3(b.hi)


def seg_rows(plan, src_rank_of, dst_rank_of):
    """All plan segments in CommPlan order with their (src, dst) rank group."""
    segs = []
    for lst in plan.local_by_rank.values():
        segs.extend(lst)
    for lst in plan.pair_segments.values():
        segs.extend(lst)
    segs.sort(key=lambda s: (s.dst_fab, s.dst_box.lo.comps, s.src_fab, s.shift))
    rows = []
    for s in segs:
        rows.append([s.src_fab, s.dst_fab] + box6(s.dst_box) + pad3(s.shift)
                    + [src_rank_of[s.src_fab], dst_rank_of[s.dst_fab]])
    return np.asarray(rows, np.int64).reshape(-1, 13)


def random_split(rng, lo, hi, max_boxes, min_extent=2):
    boxes = [(list(lo), list(hi))]
    while len(boxes) < max_boxes:
        cand = [n for n, (l, h) in enumerate(boxes)
                if max(hh - ll + 1 for ll, hh in zip(l, h)) >= 2 * min_extent]
        if not cand or rng.random() < 0.12:
            break
        l, h = boxes.pop(int(rng.choice(cand)))
        axes = [d for d in range(len(l)) if h[d] - l[d] + 1 >= 2 * min_extent]
        d = int(rng.choice(axes))
        cut = int(rng.integers(l[d] + min_extent, h[d] - min_extent + 2))
        h1 = list(h)
        h1[d] = cut - 1
        l2 = list(l)
        l2[d] = cut
        boxes += [(list(l), h1), (l2, list(h))]
    boxes.sort(key=lambda b: tuple(b[0]))
    return boxes


def stats_delta(a, b):
    out = []
    for pair in sorted(b):
        n = b[pair][0] - a[pair][0]
        nb = b[pair][1] - a[pair][1]
        if n or nb:
            out.append([pair[0], pair[1], n, nb])
    return np.asarray(out, np.int64).reshape(-1, 4)


def digest(arr):
    return hashlib.sha256(np.ascontiguousarray(inputs.bits(arr).ravel(order="F")).tobytes()).hexdigest()


# ---------------------------------------------------------------- FillBoundary

def run_fb_case(name, dim, domain_lo, domain_hi, boxes, rank_of, nranks, ngrow, periodic,
                ncomp, dtype, nodal=False, store="bits", calls=1):
    config.set_spacedim(dim)
    config.set_real_dtype(dtype)
    ixt = IndexType.node() if nodal else IndexType.cell()
    ba = BoxArray([Box(l, h, ixt) for l, h in boxes])
    dm = DistributionMapping(rank_of, nranks)
    geom = Geometry(Box(domain_lo, domain_hi), [0.0] * dim, [1.0] * dim, periodic)
    dlo, dhi = pad3(domain_lo), pad3(domain_hi)
    hhi = [h + (1 if nodal else 0) for h in dhi]  # hash domain (nodes incl. upper face)

    def program(ctx):
        mf = MultiFab(ba, dm, ncomp, ngrow, geom)
        for gi in mf.local_indices:
            fab = mf.fabs[gi]
            inputs.fill_fab(fab.data, pad3(fab.box.lo), pad3(ba[gi].lo), pad3(ba[gi].hi),
                            dlo, hhi)
        ctx.barrier()
        s0 = ctx.bus.stats_snapshot()
        ctx.barrier()
        for _ in range(calls):
            comm.fill_boundary(mf, geom, backend=Backend("serial"))
        ctx.barrier()
        s1 = ctx.bus.stats_snapshot()
        ctx.barrier()
        plan = comm.plan_build_fill_boundary(mf, geom)
        out = {gi: inputs.bits(mf.fabs[gi].data).copy(order="F") for gi in mf.local_indices}
        return out, stats_delta(s0, s1), plan, mf.plan_builds

    res = comm.runtime_spawn(nranks, program)
    fabs = {}
    for out, _, _, _ in res:
        fabs.update(out)
    stats = res[0][1]
    plan = res[0][2]
    rows = seg_rows(plan, dm.rank_of, dm.rank_of)
    case = dict(name=name, kind="fill_boundary", dim=dim, domain=[dlo, dhi], hash_domain=[dlo, hhi],
                boxes=[pad3(l) + pad3(h) for l, h in boxes], rank_of=list(rank_of),
                nranks=nranks, ngrow=pad3([ngrow] * dim if np.isscalar(ngrow) else ngrow),
                periodic=[bool(p) for p in periodic] + [False] * (3 - dim),
                ncomp=ncomp, dtype=np.dtype(dtype).name, nodal=nodal, calls=calls,
                num_segments=int(plan.num_segments), plan_builds=[r[3] for r in res],
                store=store)
    ARRAYS[f"{name}/segments"] = rows
    ARRAYS[f"{name}/stats"] = stats
    if store == "bits":
        for gi, a in fabs.items():
            ARRAYS[f"{name}/fab{gi}"] = a
    else:
        case["fab_sha256"] = {str(gi): hashlib.sha256(
            np.ascontiguousarray(a.ravel(order="F")).tobytes()).hexdigest()
            for gi, a in sorted(fabs.items())}
    CASES.append(case)
    config.set_spacedim(3)
    config.set_real_dtype(np.float64)


def gen_fb_random(rng, n):
    for t in range(n):
        dim = [1, 2, 2, 3, 3][t % 5]
        nranks = int(rng.integers(1, 5))
        ext = [int(rng.integers(5, 11)) for _ in range(dim)]
        periodic = [bool(rng.integers(0, 2)) for _ in range(dim)]
        boxes = random_split(rng, [0] * dim, [e - 1 for e in ext], int(rng.integers(1, 13)))
        minext = min(min(h[d] - l[d] + 1 for d in range(dim)) for l, h in boxes)
        ngrow = min(int(rng.integers(1, 3)), minext)
        nodal = (t % 4 == 3)
        if nodal and rng.random() < 0.5:
            # duplicate periodic nodes: boxes on the upper faces also own node
            # == extent (the periodic image of node 0) -> overlapping writers
            for b in boxes:
                for d in range(dim):
                    if b[1][d] == ext[d] - 1:
                        b[1][d] = ext[d]
        ncomp = int(rng.integers(1, 4))
        dtype = np.float32 if t % 6 == 5 else np.float64
        rank_of = [i % nranks for i in range(len(boxes))] if rng.random() < 0.6 else \
            [int(rng.integers(0, nranks)) for _ in boxes]
        run_fb_case(f"fb_rand_{t:02d}", dim, [0] * dim, [e - 1 for e in ext], boxes, rank_of,
                    nranks, ngrow, periodic, ncomp, dtype, nodal=nodal,
                    calls=1 + (t % 2))


# ---------------------------------------------------------------- ParallelCopy

def run_pc_case(name, dim, domain_lo, domain_hi, src_boxes, src_rank, dst_boxes, dst_rank,
                nranks, src_ngrow, dst_ngrow, ngrow_src, ngrow_dst, src_ncomp, dst_ncomp,
                scomp, dcomp, ncomp, periodic, dtype, nodal=False):
    config.set_spacedim(dim)
    config.set_real_dtype(dtype)
    ixt = IndexType.node() if nodal else IndexType.cell()
    sba = BoxArray([Box(l, h, ixt) for l, h in src_boxes])
    dba = BoxArray([Box(l, h, ixt) for l, h in dst_boxes])
    sdm = DistributionMapping(src_rank, nranks)
    ddm = DistributionMapping(dst_rank, nranks)
    geom = None if periodic is None else Geometry(Box(domain_lo, domain_hi), [0.0] * dim,
                                                   [1.0] * dim, periodic)
    dlo, dhi = pad3(domain_lo), pad3(domain_hi)
    hhi = [h + (1 if nodal else 0) for h in dhi]

    def program(ctx):
        src = MultiFab(sba, sdm, src_ncomp, src_ngrow)
        dst = MultiFab(dba, ddm, dst_ncomp, dst_ngrow)
        for gi in src.local_indices:
            fab = src.fabs[gi]
            inputs.fill_fab(fab.data, pad3(fab.box.lo), pad3(sba[gi].lo), pad3(sba[gi].hi),
                            dlo, hhi, ghost_tag=gi + 1)
        for gi in dst.local_indices:
            fab = dst.fabs[gi]
            inputs.fill_fab(fab.data, pad3(fab.box.lo), pad3(dba[gi].lo), pad3(dba[gi].hi),
                            dlo, hhi, seed=inputs.SEED + 1)
        ctx.barrier()
        s0 = ctx.bus.stats_snapshot()
        ctx.barrier()
        comm.parallel_copy(dst, src, scomp=scomp, dcomp=dcomp, ncomp=ncomp,
                           ngrow_src=ngrow_src, ngrow_dst=ngrow_dst, geom=geom,
                           backend=Backend("serial"))
        ctx.barrier()
        s1 = ctx.bus.stats_snapshot()
        ctx.barrier()
        plan = list(dst.plan_cache.values())[0]
        out = {gi: inputs.bits(dst.fabs[gi].data).copy(order="F") for gi in dst.local_indices}
        return out, stats_delta(s0, s1), plan

    res = comm.runtime_spawn(nranks, program)
    fabs = {}
    for out, _, _ in res:
        fabs.update(out)
    plan = res[0][2]
    case = dict(name=name, kind="parallel_copy", dim=dim, domain=[dlo, dhi], hash_domain=[dlo, hhi],
                src_boxes=[pad3(l) + pad3(h) for l, h in src_boxes], src_rank=list(src_rank),
                dst_boxes=[pad3(l) + pad3(h) for l, h in dst_boxes], dst_rank=list(dst_rank),
                nranks=nranks, src_ngrow=pad3([src_ngrow] * dim), dst_ngrow=pad3([dst_ngrow] * dim),
                ngrow_src=pad3([ngrow_src] * dim), ngrow_dst=pad3([ngrow_dst] * dim),
                src_ncomp=src_ncomp, dst_ncomp=dst_ncomp, scomp=scomp, dcomp=dcomp, ncomp=ncomp,
                periodic=None if periodic is None else [bool(p) for p in periodic] + [False] * (3 - dim),
                dtype=np.dtype(dtype).name, nodal=nodal, num_segments=int(plan.num_segments),
                store="bits")
    ARRAYS[f"{name}/segments"] = seg_rows(plan, sdm.rank_of, ddm.rank_of)
    ARRAYS[f"{name}/stats"] = res[0][1]
    for gi, a in fabs.items():
        ARRAYS[f"{name}/fab{gi}"] = a
    CASES.append(case)
    config.set_spacedim(3)
    config.set_real_dtype(np.float64)


def gen_pc_random(rng, n):
    for t in range(n):
        dim = [1, 2, 3][t % 3]
        nranks = int(rng.integers(1, 5))
        ext = [int(rng.integers(5, 11)) for _ in range(dim)]
        hi = [e - 1 for e in ext]
        sb = random_split(rng, [0] * dim, hi, int(rng.integers(1, 9)))
        db = random_split(rng, [0] * dim, hi, int(rng.integers(1, 9)))
        ngrow_src = int(rng.integers(0, 2))
        ngrow_dst = int(rng.integers(0, 2))
        src_ncomp = int(rng.integers(1, 4))
        dst_ncomp = int(rng.integers(1, 4))
        scomp = int(rng.integers(0, src_ncomp))
        dcomp = int(rng.integers(0, dst_ncomp))
        ncomp = int(rng.integers(1, min(src_ncomp - scomp, dst_ncomp - dcomp) + 1))
        periodic = None if t % 2 == 0 else [bool(rng.integers(0, 2)) for _ in range(dim)]
        dtype = np.float32 if t % 5 == 4 else np.float64
        nodal = (t % 7 == 6)
        run_pc_case(f"pc_rand_{t:02d}", dim, [0] * dim, hi,
                    sb, [int(rng.integers(0, nranks)) for _ in sb],
                    db, [i % nranks for i in range(len(db))], nranks,
                    src_ngrow=ngrow_src + int(rng.integers(0, 2)), dst_ngrow=ngrow_dst,
                    ngrow_src=ngrow_src, ngrow_dst=ngrow_dst, src_ncomp=src_ncomp,
                    dst_ncomp=dst_ncomp, scomp=scomp, dcomp=dcomp, ncomp=ncomp,
                    periodic=periodic, dtype=dtype, nodal=nodal)


# ---------------------------------------------------------------- scale plans

def scale_plan(name, n, bsize, ng, nranks_list, ncomp, extra=None):
    config.set_spacedim(3)
    dom = Box((0, 0, 0), (n - 1,) * 3)
    geom = Geometry(dom, (0.0,) * 3, (1.0,) * 3, (True,) * 3)
    boxes = []
    for bz in range(0, n, bsize):
        for by in range(0, n, bsize):
            for bx in range(0, n, bsize):
                boxes.append(Box((bx, by, bz), (bx + bsize - 1, by + bsize - 1, bz + bsize - 1)))
    t0 = time.time()
    from miniamr_core.index_space import grow
    segs = comm._build_copy_segments([(grow(b, ng), b) for b in boxes], boxes, geom,
                                     exclude_valid=True)
    t_build = time.time() - t0
    for G in nranks_list:
        rank_of = [i % G for i in range(len(boxes))]
        plan = comm.CommPlan(segs, rank_of, rank_of, G)
        rows = seg_rows(plan, rank_of, rank_of)
        pair_bytes = {f"{s}->{d}": int(sum(x.cells for x in lst)) * ncomp * 8
                      for (s, d), lst in sorted(plan.pair_segments.items())}
        local_cells = {str(r): int(sum(x.cells for x in lst))
                       for r, lst in sorted(plan.local_by_rank.items())}
        case = dict(name=f"{name}_x{G}", kind="plan_fill_boundary", n=n, box=bsize, ngrow=ng,
                    ncomp=ncomp, nranks=G, num_segments=int(plan.num_segments),
                    seg_sha256=hashlib.sha256(np.ascontiguousarray(rows).astype("<i8").tobytes()).hexdigest(),
                    pair_bytes=pair_bytes, local_cells=local_cells,
                    ref_build_seconds=round(t_build, 3))
        if plan.num_segments <= 20000:
            ARRAYS[f"{name}_x{G}/segments"] = rows.astype(np.int32)
        CASES.append(case)
        print(f"  {name}_x{G}: {plan.num_segments} segs, build {t_build:.1f}s", flush=True)


def scale_pc_plan(name, n, sb, db, nranks, ncomp):
    config.set_spacedim(3)

    def chop(b):
        return [Box((x, y, z), (x + b - 1, y + b - 1, z + b - 1))
                for z in range(0, n, b) for y in range(0, n, b) for x in range(0, n, b)]
    src = chop(sb)
    dst = chop(db)
    t0 = time.time()
    segs = comm._build_copy_segments([(b, b) for b in dst], src, None, exclude_valid=False)
    t_build = time.time() - t0
    srank = [i % nranks for i in range(len(src))]
    drank = [i % nranks for i in range(len(dst))]
    plan = comm.CommPlan(segs, srank, drank, nranks)
    rows = seg_rows(plan, srank, drank)
    pair_bytes = {f"{s}->{d}": int(sum(x.cells for x in lst)) * ncomp * 8
                  for (s, d), lst in sorted(plan.pair_segments.items())}
    local_cells = {str(r): int(sum(x.cells for x in lst))
                   for r, lst in sorted(plan.local_by_rank.items())}
    CASES.append(dict(name=name, kind="plan_parallel_copy", n=n, src_box=sb, dst_box=db,
                      ncomp=ncomp, nranks=nranks, num_segments=int(plan.num_segments),
                      seg_sha256=hashlib.sha256(np.ascontiguousarray(rows).astype("<i8").tobytes()).hexdigest(),
                      pair_bytes=pair_bytes, local_cells=local_cells,
                      ref_build_seconds=round(t_build, 3)))
    ARRAYS[f"{name}/segments"] = rows.astype(np.int32)
    print(f"  {name}: {plan.num_segments} segs, build {t_build:.1f}s", flush=True)


def main():
    rng = np.random.default_rng(20261017)
    t0 = time.time()
    # reference known-answer layout (tests/test_comm.py:168-210): 1-D periodic
    run_fb_case("fb_1d_known", 1, [0], [7], [([0], [3]), ([4], [7])], [0, 0], 1, 1, [True],
                1, np.float64)
    run_fb_case("fb_1d_known_2rank", 1, [0], [7], [([0], [3]), ([4], [7])], [0, 1], 2, 1,
                [True], 2, np.float64)
    # aggregation layout (tests/test_comm.py:407-422): 12x12, 2x2 boxes, 4 ranks
    boxes = [([x, y], [x + 5, y + 5]) for y in (0, 6) for x in (0, 6)]
    run_fb_case("fb_2d_aggregation", 2, [0, 0], [11, 11], boxes, [0, 1, 2, 3], 4, 1,
                [True, True], 1, np.float64)
    gen_fb_random(rng, 60)
    gen_pc_random(rng, 36)
    # C1 end to end (1 and 2 ranks): data digests
    boxes = [([x, y, z], [x + 31, y + 31, z + 31]) for z in (0, 32) for y in (0, 32) for x in (0, 32)]
    for G in (1, 2):
        run_fb_case(f"C1_data_x{G}", 3, [0] * 3, [63] * 3, boxes, [i % G for i in range(8)], G, 1,
                    [True] * 3, 1, np.float64, store="sha256")
    print(f"small cases done in {time.time() - t0:.1f}s", flush=True)
    scale_plan("C1", 64, 32, 1, [1, 2], 1)
    scale_plan("C2", 256, 64, 2, [1], 4)
    scale_plan("C3", 512, 128, 2, [1, 2, 4, 8], 8)
    scale_pc_plan("C5", 1024, 64, 128, 8, 4)
    if os.environ.get("GOLDEN_SKIP_C4") != "1":
        scale_plan("C4", 256, 16, 2, [1], 4)
    with open(os.path.join(HERE, "golden_cases.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py",
                   "reference": "miniamr_core (pkg/src) from /root/reference",
                   "cases": CASES}, f, indent=1)
    np.savez_compressed(os.path.join(HERE, "golden_data.npz"), **ARRAYS)
    print(f"wrote {len(CASES)} cases, {len(ARRAYS)} arrays in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
