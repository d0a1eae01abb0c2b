"""Coarse/fine level-transfer throughput on one B200 (SURVEY.md section 8f
rows 1-2): fill_patch (FillBoundary + coarse gather + interpolation) and
average_down (restriction + ParallelCopy).

    python bench_amr.py [--op fill_patch|average_down|heat|heat2] [--steps K] [--warmup W]

Workload (synthetic, splitmix64 hash data): a 256^3 periodic coarse level
cut into 64^3 boxes, ncomp 4, float64; the fine level refines the central
128^3 coarse cells by 2 (a 256^3 fine patch of 64 boxes of 64^3, nghost 2).
fill_patch is LINEAR.  One JSON line per op: whole-call time (CUDA events
around the public call, L2 flushed before each step), the dominant kernel's
event time against the measured HBM copy bandwidth, the numpy oracle of
the reference arithmetic timed on a sample on the host, and the reference's
OWN public call on the same full workload (``reference_cpu``: miniamr_core
from baseline/_ref, Backend("parallel", all host cores); GHX_AMR_NO_REF=1
skips it).
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

import bench  # noqa: E402  (the CPU-baseline legs live in bench.py)

N_CRSE, BOX, NCOMP, NGROW, RATIO = 256, 64, 4, 2, 2
PATCH_LO, PATCH_HI = 64, 191  # coarse cells refined


def peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def layout(amr):
    amr.config.set_spacedim(3)
    cdom = amr.Box((0, 0, 0), (N_CRSE - 1,) * 3)
    cgeom = amr.Geometry(cdom, (0.0,) * 3, (1.0,) * 3, (True,) * 3)
    fgeom = cgeom.refined(RATIO)
    cba = amr.decompose(cdom, BOX)
    patch = amr.Box((PATCH_LO * RATIO,) * 3, ((PATCH_HI + 1) * RATIO - 1,) * 3)
    fba = amr.decompose(patch, BOX)
    return cdom, cgeom, fgeom, cba, fba


def timed(fn, steps, warmup, flush, clean):
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(steps):
        flush.zero_()
        torch.sum(clean)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    return statistics.mean(ts), min(ts)


def reference_leg(op, seconds=20.0, max_reps=20):
    """The reference's OWN level transfer on the same workload, on the host
    cores: miniamr_core (baseline/_ref) with Backend("parallel",
    os.cpu_count()), its public amr.fill_patch / amr.average_down, and for
    the heat ops its demo loop body (comm.fill_boundary + heat._advance_level
    [+ fill_patch + average_down], reference core/heat.py:264-273).  Valid
    cells: the splitmix64 hash of oracle/inputs.py.  The first call builds
    the plans (reported separately); then timed calls (perf_counter) until
    ``seconds`` or ``max_reps``, at least 2.  Returns (seconds per call,
    dict) or (None, reason)."""
    ref, where = bench.import_reference()
    if ref is None:
        return None, "reference package not importable (baseline/_ref missing)"
    from concurrent.futures import ThreadPoolExecutor
    from miniamr_core import amr as ramr, comm as rcomm, config as rconfig, heat as rheat
    from miniamr_core.index_space import Box as RBox, Geometry as RGeometry
    from miniamr_core.kernels import Backend
    from miniamr_core.mesh import DistributionMapping as RDM, MultiFab as RMF, decompose as rdecompose
    from oracle import inputs
    rconfig.set_spacedim(3)
    rconfig.set_real_dtype(np.float64)
    cdom = RBox((0, 0, 0), (N_CRSE - 1,) * 3)
    cgeom = RGeometry(cdom, (0.0,) * 3, (1.0,) * 3, (True,) * 3)
    fgeom = cgeom.refined(RATIO)
    cba = rdecompose(cdom, BOX)
    fba = rdecompose(RBox((PATCH_LO * RATIO,) * 3, ((PATCH_HI + 1) * RATIO - 1,) * 3), BOX)
    backend = Backend("parallel", os.cpu_count())
    pool = ThreadPoolExecutor(os.cpu_count() or 1)

    def mf(ba, geom, nc, ng):
        m = RMF(ba, RDM.round_robin(len(ba), 1), nc, ng, geom)
        dlo, dhi = list(geom.domain.lo), list(geom.domain.hi)

        def one(gi):
            f = m.fabs[gi]
            inputs.fill_fab(f.data, list(f.box.lo), list(ba[gi].lo), list(ba[gi].hi), dlo, dhi)
        list(pool.map(one, m.local_indices))
        return m

    dt, kappa = 1e-6, 1.0
    if op == "fill_patch":
        coarse, fine = mf(cba, cgeom, NCOMP, 0), mf(fba, fgeom, NCOMP, NGROW)
        call = lambda: ramr.fill_patch(fine, coarse, fgeom, cgeom, RATIO, ramr.LINEAR, backend=backend)  # noqa: E731
    elif op == "average_down":
        coarse, fine = mf(cba, cgeom, NCOMP, 0), mf(fba, fgeom, NCOMP, NGROW)
        call = lambda: ramr.average_down(fine, coarse, RATIO, backend)  # noqa: E731
    elif op == "heat":
        u, w = mf(cba, cgeom, 1, 1), mf(cba, cgeom, 1, 1)

        def call():
            rcomm.fill_boundary(u, cgeom, backend=backend)
            rheat._advance_level(u, w, dt, kappa, cgeom, backend)
    else:  # heat2: the two-level step
        lv = [(mf(cba, cgeom, 1, 1), mf(cba, cgeom, 1, 1)), (mf(fba, fgeom, 1, 1), mf(fba, fgeom, 1, 1))]
        geoms = [cgeom, fgeom]

        def call():
            rcomm.fill_boundary(lv[0][0], cgeom, backend=backend)
            ramr.fill_patch(lv[1][0], lv[0][0], fgeom, cgeom, RATIO, ramr.LINEAR, backend=backend)
            for k, (u, w) in enumerate(lv):
                rheat._advance_level(u, w, dt, kappa, geoms[k], backend)
            ramr.average_down(lv[1][1], lv[0][1], RATIO, backend)
    pool.shutdown()
    t0 = time.perf_counter()
    call()  # plans built and cached, pages touched
    first = time.perf_counter() - t0
    times, t_end = [], time.perf_counter() + seconds
    while len(times) < 2 or (time.perf_counter() < t_end and len(times) < max_reps):
        a = time.perf_counter()
        call()
        times.append(time.perf_counter() - a)
    t = statistics.median(times)
    return t, {"kind": "reference", "cores": backend.nworkers, "reps": len(times),
               "ms_per_call": round(t * 1e3, 2), "first_call_s": round(first, 3), "where": where,
               "sample": "the full workload through the reference's public call (miniamr_core from baseline/_ref, "
                         f"Backend('parallel', {backend.nworkers})), same layout, splitmix64 valid cells; median "
                         f"of {len(times)} calls after the plan-building first call",
               "cpu_model": bench.cpu_model()}


def attach_reference(out, op, work):
    """Add the reference's timing on the same metric to the line."""
    if os.environ.get("GHX_AMR_NO_REF"):
        return
    t, info = reference_leg(op)
    if t is None:
        out["reference_cpu"] = {"unavailable": info}
        return
    info["value"] = round(work / t / (1e9 if out["unit"] in ("GB/s", "Gcell/s") else 1), 4)
    info["unit"] = out["unit"]
    out["reference_cpu"] = info
    out["speedup_vs_reference"] = round(out["value"] / info["value"], 1) if info["value"] else None


def run(args):
    import torch
    import paper_2403_12179_b200 as amr
    from paper_2403_12179_b200 import _native as N
    from paper_2403_12179_b200 import amr as A
    torch.cuda.set_device(0)
    cdom, cgeom, fgeom, cba, fba = layout(amr)
    coarse = amr.MultiFab(cba, amr.DistributionMapping([0] * len(cba)), NCOMP, 0, cgeom)
    fine = amr.MultiFab(fba, amr.DistributionMapping([0] * len(fba)), NCOMP, NGROW, fgeom)
    coarse.fill_hash(20261018, cdom)
    fine.fill_hash(20261017, fgeom.domain)
    torch.cuda.synchronize()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    clean = torch.ones(64 << 20, dtype=torch.int32, device="cuda")
    hbm, peak_src = peaks()
    item = 8
    out = {"op": args.op, "unit": "GB/s", "dtype": "f64", "steps": args.steps, "warmup": args.warmup,
           "data": "synthetic (splitmix64 hash valid cells)",
           "config": {"workload": f"coarse {N_CRSE}^3 periodic / {BOX}^3 boxes, fine patch = coarse cells "
                                  f"[{PATCH_LO},{PATCH_HI}]^3 refined x{RATIO} ({len(fba)} boxes of {BOX}^3, "
                                  f"nghost {NGROW}), ncomp {NCOMP}, float64",
                      "l2": "flushed before every step (512 MiB write + 256 MiB clean read, outside the events)"}}
    if args.op in ("heat", "heat2"):
        pass
    elif args.op == "fill_patch":
        call = lambda: A.fill_patch(fine, coarse, fgeom, cgeom, RATIO, A.LINEAR)  # noqa: E731
        t_mean, t_min = timed(call, args.steps, args.warmup, flush, clean)
        ghost_cells = sum(amr.grow(b, NGROW).num_pts - b.num_pts for b in fba)
        ghost_bytes = ghost_cells * NCOMP * item
        # the interp launch alone: the plan-cached prepared transfer
        key = [k for k in fine.plan_cache if getattr(k, "op", "") == "fill_patch"][0]
        targets = fine.plan_cache[key][0]
        xf = [v for k, v in fine._peer_cache.items() if isinstance(k, tuple) and k[0] == "fill_patch_interp"][0]
        regions = [r for gi in targets for r in targets[gi]]
        interp_cells = sum(r.num_pts for r in regions)
        assert interp_cells == xf.cells
        # coarse cells the LINEAR stencil reads (parents grown by 1), per region
        crse_cells = sum(amr.grow(amr.coarsen(r, RATIO), 1).num_pts for r in regions)
        k_mean, _ = timed(xf.run, args.steps, args.warmup, flush, clean)
        alg = (interp_cells + crse_cells) * NCOMP * item
        out.update(metric="fill_patch fine-ghost GB/s (FillBoundary + coarse gather + LINEAR interp)",
                   value=round(ghost_bytes / t_mean / 1e9, 2), ms_per_step=round(t_mean * 1e3, 4),
                   ghost_bytes_per_step=ghost_bytes, interp_cells=interp_cells,
                   roofline={"kernel": "interp_kernel<double,LINEAR>", "bound": "hbm",
                             "algorithmic_bytes_per_launch": alg,
                             "achieved": round(alg / k_mean / 1e9, 1), "peak": hbm,
                             "frac": round(alg / k_mean / 1e9 / hbm, 4), "unit": "GB/s", "peak_source": peak_src,
                             "kernel_ms": round(k_mean * 1e3, 4)})
        out["cpu_baseline"] = bench.cpu_sample_interp(fine, targets, NCOMP, NGROW, RATIO)
        attach_reference(out, "fill_patch", ghost_bytes)
    else:
        crse_fine = amr.MultiFab(cba, amr.DistributionMapping([0] * len(cba)), NCOMP, 0, cgeom)
        call = lambda: A.average_down(fine, crse_fine, RATIO)  # noqa: E731
        t_mean, t_min = timed(call, args.steps, args.warmup, flush, clean)
        fine_cells = sum(b.num_pts for b in fba)
        crse_cells = fine_cells // RATIO ** 3
        xf = [v for k, v in fine._peer_cache.items()
              if isinstance(k, tuple) and k[0] in ("average_down_xfer", "average_down_direct")][0]
        k_mean, _ = timed(xf.run, args.steps, args.warmup, flush, clean)
        alg = (fine_cells + crse_cells) * NCOMP * item
        out.update(metric="average_down GB/s (fine bytes restricted, restriction + ParallelCopy)",
                   path="direct restriction into the coarse fabs (single rank)"
                   if os.environ.get("GHX_AVGDOWN_DIRECT", "1") != "0" else "restriction into tmp + ParallelCopy",
                   value=round(fine_cells * NCOMP * item / t_mean / 1e9, 2), ms_per_step=round(t_mean * 1e3, 4),
                   roofline={"kernel": "avgdown_kernel<double>", "bound": "hbm", "algorithmic_bytes_per_launch": alg,
                             "achieved": round(alg / k_mean / 1e9, 1), "peak": hbm,
                             "frac": round(alg / k_mean / 1e9 / hbm, 4), "unit": "GB/s", "peak_source": peak_src,
                             "kernel_ms": round(k_mean * 1e3, 4)})
        out["cpu_baseline"] = bench.cpu_sample_restrict(BOX, NGROW, NCOMP, RATIO)
        attach_reference(out, "average_down", fine_cells * NCOMP * item)
    if args.op == "heat":
        out.update(heat_bench(args, amr, cdom, cgeom, cba, flush, clean, hbm, peak_src))
        attach_reference(out, "heat", sum(b.num_pts for b in cba))
    if args.op == "heat2":
        out.update(heat2_bench(args, amr, cdom, cgeom, cba, fba, fgeom, flush, clean))
        attach_reference(out, "heat2", sum(b.num_pts for b in cba) + sum(b.num_pts for b in fba))
    out["amr_launches"] = int(N.lib.ghx_amr_launch_count())
    print(json.dumps(out), flush=True)


def heat_bench(args, amr, cdom, cgeom, cba, flush, clean, hbm, peak_src):
    """One heat_step (FillBoundary + stencil, the reference demo's single-level
    loop body) on the coarse layout with ncomp 1, nghost 1; overlap on/off."""
    from paper_2403_12179_b200 import heat as H
    dm = amr.DistributionMapping([0] * len(cba))
    u = amr.MultiFab(cba, dm, 1, 1, cgeom)
    w = amr.MultiFab(cba, dm, 1, 1, cgeom)
    u.fill_hash(20261017, cdom)
    w.setval(0.0)
    state = {"levels": [(u, w)]}
    dt, kappa = 1e-6, 1.0
    res = {}
    for ov in (True, False):
        def step(ov=ov):
            state["levels"] = H.heat_step(state["levels"], [cgeom], dt, kappa, overlap=ov)
        t_mean, _ = timed(step, args.steps, args.warmup, flush, clean)
        res["overlap" if ov else "serial"] = round(t_mean * 1e3, 4)
    loop = H.HeatLoop(state["levels"], [cgeom], dt, kappa)
    t_graph, _ = timed(loop.step, args.steps, args.warmup, flush, clean)
    res["graph"] = round(t_graph * 1e3, 4)
    state["levels"] = loop.levels
    cells = sum(b.num_pts for b in cba)
    xf = H._stencil(state["levels"][0][0], state["levels"][0][1], dt, kappa, cgeom, "all")
    k_mean, _ = timed(xf.run, args.steps, args.warmup, flush, clean)
    alg = cells * 16  # read u + write unew, 8 B each (neighbour reads hit L1/L2)
    return {"metric": "heat_step cells/s (FillBoundary + 7-point stencil, reference demo loop body)",
            "value": round(cells / (res["serial"] * 1e-3) / 1e9, 3), "unit": "Gcell/s",
            "ms_per_step": res["serial"], "ms_per_step_overlap": res["overlap"],
            "ms_per_step_cuda_graph": res["graph"],
            "config": {"workload": f"{N_CRSE}^3 periodic, {BOX}^3 boxes, ncomp 1, nghost 1, float64 "
                                   "(the reference heat demo layout)",
                       "l2": "flushed before every step (512 MiB write + 256 MiB clean read, outside the events)"},
            "roofline": {"kernel": "advance_kernel<double,3>", "bound": "hbm", "algorithmic_bytes_per_launch": alg,
                         "achieved": round(alg / k_mean / 1e9, 1), "peak": hbm,
                         "frac": round(alg / k_mean / 1e9 / hbm, 4), "unit": "GB/s", "peak_source": peak_src,
                         "kernel_ms": round(k_mean * 1e3, 4)}}


def heat2_bench(args, amr, cdom, cgeom, cba, fba, fgeom, flush, clean):
    """The two-level heat step (FillBoundary, fill_patch LINEAR, stencil on
    both levels, average_down): eager vs CUDA-graph replay (HeatLoop)."""
    from paper_2403_12179_b200 import heat as H

    def make():
        levels = []
        for lv, (ba, geom) in enumerate(((cba, cgeom), (fba, fgeom))):
            dm = amr.DistributionMapping([0] * len(ba))
            u = amr.MultiFab(ba, dm, 1, 1, geom)
            w = amr.MultiFab(ba, dm, 1, 1, geom)
            u.fill_hash(20261017 + lv, geom.domain)
            w.setval(0.0)
            levels.append((u, w))
        return levels
    geoms = [cgeom, fgeom]
    state = {"levels": make()}

    def eager():
        state["levels"] = H.heat_step(state["levels"], geoms, 1e-7, 1.0, RATIO)
    t_eager, _ = timed(eager, args.steps, args.warmup, flush, clean)
    loop = H.HeatLoop(make(), geoms, 1e-7, 1.0, RATIO)
    t_graph, _ = timed(loop.step, args.steps, args.warmup, flush, clean)
    cells = sum(b.num_pts for b in cba) + sum(b.num_pts for b in fba)
    return {"metric": "two-level heat step cells/s (FB + fill_patch + stencils + average_down)",
            "value": round(cells / t_graph / 1e9, 3), "unit": "Gcell/s",
            "ms_per_step": round(t_graph * 1e3, 4), "ms_per_step_eager": round(t_eager * 1e3, 4),
            "config": {"workload": f"coarse {N_CRSE}^3 periodic / {BOX}^3 boxes + fine patch of {len(fba)} "
                                   f"{BOX}^3 boxes at ratio {RATIO}, ncomp 1, nghost 1, float64",
                       "l2": "flushed before every step (512 MiB write + 256 MiB clean read, outside the events)"}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--op", default="fill_patch", choices=["fill_patch", "average_down", "heat", "heat2"])
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    run(args)


if __name__ == "__main__":
    main()
