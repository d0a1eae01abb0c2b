"""FillBoundary / ParallelCopy ghost-cell throughput on B200 (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3]
                    [--impl ours|reference] [--transport p2p|nccl]

N>1 runs under torchrun (one process per GPU, NCCL process group for the
plumbing).  Rank 0 prints ONE JSON line.

Default workload: C3 = BASELINE.json configs[2] (512^3 periodic, 128^3
boxes, 8 components, 2 ghosts, float64) -- the north-star config -- at every
N (strong scaling: the same 64 boxes round-robin over N GPUs; 9.4 GB, so it
also fits one B200).  ``--config C2`` etc. select the other BASELINE configs.

A "step" is one FillBoundary (C1-C4) or ParallelCopy (C5) of the whole
synthetic MultiFab.  ``value`` is whole-job ghost bytes per second (ghost
cells x ncomp x 8 B, counted once) with the fabs
resident in HBM, timed on the device with CUDA events around each step
(L2 flushed before every step, outside the events), max over ranks.
``e2e`` is the same metric through the public API on host-resident (pinned,
mapped) fabs: every byte the exchange reads crosses PCIe host->device and
every ghost it writes crosses device->host inside the timed region.
``roofline`` (N=1) is the fused kernel's algorithmic bytes (8 B read + 8 B
write per ghost value) over its event-timed duration against the measured
HBM copy bandwidth; at N>1 it is the per-GPU NVLink bytes (max over GPUs of
max(send, recv)) against the measured 770 GB/s peer copy when that term
dominates, with the HBM share reported beside it.

``cpu_baseline`` (rank 0, N=1) and ``--impl reference`` run the REFERENCE
itself -- ``miniamr_core`` installed in ``baseline/_ref`` (or
``$MINIAMR_REF``) -- through its public ``comm.fill_boundary`` /
``comm.parallel_copy`` with ``Backend("parallel", os.cpu_count())`` on the
same layout and the same splitmix64 inputs, ranks as ``runtime_spawn``
threads (reference comm.py:143-180).  Only when the reference is not
importable (or the config needs more host RAM than the box has) does it
fall back to the numpy port of the reference algorithm (oracle/), and the
line then says ``"kind": "port"``.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

SEED = 20261017
CONFIGS = {
    "C1": dict(kind="fb", n=64, box=32, ncomp=1, ngrow=1,
               desc="C1: 64^3 periodic domain, 32^3 boxes, ncomp 1, nghost 1, float64 FillBoundary"),
    "C2": dict(kind="fb", n=256, box=64, ncomp=4, ngrow=2,
               desc="C2: 256^3 periodic domain, 64^3 boxes, ncomp 4, nghost 2, float64 FillBoundary"),
    "C3": dict(kind="fb", n=512, box=128, ncomp=8, ngrow=2,
               desc="C3: 512^3 periodic domain, 128^3 boxes, ncomp 8, nghost 2, float64 FillBoundary"),
    "C4": dict(kind="fb", n=256, box=16, ncomp=4, ngrow=2,
               desc="C4: 256^3 periodic domain, 16^3 boxes (many-small-box stress), ncomp 4, nghost 2, float64 FillBoundary"),
    # not a BASELINE config: the heat demo's exchange (the FillBoundary inside bench_amr.py --op heat)
    "H1": dict(kind="fb", n=256, box=64, ncomp=1, ngrow=1,
               desc="H1: 256^3 periodic domain, 64^3 boxes, ncomp 1, nghost 1, float64 FillBoundary (heat demo layout)"),
    "C5": dict(kind="pc", n=1024, src_box=64, box=128, ncomp=4, ngrow=0,
               desc="C5: ParallelCopy regrid 1024^3, 64^3-box layout -> 128^3-box layout, ncomp 4, float64"),
}
METRIC = "FillBoundary ghost-cell GB/s (+% HBM/NVLink roofline) at 1/2/4/8 B200 vs host CPU"
NVLINK_PEER_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def traffic_model_min(cfg):
    """Minimum DRAM bytes of one FillBoundary launch on the uniform periodic
    layout (scripts/traffic_model.py): 128-B lines holding source cells must
    be read, 32-B sectors holding ghost cells must be written."""
    if cfg["kind"] != "fb" or not isinstance(cfg["ngrow"], int):
        return None
    b, g = cfg["box"], cfg["ngrow"]
    n = b + 2 * g
    idx = np.arange(n)
    valid = (idx >= g) & (idx < g + b)
    src1 = valid & ((idx < 2 * g) | (idx >= b))
    X, Y, Z = np.meshgrid(idx, idx, idx, indexing="ij")
    isvalid = valid[X] & valid[Y] & valid[Z]
    src = isvalid & (src1[X] | src1[Y] | src1[Z])
    off = (X + n * (Y + n * Z)) * 8
    lines = np.unique(off[src] // 128).size
    sectors = np.unique(off[~isvalid] // 32).size
    nfabs = int(np.prod([e // b for e in cfg["ext"]]))
    return float((lines * 128 + sectors * 32) * cfg["ncomp"] * nfabs)


def ncu_traffic(cfg_name):
    p = os.path.join(REPO, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        v = d.get(cfg_name)
        return None if v is None else float(v["dram_bytes_per_launch"])
    except Exception:
        return None


# ----------------------------------------------------------------- layout

def scaled(cfg, world):
    """Every config is fixed-size: at N GPUs the same global MultiFab is
    distributed round-robin over N ranks (strong scaling)."""
    cfg = dict(cfg)
    cfg["ext"] = (cfg["n"],) * 3
    return cfg


def layout(amr, cfg, G):
    amr.config.set_spacedim(3)
    ext = cfg.get("ext", (cfg["n"],) * 3)
    dom = amr.Box((0, 0, 0), tuple(e - 1 for e in ext))
    geom = amr.Geometry(dom, (0.0,) * 3, (1.0,) * 3, (True,) * 3)
    t0 = time.perf_counter()
    ba = amr.decompose(dom, cfg["box"])  # BoxArray ctor incl. the disjointness check
    dm = amr.DistributionMapping.round_robin(len(ba), G)
    out = dict(dom=dom, geom=geom, ba=ba, dm=dm)
    if cfg["kind"] == "pc":
        out["sba"] = amr.decompose(dom, cfg["src_box"])
        out["sdm"] = amr.DistributionMapping.round_robin(len(out["sba"]), G)
    out["boxarray_s"] = time.perf_counter() - t0
    return out


def make_fields(amr, cfg, L, memory="device"):
    if cfg["kind"] == "fb":
        ng = cfg["ngrow"]
        ng = amr.IntVect(*ng) if isinstance(ng, tuple) else ng
        mf = amr.MultiFab(L["ba"], L["dm"], cfg["ncomp"], ng, L["geom"], memory=memory)
        mf.fill_hash(SEED, L["dom"])
        return mf, None
    src = amr.MultiFab(L["sba"], L["sdm"], cfg["ncomp"], 0, memory=memory)
    dst = amr.MultiFab(L["ba"], L["dm"], cfg["ncomp"], 0, memory=memory)
    src.fill_hash(SEED, L["dom"])
    return dst, src


def prepare(amr, cfg, L, mf, src):
    from paper_2403_12179_b200 import comm
    t0 = time.perf_counter()
    if cfg["kind"] == "fb":
        plan = comm.plan_build_fill_boundary(mf, L["geom"])
        t1 = time.perf_counter()
        x = comm.exchange_for(plan, mf, mf, 0, 0, mf.ncomp)
    else:
        plan = comm._parallel_copy_plan(mf, src, amr.IntVect.zero(), amr.IntVect.zero(), None)
        t1 = time.perf_counter()
        x = comm.exchange_for(plan, src, mf, 0, 0, mf.ncomp)
    t2 = time.perf_counter()
    return plan, x, t1 - t0, t2 - t1


def public_call(amr, cfg, L, mf, src):
    if cfg["kind"] == "fb":
        amr.fill_boundary(mf, L["geom"])
    else:
        amr.parallel_copy(mf, src)


# ----------------------------------------------------------------- clocks

class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device, period=0.01):
        self.ok = False
        self.samples, self.reasons, self.mem_samples = [], set(), []
        try:
            import pynvml
            pynvml.nvmlInit()
            uuid = None
            try:
                import torch
                uuid = str(torch.cuda.get_device_properties(device).uuid)
            except Exception:
                pass
            self.h = None
            if uuid:
                for i in range(pynvml.nvmlDeviceGetCount()):
                    h = pynvml.nvmlDeviceGetHandleByIndex(i)
                    u = pynvml.nvmlDeviceGetUUID(h)
                    u = u.decode() if isinstance(u, bytes) else u
                    if u.replace("GPU-", "") == uuid.replace("GPU-", ""):
                        self.h = h
            if self.h is None:
                self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # noqa: BLE001
            log(f"[bench] clock sampling unavailable: {e}")
        self.period = period
        self._stop = threading.Event()

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.mem_samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_MEM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self._t.join()

    def result(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": getattr(self, "max_mhz", None), "reasons": sorted(self.reasons),
                    "samples": len(self.samples)}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "mem_mhz": statistics.median(self.mem_samples) if self.mem_samples else None,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------- CPU leg

def cpu_sample(cfg, seconds=10.0, max_reps=100000, workers=None, reps=None, budget=256e6):
    """The oracle (numpy restatement of the reference CPU path) on a bounded
    sample of the workload: every segment whose destination is one of the
    first S dst fabs (S = 1/8 of the fabs, capped so a rep moves <= 256 MB),
    sources allocated as full fabs.  Same per-segment numpy slice copies,
    chunked over a thread pool, as the reference's fused_segments launch.
    Returns (GB/s, description, per-rep seconds, bytes per rep, workers)."""
    from oracle import ghost_oracle as go
    workers = workers or os.cpu_count() or 1
    n, b, nc, ng = cfg["n"], cfg["box"], cfg["ncomp"], cfg["ngrow"]

    def chop(bs):
        return np.asarray([[x, y, z, x + bs - 1, y + bs - 1, z + bs - 1]
                           for z in range(0, n, bs) for y in range(0, n, bs) for x in range(0, n, bs)], np.int64)
    boxes = chop(b)
    if cfg["kind"] == "fb":
        per_fab = ((b + 2 * ng) ** 3 - b ** 3) * nc * 8
        src_boxes, src_grow = boxes, ng
    else:
        per_fab = b ** 3 * nc * 8
        src_boxes, src_grow = chop(cfg["src_box"]), 0
    S = max(1, min(len(boxes) // 8, int(budget // per_fab)))
    t = boxes[:S].copy()
    t[:, :3] -= ng
    t[:, 3:] += ng
    if cfg["kind"] == "fb":
        segs = go.build_segments(t, boxes[:S], src_boxes, [True] * 3, [n] * 3, exclude_valid=True)
    else:
        segs = go.build_segments(t, t, src_boxes, None, [n] * 3, exclude_valid=False)
    plan = go.OraclePlan(segs, np.zeros(len(src_boxes), np.int64), np.zeros(len(boxes), np.int64), 1)
    fabs, lo, dst, dlo = {}, {}, {}, {}
    for si in sorted(set(int(v) for v in segs[:, 0])):
        g = src_boxes[si].copy()
        g[:3] -= src_grow
        g[3:] += src_grow
        fabs[si] = np.full(tuple(g[3:] - g[:3] + 1) + (nc,), 0.5, np.float64, order="F")
        lo[si] = g[:3]
    for dj in range(S):
        if cfg["kind"] == "fb" and dj in fabs:
            dst[dj], dlo[dj] = fabs[dj], lo[dj]
        else:
            dst[dj] = np.full(tuple(t[dj, 3:] - t[dj, :3] + 1) + (nc,), 0.5, np.float64, order="F")
            dlo[dj] = t[dj, :3]
    if cfg["kind"] == "fb":
        for dj in range(S):
            fabs.setdefault(dj, dst[dj])
            lo.setdefault(dj, dlo[dj])
    nbytes = go.ghost_bytes(plan, nc, 8)
    pool = go._Pool(workers)
    try:
        # warm-up: freshly committed pages run several times slower for the first
        # ~second (kernel page housekeeping); settle before timing
        t_w = time.perf_counter() + 2.0
        go.execute(plan, fabs, lo, dst, dlo, 0, 0, nc, pool=pool)
        while time.perf_counter() < t_w:
            go.execute(plan, fabs, lo, dst, dlo, 0, 0, nc, pool=pool)
        times = []
        t_end = time.perf_counter() + seconds
        while (reps is None and time.perf_counter() < t_end and len(times) < max_reps) or \
                (reps is not None and len(times) < reps):
            t0 = time.perf_counter()
            go.execute(plan, fabs, lo, dst, dlo, 0, 0, nc, pool=pool)
            times.append(time.perf_counter() - t0)
    finally:
        pool.close()
    desc = (f"{cfg['desc'].split(':')[0]} sample: the {len(segs)} segments into the first {S} of {len(boxes)} "
            f"dst fabs ({nbytes / 1e6:.2f} MB ghost per rep), numpy slice copies chunked over a {workers}-thread "
            f"pool (reference algorithm, comm.py:316-380 + kernels.py:280-297), {len(times)} reps")
    return nbytes / statistics.median(times) / 1e9, desc, times, nbytes, workers


def import_reference():
    """The reference package (miniamr_core) from ``$MINIAMR_REF`` or
    ``baseline/_ref`` (the offline pip install recorded in DESIGN.md)."""
    for c in (os.environ.get("MINIAMR_REF"), os.path.join(REPO, "baseline", "_ref")):
        if c and os.path.isdir(os.path.join(c, "miniamr_core")):
            if c not in sys.path:
                sys.path.insert(0, c)
            import miniamr_core
            return miniamr_core, c
    return None, None


def _host_ram_bytes():
    try:
        return os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_AVPHYS_PAGES")
    except (ValueError, OSError):
        return None


def reference_bytes(cfg):
    """Host bytes of the reference's MultiFab(s) for cfg."""
    n, nc = cfg["n"], cfg["ncomp"]
    if cfg["kind"] == "pc":
        return 2 * n ** 3 * nc * 8
    b, g = cfg["box"], cfg["ngrow"]
    return (n // b) ** 3 * (b + 2 * g) ** 3 * nc * 8


def reference_run(cfg, G, warmup=1, reps=None, seconds=10.0, max_reps=1000, keep=False):
    """Time the reference's own public call on the full workload.

    Layout: ``decompose(domain, B)`` + ``DistributionMapping.round_robin(n,
    G)``; G ranks as ``runtime_spawn`` threads (reference comm.py:143-180);
    valid cells = the splitmix64 counter hash of oracle/inputs.py (the same
    inputs the GPU arm generates on the device), ghosts = the sNaN poison.
    The first call builds and caches the plan (timed separately, as
    BASELINE.md asks); then ``warmup`` untimed calls, then timed calls
    (perf_counter around the collective call on rank 0, every rank between
    barriers) until ``reps`` calls or ``seconds`` elapsed (>= 5 calls).
    Returns a dict (median seconds per call etc.); with ``keep`` the rank-0
    MultiFab is returned too (parity cross-check)."""
    ref, where = import_reference()
    if ref is None:
        raise RuntimeError("reference package not importable (baseline/_ref missing)")
    from concurrent.futures import ThreadPoolExecutor
    from miniamr_core import comm as rcomm, config as rconfig
    from miniamr_core.index_space import Box as RBox, Geometry as RGeometry
    from miniamr_core.kernels import Backend
    from miniamr_core.mesh import DistributionMapping as RDM, MultiFab as RMF, decompose as rdecompose
    from oracle import inputs
    rconfig.set_spacedim(3)
    rconfig.set_real_dtype(np.float64)
    ext = cfg["ext"]
    dom = RBox((0, 0, 0), tuple(e - 1 for e in ext))
    geom = RGeometry(dom, (0.0,) * 3, (1.0,) * 3, (True,) * 3)
    t0 = time.perf_counter()
    ba = rdecompose(dom, cfg["box"])  # BoxArray ctor incl. the reference's O(n^2) disjointness check
    dm = RDM.round_robin(len(ba), G)
    sba = sdm = None
    if cfg["kind"] == "pc":
        sba = rdecompose(dom, cfg["src_box"])
        sdm = RDM.round_robin(len(sba), G)
    t_ba = time.perf_counter() - t0
    backend = Backend("parallel", os.cpu_count())
    nc, ng = cfg["ncomp"], cfg["ngrow"]
    dlo, dhi = [0, 0, 0], [e - 1 for e in ext]
    fill_pool = ThreadPoolExecutor(max(1, (os.cpu_count() or 1) // max(1, G)))

    def fill(mf, boxes):
        def one(gi):
            f = mf.fabs[gi]
            lo, hi = list(boxes[gi].lo), list(boxes[gi].hi)
            inputs.fill_fab(f.data, list(f.box.lo), lo, hi, dlo, dhi)
        list(fill_pool.map(one, mf.local_indices))

    out, decision = {}, {}

    def program(ctx):
        if cfg["kind"] == "fb":
            dst = RMF(ba, dm, nc, ng, geom)
            fill(dst, ba)
            src = None
        else:
            src = RMF(sba, sdm, nc, 0)
            dst = RMF(ba, dm, nc, 0)
            fill(src, sba)
            for gi in dst.local_indices:  # dst poisoned
                inputs.bits(dst.fabs[gi].data)[...] = inputs.POISON64

        def call():
            if src is None:
                rcomm.fill_boundary(dst, geom, backend=backend)
            else:
                rcomm.parallel_copy(dst, src, backend=backend)
        ctx.barrier()
        tp = time.perf_counter()
        if src is None:
            rcomm.plan_build_fill_boundary(dst, geom)
        call()  # first call: (PC) plan build + execution, pages touched
        ctx.barrier()
        t_first = time.perf_counter() - tp
        for _ in range(warmup):
            call()
        times = []
        t_end = time.perf_counter() + seconds
        while True:
            ctx.barrier()
            a = time.perf_counter()
            call()  # ends with the reference's own barrier
            times.append(time.perf_counter() - a)
            go_on = (len(times) < reps) if reps is not None else \
                (len(times) < 5 or (time.perf_counter() < t_end and len(times) < max_reps))
            # rank 0 decides; every rank follows (collective call)
            if ctx.rank == 0:
                decision["go"] = go_on
            ctx.barrier()
            if not decision["go"]:
                break
        if ctx.rank == 0:
            out.update(times=times, first_call_s=t_first)
            if keep:
                out["mf"] = dst
        ctx.barrier()
        return None

    t1 = time.perf_counter()
    rcomm.runtime_spawn(G, program)
    fill_pool.shutdown()
    t = statistics.median(out["times"])
    res = {"median_s": t, "reps": len(out["times"]), "boxarray_s": round(t_ba, 3),
           "first_call_s": round(out["first_call_s"], 3), "wall_s": round(time.perf_counter() - t1, 1),
           "ranks": G, "workers": backend.nworkers, "where": where}
    if keep:
        res["mf"] = out.get("mf")
    return res


def reference_baseline(cfg, G, ghost_bytes, seconds=10.0, reps=None, warmup=1, keep=False):
    """cpu_baseline dict for the reference on cfg with G simulated ranks;
    falls back to the numpy port (kind "port") when the reference is not
    importable or the workload does not fit the host's free RAM."""
    ref, _ = import_reference()
    ram = _host_ram_bytes()
    need = reference_bytes(cfg)
    why = None
    if ref is None:
        why = "reference package not importable (baseline/_ref missing)"
    elif ram is not None and need > 0.7 * ram:
        why = f"reference MultiFabs need {need / 1e9:.1f} GB, host has {ram / 1e9:.1f} GB free"
    if why is None:
        r = reference_run(cfg, G, warmup=warmup, reps=reps, seconds=seconds, keep=keep)
        d = {"value": round(ghost_bytes / r["median_s"] / 1e9, 4), "unit": "GB/s", "cores": r["workers"],
             "kind": "reference",
             "sample": (f"{cfg['desc']}: the full workload through the reference's public "
                        f"comm.{'fill_boundary' if cfg['kind'] == 'fb' else 'parallel_copy'} (miniamr_core from "
                        f"{os.path.relpath(r['where'], REPO) if r['where'].startswith(REPO) else r['where']}), "
                        f"Backend('parallel', {r['workers']}), {G} runtime_spawn rank(s), same splitmix64 inputs; "
                        f"median of {r['reps']} calls after the plan-building first call"),
             "ms_per_call": round(r["median_s"] * 1e3, 3), "reps": r["reps"], "ranks": G,
             "boxarray_s": r["boxarray_s"], "plan_build_and_first_call_s": r["first_call_s"],
             "cpu_model": cpu_model(), "os_cpu_count": os.cpu_count()}
        if keep:
            d["_mf"] = r.get("mf")
        return d
    gbs, desc, times, nbytes, workers = cpu_sample(cfg, seconds=min(seconds, 5.0))
    return {"value": round(gbs, 4), "unit": "GB/s", "cores": workers, "kind": "port", "sample": desc,
            "fallback_reason": why, "cpu_model": cpu_model(), "os_cpu_count": os.cpu_count()}


def cpu_sample_interp(fine_mf, targets, NCOMP, NGROW, RATIO, seconds=5.0):
    """cpu_baseline leg of bench_amr.py --op fill_patch: the numpy oracle of
    interp_box (reference amr.py:269-314 arithmetic) on the first regions."""
    import paper_2403_12179_b200 as amr
    from oracle import amr_oracle as ao
    rng = np.random.default_rng(1)
    t0 = time.perf_counter()
    done = 0
    jobs = [(gi, r) for gi in sorted(targets) for r in targets[gi]]
    for gi, region in jobs[:64]:
        fb = amr.grow(fine_mf.ba[gi], NGROW)
        cb = amr.grow(amr.coarsen(fb, RATIO), 1)
        crse = rng.random(tuple(cb.extents) + (NCOMP,))
        fine = np.empty(tuple(fb.extents) + (NCOMP,))
        ao.interp(crse, np.asarray(cb.as_row()), fine, np.asarray(fb.as_row()), np.asarray(region.as_row()),
                  [RATIO] * 3, True, 3)
        done += region.num_pts
        if time.perf_counter() - t0 > seconds:
            break
    dt = time.perf_counter() - t0
    return {"value": round(done * NCOMP * 8 / dt / 1e9, 3), "unit": "GB/s (interpolated fine bytes)", "cores": 1,
            "kind": "port", "sample": f"oracle interp (reference amr.py:269-314 arithmetic) on {done} fine cells"}


def cpu_sample_restrict(BOX, NGROW, NCOMP, RATIO, seconds=5.0):
    """cpu_baseline leg of bench_amr.py --op average_down: the numpy oracle of
    the restriction (reference amr.py:251-264) of one fab."""
    from oracle import amr_oracle as ao
    rng = np.random.default_rng(2)
    fine = rng.random((BOX + 2 * NGROW,) * 3 + (NCOMP,))
    fb = np.asarray([-NGROW] * 3 + [BOX + NGROW - 1] * 3)
    vb = np.asarray([0] * 3 + [BOX - 1] * 3)
    t0 = time.perf_counter()
    n = 0
    while time.perf_counter() - t0 < seconds and n < 50:
        ao.restrict(fine, fb, vb, [RATIO] * 3, 3)
        n += 1
    dt = time.perf_counter() - t0
    return {"value": round(n * BOX ** 3 * NCOMP * 8 / dt / 1e9, 3), "unit": "GB/s (fine bytes restricted)",
            "cores": 1, "kind": "port", "sample": f"oracle restriction (amr.py:251-264) of one {BOX}^3 fab x{n}"}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


# ----------------------------------------------------------------- arms

def ghost_bytes_of(cfg):
    """Ghost bytes one step moves (counted once): every ghost cell of the
    fully periodic uniform FillBoundary layouts is coverable, and the C5
    regrid covers every destination cell."""
    nc, n = cfg["ncomp"], cfg["n"]
    if cfg["kind"] == "pc":
        return n ** 3 * nc * 8
    b, g = cfg["box"], cfg["ngrow"]
    return (n // b) ** 3 * ((b + 2 * g) ** 3 - b ** 3) * nc * 8


def run_reference(args, cfg, rank, world):
    """--impl reference: the reference's own CPU implementation (miniamr_core
    from baseline/_ref) on the host cores, rank 0 only, G = N simulated ranks
    as threads; every step is one full public call (bounded: W warm-up + K
    timed calls)."""
    if rank != 0:
        return
    W, K = args.warmup, args.steps
    gb = ghost_bytes_of(cfg)
    cb = reference_baseline(cfg, world, gb, reps=K, warmup=W)
    value = cb["value"]
    ms = cb.get("ms_per_call") or round(gb / (value * 1e9) * 1e3, 4)
    line = {
        "metric": METRIC, "impl": "reference", "value": value, "unit": "GB/s",
        "n_gpus": args.gpus, "steps": cb.get("reps", K), "warmup": W, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (splitmix64 counter-hash valid cells, sNaN-poisoned ghosts)",
        "config": {"workload": cfg["desc"], "domain": list(cfg["ext"]), "box": cfg["box"], "ncomp": cfg["ncomp"],
                   "nghost": cfg["ngrow"], "ghost_bytes_per_step": gb,
                   "parallelism": f"boxes round-robin over {world} simulated rank(s) (runtime_spawn threads)"},
        "cpu_baseline": cb,
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, cfg, rank, world):
    import torch
    import paper_2403_12179_b200 as amr
    from paper_2403_12179_b200 import _native as N
    dev = torch.cuda.current_device()
    dist = torch.distributed if world > 1 else None
    L = layout(amr, cfg, world)
    t0 = time.perf_counter()
    mf, src = make_fields(amr, cfg, L)
    torch.cuda.synchronize()
    t_alloc = time.perf_counter() - t0
    plan, x, t_plan, t_exec = prepare(amr, cfg, L, mf, src)
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        public_call(amr, cfg, L, mf, src)
    torch.cuda.synchronize()
    # device-timed region
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    # write_read: after the 512 MiB write, read a clean 256 MiB buffer so the
    # flush's dirty lines are written back before the timed region instead of
    # inside it (the kernel then starts from a cold, clean L2, like ncu's
    # --cache-control all)
    clean = torch.ones(64 << 20, dtype=torch.int32, device=dev) if args.l2 == "write_read" else None
    K = args.steps
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = N.lib.ghx_launch_count()
    can_enqueue = x.mode == "serial" or x.transport == "nccl" or x.sync == "device"
    with ClockSampler(dev) as clk:
        for i in range(K):
            flush.zero_()
            if clean is not None:
                torch.sum(clean)
            ev0[i].record(stream)
            if can_enqueue:
                x.enqueue(stream.cuda_stream)
            else:  # ranks sharing one GPU: host-synchronised exchange
                x.run()
            ev1[i].record(stream)
        torch.cuda.synchronize()
    launches = N.lib.ghx_launch_count() - l0  # the timed region only (not the diagnostic steps below)
    if x.mode == "process" and x.sync == "device":
        from paper_2403_12179_b200 import comm as _comm
        _comm.check_barriers()
    breakdown = None
    if world > 1 and getattr(x, "fused", False) and os.environ.get("GHX_BENCH_BREAKDOWN", "1") != "0":
        # diagnostic steps (outside the timed region): this rank's push kernel
        # (incl. its READY waits) and the unpack / DONE wait, each timed on
        # the device; the max over ranks is reported
        push, tail = [], []
        for _ in range(max(3, min(K, 10))):
            flush.zero_()
            dist.barrier()
            m = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            x.enqueue(stream.cuda_stream, marks=[lambda e=e: e.record(stream) for e in m])
            torch.cuda.synchronize()
            try:  # never let a diagnostic raise on one rank only (the peers would wait in a collective)
                push.append(m[0].elapsed_time(m[1]))
                tail.append(m[1].elapsed_time(m[2]))
            except RuntimeError:
                push.append(float("nan"))
                tail.append(float("nan"))
        _comm.check_barriers()
        v = torch.tensor([statistics.median(push), statistics.median(tail)], dtype=torch.float64, device=dev)
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        breakdown = {"push_kernel_ms": round(float(v[0]), 5), "unpack_or_wait_ms": round(float(v[1]), 5),
                     "remote": x.remote, "one_kernel": bool(getattr(x, "one_kernel", False)),
                     "note": "median per rank, max over ranks; push includes the READY waits"
                             + ("; one kernel: push_kernel_ms is the whole exchange (pushes, local tags and "
                                "unpacks in one launch)" if getattr(x, "one_kernel", False) else "")}
    if dist:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in zip(ev0, ev1)]
    mean_ms = sum(step_ms) / K
    if dist:
        t = torch.tensor([mean_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        mean_ms_max = float(t.item())
    else:
        mean_ms_max = mean_ms
    ghost_bytes = x.ghost_bytes
    value = ghost_bytes / (mean_ms_max * 1e-3) / 1e9
    # correctness spot check (outside the timed region)
    verified = None
    if cfg["kind"] == "fb" and mf.local_indices:
        import ctypes as C
        f = mf.fabs[mf.local_indices[0]]
        flat = f.raw().view(torch.int64)
        exp = torch.empty_like(flat)
        N.check(N.lib.ghx_fill_hash_wrapped(
            C.c_void_p(exp.data_ptr()), N.i64p(np.asarray(f.box.as_row(), np.int64)), mf.ncomp,
            N.i64p(np.asarray(L["dom"].as_row(), np.int64)), N.i32p(np.ones(3, np.int32)),
            C.c_uint64(SEED), 8, None))
        verified = bool(torch.equal(flat, exp))
    hbm_peak, peak_src = peaks()
    # context only: this box's device-to-device copy rate right now (2 GiB,
    # best of 3); the roofline denominator stays MEASURED_PEAKS.json
    big = torch.empty(1 << 30, dtype=torch.int16, device=dev)
    big2 = torch.empty_like(big)
    best = 0.0
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        big2.copy_(big)
        e1.record()
        e1.synchronize()
        best = max(best, 2 * big.numel() * 2 / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    del big, big2
    alg = x.ex.alg_bytes if x.transport == "p2p" else None
    split = None
    if world == 1 and cfg["kind"] == "fb" and isinstance(cfg["ngrow"], int) and not args.no_split:
        split = direction_split(amr, cfg, L, stream, flush, clean, mean_ms, mf=mf)
    roof = None
    if alg is not None:
        achieved = alg / (mean_ms * 1e-3) / 1e9
        hbm = {"bound": "hbm", "achieved": round(achieved, 2), "peak": hbm_peak, "unit": "GB/s",
               "frac": round(achieved / hbm_peak, 4),
               "traffic": ncu_traffic(args.config) if world == 1 else None,
               "traffic_model_min": traffic_model_min(cfg) if world == 1 else None,
               "kernel": "ghx_copy_kernel", "algorithmic_bytes_per_launch": int(alg),
               "peak_source": peak_src, "box_copy_gbs_now": round(best, 1)}
        tmin = hbm["traffic_model_min"]
        if tmin:
            # the floor of this layout: the modelled minimum DRAM bytes at the
            # measured copy rate
            floor_ms = tmin / (hbm_peak * 1e9) * 1e3
            hbm["modelled_floor_ms"] = round(floor_ms, 5)
            hbm["frac_of_modelled_floor"] = round(floor_ms / mean_ms, 4)
        if split is not None:
            hbm["direction_split"] = split
        roof = hbm
        if world > 1:
            pc = x.plan.pair_cells.astype(np.float64) * x.ncomp * x.item
            off = pc - np.diag(np.diag(pc))
            send, recv = off.sum(axis=1), off.sum(axis=0)
            per_gpu = np.maximum(send, recv)
            nv_bytes = float(per_gpu.max())
            local_alg = 2.0 * float(np.diag(pc).max())  # busiest GPU's local HBM bytes (read + write)
            t = mean_ms_max * 1e-3
            nv = {"bound": "nvlink", "achieved": round(nv_bytes / t / 1e9, 2), "peak": NVLINK_PEER_GBS,
                  "unit": "GB/s", "frac": round(nv_bytes / t / 1e9 / NVLINK_PEER_GBS, 4), "traffic": None,
                  "bytes_per_gpu_max_send_recv": int(nv_bytes),
                  "send_bytes_this_rank": int(send[rank]), "recv_bytes_this_rank": int(recv[rank]),
                  "peak_source": "measured peer copy per direction (B200_PROFILING.md); nominal 900 GB/s",
                  "frac_of_nominal_900": round(nv_bytes / t / 1e9 / 900.0, 4),
                  "kernel": "ghx_copy_kernel", "launches_per_step": x.launches_per_call}
            hbm_only = {"achieved": round(local_alg / t / 1e9, 2), "peak": hbm_peak,
                        "frac": round(local_alg / t / 1e9 / hbm_peak, 4),
                        "algorithmic_bytes_busiest_gpu": int(local_alg)}
            # the roofline is the term that bounds the step: NVLink when the
            # busiest GPU's remote bytes need longer at 770 GB/s than its local
            # bytes at the HBM copy rate
            if nv_bytes / NVLINK_PEER_GBS >= local_alg / hbm_peak:
                nv["hbm"] = hbm_only
                roof = nv
            else:
                hbm.update({"achieved": hbm_only["achieved"], "frac": hbm_only["frac"],
                            "algorithmic_bytes_per_launch": int(local_alg)})
                hbm["nvlink"] = {k: nv[k] for k in ("achieved", "peak", "frac", "bytes_per_gpu_max_send_recv")}
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": round(mean_ms_max, 5), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (splitmix64 counter-hash valid cells, sNaN-poisoned ghosts)",
        "config": {"workload": cfg["desc"], "domain": list(cfg["ext"]), "box": cfg["box"], "ncomp": cfg["ncomp"],
                   "nghost": cfg["ngrow"], "boxes": len(L["ba"]), "segments": plan.num_segments,
                   "ghost_bytes_per_step": ghost_bytes, "parallelism": f"boxes round-robin over {world} GPU(s)",
                   "transport": x.transport if world > 1 else "local",
                   "sync": x.sync if world > 1 else None,
                   "remote": x.remote if world > 1 else None,
                   "l2": ("flushed before every step (512 MiB write, then a 256 MiB clean read so no dirty "
                          "flush lines are written back inside the timed region; outside the events)"
                          if args.l2 == "write_read" else
                          "flushed before every step (512 MiB write, outside the events)"),
                   "tags_this_rank": x.ex.ntags if x.transport == "p2p" else None,
                   "warp_tasks_this_rank": x.ex.ntasks if x.transport == "p2p" else None,
                   "exec": x.ex.detail if x.transport == "p2p" else None},
        "roofline": roof, "gpu_launches": int(launches), "clocks": clk.result(),
        "boxarray_s": round(L["boxarray_s"], 4), "plan_build_s": round(t_plan, 4), "exec_compile_s": round(t_exec, 4), "alloc_fill_s": round(t_alloc, 3),
        "verified": verified,
        "step_ms_min": round(min(step_ms), 5), "step_ms_median": round(statistics.median(step_ms), 5),
    }
    if breakdown is not None:
        line["multi_gpu_breakdown"] = breakdown
    # e2e through the public API on host-resident fabs
    if not args.no_e2e:
        line["e2e"] = e2e_leg(args, amr, cfg, L, world, ghost_bytes, x)
        if world == 1 and cfg["kind"] == "fb" and not os.environ.get("GHX_BENCH_NO_BINDING"):
            try:
                line["e2e"]["reference_binding"] = e2e_binding_leg(cfg, L, mf, ghost_bytes,
                                                                   max(1, min(args.e2e_steps, args.steps)))
            except Exception as e:  # noqa: BLE001 - report, do not lose the GPU line
                line["e2e"]["reference_binding"] = {"error": repr(e)[:300]}
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cb = reference_baseline(cfg, 1, ghost_bytes, seconds=args.cpu_seconds, keep=True)
        except Exception as e:  # noqa: BLE001 - report, do not lose the GPU line
            cb = {"value": None, "kind": "reference", "error": repr(e)[:300]}
        rmf = cb.pop("_mf", None)
        if rmf is not None and cfg["kind"] == "fb":
            # full-size parity cross-check against the reference's own result
            import torch
            gi = mf.local_indices[0]
            ours = mf.fabs[gi].raw().view(torch.int64).cpu().numpy()
            theirs = np.ascontiguousarray(rmf.fabs[gi].data.reshape(-1, order="F")).view(np.int64)
            cb["bit_exact_vs_ours_fab0"] = bool(np.array_equal(ours, theirs))
        del rmf
        if not args.no_port:
            gbs, desc, _, _, workers = cpu_sample(cfg, seconds=3.0)
            cb["port"] = {"value": round(gbs, 4), "unit": "GB/s", "cores": workers, "sample": desc}
        line["cpu_baseline"] = cb
    del mf, src
    if rank == 0:
        print(json.dumps(line), flush=True)


def direction_split(amr, cfg, L, stream, flush, clean, all_ms, reps=20, mf=None):
    """The same FillBoundary split by direction, measured in this run: the
    x faces alone (ngrow (g,0,0): the same x-row seams at the same row
    pitch) and the y/z faces alone (ngrow (0,g,g)), each device-timed like
    the headline.  x_only + yz_only is the additive floor the fused kernel
    is compared with: the x-row seams cost one DRAM
    line read + one line write each whatever their size, and they compete
    with the face rows for the same DRAM service."""
    import torch
    from paper_2403_12179_b200 import comm
    g = cfg["ngrow"]
    out = {}
    for name, ng in (("x_only", (g, 0, 0)), ("yz_only", (0, g, g))):
        sm = amr.MultiFab(L["ba"], L["dm"], cfg["ncomp"], amr.IntVect(*ng), L["geom"])
        sm.fill_hash(SEED, L["dom"])
        xx = comm.exchange_for(comm.plan_build_fill_boundary(sm, L["geom"]), sm, sm, 0, 0, sm.ncomp)
        for _ in range(3):
            xx.enqueue(stream.cuda_stream)
        ts = []
        for _ in range(reps):
            flush.zero_()
            if clean is not None:
                torch.sum(clean)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            xx.enqueue(stream.cuda_stream)
            e1.record(stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        out[name + "_ms"] = round(sum(ts) / len(ts), 5)
        if name == "x_only":
            rows = sum(int((b.hi[1] - b.lo[1] + 1) * (b.hi[2] - b.lo[2] + 1)) for b in L["ba"]) * cfg["ncomp"]
            out["x_row_seams"] = rows
            out["x_gseam_per_s"] = round(rows / (out["x_only_ms"] * 1e-3) / 1e9, 2)
        del xx, sm
        torch.cuda.synchronize()
    add = out["x_only_ms"] + out["yz_only_ms"]
    out["additive_floor_ms"] = round(add, 5)
    out["all_ms"] = round(all_ms, 5)
    out["frac_of_additive_floor"] = round(add / all_ms, 4)
    # the same split on the headline MultiFab's own layout: its x-face tags
    # alone and every other tag alone (GHX_EXEC_ONLY_XFACES / NO_XFACES)
    if mf is not None:
        from paper_2403_12179_b200 import _native as N
        plan = comm.plan_build_fill_boundary(mf, L["geom"])
        rows = mf.storage_rows()
        for name, flag in (("x_faces_same_layout_ms", N.EXEC_ONLY_XFACES), ("rest_same_layout_ms", N.EXEC_NO_XFACES)):
            ex = comm.Executor(plan, 0, N.EXEC_DIRECT | flag, rows, mf.ncomp, rows, mf.ncomp, 0, 0, mf.ncomp,
                               mf.dtype.itemsize, mf.device)
            b = ex.bind(comm._table(ex, mf, [(mf.local_indices, mf._ptrs)]), stream.cuda_stream)
            for _ in range(3):
                b.run(stream.cuda_stream)
            ts = []
            for _ in range(reps):
                flush.zero_()
                if clean is not None:
                    torch.sum(clean)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                b.run(stream.cuda_stream)
                e1.record(stream)
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            out[name] = round(sum(ts) / len(ts), 5)
            del b, ex
        same = out["x_faces_same_layout_ms"] + out["rest_same_layout_ms"]
        out["additive_floor_same_layout_ms"] = round(same, 5)
        out["frac_of_additive_floor_same_layout"] = round(same / all_ms, 4)
    return out


def x_host_detail(cfg, L, hmf, hsrc):
    """Task mix of the host-memory executor the public call used."""
    from paper_2403_12179_b200 import comm
    try:
        if cfg["kind"] == "fb":
            xx = comm.prepare_fill_boundary(hmf, L["geom"])
        else:
            xx = comm.prepare_parallel_copy(hmf, hsrc)
        d = xx.ex.detail
        return {k: d.get(k) for k in ("tags", "tasks", "ring_tasks", "copy_tasks", "phased", "blocks")}
    except Exception as e:  # noqa: BLE001 - diagnostic only
        return {"error": repr(e)[:120]}


def e2e_leg(args, amr, cfg, L, world, ghost_bytes, x):
    """The public call on MultiFabs in pinned host memory (zero-copy: the
    exchange kernels read source cells and write ghost cells across PCIe).
    At N > 1 each rank's fabs live in its own pinned memory; remote tags
    travel packed (pack kernel -> device buffers -> message -> unpack)."""
    import torch
    steps = max(1, min(args.e2e_steps, args.steps))
    dist = torch.distributed if world > 1 else None
    hmf, hsrc = make_fields(amr, cfg, L, memory="pinned")
    torch.cuda.synchronize()
    public_call(amr, cfg, L, hmf, hsrc)  # plan + compile (cached) + warm
    ts = []
    for _ in range(steps):
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        public_call(amr, cfg, L, hmf, hsrc)  # synchronous: returns with the host fabs updated
        dt = time.perf_counter() - t0
        if dist:
            tt = torch.tensor([dt], dtype=torch.float64, device=torch.cuda.current_device())
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dt = float(tt.item())
        ts.append(dt)
    t = statistics.median(ts)
    moved = x.ghost_bytes
    verified = None
    if cfg["kind"] == "fb" and hmf.local_indices:  # every host-resident fab, checked like the device one
        import ctypes as C
        from paper_2403_12179_b200 import _native as N
        verified = True
        for gi in hmf.local_indices:
            f = hmf.fabs[gi]
            exp = torch.empty(f.raw().numel(), dtype=torch.int64, device="cuda")
            N.check(N.lib.ghx_fill_hash_wrapped(
                C.c_void_p(exp.data_ptr()), N.i64p(np.asarray(f.box.as_row(), np.int64)), hmf.ncomp,
                N.i64p(np.asarray(L["dom"].as_row(), np.int64)), N.i32p(np.ones(3, np.int32)),
                C.c_uint64(SEED), 8, None))
            verified = verified and bool(torch.equal(f.raw().view(torch.int64).to("cuda"), exp))
            del exp
    if dist:
        v = torch.tensor([0 if verified is False else 1], dtype=torch.int32, device=torch.cuda.current_device())
        dist.all_reduce(v, op=dist.ReduceOp.MIN)
        verified = bool(v.item()) if verified is not None else None
    path = ("public fill_boundary/parallel_copy on pinned host MultiFabs: the fused kernel reads source cells "
            "and writes ghost cells across PCIe (zero-copy, mapped memory; x seams as tile-ring chunks, one "
            "64-B read + write each; FillBoundary phased: faces extended over the lower-axis ghosts, no "
            "edge/corner requests); every fab verified")
    if world > 1:
        path += ("; remote tags packed by the sender's kernel (reading its host fabs) into the peer's CUDA-IPC "
                 "mapped device receive slab over NVLink, unpacked by the receiver into its host fabs")
    return {"value": round(ghost_bytes / t / 1e9, 3), "unit": "GB/s", "h2d_bytes_per_step": int(moved),
            "d2h_bytes_per_step": int(moved), "ms_per_step": round(t * 1e3, 3), "steps": steps,
            "verified": verified, "path": path, "exec": x_host_detail(cfg, L, hmf, hsrc)}


def e2e_binding_leg(cfg, L, mf, ghost_bytes, steps):
    """The same exchange through the reference-facing C ABI: the REFERENCE's
    own MultiFab (miniamr_core from baseline/_ref) with its numpy fabs in
    pinned, mapped memory (integration/reference_binding.PinnedArena), and
    integration/reference_binding.fill_boundary_native -- ctypes and
    libghostx.so only, no torch and none of this package's Python layer on
    the call path.  Every fab is compared with the device run's result."""
    ref, where = import_reference()
    if ref is None:
        return {"unavailable": "reference package not importable (baseline/_ref missing)"}
    need, ram = reference_bytes(cfg), _host_ram_bytes()
    if ram is not None and need > 0.6 * ram:
        return {"unavailable": f"needs {need / 1e9:.1f} GB pinned host memory, {ram / 1e9:.1f} GB free"}
    from concurrent.futures import ThreadPoolExecutor
    from miniamr_core import config as rconfig
    from miniamr_core.index_space import Box as RBox, Geometry as RGeometry
    from miniamr_core.mesh import DistributionMapping as RDM, MultiFab as RMF, decompose as rdecompose
    from integration.reference_binding import PinnedArena, fill_boundary_native
    from oracle import inputs
    import torch
    rconfig.set_spacedim(3)
    rconfig.set_real_dtype(np.float64)
    ext = cfg["ext"]
    dom = RBox((0, 0, 0), tuple(e - 1 for e in ext))
    geom = RGeometry(dom, (0.0,) * 3, (1.0,) * 3, (True,) * 3)
    ba = rdecompose(dom, cfg["box"])
    rmf = RMF(ba, RDM.round_robin(len(ba), 1), cfg["ncomp"], cfg["ngrow"], geom, arena=PinnedArena())
    dlo, dhi = [0, 0, 0], [e - 1 for e in ext]

    def one(gi):
        f = rmf.fabs[gi]
        inputs.fill_fab(f.data, list(f.box.lo), list(ba[gi].lo), list(ba[gi].hi), dlo, dhi)
    with ThreadPoolExecutor(os.cpu_count() or 1) as pool:
        list(pool.map(one, rmf.local_indices))
    t0 = time.perf_counter()
    fill_boundary_native(rmf, geom)  # plan + executor (cached on the MultiFab) + first exchange
    first = time.perf_counter() - t0
    ts = []
    for _ in range(steps):
        a = time.perf_counter()
        fill_boundary_native(rmf, geom)
        ts.append(time.perf_counter() - a)
    t = statistics.median(ts)
    ok = True
    for gi in rmf.local_indices:
        ours = mf.fabs[gi].raw().view(torch.int64).cpu().numpy()
        theirs = rmf.fabs[gi].data.reshape(-1, order="F").view(np.int64)
        ok = ok and bool(np.array_equal(ours, theirs))
    return {"value": round(ghost_bytes / t / 1e9, 3), "unit": "GB/s", "ms_per_step": round(t * 1e3, 3),
            "steps": steps, "first_call_s": round(first, 3), "verified": ok,
            "path": "integration/reference_binding.fill_boundary_native on the reference's own MultiFab "
                    "(miniamr_core, numpy fabs in pinned mapped memory via PinnedArena): ctypes -> libghostx.so "
                    "(phased exchange, tile-ring seams, 6-CTA grid), every fab equal to the device run's"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C3", choices=sorted(CONFIGS),
                    help="default C3 = BASELINE.json configs[2] (the north-star config), same global size at every N")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--transport", default=None, choices=["p2p", "nccl"])
    ap.add_argument("--l2", default="write_read", choices=["write", "write_read"],
                    help="L2 flush between timed steps (both outside the events)")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-split", action="store_true", help="skip the x / y-z direction split (N=1)")
    ap.add_argument("--no-port", action="store_true", help="skip the numpy-port sample next to the reference")
    ap.add_argument("--ngrow", default=None, help="diagnostic: override ghost width per axis, e.g. 2,0,0")
    args = ap.parse_args()
    if os.environ.get("GHX_DEBUG_HANG_S"):  # diagnostics: dump every thread's stack if the run hangs
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["GHX_DEBUG_HANG_S"]), exit=True)
    if args.warmup < 3:
        log("[bench] warm-up raised to 3 (timing rules)")
        args.warmup = 3
    if args.transport:
        os.environ["GHX_TRANSPORT"] = args.transport
    world = int(os.environ.get("WORLD_SIZE", "1"))
    cfg = scaled(CONFIGS[args.config], world)
    if args.ngrow:
        g = tuple(int(v) for v in args.ngrow.split(","))
        cfg["ngrow"] = g if len(g) == 3 else g[0]
        cfg["desc"] += f" [diagnostic ngrow={args.ngrow}]"
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return
    import torch
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local % max(1, torch.cuda.device_count()))
    if world > 1:
        backend = os.environ.get("GHX_BENCH_BACKEND", "nccl")  # gloo: ranks sharing one GPU (tests)
        if backend == "nccl":
            torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
        else:
            torch.distributed.init_process_group(backend)
    try:
        run_ours(args, cfg, rank, world)
    except BaseException:
        if world > 1:
            # never wait for the peers after a failure (they may sit in a
            # collective or a device wait): report and leave, torchrun then
            # tears the job down instead of hanging it
            import traceback
            traceback.print_exc()
            sys.stderr.flush()
            os._exit(1)
        raise
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
