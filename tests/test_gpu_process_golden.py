"""The reference-generated 2-rank FillBoundary golden cases (irregular
decompositions, 1-3-D, mixed periodicity, float32, nodal, several calls)
run across two PROCESSES sharing the GPU -- CUDA-IPC push with packed and
direct remote rows, host sync and the in-kernel READY/DONE protocol -- and
every rank's fabs must equal the reference's bits and message counts."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import golden_util as gu

pytestmark = pytest.mark.gpu

CASES = [n for n in gu.names("fill_boundary", store="bits") if gu.case(n)["nranks"] == 2]
if os.environ.get("GHX_TEST_CASES"):
    CASES = [n for n in CASES if n in os.environ["GHX_TEST_CASES"].split(",")]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, port, q, names, env):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE="2",
                          LOCAL_RANK="0")
        os.environ.update(env)
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=2)
        import paper_2403_12179_b200 as amr
        from gpu_util import bits_of
        from oracle import inputs
        d = gu.data()
        out = {}
        for name in names:
            c = gu.case(name)
            dim = c["dim"]
            amr.config.set_spacedim(dim)
            amr.config.set_real_dtype(np.dtype(c["dtype"]))
            ixt = amr.IndexType.node() if c["nodal"] else amr.IndexType.cell()
            ba = amr.BoxArray([amr.Box(r[:dim], r[3:3 + dim], ixt) for r in c["boxes"]])
            dm = amr.DistributionMapping(c["rank_of"], c["nranks"])
            dom = amr.Box(c["domain"][0][:dim], c["domain"][1][:dim])
            geom = amr.Geometry(dom, [0.0] * dim, [1.0] * dim, c["periodic"][:dim])
            mf = amr.MultiFab(ba, dm, c["ncomp"], amr.IntVect(*c["ngrow"][:dim]), geom)
            mf.fill_hash(inputs.SEED, list(c["hash_domain"][0]) + list(c["hash_domain"][1]))
            torch.cuda.synchronize()
            ctx = amr.current_ctx()
            s0 = ctx.bus.stats_snapshot()
            for _ in range(c["calls"]):
                amr.fill_boundary(mf, geom)
            s1 = ctx.bus.stats_snapshot()
            bad = []
            for gi in mf.local_indices:
                got, exp = bits_of(mf.fabs[gi]), d[f"{name}/fab{gi}"].ravel(order="F")
                if not np.array_equal(got, exp):
                    w = np.flatnonzero(got != exp)
                    bad.append((gi, int(w.size), int(got.size), [hex(int(v)) for v in got[w[:3]]],
                                [hex(int(v)) for v in exp[w[:3]]]) if os.environ.get("GHX_TEST_VERBOSE") else gi)
            sent = {k: (s1[k][0] - s0[k][0], s1[k][1] - s0[k][1]) for k in s1 if s1[k] != s0[k] and k[0] == rank}
            out[name] = (bad, sent)
            del mf
        amr.config.set_real_dtype(np.dtype("f8"))
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, out))
    except BaseException:  # noqa: BLE001
        import traceback
        q.put((rank, "ERROR " + traceback.format_exc()))


@pytest.mark.parametrize("env", [{}, {"GHX_SYNC": "device", "GHX_BARRIER_TIMEOUT_S": "20"},
                                 {"GHX_SYNC": "device", "GHX_BARRIER_TIMEOUT_S": "20", "GHX_REMOTE": "direct"},
                                 {"GHX_TRANSPORT": "nccl"},
                                 {"GHX_SYNC": "device", "GHX_BARRIER_TIMEOUT_S": "20", "GHX_ONE_KERNEL": "0"}],
                         ids=["host-sync-packed", "devsync-packed", "devsync-direct", "fallback", "devsync-two-kernels"])
def test_two_process_golden_fill_boundary(env):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q, CASES, env)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=900) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
    d = gu.data()
    errs = [res[r] for r in range(2) if isinstance(res[r], str)]
    assert not errs, "\n".join(e[-1500:] for e in errs)
    for name in CASES:
        assert res[0][name][0] == [] and res[1][name][0] == [], (name, res[0][name][0], res[1][name][0])
        if "stats" in gu.case(name) or f"{name}/stats" in d:
            exp = gu.stats_dict(d[f"{name}/stats"])
            got = {}
            for r in range(2):
                got.update(res[r][name][1])
            exp_sent = {k: v for k, v in exp.items() if k[0] != k[1]}
            assert got == exp_sent, (name, got, exp_sent)


PC_CASES = [n for n in gu.names("parallel_copy") if gu.case(n)["nranks"] == 2]


def _pc_worker(rank, port, q, names, env):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE="2",
                          LOCAL_RANK="0")
        os.environ.update(env)
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=2)
        import paper_2403_12179_b200 as amr
        from gpu_util import bits_of, upload
        from oracle import inputs
        d = gu.data()
        out = {}
        for name in names:
            c = gu.case(name)
            dim = c["dim"]
            dt = np.dtype(c["dtype"])
            amr.config.set_spacedim(dim)
            amr.config.set_real_dtype(dt)
            ixt = amr.IndexType.node() if c["nodal"] else amr.IndexType.cell()
            sba = amr.BoxArray([amr.Box(r[:dim], r[3:3 + dim], ixt) for r in c["src_boxes"]])
            dba = amr.BoxArray([amr.Box(r[:dim], r[3:3 + dim], ixt) for r in c["dst_boxes"]])
            sdm = amr.DistributionMapping(c["src_rank"], 2)
            ddm = amr.DistributionMapping(c["dst_rank"], 2)
            geom = None
            if c["periodic"] is not None:
                dom = amr.Box(c["domain"][0][:dim], c["domain"][1][:dim])
                geom = amr.Geometry(dom, [0.0] * dim, [1.0] * dim, c["periodic"][:dim])
            hd = c["hash_domain"]
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
            torch.cuda.synchronize()
            dist.barrier()
            amr.parallel_copy(dst, src, scomp=c["scomp"], dcomp=c["dcomp"], ncomp=c["ncomp"],
                              ngrow_src=amr.IntVect(*c["ngrow_src"][:dim]),
                              ngrow_dst=amr.IntVect(*c["ngrow_dst"][:dim]), geom=geom)
            out[name] = [gi for gi in dst.local_indices
                         if not np.array_equal(bits_of(dst.fabs[gi]), d[f"{name}/fab{gi}"].ravel(order="F"))]
            del src, dst
        amr.config.set_real_dtype(np.dtype("f8"))
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, out))
    except BaseException:  # noqa: BLE001
        import traceback
        q.put((rank, "ERROR " + traceback.format_exc()))


@pytest.mark.parametrize("env", [{}, {"GHX_SYNC": "device", "GHX_BARRIER_TIMEOUT_S": "20"},
                                 {"GHX_SYNC": "device", "GHX_BARRIER_TIMEOUT_S": "20", "GHX_REMOTE": "direct"},
                                 {"GHX_TRANSPORT": "nccl"}],
                         ids=["host-sync-packed", "devsync-packed", "devsync-direct", "fallback"])
def test_two_process_golden_parallel_copy(env):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pc_worker, args=(r, port, q, PC_CASES, env)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=900) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
    errs = [res[r] for r in range(2) if isinstance(res[r], str)]
    assert not errs, "\n".join(e[-1500:] for e in errs)
    for name in PC_CASES:
        assert res[0][name] == [] and res[1][name] == [], (name, res[0][name], res[1][name])
