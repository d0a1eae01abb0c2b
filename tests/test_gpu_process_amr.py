"""Level transfers in process-per-GPU mode: two processes (gloo plumbing)
share cuda:0 and run the 2-rank reference fixtures of fill_patch,
average_down and the heat loop (tests/golden/make_golden_amr.py) through the
public API -- gathers and ParallelCopies cross processes via CUDA IPC.
Raw bits compared with the reference."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from test_amr_oracle import case, data, names

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _g3(v, dim):
    return [v if d < dim else 0 for d in range(3)]


def _worker(rank, world, port, q, name, env=None):
    try:
        os.environ.update(env or {})
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                          LOCAL_RANK="0")
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2403_12179_b200 as amr
        from paper_2403_12179_b200 import amr as A
        from paper_2403_12179_b200 import heat as H
        from gpu_util import bits_of, upload
        from oracle import inputs
        from test_amr_oracle import grown, hashed, meta
        c = case(name)
        dim, dt, r = c["dim"], np.dtype(c["dtype"]), c.get("ratio", 1)
        amr.config.set_spacedim(dim)
        amr.config.set_real_dtype(dt)
        box = lambda b6: amr.Box(tuple(b6[:dim]), tuple(b6[3:3 + dim]))  # noqa: E731
        if c["kind"] != "index_copy":
            cdom6 = [0, 0, 0] + [e - 1 for e in c["cext"]]
            fdom6 = [0, 0, 0] + [e * (r if d < dim else 1) - 1 for d, e in enumerate(c["cext"])]
            per = tuple(bool(p) for p in c.get("periodic", [True] * 3)[:dim])
            cgeom = amr.Geometry(box(cdom6), (0.0,) * dim, (1.0,) * dim, per)
            fgeom = cgeom.refined(r)
            cba = amr.BoxArray([box(b) for b in c["crse_boxes"]])
            cdm = amr.DistributionMapping(c["crse_rank"], c["nranks"])
        out = {}
        if c["kind"] == "index_copy":
            from test_index_copy import MAPPINGS, _inputs
            sba = amr.BoxArray([box(b) for b in c["src_boxes"]])
            dba = amr.BoxArray([box(b) for b in c["dst_boxes"]])
            src = amr.MultiFab(sba, amr.DistributionMapping(c["src_rank"], c["nranks"]), c["ncomp"], c["sng"])
            dst = amr.MultiFab(dba, amr.DistributionMapping(c["dst_rank"], c["nranks"]), c["ncomp"], c["dng"])
            hsrc, hdst = _inputs(c)
            for gi in src.local_indices:
                upload(src.fabs[gi], hsrc[gi])
            for gi in dst.local_indices:
                upload(dst.fabs[gi], hdst[gi])
            dist.barrier()
            region = None if c["region"] is None else amr.Box(tuple(c["region"][0][:dim]), tuple(c["region"][1][:dim]))
            amr.index_mapped_copy(dst, src, MAPPINGS[c["mapping"]](c["ext"]), region=region)
            out = {f"dst{gi}": bits_of(dst.fabs[gi]) for gi in dst.local_indices}
        elif c["kind"] == "heat":
            specs = [(cba, cdm)]
            if c["fine_boxes"]:
                specs.append((amr.BoxArray([box(b) for b in c["fine_boxes"]]),
                              amr.DistributionMapping(c["fine_rank"], c["nranks"])))
            geoms = [cgeom, fgeom]
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
            dist.barrier()
            for _ in range(c["steps"]):
                levels = H.heat_step(levels, geoms, c["dt"], c["diffusivity"], r)
            for lv, (u, w) in enumerate(levels):
                for gi in u.local_indices:
                    out[f"l{lv}u{gi}"] = bits_of(u.fabs[gi])
                    out[f"l{lv}w{gi}"] = bits_of(w.fabs[gi])
        else:
            nc = c["ncomp"]
            fba = amr.BoxArray([box(b) for b in c["fine_boxes"]])
            fdm = amr.DistributionMapping(c["fine_rank"], c["nranks"])
            cng = c.get("cngrow", 0)
            coarse = amr.MultiFab(cba, cdm, nc, cng, cgeom)
            fine = amr.MultiFab(fba, fdm, nc, c["fngrow"], fgeom)
            for gi in coarse.local_indices:
                vb = np.asarray(c["crse_boxes"][gi])
                upload(coarse.fabs[gi], hashed(grown(vb, _g3(cng, dim)), vb, np.asarray(cdom6), nc, dt,
                                               meta()["seed_crse"]))
            for gi in fine.local_indices:
                vb = np.asarray(c["fine_boxes"][gi])
                upload(fine.fabs[gi], hashed(grown(vb, _g3(c["fngrow"], dim)), vb, np.asarray(fdom6), nc, dt,
                                             meta()["seed_fine"]))
            dist.barrier()
            if c["kind"] == "fill_patch":
                A.fill_patch(fine, coarse, fgeom, cgeom, r, c["scheme"])
                A.fill_patch(fine, coarse, fgeom, cgeom, r, c["scheme"])
                out = {f"fine{gi}": bits_of(fine.fabs[gi]) for gi in fine.local_indices}
            else:
                A.average_down(fine, coarse, r)
                out = {f"crse{gi}": bits_of(coarse.fabs[gi]) for gi in coarse.local_indices}
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, out))
    except BaseException:  # noqa: BLE001
        import traceback
        q.put((rank, "ERROR " + traceback.format_exc()))


# three 2-rank cases per kind keep the suite short (each case spawns two processes)
TWO_RANK = [n for kind in ("fill_patch", "average_down", "heat", "index_copy")
            for n in [m for m in names(kind) if case(m)["nranks"] == 2][:3]]


ENVS = {"host-sync": {}, "devsync": {"GHX_SYNC": "device", "GHX_BARRIER_TIMEOUT_S": "20"},
        "fallback": {"GHX_TRANSPORT": "nccl"}}


@pytest.mark.parametrize("mode", sorted(ENVS))
@pytest.mark.parametrize("name", TWO_RANK)
def test_level_transfers_two_processes(name, mode):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, name, ENVS[mode])) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
    got = {}
    for r in range(world):
        assert not isinstance(res[r], str), res[r]
        got.update(res[r])
    assert got
    for key, a in got.items():
        assert np.array_equal(a, data()[f"{name}/{key}"].ravel(order="F")), key
