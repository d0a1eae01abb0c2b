"""Process-per-GPU host logic over torch.distributed with the gloo backend,
world_size 2, 4 and 8, on CPU: collectives of ProcessContext, identical plans on
every rank, reference message accounting, and the NCCL-fallback buffer
contract (what rank s packs for rank d is exactly what d unpacks from s)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import golden_util as gu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                          WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2403_12179_b200 as amr
        from paper_2403_12179_b200 import _native as N
        from paper_2403_12179_b200 import comm
        ctx = comm.current_ctx()
        assert ctx.kind == "process" and ctx.rank == rank and ctx.nranks == world
        assert ctx.allgather(rank * 10) == [10 * r for r in range(world)]
        assert ctx.allreduce([amr.SUM, amr.MAX], [rank + 1, rank]) == (world * (world + 1) / 2, world - 1.0)
        ctx.barrier()
        out = {}
        # C3 at `world` ranks: plan + accounting vs the reference-generated fixture
        amr.config.set_spacedim(3)
        n, b, nc, ng = 512, 128, 8, 2
        dom = amr.Box((0, 0, 0), (n - 1,) * 3)
        geom = amr.Geometry(dom, (0.0,) * 3, (1.0,) * 3, (True,) * 3)
        ba = amr.decompose(dom, b)
        # an extra, box-less rank index keeps MultiFab from allocating on CPU
        dm = amr.DistributionMapping([i % world for i in range(len(ba))], world)
        mfv = amr.MultiFab(ba, amr.DistributionMapping(dm.rank_of, world + 1), nc, ng, geom, rank=world)
        plan = amr.plan_build_fill_boundary(mfv, geom)
        out["segments"] = plan.num_segments
        out["digest"] = gu.seg_digest(plan.rows())
        # rank-local executors for the real layout (host-side compile only)
        import ctypes as C
        rows = ba.rows(amr.IntVect(ng, ng, ng))
        h = C.c_void_p()
        N.check(N.lib.ghx_plan_build_fill_boundary(len(ba), N.i64p(ba.rows()), N.i64p(np.full(3, ng, np.int64)),
                                                   N.i32p(np.ones(3, np.int32)), N.i64p(np.full(3, n, np.int64)),
                                                   N.i32p(dm.array()), world, C.byref(h)))
        plan2 = comm.CommPlan(h.value, world, 3, ba.ixtype)
        pack = comm.Executor(plan2, rank, N.EXEC_PACK, rows, nc, rows, nc, 0, 0, nc, 8, 0)
        unpack = comm.Executor(plan2, rank, N.EXEC_UNPACK, rows, nc, rows, nc, 0, 0, nc, 8, 0)
        direct = comm.Executor(plan2, rank, N.EXEC_DIRECT, rows, nc, rows, nc, 0, 0, nc, 8, 0)
        local = comm.Executor(plan2, rank, N.EXEC_LOCAL, rows, nc, rows, nc, 0, 0, nc, 8, 0)
        sizes = ctx.allgather((pack.buffer_elems.tolist(), unpack.buffer_elems.tolist()))
        for s in range(world):
            for d in range(world):
                if s != d:
                    assert sizes[s][0][d] == sizes[d][1][s], (s, d)
        out["pair_bytes"] = {f"{rank}->{d}": int(plan2.pair_cells[rank, d]) * nc * 8
                             for d in range(world) if d != rank and plan2.pair_cells[rank, d]}
        out["elems"] = (direct.elems, local.elems + pack.elems, local.elems + unpack.elems)
        out["sync"] = comm._sync_mode(ctx)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, out))
    except BaseException as e:  # noqa: BLE001
        import traceback
        q.put((rank, "ERROR " + traceback.format_exc()))


@pytest.mark.parametrize("world", [2, 4, 8])
def test_process_group_plans_accounting_and_buffers(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert not isinstance(res[r], str), res[r]
    c = gu.case(f"C3_x{world}")
    got_pairs = {}
    for r in range(world):
        assert res[r]["segments"] == c["num_segments"]
        got_pairs.update(res[r]["pair_bytes"])
        direct, pack_side, unpack_side = res[r]["elems"]
        assert direct == pack_side  # push = local + everything I send
        # host sync when both ranks share one device (this container: device 0)
        assert res[r]["sync"] == "host"
    assert got_pairs == c["pair_bytes"]
    assert all(res[r]["digest"] == res[0]["digest"] for r in range(world))
