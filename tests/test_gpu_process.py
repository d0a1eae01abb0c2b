"""Process-per-GPU exchange path on one GPU: two processes (gloo process
group for the plumbing) share cuda:0, map each other's fab slabs with CUDA
IPC and push remote tags straight into the peer's ghost cells (host-side
synchronisation, since both ranks share the device).  Checked against the
wrapped-hash property and the reference's per-pair message accounting."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import golden_util as gu

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q, n, b, nc, ng, env=None):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                          WORLD_SIZE=str(world), LOCAL_RANK="0")
        os.environ.update(env or {})
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2403_12179_b200 as amr
        from gpu_util import device_bits, expected_wrapped
        from oracle import inputs
        amr.config.set_spacedim(3)
        dom = amr.Box((0, 0, 0), (n - 1,) * 3)
        geom = amr.Geometry(dom, (0.0,) * 3, (1.0,) * 3, (True,) * 3)
        ba = amr.decompose(dom, b)
        dm = amr.DistributionMapping.round_robin(len(ba), world)
        arena = None
        if os.environ.get("GHX_TEST_ARENA"):  # storage inside a pooled slab, after a 4 KiB block
            from paper_2403_12179_b200.arena import Arena
            arena = Arena(0)
            arena.alloc(4096)
        memory = "pinned" if os.environ.get("GHX_TEST_PINNED") else "device"  # host-resident fabs
        mf = amr.MultiFab(ba, dm, nc, ng, geom, arena=arena, memory=memory)
        mf.fill_hash(inputs.SEED, dom)
        torch.cuda.synchronize()
        ctx = amr.current_ctx()
        s0 = ctx.bus.stats_snapshot()
        # GHX_TEST_DELAY="r:s": rank r enters each exchange s seconds late,
        # so the peers' kernels really wait in the READY / DONE spins
        delay = os.environ.get("GHX_TEST_DELAY")
        for _ in range(2):
            if delay and int(delay.split(":")[0]) == rank:
                import time
                time.sleep(float(delay.split(":")[1]))
            amr.fill_boundary(mf, geom)
        s1 = ctx.bus.stats_snapshot()
        bad = 0
        for gi in mf.local_indices:
            f = mf.fabs[gi]
            exp = expected_wrapped(f, nc, dom.as_row(), (1, 1, 1), inputs.SEED, 8)
            bad += int((device_bits(f).to(exp.device) != exp).sum().item())
        stats = {f"{s}->{d}": (s1[(s, d)][0] - s0[(s, d)][0], s1[(s, d)][1] - s0[(s, d)][1])
                 for (s, d) in s1 if s1[(s, d)] != s0[(s, d)]}
        if os.environ.get("GHX_TEST_NO_IPC"):  # the probe must have picked the NCCL transport
            assert amr.comm.prepare_fill_boundary(mf, geom).transport == "nccl"
        dist.barrier()
        del mf
        dist.destroy_process_group()
        q.put((rank, (bad, stats)))
    except BaseException:  # noqa: BLE001
        import traceback
        q.put((rank, "ERROR " + traceback.format_exc()))


CASES = [("C1", 64, 32, 1, 1, "C1_x2", {"GHX_REMOTE": "direct"}), ("C3", 512, 128, 8, 2, "C3_x2", {}),
         ("C3", 512, 128, 8, 2, "C3_x2", {"GHX_REMOTE": "direct"}),
         # device flag barriers between two processes time-sliced on one GPU:
         # the in-kernel READY / DONE protocol (default), packed and direct,
         # and the standalone barrier kernels (GHX_FUSED_SYNC=0)
         ("C1", 64, 32, 1, 1, "C1_x2", {"GHX_SYNC": "device", "GHX_BARRIER_TIMEOUT_S": "20"}),
         ("C1", 64, 32, 1, 1, "C1_x2", {"GHX_SYNC": "device", "GHX_BARRIER_TIMEOUT_S": "20", "GHX_REMOTE": "direct"}),
         ("C3", 512, 128, 8, 2, "C3_x2", {"GHX_SYNC": "device", "GHX_BARRIER_TIMEOUT_S": "20"}),
         ("C3", 512, 128, 8, 2, "C3_x2", {"GHX_SYNC": "device", "GHX_BARRIER_TIMEOUT_S": "20", "GHX_REMOTE": "direct"}),
         ("C1", 64, 32, 1, 1, "C1_x2", {"GHX_SYNC": "device", "GHX_BARRIER_TIMEOUT_S": "20", "GHX_FUSED_SYNC": "0"}),
         ("C1", 64, 32, 1, 1, "C1_x2", {"GHX_SYNC": "device", "GHX_BARRIER_TIMEOUT_S": "20",
                                        "GHX_REMOTE_ORDER": "interleave"}),
         # one rank late: the other's remote tasks wait for its READY, its
         # unpack (packed) / exit wait (direct) for its DONE
         ("C1", 64, 32, 1, 1, "C1_x2", {"GHX_SYNC": "device", "GHX_BARRIER_TIMEOUT_S": "20", "GHX_TEST_DELAY": "1:0.3"}),
         ("C3", 512, 128, 8, 2, "C3_x2", {"GHX_SYNC": "device", "GHX_BARRIER_TIMEOUT_S": "20",
                                          "GHX_TEST_DELAY": "0:0.3", "GHX_REMOTE": "direct"}),
         # the pack -> message -> unpack fallback (host-staged over gloo here),
         # selected explicitly or because CUDA IPC is unavailable
         ("C1", 64, 32, 1, 1, "C1_x2", {"GHX_TRANSPORT": "nccl"}),
         ("C1", 64, 32, 1, 1, "C1_x2", {"GHX_TEST_NO_IPC": "1"}),
         ("C3", 512, 128, 8, 2, "C3_x2", {"GHX_TRANSPORT": "nccl"}),
         # fab storage at an offset inside an arena slab: IPC maps whole allocations
         ("C1", 64, 32, 1, 1, "C1_x2", {"GHX_TEST_ARENA": "1", "GHX_REMOTE": "direct"}),
         # fabs in pinned host memory: pack -> message -> unpack, kernels over PCIe
         ("C1", 64, 32, 1, 1, "C1_x2", {"GHX_TEST_PINNED": "1"}),
         ("C3", 512, 128, 8, 2, "C3_x2", {"GHX_TEST_PINNED": "1"}),
         # pinned host fabs with the in-kernel READY/DONE protocol
         ("C1", 64, 32, 1, 1, "C1_x2", {"GHX_TEST_PINNED": "1", "GHX_SYNC": "device", "GHX_BARRIER_TIMEOUT_S": "20"})]


@pytest.mark.parametrize("cfg", CASES, ids=["C1-ipc-direct", "C3-ipc-packed", "C3-ipc-direct", "C1-devbarrier-packed",
                                            "C1-devsync-direct", "C3-devsync-packed", "C3-devsync-direct",
                                            "C1-devbarrier-unfused", "C1-devsync-interleave", "C1-devsync-late1",
                                            "C3-devsync-late0-direct", "C1-fallback", "C1-no-ipc-fallback", "C3-fallback", "C1-arena-ipc", "C1-pinned",
                                            "C3-pinned", "C1-pinned-devsync"])
def test_two_processes_one_gpu(cfg):
    _run(cfg, 2)


# C3 at 4 and 8 ranks (8 and 40 ordered pairs): every rank maps
# every peer it pushes to; message accounting against the reference's plan
@pytest.mark.parametrize("world,env", [(4, {}), (4, {"GHX_TRANSPORT": "nccl"}), (8, {}),
                                       (4, {"GHX_SYNC": "device", "GHX_BARRIER_TIMEOUT_S": "30"}),
                                       (4, {"GHX_SYNC": "device", "GHX_BARRIER_TIMEOUT_S": "30", "GHX_REMOTE": "direct"}),
                                       (8, {"GHX_SYNC": "device", "GHX_BARRIER_TIMEOUT_S": "60"}),
                                       (8, {"GHX_SYNC": "device", "GHX_BARRIER_TIMEOUT_S": "60", "GHX_ONE_KERNEL": "0"})],
                         ids=["C3x4-ipc-packed", "C3x4-fallback", "C3x8-ipc-packed", "C3x4-devbarrier",
                              "C3x4-devsync-direct", "C3x8-devsync", "C3x8-devsync-two-kernels"])
def test_many_processes_one_gpu(world, env):
    _run(("C3", 512, 128, 8, 2, f"C3_x{world}", env), world)


def _run(cfg, world):
    name, n, b, nc, ng, golden, env = cfg
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, n, b, nc, ng, env)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
    for r in range(world):
        assert not isinstance(res[r], str), res[r]
        assert res[r][0] == 0, f"rank {r}: {res[r][0]} cells differ"
    c = gu.case(golden)
    pair_bytes = {}
    for r in range(world):
        for k, (msgs, nbytes) in res[r][1].items():
            assert msgs == 2  # two calls, one message per ordered pair per call
            pair_bytes[k] = nbytes // 2
    assert pair_bytes == {k: v * nc // c["ncomp"] for k, v in c["pair_bytes"].items()}


def _absent_worker(rank, world, port, q):
    """Rank 1 never enters the exchange: rank 0's kernel must give up after
    GHX_BARRIER_TIMEOUT_S and its synchronous call raise, not hang the GPU."""
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                          WORLD_SIZE=str(world), LOCAL_RANK="0", GHX_SYNC="device", GHX_BARRIER_TIMEOUT_S="2")
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2403_12179_b200 as amr
        from paper_2403_12179_b200 import comm
        amr.config.set_spacedim(3)
        dom = amr.Box((0, 0, 0), (63, 63, 63))
        geom = amr.Geometry(dom, (0.0,) * 3, (1.0,) * 3, (True,) * 3)
        ba = amr.decompose(dom, 32)
        mf = amr.MultiFab(ba, amr.DistributionMapping.round_robin(len(ba), world), 1, 1, geom)
        x = comm.prepare_fill_boundary(mf, geom)  # collective setup (IPC handles, flags)
        dist.barrier()
        out = "skipped"
        if rank == 0:
            try:
                x.run()
                out = "no error"
            except Exception as e:  # noqa: BLE001
                out = type(e).__name__ + ": " + str(e)
        dist.barrier()
        del x, mf
        dist.destroy_process_group()
        q.put((rank, out))
    except BaseException:  # noqa: BLE001
        import traceback
        q.put((rank, "ERROR " + traceback.format_exc()))


def test_device_sync_times_out_when_a_peer_never_arrives():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_absent_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    assert "timed out" in res[0], res[0]
    assert res[1] == "skipped", res[1]


def _pc_worker(rank, world, port, q, env):
    """ParallelCopy between two layouts (64^3-box source -> 32^3-box
    destination of a 128^3 domain, 2 comps) across processes sharing the GPU:
    every destination cell must hold the source hash of its cell."""
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                          WORLD_SIZE=str(world), LOCAL_RANK="0")
        os.environ.update(env or {})
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2403_12179_b200 as amr
        from gpu_util import device_bits, expected_wrapped
        from oracle import inputs
        amr.config.set_spacedim(3)
        dom = amr.Box((0, 0, 0), (127, 127, 127))
        sba, dba = amr.decompose(dom, 64), amr.decompose(dom, 32)
        src = amr.MultiFab(sba, amr.DistributionMapping.round_robin(len(sba), world), 2, 0)
        dst = amr.MultiFab(dba, amr.DistributionMapping.round_robin(len(dba), world), 2, 0)
        src.fill_hash(inputs.SEED, dom)
        dst.setval(0.0)
        torch.cuda.synchronize()
        for _ in range(2):
            amr.parallel_copy(dst, src)
        bad = 0
        for gi in dst.local_indices:
            f = dst.fabs[gi]
            exp = expected_wrapped(f, 2, dom.as_row(), (0, 0, 0), inputs.SEED, 8)
            bad += int((device_bits(f) != exp).sum().item())
        x = amr.comm.prepare_parallel_copy(dst, src)
        dist.barrier()
        del src, dst, x
        dist.destroy_process_group()
        q.put((rank, bad))
    except BaseException:  # noqa: BLE001
        import traceback
        q.put((rank, "ERROR " + traceback.format_exc()))


@pytest.mark.parametrize("env", [{}, {"GHX_SYNC": "device", "GHX_BARRIER_TIMEOUT_S": "20"},
                                 {"GHX_SYNC": "device", "GHX_BARRIER_TIMEOUT_S": "20", "GHX_REMOTE": "direct"},
                                 {"GHX_TRANSPORT": "nccl"}],
                         ids=["host-sync", "devsync-packed", "devsync-direct", "fallback"])
def test_parallel_copy_two_processes(env):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pc_worker, args=(r, 2, port, q, env)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
    for r in range(2):
        assert res[r] == 0, res[r]


def test_torch_stream_zero_orders_against_native_launches():
    """comm.torch_stream(0) must be torch's view of the SAME legacy default
    stream the native library launches on when handed 0 (torch's
    ExternalStream(0) is another stream): its synchronize waits for them."""
    import time

    import torch

    import paper_2403_12179_b200 as amr
    from paper_2403_12179_b200 import comm
    amr.config.set_spacedim(3)
    dom = amr.Box((0, 0, 0), (255, 255, 255))
    geom = amr.Geometry(dom, (0.0,) * 3, (1.0,) * 3, (True,) * 3)
    mf = amr.MultiFab(amr.decompose(dom, 64), amr.DistributionMapping.round_robin(64, 1), 4, 2, geom)
    mf.fill_hash(1, dom)
    x = comm.prepare_fill_boundary(mf, geom)
    torch.cuda.synchronize()
    with comm.torch_stream(0, 0) as ts:
        assert ts.cuda_stream == 0
        for _ in range(40):  # ~3.5 ms of native work on stream 0
            x.b_ex.run(0)
        t0 = time.perf_counter()
        ts.synchronize()
        waited = time.perf_counter() - t0
    assert waited > 1e-3, waited
