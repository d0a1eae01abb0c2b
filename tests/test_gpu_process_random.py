"""Randomised FillBoundary layouts across 2 and 3 PROCESSES sharing the GPU
(round-robin boxes, so most faces are remote): anisotropic ghosts, odd
extents, mixed periodicity, float32/float64 -- every remote transport and
sync mode, packed unpacks with sector fills included -- against the CPU
oracle (oracle/ghost_oracle.py) on every rank's fabs, raw bits."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

NLAYOUTS = 10


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _layout(rng):
    ext = [int(rng.integers(8, 40)) for _ in range(3)]
    cuts = [np.unique(np.concatenate([[0], rng.integers(3, e - 2, int(rng.integers(1, 3))), [e]])) for e in ext]
    boxes = np.asarray([[x0, y0, z0, x1 - 1, y1 - 1, z1 - 1]
                        for z0, z1 in zip(cuts[2][:-1], cuts[2][1:])
                        for y0, y1 in zip(cuts[1][:-1], cuts[1][1:])
                        for x0, x1 in zip(cuts[0][:-1], cuts[0][1:])], np.int64)
    minext = int((boxes[:, 3:] - boxes[:, :3] + 1).min())
    ng = [int(rng.integers(0, min(4, minext) + 1)) for _ in range(3)]
    per = [bool(v) for v in rng.integers(0, 2, 3)]
    return ext, boxes, ng, per


def _fixed_layout(_rng):
    """Two boxes of a periodic 16 x 8 x 8 domain: with 3 or 4 ranks, ranks 2
    and 3 own no box and take part in the in-kernel protocol with empty
    executors."""
    return [16, 8, 8], np.asarray([[0, 0, 0, 7, 7, 7], [8, 0, 0, 15, 7, 7]], np.int64), [2, 1, 2], [True] * 3


def _worker(rank, world, port, q, seed0, env, fixed=False):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                          LOCAL_RANK="0")
        env = dict(env)
        memory = env.pop("_MEMORY", "device")
        os.environ.update(env)
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2403_12179_b200 as amr
        from gpu_util import bits_of
        from oracle import ghost_oracle as go
        from oracle import inputs
        bad = []
        for k in range(1 if fixed else NLAYOUTS):
            rng = np.random.default_rng(seed0 + k)
            ext, boxes, ng, per = (_fixed_layout if fixed else _layout)(rng)
            nc = int(rng.integers(1, 4))
            dt = np.float32 if k % 3 == 2 else np.float64
            amr.config.set_spacedim(3)
            amr.config.set_real_dtype(dt)
            dom = amr.Box((0, 0, 0), tuple(e - 1 for e in ext))
            geom = amr.Geometry(dom, (0.0,) * 3, (1.0,) * 3, tuple(per))
            ba = amr.BoxArray([amr.Box(tuple(b[:3]), tuple(b[3:])) for b in boxes])
            ranks = [i % world for i in range(len(boxes))]
            mf = amr.MultiFab(ba, amr.DistributionMapping(ranks, world), nc, amr.IntVect(*ng), geom, memory=memory)
            mf.fill_hash(inputs.SEED, dom)
            torch.cuda.synchronize()
            for _ in range(2):
                amr.fill_boundary(mf, geom)
            plan = go.plan_fill_boundary(boxes, ng, per, ext, ranks, world)
            fabs, lo = {}, {}
            for gi, b in enumerate(boxes):
                g = b.copy()
                g[:3] -= ng
                g[3:] += ng
                fabs[gi] = inputs.make_fab(g[:3], g[3:], nc, dt, b[:3], b[3:], [0] * 3, [e - 1 for e in ext])
                lo[gi] = g[:3]
            go.execute(plan, fabs, lo, fabs, lo, 0, 0, nc)
            for gi in mf.local_indices:
                if not np.array_equal(bits_of(mf.fabs[gi]), inputs.bits(fabs[gi]).ravel(order="F")):
                    bad.append((k, gi))
            del mf
        amr.config.set_real_dtype(np.dtype("f8"))
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, bad))
    except BaseException:  # noqa: BLE001
        import traceback
        q.put((rank, "ERROR " + traceback.format_exc()))


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("env", [{}, {"GHX_SYNC": "device", "GHX_BARRIER_TIMEOUT_S": "20"},
                                 {"GHX_SYNC": "device", "GHX_BARRIER_TIMEOUT_S": "20", "GHX_REMOTE": "direct"},
                                 {"GHX_TRANSPORT": "nccl"}, {"GHX_SECTOR_FILL": "0"},
                                 {"GHX_SYNC": "device", "GHX_BARRIER_TIMEOUT_S": "20", "GHX_ONE_KERNEL": "0"},
                                 {"_MEMORY": "pinned"}, {"_MEMORY": "pinned", "GHX_SEAM_TASKS": "0"},
                                 {"_MEMORY": "pinned", "GHX_SYNC": "device", "GHX_BARRIER_TIMEOUT_S": "20"}],
                         ids=["host-sync-packed", "devsync-packed", "devsync-direct", "fallback", "no-sector-fill",
                              "devsync-two-kernels", "pinned", "pinned-no-seam-tasks", "pinned-devsync"])
def test_random_layouts_across_processes(world, env):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    seed0 = 5000 + 100 * world
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, seed0, env)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=900) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
    errs = [res[r] for r in range(world) if isinstance(res[r], str)]
    assert not errs, "\n".join(e[-1500:] for e in errs)
    assert all(res[r] == [] for r in range(world)), res


@pytest.mark.parametrize("world", [3, 4])
@pytest.mark.parametrize("env", [{"GHX_SYNC": "device", "GHX_BARRIER_TIMEOUT_S": "20"},
                                 {"GHX_SYNC": "device", "GHX_BARRIER_TIMEOUT_S": "20", "GHX_ONE_KERNEL": "0"}, {}],
                         ids=["devsync-one-kernel", "devsync-two-kernels", "host-sync"])
def test_ranks_without_boxes(world, env):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, 0, env, True)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
    errs = [res[r] for r in range(world) if isinstance(res[r], str)]
    assert not errs, "\n".join(e[-1500:] for e in errs)
    assert all(res[r] == [] for r in range(world)), res
