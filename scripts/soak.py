"""Soak test (diagnostic): many back-to-back exchanges in thread mode
(runtime_spawn, 4 rank threads on one GPU) and, under torchrun, in process
mode, then the wrapped-hash check -- looks for rare hangs or races in the
rank synchronisation.  Usage:
    python scripts/soak.py [calls]
    torchrun --nproc-per-node 4 scripts/soak.py [calls]   (GHX_BENCH_BACKEND-style gloo)
SOAK_MEMORY=pinned puts the fabs in pinned host memory.
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch

import paper_2403_12179_b200 as amr
from gpu_util import device_bits, expected_wrapped
from oracle import inputs

CALLS = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
amr.config.set_spacedim(3)
dom = amr.Box((0, 0, 0), (63, 63, 63))
geom = amr.Geometry(dom, (0.0,) * 3, (1.0,) * 3, (True,) * 3)
ba = amr.decompose(dom, 16)


def program(ctx):
    dm = amr.DistributionMapping.round_robin(len(ba), ctx.nranks)
    mf = amr.MultiFab(ba, dm, 2, 2, geom, memory=os.environ.get("SOAK_MEMORY", "device"))
    mf.fill_hash(inputs.SEED, dom)
    torch.cuda.synchronize()
    for _ in range(CALLS):
        amr.fill_boundary(mf, geom)
    bad = 0
    for gi in mf.local_indices:
        f = mf.fabs[gi]
        exp = expected_wrapped(f, 2, dom.as_row(), (1, 1, 1), inputs.SEED, 8)
        bad += int((device_bits(f).to(exp.device) != exp).sum())  # (pinned fabs: a host view)
    return bad


if "RANK" in os.environ:
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    t0 = time.perf_counter()
    bad = program(amr.current_ctx())
    t = torch.tensor([bad])
    dist.all_reduce(t)
    if dist.get_rank() == 0:
        print(f"process mode x{dist.get_world_size()} ({os.environ.get('SOAK_MEMORY', 'device')}): {CALLS} calls "
              f"in {time.perf_counter() - t0:.1f} s, {int(t.item())} bad cells")
    dist.destroy_process_group()
else:
    t0 = time.perf_counter()
    res = amr.runtime_spawn(4, program)
    print(f"thread mode x4: {CALLS} calls in {time.perf_counter() - t0:.1f} s, {sum(res)} bad cells")
