"""C3 FillBoundary with G thread ranks sharing one GPU (runtime_spawn): every
rank's DIRECT executor stores its remote tags straight into the other ranks'
fabs through plain device pointers (no IPC).  Run under ncu to time each
rank's launch alone:  python scripts/thread_ranks_c3.py G [calls]"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2403_12179_b200 as amr  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 8
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 3
amr.config.set_spacedim(3)
dom = amr.Box((0, 0, 0), (511, 511, 511))
geom = amr.Geometry(dom, (0.0,) * 3, (1.0,) * 3, (True,) * 3)
ba = amr.decompose(dom, 128)
dm = amr.DistributionMapping.round_robin(len(ba), G)


def program(ctx):
    mf = amr.MultiFab(ba, dm, 8, 2, geom)
    mf.fill_hash(20261017, dom)
    torch.cuda.synchronize()
    ctx.barrier()
    for _ in range(calls):
        amr.fill_boundary(mf, geom)
    ctx.barrier()
    x = amr.comm.prepare_fill_boundary(mf, geom)
    return x.ex.detail


for r, d in enumerate(amr.runtime_spawn(G, program)):
    if r == 0:
        print(d)
