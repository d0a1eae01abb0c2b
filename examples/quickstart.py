"""Quick start: FillBoundary, fill_patch, average_down and the CUDA-graph
heat loop through the drop-in API on one B200 (python examples/quickstart.py)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2403_12179_b200 as amr  # noqa: E402

amr.config.set_spacedim(3)
dom = amr.Box((0, 0, 0), (127, 127, 127))
geom = amr.Geometry(dom, (0.0,) * 3, (1.0,) * 3, (True, True, True))
ba = amr.decompose(dom, 64)
dm = amr.DistributionMapping.round_robin(len(ba), 1)
mf = amr.MultiFab(ba, dm, 4, 2, geom)
mf.fill_hash(1, dom)
amr.fill_boundary(mf, geom)                 # one fused sm_100a launch, bit-exact
x = amr.prepare_fill_boundary(mf, geom)     # enqueue-only variant
x.enqueue(torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()

# a fine patch at ratio 2 over the coarse cells [32, 95]^3
fgeom = geom.refined(2)
fba = amr.decompose(amr.Box((64, 64, 64), (191, 191, 191)), 64)
fdm = amr.DistributionMapping([0] * len(fba))
coarse = amr.MultiFab(ba, dm, 1, 1, geom)
fine = amr.MultiFab(fba, fdm, 1, 1, fgeom)
coarse.fill_hash(2, dom)
fine.fill_hash(3, fgeom.domain)
amr.fill_patch(fine, coarse, fgeom, geom, 2, amr.LINEAR)
amr.average_down(fine, coarse, 2)

# the heat demo's step loop, replayed from CUDA graphs after two eager steps
levels = [(coarse, amr.MultiFab(ba, dm, 1, 1, geom)), (fine, amr.MultiFab(fba, fdm, 1, 1, fgeom))]
for _, w in levels:
    w.setval(0.0)
loop = amr.heat.HeatLoop(levels, [geom, fgeom], 1e-6, 1.0, 2)
for _ in range(5):
    loop.step()
print("quickstart ok:", len(ba), "coarse fabs,", len(fba), "fine fabs,", loop.nsteps, "heat steps")
