"""Host overhead of one public fill_boundary call on a small MultiFab (C1
shape, device-resident): wall time per call vs the kernel time, plus a
cProfile of the Python side.  Diagnostic, not part of the bench."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import torch

import paper_2403_12179_b200 as amr

amr.config.set_spacedim(3)
dom = amr.Box((0, 0, 0), (63, 63, 63))
geom = amr.Geometry(dom, (0.0,) * 3, (1.0,) * 3, (True,) * 3)
ba = amr.decompose(dom, 32)
dm = amr.DistributionMapping.round_robin(len(ba), 1)
mf = amr.MultiFab(ba, dm, 1, 1, geom)
mf.setval(1.0)
for _ in range(10):
    amr.fill_boundary(mf, geom)
torch.cuda.synchronize()
n = 2000
t0 = time.perf_counter()
for _ in range(n):
    amr.fill_boundary(mf, geom)
dt = (time.perf_counter() - t0) / n
x = amr.prepare_fill_boundary(mf, geom)
st = torch.cuda.current_stream()
t0 = time.perf_counter()
for _ in range(n):
    x.enqueue(st.cuda_stream)
st.synchronize()
dq = (time.perf_counter() - t0) / n
print(f"fill_boundary wall per call {dt * 1e6:.1f} us; enqueue-only {dq * 1e6:.1f} us")
pr = cProfile.Profile()
pr.enable()
for _ in range(500):
    amr.fill_boundary(mf, geom)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
