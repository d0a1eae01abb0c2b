"""Profile helper: FillBoundary on pinned host fabs (zero-copy over PCIe).

    python scripts/e2e_probe.py N BOX NCOMP NGX NGY NGZ [memory]

Prints the public-call wall time and the kernel's CUDA-event time."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2403_12179_b200 as amr  # noqa: E402
from paper_2403_12179_b200 import comm  # noqa: E402

amr.config.set_spacedim(3)
a = sys.argv[1:]
n, b, nc = int(a[0]), int(a[1]), int(a[2])
ng = amr.IntVect(int(a[3]), int(a[4]), int(a[5]))
memory = a[6] if len(a) > 6 else "pinned"
dom = amr.Box((0, 0, 0), (n - 1,) * 3)
geom = amr.Geometry(dom, (0.0,) * 3, (1.0,) * 3, (True,) * 3)
ba = amr.decompose(dom, b)
mf = amr.MultiFab(ba, amr.DistributionMapping([0] * len(ba)), nc, ng, geom, memory=memory)
mf.fill_hash(1, dom)
torch.cuda.synchronize()
amr.fill_boundary(mf, geom)
plan = comm.plan_build_fill_boundary(mf, geom)
x = comm.exchange_for(plan, mf, mf, 0, 0, nc)
st = torch.cuda.current_stream()
walls, kern = [], []
for i in range(5):
    t0 = time.perf_counter()
    amr.fill_boundary(mf, geom)
    walls.append(1e3 * (time.perf_counter() - t0))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    x.enqueue(st.cuda_stream)
    e1.record(st)
    e1.synchronize()
    kern.append(e0.elapsed_time(e1))
gb = x.ghost_bytes / 1e9
print(f"{memory} n={n} box={b} nc={nc} ng={tuple(ng)}: public call {min(walls):.3f} ms, kernel {min(kern):.3f} ms, "
      f"{gb / (min(kern) * 1e-3):.2f} GB/s ghost (kernel)", flush=True)
