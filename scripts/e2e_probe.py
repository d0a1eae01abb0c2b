"""Profile helper: C3 FillBoundary on pinned host fabs (zero-copy)."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2403_12179_b200 as amr
amr.config.set_spacedim(3)
n, b, nc, ng = [int(v) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (512, 128, 8, 2))]
dom = amr.Box((0, 0, 0), (n - 1,) * 3)
geom = amr.Geometry(dom, (0.0,) * 3, (1.0,) * 3, (True,) * 3)
ba = amr.decompose(dom, b)
mf = amr.MultiFab(ba, amr.DistributionMapping([0] * len(ba)), nc, ng, geom, memory="pinned")
mf.fill_hash(1, dom)
torch.cuda.synchronize()
for i in range(4):
    t0 = time.perf_counter()
    amr.fill_boundary(mf, geom)
    print(f"call {i}: {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
