import sys, time
sys.path.insert(0, ".")
import torch, ctypes as C
import paper_2403_12179_b200 as amr
from paper_2403_12179_b200 import comm, _native as N
amr.config.set_spacedim(3)
dom = amr.Box((0,0,0),(511,511,511)); geom = amr.Geometry(dom,(0.0,)*3,(1.0,)*3,(True,)*3)
ba = amr.decompose(dom, 128); dm = amr.DistributionMapping.round_robin(len(ba), 1)
mf = amr.MultiFab(ba, dm, 8, 2, geom); mf.fill_hash(1, dom)
x = comm.prepare_fill_boundary(mf, geom)
torch.cuda.synchronize()
cs = torch.cuda.current_stream()
print("torch current stream handle:", cs.cuda_stream, "default:", torch.cuda.default_stream().cuda_stream)
for label, sync in (("torch stream.synchronize", lambda: cs.synchronize()),
                    ("ExternalStream(0).synchronize", lambda: torch.cuda.ExternalStream(0).synchronize()),
                    ("ghx_stream_sync(0)", lambda: N.lib.ghx_stream_sync(None)),
                    ("torch.cuda.synchronize", lambda: torch.cuda.synchronize())):
    for _ in range(2):
        torch.cuda.synchronize()
        for _ in range(5): x.b_ex.run(0)  # 5 x 0.7 ms on OUR stream 0
        t0 = time.perf_counter(); sync(); t1 = time.perf_counter()
        torch.cuda.synchronize()
    print(f"{label:32s} waited {1e3*(t1-t0):.3f} ms (5 launches = ~3.5 ms)")
with torch.cuda.stream(torch.cuda.ExternalStream(0)):
    torch.cuda.synchronize()
    for _ in range(5): x.b_ex.run(0)
    t0 = time.perf_counter(); torch.cuda.current_stream().synchronize(); t1 = time.perf_counter()
    print(f"inside ExternalStream(0) ctx: current().synchronize waited {1e3*(t1-t0):.3f} ms, current handle {torch.cuda.current_stream().cuda_stream}")
