"""A reference user's switch, end to end: the reference's OWN MultiFab
(miniamr_core from baseline/_ref or $MINIAMR_REF), its numpy fabs in pinned
memory, exchanged by libghostx.so through integration/reference_binding.py
(ctypes only) -- checked bit for bit against the reference's own
comm.fill_boundary on a twin MultiFab, both timed.

    python examples/reference_binding_demo.py [n] [box] [ncomp]   (default 256 64 4: C2)
"""
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
ref_dir = os.environ.get("MINIAMR_REF", os.path.join(REPO, "baseline", "_ref"))
if not os.path.isdir(os.path.join(ref_dir, "miniamr_core")):
    sys.exit(f"reference install not found in {ref_dir} (python -c 'import __graft_entry__ as g; g.build()')")
sys.path.insert(0, ref_dir)

from miniamr_core import comm, config, index_space as ix, kernels, mesh  # noqa: E402

from integration.reference_binding import PinnedArena, fill_boundary_native  # noqa: E402

n, b, nc = (int(v) for v in (sys.argv[1:4] + ["256", "64", "4"][len(sys.argv[1:4]):]))
config.set_spacedim(3)
dom = ix.Box((0, 0, 0), (n - 1,) * 3)
geom = ix.Geometry(dom, (0.0,) * 3, (1.0,) * 3, (True,) * 3)
ba = mesh.decompose(dom, b)
dm = mesh.DistributionMapping.round_robin(len(ba), 1)
ours = mesh.MultiFab(ba, dm, nc, 2, geom, arena=PinnedArena())
theirs = mesh.MultiFab(ba, dm, nc, 2, geom)
for i in ours.local_indices:
    v = np.random.default_rng(i).standard_normal(ours.fabs[i].data.shape)
    ours.fabs[i].data[...] = v
    theirs.fabs[i].data[...] = v

fill_boundary_native(ours, geom)  # plan + executor, cached on the MultiFab
t0 = time.perf_counter()
for _ in range(5):
    fill_boundary_native(ours, geom)
t_ours = (time.perf_counter() - t0) / 5
backend = kernels.Backend("parallel", os.cpu_count())
comm.fill_boundary(theirs, geom, backend=backend)
t0 = time.perf_counter()
for _ in range(5):
    comm.fill_boundary(theirs, geom, backend=backend)
t_ref = (time.perf_counter() - t0) / 5
same = all(np.array_equal(ours.fabs[i].data.view(np.uint64), theirs.fabs[i].data.view(np.uint64))
           for i in ours.local_indices)
print(f"{n}^3 / {b}^3 boxes, {nc} comps, 2 ghosts, {len(ba)} fabs on the reference's own MultiFab")
print(f"  B200 through the C-ABI binding (host fabs over PCIe): {t_ours * 1e3:8.2f} ms per call")
print(f"  reference comm.fill_boundary, {backend.nworkers} threads:       {t_ref * 1e3:8.2f} ms per call")
print(f"  bit-identical: {same}")
sys.exit(0 if same else 1)
