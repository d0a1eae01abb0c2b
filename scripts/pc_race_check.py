# Diagnostic: repeat one ParallelCopy (source ghosts, periodic) through the reference binding and
# compare with the reference serial backend (its parallel backend races on overlapping destinations).
import sys, os
import numpy as np
sys.path.insert(0, "baseline/_ref"); sys.path.insert(0, ".")
from miniamr_core import comm, config, index_space as ix, mesh
from integration.reference_binding import PinnedArena, parallel_copy_native
config.set_spacedim(3)
n, sb, db, nc, gs, gd = 24, 12, 8, 1, 1, 2
dom = ix.Box((0, 0, 0), (n - 1,) * 3)
geom = ix.Geometry(dom, (0.0,) * 3, (1.0,) * 3, (1, 1, 1))
sba, dba = mesh.decompose(dom, sb), mesh.decompose(dom, db)
sdm = mesh.DistributionMapping.round_robin(len(sba), 1)
ddm = mesh.DistributionMapping.round_robin(len(dba), 1)
def fill(mf, seed):
    rng = np.random.default_rng(seed)
    for i in mf.local_indices:
        a = mf.fabs[i].data; a[...] = rng.standard_normal(a.shape)
src_r, dst_r = mesh.MultiFab(sba, sdm, nc, gs), mesh.MultiFab(dba, ddm, nc + 1, gd)
fill(src_r, 11); fill(dst_r, 12)
from miniamr_core import kernels
comm.parallel_copy(dst_r, src_r, 0, 1, nc, gs, gd, geom, backend=kernels.Backend("serial"))
bad_runs = 0
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 20):
    arena = PinnedArena()
    src_o, dst_o = mesh.MultiFab(sba, sdm, nc, gs, arena=arena), mesh.MultiFab(dba, ddm, nc + 1, gd, arena=arena)
    fill(src_o, 11); fill(dst_o, 12)
    parallel_copy_native(dst_o, src_o, 0, 1, nc, gs, gd, geom)
    nbad = 0
    for i in dst_o.local_indices:
        a, b = dst_o.fabs[i].data, dst_r.fabs[i].data
        d = np.argwhere(a.view(np.uint64) != b.view(np.uint64))
        if len(d):
            nbad += len(d)
            if bad_runs == 0:
                print("rep", rep, "fab", i, "box", dba[i], "first bad (i,j,k,c):", d[:6].tolist(), "of", len(d))
    if nbad:
        bad_runs += 1
print("bad runs", bad_runs)
