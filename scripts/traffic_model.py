#!/usr/bin/env python3
"""Minimal DRAM traffic of a FillBoundary (lines read that hold source cells +
sectors written that hold ghost cells) for a uniform periodic decomposition:
    python scripts/traffic_model.py BOX NGHOST NCOMP NFABS
Compared with ncu dram__bytes in DESIGN.md section 3."""
# Minimal DRAM traffic model for FillBoundary on one fab-comp of a uniform periodic
# decomposition (box B, ghosts g, float64): lines read (128 B) containing source
# cells, sectors written (32 B) containing ghost cells.
import numpy as np, sys
B, g, nc, nfab = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
n = B + 2 * g
idx = np.arange(n)
valid = (idx >= g) & (idx < g + B)
# source cells of this fab: valid cells within g of its boundary (sent to neighbours)
src1 = valid & ((idx < 2 * g) | (idx >= B))
X, Y, Z = np.meshgrid(idx, idx, idx, indexing="ij")
vx, vy, vz = valid[X], valid[Y], valid[Z]
sx, sy, sz = src1[X], src1[Y], src1[Z]
isvalid = vx & vy & vz
src = isvalid & (sx | sy | sz)
ghost = ~isvalid
off = (X + n * (Y + n * Z)) * 8  # byte offset within the component (F order)
base = 0  # assume component start 128-B aligned (fabs are 256-B aligned; comps are n^3*8 apart)
lines_read = np.unique(off[src] // 128).size
sect_w = np.unique(off[ghost] // 32).size
lines_w = np.unique(off[ghost] // 128).size
alg = (ghost.sum()) * 16
tot = (lines_read * 128 + sect_w * 32)
print(f"B={B} g={g}: ghost cells {ghost.sum()}, alg {alg/1e6:.3f} MB/fab-comp; lines read {lines_read} "
      f"({lines_read*128/1e6:.3f} MB), sectors written {sect_w} ({sect_w*32/1e6:.3f} MB), "
      f"min DRAM {tot/1e6:.3f} MB = {tot/alg:.3f}x alg; whole job {tot*nc*nfab/1e6:.1f} MB")
