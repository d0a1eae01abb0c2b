"""Debug helper: FillBoundary with seam-chunk ring tasks (GHX_RING=1) on
device memory for several x-line lengths; prints bad cells per layout."""
import os
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
os.environ.setdefault("GHX_RING", "1")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2403_12179_b200 as amr  # noqa: E402

_bad_total = 0
from gpu_util import device_bits, expected_wrapped  # noqa: E402

amr.config.set_spacedim(3)
for (nx, ny, nz, b, nc) in [(128, 64, 64, 64, 1), (192, 64, 64, 64, 1), (256, 64, 64, 64, 1), (64, 64, 64, 64, 1),
                            (128, 128, 128, 64, 2), (128, 32, 32, 32, 1), (96, 40, 24, 32, 1),
                            (256, 32, 48, 32, 2), (512, 32, 32, 32, 1), (64, 200, 16, 64, 1)]:
    dom = amr.Box((0, 0, 0), (nx - 1, ny - 1, nz - 1))
    geom = amr.Geometry(dom, (0.0,) * 3, (1.0,) * 3, (True,) * 3)
    ba = amr.decompose(dom, b)
    mf = amr.MultiFab(ba, amr.DistributionMapping([0] * len(ba)), nc, 2, geom)
    mf.fill_hash(7, dom)
    amr.fill_boundary(mf, geom)
    ex = amr.comm.prepare_fill_boundary(mf, geom).ex
    bad = 0
    for gi in mf.local_indices:
        f = mf.fabs[gi]
        exp = expected_wrapped(f, nc, dom.as_row(), (1, 1, 1), 7, 8)
        bad += int((device_bits(f) != exp).sum().item())
    print(nx, ny, nz, b, nc, "ring tasks", ex.detail["ring_tasks"], "swap", ex.detail["swap_tasks"], "bad", bad,
          flush=True)
    _bad_total += bad
sys.exit(1 if _bad_total else 0)
