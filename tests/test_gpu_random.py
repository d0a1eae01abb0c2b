"""Randomised FillBoundary layouts (anisotropic ghosts, odd extents, mixed
periodicity, float32/float64, device and pinned host memory, every task
variant of the fused kernel) against the CPU oracle (oracle/ghost_oracle.py,
itself pinned to the reference's golden vectors): raw bits."""

import numpy as np
import pytest

from gpu_util import bits_of
from oracle import ghost_oracle as go
from oracle import inputs

pytestmark = pytest.mark.gpu

VARIANTS = [{}, {"GHX_FAB_LOCAL": "0", "GHX_BULK": "1"}, {"GHX_FAB_LOCAL": "1"}, {"GHX_RING": "1"}]


def _layout(rng):
    ext = [int(rng.integers(6, 40)) for _ in range(3)]
    cuts = [np.unique(np.concatenate([[0], rng.integers(3, e - 2, int(rng.integers(0, 3))), [e]])) for e in ext]
    boxes = np.asarray([[x0, y0, z0, x1 - 1, y1 - 1, z1 - 1]
                        for z0, z1 in zip(cuts[2][:-1], cuts[2][1:])
                        for y0, y1 in zip(cuts[1][:-1], cuts[1][1:])
                        for x0, x1 in zip(cuts[0][:-1], cuts[0][1:])], np.int64)
    minext = int((boxes[:, 3:] - boxes[:, :3] + 1).min())  # the reference bounds max(ngrow) by it
    ng = [int(rng.integers(0, min(3, minext) + 1)) for _ in range(3)]
    per = [bool(v) for v in rng.integers(0, 2, 3)]
    return ext, boxes, ng, per


@pytest.mark.parametrize("seed", range(24))
def test_random_fill_boundary_matches_oracle(seed, monkeypatch):
    import paper_2403_12179_b200 as amr
    rng = np.random.default_rng(1000 + seed)
    ext, boxes, ng, per = _layout(rng)
    nc = int(rng.integers(1, 4))
    dt = np.float32 if seed % 5 == 4 else np.float64
    memory = "pinned" if seed % 6 == 5 else "device"
    for k, v in VARIANTS[seed % len(VARIANTS)].items():
        monkeypatch.setenv(k, v)
    amr.config.set_spacedim(3)
    amr.config.set_real_dtype(dt)
    dom = amr.Box((0, 0, 0), tuple(e - 1 for e in ext))
    geom = amr.Geometry(dom, (0.0,) * 3, (1.0,) * 3, tuple(per))
    ba = amr.BoxArray([amr.Box(tuple(b[:3]), tuple(b[3:])) for b in boxes])
    dm = amr.DistributionMapping([0] * len(ba))
    mf = amr.MultiFab(ba, dm, nc, amr.IntVect(*ng), geom, memory=memory)
    mf.fill_hash(inputs.SEED, dom)
    import torch
    torch.cuda.synchronize()
    amr.fill_boundary(mf, geom)
    # oracle
    plan = go.plan_fill_boundary(boxes, ng, per, ext, [0] * len(boxes), 1)
    fabs, lo = {}, {}
    for gi, b in enumerate(boxes):
        g = b.copy()
        g[:3] -= ng
        g[3:] += ng
        fabs[gi] = inputs.make_fab(g[:3], g[3:], nc, dt, b[:3], b[3:], [0] * 3, [e - 1 for e in ext])
        lo[gi] = g[:3]
    go.execute(plan, fabs, lo, fabs, lo, 0, 0, nc)
    for gi in range(len(boxes)):
        assert np.array_equal(bits_of(mf.fabs[gi]), inputs.bits(fabs[gi]).ravel(order="F")), f"fab {gi}"
