"""Host-side logic of the level transfers (no GPU): the uncovered-ghost
target computation of fill_patch against the oracle restatement of the
reference (amr.py:322-352), on every fill_patch golden case."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import amr_oracle as ao
from test_amr_oracle import case, names


@pytest.mark.parametrize("name", names("fill_patch"))
def test_coarse_fill_targets_match_oracle(name):
    import paper_2403_12179_b200 as amr
    from paper_2403_12179_b200 import amr as A
    c = case(name)
    dim, r = c["dim"], c["ratio"]
    amr.config.set_spacedim(dim)
    fdom = amr.Box((0,) * dim, tuple(e * r - 1 for e in c["cext"][:dim]))
    per = tuple(bool(p) for p in c["periodic"][:dim])
    fgeom = amr.Geometry(fdom, (0.0,) * dim, (1.0,) * dim, per)
    fba = amr.BoxArray([amr.Box(tuple(b[:dim]), tuple(b[3:3 + dim])) for b in c["fine_boxes"]])
    got = A._coarse_fill_targets(fba, amr.IntVect.filled(c["fngrow"]), fgeom)
    ng = [c["fngrow"] if d < dim else 0 for d in range(3)]
    exp = ao.fill_targets([np.asarray(b, np.int64) for b in c["fine_boxes"]], ng, np.asarray(fdom.as_row()),
                          list(per) + [False] * (3 - dim), dim)
    assert sorted(got) == sorted(exp)
    for gi in got:
        cells = lambda bs: sorted(tuple(x) for b in bs for x in np.stack(np.meshgrid(
            *[np.arange(b[d], b[3 + d] + 1) for d in range(3)], indexing="ij"), -1).reshape(-1, 3))
        assert cells([np.asarray(b.as_row()) for b in got[gi]]) == cells(exp[gi])


def test_amr_public_names():
    import paper_2403_12179_b200 as amr
    for n in ("fill_patch", "average_down", "interp_box", "LINEAR", "PIECEWISE_CONSTANT", "gather_fabs",
              "build_gather_plan"):
        assert hasattr(amr, n), n
    from paper_2403_12179_b200 import amr as A
    assert A.LINEAR == "linear" and A.PIECEWISE_CONSTANT == "piecewise_constant"
