"""Zero-copy fab views (reference frontend/tests/test_bridge.py semantics) on
device and pinned-host fabs."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _amr():
    import paper_2403_12179_b200 as amr
    return amr


def make_mf(amr, ncomp=1, ngrow=0, extent=8, split=4, dim=2, memory="device"):
    amr.config.set_spacedim(dim)
    dom = amr.Box([0] * dim, [extent - 1] * dim)
    ba = amr.decompose(dom, split)
    return amr.multifab_define(ba, amr.DistributionMapping([0] * len(ba)), ncomp, ngrow, memory=memory)


def test_shape_strides_and_interface():
    amr = _amr()
    from paper_2403_12179_b200.bridge import array_view
    amr.config.set_spacedim(2)
    fab = amr.Fab(amr.Box((0, 0), (3, 3)), 2)
    v = array_view(fab)
    assert v.shape == (4, 4, 1, 2)
    assert v.strides == (8, 32, 128, 128)
    assert v.typestr == "<f8"
    ai = v.__cuda_array_interface__
    assert ai["version"] == 3 and ai["data"] == (v.address, False)
    import torch
    t = torch.as_tensor(v, device="cuda")
    assert t.data_ptr() == fab.data.data_ptr()


def test_zero_copy_mutation_visible_to_exchange():
    amr = _amr()
    from paper_2403_12179_b200.bridge import multifab_iter
    amr.config.set_spacedim(2)
    dom = amr.Box((0, 0), (7, 7))
    geom = amr.Geometry(dom, (0, 0), (1, 1), (True, True))
    ba = amr.decompose(dom, 4)
    mf = amr.multifab_define(ba, amr.DistributionMapping([0] * len(ba)), 1, 1, geom)
    mf.setval(0.0)
    for mfi in multifab_iter(mf):
        t = mfi.to_torch()
        t.fill_(float(mfi.index + 1))  # whole fab incl. ghosts
        g = mfi.fabbox()
        assert mfi.tilebox().grow(mfi.n_grow_vect) == g
    amr.fill_boundary(mf, geom)
    # ghosts now hold the neighbours' values, valid cells their own
    v0 = mf.view(0)
    assert v0[0, 0] == 1.0 and v0[4, 0] == 2.0 and v0[-1, 0] == 2.0


def test_copy_semantics_and_order_duality():
    amr = _amr()
    from paper_2403_12179_b200.bridge import array_view
    amr.config.set_spacedim(3)
    fab = amr.Fab(amr.Box((0, 0, 0), (3, 2, 1)), 2)
    import torch
    ramp = torch.arange(fab.data.numel(), dtype=torch.float64, device="cuda")
    fab.raw().copy_(ramp)
    v = array_view(fab)
    f = v.to_host_array("F")
    c = v.to_host_array("C")
    for x in range(4):
        for y in range(3):
            for z in range(2):
                for comp in range(2):
                    assert f[x, y, z, comp] == c[comp, z, y, x]
    f[...] = -7.0  # a device fab's host array is a copy
    assert float(fab.data.min()) == 0.0
    tf, tc = v.to_torch("F"), v.to_torch("C")
    assert tf.data_ptr() == tc.data_ptr() and tc.shape == (2, 2, 3, 4)


def test_pinned_fab_is_zero_copy_on_host():
    amr = _amr()
    from paper_2403_12179_b200.bridge import multifab_iter
    mf = make_mf(amr, memory="pinned")
    mf.setval(0.0)
    for mfi in multifab_iter(mf):
        arr = mfi.to_host_array(copy=False)
        arr[()] = 42.0
        assert arr.__array_interface__["data"][0] == mf.fab(mfi.index).ptr
    for gi in mf.local_indices:
        assert bool((mf.fabs[gi].data == 42.0).all())
    dup = mfi.to_host_array(copy=True)
    dup[...] = 1.0
    assert bool((mf.fabs[mfi.index].data == 42.0).all())


def test_const_view_read_only_pinned():
    amr = _amr()
    from paper_2403_12179_b200.bridge import BoundArray4
    mf = make_mf(amr, memory="pinned")
    arr = np.asarray(BoundArray4(mf.const_view(mf.local_indices[0])))
    assert not arr.flags.writeable
    with pytest.raises(ValueError):
        arr[0, 0, 0, 0] = 1.0


def test_multifab_iter_detects_structure_change():
    amr = _amr()
    from paper_2403_12179_b200.bridge import multifab_iter
    mf = make_mf(amr)
    with pytest.raises(RuntimeError):
        for n, _ in enumerate(multifab_iter(mf)):
            if n == 0:
                mf.close()
