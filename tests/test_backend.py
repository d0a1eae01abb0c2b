"""The reference's backend handle (kernels.Backend) on the exchange API:
accepted for signature compatibility, "gpu" and other kinds raise like the
reference (tests/test_kernels.py:202-205), and launch_counter counts the
device launches of each call."""

import pytest

import paper_2403_12179_b200 as amr
from paper_2403_12179_b200 import kernels


def test_backend_kinds():
    assert kernels.Backend().kind == kernels.SERIAL
    assert kernels.Backend(kernels.CPU_PARALLEL, 3).nworkers == 3
    with pytest.raises(ValueError):
        kernels.Backend("gpu")
    with pytest.raises(ValueError):
        kernels.Backend(kernels.SERIAL, -1)
    b = kernels.Backend()
    kernels.set_default_backend(b)
    assert kernels.default_backend() is b


@pytest.mark.gpu
def test_backend_launch_counter_single_rank():
    amr.config.set_spacedim(3)
    dom = amr.Box((0, 0, 0), (31, 31, 31))
    geom = amr.Geometry(dom, (0.0,) * 3, (1.0,) * 3, (True,) * 3)
    ba = amr.decompose(dom, 16)
    dm = amr.DistributionMapping.round_robin(len(ba), 1)
    mf = amr.MultiFab(ba, dm, 2, 1, geom)
    mf.setval(1.0)
    b = kernels.Backend(kernels.CPU_PARALLEL)
    amr.fill_boundary(mf, geom, backend=b)
    assert b.launch_counter == 1  # one fused launch; the reference's single local phase is one dispatch too
    src = amr.MultiFab(ba, dm, 2, 0)
    src.setval(2.0)
    amr.parallel_copy(mf, src, backend=b)
    assert b.launch_counter == 2
    amr.fill_boundary(mf, geom)  # no backend: nothing counted
    assert b.launch_counter == 2


@pytest.mark.gpu
def test_cached_exchanges_do_not_keep_sources_alive():
    """A long-lived destination copied from a fresh source each call (a
    regrid loop) must not accumulate the sources' device memory: the
    cached executors evict themselves when their source is collected."""
    import gc
    import weakref
    import torch
    amr.config.set_spacedim(3)
    dom = amr.Box((0, 0, 0), (31, 31, 31))
    geom = amr.Geometry(dom, (0.0,) * 3, (1.0,) * 3, (True,) * 3)
    ba = amr.decompose(dom, 16)
    dm = amr.DistributionMapping.round_robin(len(ba), 1)
    dst = amr.MultiFab(ba, dm, 1, 1, geom)
    refs = []
    for it in range(4):
        src = amr.MultiFab(amr.decompose(dom, 8), amr.DistributionMapping.round_robin(64, 1), 1, 0)
        src.setval(float(it))
        amr.parallel_copy(dst, src)
        assert float(dst.fabs[0].data[2, 2, 2, 0]) == float(it)
        refs.append(weakref.ref(src))
        del src
        gc.collect()
    torch.cuda.synchronize()
    assert all(r() is None for r in refs)
    assert sum(1 for k in dst._peer_cache if isinstance(k, tuple) and k[0] == "xchg") == 0
    amr.fill_boundary(dst, geom)  # still works after the evictions


@pytest.mark.gpu
def test_closed_multifab_raises_instead_of_touching_freed_memory():
    amr.config.set_spacedim(3)
    dom = amr.Box((0, 0, 0), (15, 15, 15))
    geom = amr.Geometry(dom, (0.0,) * 3, (1.0,) * 3, (True,) * 3)
    ba = amr.decompose(dom, 8)
    dm = amr.DistributionMapping.round_robin(len(ba), 1)
    mf = amr.MultiFab(ba, dm, 1, 1, geom)
    other = amr.MultiFab(ba, dm, 1, 1, geom)
    amr.fill_boundary(mf, geom)  # plan + executor cached
    amr.parallel_copy(other, mf)
    mf.close()
    with pytest.raises(ValueError):
        amr.fill_boundary(mf, geom)
    with pytest.raises(ValueError):
        amr.parallel_copy(other, mf)
    amr.fill_boundary(other, geom)  # unaffected
