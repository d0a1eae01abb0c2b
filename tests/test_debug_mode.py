"""Debug-mode parity (reference config.py:16-21, mesh.py:59-60, :172-174).

With ``config.debug`` on, fresh fabs hold the reference's poison: the
float64 signalling NaN 0x7FF40000DEADBEEF, and for float32 storage numpy's
narrowing of it (0x7FE00006).  Uncoverable ghost cells keep those bits
through FillBoundary / ParallelCopy.  The fixtures come from the reference
itself (tests/golden/make_golden_debug.py).  CPU tests pin the constants and
the oracle; ``-m gpu`` tests run the CUDA path through the public API and
compare every fab bit for bit.
"""

import functools
import json
import os

import numpy as np
import pytest

import golden_util as gu
from oracle import ghost_oracle as go
from oracle import inputs

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@functools.lru_cache(maxsize=1)
def meta():
    with open(os.path.join(HERE, "golden_debug.json")) as f:
        return json.load(f)


@functools.lru_cache(maxsize=1)
def data():
    return dict(np.load(os.path.join(HERE, "golden_debug.npz")))


def names(kind):
    return [c["name"] for c in meta()["cases"] if c["kind"] == kind]


def case(name):
    return next(c for c in meta()["cases"] if c["name"] == name)


def _valid_filled(c, gi, box, grow, fresh):
    """The reference's pre-call fab: debug poison, hash values on valid cells."""
    dt = np.dtype(c["dtype"])
    b = np.asarray(box, np.int64)
    g = gu.grown(b, grow)
    shape = tuple(int(v) for v in g[3:] - g[:3] + 1) + (c["ncomp"],)
    arr = np.empty(shape, dt, order="F")
    inputs.bits(arr)[...] = fresh
    ext = c["ext"]
    tmp = inputs.make_fab(b[:3], b[3:], c["ncomp"], dt, b[:3], b[3:], [0, 0, 0], [e - 1 for e in ext])
    sl = tuple(slice(int(b[d] - g[d]), int(b[3 + d] - g[d] + 1)) for d in range(3))
    arr[sl] = tmp
    return arr, g[:3]


def test_poison_constants_match_reference():
    from paper_2403_12179_b200 import config
    assert config.POISON_BITS32 == meta()["poison32_bits"] == 0x7FE00006
    assert config.POISON_BITS64 == 0x7FF40000DEADBEEF
    for c in meta()["cases"]:
        if c["kind"] != "fill_boundary":
            continue
        word = config.poison_bits(np.dtype(c["dtype"]).itemsize)
        for k, v in data().items():
            if k.startswith(c["name"] + "/fresh"):
                assert (v == word).all(), k


@pytest.mark.parametrize("name", names("fill_boundary"))
def test_oracle_debug_fill_boundary_matches_reference(name):
    c, d = case(name), data()
    boxes = np.asarray(c["boxes"], np.int64)
    plan = go.plan_fill_boundary(boxes, c["ngrow"], c["periodic"], c["ext"], c["rank_of"], c["nranks"])
    fabs, lo = {}, {}
    for gi, b in enumerate(boxes):
        fabs[gi], lo[gi] = _valid_filled(c, gi, b, c["ngrow"], d[f"{name}/fresh{gi}"])
    st = go.execute(plan, fabs, lo, fabs, lo, 0, 0, c["ncomp"])
    for gi in fabs:
        np.testing.assert_array_equal(inputs.bits(fabs[gi]), d[f"{name}/fab{gi}"])
    assert {k: tuple(v) for k, v in st.items()} == gu.stats_dict(d[f"{name}/stats"])


def test_fabview_debug_vector_bounds():
    """Debug builds reject out-of-range vector indices (reference mesh.py:172-174);
    the check only needs host logic, so a CPU tensor stands in for the fab."""
    import torch
    from paper_2403_12179_b200 import config
    from paper_2403_12179_b200.mesh import FabView
    a = torch.arange(4 * 3 * 2, dtype=torch.float64).reshape(4, 3, 2, 1)
    v = FabView(a, (10, 0, 0), 1, True)
    idx = np.asarray([10, 13])
    want = [float(a[0, 0, 0, 0]), float(a[3, 0, 0, 0])]
    assert v[idx, 0, 0].tolist() == want
    bad = np.asarray([9, 10])  # global 9 is local -1: wraps silently without debug
    assert v[bad, 0, 0].tolist() == want[::-1]
    old = config.debug
    config.set_debug(True)
    try:
        with pytest.raises(IndexError):
            v[bad, 0, 0]
        with pytest.raises(IndexError):
            v[10, np.asarray([0, 3]), 0]
        assert v[idx, 0, 0].tolist() == want
    finally:
        config.set_debug(old)


# ------------------------------------------------------------------- CUDA path

def _setup(amr, c):
    amr.config.set_spacedim(c["dim"])
    amr.config.set_real_dtype(np.dtype(c["dtype"]))
    amr.config.set_debug(True)


def _restore(amr):
    amr.config.set_debug(False)
    amr.config.set_spacedim(3)
    amr.config.set_real_dtype(np.float64)


@pytest.mark.gpu
@pytest.mark.parametrize("name", names("fill_boundary"))
def test_gpu_debug_fill_boundary_matches_reference(name):
    import paper_2403_12179_b200 as amr
    from gpu_util import bits_of, upload
    c, d = case(name), data()
    dim = c["dim"]
    _setup(amr, c)
    try:
        ba = amr.BoxArray([amr.Box(r[:dim], r[3:3 + dim]) for r in c["boxes"]])
        dm = amr.DistributionMapping(c["rank_of"], c["nranks"])
        geom = amr.Geometry(amr.Box([0] * dim, [e - 1 for e in c["ext"][:dim]]), [0.0] * dim, [1.0] * dim,
                            c["periodic"][:dim])

        def program(ctx):
            mf = amr.MultiFab(ba, dm, c["ncomp"], c["ngrow"][0], geom)
            for gi in mf.local_indices:
                # the fresh device fab carries the reference's debug poison
                np.testing.assert_array_equal(bits_of(mf.fabs[gi]), d[f"{name}/fresh{gi}"].ravel(order="F"))
                arr, _ = _valid_filled(c, gi, c["boxes"][gi], c["ngrow"], d[f"{name}/fresh{gi}"])
                upload(mf.fabs[gi], arr)
            ctx.barrier()
            s0 = ctx.bus.stats_snapshot()
            ctx.barrier()
            amr.fill_boundary(mf, geom)
            ctx.barrier()
            s1 = ctx.bus.stats_snapshot()
            out = {gi: bits_of(mf.fabs[gi]) for gi in mf.local_indices}
            return out, {k: (s1[k][0] - s0[k][0], s1[k][1] - s0[k][1]) for k in s1 if s1[k] != s0[k]}

        res = amr.runtime_spawn(c["nranks"], program)
        for out, stats in res:
            for gi, got in out.items():
                np.testing.assert_array_equal(got, d[f"{name}/fab{gi}"].ravel(order="F"), err_msg=f"fab {gi}")
        if c["nranks"] > 1:
            assert res[0][1] == gu.stats_dict(d[f"{name}/stats"])
    finally:
        _restore(amr)


@pytest.mark.gpu
@pytest.mark.parametrize("name", names("parallel_copy"))
def test_gpu_debug_parallel_copy_matches_reference(name):
    import paper_2403_12179_b200 as amr
    from gpu_util import bits_of, upload
    c, d = case(name), data()
    dim = c["dim"]
    _setup(amr, c)
    try:
        sba = amr.BoxArray([amr.Box(r[:dim], r[3:3 + dim]) for r in c["src_boxes"]])
        dba = amr.BoxArray([amr.Box(r[:dim], r[3:3 + dim]) for r in c["dst_boxes"]])
        sdm = amr.DistributionMapping(c["src_rank"], c["nranks"])
        ddm = amr.DistributionMapping(c["dst_rank"], c["nranks"])
        dt = np.dtype(c["dtype"])
        word = amr.config.poison_bits(dt.itemsize)

        def program(ctx):
            src = amr.MultiFab(sba, sdm, c["ncomp"], 0)
            dst = amr.MultiFab(dba, ddm, c["ncomp"], c["ngrow_dst"][0])
            for gi in src.local_indices:
                b = np.asarray(c["src_boxes"][gi], np.int64)
                upload(src.fabs[gi], inputs.make_fab(b[:3], b[3:], c["ncomp"], dt, b[:3], b[3:], [0, 0, 0],
                                                     [e - 1 for e in c["ext"]]))
            for gi in dst.local_indices:
                assert (bits_of(dst.fabs[gi]) == word).all()
            ctx.barrier()
            s0 = ctx.bus.stats_snapshot()
            ctx.barrier()
            amr.parallel_copy(dst, src, ngrow_dst=c["ngrow_dst"][0])
            ctx.barrier()
            s1 = ctx.bus.stats_snapshot()
            out = {gi: bits_of(dst.fabs[gi]) for gi in dst.local_indices}
            return out, {k: (s1[k][0] - s0[k][0], s1[k][1] - s0[k][1]) for k in s1 if s1[k] != s0[k]}

        res = amr.runtime_spawn(c["nranks"], program)
        for out, stats in res:
            for gi, got in out.items():
                np.testing.assert_array_equal(got, d[f"{name}/fab{gi}"].ravel(order="F"), err_msg=f"fab {gi}")
        assert res[0][1] == gu.stats_dict(d[f"{name}/stats"])
    finally:
        _restore(amr)


def _debug_arena_roundtrip(memory):
    from paper_2403_12179_b200 import config
    from paper_2403_12179_b200.arena import Arena
    prev = config.debug
    config.debug = True
    try:
        a = Arena(1 << 16, memory=memory)
        blk = a.alloc(4096)
        ptr, padded = blk.ptr, blk.padded
        view = blk.as_array(np.uint8, padded)
        view[:] = 7
        a.free(blk)
        if memory == "device":
            import torch
            torch.cuda.synchronize()
            got = view.cpu().numpy()
        else:
            got = np.asarray(view)
        assert got.size == padded and (got == 0xAB).all()  # freed bytes scribbled (reference arena.py:157-161)
        again = a.alloc(4096)
        assert again.ptr == ptr  # the pool hands the scribbled block back
        with pytest.raises(RuntimeError, match="double free"):
            a.free(blk)
    finally:
        config.debug = prev


def test_debug_arena_scribbles_freed_host_blocks():
    _debug_arena_roundtrip("host")


@pytest.mark.gpu
def test_debug_arena_scribbles_freed_device_blocks():
    _debug_arena_roundtrip("device")
