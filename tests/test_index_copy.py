"""index_mapped_copy (reference comm.py:465-560): the oracle against fixtures
from the reference (CPU) and the CUDA path against the same fixtures and the
reference's own known-answer tests (GPU)."""

import numpy as np
import pytest

from oracle import ghost_oracle as go
from oracle import inputs
from test_amr_oracle import case, data, grown, hashed, meta, names

MAPPINGS = {
    "identity": lambda n: (lambda i, j, k: (i, j, k)),
    "reflect_x": lambda n: (lambda i, j, k: (n[0] - 1 - i, j, k)),
    "shift_wrap": lambda n: (lambda i, j, k: ((i + 3) % n[0], (j + 5) % n[1], k)),
    "transpose_xy": lambda n: (lambda i, j, k: (j, i, k)),
}


def _g3(v, dim):
    return [v if d < dim else 0 for d in range(3)]


def _inputs(c):
    dim, nc, dt = c["dim"], c["ncomp"], np.dtype(c["dtype"])
    dom = np.asarray([0, 0, 0] + [e - 1 for e in c["ext"]], np.int64)
    src = {gi: hashed(grown(b, _g3(c["sng"], dim)), np.asarray(b), dom, nc, dt, inputs.SEED)
           for gi, b in enumerate(c["src_boxes"])}
    dst = {gi: hashed(grown(b, _g3(c["dng"], dim)), np.asarray(b), dom, nc, dt, meta()["seed_crse"])
           for gi, b in enumerate(c["dst_boxes"])}
    return src, dst


@pytest.mark.parametrize("name", names("index_copy"))
def test_index_copy_oracle_matches_reference(name):
    c = case(name)
    dim = c["dim"]
    src, dst = _inputs(c)
    region = None if c["region"] is None else np.asarray(c["region"][0] + c["region"][1], np.int64)
    go.index_copy(c["dst_boxes"], dst, {gi: grown(b, _g3(c["dng"], dim))[:3] for gi, b in enumerate(c["dst_boxes"])},
                  c["src_boxes"], src, {gi: grown(b, _g3(c["sng"], dim))[:3] for gi, b in enumerate(c["src_boxes"])},
                  MAPPINGS[c["mapping"]](c["ext"]), region)
    for gi, a in dst.items():
        assert np.array_equal(inputs.bits(a), data()[f"{name}/dst{gi}"]), gi


@pytest.mark.gpu
@pytest.mark.parametrize("name", names("index_copy"))
def test_index_mapped_copy_bit_exact(name):
    import paper_2403_12179_b200 as amr
    from gpu_util import bits_of, upload
    c = case(name)
    dim, nc, dt = c["dim"], c["ncomp"], np.dtype(c["dtype"])
    amr.config.set_spacedim(dim)
    amr.config.set_real_dtype(dt)
    box = lambda b6: amr.Box(tuple(b6[:dim]), tuple(b6[3:3 + dim]))  # noqa: E731
    sba = amr.BoxArray([box(b) for b in c["src_boxes"]])
    dba = amr.BoxArray([box(b) for b in c["dst_boxes"]])
    sdm = amr.DistributionMapping(c["src_rank"], c["nranks"])
    ddm = amr.DistributionMapping(c["dst_rank"], c["nranks"])
    hsrc, hdst = _inputs(c)
    region = None if c["region"] is None else amr.Box(tuple(c["region"][0][:dim]), tuple(c["region"][1][:dim]))
    fn = MAPPINGS[c["mapping"]](c["ext"])

    def program(ctx):
        src = amr.MultiFab(sba, sdm, nc, c["sng"])
        dst = amr.MultiFab(dba, ddm, nc, c["dng"])
        for gi in src.local_indices:
            upload(src.fabs[gi], hsrc[gi])
        for gi in dst.local_indices:
            upload(dst.fabs[gi], hdst[gi])
        ctx.barrier()
        s0 = ctx.bus.stats_snapshot()
        ctx.barrier()
        amr.index_mapped_copy(dst, src, fn, region=region)
        ctx.barrier()
        s1 = ctx.bus.stats_snapshot()
        stats = {f"{a}->{b}": [s1[(a, b)][0] - s0[(a, b)][0], s1[(a, b)][1] - s0[(a, b)][1]]
                 for (a, b) in s1 if s1[(a, b)] != s0[(a, b)]}
        return {gi: bits_of(dst.fabs[gi]) for gi in dst.local_indices}, stats

    res = amr.runtime_spawn(c["nranks"], program)
    for out, _ in res:
        for gi, a in out.items():
            assert np.array_equal(a, data()[f"{name}/dst{gi}"].ravel(order="F")), gi
    assert res[0][1] == {k: list(v) for k, v in c["stats"].items()}


@pytest.mark.gpu
def test_index_mapped_copy_known_answers():
    """Reference tests/test_comm.py:283-330: identity == parallel_copy,
    reflection, 90-degree rotation; uncovered mapping raises."""
    import paper_2403_12179_b200 as amr
    from gpu_util import bits_of
    amr.config.set_spacedim(2)
    ba = amr.BoxArray([amr.Box((0, 0), (7, 7))])
    dm = amr.DistributionMapping([0])
    src = amr.MultiFab(ba, dm, 1, 0)
    dst = amr.MultiFab(ba, dm, 1, 0)
    rng = np.random.default_rng(6)
    g = rng.random((8, 8))
    src.fabs[0].data[:, :, 0, 0] = __import__("torch").from_numpy(g).to(src.fabs[0].data.device)
    amr.index_mapped_copy(dst, src, lambda i, j, k: (j, 7 - i, k))
    got = dst.fabs[0].data[:, :, 0, 0].cpu().numpy()
    expect = np.array([[g[j, 7 - i] for j in range(8)] for i in range(8)])
    assert np.array_equal(got, expect)
    d2 = amr.MultiFab(ba, dm, 1, 0)
    amr.index_mapped_copy(d2, src, lambda i, j, k: (i, j, k))
    d1 = amr.MultiFab(ba, dm, 1, 0)
    amr.parallel_copy(d1, src)
    assert np.array_equal(bits_of(d1.fabs[0]), bits_of(d2.fabs[0]))
    with pytest.raises(ValueError):
        amr.index_mapped_copy(dst, src, lambda i, j, k: (i + 1, j, k))
