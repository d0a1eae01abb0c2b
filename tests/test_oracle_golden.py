"""Pin the CPU oracle (oracle/ghost_oracle.py) against fixtures produced by
running the reference implementation itself (tests/golden/make_golden.py),
and against the reference's own known-answer tests.  CPU only."""

import numpy as np
import pytest

import golden_util as gu
from oracle import ghost_oracle as go
from oracle import inputs


def _fb_oracle(c):
    boxes = np.asarray(c["boxes"], np.int64)
    period = [c["domain"][1][d] - c["domain"][0][d] + 1 for d in range(3)]
    plan = go.plan_fill_boundary(boxes, c["ngrow"], c["periodic"], period, c["rank_of"],
                                 c["nranks"])
    return boxes, plan


def _rows13(plan, src_rank, dst_rank):
    s = plan.segments
    return np.concatenate([s, np.asarray(src_rank)[s[:, 0]][:, None],
                           np.asarray(dst_rank)[s[:, 1]][:, None]], axis=1)


@pytest.mark.parametrize("name", gu.names("fill_boundary"))
def test_oracle_fill_boundary_matches_reference(name):
    c = gu.case(name)
    d = gu.data()
    boxes, plan = _fb_oracle(c)
    assert plan.num_segments == c["num_segments"]
    np.testing.assert_array_equal(_rows13(plan, c["rank_of"], c["rank_of"]), d[f"{name}/segments"])
    dtype = np.dtype(c["dtype"])
    fabs, lo = {}, {}
    hd = c["hash_domain"]
    for gi, b in enumerate(boxes):
        g = gu.grown(b, c["ngrow"])
        fabs[gi] = inputs.make_fab(g[:3], g[3:], c["ncomp"], dtype, b[:3], b[3:], hd[0], hd[1])
        lo[gi] = g[:3]
    total = {}
    for _ in range(c["calls"]):
        st = go.execute(plan, fabs, lo, fabs, lo, 0, 0, c["ncomp"])
        for k, v in st.items():
            t = total.setdefault(k, [0, 0])
            t[0] += v[0]
            t[1] += v[1]
    assert {k: tuple(v) for k, v in total.items()} == gu.stats_dict(d[f"{name}/stats"])
    for gi in fabs:
        got = inputs.bits(fabs[gi])
        if c["store"] == "bits":
            np.testing.assert_array_equal(got, d[f"{name}/fab{gi}"])
        else:
            assert gu.fab_digest(got) == c["fab_sha256"][str(gi)]


@pytest.mark.parametrize("name", gu.names("parallel_copy"))
def test_oracle_parallel_copy_matches_reference(name):
    c = gu.case(name)
    d = gu.data()
    sb = np.asarray(c["src_boxes"], np.int64)
    db = np.asarray(c["dst_boxes"], np.int64)
    per = c["periodic"]
    period = [c["domain"][1][k] - c["domain"][0][k] + 1 for k in range(3)]
    plan = go.plan_parallel_copy(db, sb, c["ngrow_dst"], c["ngrow_src"], per, period,
                                 c["src_rank"], c["dst_rank"], c["nranks"])
    assert plan.num_segments == c["num_segments"]
    np.testing.assert_array_equal(_rows13(plan, c["src_rank"], c["dst_rank"]), d[f"{name}/segments"])
    dtype = np.dtype(c["dtype"])
    hd = c["hash_domain"]
    src, slo, dst, dlo = {}, {}, {}, {}
    for gi, b in enumerate(sb):
        g = gu.grown(b, c["src_ngrow"])
        src[gi] = inputs.make_fab(g[:3], g[3:], c["src_ncomp"], dtype, b[:3], b[3:], hd[0], hd[1],
                                  ghost_tag=gi + 1)
        slo[gi] = g[:3]
    for gi, b in enumerate(db):
        g = gu.grown(b, c["dst_ngrow"])
        dst[gi] = inputs.make_fab(g[:3], g[3:], c["dst_ncomp"], dtype, b[:3], b[3:], hd[0], hd[1],
                                  seed=inputs.SEED + 1)
        dlo[gi] = g[:3]
    st = go.execute(plan, src, slo, dst, dlo, c["scomp"], c["dcomp"], c["ncomp"])
    assert st == gu.stats_dict(d[f"{name}/stats"])
    for gi in dst:
        np.testing.assert_array_equal(inputs.bits(dst[gi]), d[f"{name}/fab{gi}"])


@pytest.mark.parametrize("name", [c["name"] for c in gu.cases() if c["kind"] == "plan_fill_boundary"])
def test_oracle_scale_plans_match_reference(name):
    c = gu.case(name)
    n, b, ng, G = c["n"], c["box"], c["ngrow"], c["nranks"]
    boxes = gu.scale_boxes(n, b)
    rank_of = np.arange(len(boxes)) % G
    plan = go.plan_fill_boundary(boxes, [ng] * 3, [True] * 3, [n] * 3, rank_of, G)
    assert plan.num_segments == c["num_segments"]
    rows = _rows13(plan, rank_of, rank_of)
    assert gu.seg_digest(rows) == c["seg_sha256"]
    pair_bytes = {f"{s}->{d}": int((segs[:, 5:8] - segs[:, 2:5] + 1).prod(axis=1).sum()) * c["ncomp"] * 8
                  for (s, d), segs in plan.pair_segments.items()}
    assert pair_bytes == c["pair_bytes"]


def test_oracle_regrid_plan_matches_reference():
    c = gu.case("C5")
    n = c["n"]
    sb = gu.scale_boxes(n, c["src_box"])
    db = gu.scale_boxes(n, c["dst_box"])
    G = c["nranks"]
    plan = go.plan_parallel_copy(db, sb, [0] * 3, [0] * 3, None, [n] * 3,
                                 np.arange(len(sb)) % G, np.arange(len(db)) % G, G)
    assert plan.num_segments == c["num_segments"]
    rows = _rows13(plan, np.arange(len(sb)) % G, np.arange(len(db)) % G)
    assert gu.seg_digest(rows) == c["seg_sha256"]


def test_oracle_known_values_1d():
    """Reference tests/test_comm.py:198-210: data(i)=i on [0..7], periodic,
    two boxes, ngrow 1 -> fab0 ghost(-1)=7, ghost(4)=4; fab1 ghost(3)=3,
    ghost(8)=0; and tests/test_comm.py:168-177: 4 segments."""
    boxes = np.array([[0, 0, 0, 3, 0, 0], [4, 0, 0, 7, 0, 0]])
    plan = go.plan_fill_boundary(boxes, [1, 0, 0], [True, False, False], [8, 1, 1], [0, 0], 1)
    assert plan.num_segments == 4
    fabs = {0: np.zeros((6, 1, 1, 1), order="F"), 1: np.zeros((6, 1, 1, 1), order="F")}
    lo = {0: np.array([-1, 0, 0]), 1: np.array([3, 0, 0])}
    for gi in (0, 1):
        for i in range(boxes[gi, 0], boxes[gi, 3] + 1):
            fabs[gi][i - lo[gi][0], 0, 0, 0] = float(i)
    go.execute(plan, fabs, lo, fabs, lo, 0, 0, 1)
    assert (fabs[0][0, 0, 0, 0], fabs[0][5, 0, 0, 0]) == (7.0, 4.0)
    assert (fabs[1][0, 0, 0, 0], fabs[1][5, 0, 0, 0]) == (3.0, 0.0)


def test_oracle_ngrow_zero_is_empty():
    boxes = np.array([[0, 0, 0, 3, 0, 0], [4, 0, 0, 7, 0, 0]])
    plan = go.plan_fill_boundary(boxes, [0, 0, 0], [True, False, False], [8, 1, 1], [0, 0], 1)
    assert plan.num_segments == 0


def test_box_diff_partition_property():
    rng = np.random.default_rng(3)
    for _ in range(300):
        a = np.concatenate([rng.integers(-5, 5, 3), np.zeros(3, np.int64)])
        a[3:] = a[:3] + rng.integers(0, 6, 3)
        b = np.concatenate([rng.integers(-5, 5, 3), np.zeros(3, np.int64)])
        b[3:] = b[:3] + rng.integers(0, 6, 3)
        parts = go.box_diff(a, b)
        lo = np.maximum(a[:3], b[:3])
        hi = np.minimum(a[3:], b[3:])
        inter = int(np.prod(np.maximum(hi - lo + 1, 0)))
        vol = lambda x: int(np.prod(x[3:] - x[:3] + 1))  # noqa: E731
        assert vol(a) == inter + sum(vol(p) for p in parts)


def test_inputs_hash_known_values():
    # splitmix64 reference outputs for seed 0 sequence (public algorithm constants)
    assert int(inputs.splitmix64(np.uint64(0))) == 0xE220A8397B1DCDAF
    assert int(inputs.splitmix64(np.uint64(1))) == 0x910A2DEC89025CC1
