"""Native plan builder (libghostx, C ABI) against the reference-generated
golden plans and the oracle; host-side plan API semantics.  CPU only: plan
building never touches a device."""

import ctypes as C

import numpy as np
import pytest

import golden_util as gu
from oracle import ghost_oracle as go
from paper_2403_12179_b200 import _native as N


def native_fb(boxes, ngrow, periodic, period, rank_of, nranks):
    boxes = np.ascontiguousarray(np.asarray(boxes, np.int64).reshape(-1, 6))
    h = C.c_void_p()
    N.check(N.lib.ghx_plan_build_fill_boundary(
        len(boxes), N.i64p(boxes), N.i64p(np.asarray(ngrow, np.int64)), N.i32p(np.asarray(periodic, np.int32)),
        N.i64p(np.asarray(period, np.int64)), N.i32p(np.asarray(rank_of, np.int32)), nranks, C.byref(h)))
    return h


def native_pc(db, ngd, sb, ngs, periodic, period, srank, drank, nranks):
    db = np.ascontiguousarray(np.asarray(db, np.int64).reshape(-1, 6))
    sb = np.ascontiguousarray(np.asarray(sb, np.int64).reshape(-1, 6))
    per = None if periodic is None else N.i32p(np.asarray(periodic, np.int32))
    h = C.c_void_p()
    N.check(N.lib.ghx_plan_build_parallel_copy(
        len(db), N.i64p(db), N.i64p(np.asarray(ngd, np.int64)), len(sb), N.i64p(sb),
        N.i64p(np.asarray(ngs, np.int64)), per, N.i64p(np.asarray(period, np.int64)),
        N.i32p(np.asarray(srank, np.int32)), N.i32p(np.asarray(drank, np.int32)), nranks, C.byref(h)))
    return h


def rows(h):
    n = N.lib.ghx_plan_num_segments(h)
    r = np.zeros((n, 13), np.int64)
    if n:
        N.check(N.lib.ghx_plan_get_segments(h, N.i64p(r)))
    return r


def period_of(c):
    return [c["domain"][1][d] - c["domain"][0][d] + 1 for d in range(3)]


@pytest.mark.parametrize("name", gu.names("fill_boundary"))
def test_native_fill_boundary_plan_matches_reference(name):
    c = gu.case(name)
    h = native_fb(c["boxes"], c["ngrow"], c["periodic"], period_of(c), c["rank_of"], c["nranks"])
    try:
        np.testing.assert_array_equal(rows(h), gu.data()[f"{name}/segments"])
    finally:
        N.lib.ghx_plan_free(h)


@pytest.mark.parametrize("name", gu.names("parallel_copy"))
def test_native_parallel_copy_plan_matches_reference(name):
    c = gu.case(name)
    h = native_pc(c["dst_boxes"], c["ngrow_dst"], c["src_boxes"], c["ngrow_src"], c["periodic"], period_of(c),
                  c["src_rank"], c["dst_rank"], c["nranks"])
    try:
        np.testing.assert_array_equal(rows(h), gu.data()[f"{name}/segments"])
    finally:
        N.lib.ghx_plan_free(h)


@pytest.mark.parametrize("name", [c["name"] for c in gu.cases() if c["kind"] == "plan_fill_boundary"])
def test_native_scale_plans_match_reference(name):
    c = gu.case(name)
    n, b, ng, G = c["n"], c["box"], c["ngrow"], c["nranks"]
    boxes = gu.scale_boxes(n, b)
    h = native_fb(boxes, [ng] * 3, [1, 1, 1], [n] * 3, np.arange(len(boxes)) % G, G)
    try:
        r = rows(h)
        assert len(r) == c["num_segments"]
        assert gu.seg_digest(r) == c["seg_sha256"]
        pc = np.zeros(G * G, np.int64)
        N.check(N.lib.ghx_plan_pair_cells(h, N.i64p(pc)))
        pc = pc.reshape(G, G)
        got = {f"{s}->{d}": int(pc[s, d]) * c["ncomp"] * 8 for s in range(G) for d in range(G)
               if s != d and pc[s, d]}
        assert got == c["pair_bytes"]
        assert N.lib.ghx_plan_num_write_tags(h) == len(r)  # cell-centred FB: disjoint writes
    finally:
        N.lib.ghx_plan_free(h)


def test_native_regrid_plan_matches_reference():
    c = gu.case("C5")
    n = c["n"]
    sb, db = gu.scale_boxes(n, c["src_box"]), gu.scale_boxes(n, c["dst_box"])
    G = c["nranks"]
    h = native_pc(db, [0] * 3, sb, [0] * 3, None, [n] * 3, np.arange(len(sb)) % G, np.arange(len(db)) % G, G)
    try:
        assert gu.seg_digest(rows(h)) == c["seg_sha256"]
    finally:
        N.lib.ghx_plan_free(h)


def test_native_matches_oracle_random_periodic_3d():
    rng = np.random.default_rng(5)
    for _ in range(25):
        ext = rng.integers(4, 14, 3)
        # random decomposition via oracle-independent slicing
        cuts = [np.unique(np.concatenate([[0], rng.integers(1, e, rng.integers(0, 3)), [e]])) for e in ext]
        boxes = [[x0, y0, z0, x1 - 1, y1 - 1, z1 - 1]
                 for z0, z1 in zip(cuts[2][:-1], cuts[2][1:])
                 for y0, y1 in zip(cuts[1][:-1], cuts[1][1:])
                 for x0, x1 in zip(cuts[0][:-1], cuts[0][1:])]
        boxes = np.asarray(boxes, np.int64)
        minext = int((boxes[:, 3:] - boxes[:, :3] + 1).min())
        ng = [int(rng.integers(0, minext + 1))] * 3
        per = [bool(v) for v in rng.integers(0, 2, 3)]
        G = int(rng.integers(1, 5))
        ranks = rng.integers(0, G, len(boxes))
        ref = go.plan_fill_boundary(boxes, ng, per, ext, ranks, G)
        h = native_fb(boxes, ng, per, ext, ranks, G)
        try:
            r = rows(h)
            np.testing.assert_array_equal(r[:, :11], ref.segments)
        finally:
            N.lib.ghx_plan_free(h)


def test_c4_native_plan_is_fast():
    import time
    boxes = gu.scale_boxes(256, 16)
    t0 = time.perf_counter()
    h = native_fb(boxes, [2] * 3, [1, 1, 1], [256] * 3, np.zeros(len(boxes)), 1)
    dt = time.perf_counter() - t0
    n = N.lib.ghx_plan_num_segments(h)
    N.lib.ghx_plan_free(h)
    assert n == 106496
    assert dt < 5.0  # the reference needs ~75 s


def test_boxes_disjoint_matches_bruteforce():
    rng = np.random.default_rng(11)
    for _ in range(200):
        n = int(rng.integers(1, 12))
        lo = rng.integers(-6, 6, (n, 3))
        hi = lo + rng.integers(0, 4, (n, 3))
        b = np.ascontiguousarray(np.concatenate([lo, hi], axis=1).astype(np.int64))
        oa, ob = C.c_int64(), C.c_int64()
        N.check(N.lib.ghx_boxes_disjoint(n, N.i64p(b), C.byref(oa), C.byref(ob)))
        first = (-1, -1)
        for i in range(n):
            for j in range(i + 1, n):
                if np.all(np.maximum(lo[i], lo[j]) <= np.minimum(hi[i], hi[j])):
                    first = (i, j)
                    break
            if first[0] >= 0:
                break
        assert (oa.value, ob.value) == first


def test_write_tags_clip_overlapping_parallel_copy():
    """ngrow_src > 0: two sources cover the same dst cells; the later
    writer (reference order) keeps them, earlier ones are clipped."""
    sb = [[0, 0, 0, 3, 0, 0], [4, 0, 0, 7, 0, 0]]
    db = [[0, 0, 0, 7, 0, 0]]
    h = native_pc(db, [0, 0, 0], sb, [1, 0, 0], None, [8, 1, 1], [0, 0], [0], 1)
    try:
        assert N.lib.ghx_plan_num_segments(h) == 2
        assert N.lib.ghx_plan_num_write_tags(h) == 2
        r = rows(h)
        # reference segments overlap on cells 3..4
        assert r[0, 2] == 0 and r[0, 5] == 4 and r[1, 2] == 3 and r[1, 5] == 7
    finally:
        N.lib.ghx_plan_free(h)
