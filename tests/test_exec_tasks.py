"""Executor task building (host only, no GPU): which task kinds the fused
kernel gets for the benchmark layouts -- x-line chains for large fabs,
fab-ordered per-tag sector swaps for small fabs, seam-chunk rings for
host-memory executors of periodic x-lines (and not for open ones)."""

import ctypes as C

import numpy as np
import pytest

import golden_util as gu
from paper_2403_12179_b200 import _native as N
from test_plan_native import native_fb


def kinds(n, b, nc, ng, periodic=(1, 1, 1), ring=False):
    boxes = gu.scale_boxes(n, b)
    h = native_fb(boxes, [ng] * 3, list(periodic), [n] * 3, [0] * len(boxes), 1)
    storage = boxes.copy()
    storage[:, :3] -= ng
    storage[:, 3:] += ng
    storage = np.ascontiguousarray(storage)
    ex = C.c_void_p()
    try:
        N.check(N.lib.ghx_exec_create(h, 0, N.EXEC_DIRECT, N.i64p(storage), nc, N.i64p(storage), nc, 0, 0, nc, 8, 0,
                                      C.byref(ex)))
        if ring:
            N.check(N.lib.ghx_exec_set_ring(ex, 1))
        out = np.zeros(6, np.int64)
        N.check(N.lib.ghx_exec_task_kinds(ex, N.i64p(out)))
        return dict(zip(("copy", "swap", "chain", "ring", "ring_mode", "fab_local"), (int(v) for v in out)))
    finally:
        if ex:
            N.lib.ghx_exec_free(ex)
        N.lib.ghx_plan_free(h)


def test_large_fabs_use_xline_chains():
    k = kinds(512, 128, 8, 2)  # C3: 147 MB fabs
    assert k["fab_local"] == 0 and k["chain"] > 0 and k["swap"] == 0 and k["ring"] == 0


@pytest.mark.parametrize("n,b", [(256, 64), (256, 16)])
def test_small_fabs_use_fab_ordered_swaps(n, b):
    k = kinds(n, b, 4, 2)  # C2 / C4
    assert k["fab_local"] == 1 and k["chain"] == 0 and k["swap"] > 0 and k["ring"] == 0


def test_ring_tasks_for_periodic_xlines():
    k = kinds(256, 64, 4, 2, ring=True)
    assert k["ring_mode"] == 1 and k["ring"] > 0 and k["swap"] == 0 and k["chain"] == 0
    # tile ring tasks: 16 x-lines of 4 fabs, one task per (z, comp) column and
    # balanced range of the 65 seam chunks (rows -1 .. 63): at most 8 steps of
    # 16/4 = 4 chunks -> 3 tasks of 22 / 22 / 21 chunks per column
    nch, per = 64 + 1, 8 * (16 // 4)
    assert k["ring"] == 16 * (64 * 4) * (-(-nch // per))


def test_open_xlines_fall_back_to_swaps():
    k = kinds(256, 64, 4, 2, periodic=(0, 1, 1), ring=True)
    assert k["ring"] == 0 and k["swap"] > 0


def test_set_ring_rebuilds_tasks_only_before_first_run():
    k0 = kinds(256, 64, 4, 2, ring=False)
    k1 = kinds(256, 64, 4, 2, ring=True)
    assert k0["copy"] == k1["copy"]  # face copies unchanged; seams change form


def phases(boxes, n, ng, nc, periodic, ranks=None, nranks=1, phased=True, rank=0):
    ranks = [0] * len(boxes) if ranks is None else ranks
    h = native_fb(boxes, [ng] * 3, list(periodic), [n] * 3, ranks, nranks)
    storage = boxes.copy()
    storage[:, :3] -= ng
    storage[:, 3:] += ng
    storage = np.ascontiguousarray(storage)
    ex = C.c_void_p()
    try:
        kind = N.EXEC_DIRECT | (N.EXEC_PHASED if phased else 0)
        N.check(N.lib.ghx_exec_create(h, rank, kind, N.i64p(storage), nc, N.i64p(storage), nc, 0, 0, nc, 8, 0,
                                      C.byref(ex)))
        ph = np.zeros(4, np.int64)
        N.check(N.lib.ghx_exec_phases(ex, N.i64p(ph)))
        a = [C.c_int64() for _ in range(4)]
        N.check(N.lib.ghx_exec_info(ex, *[C.byref(v) for v in a]))
        return dict(phased=int(ph[0]), pe0=int(ph[1]), pe1=int(ph[2]), tags=int(ph[3]), tasks=a[1].value,
                    elems=a[2].value)
    finally:
        if ex:
            N.lib.ghx_exec_free(ex)
        N.lib.ghx_plan_free(h)


@pytest.mark.parametrize("n,b,nc,ng", [(512, 128, 8, 2), (256, 64, 4, 2), (64, 32, 1, 1), (256, 16, 4, 2)])
def test_phased_exchange_drops_edge_and_corner_tags(n, b, nc, ng):
    """Uniform periodic layouts: every fab's faces are extended over the
    lower-axis ghosts, so only the 6 face tags per fab remain (x faces: two
    tags per side pair), moving exactly the same ghost elements."""
    boxes = gu.scale_boxes(n, b)
    p = phases(boxes, n, ng, nc, (1, 1, 1))
    q = phases(boxes, n, ng, nc, (1, 1, 1), phased=False)
    assert p["phased"] == 1 and q["phased"] == 0
    assert p["elems"] == q["elems"]
    assert p["tags"] < q["tags"]
    assert 0 < p["pe0"] <= p["pe1"] < p["tasks"]


@pytest.mark.parametrize("periodic", [(0, 1, 1), (1, 0, 1), (0, 0, 0), (1, 1, 0)])
def test_phased_exchange_keeps_element_count_with_physical_boundaries(periodic):
    # fabs at a non-periodic face keep their own tags where an extension
    # would reach uncovered ghosts; the element count never changes
    boxes = gu.scale_boxes(256, 64)
    p = phases(boxes, 256, 2, 2, periodic)
    q = phases(boxes, 256, 2, 2, periodic, phased=False)
    assert p["elems"] == q["elems"] and p["tags"] <= q["tags"]


def test_phased_exchange_irregular_boxes_keep_element_count():
    rng = np.random.default_rng(7)
    for _ in range(20):
        # random slab cuts of a 48^3 domain (irregular neighbours)
        cuts = [np.unique(np.concatenate([[0, 48], rng.integers(4, 44, size=2)])) for _ in range(3)]
        boxes = np.asarray([[x0, y0, z0, x1 - 1, y1 - 1, z1 - 1]
                            for z0, z1 in zip(cuts[2][:-1], cuts[2][1:])
                            for y0, y1 in zip(cuts[1][:-1], cuts[1][1:])
                            for x0, x1 in zip(cuts[0][:-1], cuts[0][1:])], np.int64)
        for per in [(1, 1, 1), (0, 1, 0)]:
            p = phases(boxes, 48, 2, 1, per)
            q = phases(boxes, 48, 2, 1, per, phased=False)
            assert p["elems"] == q["elems"]


def test_phased_exchange_needs_all_tags_local():
    boxes = gu.scale_boxes(256, 64)
    ranks = [i % 2 for i in range(len(boxes))]
    p = phases(boxes, 256, 2, 2, (1, 1, 1), ranks=ranks, nranks=2)
    assert p["phased"] == 0


@pytest.mark.parametrize("n,b,nc,ng", [(512, 128, 8, 2), (256, 64, 4, 2), (256, 16, 4, 2)])
def test_diagnostic_xface_split_partitions_the_exchange(n, b, nc, ng):
    """bench.py's same-layout direction split: the x-face tags and the rest
    are disjoint halves of the exchange (their elements add up)."""
    boxes = gu.scale_boxes(n, b)
    h = native_fb(boxes, [ng] * 3, [1, 1, 1], [n] * 3, [0] * len(boxes), 1)
    storage = boxes.copy()
    storage[:, :3] -= ng
    storage[:, 3:] += ng
    storage = np.ascontiguousarray(storage)
    elems = {}
    try:
        for name, flag in (("all", 0), ("x", N.EXEC_ONLY_XFACES), ("rest", N.EXEC_NO_XFACES)):
            ex = C.c_void_p()
            N.check(N.lib.ghx_exec_create(h, 0, N.EXEC_DIRECT | flag, N.i64p(storage), nc, N.i64p(storage), nc, 0, 0,
                                          nc, 8, 0, C.byref(ex)))
            a = [C.c_int64() for _ in range(4)]
            N.check(N.lib.ghx_exec_info(ex, *[C.byref(v) for v in a]))
            elems[name] = a[2].value
            N.lib.ghx_exec_free(ex)
    finally:
        N.lib.ghx_plan_free(h)
    assert elems["x"] + elems["rest"] == elems["all"] and elems["x"] > 0 and elems["rest"] > 0
    assert elems["x"] == len(boxes) * 2 * ng * b * b * nc


def sector_fills(n, b, nc, ng, kind, item=8, env=None, ring=False, monkeypatch=None):
    """Tags an executor of rank 0 (2 ranks, round-robin boxes) runs as sector fills."""
    if env is not None:
        monkeypatch.setenv("GHX_SECTOR_FILL", env)
    boxes = gu.scale_boxes(n, b)
    h = native_fb(boxes, [ng] * 3, [1, 1, 1], [n] * 3, [i % 2 for i in range(len(boxes))], 2)
    storage = boxes.copy()
    storage[:, :3] -= ng
    storage[:, 3:] += ng
    storage = np.ascontiguousarray(storage)
    ex = C.c_void_p()
    try:
        N.check(N.lib.ghx_exec_create(h, 0, kind, N.i64p(storage), nc, N.i64p(storage), nc, 0, 0, nc, item, 0,
                                      C.byref(ex)))
        if ring:
            N.check(N.lib.ghx_exec_set_ring(ex, 1))
        v = C.c_int64()
        N.check(N.lib.ghx_exec_sector_fills(ex, C.byref(v)))
        return v.value
    finally:
        if ex:
            N.lib.ghx_exec_free(ex)
        N.lib.ghx_plan_free(h)


def test_unpack_x_ghosts_run_as_sector_fills(monkeypatch):
    # 4 x 4 x 4 boxes, ranks alternate along x: every x-face is remote.  Rank
    # 0 receives, per fab, a lo- and a hi-x ghost tag of 16-byte rows (f64,
    # ng 2) whose sectors' other halves are valid cells
    assert sector_fills(64, 16, 2, 2, N.EXEC_UNPACK_PACKED) == 32 * 2
    assert sector_fills(64, 16, 2, 2, N.EXEC_UNPACK) == 32 * 2
    assert sector_fills(64, 16, 2, 2, N.EXEC_UNPACK_PACKED, env="0", monkeypatch=monkeypatch) == 0
    # pushes, host-memory (ring) executors, rows that are not one 16-byte
    # vector (ng 1: 8-byte rows; f32 ng 2: 8-byte rows) -> no fills
    monkeypatch.delenv("GHX_SECTOR_FILL", raising=False)
    assert sector_fills(64, 16, 2, 2, N.EXEC_PUSH_PACKED) == 0
    assert sector_fills(64, 16, 2, 2, N.EXEC_UNPACK_PACKED, ring=True) == 0
    assert sector_fills(64, 16, 2, 1, N.EXEC_UNPACK_PACKED) == 0
    assert sector_fills(64, 16, 2, 2, N.EXEC_UNPACK_PACKED, item=4) == 0
    # f32 ng 4: 16-byte rows again
    assert sector_fills(64, 16, 2, 4, N.EXEC_UNPACK_PACKED, item=4) == 32 * 2


def test_exchange_packed_combines_push_and_unpack():
    """GHX_EXEC_EXCHANGE_PACKED = PUSH_PACKED + UNPACK_PACKED of one rank in
    one task list: same tags, same send / receive buffer sizes."""
    boxes = gu.scale_boxes(64, 16)
    ranks = [i % 4 for i in range(len(boxes))]
    h = native_fb(boxes, [2] * 3, [1, 1, 1], [64] * 3, ranks, 4)
    storage = boxes.copy()
    storage[:, :3] -= 2
    storage[:, 3:] += 2
    storage = np.ascontiguousarray(storage)

    def info(kind):
        ex = C.c_void_p()
        N.check(N.lib.ghx_exec_create(h, 1, kind, N.i64p(storage), 2, N.i64p(storage), 2, 0, 0, 2, 8, 0,
                                      C.byref(ex)))
        try:
            a = [C.c_int64() for _ in range(4)]
            N.check(N.lib.ghx_exec_info(ex, *[C.byref(v) for v in a]))
            send, recv = np.zeros(4, np.int64), np.zeros(4, np.int64)
            N.check(N.lib.ghx_exec_buffer_elems(ex, N.i64p(send)))
            N.check(N.lib.ghx_exec_recv_elems(ex, N.i64p(recv)))
            fills, kinds = C.c_int64(), np.zeros(6, np.int64)
            N.check(N.lib.ghx_exec_sector_fills(ex, C.byref(fills)))
            N.check(N.lib.ghx_exec_task_kinds(ex, N.i64p(kinds)))
            if kind == N.EXEC_EXCHANGE_PACKED:  # fills ride in the instantiation without swap / chain tasks
                assert fills.value > 0 and kinds[1] == 0 and kinds[2] == 0
            return a[0].value, a[2].value, send, recv
        finally:
            N.lib.ghx_exec_free(ex)
    try:
        tp, ep, sp, _ = info(N.EXEC_PUSH_PACKED)
        tu, eu, _, ru = info(N.EXEC_UNPACK_PACKED)
        tx, ex_, sx, rx = info(N.EXEC_EXCHANGE_PACKED)
        assert tx == tp + tu and ex_ == ep + eu
        assert np.array_equal(sx, sp) and np.array_equal(rx, ru) and rx.sum() > 0
    finally:
        N.lib.ghx_plan_free(h)


def test_exchange_packed_runs_only_synced():
    boxes = gu.scale_boxes(64, 16)
    h = native_fb(boxes, [2] * 3, [1, 1, 1], [64] * 3, [i % 2 for i in range(len(boxes))], 2)
    storage = boxes.copy()
    storage[:, :3] -= 2
    storage[:, 3:] += 2
    storage = np.ascontiguousarray(storage)
    ex = C.c_void_p()
    try:
        N.check(N.lib.ghx_exec_create(h, 0, N.EXEC_EXCHANGE_PACKED, N.i64p(storage), 2, N.i64p(storage), 2, 0, 0, 2,
                                      8, 0, C.byref(ex)))
        table = np.zeros(2 * len(boxes) + 4, np.uint64)
        rc = N.lib.ghx_exec_run(ex, table.ctypes.data_as(C.POINTER(C.c_void_p)), len(table), None)
        assert rc == 1 and b"run_synced" in N.lib.ghx_last_error()
    finally:
        if ex:
            N.lib.ghx_exec_free(ex)
        N.lib.ghx_plan_free(h)
