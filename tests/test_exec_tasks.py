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
