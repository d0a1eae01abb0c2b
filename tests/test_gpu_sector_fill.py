"""GPU: the unpack executor's sector fills (x-face ghost halves stored with
the valid half of their 32-byte sector) write exactly what the plain
16-byte unpack writes -- for 32-byte aligned fab bases (the fill path) and
for 16-byte aligned ones (the kernel's per-tag fallback) -- through the C
ABI, f64 ng 2 and f32 ng 4, every x-face remote (2 ranks alternating
along x)."""

import ctypes as C

import numpy as np
import pytest
import torch

import golden_util as gu
from paper_2403_12179_b200 import _native as N
from test_plan_native import native_fb

pytestmark = pytest.mark.gpu


def _unpack(h, storage, nc, item, kind, fab_bytes, base_off, fabs0, slab0, monkeypatch, fill):
    monkeypatch.setenv("GHX_SECTOR_FILL", "1" if fill else "0")
    ex = C.c_void_p()
    N.check(N.lib.ghx_exec_create(h, 0, kind, N.i64p(storage), nc, N.i64p(storage), nc, 0, 0, nc, item, 0,
                                  C.byref(ex)))
    try:
        sf = C.c_int64()
        N.check(N.lib.ghx_exec_sector_fills(ex, C.byref(sf)))
        assert (sf.value > 0) == fill
        nf = len(storage)
        fabs = fabs0.clone()
        slab = slab0.clone()
        table = np.zeros(2 * nf + 4, np.uint64)
        for i in range(nf):
            table[nf + i] = fabs.data_ptr() + base_off + i * fab_bytes
        table[2 * nf + 2 + 1] = slab.data_ptr()  # receive buffer from rank 1
        stream = torch.cuda.current_stream().cuda_stream
        N.check(N.lib.ghx_exec_run(ex, table.ctypes.data_as(C.POINTER(C.c_void_p)), len(table), C.c_void_p(stream)))
        torch.cuda.synchronize()
        return fabs
    finally:
        N.lib.ghx_exec_free(ex)


@pytest.mark.parametrize("item,ng", [(8, 2), (4, 4)])
@pytest.mark.parametrize("base_off", [0, 16])
@pytest.mark.parametrize("kind", ["UNPACK_PACKED", "UNPACK"])
def test_sector_fill_matches_plain_unpack(item, ng, base_off, kind, monkeypatch):
    n, b, nc = 64, 16, 2
    boxes = gu.scale_boxes(n, b)
    h = native_fb(boxes, [ng] * 3, [1, 1, 1], [n] * 3, [i % 2 for i in range(len(boxes))], 2)
    try:
        storage = boxes.copy()
        storage[:, :3] -= ng
        storage[:, 3:] += ng
        storage = np.ascontiguousarray(storage)
        fab_bytes = (b + 2 * ng) ** 3 * nc * item
        fab_bytes = -(-fab_bytes // 256) * 256
        g = torch.Generator(device="cuda").manual_seed(7)
        fabs0 = torch.randint(0, 256, (base_off + fab_bytes * len(storage),), dtype=torch.uint8, device="cuda",
                              generator=g)
        k = getattr(N, "EXEC_" + kind)
        # receive-buffer size from a throwaway executor
        ex = C.c_void_p()
        N.check(N.lib.ghx_exec_create(h, 0, k, N.i64p(storage), nc, N.i64p(storage), nc, 0, 0, nc, item, 0,
                                      C.byref(ex)))
        be = np.zeros(2, np.int64)
        N.check(N.lib.ghx_exec_buffer_elems(ex, N.i64p(be)))
        N.lib.ghx_exec_free(ex)
        assert be[1] > 0
        slab0 = torch.randint(0, 256, (int(be[1]) * item,), dtype=torch.uint8, device="cuda", generator=g)
        plain = _unpack(h, storage, nc, item, k, fab_bytes, base_off, fabs0, slab0, monkeypatch, False)
        fill = _unpack(h, storage, nc, item, k, fab_bytes, base_off, fabs0, slab0, monkeypatch, True)
        assert not torch.equal(plain, fabs0)  # the unpack wrote ghost cells
        assert torch.equal(fill, plain)
    finally:
        N.lib.ghx_plan_free(h)
