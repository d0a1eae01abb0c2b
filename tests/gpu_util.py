"""Helpers for the GPU parity tests (device-side inputs, raw-bit readback)."""

from __future__ import annotations

import ctypes as C

import numpy as np


def bits_of(fab) -> np.ndarray:
    """Raw storage of a fab (F-order flat) as uint64/uint32 on the host."""
    import torch
    flat = fab.raw()
    it = torch.int64 if flat.element_size() == 8 else torch.int32
    a = flat.view(it).cpu().numpy()
    return a.view(np.uint64 if flat.element_size() == 8 else np.uint32)


def upload(fab, arr: np.ndarray) -> None:
    """Copy an F-order numpy array (nx, ny, nz, nc) into the fab bit-exactly."""
    import torch
    flat = fab.raw()
    src = np.ascontiguousarray(arr.ravel(order="F"))
    it = np.int64 if src.dtype.itemsize == 8 else np.int32
    t = torch.from_numpy(src.view(it))
    flat.view(torch.int64 if src.dtype.itemsize == 8 else torch.int32).copy_(t)


def expected_wrapped(fab, ncomp, domain_row, periodic, seed, itemsize):
    """Device tensor holding the wrapped-hash expectation for one fab."""
    import torch
    from paper_2403_12179_b200 import _native as N
    n = fab.raw().numel()
    dev = fab.data.device if fab.data.is_cuda else torch.device("cuda", torch.cuda.current_device())  # host fabs
    out = torch.empty(n, dtype=torch.int64 if itemsize == 8 else torch.int32, device=dev)
    fb = np.ascontiguousarray(np.asarray(fab.box.as_row(), np.int64))
    dom = np.ascontiguousarray(np.asarray(domain_row, np.int64))
    per = np.ascontiguousarray(np.asarray(list(periodic) + [0] * (3 - len(periodic)), np.int32))
    N.check(N.lib.ghx_fill_hash_wrapped(C.c_void_p(out.data_ptr()), N.i64p(fb), ncomp, N.i64p(dom), N.i32p(per),
                                        C.c_uint64(seed), itemsize, None))
    return out


def device_bits(fab):
    import torch
    flat = fab.raw()
    return flat.view(torch.int64 if flat.element_size() == 8 else torch.int32)
