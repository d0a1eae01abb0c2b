"""ctypes binding of libghostx.so (the C ABI declared in include/ghostx.h).

The library is the only compute path: if it is missing or fails to load,
importing the exchange layer raises -- there is no Python/CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# GHX_LIB: developer override (kernel-variant experiments, scripts/variants.sh)
LIB_PATH = os.environ.get("GHX_LIB") or os.path.join(_HERE, "_lib", "libghostx.so")

GHX_OK, GHX_EINVAL, GHX_ECUDA, GHX_ENOMEM, GHX_EOVERLAP = 0, 1, 2, 3, 4
MODE_FILL_BOUNDARY, MODE_PARALLEL_COPY = 0, 1
EXEC_DIRECT, EXEC_LOCAL, EXEC_PACK, EXEC_UNPACK, EXEC_PUSH_PACKED, EXEC_UNPACK_PACKED = 0, 1, 2, 3, 4, 5
EXEC_PHASED = 0x100  # flag OR-ed into the kind (include/ghostx.h)
EXEC_ONLY_XFACES, EXEC_NO_XFACES = 0x200, 0x400  # diagnostic direction split
EXEC_PUSH_PACKED_ALL, EXEC_UNPACK_PACKED_ALL = 6, 7
EXEC_EXCHANGE_PACKED = 8

P = C.c_void_p
I32 = C.c_int32
I64 = C.c_int64
PI64 = C.POINTER(C.c_int64)
PI32 = C.POINTER(C.c_int32)


class GhostxError(RuntimeError):
    """A libghostx call failed (CUDA error, out of memory, ...)."""


# name: (restype, argtypes)
_SIGS = {
    "ghx_last_error": (C.c_char_p, []),
    "ghx_version": (C.c_int, []),
    "ghx_boxes_disjoint": (C.c_int, [I64, PI64, PI64, PI64]),
    "ghx_plan_build_fill_boundary": (C.c_int, [I64, PI64, PI64, PI32, PI64, PI32, I32, C.POINTER(P)]),
    "ghx_plan_build_parallel_copy": (C.c_int, [I64, PI64, PI64, I64, PI64, PI64, PI32, PI64, PI32, PI32,
                                               I32, C.POINTER(P)]),
    "ghx_plan_free": (None, [P]),
    "ghx_plan_num_segments": (I64, [P]),
    "ghx_plan_get_segments": (C.c_int, [P, PI64]),
    "ghx_plan_num_write_tags": (I64, [P]),
    "ghx_plan_pair_cells": (C.c_int, [P, PI64]),
    "ghx_exec_create": (C.c_int, [P, I32, I32, PI64, I32, PI64, I32, I32, I32, I32, I32, I32, C.POINTER(P)]),
    "ghx_exec_free": (None, [P]),
    "ghx_exec_run": (C.c_int, [P, C.POINTER(P), I64, P]),
    "ghx_exec_bind": (C.c_int, [P, C.POINTER(P), I64, P, PI64]),
    "ghx_exec_run_bound": (C.c_int, [P, I64, P]),
    "ghx_exec_unbind": (C.c_int, [P, I64]),
    "ghx_exec_info": (C.c_int, [P, PI64, PI64, PI64, PI64]),
    "ghx_exec_buffer_elems": (C.c_int, [P, PI64]),
    "ghx_exec_detail": (C.c_int, [P, PI64]),
    "ghx_exec_set_grid": (C.c_int, [P, I32, I32]),
    "ghx_exec_set_ring": (C.c_int, [P, I32]),
    "ghx_exec_task_kinds": (C.c_int, [P, PI64]),
    "ghx_exec_set_bulk": (C.c_int, [P, I32]),
    "ghx_exec_set_sync": (C.c_int, [P, C.POINTER(P), I32, I32]),
    "ghx_exec_phases": (C.c_int, [P, PI64]),
    "ghx_exec_sector_fills": (C.c_int, [P, PI64]),
    "ghx_exec_recv_elems": (C.c_int, [P, PI64]),
    "ghx_exec_run_synced": (C.c_int, [P, I64, C.c_uint64, P]),
    "ghx_exec_sync_wait": (C.c_int, [P, C.c_uint64, P]),
    "ghx_arena_create": (C.c_int, [I32, I32, I32, C.c_size_t, C.POINTER(P)]),
    "ghx_arena_alloc": (C.c_int, [P, C.c_size_t, C.c_size_t, C.POINTER(P)]),
    "ghx_arena_free": (C.c_int, [P, P]),
    "ghx_arena_free_after": (C.c_int, [P, P, C.POINTER(P), I32]),
    "ghx_arena_poll": (C.c_int, [P, PI64]),
    "ghx_arena_block_size": (C.c_int, [P, P, C.POINTER(C.c_size_t)]),
    "ghx_arena_stats": (C.c_int, [P, PI64]),
    "ghx_arena_destroy": (None, [P]),
    "ghx_device_alloc": (C.c_int, [I32, C.c_size_t, C.POINTER(P)]),
    "ghx_device_free": (C.c_int, [P]),
    "ghx_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(P)]),
    "ghx_host_free": (C.c_int, [P]),
    "ghx_memset_u64": (C.c_int, [P, C.c_uint64, C.c_size_t, P]),
    "ghx_enable_peer_access": (C.c_int, [I32, I32]),
    "ghx_ipc_get_handle": (C.c_int, [P, C.POINTER(C.c_uint8)]),
    "ghx_ipc_open_handle": (C.c_int, [I32, C.POINTER(C.c_uint8), C.POINTER(P)]),
    "ghx_ipc_close_handle": (C.c_int, [P]),
    "ghx_alloc_offset": (C.c_int, [P, C.POINTER(C.c_uint64)]),
    "ghx_index_copy": (C.c_int, [P, I64, I32, I32, P]),
    "ghx_stream_sync": (C.c_int, [P]),
    "ghx_signal_barrier": (C.c_int, [C.POINTER(P), I32, I32, C.c_uint64, P]),
    "ghx_barrier_timeouts": (I64, []),
    "ghx_fill_hash": (C.c_int, [P, PI64, I32, PI64, PI64, C.c_uint64, I32, P]),
    "ghx_fill_hash_wrapped": (C.c_int, [P, PI64, I32, PI64, PI32, C.c_uint64, I32, P]),
    "ghx_launch_count": (I64, []),
    # job arrays: int64[njobs, 20] rows laid out like ghx_interp_job / ghx_avgdown_job
    "ghx_interp": (C.c_int, [P, I64, I32, PI32, I32, I32, I32, P]),
    "ghx_average_down": (C.c_int, [P, I64, I32, PI32, I32, I32, P]),
    "ghx_amr_launch_count": (I64, []),
    "ghx_interp_prepare": (C.c_int, [P, I64, I32, PI32, I32, I32, I32, I32, C.POINTER(P)]),
    "ghx_average_down_prepare": (C.c_int, [P, I64, I32, PI32, I32, I32, I32, C.POINTER(P)]),
    "ghx_advance_prepare": (C.c_int, [P, I64, C.POINTER(C.c_double), I32, I32, I32, I32, C.POINTER(P)]),
    "ghx_xfer_run": (C.c_int, [P, P]),
    "ghx_xfer_cells": (I64, [P]),
    "ghx_xfer_free": (None, [P]),
}

INTERP_PC, INTERP_LINEAR = 0, 1
ADVANCE_TILES, ADVANCE_CELLS = 0, 1
ARENA_POOLED, ARENA_SYSTEM = 0, 1
ARENA_DEVICE, ARENA_PINNED, ARENA_HOST = 0, 1, 2
JOB_WORDS = 20  # int64 words per ghx_interp_job / ghx_avgdown_job

EXPORTED = tuple(_SIGS)


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libghostx.so not found at {LIB_PATH}; build it with "
            "`python -m paper_2403_12179_b200._build` (there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def last_error() -> str:
    msg = lib.ghx_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> None:
    if rc == GHX_OK:
        return
    msg = last_error() or what
    if rc == GHX_EINVAL:
        raise ValueError(msg)
    if rc == GHX_ENOMEM:
        raise MemoryError(msg)
    raise GhostxError(msg)


def i64p(a: np.ndarray):
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(PI64)


def i32p(a: np.ndarray):
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(PI32)


def ptr_array(values) -> "C.Array":
    arr = np.ascontiguousarray(np.asarray(values, dtype=np.uint64))
    return arr, arr.ctypes.data_as(C.POINTER(P))
