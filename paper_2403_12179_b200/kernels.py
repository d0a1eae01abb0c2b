"""The reference's launch-backend handle, kept for signature compatibility
(reference kernels.py:47-111).

``fill_boundary(..., backend=b)`` / ``parallel_copy(..., backend=b)`` accept
the same object the reference does, but there is exactly one execution
path -- the fused CUDA kernels -- so the backend selects nothing.  Its
``launch_counter`` counts the device launches each exchange call makes (the
reference counts one dispatch per non-empty phase: a single-rank
FillBoundary is one launch in both).  Kinds are the reference's
``"serial"`` / ``"parallel"``; anything else raises ValueError, as
``Backend("gpu")`` does in the reference (tests/test_kernels.py:202-205).
"""

from __future__ import annotations

import os
import threading

SERIAL = "serial"
CPU_PARALLEL = "parallel"


class Backend:
    def __init__(self, kind: str = SERIAL, nworkers: int | None = None):
        if kind not in (SERIAL, CPU_PARALLEL):
            raise ValueError(f"backend kind must be '{SERIAL}' or '{CPU_PARALLEL}'")
        self.kind = kind
        self.nworkers = int(nworkers) if nworkers else (os.cpu_count() or 1)
        if self.nworkers < 1:
            raise ValueError("nworkers must be >= 1")
        self._counter_lock = threading.Lock()
        self.launch_counter = 0

    def _bump(self, n: int = 1) -> None:
        with self._counter_lock:
            self.launch_counter += n


_default_backend: Backend | None = None
_default_lock = threading.Lock()


def default_backend() -> Backend:
    global _default_backend
    with _default_lock:
        if _default_backend is None:
            _default_backend = Backend(CPU_PARALLEL)
        return _default_backend


def set_default_backend(backend: Backend) -> None:
    global _default_backend
    with _default_lock:
        _default_backend = backend
