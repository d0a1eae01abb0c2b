"""Zero-copy array access to fab storage (drop-in for the reference's
``miniamr.bridge`` fab views, frontend/src/miniamr/bridge.py:23-123).

A ``BoundArray4`` publishes one fab's ``(nx, ny, nz, ncomp)`` storage
(F-order, byte strides, zero-based per fab) through the CUDA array interface
(version 3) when the fab lives in HBM -- the device analogue of the
reference's ``__array_interface__`` (PAPER.md: ``__cuda_array_interface__``
/ ``to_cupy``) -- and additionally through ``__array_interface__`` when the
MultiFab uses pinned host memory.  ``to_torch`` / ``__dlpack__`` hand out the
same memory; ``to_host_array`` returns a host ndarray (a copy for device
fabs, a zero-copy view for pinned fabs unless ``copy=True``).
"""

from __future__ import annotations

from typing import Iterator

import numpy as np

from .mesh import Fab, FabView, MultiFab


class BoundArray4:
    """Array-protocol handle onto one fab's (nx, ny, nz, ncomp) storage."""

    def __init__(self, source, writable: bool | None = None):
        if isinstance(source, Fab):
            t = source.data
            w = True if writable is None else writable
        elif isinstance(source, FabView):
            t = source.array
            w = source.writable if writable is None else writable
        else:
            raise TypeError(f"expected a Fab or FabView, got {type(source).__name__}")
        self._keepalive = source
        self._t = t
        self._writable = bool(w)

    @property
    def shape(self) -> tuple:
        return tuple(self._t.shape)

    @property
    def strides(self) -> tuple:
        es = self._t.element_size()
        return tuple(s * es for s in self._t.stride())

    @property
    def typestr(self) -> str:
        return "<f8" if self._t.element_size() == 8 else "<f4"

    @property
    def address(self) -> int:
        return int(self._t.data_ptr())

    @property
    def is_device(self) -> bool:
        return bool(self._t.is_cuda)

    def _iface(self) -> dict:
        return {"shape": self.shape, "typestr": self.typestr, "strides": self.strides,
                "data": (self.address, not self._writable), "version": 3}

    @property
    def __cuda_array_interface__(self) -> dict:
        if not self.is_device:
            raise AttributeError("host (pinned) fab: use __array_interface__")
        d = self._iface()
        d["stream"] = None  # the exchange API is synchronous
        return d

    @property
    def __array_interface__(self) -> dict:
        if self.is_device:
            raise AttributeError("device fab: use __cuda_array_interface__ / to_torch()")
        return self._iface()

    def __dlpack__(self, stream=None):
        return self._t.__dlpack__() if stream is None else self._t.__dlpack__(stream=stream)

    def __dlpack_device__(self):
        return self._t.__dlpack_device__()

    def to_torch(self, order: str = "F"):
        """Zero-copy torch tensor: order "F" axes (x, y, z, comp), order "C"
        axes (comp, z, y, x) over the same storage."""
        if order == "F":
            return self._t
        if order == "C":
            return self._t.permute(3, 2, 1, 0)
        raise ValueError(f"order must be 'F' or 'C', got {order!r}")

    def to_host_array(self, order: str = "F", copy: bool = False) -> np.ndarray:
        """Host ndarray of the storage.  Device fabs are always copied
        (device->host); pinned fabs are zero-copy unless ``copy``."""
        if order not in ("F", "C"):
            raise ValueError(f"order must be 'F' or 'C', got {order!r}")
        if self.is_device:
            t = self.to_torch(order)
            out = t.cpu().numpy()
            return np.asfortranarray(out) if order == "F" else np.ascontiguousarray(out)
        base = np.asarray(self)
        if not self._writable:
            base = base.view()
            base.flags.writeable = False
        out = base if order == "F" else base.transpose(3, 2, 1, 0)
        if copy:
            out = out.copy(order="F" if order == "F" else "C")
        return out

    def to_numpy(self, order: str = "F", copy: bool = False) -> np.ndarray:
        return self.to_host_array(order, copy)


def array_view(source) -> BoundArray4:
    return BoundArray4(source)


class MfiAccessor:
    """Per-fab handle yielded by multifab_iter."""

    def __init__(self, mf: MultiFab, index: int):
        self._mf = mf
        self.index = index

    def tilebox(self):
        return self._mf.valid_box(self.index)

    def validbox(self):
        return self._mf.valid_box(self.index)

    def fabbox(self):
        return self._mf.grown_box(self.index)

    @property
    def n_grow_vect(self):
        return self._mf.ngrow

    def array_view(self, writable: bool = True) -> BoundArray4:
        return BoundArray4(self._mf.fab(self.index).view(writable=writable))

    def to_host_array(self, order: str = "F", copy: bool = False) -> np.ndarray:
        return self.array_view().to_host_array(order, copy)

    def to_torch(self, order: str = "F"):
        return self.array_view().to_torch(order)


def multifab_iter(mf: MultiFab) -> Iterator[MfiAccessor]:
    """One accessor per locally owned fab; structural mutation of the
    MultiFab while iterating raises RuntimeError (bridge.py:113-123)."""
    snapshot = tuple(mf.local_indices)
    live = tuple(sorted(mf.fabs))
    for gi in snapshot:
        if tuple(sorted(mf.fabs)) != live:
            raise RuntimeError("MultiFab structure changed during iteration")
        yield MfiAccessor(mf, gi)
