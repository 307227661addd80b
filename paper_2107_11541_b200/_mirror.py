"""Write-back host views of device arrays.

The reference's data structures are plain numpy arrays that callers read
*and edit in place* (`mesh.groups[0].conn[1, [1, 3]] = ...`,
`A.vals[k] = 1.0` in the reference's own sparse.py:249-253).  Here the data
live in HBM, so the numpy attribute is a host mirror with write-back:

* `host()` returns the same ndarray object every time (identity is stable, as
  for the reference's attributes) and refreshes it in place whenever the
  device copy was written since (torch version counter; kernel writes through
  raw pointers call `sparse.mark_written`).
* `device()` uploads the mirror first if the caller edited it (byte compare
  against the snapshot taken when it was last synchronised), so the next
  kernel sees the edit.

Large arrays (> WRITE_BACK_MAX bytes, e.g. a 100 M-tet matrix's 2 GB of
values) get a read-only mirror instead: downloaded through pinned staging at
PCIe speed, no snapshot copy, and an in-place write raises ("assignment
destination is read-only") instead of being lost — assign a new array
(`A.vals = ...`, `CsrMatrix.with_vals`) to change them.

Nothing here runs unless a caller touches the numpy attribute: the device
paths never create a mirror.
"""

from __future__ import annotations

import weakref

import numpy as np
import torch


WRITE_BACK_MAX = 64 << 20  # bytes: larger mirrors are read-only (no snapshot)


def _download(t: torch.Tensor) -> np.ndarray:
    """Device -> numpy through pinned staging (DMA speed, not pageable)."""
    if not t.is_cuda:
        return t.detach().numpy().copy()
    out = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    out.copy_(t, non_blocking=True)
    torch.cuda.current_stream(t.device).synchronize()
    return out.numpy()


class DeviceArray:
    """A device tensor plus an optional write-back numpy mirror."""

    __slots__ = ("_tt", "_weak", "_host_dtype", "_h", "_snap", "_ver")

    def __init__(self, t: torch.Tensor, host_dtype=None, weak: bool = False):
        """weak = True: hold the tensor by weak reference (a registry keyed by
        the tensor — sparse._vals_store — must not keep its key alive; the
        owners hold the tensor)."""
        self._weak = weak
        self._tt = weakref.ref(t) if weak else t
        self._host_dtype = np.dtype(host_dtype) if host_dtype is not None else None
        self._h = None
        self._snap = None
        self._ver = None

    def _sync_up(self) -> None:
        h = self._h
        if h is None or self._snap is None or self._ver != self._t._version:
            return  # no (writable) mirror, or the device copy is newer (device wins)
        if h.shape == self._snap.shape and np.array_equal(h.view(np.uint8), self._snap.view(np.uint8)):
            return
        if tuple(h.shape) != tuple(self._t.shape):
            raise ValueError("host mirror changed shape; assign a new array instead")
        src = torch.from_numpy(np.ascontiguousarray(h).astype(
            torch.empty((), dtype=self._t.dtype).numpy().dtype, copy=False))
        self._t.copy_(src)  # bumps the version counter
        self._snap = h.copy()
        self._ver = self._t._version

    def device(self) -> torch.Tensor:
        self._sync_up()
        return self._t

    @property
    def _t(self) -> torch.Tensor:
        return self._tt() if self._weak else self._tt

    def set_device(self, t: torch.Tensor) -> None:
        self._tt = weakref.ref(t) if self._weak else t
        self._h = self._snap = self._ver = None

    def host(self) -> np.ndarray:
        t = self._t
        if self._h is not None and self._ver == t._version:
            return self._h
        fresh = _download(t)
        if self._host_dtype is not None and fresh.dtype != self._host_dtype:
            fresh = fresh.astype(self._host_dtype)
        if fresh.nbytes > WRITE_BACK_MAX:
            fresh.flags.writeable = False  # no write-back for huge arrays: writes raise
            self._h, self._snap = fresh, None
        elif (self._h is not None and self._h.shape == fresh.shape and self._h.dtype == fresh.dtype
              and self._h.flags.writeable):
            self._h[...] = fresh  # keep the handed-out object current
            self._snap = self._h.copy()
        else:
            self._h = np.ascontiguousarray(fresh)
            self._snap = self._h.copy()
        self._ver = t._version
        return self._h

    def forget(self) -> None:
        """Drop the mirror (the next host() downloads a new array)."""
        self._h = self._snap = self._ver = None
