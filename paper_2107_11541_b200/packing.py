"""Lane-major element packs (packing.py:1-151), built in HBM.

The paper's SIMD layout: elements of one type grouped in packs of
`vector_size` lanes, lane index fastest, tail padded by replicating the last
element.  The assembly kernels always run at 32 lanes — one warp per pack, so
lane_conn[p][a][0:32] is one coalesced 128-byte row; a context additionally
exposes the packs at the caller's `vector_size` for parity with the
reference's `PackSet` (bit-exact, tests/test_gpu_setup.py).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .elements import ElementType
from .errors import ConfigurationError

VALID_VECTOR_SIZES = (1, 2, 4, 8, 16, 32)
KERNEL_LANES = 32  # one warp per pack
#: host allocation alignment in bytes (packing.py:25)
ALIGNMENT = 64


def aligned_zeros(shape, dtype=np.float64, alignment: int = ALIGNMENT) -> np.ndarray:
    """Zero-filled C-contiguous host array whose data start is aligned
    (packing.py:40-48); the host-side container of lane-major results."""
    dtype = np.dtype(dtype)
    size = int(np.prod(shape)) * dtype.itemsize
    buf = np.zeros(size + alignment, dtype=np.uint8)
    off = (-buf.ctypes.data) % alignment
    return buf[off:off + size].view(dtype).reshape(shape)


@dataclass(frozen=True)
class PackConfig:
    vector_size: int = 8

    def __post_init__(self):
        if self.vector_size not in VALID_VECTOR_SIZES:
            raise ConfigurationError(
                f"vector_size must be one of {VALID_VECTOR_SIZES}, got {self.vector_size}")


def pack_lanes(conn_d: torch.Tensor, vs: int) -> torch.Tensor:
    """lane_conn[npacks][nn][vs] (int32, HBM) — packing.py:104-115."""
    ne, nn = conn_d.shape
    npacks = -(-ne // vs)
    out = torch.empty((npacks, nn, vs), dtype=torch.int32, device=conn_d.device)
    _lib.call("fpb_build_packs", ne, nn, vs, conn_d.data_ptr(), out.data_ptr(), _lib.stream())
    return out


@dataclass
class PackSet:
    """Packed connectivity of one element type (packing.py:50-82)."""

    etype: ElementType
    vector_size: int
    nelem: int
    offset: int
    lane_conn_d: torch.Tensor
    _cache: dict = field(default_factory=dict, repr=False)

    @property
    def npacks(self) -> int:
        return int(self.lane_conn_d.shape[0])

    @property
    def npadded(self) -> int:
        return self.npacks * self.vector_size - self.nelem

    @property
    def lane_conn(self) -> np.ndarray:
        if "lane_conn" not in self._cache:
            self._cache["lane_conn"] = self.lane_conn_d.cpu().numpy().astype(np.int64)
        return self._cache["lane_conn"]

    @property
    def elem_index(self) -> np.ndarray:
        flat = np.empty(self.npacks * self.vector_size, dtype=np.int64)
        flat[: self.nelem] = self.offset + np.arange(self.nelem)
        flat[self.nelem:] = self.offset + self.nelem - 1
        return flat.reshape(self.npacks, self.vector_size)

    @property
    def active_mask(self) -> np.ndarray:
        m = np.zeros(self.npacks * self.vector_size, dtype=bool)
        m[: self.nelem] = True
        return m.reshape(self.npacks, self.vector_size)


def build_packs(mesh, config: PackConfig) -> list[PackSet]:
    """One PackSet per non-empty type block (packing.py:85-127)."""
    from .mesh import as_device_mesh

    mesh = as_device_mesh(mesh)
    if not mesh.is_grouped_by_type():
        raise ConfigurationError("mesh has repeated element-type blocks; renumber_by_type first")
    out, offset = [], 0
    for g in mesh.groups:
        if g.nelem:
            out.append(PackSet(g.etype, config.vector_size, g.nelem, offset,
                               pack_lanes(g.conn_d, config.vector_size)))
        offset += g.nelem
    return out


def pack_array(values, packset: PackSet, zero_pad: bool = True) -> np.ndarray:
    """Gather per-element data (nelem_total, ...) into lane-major form
    (npacks, ..., vector_size) (packing.py:130-142): a device gather by the
    pack's element index; padded lanes zeroed unless zero_pad is False (then
    they repeat the last active element)."""
    a = np.asarray(values)
    dev = _lib.device()
    src = torch.as_tensor(np.ascontiguousarray(a), device=dev)
    idx = torch.as_tensor(packset.elem_index.reshape(-1), device=dev)
    g = src.index_select(0, idx).reshape((packset.npacks, packset.vector_size) + a.shape[1:])
    g = torch.movedim(g, 1, -1).contiguous()
    if zero_pad and packset.npadded:
        g[packset.npacks - 1, ..., packset.vector_size - packset.npadded:] = 0
    out = aligned_zeros(tuple(g.shape), dtype=a.dtype)
    out[...] = g.cpu().numpy()
    return out


def unpack_array(packed, packset: PackSet, nelem_total: int) -> np.ndarray:
    """Scatter the active lanes of a lane-major array back to per-element
    rows (packing.py:145-151), on the device."""
    a = np.asarray(packed)
    dev = _lib.device()
    src = torch.movedim(torch.as_tensor(np.ascontiguousarray(a), device=dev), -1, 1)
    src = src.reshape((-1,) + tuple(src.shape[2:]))[: packset.nelem]
    out = torch.zeros((nelem_total,) + a.shape[1:-1], dtype=src.dtype, device=dev)
    out[packset.offset: packset.offset + packset.nelem] = src
    return out.cpu().numpy()
