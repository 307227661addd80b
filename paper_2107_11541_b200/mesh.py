"""Device-resident meshes and the synthetic box generators.

`generate_box_mesh` / `generate_mixed_mesh` build the reference's meshes
(mesh.py:227-336) directly in HBM with CUDA kernels: node coordinates are
np.linspace-exact and connectivity follows the reference's cell order, Kuhn
permutations and pyramid faces, so coords and conn are bitwise identical to
the reference's (tests/test_gpu_setup.py).  Connectivity is int32 on the
device; the numpy views (`.coords`, `.conn`) are materialised on demand with
the reference dtypes (float64 / int64).

Boundary faces (mesh.py:115-155) are extracted on the device on first use
(`Mesh.boundary`): faces shared by exactly one element, outward-oriented, in
the reference's template order; they feed the Robin boundary assembly and
`boundary_nodes()`.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._mirror import DeviceArray
from .elements import DIM, ELEMENT_FACES, ETYPE_ID, NNODES, ElementType


def _as_conn_d(conn) -> torch.Tensor:
    if isinstance(conn, torch.Tensor) and conn.is_cuda and conn.dtype == torch.int32:
        return conn
    if isinstance(conn, torch.Tensor):
        conn = conn.cpu().numpy()
    conn = np.asarray(conn)
    if conn.size and conn.max() >= np.iinfo(np.int32).max:
        raise ValueError("node ids exceed int32")
    return torch.as_tensor(np.ascontiguousarray(conn, dtype=np.int32), device=_lib.device())


class ElementGroup:
    """Connectivity of one element type (mesh.py:20-30); conn_d is int32
    [nelem, nn] in HBM.  `conn` is the reference's int64 ndarray, a
    write-back mirror: in-place edits reach the device before the next
    kernel reads the connectivity (_mirror.py)."""

    def __init__(self, etype: ElementType, conn):
        self.etype = etype
        self._conn = DeviceArray(_as_conn_d(conn), np.int64)

    @property
    def conn_d(self) -> torch.Tensor:
        return self._conn.device()

    @conn_d.setter
    def conn_d(self, t: torch.Tensor) -> None:
        self._conn.set_device(_as_conn_d(t))

    @property
    def conn(self) -> np.ndarray:
        return self._conn.host()

    @conn.setter
    def conn(self, value) -> None:
        self._conn.set_device(_as_conn_d(value))

    @property
    def nelem(self) -> int:
        return int(self._conn._t.shape[0])

    def __repr__(self) -> str:
        return f"ElementGroup({self.etype}, nelem={self.nelem})"


def _as_coords_d(coords) -> torch.Tensor:
    if isinstance(coords, torch.Tensor) and coords.is_cuda and coords.dtype == torch.float64:
        return coords.contiguous()
    if isinstance(coords, torch.Tensor):
        coords = coords.cpu().numpy()
    return torch.as_tensor(np.ascontiguousarray(coords, dtype=np.float64), device=_lib.device())


class Mesh:
    """dim, node coordinates float64 [nnode, dim] and element groups, all in
    HBM (mesh.py:57-113).  Accepts numpy or torch arguments like the
    reference's dataclass; `coords` is a write-back host mirror."""

    def __init__(self, dim: int, coords, groups=None, boundary=None):
        self.dim = int(dim)
        self._coords = DeviceArray(_as_coords_d(coords))
        self.groups = list(groups) if groups is not None else []
        self._boundary = list(boundary) if boundary is not None else None

    @property
    def coords_d(self) -> torch.Tensor:
        return self._coords.device()

    @coords_d.setter
    def coords_d(self, t) -> None:
        self._coords.set_device(_as_coords_d(t))

    @property
    def coords(self) -> np.ndarray:
        return self._coords.host()

    @coords.setter
    def coords(self, value) -> None:
        self._coords.set_device(_as_coords_d(value))

    @property
    def boundary(self) -> list:
        """Boundary FaceGroups (mesh.py:140-155), extracted on first use."""
        if self._boundary is None:
            self._boundary = extract_boundary(self.groups)
        return self._boundary

    @boundary.setter
    def boundary(self, value) -> None:
        self._boundary = list(value)

    def boundary_nodes(self) -> np.ndarray:
        """Sorted unique node ids on any boundary face (mesh.py:82-86)."""
        if not self.boundary:
            return np.empty(0, dtype=np.int64)
        allnodes = torch.cat([fg.conn_d.reshape(-1) for fg in self.boundary])
        return torch.unique(allnodes).cpu().numpy().astype(np.int64)

    @property
    def nnode(self) -> int:
        return int(self._coords._t.shape[0])

    @property
    def nelem(self) -> int:
        return sum(g.nelem for g in self.groups)

    def element_counts(self) -> dict:
        out: dict = {}
        for g in self.groups:
            out[g.etype] = out.get(g.etype, 0) + g.nelem
        return out

    def is_grouped_by_type(self) -> bool:
        types = [g.etype for g in self.groups]
        return len(types) == len(set(types))

    def validate(self) -> None:
        """Raise ValueError on structural defects (mesh.py:88-113); the
        range, finiteness and shared-face checks run on the device."""
        if self.dim not in (2, 3):
            raise ValueError(f"unsupported dimension {self.dim}")
        x = self.coords_d
        if x.ndim != 2 or x.shape[1] != self.dim:
            raise ValueError("coords must have shape (nnode, dim)")
        if x.numel() and not bool(torch.isfinite(x).all()):
            raise ValueError("non-finite node coordinates")
        n = self.nnode
        for g in self.groups:
            c = g.conn_d
            if DIM[g.etype] != self.dim:
                raise ValueError(f"{g.etype.value} in a {self.dim}D mesh")
            if c.ndim != 2 or c.shape[1] != NNODES[g.etype]:
                raise ValueError(f"bad connectivity shape for {g.etype.value}")
            if g.nelem and (int(c.min()) < 0 or int(c.max()) >= n):
                raise ValueError(f"node index out of range in {g.etype.value}")
        if self._boundary is not None:
            for fg in self._boundary:
                if fg.conn_d.shape[1] != fg.nnodes:
                    raise ValueError("face group width mismatch")
                if fg.nfaces and (int(fg.conn_d.min()) < 0 or int(fg.conn_d.max()) >= n):
                    raise ValueError("face node index out of range")
                if fg.nfaces and (int(fg.owner_d.min()) < 0 or int(fg.owner_d.max()) >= self.nelem):
                    raise ValueError("face owner out of range")
        for size, counts in _face_counts(self.groups).items():
            if counts.numel() and int(counts.max()) > 2:
                raise ValueError(f"{size}-node face shared by more than 2 elements")

    def __repr__(self) -> str:
        return f"Mesh(dim={self.dim}, nnode={self.nnode}, groups={self.groups})"


@dataclass
class FaceGroup:
    """Boundary faces of one node count (mesh.py:33-47): owner element ids and
    outward-oriented face nodes, in HBM."""

    nnodes: int
    owner_d: torch.Tensor
    conn_d: torch.Tensor

    @property
    def nfaces(self) -> int:
        return int(self.conn_d.shape[0])

    @property
    def owner(self) -> np.ndarray:
        return self.owner_d.cpu().numpy()

    @property
    def conn(self) -> np.ndarray:
        return self.conn_d.cpu().numpy().astype(np.int64)


def _faces_by_size(groups) -> dict:
    """{size: [(owner ids, face nodes)]} per face template (mesh.py:117-125)."""
    buckets: dict = {}
    offset = 0
    for g in groups:
        for tmpl in ELEMENT_FACES[g.etype]:
            idx = torch.as_tensor(tmpl, dtype=torch.int64, device=g.conn_d.device)
            owner = torch.arange(offset, offset + g.nelem, dtype=torch.int64, device=g.conn_d.device)
            buckets.setdefault(len(tmpl), []).append((owner, g.conn_d.index_select(1, idx)))
        offset += g.nelem
    return buckets


def _face_counts(groups) -> dict:
    """{size: multiplicity of every distinct face} (mesh.py:127-137)."""
    out = {}
    for size, parts in _faces_by_size(groups).items():
        faces = torch.cat([f for _, f in parts], dim=0)
        if faces.shape[0] == 0:
            out[size] = torch.empty(0, dtype=torch.int64)
            continue
        key = torch.sort(faces.to(torch.int64), dim=1).values
        out[size] = torch.unique(key, dim=0, return_counts=True)[1]
    return out


def extract_boundary(groups) -> list:
    """Faces that belong to exactly one element (mesh.py:140-155), grouped by
    node count in ascending size, each group in the reference's (group,
    template, element) order.  Face counting by sorted node tuples on the
    device (setup only)."""
    buckets = _faces_by_size(groups)
    out = []
    for size in sorted(buckets):
        owners = torch.cat([o for o, _ in buckets[size]])
        faces = torch.cat([f for _, f in buckets[size]], dim=0)
        if faces.shape[0] == 0:
            continue
        key = torch.sort(faces.to(torch.int64), dim=1).values
        _, inverse, counts = torch.unique(key, dim=0, return_inverse=True, return_counts=True)
        keep = counts[inverse] == 1
        if bool(keep.any()):
            out.append(FaceGroup(size, owners[keep].contiguous(), faces[keep].contiguous()))
    return out


def as_device_mesh(mesh) -> Mesh:
    """Accept this package's Mesh or any reference-style mesh (numpy
    `coords` and groups with `.etype` / `.conn`) and return a device Mesh."""
    if isinstance(mesh, Mesh):
        return mesh
    dev = _lib.device()
    coords = torch.as_tensor(np.ascontiguousarray(mesh.coords, dtype=np.float64), device=dev)
    groups = []
    for g in mesh.groups:
        et = g.etype if isinstance(g.etype, ElementType) else ElementType(g.etype.value)
        conn = np.asarray(g.conn)
        if conn.size and (conn.max() >= np.iinfo(np.int32).max):
            raise ValueError("node ids exceed int32")
        groups.append(ElementGroup(et, torch.as_tensor(conn.astype(np.int32), device=dev)))
    return Mesh(int(mesh.dim), coords, groups)


def _grid(dim, nx, ny, nz, lengths):
    dev = _lib.device()
    nnode = (nx + 1) * (ny + 1) * ((nz + 1) if dim == 3 else 1)
    coords = torch.empty((nnode, dim), dtype=torch.float64, device=dev)
    lz = lengths[2] if dim == 3 else 0.0
    _lib.call("fpb_grid_coords", dim, nx, ny, nz, float(lengths[0]), float(lengths[1]), float(lz),
              coords.data_ptr(), _lib.stream())
    return coords


def generate_box_mesh(etype: ElementType, nx: int, ny: int, nz: int = 1, lengths=None) -> Mesh:
    """Single-type box mesh in HBM (mesh.py:227-289)."""
    if min(nx, ny) < 1 or (DIM[etype] == 3 and nz < 1):
        raise ValueError("cell counts must be at least 1")
    dim = DIM[etype]
    if lengths is None:
        lengths = (1.0,) * dim
    if etype is ElementType.PYR05:
        return generate_mixed_mesh(nx, ny, nz, fraction=1.0, lengths=lengths)
    if dim == 2 and etype not in (ElementType.TRI03, ElementType.QUAD04):
        raise ValueError(f"{etype.value} is not a 2D type")
    coords = _grid(dim, nx, ny, nz, lengths)
    ncell = nx * ny * (nz if dim == 3 else 1)
    per = {ElementType.TET04: 6, ElementType.TRI03: 2}.get(etype, 1)
    conn = torch.empty((ncell * per, NNODES[etype]), dtype=torch.int32, device=coords.device)
    _lib.call("fpb_box_conn", ETYPE_ID[etype], nx, ny, nz, conn.data_ptr(), _lib.stream())
    return Mesh(dim, coords, [ElementGroup(etype, conn)])


def generate_mixed_mesh(nx: int, ny: int, nz: int, fraction: float = 0.5, lengths=None) -> Mesh:
    """Pyramid layers (i < ceil(fraction*nx)) plus hexes (mesh.py:292-336)."""
    if not 0.0 <= fraction <= 1.0:
        raise ValueError("fraction must lie in [0, 1]")
    if min(nx, ny, nz) < 1:
        raise ValueError("cell counts must be at least 1")
    if lengths is None:
        lengths = (1.0, 1.0, 1.0)
    nlayers = int(np.ceil(fraction * nx))
    npyr_cells = nlayers * ny * nz
    nhex = (nx - nlayers) * ny * nz
    ngrid = (nx + 1) * (ny + 1) * (nz + 1)
    dev = _lib.device()
    coords = torch.empty((ngrid + npyr_cells, 3), dtype=torch.float64, device=dev)
    _lib.call("fpb_grid_coords", 3, nx, ny, nz, float(lengths[0]), float(lengths[1]),
              float(lengths[2]), coords.data_ptr(), _lib.stream())
    pyr = torch.empty((6 * npyr_cells, 5), dtype=torch.int32, device=dev)
    hexc = torch.empty((nhex, 8), dtype=torch.int32, device=dev)
    _lib.call("fpb_mixed_conn", nx, ny, nz, nlayers, coords.data_ptr(), pyr.data_ptr(),
              hexc.data_ptr(), _lib.stream())
    groups = []
    if npyr_cells:
        groups.append(ElementGroup(ElementType.PYR05, pyr))
    if nhex:
        groups.append(ElementGroup(ElementType.HEX08, hexc))
    return Mesh(3, coords, groups)


@dataclass(frozen=True)
class Permutation:
    forward: np.ndarray
    inverse: np.ndarray


def renumber_by_type(mesh) -> tuple[Mesh, Permutation]:
    """Stable regroup so each type is one block (mesh.py:339-364)."""
    mesh = as_device_mesh(mesh)
    order: list = []
    for g in mesh.groups:
        if g.etype not in order:
            order.append(g.etype)
    keys = np.concatenate([np.full(g.nelem, order.index(g.etype), dtype=np.int64)
                           for g in mesh.groups]) if mesh.groups else np.empty(0, np.int64)
    inverse = np.argsort(keys, kind="stable")
    forward = np.empty_like(inverse)
    forward[inverse] = np.arange(len(inverse))
    groups = [ElementGroup(t, torch.cat([g.conn_d for g in mesh.groups if g.etype is t], dim=0))
              for t in order]
    boundary = None
    if mesh._boundary is not None:  # remap face owners with the permutation (mesh.py:360-362)
        fwd = torch.as_tensor(forward, device=mesh.coords_d.device)
        boundary = [FaceGroup(fg.nnodes, fwd.index_select(0, fg.owner_d.to(torch.int64)), fg.conn_d.clone())
                    for fg in mesh._boundary]
    return Mesh(mesh.dim, mesh.coords_d, groups, boundary), Permutation(forward, inverse)
