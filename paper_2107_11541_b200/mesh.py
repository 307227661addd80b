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

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .elements import DIM, ETYPE_ID, NNODES, ElementType


@dataclass
class ElementGroup:
    """Connectivity of one element type; conn_d is int32 [nelem, nn] in HBM."""

    etype: ElementType
    conn_d: torch.Tensor
    _conn_h: np.ndarray | None = field(default=None, repr=False)

    @property
    def nelem(self) -> int:
        return int(self.conn_d.shape[0])

    @property
    def conn(self) -> np.ndarray:
        if self._conn_h is None:
            self._conn_h = self.conn_d.cpu().numpy().astype(np.int64)
        return self._conn_h


@dataclass
class Mesh:
    """dim, coords_d float64 [nnode, dim] and element groups, all in HBM."""

    dim: int
    coords_d: torch.Tensor
    groups: list[ElementGroup] = field(default_factory=list)
    _boundary: list | None = field(default=None, repr=False)
    _coords_h: np.ndarray | None = field(default=None, repr=False)

    @property
    def boundary(self) -> list:
        """Boundary FaceGroups (mesh.py:140-155), extracted on first use."""
        if self._boundary is None:
            self._boundary = extract_boundary(self.groups)
        return self._boundary

    def boundary_nodes(self) -> np.ndarray:
        """Sorted unique node ids on any boundary face (mesh.py:82-86)."""
        if not self.boundary:
            return np.empty(0, dtype=np.int64)
        allnodes = torch.cat([fg.conn_d.reshape(-1) for fg in self.boundary])
        return torch.unique(allnodes).cpu().numpy().astype(np.int64)

    @property
    def coords(self) -> np.ndarray:
        if self._coords_h is None:
            self._coords_h = self.coords_d.cpu().numpy()
        return self._coords_h

    @property
    def nnode(self) -> int:
        return int(self.coords_d.shape[0])

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


# outward-oriented face templates (elements.py:73-86)
ELEMENT_FACES = {
    ElementType.TRI03: ((0, 1), (1, 2), (2, 0)),
    ElementType.QUAD04: ((0, 1), (1, 2), (2, 3), (3, 0)),
    ElementType.TET04: ((0, 2, 1), (0, 1, 3), (1, 2, 3), (0, 3, 2)),
    ElementType.PYR05: ((0, 3, 2, 1), (0, 1, 4), (1, 2, 4), (2, 3, 4), (3, 0, 4)),
    ElementType.HEX08: ((0, 3, 2, 1), (4, 5, 6, 7), (0, 1, 5, 4), (2, 3, 7, 6), (0, 4, 7, 3), (1, 2, 6, 5)),
}


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


def extract_boundary(groups) -> list:
    """Faces that belong to exactly one element (mesh.py:140-155), grouped by
    node count in ascending size, each group in the reference's (group,
    template, element) order.  Face counting by sorted node tuples on the
    device (setup only)."""
    buckets: dict = {}
    offset = 0
    for g in groups:
        for tmpl in ELEMENT_FACES[g.etype]:
            idx = torch.as_tensor(tmpl, dtype=torch.int64, device=g.conn_d.device)
            owner = torch.arange(offset, offset + g.nelem, dtype=torch.int64, device=g.conn_d.device)
            buckets.setdefault(len(tmpl), []).append((owner, g.conn_d.index_select(1, idx)))
        offset += g.nelem
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
    return Mesh(mesh.dim, mesh.coords_d, groups), Permutation(forward, inverse)
