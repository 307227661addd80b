"""Z-slab domain decomposition of the synthetic box meshes across GPUs.

The reference has no partitioner; this module defines one
 and is pinned by its own restatement in the tests:

* Cells are visited k-major (mesh.py:220-224) and nodes are numbered
  i + (nx+1)(j + (ny+1)k) (mesh.py:183-184), so a contiguous range of cell
  layers [k0, k1) is a contiguous range of elements and its node planes
  k0..k1 a contiguous range of nodes.  Rank r owns layers
  [k0_r, k1_r) = balanced split of nz (first ranks take the remainder).
* Every rank keeps one ghost cell layer on each side that has a neighbour.
  Ghost elements are never integrated; they only shape the local CSR graph,
  so the rows of an interface plane have the same global column set on both
  sides and their values can be summed entry by entry.
* Halo sum: after local assembly, each interface plane's RHS rows / CSR row
  segments are exchanged with the neighbour (one grouped send/recv pair per
  interface — NCCL over NVLink on GPUs, gloo on CPU) and added, so both
  copies hold the global value (a + b == b + a bit for bit).
* Ownership for gathering a global result: rank r owns node planes
  [k0_r + (r > 0), k1_r] — interface plane k1_r belongs to the lower rank.

Everything here is device-agnostic torch code except `SlabDomain.build`,
which generates the local mesh with the CUDA setup kernels.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from .elements import ElementType


def slab_ranges(nz: int, world: int) -> list[tuple[int, int]]:
    """Balanced cell-layer ranges [k0, k1) per rank."""
    if world < 1 or nz < world:
        raise ValueError(f"cannot split {nz} cell layers over {world} ranks")
    base, rem = divmod(nz, world)
    out, k = [], 0
    for r in range(world):
        n = base + (1 if r < rem else 0)
        out.append((k, k + n))
        k += n
    return out


@dataclass(frozen=True)
class SlabLayout:
    """Index bookkeeping of one rank's slab (all counts in the box grid)."""

    nx: int
    ny: int
    nz: int
    rank: int
    world: int
    k0: int  # first owned cell layer
    k1: int  # one past the last owned cell layer
    kA: int  # first local node plane (k0 - 1 with a lower neighbour)
    kB: int  # last local node plane (k1 + 1 with an upper neighbour)
    cells_per_layer: int
    elems_per_cell: int

    @classmethod
    def make(cls, nx, ny, nz, rank, world, etype: ElementType = ElementType.TET04) -> "SlabLayout":
        k0, k1 = slab_ranges(nz, world)[rank]
        kA = k0 - (1 if rank > 0 else 0)
        kB = k1 + (1 if rank < world - 1 else 0)
        per = {ElementType.TET04: 6, ElementType.HEX08: 1}[etype]
        return cls(nx, ny, nz, rank, world, k0, k1, kA, kB, nx * ny, per)

    @property
    def plane(self) -> int:
        return (self.nx + 1) * (self.ny + 1)

    @property
    def nplanes(self) -> int:
        return self.kB - self.kA + 1

    @property
    def nnode(self) -> int:
        return self.plane * self.nplanes

    @property
    def node_offset(self) -> int:
        """global node id = local node id + node_offset."""
        return self.plane * self.kA

    @property
    def elems_per_layer(self) -> int:
        return self.cells_per_layer * self.elems_per_cell

    @property
    def own_elems(self) -> tuple[int, int]:
        """Own elements as a local element range of the extended slab."""
        return ((self.k0 - self.kA) * self.elems_per_layer, (self.k1 - self.kA) * self.elems_per_layer)

    @property
    def global_elem_offset(self) -> int:
        return self.k0 * self.elems_per_layer

    def plane_rows(self, k: int) -> tuple[int, int]:
        """Local node range of global node plane k."""
        lo = (k - self.kA) * self.plane
        return lo, lo + self.plane

    @property
    def owned_rows(self) -> tuple[int, int]:
        first = self.k0 + (1 if self.rank > 0 else 0)
        return (first - self.kA) * self.plane, (self.k1 - self.kA + 1) * self.plane

    def interfaces(self) -> list[tuple[int, int]]:
        """(neighbour rank, global plane) for each interface of this rank."""
        out = []
        if self.rank > 0:
            out.append((self.rank - 1, self.k0))
        if self.rank < self.world - 1:
            out.append((self.rank + 1, self.k1))
        return out


def _exchange(sends: list[tuple[int, torch.Tensor]], group=None) -> list[torch.Tensor]:
    """Grouped point-to-point exchange; returns one received buffer per send."""
    recvs = [torch.empty_like(t) for _, t in sends]
    ops = []
    for (peer, t), r in zip(sends, recvs):
        ops.append(dist.P2POp(dist.isend, t, peer, group))
        ops.append(dist.P2POp(dist.irecv, r, peer, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    return recvs


def halo_sum_nodes(layout: SlabLayout, x: torch.Tensor, group=None) -> torch.Tensor:
    """Sum a node-major field (x[n] or x[n, c]) across every interface plane,
    in place: both copies of an interface row end up with mine + theirs."""
    segs = [(peer, layout.plane_rows(k)) for peer, k in layout.interfaces()]
    sends = [(peer, x[lo:hi].contiguous()) for peer, (lo, hi) in segs]
    recvs = _exchange(sends, group)
    for (peer, (lo, hi)), r in zip(segs, recvs):
        x[lo:hi] += r
    return x


def interface_segments(layout: SlabLayout, rowptr) -> list[tuple[int, int, int]]:
    """(peer, first entry, end entry) of each interface plane's CSR rows."""
    segs = []
    for peer, k in layout.interfaces():
        lo, hi = layout.plane_rows(k)
        segs.append((peer, int(rowptr[lo]), int(rowptr[hi])))
    return segs


def halo_sum_rows(layout: SlabLayout, rowptr: torch.Tensor, vals: torch.Tensor, nmat: int = 1,
                  nnz: int | None = None, group=None, segs=None) -> torch.Tensor:
    """Sum the CSR values of every interface-plane row across the interface,
    in place.  vals holds nmat matrices back to back (vals[m*nnz + k]); the
    interface rows are contiguous, and have identical global column lists on
    both sides (ghost layers), so the segments line up entry for entry."""
    if nnz is None:
        nnz = vals.numel() // nmat
    if segs is None:
        segs = interface_segments(layout, rowptr)
    sends = []
    for peer, a, b in segs:
        parts = [vals[m * nnz + a:m * nnz + b] for m in range(nmat)]
        sends.append((peer, torch.cat(parts) if nmat > 1 else parts[0].contiguous()))
    recvs = _exchange(sends, group)
    for (peer, a, b), r in zip(segs, recvs):
        w = b - a
        for m in range(nmat):
            vals[m * nnz + a:m * nnz + b] += r[m * w:(m + 1) * w]
    return vals


class SlabDomain:
    """One rank's slab of an (nx, ny, nz) box mesh on its GPU: local mesh
    (own + ghost layers), CSR graph of the extended slab, an assembly
    context integrating own elements only, and the halo sums."""

    def __init__(self, layout: SlabLayout, mesh, ctx, group=None):
        self.layout, self.mesh, self.ctx, self.group = layout, mesh, ctx, group
        self.segs = interface_segments(layout, ctx.pattern.rowptr)  # host copy, once

    @classmethod
    def build(cls, nx: int, ny: int, nz: int, rank: int, world: int,
              etype: ElementType = ElementType.TET04, vector_size: int = 8, group=None,
              lengths=(1.0, 1.0, 1.0)) -> "SlabDomain":
        from . import _lib
        from .assembly import AssemblyContext
        from .elements import ETYPE_ID, NNODES
        from .mesh import ElementGroup, Mesh
        from .sparse import build_node_pattern

        L = SlabLayout.make(nx, ny, nz, rank, world, etype)
        dev = _lib.device()
        coords = torch.empty((L.nnode, 3), dtype=torch.float64, device=dev)
        _lib.call("fpb_grid_coords_slab", nx, ny, nz, L.kA, L.nplanes, float(lengths[0]),
                  float(lengths[1]), float(lengths[2]), coords.data_ptr(), _lib.stream())
        nlay = L.kB - L.kA
        conn = torch.empty((nlay * L.elems_per_layer, NNODES[etype]), dtype=torch.int32, device=dev)
        _lib.call("fpb_box_conn", ETYPE_ID[etype], nx, ny, nlay, conn.data_ptr(), _lib.stream())
        e0, e1 = L.own_elems
        ext = Mesh(3, coords, [ElementGroup(etype, conn)])
        pattern = build_node_pattern(ext)  # own + ghost elements
        own = Mesh(3, coords, [ElementGroup(etype, conn[e0:e1].contiguous())])
        ctx = AssemblyContext.build(own, vector_size, pattern=pattern)
        return cls(L, own, ctx, group)

    def halo_sum_rhs(self, rhs: torch.Tensor) -> torch.Tensor:
        return halo_sum_nodes(self.layout, rhs, self.group)

    def halo_sum_matrix(self, vals: torch.Tensor, nmat: int = 1) -> torch.Tensor:
        return halo_sum_rows(self.layout, self.ctx.pattern.rowptr_d, vals, nmat, self.ctx.pattern.nnz,
                             self.group, self.segs)
