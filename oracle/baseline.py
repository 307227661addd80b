"""CPU baseline workload (BASELINE INFRASTRUCTURE ONLY): the reference's
bench step run by the C restatement of the reference packed kernels
(oracle/fempack_ref.c) on the host cores, on a z-slab sample of a config
mesh.

The sample is the first `kz` cell layers of the (nx, ny, nz) box mesh,
exactly as `generate_box_mesh` numbers and places them: cells are visited
k-major and nodes numbered i + (nx+1)(j + (ny+1)k) (mesh.py:183-184,
:220-224), so the slab's connectivity is the box (nx, ny, kz)'s and its
nodes are the first (kz+1) node planes of the full mesh, with the full
mesh's coordinates and the leading rows of its default_rng(0) fields
(bench.py:178-179, :196-197).  The per-element work is the full mesh's;
elements/s measured on the slab is reported as the extrapolated rate of
the whole mesh (chunk-wise reference kernels at config
4/5 sizes, labelled extrapolated).

Step kinds (the reference's calls, packed layout, vs = 8):
  "momentum"  assemble_rhs(MOMENTUM_RHS, rho 1, mu 1e-2)    _kernels.py:320-382
  "gradients" gradient_matrices = 3 x CONVECTION(e_k)       timeloop.py:159-171
  "scalars"   3 x assemble_rhs(SCALAR_RHS, kappa = D = 1e-2) _kernels.py:420-461

Setup (mesh, CSR pattern, element->CSR map, cached geometry) follows the
reference and is not timed, as the reference bench keeps refresh_geometry
out of its timed region (bench.py:195).  Each step allocates zeroed
outputs like the reference."""

from __future__ import annotations

import time

import numpy as np

from . import cport
from . import fempack_np as O

ETYPES = {"TET04": O.TET04, "HEX08": O.HEX08}


def slab_sample(etype: str, nx: int, ny: int, nz: int, kz: int):
    """(conn int64, coords, velocity, [3 scalars]) of the first kz cell
    layers of the (nx, ny, nz) unit-cube box mesh."""
    et = ETYPES[etype]
    _, _, groups = O.generate_box_mesh(et, nx, ny, kz)
    (_, conn), = groups
    plane = (nx + 1) * (ny + 1)
    nloc = plane * (kz + 1)
    coords = O.grid_coords(nx, ny, nz, (1.0, 1.0, 1.0), 3)[:nloc].copy()
    nglob = plane * (nz + 1)
    rng = np.random.default_rng(0)
    vel = rng.standard_normal((nglob, 3))[:nloc].copy()
    scal = [rng.standard_normal(nglob)[:nloc].copy() for _ in range(3)]
    return conn, coords, vel, scal


class CpuWorkload:
    def __init__(self, etype: str, nx: int, ny: int, nz: int, kz: int, nthreads: int,
                 kinds=("momentum", "gradients"), vs: int = 8):
        conn, coords, self.vel, self.scal = slab_sample(etype, nx, ny, nz, kz)
        self.nnode = coords.shape[0]
        self.nelem = conn.shape[0]
        self.kinds = tuple(kinds)
        self.nthreads = nthreads
        self.group = cport.PackedGroup(ETYPES[etype], conn, coords, vs=vs, nthreads=nthreads)
        self.nnz = 0
        if "gradients" in self.kinds:
            self.rowptr, self.colind = O.build_node_pattern(self.nnode, [conn])
            pos = O.matrix_positions(conn, self.rowptr, self.colind)
            self.pos_packed = np.ascontiguousarray(O.packed_positions(pos, self.group.elem_index))
            del pos
            self.nnz = self.colind.size
            self.units = []
            for k in range(3):
                u = np.zeros((self.nnode, 3))
                u[:, k] = 1.0
                self.units.append(u)

    def step(self):
        out = {}
        if "momentum" in self.kinds:
            out["momentum"] = self.group.momentum_rhs(self.vel, 1.0, 1e-2, np.zeros((self.nnode, 3)))
        if "gradients" in self.kinds:
            out["gradients"] = [self.group.convection(self.units[k], self.pos_packed, np.zeros(self.nnz))
                                for k in range(3)]
        if "scalars" in self.kinds:
            out["scalars"] = [self.group.scalar_rhs(self.vel, self.scal[f], 1e-2, np.zeros(self.nnode))
                              for f in range(3)]
        return out

    def time_steps(self, steps: int, warmup: int) -> list[float]:
        for _ in range(warmup):
            self.step()
        out = []
        for _ in range(steps):
            t0 = time.perf_counter()
            self.step()
            out.append(time.perf_counter() - t0)
        return out
