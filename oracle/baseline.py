"""CPU baseline workload (BASELINE INFRASTRUCTURE ONLY): the reference's
bench step for config 2 — `assemble_rhs(MOMENTUM_RHS)` plus the continuity
matrices `gradient_matrices` (3x CONVECTION with unit e_k), packed layout,
vs=8 (bench.py:193-211, timeloop.py:159-171) — run by the C restatement of
the reference kernels (oracle/fempack_ref.c) on the host cores.

Setup follows the reference (mesh, CSR pattern, element->CSR map, cached
geometry; all NumPy/C oracle, no GPU code) and is not timed, exactly as the
reference bench keeps refresh_geometry out of its timed region
(bench.py:195).  Each step allocates zeroed outputs like the reference."""

from __future__ import annotations

import time

import numpy as np

from . import cport
from . import fempack_np as O


class CpuWorkload:
    def __init__(self, nx: int, ny: int, nz: int, nthreads: int, vs: int = 8):
        self.mesh = O.box(O.TET04, nx, ny, nz)
        (et, conn), = self.mesh.groups
        self.nthreads = nthreads
        self.rowptr, self.colind = O.build_node_pattern(self.mesh.nnode, [conn])
        self.group = cport.PackedGroup(et, conn, self.mesh.coords, vs=vs, nthreads=nthreads)
        pos = O.matrix_positions(conn, self.rowptr, self.colind)
        self.pos_packed = np.ascontiguousarray(O.packed_positions(pos, self.group.elem_index))
        del pos
        self.vel, _ = O.bench_fields(self.mesh.nnode, 3)
        self.units = []
        for k in range(3):
            u = np.zeros((self.mesh.nnode, 3))
            u[:, k] = 1.0
            self.units.append(u)
        self.nelem = self.mesh.nelem

    def step(self):
        rhs = np.zeros((self.mesh.nnode, 3))
        self.group.momentum_rhs(self.vel, 1.0, 1e-2, rhs)
        mats = []
        for k in range(3):
            vals = np.zeros(self.colind.size)
            self.group.convection(self.units[k], self.pos_packed, vals)
            mats.append(vals)
        return rhs, mats

    def time_steps(self, steps: int, warmup: int) -> list[float]:
        for _ in range(warmup):
            self.step()
        out = []
        for _ in range(steps):
            t0 = time.perf_counter()
            self.step()
            out.append(time.perf_counter() - t0)
        return out
