"""ctypes wrapper of oracle/build/liboracle.so — the C restatement of the
reference packed kernels (TEST/BASELINE INFRASTRUCTURE ONLY; see
fempack_ref.c).  Used by tests and by bench.py's cpu_baseline /
`--impl reference` arm."""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import fempack_np as O

_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "build", "liboracle.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(_LIB)
        _lib.orc_geometry.restype = C.c_int64
        _lib.orc_max_threads.restype = C.c_int
    return _lib


def _p(a, offset_items=0):
    return C.c_void_p(a.ctypes.data + offset_items * a.itemsize)


class PackedGroup:
    """Reference packed state of one element group at pack width vs, with
    cached geometry (the reference's refresh_geometry, assembly.py:121-142).

    cache_geometry=False keeps only the packs and recomputes geometry chunk
    by chunk inside every kernel call (`chunk` packs at a time) — the same
    arithmetic as the cached path (geometry_packed per pack, bit for bit),
    for meshes whose cached gradN would not fit in host memory (config 4's
    20 M hexes: 31 GB at vs = 8)."""

    def __init__(self, etype, conn, coords, vs=8, nthreads=1, cache_geometry=True, chunk=1 << 14):
        self.etype, self.vs, self.nthreads = etype, vs, nthreads
        self.N, self.dN, self.w = O.reference_element(etype)
        self.nn, self.ng, self.dim = self.N.shape[0], self.N.shape[1], self.dN.shape[0]
        self.nelem = conn.shape[0]
        self.coords = np.ascontiguousarray(coords)
        self.lane_conn, self.elem_index = O.build_packs(conn.astype(np.int64), vs)
        self.npacks = self.lane_conn.shape[0]
        self.cached = cache_geometry
        self.chunk = self.npacks if cache_geometry else min(chunk, self.npacks)
        self.detjw = np.zeros((self.chunk, self.ng, vs))
        self.gradn = np.zeros((self.chunk, self.dim, self.nn, self.ng, vs))
        if cache_geometry:
            self._geometry(0, self.npacks)

    def _geometry(self, p0, p1):
        bad_g = C.c_int(-1)
        bad = lib().orc_geometry(
            C.c_int64(p1 - p0), self.nn, self.ng, self.dim, self.vs, C.c_int64(self.nelem - p0 * self.vs),
            _p(self.lane_conn, p0 * self.nn * self.vs), _p(self.coords), _p(self.dN), _p(self.w),
            _p(self.detjw), _p(self.gradn), C.byref(bad_g), self.nthreads)
        if bad >= 0:
            raise ArithmeticError(f"inverted element {p0 * self.vs + bad} gauss {bad_g.value}")

    def _chunks(self):
        """(first pack, pack count) per kernel call; geometry refreshed per chunk."""
        if self.cached:
            yield 0, self.npacks
            return
        for p0 in range(0, self.npacks, self.chunk):
            p1 = min(p0 + self.chunk, self.npacks)
            self._geometry(p0, p1)
            yield p0, p1 - p0

    def momentum_rhs(self, vel, rho, mu, rhs):
        vel = np.ascontiguousarray(vel)
        for p0, np_ in self._chunks():
            lib().orc_momentum_rhs(C.c_int64(np_), self.nn, self.ng, self.dim, self.vs,
                                   _p(self.lane_conn, p0 * self.nn * self.vs), _p(self.N), _p(self.detjw),
                                   _p(self.gradn), _p(vel), C.c_double(rho), C.c_double(mu), _p(rhs),
                                   self.nthreads)
        return rhs

    def scalar_rhs(self, vel, phi, kappa, rhs):
        vel, phi = np.ascontiguousarray(vel), np.ascontiguousarray(phi)
        for p0, np_ in self._chunks():
            lib().orc_scalar_rhs(C.c_int64(np_), self.nn, self.ng, self.dim, self.vs,
                                 _p(self.lane_conn, p0 * self.nn * self.vs), _p(self.N), _p(self.detjw),
                                 _p(self.gradn), _p(vel), _p(phi), C.c_double(kappa), _p(rhs), self.nthreads)
        return rhs

    def convection(self, vel, pos_packed, vals):
        vel = np.ascontiguousarray(vel)
        for p0, np_ in self._chunks():
            lib().orc_convection(C.c_int64(np_), self.nn, self.ng, self.dim, self.vs,
                                 _p(self.lane_conn, p0 * self.nn * self.vs), _p(self.N), _p(self.detjw),
                                 _p(self.gradn), _p(vel), _p(pos_packed, p0 * self.nn * self.nn * self.vs),
                                 _p(vals), self.nthreads)
        return vals


def spmv(rowptr, colind, vals, x, nthreads=1):
    y = np.empty(rowptr.size - 1)
    lib().orc_spmv(C.c_int64(y.size), _p(rowptr), _p(colind), _p(vals), _p(x), _p(y), nthreads)
    return y


def max_threads() -> int:
    """Host threads this process may run on (its CPU affinity), not
    omp_get_max_threads(): torchrun exports OMP_NUM_THREADS=1 to every rank,
    and the baseline should use every core it is allowed."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or int(lib().orc_max_threads())
