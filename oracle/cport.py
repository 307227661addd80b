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


def _p(a):
    return C.c_void_p(a.ctypes.data)


class PackedGroup:
    """Reference packed state of one element group at pack width vs, with
    cached geometry (the reference's refresh_geometry, assembly.py:121-142)."""

    def __init__(self, etype, conn, coords, vs=8, nthreads=1):
        self.etype, self.vs, self.nthreads = etype, vs, nthreads
        self.N, self.dN, self.w = O.reference_element(etype)
        self.nn, self.ng, self.dim = self.N.shape[0], self.N.shape[1], self.dN.shape[0]
        self.nelem = conn.shape[0]
        self.lane_conn, self.elem_index = O.build_packs(conn.astype(np.int64), vs)
        self.npacks = self.lane_conn.shape[0]
        self.detjw = np.zeros((self.npacks, self.ng, vs))
        self.gradn = np.zeros((self.npacks, self.dim, self.nn, self.ng, vs))
        bad_g = C.c_int(-1)
        bad = lib().orc_geometry(
            C.c_int64(self.npacks), self.nn, self.ng, self.dim, vs, C.c_int64(self.nelem),
            _p(self.lane_conn), _p(np.ascontiguousarray(coords)), _p(self.dN), _p(self.w),
            _p(self.detjw), _p(self.gradn), C.byref(bad_g), nthreads)
        if bad >= 0:
            raise ArithmeticError(f"inverted element {bad} gauss {bad_g.value}")

    def momentum_rhs(self, vel, rho, mu, rhs):
        lib().orc_momentum_rhs(C.c_int64(self.npacks), self.nn, self.ng, self.dim, self.vs,
                               _p(self.lane_conn), _p(self.N), _p(self.detjw), _p(self.gradn),
                               _p(np.ascontiguousarray(vel)), C.c_double(rho), C.c_double(mu),
                               _p(rhs), self.nthreads)
        return rhs

    def convection(self, vel, pos_packed, vals):
        lib().orc_convection(C.c_int64(self.npacks), self.nn, self.ng, self.dim, self.vs,
                             _p(self.lane_conn), _p(self.N), _p(self.detjw), _p(self.gradn),
                             _p(np.ascontiguousarray(vel)), _p(pos_packed), _p(vals), self.nthreads)
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
