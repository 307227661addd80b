"""Reference elements: quadrature rules and shape-function tables.

Same five first-order types, rules and tables as the reference
(elements.py:28-274); the tables are the constant inputs of every assembly
kernel and are uploaded once per device into `__constant__` memory
(`fpb_set_reference_element`).  They are bitwise identical to the
reference's (tests/test_host.py::test_tables_match_reference).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum
from functools import lru_cache

import numpy as np


class ElementType(Enum):
    TRI03 = "TRI03"
    QUAD04 = "QUAD04"
    TET04 = "TET04"
    PYR05 = "PYR05"
    HEX08 = "HEX08"


#: C-ABI enum value (include/fempack_b200.h fpb_etype)
ETYPE_ID = {ElementType.TRI03: 0, ElementType.QUAD04: 1, ElementType.TET04: 2,
            ElementType.PYR05: 3, ElementType.HEX08: 4}
NNODES = {ElementType.TRI03: 3, ElementType.QUAD04: 4, ElementType.TET04: 4,
          ElementType.PYR05: 5, ElementType.HEX08: 8}
DIM = {ElementType.TRI03: 2, ElementType.QUAD04: 2, ElementType.TET04: 3,
       ElementType.PYR05: 3, ElementType.HEX08: 3}
REFERENCE_VOLUME = {ElementType.TRI03: 0.5, ElementType.QUAD04: 4.0, ElementType.TET04: 1.0 / 6.0,
                    ElementType.PYR05: 4.0 / 3.0, ElementType.HEX08: 8.0}


@dataclass(frozen=True)
class ReferenceElement:
    """N[nn, ng], dN[dim, nn, ng], weights[ng] at the Gauss points."""

    etype: ElementType
    dim: int
    nnodes: int
    ngauss: int
    gauss_points: np.ndarray
    weights: np.ndarray
    N: np.ndarray
    dN: np.ndarray


_G2 = (-1.0 / math.sqrt(3.0), 1.0 / math.sqrt(3.0))
_SQ_CORNERS = ((-1, -1), (1, -1), (1, 1), (-1, 1))
_CUBE_CORNERS = tuple((x, y, z) for z in (-1, 1) for (x, y) in _SQ_CORNERS)


def _points_and_weights(et: ElementType):
    if et is ElementType.TRI03:
        return np.array([(1 / 6, 1 / 6), (2 / 3, 1 / 6), (1 / 6, 2 / 3)]), np.full(3, 1 / 6)
    if et is ElementType.QUAD04:
        return np.array([(x, y) for y in _G2 for x in _G2]), np.ones(4)
    if et is ElementType.TET04:
        hi = (5.0 + 3.0 * math.sqrt(5.0)) / 20.0
        lo = (5.0 - math.sqrt(5.0)) / 20.0
        return np.array([(lo, lo, lo), (hi, lo, lo), (lo, hi, lo), (lo, lo, hi)]), np.full(4, 1 / 24)
    if et is ElementType.HEX08:
        return np.array([(x, y, z) for z in _G2 for y in _G2 for x in _G2]), np.ones(8)
    # PYR05: 2x2 Gauss on the base times 2-point Gauss-Jacobi (weight (1-z)^2)
    r10 = math.sqrt(10)
    axial = ((1 / 3 - r10 / 15, 1 / 6 + r10 / 48), (1 / 3 + r10 / 15, 1 / 6 - r10 / 48))
    pts = [(a * (1.0 - z), b * (1.0 - z), z) for z, _ in axial for b in _G2 for a in _G2]
    wts = [wz for _, wz in axial for _b in _G2 for _a in _G2]
    return np.array(pts), np.array(wts)


def _tables(et: ElementType, pts: np.ndarray):
    ng = pts.shape[0]
    if et is ElementType.TRI03:
        xi, eta = pts.T
        N = np.stack([1.0 - xi - eta, xi, eta])
        dN = np.zeros((2, 3, ng))
        dN[0, 0], dN[0, 1], dN[1, 0], dN[1, 2] = -1.0, 1.0, -1.0, 1.0
        return N, dN
    if et is ElementType.TET04:
        xi, eta, zeta = pts.T
        N = np.stack([1.0 - xi - eta - zeta, xi, eta, zeta])
        dN = np.zeros((3, 4, ng))
        dN[:, 0] = -1.0
        dN[0, 1] = dN[1, 2] = dN[2, 3] = 1.0
        return N, dN
    if et is ElementType.QUAD04:
        xi, eta = pts.T
        N, dN = np.empty((4, ng)), np.empty((2, 4, ng))
        for a, (xc, yc) in enumerate(_SQ_CORNERS):
            fx, fy = 1 + float(xc) * xi, 1 + float(yc) * eta
            N[a] = 0.25 * fx * fy
            dN[0, a] = 0.25 * xc * fy
            dN[1, a] = 0.25 * yc * fx
        return N, dN
    if et is ElementType.HEX08:
        xi, eta, zeta = pts.T
        N, dN = np.empty((8, ng)), np.empty((3, 8, ng))
        for a, (xc, yc, zc) in enumerate(_CUBE_CORNERS):
            fx, fy, fz = 1 + float(xc) * xi, 1 + float(yc) * eta, 1 + float(zc) * zeta
            N[a] = 0.125 * fx * fy * fz
            dN[0, a] = 0.125 * xc * fy * fz
            dN[1, a] = 0.125 * yc * fx * fz
            dN[2, a] = 0.125 * zc * fx * fy
        return N, dN
    # PYR05: rational basis, apex (0,0,1); the quadrature never reaches z = 1
    xi, eta, zeta = pts.T
    om = 1.0 - zeta
    safe = np.where(np.abs(om) > 1e-14, om, 1.0)
    r, s = zeta / safe, 1.0 / safe**2
    N, dN = np.empty((5, ng)), np.empty((3, 5, ng))
    for a, ((xc, yc), sg) in enumerate(zip(_SQ_CORNERS, (1.0, -1.0, 1.0, -1.0))):
        N[a] = 0.25 * ((1 + xc * xi) * (1 + yc * eta) - zeta + sg * xi * eta * r)
        dN[0, a] = 0.25 * (xc * (1 + yc * eta) + sg * eta * r)
        dN[1, a] = 0.25 * (yc * (1 + xc * xi) + sg * xi * r)
        dN[2, a] = 0.25 * (-1.0 + sg * xi * eta * s)
    N[4] = zeta
    dN[0, 4] = dN[1, 4] = 0.0
    dN[2, 4] = 1.0
    return N, dN


@lru_cache(maxsize=None)
def reference_element(etype: ElementType) -> ReferenceElement:
    pts, w = _points_and_weights(etype)
    N, dN = _tables(etype, pts)
    arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (pts, w, N, dN)]
    for a in arrs:
        a.flags.writeable = False
    return ReferenceElement(etype, DIM[etype], NNODES[etype], len(w), arrs[0], arrs[1], arrs[2], arrs[3])


_uploaded: set = set()


def upload_tables(etype: ElementType) -> None:
    """Copy one type's tables into device constant memory (once per device)."""
    import torch

    from . import _lib

    lib = _lib.load()
    key = (torch.cuda.current_device(), etype)
    if key in _uploaded:
        return
    ref = reference_element(etype)
    N = np.ascontiguousarray(ref.N)
    dN = np.ascontiguousarray(ref.dN)
    w = np.ascontiguousarray(ref.weights)
    _lib.check(lib.fpb_set_reference_element(ETYPE_ID[etype], ref.nnodes, ref.ngauss, ref.dim,
                                             N.ctypes.data, dN.ctypes.data, w.ctypes.data),
               "fpb_set_reference_element")
    _uploaded.add(key)
