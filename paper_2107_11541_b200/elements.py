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
#: polynomial degree up to which each rule is exact (elements.py:63-70)
QUADRATURE_DEGREE = {ElementType.TRI03: 2, ElementType.QUAD04: 3, ElementType.TET04: 2,
                     ElementType.PYR05: 2, ElementType.HEX08: 3}
#: outward-oriented faces as local node indices (elements.py:73-86)
ELEMENT_FACES = {
    ElementType.TRI03: ((0, 1), (1, 2), (2, 0)),
    ElementType.QUAD04: ((0, 1), (1, 2), (2, 3), (3, 0)),
    ElementType.TET04: ((0, 2, 1), (0, 1, 3), (1, 2, 3), (0, 3, 2)),
    ElementType.PYR05: ((0, 3, 2, 1), (0, 1, 4), (1, 2, 4), (2, 3, 4), (3, 0, 4)),
    ElementType.HEX08: ((0, 3, 2, 1), (4, 5, 6, 7), (0, 1, 5, 4), (2, 3, 7, 6), (0, 4, 7, 3), (1, 2, 6, 5)),
}


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


#: shape-function evaluators by type, (pts[np, dim]) -> (N[nn, np], dN[dim, nn, np])
#: (elements.py:230-236)
_SHAPE_FUNCS = {et: (lambda pts, _et=et: _tables(_et, np.asarray(pts, dtype=np.float64))) for et in ElementType}


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


@dataclass
class ElementGeometry:
    """Geometry of one element at the Gauss points (elements.py:278-286):
    detJw[ng] = det J * weight, gradN[dim, nn, ng] physical gradients."""

    detJw: np.ndarray
    gradN: np.ndarray


def compute_geometry(ref: ReferenceElement, node_coords) -> ElementGeometry:
    """One element's Gauss-point geometry (elements.py:289-313), evaluated by
    the device geometry kernel (`fpb_geometry`, the same code that validates
    whole meshes).  Raises InvertedElementError(-1, gauss, det) for the first
    Gauss point with det J <= 0, like the reference."""
    import ctypes

    import torch

    from . import _lib
    from .errors import InvertedElementError

    x = np.ascontiguousarray(node_coords, dtype=np.float64)
    if x.shape != (ref.nnodes, ref.dim):
        raise ValueError(f"node_coords must have shape ({ref.nnodes}, {ref.dim})")
    upload_tables(ref.etype)
    dev = _lib.device()
    xd = torch.as_tensor(x, device=dev)
    conn = torch.arange(ref.nnodes, dtype=torch.int32, device=dev).reshape(1, -1)
    detjw = torch.empty((1, ref.ngauss, 1), dtype=torch.float64, device=dev)
    gradn = torch.empty((1, ref.dim, ref.nnodes, ref.ngauss, 1), dtype=torch.float64, device=dev)
    bad_e = np.zeros(1, dtype=np.int64)
    bad_g = np.zeros(1, dtype=np.int32)
    rc = _lib.load().fpb_geometry(ETYPE_ID[ref.etype], 1, 1, conn.data_ptr(), xd.data_ptr(), detjw.data_ptr(),
                                  gradn.data_ptr(), bad_e.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                  bad_g.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), _lib.stream())
    if rc == _lib.FPB_EINVERTED:
        ig = int(bad_g[0])
        # det for the message only (the device reports where, not the value)
        raise InvertedElementError(-1, ig, float(np.linalg.det(x.T @ ref.dN[:, :, ig].T)))
    _lib.check(rc, "fpb_geometry")
    return ElementGeometry(detJw=detjw.reshape(ref.ngauss).cpu().numpy(),
                           gradN=gradn.reshape(ref.dim, ref.nnodes, ref.ngauss).cpu().numpy())


def integrate_reference_monomial(etype: ElementType, powers) -> float:
    """Quadrature value of x^a y^b (z^c) over the reference domain
    (elements.py:316-328) — a property of the rule tables only."""
    ref = reference_element(etype)
    vals = np.ones(ref.ngauss)
    for d, p in enumerate(powers):
        if p:
            vals = vals * ref.gauss_points[:, d] ** p
    return float(np.dot(vals, ref.weights))


@dataclass(frozen=True)
class FaceRule:
    """Quadrature and shape tables of a boundary face (elements.py:331-345):
    dN is [face_dim, node, gauss point]."""

    nnodes: int
    dim: int
    ngauss: int
    weights: np.ndarray
    N: np.ndarray
    dN: np.ndarray


@lru_cache(maxsize=None)
def face_rule(nnodes: int) -> FaceRule:
    """Face rule for `nnodes`-node faces (elements.py:348-363): 2-point Gauss
    on [-1, 1] for edges, the TRI03 / QUAD04 tables for 3- / 4-node faces."""
    if nnodes == 2:
        pts = np.array([_G2[0], _G2[1]])
        N = np.stack([0.5 * (1.0 - pts), 0.5 * (1.0 + pts)])
        dN = np.empty((1, 2, 2))
        dN[0, 0], dN[0, 1] = -0.5, 0.5
        return FaceRule(2, 1, 2, np.ones(2), N, dN)
    if nnodes in (3, 4):
        ref = reference_element(ElementType.TRI03 if nnodes == 3 else ElementType.QUAD04)
        return FaceRule(nnodes, ref.dim, ref.ngauss, ref.weights, ref.N, ref.dN)
    raise ValueError(f"no face rule for {nnodes}-node faces")
