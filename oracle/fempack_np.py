"""CPU oracle (TEST INFRASTRUCTURE ONLY) — NumPy restatement of the reference
`fempack` hot path (arXiv 2107.11541 mini-app, /root/reference/pkg/src/fempack).

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline leg may
import this module, and only as the checker.  The product package
(`paper_2107_11541_b200`) never imports it; the product fails loudly without
its CUDA library.

Parity pinning: every function below is checked against golden vectors that
`tools/make_golden.py` produced by importing the unmodified reference in the
build container (`tests/golden/*.npz`, `tests/test_oracle_golden.py`).

Arithmetic order follows the reference's *packed* kernels element by element
(vectorised over elements instead of over lanes), so per-element results are
bitwise identical to `_kernels.*_packed`; scatters use `np.add.at` in the
reference's (p, i, j, v) order, which is sequential, so global results are
bitwise identical to the reference packed path as well.
"""

from __future__ import annotations

import math

import numpy as np

# --------------------------------------------------------------------------
# reference elements  (elements.py)
# --------------------------------------------------------------------------

TRI03, QUAD04, TET04, PYR05, HEX08 = "TRI03", "QUAD04", "TET04", "PYR05", "HEX08"
NNODES = {TRI03: 3, QUAD04: 4, TET04: 4, PYR05: 5, HEX08: 8}  # elements.py:36-42
DIM = {TRI03: 2, QUAD04: 2, TET04: 3, PYR05: 3, HEX08: 3}  # elements.py:45-51
_SQ3 = 1.0 / math.sqrt(3.0)  # elements.py:24


def _shape(etype, pts):
    """Shape tables N[nn, ng], dN[dim, nn, ng] (elements.py:118-204)."""
    ng = len(pts)
    if etype == TRI03:  # elements.py:118-124
        xi, eta = pts[:, 0], pts[:, 1]
        N = np.stack([1.0 - xi - eta, xi, eta])
        dN = np.zeros((2, 3, ng))
        dN[0, 0], dN[0, 1] = -1.0, 1.0
        dN[1, 0], dN[1, 2] = -1.0, 1.0
        return N, dN
    if etype == QUAD04:  # elements.py:127-136
        corners = np.array([(-1, -1), (1, -1), (1, 1), (-1, 1)], dtype=float)
        xi, eta = pts[:, 0], pts[:, 1]
        N = np.empty((4, ng))
        dN = np.empty((2, 4, ng))
        for i, (xc, yc) in enumerate(corners):
            N[i] = 0.25 * (1 + xc * xi) * (1 + yc * eta)
            dN[0, i] = 0.25 * xc * (1 + yc * eta)
            dN[1, i] = 0.25 * yc * (1 + xc * xi)
        return N, dN
    if etype == TET04:  # elements.py:139-145
        xi, eta, zeta = pts[:, 0], pts[:, 1], pts[:, 2]
        N = np.stack([1.0 - xi - eta - zeta, xi, eta, zeta])
        dN = np.zeros((3, 4, ng))
        dN[:, 0] = -1.0
        dN[0, 1] = dN[1, 2] = dN[2, 3] = 1.0
        return N, dN
    if etype == HEX08:  # elements.py:148-171
        corners = np.array(
            [(-1, -1, -1), (1, -1, -1), (1, 1, -1), (-1, 1, -1),
             (-1, -1, 1), (1, -1, 1), (1, 1, 1), (-1, 1, 1)], dtype=float)
        xi, eta, zeta = pts[:, 0], pts[:, 1], pts[:, 2]
        N = np.empty((8, ng))
        dN = np.empty((3, 8, ng))
        for i, (xc, yc, zc) in enumerate(corners):
            N[i] = 0.125 * (1 + xc * xi) * (1 + yc * eta) * (1 + zc * zeta)
            dN[0, i] = 0.125 * xc * (1 + yc * eta) * (1 + zc * zeta)
            dN[1, i] = 0.125 * yc * (1 + xc * xi) * (1 + zc * zeta)
            dN[2, i] = 0.125 * zc * (1 + xc * xi) * (1 + yc * eta)
        return N, dN
    if etype == PYR05:  # elements.py:174-196
        xi, eta, zeta = pts[:, 0], pts[:, 1], pts[:, 2]
        om = 1.0 - zeta
        safe = np.where(np.abs(om) > 1e-14, om, 1.0)
        r = zeta / safe
        s = 1.0 / safe**2
        N = np.empty((5, ng))
        dN = np.empty((3, 5, ng))
        signs = (1.0, -1.0, 1.0, -1.0)
        corners = ((-1, -1), (1, -1), (1, 1), (-1, 1))
        for i, ((xc, yc), sg) in enumerate(zip(corners, signs)):
            N[i] = 0.25 * ((1 + xc * xi) * (1 + yc * eta) - zeta + sg * xi * eta * r)
            dN[0, i] = 0.25 * (xc * (1 + yc * eta) + sg * eta * r)
            dN[1, i] = 0.25 * (yc * (1 + xc * xi) + sg * xi * r)
            dN[2, i] = 0.25 * (-1.0 + sg * xi * eta * s)
        N[4] = zeta
        dN[0, 4] = dN[1, 4] = 0.0
        dN[2, 4] = 1.0
        return N, dN
    raise ValueError(etype)


def _rule(etype):
    """Quadrature points and weights (elements.py:207-246)."""
    if etype == TRI03:
        return np.array([(1 / 6, 1 / 6), (2 / 3, 1 / 6), (1 / 6, 2 / 3)]), np.full(3, 1 / 6)
    if etype == QUAD04:
        g = [-_SQ3, _SQ3]
        return np.array([(x, y) for y in g for x in g]), np.ones(4)
    if etype == TET04:
        a = (5.0 + 3.0 * math.sqrt(5.0)) / 20.0
        b = (5.0 - math.sqrt(5.0)) / 20.0
        return np.array([(b, b, b), (a, b, b), (b, a, b), (b, b, a)]), np.full(4, 1 / 24)
    if etype == HEX08:
        g = [-_SQ3, _SQ3]
        return np.array([(x, y, z) for z in g for y in g for x in g]), np.ones(8)
    if etype == PYR05:
        zj = np.array([1 / 3 - math.sqrt(10) / 15, 1 / 3 + math.sqrt(10) / 15])
        wj = np.array([1 / 6 + math.sqrt(10) / 48, 1 / 6 - math.sqrt(10) / 48])
        g = [-_SQ3, _SQ3]
        pts, wts = [], []
        for z, wz in zip(zj, wj):
            for b in g:
                for a in g:
                    pts.append((a * (1.0 - z), b * (1.0 - z), z))
                    wts.append(wz)
        return np.array(pts), np.array(wts)
    raise ValueError(etype)


def reference_element(etype):
    """(N[nn,ng], dN[dim,nn,ng], w[ng]) — elements.py:258-274."""
    pts, w = _rule(etype)
    N, dN = _shape(etype, pts)
    return np.ascontiguousarray(N), np.ascontiguousarray(dN), w


# --------------------------------------------------------------------------
# synthetic meshes  (mesh.py)
# --------------------------------------------------------------------------

_HEX_CORNERS = ((0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0),
                (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1))  # mesh.py:190-199
_HEX_INWARD_FACES = ((0, 1, 2, 3), (4, 7, 6, 5), (0, 4, 5, 1),
                     (2, 6, 7, 3), (0, 3, 7, 4), (1, 5, 6, 2))  # mesh.py:202-209
_KUHN_PERMS = ((0, 1, 2), (1, 2, 0), (2, 0, 1), (0, 2, 1), (2, 1, 0), (1, 0, 2))
_KUHN_ODD = (False, False, False, True, True, True)  # mesh.py:212-213


def grid_coords(nx, ny, nz, lengths, dim):
    """Structured-grid node coordinates, i fastest (mesh.py:158-187)."""
    if dim == 2:
        xs = np.linspace(0.0, lengths[0], nx + 1)
        ys = np.linspace(0.0, lengths[1], ny + 1)
        X, Y = np.meshgrid(xs, ys, indexing="ij")
        return np.stack([X.T.ravel(), Y.T.ravel()], axis=1)
    xs = np.linspace(0.0, lengths[0], nx + 1)
    ys = np.linspace(0.0, lengths[1], ny + 1)
    zs = np.linspace(0.0, lengths[2], nz + 1)
    Z, Y, X = np.meshgrid(zs, ys, xs, indexing="ij")
    return np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1)


def _cell_ijk(nx, ny, nz):
    """Cells visited k-major, i fastest (mesh.py:220-224)."""
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    return i.ravel(), j.ravel(), k.ravel()


def _hex_cells(nx, ny, nz):
    i, j, k = _cell_ijk(nx, ny, nz)

    def nid(a, b, c):
        return a + (nx + 1) * (b + (ny + 1) * c)  # mesh.py:183-184

    return np.stack([nid(i + di, j + dj, k + dk) for di, dj, dk in _HEX_CORNERS], axis=1)


def generate_box_mesh(etype, nx, ny, nz=1, lengths=None):
    """Returns (dim, coords, [(etype, conn int64)]) — mesh.py:227-289."""
    dim = DIM[etype]
    if lengths is None:
        lengths = (1.0,) * dim
    if dim == 2:
        coords = grid_coords(nx, ny, 0, lengths, 2)
        jj, ii = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
        i, j = ii.ravel(), jj.ravel()

        def nid(a, b):
            return a + (nx + 1) * b

        v = np.stack([nid(i, j), nid(i + 1, j), nid(i + 1, j + 1), nid(i, j + 1)], axis=1)
        if etype == QUAD04:
            conn = v
        else:  # mesh.py:252-254, two triangles per cell
            conn = np.stack([v[:, [0, 1, 2]], v[:, [0, 2, 3]]], axis=1).reshape(-1, 3)
        return 2, coords, [(etype, conn.astype(np.int64))]
    if etype == PYR05:
        return generate_mixed_mesh(nx, ny, nz, 1.0, lengths)
    coords = grid_coords(nx, ny, nz, lengths, 3)
    if etype == HEX08:
        return 3, coords, [(HEX08, _hex_cells(nx, ny, nz).astype(np.int64))]
    # Kuhn subdivision (mesh.py:268-282)
    i, j, k = _cell_ijk(nx, ny, nz)

    def nid(c):
        return c[0] + (nx + 1) * (c[1] + (ny + 1) * c[2])

    v7 = nid((i + 1, j + 1, k + 1))
    tets = []
    for perm, odd in zip(_KUHN_PERMS, _KUHN_ODD):
        p = [i.copy(), j.copy(), k.copy()]
        v0 = nid(p)
        p[perm[0]] = p[perm[0]] + 1
        v1 = nid(p)
        p[perm[1]] = p[perm[1]] + 1
        v2 = nid(p)
        tets.append(np.stack([v0, v1, v7, v2] if odd else [v0, v1, v2, v7], axis=1))
    conn = np.stack(tets, axis=1).reshape(-1, 4)
    return 3, coords, [(TET04, conn.astype(np.int64))]


def generate_mixed_mesh(nx, ny, nz, fraction=0.5, lengths=None):
    """Pyramid layers (i < ceil(fraction*nx)) then hexes — mesh.py:292-336."""
    if lengths is None:
        lengths = (1.0, 1.0, 1.0)
    coords = grid_coords(nx, ny, nz, lengths, 3)
    nlayers = int(np.ceil(fraction * nx))
    cells = _hex_cells(nx, ny, nz)
    i, _, _ = _cell_ijk(nx, ny, nz)
    is_pyr = i < nlayers
    pc = cells[is_pyr]
    groups = []
    if pc.shape[0]:
        # centre = coords[cell].mean(axis=0): numpy pairwise-sums 8 rows
        centers = coords[pc].mean(axis=1)
        cid = coords.shape[0] + np.arange(pc.shape[0])
        pyr = np.stack(
            [np.concatenate([pc[:, list(f)], cid[:, None]], axis=1) for f in _HEX_INWARD_FACES],
            axis=1,
        ).reshape(-1, 5)
        coords = np.vstack([coords, centers])
        groups.append((PYR05, pyr.astype(np.int64)))
    hc = cells[~is_pyr]
    if hc.shape[0]:
        groups.append((HEX08, hc.astype(np.int64)))
    return 3, coords, groups


# --------------------------------------------------------------------------
# packing  (packing.py:85-127)
# --------------------------------------------------------------------------

def build_packs(conn, vs, offset=0):
    """(lane_conn[npacks,nn,vs], elem_index[npacks,vs]); tail replicates
    the last element (packing.py:104-115)."""
    ne = conn.shape[0]
    npacks = -(-ne // vs)
    flat = np.empty(npacks * vs, dtype=np.int64)
    flat[:ne] = offset + np.arange(ne)
    flat[ne:] = offset + ne - 1
    elem_index = flat.reshape(npacks, vs)
    lane_conn = np.ascontiguousarray(np.moveaxis(conn[elem_index - offset], 1, 2))
    return lane_conn, elem_index


# --------------------------------------------------------------------------
# CSR pattern and element->CSR map  (sparse.py:59-75, assembly.py:44-52)
# --------------------------------------------------------------------------

def build_node_pattern(n, conns):
    keys = [np.arange(n, dtype=np.int64) * (n + 1)]
    for c in conns:
        keys.append((c[:, :, None] * n + c[:, None, :]).ravel())
    uniq = np.unique(np.concatenate(keys))
    rows = uniq // n
    rowptr = np.zeros(n + 1, dtype=np.int64)
    rowptr[1:] = np.cumsum(np.bincount(rows, minlength=n))
    return rowptr, (uniq % n).astype(np.int64)


def matrix_positions(conn, rowptr, colind):
    n = rowptr.size - 1
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rowptr))
    keys = rows * n + colind
    want = conn[..., :, None] * n + conn[..., None, :]
    pos = np.searchsorted(keys, want)
    if pos.max(initial=0) >= keys.size or not np.array_equal(keys[pos], want):
        raise KeyError("element node pair missing from CSR pattern")
    return pos.astype(np.int64)


def packed_positions(pos_scalar, elem_index, offset=0):
    """pos_packed[p,i,j,v] (assembly.py:89-93)."""
    return np.ascontiguousarray(np.moveaxis(pos_scalar[elem_index - offset], 1, -1))


# --------------------------------------------------------------------------
# element kernels — per-element arithmetic of _kernels.py *_packed
# (vectorised over elements; e is the leading axis)
# --------------------------------------------------------------------------

def geometry(conn, coords, dN, w):
    """detjw[e,g], gradn[e,d,a,g]; first bad (e, g) — _kernels.py:78-147."""
    ne, nn = conn.shape
    dim, _, ng = dN.shape
    xe = coords[conn]  # [e, a, d]
    detjw = np.empty((ne, ng))
    gradn = np.empty((ne, dim, nn, ng))
    bad = (-1, -1)
    for ig in range(ng):
        J = np.empty((ne, dim, dim))
        for d in range(dim):
            for l in range(dim):
                acc = np.zeros(ne)
                for a in range(nn):
                    acc = acc + xe[:, a, d] * dN[l, a, ig]
                J[:, d, l] = acc
        if dim == 2:
            det = J[:, 0, 0] * J[:, 1, 1] - J[:, 0, 1] * J[:, 1, 0]
        else:
            det = (J[:, 0, 0] * (J[:, 1, 1] * J[:, 2, 2] - J[:, 1, 2] * J[:, 2, 1])
                   - J[:, 0, 1] * (J[:, 1, 0] * J[:, 2, 2] - J[:, 1, 2] * J[:, 2, 0])
                   + J[:, 0, 2] * (J[:, 1, 0] * J[:, 2, 1] - J[:, 1, 1] * J[:, 2, 0]))
        nz = np.nonzero(det <= 0.0)[0]
        if nz.size and (bad[0] < 0 or nz[0] < bad[0]):
            bad = (int(nz[0]), ig)
        detjw[:, ig] = det * w[ig]
        inv = 1.0 / det
        Ji = np.empty((ne, dim, dim))
        if dim == 2:
            Ji[:, 0, 0] = J[:, 1, 1] * inv
            Ji[:, 0, 1] = -J[:, 0, 1] * inv
            Ji[:, 1, 0] = -J[:, 1, 0] * inv
            Ji[:, 1, 1] = J[:, 0, 0] * inv
        else:
            Ji[:, 0, 0] = (J[:, 1, 1] * J[:, 2, 2] - J[:, 1, 2] * J[:, 2, 1]) * inv
            Ji[:, 0, 1] = (J[:, 0, 2] * J[:, 2, 1] - J[:, 0, 1] * J[:, 2, 2]) * inv
            Ji[:, 0, 2] = (J[:, 0, 1] * J[:, 1, 2] - J[:, 0, 2] * J[:, 1, 1]) * inv
            Ji[:, 1, 0] = (J[:, 1, 2] * J[:, 2, 0] - J[:, 1, 0] * J[:, 2, 2]) * inv
            Ji[:, 1, 1] = (J[:, 0, 0] * J[:, 2, 2] - J[:, 0, 2] * J[:, 2, 0]) * inv
            Ji[:, 1, 2] = (J[:, 0, 2] * J[:, 1, 0] - J[:, 0, 0] * J[:, 1, 2]) * inv
            Ji[:, 2, 0] = (J[:, 1, 0] * J[:, 2, 1] - J[:, 1, 1] * J[:, 2, 0]) * inv
            Ji[:, 2, 1] = (J[:, 0, 1] * J[:, 2, 0] - J[:, 0, 0] * J[:, 2, 1]) * inv
            Ji[:, 2, 2] = (J[:, 0, 0] * J[:, 1, 1] - J[:, 0, 1] * J[:, 1, 0]) * inv
        for a in range(nn):
            for d in range(dim):
                acc = np.zeros(ne)
                for l in range(dim):
                    acc = acc + Ji[:, l, d] * dN[l, a, ig]
                gradn[:, d, a, ig] = acc
    return detjw, gradn, bad


def mass(detjw, N):  # _kernels.py:163-172
    ne, ng = detjw.shape
    nn = N.shape[0]
    out = np.zeros((ne, nn, nn))
    for ig in range(ng):
        for j in range(nn):
            for i in range(nn):
                out[:, i, j] += detjw[:, ig] * N[j, ig] * N[i, ig]
    return out


def laplacian(detjw, gradn):  # _kernels.py:191-207
    ne, dim, nn, ng = gradn.shape
    out = np.zeros((ne, nn, nn))
    for ig in range(ng):
        for j in range(nn):
            for i in range(nn):
                acc = np.zeros(ne)
                for d in range(dim):
                    acc = acc + gradn[:, d, i, ig] * gradn[:, d, j, ig]
                out[:, i, j] += detjw[:, ig] * acc
    return out


def convection(detjw, gradn, N, conn, vel):  # _kernels.py:238-266
    ne, dim, nn, ng = gradn.shape
    ue = vel[conn]  # [e, a, d]
    out = np.zeros((ne, nn, nn))
    for ig in range(ng):
        ug = []
        for d in range(dim):
            acc = np.zeros(ne)
            for a in range(nn):
                acc = acc + ue[:, a, d] * N[a, ig]
            ug.append(acc)
        for j in range(nn):
            adv = np.zeros(ne)
            for d in range(dim):
                adv = adv + ug[d] * gradn[:, d, j, ig]
            for i in range(nn):
                out[:, i, j] += detjw[:, ig] * adv * N[i, ig]
    return out


def momentum_rhs(detjw, gradn, N, conn, vel, rho, mu):  # _kernels.py:320-382
    ne, dim, nn, ng = gradn.shape
    ue = vel[conn]
    out = np.zeros((ne, nn, dim))
    for ig in range(ng):
        ug = []
        for d in range(dim):
            acc = np.zeros(ne)
            for a in range(nn):
                acc = acc + ue[:, a, d] * N[a, ig]
            ug.append(acc)
        G = [[None] * dim for _ in range(dim)]
        for l in range(dim):
            for k in range(dim):
                acc = np.zeros(ne)
                for a in range(nn):
                    acc = acc + ue[:, a, k] * gradn[:, l, a, ig]
                G[l][k] = acc
        divu = np.zeros(ne)
        for d in range(dim):
            divu = divu + G[d][d]
        S = [[0.5 * (G[l][k] + G[k][l]) for k in range(dim)] for l in range(dim)]
        c = []
        for k in range(dim):
            us = np.zeros(ne)
            gk = np.zeros(ne)
            for l in range(dim):
                us = us + ug[l] * S[l][k]
                gk = gk + ug[l] * G[k][l]
            c.append(2.0 * us + divu * ug[k] - gk)
        for i in range(nn):
            for k in range(dim):
                visc = np.zeros(ne)
                for l in range(dim):
                    visc = visc + S[k][l] * gradn[:, l, i, ig]
                out[:, i, k] -= detjw[:, ig] * (rho * N[i, ig] * c[k] + 2.0 * mu * visc)
    return out


def scalar_rhs(detjw, gradn, N, conn, vel, phi, kappa):  # _kernels.py:420-461
    ne, dim, nn, ng = gradn.shape
    ue = vel[conn]
    fe = phi[conn]
    out = np.zeros((ne, nn))
    for ig in range(ng):
        ug, gphi = [], []
        for d in range(dim):
            au = np.zeros(ne)
            ap = np.zeros(ne)
            for a in range(nn):
                au = au + ue[:, a, d] * N[a, ig]
                ap = ap + fe[:, a] * gradn[:, d, a, ig]
            ug.append(au)
            gphi.append(ap)
        adv = np.zeros(ne)
        for d in range(dim):
            adv = adv + ug[d] * gphi[d]
        for i in range(nn):
            diff = np.zeros(ne)
            for d in range(dim):
                diff = diff + gphi[d] * gradn[:, d, i, ig]
            out[:, i] -= detjw[:, ig] * (N[i, ig] * adv + kappa * diff)
    return out


# --------------------------------------------------------------------------
# global assembly  (assembly.py:209-270, packed path; scatter _kernels.py:473-519)
# --------------------------------------------------------------------------

class OracleMesh:
    """dim, coords, groups [(etype, conn)] in the reference's group order."""

    def __init__(self, dim, coords, groups):
        self.dim, self.coords, self.groups = dim, coords, [g for g in groups if g[1].shape[0]]

    @property
    def nnode(self):
        return self.coords.shape[0]

    @property
    def nelem(self):
        return sum(c.shape[0] for _, c in self.groups)


def box(etype, nx, ny, nz=1):
    return OracleMesh(*generate_box_mesh(etype, nx, ny, nz))


def mixed(nx, ny, nz, fraction=0.5):
    return OracleMesh(*generate_mixed_mesh(nx, ny, nz, fraction))


def element_blocks(mesh, kind, velocity=None, scalar=None, rho=1.0, mu=0.0, kappa=0.0):
    """Per-group element contributions, scalar (per-element) indexing."""
    out = []
    for etype, conn in mesh.groups:
        N, dN, w = reference_element(etype)
        detjw, gradn, bad = geometry(conn, mesh.coords, dN, w)
        if bad[0] >= 0:
            raise ArithmeticError(f"inverted element {bad}")
        if kind == "mass":
            blk = mass(detjw, N)
        elif kind == "laplacian":
            blk = laplacian(detjw, gradn)
        elif kind == "convection":
            blk = convection(detjw, gradn, N, conn, velocity)
        elif kind == "momentum_rhs":
            blk = momentum_rhs(detjw, gradn, N, conn, velocity, rho, mu)
        elif kind == "scalar_rhs":
            blk = scalar_rhs(detjw, gradn, N, conn, velocity, scalar, kappa)
        else:
            raise ValueError(kind)
        out.append((etype, conn, blk))
    return out


def assemble_matrix(mesh, kind, velocity=None, vs=8, pattern=None):
    """Global CSR values in the reference packed scatter order."""
    if pattern is None:
        pattern = build_node_pattern(mesh.nnode, [c for _, c in mesh.groups])
    rowptr, colind = pattern
    vals = np.zeros(colind.size)
    for _, conn, blk in element_blocks(mesh, kind, velocity):
        pos = matrix_positions(conn, rowptr, colind)
        lane_conn, eidx = build_packs(conn, vs)
        ne = conn.shape[0]
        # padded lanes contribute exact zeros (zero detJw), so they are skipped
        Ae = np.moveaxis(blk[eidx], 1, -1).copy()  # [p,i,j,v]
        pp = np.moveaxis(pos[eidx], 1, -1)
        act = (np.arange(eidx.size) < ne).reshape(eidx.shape)
        Ae[np.broadcast_to(~act[:, None, None, :], Ae.shape)] = 0.0
        np.add.at(vals, pp.ravel(), Ae.ravel())
    return rowptr, colind, vals


def assemble_rhs(mesh, kind, velocity, scalar=None, rho=1.0, mu=0.0, kappa=0.0, vs=8):
    n, dim = mesh.nnode, mesh.dim
    rhs = np.zeros((n, dim)) if kind == "momentum_rhs" else np.zeros(n)
    for _, conn, blk in element_blocks(mesh, kind, velocity, scalar, rho, mu, kappa):
        lane_conn, eidx = build_packs(conn, vs)
        ne = conn.shape[0]
        act = (np.arange(eidx.size) < ne).reshape(eidx.shape)
        if kind == "momentum_rhs":
            Re = np.moveaxis(blk[eidx], 1, -1).copy()  # [p, a, d, v]
            Re[np.broadcast_to(~act[:, None, None, :], Re.shape)] = 0.0
            # order p, i, v, d (_kernels.py:511-519)
            idx = np.moveaxis(lane_conn, 2, 2)[:, :, :, None] * dim + np.arange(dim)
            vals = np.moveaxis(Re, 3, 2)  # [p, a, v, d]
            np.add.at(rhs.reshape(-1), idx.ravel(), vals.ravel())
        else:
            Re = np.moveaxis(blk[eidx], 1, -1).copy()  # [p, a, v]
            Re[np.broadcast_to(~act[:, None, :], Re.shape)] = 0.0
            np.add.at(rhs, lane_conn.ravel(), Re.ravel())
    return rhs


# --------------------------------------------------------------------------
# CSR + vector kernels  (sparse.py:78-130) and PCG  (krylov.py:27-89)
# --------------------------------------------------------------------------

def spmv(rowptr, colind, vals, x):
    """y_i = sum_k vals[k] x[col[k]] in ascending k (sparse.py:78-84)."""
    prod = vals * x[colind]
    n = rowptr.size - 1
    # sequential per-row sum: cumulative sum restarted at each row start
    y = np.zeros(n)
    lens = np.diff(rowptr)
    maxlen = int(lens.max(initial=0))
    for t in range(maxlen):
        live = lens > t
        y[live] = y[live] + prod[rowptr[:-1][live] + t]
    return y


def axpy(alpha, x, y):  # sparse.py:96-99
    return alpha * x + y


def dot(x, y):
    """Left-to-right sequential sum (sparse.py:102-107)."""
    prod = x * y
    return float(np.cumsum(prod)[-1]) if prod.size else 0.0


def norm2(x):  # sparse.py:129-130
    return float(np.sqrt(dot(x, x)))


def diagonal(rowptr, colind, vals):  # sparse.py:48-56
    n = rowptr.size - 1
    out = np.zeros(n)
    for i in range(n):
        lo, hi = rowptr[i], rowptr[i + 1]
        k = lo + np.searchsorted(colind[lo:hi], i)
        if k < hi and colind[k] == i:
            out[i] = vals[k]
    return out


def apply_dirichlet_pin(rowptr, colind, vals, nodes):
    """Symmetric elimination without RHS (sparse.py:219-254)."""
    n = rowptr.size - 1
    flag = np.zeros(n, dtype=bool)
    flag[nodes] = True
    rows = np.repeat(np.arange(n), np.diff(rowptr))
    out = vals.copy()
    out[flag[rows] | flag[colind]] = 0.0
    for i in nodes:
        lo, hi = rowptr[i], rowptr[i + 1]
        out[lo + np.searchsorted(colind[lo:hi], i)] = 1.0
    return out


def pcg_solve(rowptr, colind, vals, b, x0=None, tol=1e-8, max_iter=None, jacobi=True):
    """Returns (x, iterations, converged, history, true_residual) — krylov.py:27-89."""
    n = rowptr.size - 1
    if max_iter is None:
        max_iter = 10 * n
    d = diagonal(rowptr, colind, vals) if jacobi else np.ones(n)
    if jacobi and (d <= 0.0).any():
        raise ArithmeticError("Jacobi preconditioner needs a positive diagonal")
    bnorm = norm2(b)
    if bnorm == 0.0:
        return np.zeros(n), 0, True, [0.0], 0.0
    if x0 is None:
        x = np.zeros(n)
        r = b.copy()
    else:
        x = x0.copy()
        r = axpy(-1.0, spmv(rowptr, colind, vals, x), b)
    relres = norm2(r) / bnorm
    hist = [relres]
    if relres <= tol:
        return x, 0, True, hist, relres
    z = r / d
    p = z.copy()
    rz = dot(r, z)
    it, conv = 0, False
    for _ in range(max_iter):
        q = spmv(rowptr, colind, vals, p)
        pq = dot(p, q)
        if pq <= 0.0:
            raise ArithmeticError(f"non-positive curvature p^T A p = {pq:.6e}")
        alpha = rz / pq
        x = axpy(alpha, p, x)
        r = axpy(-alpha, q, r)
        it += 1
        relres = norm2(r) / bnorm
        hist.append(relres)
        if relres <= tol:
            conv = True
            break
        z = r / d
        rz_new = dot(r, z)
        p = axpy(rz_new / rz, p, z)
        rz = rz_new
    tr = norm2(axpy(-1.0, spmv(rowptr, colind, vals, x), b)) / bnorm
    return x, it, conv, hist, tr


def bicgstab(rowptr, colind, vals, b, x0=None, tol=1e-8, max_iter=None, jacobi=True):
    """Jacobi-BiCGSTAB, restated operation for operation from
    scipy.sparse.linalg.bicgstab (scipy 1.18.1, _isolve/iterative.py; the
    reference has no BiCGSTAB — SURVEY.md 8(f) rank 1) with this module's
    sequential spmv / dot.  Returns (x, iterations, status, history) with
    status 0 converged, 2 rho breakdown, 3 (r~, v) = 0, 4 omega breakdown,
    -1 iteration cap; history[i] = ||r_i|| / ||b||.  Pinned against scipy in
    tests/test_bicgstab.py."""
    n = rowptr.size - 1
    if max_iter is None:
        max_iter = 10 * n
    d = diagonal(rowptr, colind, vals) if jacobi else None
    psolve = (lambda v: v / d) if jacobi else (lambda v: v.copy())
    eps2 = np.finfo(float).eps ** 2
    bnorm = norm2(b)
    if bnorm == 0.0:
        return np.zeros(n), 0, 0, [0.0]
    atol = tol * bnorm
    x = np.zeros(n) if x0 is None else x0.copy()
    r = b.copy() if x0 is None else b - spmv(rowptr, colind, vals, x)
    rt = r.copy()
    hist = [norm2(r) / bnorm]
    rho_prev = alpha = omega = 1.0
    p = v = None
    for it in range(max_iter):
        if norm2(r) < atol:
            return x, it, 0, hist
        rho = dot(rt, r)
        if abs(rho) < eps2:
            return x, it, 2, hist
        if it > 0:
            if abs(omega) < eps2:
                return x, it, 4, hist
            beta = (rho / rho_prev) * (alpha / omega)
            p = (p - omega * v) * beta + r
        else:
            p = r.copy()
        ph = psolve(p)
        v = spmv(rowptr, colind, vals, ph)
        rv = dot(rt, v)
        if rv == 0.0:
            return x, it, 3, hist
        alpha = rho / rv
        s = r - alpha * v
        if norm2(s) < atol:
            x = x + alpha * ph
            hist.append(norm2(s) / bnorm)
            return x, it + 1, 0, hist
        sh = psolve(s)
        t = spmv(rowptr, colind, vals, sh)
        omega = dot(t, s) / dot(t, t)
        x = x + alpha * ph
        x = x + omega * sh
        r = s - omega * t
        hist.append(norm2(r) / bnorm)
        rho_prev = rho
    if norm2(r) < atol:
        return x, max_iter, 0, hist
    return x, max_iter, -1, hist


# --------------------------------------------------------------------------
# bench fields  (bench.py:178-179, :196-197; test_assembly.py:199-213)
# --------------------------------------------------------------------------

def bench_fields(nnode, dim, seed=0):
    """velocity then three scalars from one default_rng(seed) stream."""
    rng = np.random.default_rng(seed)
    vel = rng.standard_normal((nnode, dim))
    scalars = [rng.standard_normal(nnode) for _ in range(3)]
    return vel, scalars


def smooth_fields(coords):
    x = coords
    if x.shape[1] == 2:
        vel = np.stack([np.sin(x[:, 0]) + 0.2 * x[:, 1], np.cos(x[:, 1])], axis=1)
    else:
        vel = np.stack([np.sin(x[:, 0]) + 0.2 * x[:, 1], np.cos(x[:, 1]) * x[:, 2],
                        x[:, 0] * x[:, 1] + 0.5], axis=1)
    phi = np.cos(x[:, 0]) * np.sin(x[:, 1]) + x[:, -1]
    return np.ascontiguousarray(vel), np.ascontiguousarray(phi)


def rel_diff(a, b):
    """Max-normalised difference (test_assembly.py:216-218)."""
    scale = max(np.abs(a).max(initial=0), np.abs(b).max(initial=0), 1e-30)
    return float(np.abs(a - b).max(initial=0) / scale)
