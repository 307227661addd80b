"""Assembly on distorted meshes.  The reference goldens are box meshes, whose
elements are all affine images of one cell — constant Jacobians hide bugs in
the per-Gauss-point geometry (e.g. the cross terms of the sum-factorised Q1
Jacobian) and in the closed forms' use of per-element geometry.  Here every
interior node is moved by up to 0.2 h (the SURVEY's "burner-like" jitter,
applied identically to both sides) and each kernel kind is checked against
the oracle, whose element loops follow the reference's Gauss-point
arithmetic for any coordinates (pinned bitwise on the goldens)."""

import numpy as np
import pytest
import torch

from oracle import fempack_np as O

pytestmark = pytest.mark.gpu

CASES = {
    "tet": ("TET04", (6, 5, 4)),
    "hex": ("HEX08", (5, 4, 4)),
    "quad": ("QUAD04", (7, 6)),
    "tri": ("TRI03", (7, 6)),
    "pyr": ("PYR05", (3, 3, 3)),
    "mixed": ("mixed", (4, 3, 3)),
}


def _jitter(coords, dims, seed=3):
    """Move interior nodes by up to 0.2 h per axis (boundary nodes stay)."""
    rng = np.random.default_rng(seed)
    x = coords.copy()
    h = np.array([1.0 / d for d in dims])
    lo, hi = x.min(axis=0), x.max(axis=0)
    interior = np.all((x > lo + 1e-12) & (x < hi - 1e-12), axis=1)
    x[interior] += 0.2 * h * rng.uniform(-1.0, 1.0, size=(int(interior.sum()), x.shape[1]))
    return x


@pytest.fixture(scope="module", params=sorted(CASES))
def case(request, cuda_ok):
    import paper_2107_11541_b200 as P

    et, dims = CASES[request.param]
    if et == "mixed":
        mesh = P.renumber_by_type(P.generate_mixed_mesh(*dims, fraction=0.5))[0]
        om = O.OracleMesh(3, mesh.coords.copy(), [(g.etype.value, g.conn) for g in mesh.groups])
    else:
        mesh = P.generate_box_mesh(P.ElementType[et], *dims)
        om = O.box(et, *dims)
    x = _jitter(om.coords, dims if et != "pyr" else dims)
    om = O.OracleMesh(om.dim, x, om.groups)
    mesh.coords_d.copy_(torch.as_tensor(x, device="cuda"))
    mesh._coords_h = None
    ctx = P.AssemblyContext.build(mesh, 8)
    return request.param, P, ctx, om


def _fields(om, seed=5):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((om.nnode, om.dim)), rng.standard_normal(om.nnode)


@pytest.mark.parametrize("kind", ["mass", "laplacian", "convection"])
def test_matrices_on_distorted_mesh(case, kind):
    name, P, ctx, om = case
    vel, _ = _fields(om)
    A = ctx.assemble_matrix(P.KernelKind[kind.upper()], "packed", velocity=vel if kind == "convection" else None)
    _, _, want = O.assemble_matrix(om, kind, vel if kind == "convection" else None)
    assert O.rel_diff(A.vals, want) < 1e-12, (name, kind)


def test_gradient_matrices_on_distorted_mesh(case):
    name, P, ctx, om = case
    grads = P.gradient_matrices(ctx)
    for k, B in enumerate(grads):
        unit = np.zeros((om.nnode, om.dim))
        unit[:, k] = 1.0
        _, _, want = O.assemble_matrix(om, "convection", unit)
        assert O.rel_diff(B.vals, want) < 1e-12, (name, k)


@pytest.mark.parametrize("kind", ["momentum_rhs", "scalar_rhs"])
def test_rhs_on_distorted_mesh(case, kind):
    name, P, ctx, om = case
    vel, phi = _fields(om)
    args = (vel, None, 1.3, 2e-2, 0.0) if kind == "momentum_rhs" else (vel, phi, 1.0, 0.0, 3e-2)
    got = ctx.assemble_rhs(P.KernelKind[kind.upper()], "packed", *args)
    want = O.assemble_rhs(om, kind, *args)
    assert O.rel_diff(got, want) < 1e-12, (name, kind)


@pytest.mark.parametrize("dims", [(20, 17, 13), (9, 33, 5)])
def test_hex_once_gradients_match_row_kernel(cuda_ok, dims):
    """hexblock.cu (element geometry once: element pass + canonical / generic
    row passes) against the per-row kernel (rowsq.cu) and the oracle on a
    jittered HEX08 box; bitwise run-to-run."""
    import paper_2107_11541_b200 as P
    from paper_2107_11541_b200 import assembly as A

    mesh = P.generate_box_mesh(P.ElementType.HEX08, *dims)
    om = O.box("HEX08", *dims)
    x = _jitter(om.coords, dims, seed=11)
    om = O.OracleMesh(3, x, om.groups)
    mesh.coords_d.copy_(torch.as_tensor(x, device="cuda"))
    ctx = P.AssemblyContext.build(mesh, 8)
    nnz = ctx.pattern.nnz
    brick = torch.empty(3 * nnz, dtype=torch.float64, device="cuda")
    ctx.assemble_gradients_d(brick)
    plan = ctx.groups[0].hexrows
    assert plan is not None and plan.ncanon > 0 and plan.ngblocks > 0, "both row kinds exercised"
    again = torch.empty_like(brick)
    ctx.assemble_gradients_d(again)
    assert torch.equal(brick, again)
    A.HEX_ONCE = False
    try:
        rows = torch.empty_like(brick)
        ctx.assemble_gradients_d(rows)
    finally:
        A.HEX_ONCE = True
    b, r = brick.cpu().numpy(), rows.cpu().numpy()
    assert O.rel_diff(b, r) < 1e-13
    for k in range(3):
        unit = np.zeros((om.nnode, 3))
        unit[:, k] = 1.0
        _, _, want = O.assemble_matrix(om, "convection", unit)
        assert O.rel_diff(b[k * nnz:(k + 1) * nnz], want) < 1e-12, k
