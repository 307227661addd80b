"""Assembly kernels on the B200 vs the reference (goldens) and the oracle.

Bar (north star): matrices and RHS within 1e-12 max-normalised relative
difference (rel_diff, test_assembly.py:216-218) of the reference's packed
path.  The device sums contributions in a different order (FP64 reductions
at L2, DFMA contraction), so agreement is to rounding, not bitwise."""

import numpy as np
import pytest

from conftest import load_golden
from oracle import fempack_np as O

pytestmark = pytest.mark.gpu
TOL = 1e-12

NAMES = ["tri_4x3", "quad_4x3", "tet_6", "pyr_6", "hex_8", "mixed_8", "mixed_3x2x2", "tet_c1"]


@pytest.fixture(scope="module", params=[(n, s) for n in NAMES for s in ("auto", "rows", "atomic")
                                        if s == "auto" or n in ("tri_4x3", "tet_6", "tet_c1", "mixed_8")],
                ids=lambda p: f"{p[0]}-{p[1]}")
def case(request, cuda_ok):
    """Every golden mesh through the default dispatch (row-owned kernels for
    TRI03/TET04, element kernels + FP64 reductions otherwise), and the
    simplex meshes once more through the element/atomic kernels."""
    import paper_2107_11541_b200 as P
    from gpu_cases import CASES

    name, scatter = request.param
    mesh = CASES[name]()
    return name, P.AssemblyContext.build(mesh, vector_size=8, scatter=scatter), load_golden(name)


def test_matrices_match_reference(case):
    import paper_2107_11541_b200 as P

    name, ctx, g = case
    vel = g["bench_vel"]
    for key, kind, v in (("mass", P.KernelKind.MASS, None),
                         ("laplacian", P.KernelKind.LAPLACIAN, None),
                         ("convection", P.KernelKind.CONVECTION, vel)):
        if f"mat_{key}" not in g:
            continue
        for layout in ("packed", "scalar"):
            A = ctx.assemble_matrix(kind, layout, velocity=v)
            assert O.rel_diff(A.vals, g[f"mat_{key}"]) < TOL, (name, key, layout)
    A = ctx.assemble_matrix(P.KernelKind.CONVECTION, "packed", velocity=g["smooth_vel"])
    assert O.rel_diff(A.vals, g["mat_convection_smooth"]) < TOL


def test_rhs_match_reference(case):
    import paper_2107_11541_b200 as P

    name, ctx, g = case
    vel = g["bench_vel"]
    r = ctx.assemble_rhs(P.KernelKind.MOMENTUM_RHS, "packed", vel, None, 1.0, 1e-2, 0.0)
    assert r.shape == g["rhs_momentum"].shape
    assert O.rel_diff(r, g["rhs_momentum"]) < TOL, name
    assert O.rel_diff(r, g["rhs_momentum_scalar_layout"]) < TOL
    r = ctx.assemble_rhs(P.KernelKind.MOMENTUM_RHS, "packed", g["smooth_vel"], None, 1.2, 1e-2, 0.0)
    assert O.rel_diff(r, g["rhs_momentum_smooth"]) < TOL
    for s in range(3):
        r = ctx.assemble_rhs(P.KernelKind.SCALAR_RHS, "packed", vel, g[f"bench_scalar{s}"], 1.0, 0.0, 1e-2)
        assert O.rel_diff(r, g[f"rhs_scalar{s}"]) < TOL, (name, s)
    r = ctx.assemble_rhs(P.KernelKind.SCALAR_RHS, "scalar", g["smooth_vel"], g["smooth_phi"], 1.0, 0.0, 0.3)
    assert O.rel_diff(r, g["rhs_scalar_smooth"]) < TOL


def test_continuity_and_lumped_mass(case):
    import paper_2107_11541_b200 as P

    name, ctx, g = case
    grads = P.gradient_matrices(ctx)
    for k, B in enumerate(grads):
        if f"mat_grad{k}" in g:
            assert O.rel_diff(B.vals, g[f"mat_grad{k}"]) < TOL, (name, k)
    ml = P.lumped_mass(ctx)
    assert O.rel_diff(ml, g["lumped_mass"]) < TOL


def test_torch_inputs_stay_on_device(case):
    import torch

    import paper_2107_11541_b200 as P

    name, ctx, g = case
    vel = torch.as_tensor(g["bench_vel"], device="cuda")
    r = ctx.assemble_rhs(P.KernelKind.MOMENTUM_RHS, "packed", vel, None, 1.0, 1e-2, 0.0)
    assert isinstance(r, torch.Tensor) and r.is_cuda
    assert O.rel_diff(r.cpu().numpy(), g["rhs_momentum"]) < TOL


def test_vector_size_does_not_change_results(cuda_ok):
    import paper_2107_11541_b200 as P
    from gpu_cases import CASES

    g = load_golden("mixed_8")
    mesh = CASES["mixed_8"]()
    outs = [P.AssemblyContext.build(mesh, vs).assemble_matrix(P.KernelKind.LAPLACIAN).vals
            for vs in (1, 2, 4, 8, 16, 32)]
    for o in outs:
        assert O.rel_diff(o, g["mat_laplacian"]) < TOL


def test_physics_identities(cuda_ok):
    """MASS sums to the volume; LAPLACIAN rows sum to zero
    (test_assembly.py:172-196); momentum is linear in (rho, mu)
    (test_assembly.py:279-286)."""
    import paper_2107_11541_b200 as P

    for et, dims in ((P.ElementType.TET04, (5, 4, 3)), (P.ElementType.HEX08, (4, 4, 4)),
                     (P.ElementType.PYR05, (3, 3, 3))):
        mesh = P.generate_box_mesh(et, *dims)
        ctx = P.AssemblyContext.build(mesh, 8)
        M = ctx.assemble_matrix(P.KernelKind.MASS)
        assert M.vals.sum() == pytest.approx(1.0, rel=1e-12)
        L = ctx.assemble_matrix(P.KernelKind.LAPLACIAN)
        rs = np.add.reduceat(L.vals, L.rowptr[:-1])
        assert np.abs(rs).max() < 1e-12
        vel, _ = O.smooth_fields(mesh.coords)
        base = ctx.assemble_rhs(P.KernelKind.MOMENTUM_RHS, "packed", vel, rho=1.0, mu=0.0)
        visc = ctx.assemble_rhs(P.KernelKind.MOMENTUM_RHS, "packed", vel, rho=0.0, mu=1.0)
        both = ctx.assemble_rhs(P.KernelKind.MOMENTUM_RHS, "packed", vel, rho=2.0, mu=3.0)
        np.testing.assert_allclose(both, 2.0 * base + 3.0 * visc, atol=1e-12)


def test_missing_fields_raise(cuda_ok):
    import paper_2107_11541_b200 as P

    ctx = P.AssemblyContext.build(P.generate_box_mesh(P.ElementType.QUAD04, 2, 2), 4)
    with pytest.raises(P.ConfigurationError):
        ctx.assemble_matrix(P.KernelKind.CONVECTION)
    with pytest.raises(P.ConfigurationError):
        ctx.assemble_rhs(P.KernelKind.SCALAR_RHS, velocity=np.zeros((9, 2)))
    with pytest.raises(P.ConfigurationError):
        ctx.assemble_matrix(P.KernelKind.MOMENTUM_RHS)
    with pytest.raises(P.ConfigurationError):
        ctx.assemble_rhs(P.KernelKind.MASS)
    with pytest.raises(P.ConfigurationError):
        ctx.assemble_matrix(P.KernelKind.MASS, "simd")


def test_repeat_assembly_reproducible_to_rounding(cuda_ok):
    """The reference packed path is bitwise repeatable (test_assembly.py:270-276).
    Element kernels with FP64 reductions at L2 (PYR05/HEX08) reorder
    additions, so their repeats agree to rounding."""
    import paper_2107_11541_b200 as P

    mesh = P.generate_mixed_mesh(2, 2, 2, fraction=0.5)
    ctx = P.AssemblyContext.build(mesh, 8)
    vel, _ = O.smooth_fields(mesh.coords)
    a = ctx.assemble_matrix(P.KernelKind.CONVECTION, "packed", velocity=vel).vals
    b = ctx.assemble_matrix(P.KernelKind.CONVECTION, "packed", velocity=vel).vals
    # every matrix kind is row-owned (rows.cu, rowsq.cu): byte-identical,
    # as the reference asserts (test_assembly.py:270-276)
    assert a.tobytes() == b.tobytes()


@pytest.mark.parametrize("et", ["TET04", "TRI03", "HEX08", "QUAD04"])
def test_row_owned_assembly_is_bitwise_deterministic(cuda_ok, et):
    """Row-owned kernels (simplices: rows.cu; Gauss-loop elements: rowsq.cu)
    sum each row in a fixed element order: repeated assemblies are
    byte-identical, as in the reference (test_assembly.py:270-276,
    test_sparse.py:93-97)."""
    import paper_2107_11541_b200 as P

    dims = (9, 7, 5) if P.ElementType[et].value in ("TET04", "HEX08") else (9, 7)
    mesh = P.generate_box_mesh(P.ElementType[et], *dims)
    ctx = P.AssemblyContext.build(mesh, 8)
    assert ctx.groups[0].rows is not None
    vel, phi = O.smooth_fields(mesh.coords)
    for kind, kw in ((P.KernelKind.CONVECTION, dict(velocity=vel)), (P.KernelKind.LAPLACIAN, {})):
        a = ctx.assemble_matrix(kind, "packed", **kw).vals
        b = ctx.assemble_matrix(kind, "packed", **kw).vals
        assert a.tobytes() == b.tobytes()
    r1 = ctx.assemble_rhs(P.KernelKind.MOMENTUM_RHS, "packed", vel, None, 1.2, 1e-2)
    r2 = ctx.assemble_rhs(P.KernelKind.MOMENTUM_RHS, "packed", vel, None, 1.2, 1e-2)
    assert r1.tobytes() == r2.tobytes()
    g1 = [B.vals for B in P.gradient_matrices(ctx)]
    g2 = [B.vals for B in P.gradient_matrices(ctx)]
    assert all(x.tobytes() == y.tobytes() for x, y in zip(g1, g2))


@pytest.mark.parametrize("strategy", ["auto", "rows"])
def test_owner_kernels_match_atomic_kernels(cuda_ok, strategy):
    """Independent device formulations agree to rounding on a 90k-tet mesh."""
    import paper_2107_11541_b200 as P

    mesh = P.generate_box_mesh(P.ElementType.TET04, 25, 24, 25)
    rows = P.AssemblyContext.build(mesh, 8, scatter=strategy)
    atom = P.AssemblyContext.build(mesh, 8, scatter="atomic")
    vel, phi = O.smooth_fields(mesh.coords)
    for kind in (P.KernelKind.MASS, P.KernelKind.LAPLACIAN, P.KernelKind.CONVECTION):
        a = rows.assemble_matrix(kind, velocity=vel).vals
        b = atom.assemble_matrix(kind, velocity=vel).vals
        assert O.rel_diff(a, b) < 1e-13, kind
    for kind, kw in ((P.KernelKind.MOMENTUM_RHS, dict(rho=1.1, mu=0.02)),
                     (P.KernelKind.SCALAR_RHS, dict(scalar=phi, kappa=0.03))):
        a = rows.assemble_rhs(kind, "packed", vel, **kw)
        b = atom.assemble_rhs(kind, "packed", vel, **kw)
        assert O.rel_diff(a, b) < 1e-13, kind


def test_c2_momentum_and_continuity_vs_oracle(cuda_ok):
    """Config 2 at full size (5,036,520 tets): momentum RHS against the
    oracle (bitwise-pinned restatement of the reference packed path); the
    continuity matrices' row sums vanish."""
    import torch

    import paper_2107_11541_b200 as P

    mesh = P.generate_box_mesh(P.ElementType.TET04, 94, 94, 95)
    ctx = P.AssemblyContext.build(mesh, 8)
    om = O.box(O.TET04, 94, 94, 95)
    vel, _ = O.bench_fields(om.nnode, 3)
    r = ctx.assemble_rhs(P.KernelKind.MOMENTUM_RHS, "packed", vel, None, 1.0, 1e-2, 0.0)
    ro = O.assemble_rhs(om, "momentum_rhs", vel, None, 1.0, 1e-2, 0.0)
    assert O.rel_diff(r, ro) < TOL
    del ro
    grads = P.gradient_matrices(ctx)  # values vs the C port: tests/test_gpu_scale.py
    # B_k annihilates constants: row sums vanish (timeloop.py:191)
    for B in grads:
        assert float(B.row_sums_d().abs().max()) < 1e-12 * float(B.vals_d.abs().max())
    torch.cuda.synchronize()


@pytest.mark.parametrize("name", ["mixed_8", "hex_8", "pyr_6"])
def test_block_rhs_is_bitwise_deterministic(cuda_ok, name):
    """Element-block RHS (every element type) reduces in a fixed order:
    repeated assemblies are byte-identical."""
    import paper_2107_11541_b200 as P
    from gpu_cases import CASES

    mesh = CASES[name]()
    ctx = P.AssemblyContext.build(mesh, 8)
    vel, phi = O.smooth_fields(mesh.coords)
    r1 = ctx.assemble_rhs(P.KernelKind.MOMENTUM_RHS, "packed", vel, None, 1.2, 1e-2)
    r2 = ctx.assemble_rhs(P.KernelKind.MOMENTUM_RHS, "packed", vel, None, 1.2, 1e-2)
    assert r1.tobytes() == r2.tobytes()
    s1 = ctx.assemble_rhs(P.KernelKind.SCALAR_RHS, "packed", vel, phi, kappa=0.3)
    s2 = ctx.assemble_rhs(P.KernelKind.SCALAR_RHS, "packed", vel, phi, kappa=0.3)
    assert s1.tobytes() == s2.tobytes()


@pytest.mark.parametrize("name", NAMES)
def test_scalar_rhs3_fused_matches_reference(cuda_ok, name):
    """The fused three-scalar pass (config 3: enthalpy + 2 species) equals
    three SCALAR_RHS passes to rounding and the reference's goldens within
    1e-12, with a different diffusivity per field; bitwise run-to-run."""
    import torch

    import paper_2107_11541_b200 as P
    from gpu_cases import CASES

    g = load_golden(name)
    ctx = P.AssemblyContext.build(CASES[name](), vector_size=8)
    n = ctx.mesh.nnode
    vel = torch.as_tensor(g["bench_vel"], device="cuda")
    phi3 = torch.as_tensor(np.stack([g[f"bench_scalar{s}"] for s in range(3)]), device="cuda")
    out = torch.empty((3, n), dtype=torch.float64, device="cuda")
    ctx.assemble_scalar_rhs3_d(vel, phi3, (1e-2, 1e-2, 1e-2), out)
    for s in range(3):
        assert O.rel_diff(out[s].cpu().numpy(), g[f"rhs_scalar{s}"]) < TOL, (name, s)
    kap = (1e-2, 3e-3, 0.2)
    ctx.assemble_scalar_rhs3_d(vel, phi3, kap, out)
    first = out.cpu().numpy().copy()
    ctx.assemble_scalar_rhs3_d(vel, phi3, kap, out)
    assert out.cpu().numpy().tobytes() == first.tobytes()
    one = torch.empty(n, dtype=torch.float64, device="cuda")
    for s in range(3):
        ctx.assemble_rhs_d(P.KernelKind.SCALAR_RHS, vel, phi3[s], 1.0, 0.0, kap[s], one)
        assert O.rel_diff(first[s], one.cpu().numpy()) < 1e-14, (name, s)
