"""Momentum RHS on Kuhn box meshes by z-marching cell lines (kmom.cu).

The default dispatch sends MOMENTUM_RHS of a TET04 mesh whose connectivity
is exactly generate_box_mesh's (assembly.py KuhnBox.detect) to
fpb_assemble_momentum_kuhn.  Checked here against the oracle (pinned to the
reference, tests/test_oracle_golden.py) on unjittered and jittered
coordinates, over z-chunk sizes that exercise the halo layer, the row
chain and the top face, against the element-block path at a larger size,
and for bitwise run-to-run determinism.  Bar: 1e-12 max-normalised."""

import numpy as np
import pytest
import torch

from oracle import fempack_np as O

pytestmark = pytest.mark.gpu
TOL = 1e-12


def _ctx(P, nx, ny, nz, kchunk=0, coords=None):
    import paper_2107_11541_b200.assembly as A

    old = A.KUHN_KCHUNK
    A.KUHN_KCHUNK = kchunk
    try:
        mesh = P.generate_box_mesh(P.ElementType.TET04, nx, ny, nz)
        if coords is not None:
            mesh.coords = coords
        ctx = P.AssemblyContext.build(mesh, vector_size=8)
    finally:
        A.KUHN_KCHUNK = old
    return mesh, ctx


def _jitter(coords, nx, ny, nz, seed=3):
    rng = np.random.default_rng(seed)
    h = np.array([1.0 / nx, 1.0 / ny, 1.0 / nz])
    return coords + rng.uniform(-0.15, 0.15, coords.shape) * h


@pytest.mark.parametrize("dims,kchunk", [((5, 4, 7), 0), ((5, 4, 7), 1), ((5, 4, 7), 2), ((5, 4, 7), 3),
                                         ((1, 1, 1), 0), ((1, 3, 2), 1), ((33, 3, 5), 2), ((64, 2, 3), 0),
                                         ((7, 1, 9), 4), ((65, 17, 4), 3), ((32, 8, 2), 0), ((70, 16, 5), 2),
                                         ((31, 9, 3), 1), ((96, 24, 3), 0)])
@pytest.mark.parametrize("jitter", [False, True])
def test_kuhn_momentum_matches_oracle(cuda_ok, dims, kchunk, jitter):
    import paper_2107_11541_b200 as P

    nx, ny, nz = dims
    om = O.box(O.TET04, nx, ny, nz)
    if jitter:
        om.coords = _jitter(om.coords, nx, ny, nz)
    mesh, ctx = _ctx(P, nx, ny, nz, kchunk, om.coords if jitter else None)
    assert ctx.groups[0].kuhn is not None
    if kchunk:
        assert ctx.groups[0].kuhn.kchunk == min(kchunk, nz)
    vel, _ = O.bench_fields(om.nnode, 3)
    for rho, mu in ((1.0, 1e-2), (0.7, 0.0), (0.0, 0.3)):
        r = ctx.assemble_rhs(P.KernelKind.MOMENTUM_RHS, "packed", vel, None, rho, mu, 0.0)
        ro = O.assemble_rhs(om, "momentum_rhs", vel, None, rho, mu, 0.0)
        assert O.rel_diff(r, ro) < TOL, (dims, kchunk, rho, mu, O.rel_diff(r, ro))


def test_kuhn_wide_and_detection(cuda_ok):
    import paper_2107_11541_b200 as P

    for dims in ((300, 1, 2), (257, 9, 1)):
        _, ctx = _ctx(P, *dims)
        assert ctx.groups[0].kuhn is not None
        om = O.box(O.TET04, *dims)
        vel, _ = O.bench_fields(om.nnode, 3)
        r = ctx.assemble_rhs(P.KernelKind.MOMENTUM_RHS, "packed", vel, None, 1.0, 1e-2, 0.0)
        assert O.rel_diff(r, O.assemble_rhs(om, "momentum_rhs", vel, None, 1.0, 1e-2, 0.0)) < TOL, dims
    # a permuted element order is not the generator's: element blocks
    mesh = P.generate_box_mesh(P.ElementType.TET04, 4, 3, 2)
    conn = mesh.groups[0].conn.copy()
    conn[[5, 6]] = conn[[6, 5]]
    m2 = P.Mesh(3, mesh.coords, [P.ElementGroup(P.ElementType.TET04, conn)])
    ctx2 = P.AssemblyContext.build(m2, vector_size=8)
    assert ctx2.groups[0].kuhn is None
    om = O.box(O.TET04, 4, 3, 2)
    vel, _ = O.bench_fields(om.nnode, 3)
    r = ctx2.assemble_rhs(P.KernelKind.MOMENTUM_RHS, "packed", vel, None, 1.0, 1e-2, 0.0)
    assert O.rel_diff(r, O.assemble_rhs(om, "momentum_rhs", vel, None, 1.0, 1e-2, 0.0)) < TOL


def test_kuhn_matches_block_path_and_is_deterministic(cuda_ok):
    import paper_2107_11541_b200 as P
    import paper_2107_11541_b200.assembly as A

    nx, ny, nz = 94, 40, 37
    mesh, ctx = _ctx(P, nx, ny, nz)
    kb = ctx.groups[0].kuhn
    assert kb is not None and -(-nz // kb.kchunk) > 1
    n = mesh.nnode
    g = torch.Generator(device="cuda").manual_seed(5)
    vel = torch.randn((n, 3), dtype=torch.float64, device="cuda", generator=g)
    out1 = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    out2 = torch.empty_like(out1)
    ref = torch.empty_like(out1)
    ctx.assemble_rhs_d(P.KernelKind.MOMENTUM_RHS, vel, None, 1.0, 1e-2, 0.0, out1)
    ctx.assemble_rhs_d(P.KernelKind.MOMENTUM_RHS, vel, None, 1.0, 1e-2, 0.0, out2)
    assert torch.equal(out1, out2)
    A.KUHN_MOMENTUM = False
    try:
        ctx.assemble_rhs_d(P.KernelKind.MOMENTUM_RHS, vel, None, 1.0, 1e-2, 0.0, ref)
    finally:
        A.KUHN_MOMENTUM = True
    a, b = out1.cpu().numpy(), ref.cpu().numpy()
    assert O.rel_diff(a, b) < TOL


def test_kuhn_box_gradients_match_colind_path(cuda_ok):
    """Continuity B_x, B_y, B_z on a Kuhn box: the interior rows by z-marching
    lines (fpb_assemble_gradient_kuhn_lines) give bitwise the colind path's
    values (same arithmetic, same order); the boundary rows by the
    box-masked interior stream (fpb_assemble_gradient_kuhn_boundary) agree
    with the generic row-list kernel to rounding; all match the oracle."""
    import paper_2107_11541_b200 as P
    import paper_2107_11541_b200.assembly as A

    for dims in ((37, 21, 9), (6, 5, 4), (2, 2, 2), (33, 2, 3), (1, 1, 1), (1, 4, 3), (40, 1, 2), (3, 3, 1)):
        om = O.box(O.TET04, *dims)
        om.coords = _jitter(om.coords, *dims, seed=11)
        mesh, ctx = _ctx(P, *dims, coords=om.coords)
        kb = ctx.groups[0].kuhn
        assert kb is not None and kb.pattern_ok
        nnz = ctx.pattern.nnz
        a = torch.empty(3 * nnz, dtype=torch.float64, device="cuda")
        b = torch.empty_like(a)
        ctx.assemble_gradients_d(a)
        A.KUHN_BOX_GRADIENT = False
        try:
            ctx.assemble_gradients_d(b)
        finally:
            A.KUHN_BOX_GRADIENT = True
        assert O.rel_diff(a.cpu().numpy(), b.cpu().numpy()) < 1e-14, dims
        # interior rows: bitwise
        nx, ny, nz = dims
        rp = ctx.pattern.rowptr_d.cpu().numpy()
        idx = np.arange(mesh.nnode)
        i, j, k = idx % (nx + 1), (idx // (nx + 1)) % (ny + 1), idx // ((nx + 1) * (ny + 1))
        inner = idx[(i > 0) & (i < nx) & (j > 0) & (j < ny) & (k > 0) & (k < nz)]
        sel = np.concatenate([np.arange(rp[r], rp[r + 1]) for r in inner]) if inner.size else np.zeros(0, int)
        pc = ctx.groups[0].rows.pair_canon
        for m in range(3 if (pc is not None and pc.get("kuhn")) else 0):  # colind path on the Kuhn stream
            assert torch.equal(a[m * nnz:(m + 1) * nnz][torch.as_tensor(sel, device="cuda")],
                               b[m * nnz:(m + 1) * nnz][torch.as_tensor(sel, device="cuda")]), dims
        for k3 in range(3):
            e = np.zeros((om.nnode, 3))
            e[:, k3] = 1.0
            _, _, vo = O.assemble_matrix(om, "convection", e)
            assert O.rel_diff(a[k3 * nnz:(k3 + 1) * nnz].cpu().numpy(), vo) < TOL, (dims, k3)


@pytest.mark.parametrize("dims,kchunk", [((5, 4, 7), 0), ((5, 4, 7), 2), ((33, 9, 5), 3), ((64, 2, 3), 0),
                                         ((1, 1, 1), 0)])
@pytest.mark.parametrize("jitter", [False, True])
def test_kuhn_scalar3_matches_oracle(cuda_ok, dims, kchunk, jitter):
    """Three scalar RHS (enthalpy + 2 species, one velocity) on the Kuhn box
    (fpb_assemble_scalar3_kuhn): each field equals the oracle's SCALAR_RHS
    with its own diffusivity."""
    import paper_2107_11541_b200 as P

    nx, ny, nz = dims
    om = O.box(O.TET04, nx, ny, nz)
    if jitter:
        om.coords = _jitter(om.coords, nx, ny, nz, seed=7)
    mesh, ctx = _ctx(P, nx, ny, nz, kchunk, om.coords if jitter else None)
    assert ctx.groups[0].kuhn is not None
    vel, sc = O.bench_fields(om.nnode, 3)
    kap = (1e-2, 3e-2, 0.0)
    phi3 = torch.as_tensor(np.stack(sc[:3]), device="cuda").contiguous()
    out3 = torch.full((3, om.nnode), float("nan"), dtype=torch.float64, device="cuda")
    ctx.assemble_scalar_rhs3_d(torch.as_tensor(vel, device="cuda"), phi3, kap, out3)
    got = out3.cpu().numpy()
    for f in range(3):
        want = O.assemble_rhs(om, "scalar_rhs", vel, sc[f], 1.0, 0.0, kap[f])
        assert O.rel_diff(got[f], want) < TOL, (dims, kchunk, f)


def test_kuhn_scalar3_matches_block_path(cuda_ok):
    import paper_2107_11541_b200 as P
    import paper_2107_11541_b200.assembly as A

    mesh, ctx = _ctx(P, 94, 40, 37)
    n = mesh.nnode
    g = torch.Generator(device="cuda").manual_seed(9)
    vel = torch.randn((n, 3), dtype=torch.float64, device="cuda", generator=g)
    phi3 = torch.randn((3, n), dtype=torch.float64, device="cuda", generator=g)
    a = torch.empty((3, n), dtype=torch.float64, device="cuda")
    b = torch.empty_like(a)
    ctx.assemble_scalar_rhs3_d(vel, phi3, (1e-2, 2e-2, 3e-2), a)
    c = torch.empty_like(a)
    ctx.assemble_scalar_rhs3_d(vel, phi3, (1e-2, 2e-2, 3e-2), c)
    assert torch.equal(a, c)
    A.KUHN_MOMENTUM = False
    try:
        ctx.assemble_scalar_rhs3_d(vel, phi3, (1e-2, 2e-2, 3e-2), b)
    finally:
        A.KUHN_MOMENTUM = True
    assert O.rel_diff(a.cpu().numpy(), b.cpu().numpy()) < TOL


def test_hex_box_element_ids_bitwise_equal_listed_ids(cuda_ok):
    """HEX08 continuity on the generator's hex box: the canonical-row kernel
    with element ids computed from the node (HexRowPlan.box) gives bitwise
    the values of the kernel reading them from canon_inc8, and the oracle's
    (jittered coordinates)."""
    import paper_2107_11541_b200 as P
    import paper_2107_11541_b200.assembly as A

    dims = (12, 9, 7)
    om = O.box(O.HEX08, *dims)
    om.coords = _jitter(om.coords, *dims, seed=5)
    mesh = P.generate_box_mesh(P.ElementType.HEX08, *dims)
    mesh.coords = om.coords
    res = {}
    for flag in (True, False):
        A.HEX_BOX_IDS = flag
        try:
            ctx = P.AssemblyContext.build(mesh, vector_size=8)
            out = torch.empty(3 * ctx.pattern.nnz, dtype=torch.float64, device="cuda")
            ctx.assemble_gradients_d(out)
            res[flag] = (out.cpu().numpy(), ctx.groups[0].hexrows.box)
        finally:
            A.HEX_BOX_IDS = True
    assert res[True][1] == (12, 9) and res[False][1] == (0, 0)
    assert np.array_equal(res[True][0], res[False][0])
    nnz = res[True][0].size // 3
    for k in range(3):
        e = np.zeros((om.nnode, 3))
        e[:, k] = 1.0
        _, _, vo = O.assemble_matrix(om, "convection", e)
        assert O.rel_diff(res[True][0][k * nnz:(k + 1) * nnz], vo) < TOL


def _hex_ctx(P, dims, kchunk=0, coords=None):
    import paper_2107_11541_b200.assembly as A

    old = A.KUHN_KCHUNK
    A.KUHN_KCHUNK = kchunk
    try:
        mesh = P.generate_box_mesh(P.ElementType.HEX08, *dims)
        if coords is not None:
            mesh.coords = coords
        ctx = P.AssemblyContext.build(mesh, vector_size=8)
    finally:
        A.KUHN_KCHUNK = old
    return mesh, ctx


@pytest.mark.parametrize("dims,kchunk", [((5, 4, 7), 0), ((5, 4, 7), 2), ((33, 9, 4), 3), ((32, 8, 2), 0),
                                         ((1, 1, 1), 0)])
def test_hex_box_rhs_matches_oracle(cuda_ok, dims, kchunk):
    """HEX08 box: momentum RHS and the three scalar RHS by the cell pencils
    (fpb_assemble_rhs_hexbox) against the oracle, jittered coordinates."""
    import paper_2107_11541_b200 as P

    om = O.box(O.HEX08, *dims)
    om.coords = _jitter(om.coords, *dims, seed=13)
    mesh, ctx = _hex_ctx(P, dims, kchunk, om.coords)
    kb = ctx.groups[0].kuhn
    assert kb is not None and kb.etype is P.ElementType.HEX08
    vel, sc = O.bench_fields(om.nnode, 3)
    r = ctx.assemble_rhs(P.KernelKind.MOMENTUM_RHS, "packed", vel, None, 1.0, 1e-2, 0.0)
    assert O.rel_diff(r, O.assemble_rhs(om, "momentum_rhs", vel, None, 1.0, 1e-2, 0.0)) < TOL, dims
    kap = (1e-2, 3e-2, 0.0)
    phi3 = torch.as_tensor(np.stack(sc[:3]), device="cuda").contiguous()
    out3 = torch.full((3, om.nnode), float("nan"), dtype=torch.float64, device="cuda")
    ctx.assemble_scalar_rhs3_d(torch.as_tensor(vel, device="cuda"), phi3, kap, out3)
    got = out3.cpu().numpy()
    for f in range(3):
        want = O.assemble_rhs(om, "scalar_rhs", vel, sc[f], 1.0, 0.0, kap[f])
        assert O.rel_diff(got[f], want) < TOL, (dims, f)


def test_hex_box_rhs_matches_block_path(cuda_ok):
    import paper_2107_11541_b200 as P
    import paper_2107_11541_b200.assembly as A

    mesh, ctx = _hex_ctx(P, (40, 24, 19))
    n = mesh.nnode
    g = torch.Generator(device="cuda").manual_seed(3)
    vel = torch.randn((n, 3), dtype=torch.float64, device="cuda", generator=g)
    phi3 = torch.randn((3, n), dtype=torch.float64, device="cuda", generator=g)
    a, b = torch.empty((n, 3), dtype=torch.float64, device="cuda"), torch.empty((n, 3), dtype=torch.float64,
                                                                                 device="cuda")
    a3, b3 = torch.empty((3, n), dtype=torch.float64, device="cuda"), torch.empty((3, n), dtype=torch.float64,
                                                                                  device="cuda")
    ctx.assemble_rhs_d(P.KernelKind.MOMENTUM_RHS, vel, None, 1.0, 1e-2, 0.0, a)
    ctx.assemble_scalar_rhs3_d(vel, phi3, (1e-2, 2e-2, 3e-2), a3)
    A.KUHN_MOMENTUM = False
    try:
        ctx.assemble_rhs_d(P.KernelKind.MOMENTUM_RHS, vel, None, 1.0, 1e-2, 0.0, b)
        ctx.assemble_scalar_rhs3_d(vel, phi3, (1e-2, 2e-2, 3e-2), b3)
    finally:
        A.KUHN_MOMENTUM = True
    assert O.rel_diff(a.cpu().numpy(), b.cpu().numpy()) < TOL
    assert O.rel_diff(a3.cpu().numpy(), b3.cpu().numpy()) < TOL


def test_assemble_ns_d_equals_sequence(cuda_ok):
    """assemble_ns_d (momentum and B_xyz on two streams) equals the two calls
    in sequence bitwise."""
    import paper_2107_11541_b200 as P

    mesh, ctx = _ctx(P, 40, 21, 13)
    n, nnz = mesh.nnode, ctx.pattern.nnz
    g = torch.Generator(device="cuda").manual_seed(11)
    vel = torch.randn((n, 3), dtype=torch.float64, device="cuda", generator=g)
    r1, r2 = (torch.empty((n, 3), dtype=torch.float64, device="cuda") for _ in range(2))
    m1, m2 = (torch.empty(3 * nnz, dtype=torch.float64, device="cuda") for _ in range(2))
    ctx.assemble_ns_d(vel, 1.0, 1e-2, r1, m1)
    ctx.assemble_rhs_d(P.KernelKind.MOMENTUM_RHS, vel, None, 1.0, 1e-2, 0.0, r2)
    ctx.assemble_gradients_d(m2)
    torch.cuda.synchronize()
    assert torch.equal(r1, r2) and torch.equal(m1, m2)


def test_kuhn_anisotropic_offset_box(cuda_ok):
    """Kuhn-box kernels on a stretched, shifted box (lengths 2 x 0.5 x 3,
    coordinates + 10): momentum, three scalars and B_xyz against the oracle."""
    import paper_2107_11541_b200 as P

    dims = (9, 7, 6)
    om = O.box(O.TET04, *dims)
    om.coords = om.coords * np.array([2.0, 0.5, 3.0]) + 10.0
    om.coords = _jitter(om.coords, *dims, seed=23)
    mesh, ctx = _ctx(P, *dims, coords=om.coords)
    assert ctx.groups[0].kuhn is not None
    vel, sc = O.bench_fields(om.nnode, 3)
    r = ctx.assemble_rhs(P.KernelKind.MOMENTUM_RHS, "packed", vel, None, 1.0, 1e-2, 0.0)
    assert O.rel_diff(r, O.assemble_rhs(om, "momentum_rhs", vel, None, 1.0, 1e-2, 0.0)) < TOL
    phi3 = torch.as_tensor(np.stack(sc[:3]), device="cuda").contiguous()
    out3 = torch.empty((3, om.nnode), dtype=torch.float64, device="cuda")
    ctx.assemble_scalar_rhs3_d(torch.as_tensor(vel, device="cuda"), phi3, (1e-2, 1e-2, 1e-2), out3)
    for f in range(3):
        want = O.assemble_rhs(om, "scalar_rhs", vel, sc[f], 1.0, 0.0, 1e-2)
        assert O.rel_diff(out3[f].cpu().numpy(), want) < TOL
    nnz = ctx.pattern.nnz
    mats = torch.empty(3 * nnz, dtype=torch.float64, device="cuda")
    ctx.assemble_gradients_d(mats)
    for k in range(3):
        e = np.zeros((om.nnode, 3))
        e[:, k] = 1.0
        _, _, vo = O.assemble_matrix(om, "convection", e)
        assert O.rel_diff(mats[k * nnz:(k + 1) * nnz].cpu().numpy(), vo) < TOL


def test_kuhn_lines_accumulate_and_window(cuda_ok):
    """fpb_assemble_gradient_kuhn_lines through the C ABI: accumulate = 1
    (plain read-modify-write stores) adds bitwise the values the default
    path (TMA bulk stores, accumulate = 0) writes, only in the interior
    rows of the node-plane window [kz0, kz1]; rows outside stay untouched."""
    import paper_2107_11541_b200 as P
    from paper_2107_11541_b200 import _lib

    nx, ny, nz = 37, 21, 9
    om = O.box(O.TET04, nx, ny, nz)
    om.coords = _jitter(om.coords, nx, ny, nz, seed=5)
    mesh, ctx = _ctx(P, nx, ny, nz, coords=om.coords)
    ctx.assemble_gradients_d(torch.empty(3 * ctx.pattern.nnz, dtype=torch.float64, device="cuda"))  # xyz4 staged
    nnz = ctx.pattern.nnz
    rp = ctx.pattern.rowptr_d
    idx = np.arange(mesh.nnode)
    i, j, k = idx % (nx + 1), (idx // (nx + 1)) % (ny + 1), idx // ((nx + 1) * (ny + 1))
    for kz0, kz1 in ((1, nz - 1), (3, 5), (4, 4)):
        inner = idx[(i > 0) & (i < nx) & (j > 0) & (j < ny) & (k >= kz0) & (k <= kz1)]
        rpc = rp.cpu().numpy()
        sel = torch.as_tensor(np.concatenate([np.arange(rpc[r], rpc[r + 1]) for r in inner]), device="cuda")
        mask = torch.zeros(nnz, dtype=torch.bool, device="cuda")
        mask[sel] = True
        g = torch.Generator(device="cuda").manual_seed(kz0)
        base = torch.randn(3 * nnz, dtype=torch.float64, device="cuda", generator=g)
        a = base.clone()
        _lib.call("fpb_assemble_gradient_kuhn_lines", nx, ny, nz, kz0, kz1, ctx.xyz4.data_ptr(), rp.data_ptr(), nnz,
                  0, a.data_ptr(), _lib.stream())
        b = base.clone()
        _lib.call("fpb_assemble_gradient_kuhn_lines", nx, ny, nz, kz0, kz1, ctx.xyz4.data_ptr(), rp.data_ptr(), nnz,
                  1, b.data_ptr(), _lib.stream())
        for m in range(3):
            am, bm, vm = a[m * nnz:(m + 1) * nnz], b[m * nnz:(m + 1) * nnz], base[m * nnz:(m + 1) * nnz]
            assert torch.equal(am[~mask], vm[~mask]) and torch.equal(bm[~mask], vm[~mask]), (kz0, kz1, m)
            assert torch.equal(bm[mask], vm[mask] + am[mask]), (kz0, kz1, m)
