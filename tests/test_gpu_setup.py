"""Setup path on the B200, bit-exact against the reference's own outputs
(tests/golden, made by tools/make_golden.py): mesh coordinates and
connectivity, lane packs, CSR graph and element->CSR maps."""

import hashlib

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a).astype(np.int64)).tobytes()).hexdigest()


@pytest.fixture(scope="module", params=["tri_4x3", "quad_4x3", "tet_6", "pyr_6", "hex_8",
                                        "mixed_8", "mixed_3x2x2", "tet_c1"])
def case(request, cuda_ok):
    from gpu_cases import CASES

    return request.param, CASES[request.param](), load_golden(request.param)


def test_mesh_bitwise(case):
    name, mesh, g = case
    assert mesh.coords.tobytes() == g["coords"].tobytes(), name
    assert [gr.etype.value for gr in mesh.groups] == list(g["etypes"])
    for gi, gr in enumerate(mesh.groups):
        np.testing.assert_array_equal(gr.conn, g[f"conn{gi}"])


def test_pattern_bitwise(case):
    import paper_2107_11541_b200 as P

    name, mesh, g = case
    pat = P.build_node_pattern(mesh)
    np.testing.assert_array_equal(pat.rowptr, g["rowptr"])
    assert sha(pat.colind) == str(g["colind_sha"])
    if "colind" in g:
        np.testing.assert_array_equal(pat.colind, g["colind"])


@pytest.mark.parametrize("vs", [8, 32])
def test_packs_and_maps_bitwise(case, vs):
    import paper_2107_11541_b200 as P

    name, mesh, g = case
    ctx = P.AssemblyContext.build(mesh, vector_size=vs)
    for gi, gd in enumerate(ctx.groups):
        assert sha(gd.packset.lane_conn) == str(g[f"lane_conn{gi}_vs{vs}_sha"]), (name, gi)
        assert sha(gd.pos_packed) == str(g[f"pos_packed{gi}_vs{vs}_sha"]), (name, gi)
        assert sha(gd.pos_scalar) == str(g[f"pos_scalar{gi}_sha"]), (name, gi)
        assert gd.packset.npadded == gd.packset.npacks * vs - gd.nelem


def test_missing_pair_raises_scatter_pattern_error(cuda_ok):
    import paper_2107_11541_b200 as P

    mesh = P.generate_box_mesh(P.ElementType.QUAD04, 2, 2)
    other = P.build_node_pattern(P.generate_box_mesh(P.ElementType.QUAD04, 1, 1))
    with pytest.raises(P.ScatterPatternError):
        P.matrix_positions(mesh.groups[0].conn, other)


def test_pattern_keeps_diagonal_of_unused_node(cuda_ok):
    import torch

    import paper_2107_11541_b200 as P

    mesh = P.generate_box_mesh(P.ElementType.QUAD04, 1, 1)
    mesh.coords_d = torch.cat([mesh.coords_d, torch.tensor([[9.0, 9.0]], dtype=torch.float64,
                                                            device=mesh.coords_d.device)])
    A = P.build_node_pattern(mesh)
    assert A.n == 5 and np.diff(A.rowptr)[4] == 1 and A.colind[A.rowptr[4]] == 4


def test_inverted_element_reported_like_reference(cuda_ok):
    """Swapping two nodes of hex 1 inverts it (test_assembly.py:338-345)."""
    import torch

    import paper_2107_11541_b200 as P

    mesh = P.generate_box_mesh(P.ElementType.HEX08, 2, 1, 1)
    c = mesh.groups[0].conn_d
    c[1, [1, 3]] = c[1, [3, 1]].clone()
    mesh.groups[0]._conn_h = None
    ctx = P.AssemblyContext.build(mesh, vector_size=4)
    with pytest.raises(P.InvertedElementError) as ei:
        ctx.refresh_geometry("packed")
    assert ei.value.element == 1
    assert ei.value.det < 0


def test_large_mesh_setup_invariants(cuda_ok):
    """C2 (5,036,520 tets): sizes from SURVEY 8(a) a1-a3 and CSR invariants."""
    import torch

    import paper_2107_11541_b200 as P

    mesh = P.generate_box_mesh(P.ElementType.TET04, 94, 94, 95)
    assert mesh.nelem == 5_036_520 and mesh.nnode == 866_400
    pat = P.build_node_pattern(mesh)
    assert pat.nnz == 12_779_022
    rp, ci = pat.rowptr_d.long(), pat.colind_d.long()
    # strictly ascending columns within each row and every diagonal present
    rows = torch.repeat_interleave(torch.arange(pat.n, device=rp.device), rp[1:] - rp[:-1])
    same = rows[1:] == rows[:-1]
    assert bool((ci[1:][same] > ci[:-1][same]).all())
    assert int((ci == rows).sum()) == pat.n
    # symmetric graph: (i, j) present iff (j, i) present
    k1 = torch.sort(rows * pat.n + ci).values
    k2 = torch.sort(ci * pat.n + rows).values
    assert bool((k1 == k2).all())


def test_inverted_element_raised_by_assembly(cuda_ok):
    import paper_2107_11541_b200 as P

    mesh = P.generate_box_mesh(P.ElementType.HEX08, 2, 1, 1)
    c = mesh.groups[0].conn_d
    c[1, [1, 3]] = c[1, [3, 1]].clone()
    ctx = P.AssemblyContext.build(mesh, vector_size=2)
    with pytest.raises(P.InvertedElementError) as ei:
        ctx.assemble_matrix(P.KernelKind.MASS, "scalar")
    assert ei.value.element == 1 and ei.value.det < 0.0
