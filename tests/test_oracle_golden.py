"""Pin the CPU oracle (oracle/fempack_np.py) against the reference's own
outputs (tests/golden/*.npz, produced by tools/make_golden.py from the
unmodified reference).  CPU only."""

import hashlib

import numpy as np
import pytest

from conftest import golden_names, load_golden
from oracle import fempack_np as O

CASES = {
    "tri_4x3": lambda: O.box(O.TRI03, 4, 3),
    "quad_4x3": lambda: O.box(O.QUAD04, 4, 3),
    "tet_6": lambda: O.box(O.TET04, 6, 6, 6),
    "pyr_6": lambda: O.box(O.PYR05, 6, 6, 6),
    "hex_8": lambda: O.box(O.HEX08, 8, 8, 8),
    "mixed_8": lambda: O.mixed(8, 8, 8, 0.5),
    "mixed_3x2x2": lambda: O.mixed(3, 2, 2, 0.5),
    "tet_c1": lambda: O.box(O.TET04, 20, 20, 21),
}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a.astype(np.int64)).tobytes()).hexdigest()


def test_all_goldens_have_a_case():
    assert set(golden_names()) == set(CASES)


def test_reference_tables_bitwise():
    g = load_golden("elements")
    for et in (O.TRI03, O.QUAD04, O.TET04, O.PYR05, O.HEX08):
        N, dN, w = O.reference_element(et)
        assert N.tobytes() == g[f"{et}_N"].tobytes()
        assert dN.tobytes() == g[f"{et}_dN"].tobytes()
        assert w.tobytes() == g[f"{et}_w"].tobytes()


@pytest.fixture(scope="module", params=sorted(CASES))
def case(request):
    return request.param, CASES[request.param](), load_golden(request.param)


def test_mesh_bitwise(case):
    name, m, g = case
    assert m.coords.tobytes() == g["coords"].tobytes(), name
    assert [e for e, _ in m.groups] == list(g["etypes"])
    for gi, (_, conn) in enumerate(m.groups):
        np.testing.assert_array_equal(conn, g[f"conn{gi}"])


def test_pattern_and_maps_bitwise(case):
    name, m, g = case
    rowptr, colind = O.build_node_pattern(m.nnode, [c for _, c in m.groups])
    np.testing.assert_array_equal(rowptr, g["rowptr"])
    assert sha(colind) == str(g["colind_sha"])
    offset = 0
    for gi, (_, conn) in enumerate(m.groups):
        pos = O.matrix_positions(conn, rowptr, colind)
        assert sha(pos) == str(g[f"pos_scalar{gi}_sha"])
        for vs in (8, 32):
            lc, ei = O.build_packs(conn, vs)
            assert sha(lc) == str(g[f"lane_conn{gi}_vs{vs}_sha"])
            assert sha(O.packed_positions(pos, ei)) == str(g[f"pos_packed{gi}_vs{vs}_sha"])
        offset += conn.shape[0]


def test_fields_bitwise(case):
    name, m, g = case
    vel, sc = O.bench_fields(m.nnode, m.dim)
    assert vel.tobytes() == g["bench_vel"].tobytes()
    for s in range(3):
        assert sc[s].tobytes() == g[f"bench_scalar{s}"].tobytes()


def test_matrices(case):
    name, m, g = case
    vel = g["bench_vel"]
    pat = (g["rowptr"], None)
    for key, kind, v in (("mass", "mass", None), ("laplacian", "laplacian", None),
                         ("convection", "convection", vel)):
        if f"mat_{key}" not in g:
            continue
        _, _, vals = O.assemble_matrix(m, kind, v)
        # the oracle restates the packed path op for op: bitwise
        assert vals.tobytes() == g[f"mat_{key}"].tobytes(), (name, key)
    for k in range(m.dim):
        if f"mat_grad{k}" in g:
            unit = np.zeros((m.nnode, m.dim))
            unit[:, k] = 1.0
            _, _, vals = O.assemble_matrix(m, "convection", unit)
            assert vals.tobytes() == g[f"mat_grad{k}"].tobytes()


def test_rhs(case):
    name, m, g = case
    vel = g["bench_vel"]
    r = O.assemble_rhs(m, "momentum_rhs", vel, None, 1.0, 1e-2, 0.0)
    assert r.tobytes() == g["rhs_momentum"].tobytes(), name
    assert O.rel_diff(r, g["rhs_momentum_scalar_layout"]) < 1e-12
    for s in range(3):
        r = O.assemble_rhs(m, "scalar_rhs", vel, g[f"bench_scalar{s}"], 1.0, 0.0, 1e-2)
        assert r.tobytes() == g[f"rhs_scalar{s}"].tobytes()
    sv, sp = O.smooth_fields(m.coords)
    r = O.assemble_rhs(m, "momentum_rhs", sv, None, 1.2, 1e-2, 0.0)
    assert r.tobytes() == g["rhs_momentum_smooth"].tobytes()


def test_vector_ops(case):
    name, m, g = case
    rowptr, colind = O.build_node_pattern(m.nnode, [c for _, c in m.groups])
    _, _, M = O.assemble_matrix(m, "mass")
    y = O.spmv(rowptr, colind, M, g["spmv_x"])
    assert y.tobytes() == g["spmv_y"].tobytes()
    out = O.axpy(2.5, g["bench_scalar0"], g["bench_scalar1"])
    assert out.tobytes() == g["axpy_out"].tobytes()
    assert O.dot(g["bench_scalar0"], g["bench_scalar1"]) == float(g["dot"])
    assert O.norm2(g["bench_scalar0"]) == float(g["norm2"])


def test_pcg(case):
    name, m, g = case
    if "cg_b" not in g:
        pytest.skip("no PCG fixture")
    rowptr, colind = O.build_node_pattern(m.nnode, [c for _, c in m.groups])
    _, _, lap = O.assemble_matrix(m, "laplacian")
    vals = O.apply_dirichlet_pin(rowptr, colind, lap, [0])
    assert vals.tobytes() == g["cg_vals"].tobytes()
    x, it, conv, hist, tr = O.pcg_solve(rowptr, colind, vals, g["cg_b"], tol=1e-8)
    assert it == int(g["cg_iterations"])
    assert np.array(hist).tobytes() == g["cg_history"].tobytes()
    assert x.tobytes() == g["cg_x"].tobytes()


def test_c_port_bitwise_vs_reference():
    """The C restatement (bench cpu_baseline) reproduces the reference
    packed path bit for bit when run on one thread."""
    from oracle import cport

    for name in ("tet_6", "hex_8", "tet_c1"):
        g = load_golden(name)
        m = CASES[name]()
        (et, conn), = m.groups
        pg = cport.PackedGroup(et, conn, m.coords, vs=8, nthreads=1)
        rhs = pg.momentum_rhs(g["bench_vel"], 1.0, 1e-2, np.zeros((m.nnode, 3)))
        assert rhs.tobytes() == g["rhs_momentum"].tobytes(), name
        rowptr, colind = O.build_node_pattern(m.nnode, [conn])
        pos = O.packed_positions(O.matrix_positions(conn, rowptr, colind), pg.elem_index)
        vals = pg.convection(g["bench_vel"], np.ascontiguousarray(pos), np.zeros(colind.size))
        assert vals.tobytes() == g["mat_convection"].tobytes(), name
        for s in range(3):
            rs = pg.scalar_rhs(g["bench_vel"], g[f"bench_scalar{s}"], 1e-2, np.zeros(m.nnode))
            assert rs.tobytes() == g[f"rhs_scalar{s}"].tobytes(), (name, s)
        # geometry recomputed chunk by chunk (the config-4/5 scale path): same bits
        pc = cport.PackedGroup(et, conn, m.coords, vs=8, nthreads=1, cache_geometry=False, chunk=7)
        rc = pc.momentum_rhs(g["bench_vel"], 1.0, 1e-2, np.zeros((m.nnode, 3)))
        assert rc.tobytes() == g["rhs_momentum"].tobytes(), name
        vc = pc.convection(g["bench_vel"], np.ascontiguousarray(pos), np.zeros(colind.size))
        assert vc.tobytes() == g["mat_convection"].tobytes(), name
        sc = pc.scalar_rhs(g["bench_vel"], g["bench_scalar0"], 1e-2, np.zeros(m.nnode))
        assert sc.tobytes() == g["rhs_scalar0"].tobytes(), name
        y = cport.spmv(rowptr, colind, O.assemble_matrix(m, "mass")[2], g["spmv_x"])
        assert y.tobytes() == g["spmv_y"].tobytes()
        # threaded run: same values up to summation order
        pg4 = cport.PackedGroup(et, conn, m.coords, vs=8, nthreads=4)
        r4 = pg4.momentum_rhs(g["bench_vel"], 1.0, 1e-2, np.zeros((m.nnode, 3)))
        assert O.rel_diff(r4, g["rhs_momentum"]) < 1e-13
