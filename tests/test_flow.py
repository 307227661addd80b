"""Device time loop against fixtures produced by the
unmodified reference (tools/make_golden_flow.py, tests/golden/flow_*.npz):
boundary extraction, Robin structures (assembly.py:383-411), the pressure
operator built with the device transpose / spgemm / csr_add /
apply_dirichlet (timeloop.py:184-231, sparse.py:133-254) and two
FlowSolver.step calls (timeloop.py:336-440).  The sparse setup operations are
also checked one by one against scipy / numpy restatements."""

import numpy as np
import pytest

from conftest import load_golden
from oracle import fempack_np as O

CASES = ["mixed", "tet_rest", "tet_smooth", "quad_tg", "hex_uniform", "tri_smooth", "tet_jitter", "hex_jitter"]


def _close(got, want, rtol=1e-9):
    """max |got - want| <= rtol * max(|want|, 1e-3): fields that are pure
    round-off (e.g. the pressure of a uniform flow, ~1e-13) are compared
    absolutely."""
    scale = max(float(np.abs(want).max(initial=0.0)), 1e-3)
    return float(np.abs(got - want).max(initial=0.0)) <= rtol * scale


# ----------------------------------------------------------------- CPU only
def test_rk3_tableau_integrates_linear_ode():
    """SSP-RK3 with the reference tableau (timeloop.py:38-61) is third order."""
    from paper_2107_11541_b200.timeloop import integrate_ode

    errs = []
    for nsteps in (10, 20):
        y = integrate_ode(1.0, 1.0 / nsteps, nsteps, lambda v: -v)
        errs.append(abs(y - np.exp(-1.0)))
    assert errs[0] / errs[1] == pytest.approx(8.0, rel=0.1)


def test_config_and_state_validation():
    from paper_2107_11541_b200 import ConfigurationError, FlowState, TimeConfig

    with pytest.raises(ConfigurationError):
        TimeConfig(dt=0.0).validate()
    with pytest.raises(ConfigurationError):
        TimeConfig(dt=1.0, tol=0.0).validate()
    st = FlowState(np.zeros((4, 2)), np.zeros(4), np.zeros(4), np.zeros((2, 4)))
    st.validate()
    bad = st.copy()
    bad.heat[1] = np.nan
    with pytest.raises(ConfigurationError):
        bad.validate()
    with pytest.raises(ConfigurationError):
        FlowState(np.zeros((4, 2)), np.zeros(4), np.zeros(3), np.zeros((2, 4))).validate()


# ------------------------------------------------------------------ device
def _mesh(P, spec):
    import torch

    spec = [str(s) for s in spec]
    if spec[0] == "mixed":
        m, _ = P.renumber_by_type(P.generate_mixed_mesh(*map(int, spec[1:]), fraction=0.5))
        return m
    dims = list(map(int, spec[2:]))
    m = P.generate_box_mesh(P.ElementType[spec[1]], *dims)
    if spec[0] == "jitter":  # same jitter as tools/make_golden_flow.py
        rng = np.random.default_rng(3)
        x = m.coords.copy()
        h = np.array([1.0 / d for d in dims])
        lo, hi = x.min(axis=0), x.max(axis=0)
        interior = np.all((x > lo + 1e-12) & (x < hi - 1e-12), axis=1)
        x[interior] += 0.2 * h * rng.uniform(-1.0, 1.0, size=(int(interior.sum()), x.shape[1]))
        m.coords_d.copy_(torch.as_tensor(x, device="cuda"))
        m._coords_h = None
    return m


def _initial(P, name, mesh, g):
    st = P.FlowState(g["s0_velocity"].copy(), g["s0_pressure"].copy(), g["s0_heat"].copy(), g["s0_species"].copy())
    return st


def _solver(P, name, g, mesh):
    kw = {}
    if g["robin_alpha"] or g["robin_beta"]:
        kw.update(robin_alpha=float(g["robin_alpha"]), robin_beta=float(g["robin_beta"]))
    if "dirichlet_nodes" in g:
        kw.update(dirichlet_nodes=g["dirichlet_nodes"], dirichlet_values=g["dirichlet_values"])
    cfg = P.TimeConfig(dt=float(g["dt"]), nsteps=2, tol=float(g["tol"]))
    return P.FlowSolver(mesh, cfg, layout="packed", **kw)


@pytest.fixture(scope="module", params=CASES)
def case(request, cuda_ok):
    import paper_2107_11541_b200 as P

    g = load_golden(f"flow_{request.param}")
    mesh = _mesh(P, g["spec"])
    return request.param, P, g, mesh, _solver(P, request.param, g, mesh)


@pytest.mark.gpu
def test_boundary_nodes_match_reference(case):
    name, P, g, mesh, solver = case
    np.testing.assert_array_equal(mesh.boundary_nodes(), g["boundary_nodes"])


@pytest.mark.gpu
def test_robin_structures_match_reference(case):
    name, P, g, mesh, solver = case
    if "robin_vals" not in g:
        pytest.skip("no Robin terms in this case")
    R, load = P.assemble_boundary(mesh, solver.ctx.pattern, float(g["robin_alpha"]), float(g["robin_beta"]))
    assert O.rel_diff(R.vals, g["robin_vals"]) < 1e-13
    assert O.rel_diff(load, g["robin_load"]) < 1e-13


@pytest.mark.gpu
def test_pressure_operator_matches_reference(case):
    name, P, g, mesh, solver = case
    assert O.rel_diff(solver.lumped, g["lumped"]) < 1e-13
    L = solver.laplacian
    np.testing.assert_array_equal(L.rowptr, g["lap_rowptr"])
    np.testing.assert_array_equal(L.colind, g["lap_colind"])
    assert O.rel_diff(L.vals, g["lap_vals"]) < 1e-12
    D = solver.div_mats[0]
    np.testing.assert_array_equal(D.rowptr, g["div0_rowptr"])
    np.testing.assert_array_equal(D.colind, g["div0_colind"])
    assert O.rel_diff(D.vals, g["div0_vals"]) < 1e-12


@pytest.mark.gpu
def test_two_steps_match_reference(case):
    name, P, g, mesh, solver = case
    st = _initial(P, name, mesh, g)
    for k in (1, 2):
        st, diag = solver.step(st)
        if diag.solver.iterations == 0 and diag.solver.residual_history == [0.0]:
            # exactly zero pressure RHS: a uniform velocity (hex_uniform) has
            # zero interior divergence, which the continuity matrices here
            # cancel exactly and the reference's to round-off — its solve
            # then iterates on noise; the increment must be round-off there
            prev = g["s0_pressure"] if k == 1 else g[f"s{k - 1}_pressure"]
            assert np.abs(g[f"s{k}_pressure"] - prev).max() < 1e-10
        else:
            assert abs(diag.solver.iterations - int(g[f"s{k}_iterations"])) <= 1
        for f in ("velocity", "pressure", "heat", "species"):
            # the pressure solve runs to tol (1e-12 / 1e-13) on both sides
            assert _close(getattr(st, f), g[f"s{k}_{f}"]), (name, k, f)
        assert diag.div_star == pytest.approx(float(g[f"s{k}_div_star"]), rel=1e-9, abs=1e-14)
        assert diag.div_after == pytest.approx(float(g[f"s{k}_div_after"]), rel=1e-3, abs=1e-10)
        cells = diag.timings
        assert ("MatrixAssembly", "NavierStokes") in cells and ("AlgebraicSolver", "NavierStokes") in cells
        assert all(v >= 0.0 for v in cells.values())


@pytest.mark.gpu
def test_run_keeps_state_on_device_and_matches_steps(case):
    name, P, g, mesh, solver = case
    st, diags = solver.run(_initial(P, name, mesh, g), 2)
    assert len(diags) == 2
    for f in ("velocity", "pressure", "heat", "species"):
        assert _close(getattr(st, f), g[f"s2_{f}"]), (name, f)


# ----------------------------------------------------- sparse setup ops
def _rand_csr(n, density, seed):
    import scipy.sparse as sp

    rng = np.random.default_rng(seed)
    A = sp.random(n, n, density=density, random_state=rng, format="csr")
    A = A + sp.eye(n, format="csr")
    A.sort_indices()
    return A


@pytest.mark.gpu
def test_transpose_spgemm_add_dirichlet_vs_scipy(cuda_ok):
    import scipy.sparse as sp

    import paper_2107_11541_b200 as P

    A = _rand_csr(300, 0.03, 1)
    B = _rand_csr(300, 0.02, 2)
    Ad = P.CsrMatrix(300, A.indptr, A.indices, A.data)
    Bd = P.CsrMatrix(300, B.indptr, B.indices, B.data)
    T = P.transpose_csr(Ad)
    At = A.T.tocsr()
    At.sort_indices()
    np.testing.assert_array_equal(T.rowptr, At.indptr)
    np.testing.assert_array_equal(T.colind, At.indices)
    np.testing.assert_array_equal(T.vals, At.data)  # a permutation: exact
    C = P.spgemm(Ad, Bd)
    Cs = (A @ B).tocsr()
    Cs.sort_indices()
    # structural pattern: every product visited, explicit zeros kept
    assert C.nnz >= Cs.nnz
    np.testing.assert_allclose(C.to_dense(), Cs.toarray(), rtol=1e-13, atol=1e-15)
    S = P.csr_add(Ad, Bd)
    Ss = (A + B).tocsr()
    Ss.sort_indices()
    np.testing.assert_array_equal(S.rowptr, Ss.indptr)
    np.testing.assert_array_equal(S.colind, Ss.indices)
    np.testing.assert_array_equal(S.vals, Ss.data)
    d = np.random.default_rng(3).uniform(0.5, 2.0, 300)
    N = P.normal_product(Ad, d)
    np.testing.assert_allclose(N.to_dense(), (A.T @ sp.diags(d) @ A).toarray(), rtol=1e-12, atol=1e-14)
    nodes = np.array([0, 17, 299])
    vals = np.array([1.0, -2.0, 0.5])
    b = np.random.default_rng(4).standard_normal(300)
    Dd, bd = P.apply_dirichlet(Ad, nodes, vals, b)
    want = A.toarray().copy()
    lift = np.zeros(300)
    lift[nodes] = vals
    bw = b - want[:, nodes] @ vals
    bw[nodes] = vals
    want[nodes, :] = 0.0
    want[:, nodes] = 0.0
    want[nodes, nodes] = 1.0
    np.testing.assert_array_equal(Dd.to_dense(), want)
    np.testing.assert_allclose(bd, bw, rtol=1e-14, atol=1e-14)


@pytest.mark.gpu
def test_mesh_size_and_cfl_warning(cuda_ok):
    """hmin = min element volume^(1/dim) (timeloop.py:293-301) and the CFL
    warning (timeloop.py:317-330)."""
    import warnings

    import paper_2107_11541_b200 as P

    mesh = P.generate_box_mesh(P.ElementType.TET04, 5, 4, 3)
    solver = P.FlowSolver(mesh, P.TimeConfig(dt=1e-3))
    h = (1.0 / 5) * (1.0 / 4) * (1.0 / 3) / 6.0
    assert solver._hmin == pytest.approx(h ** (1.0 / 3.0), rel=1e-12)
    st = P.FlowState.zeros(mesh)
    st.velocity[:, 0] = 1.0
    with warnings.catch_warnings():
        warnings.simplefilter("error")
        solver.step(st)  # CFL = 1e-3 / hmin < 1: silent
    fast = P.FlowSolver(mesh, P.TimeConfig(dt=1.0))
    with pytest.warns(RuntimeWarning, match="CFL"):
        try:
            fast.step(st)
        except P.StepFailureError:
            pass
