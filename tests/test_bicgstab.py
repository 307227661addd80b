"""BiCGSTAB (BASELINE config 5).  The reference has no BiCGSTAB (SURVEY.md
8(f) rank 1), so the oracle's restatement is pinned against
scipy.sparse.linalg.bicgstab (CPU tests), and the device solver is checked
against the oracle on the same assembled advection-diffusion systems."""

import numpy as np
import pytest

from oracle import fempack_np as O


def _system(etype, dims, dt=0.05, kappa=0.01, seed=0):
    m = O.box(etype, *dims)
    vel, sc = O.bench_fields(m.nnode, m.dim, seed)
    rp, ci, M = O.assemble_matrix(m, "mass")
    _, _, C = O.assemble_matrix(m, "convection", vel)
    _, _, L = O.assemble_matrix(m, "laplacian")
    A = M + dt * (C + kappa * L)  # mass + dt (convection + kappa laplacian): non-symmetric
    return m, rp, ci, A, sc[0]


SYSTEMS = {
    "tet": (O.TET04, (6, 5, 4)),
    "hex": (O.HEX08, (5, 4, 4)),
    "quad": (O.QUAD04, (9, 7)),
}


def _scipy(rp, ci, A, b, tol, jacobi, x0=None):
    import scipy.sparse as sp
    import scipy.sparse.linalg as sla

    S = sp.csr_matrix((A, ci, rp), shape=(rp.size - 1,) * 2)
    M = None
    if jacobi:
        d = S.diagonal()
        M = sla.LinearOperator(S.shape, matvec=lambda v: v / d)
    it = [0]
    x, info = sla.bicgstab(S, b, x0=x0, rtol=tol, atol=0.0, M=M, callback=lambda xk: it.__setitem__(0, it[0] + 1))
    return x, it[0], info


@pytest.mark.parametrize("name", sorted(SYSTEMS))
@pytest.mark.parametrize("jacobi", [True, False])
def test_oracle_matches_scipy(name, jacobi):
    m, rp, ci, A, b = _system(*SYSTEMS[name])
    x, it, status, hist = O.bicgstab(rp, ci, A, b, tol=1e-10, jacobi=jacobi)
    xs, its, info = _scipy(rp, ci, A, b, 1e-10, jacobi)
    assert status == 0 and info == 0
    # scipy does not invoke the callback for a final half step (exit on ||s||)
    assert it - its in (0, 1)
    # scipy's dots are BLAS (blocked summation), the oracle's sequential: the
    # iterates agree to rounding, amplified by the conditioning unpreconditioned
    assert O.rel_diff(x, xs) < (1e-12 if jacobi else 1e-9)
    r = b - O.spmv(rp, ci, A, x)
    assert np.linalg.norm(r) < 1e-10 * np.linalg.norm(b) * 1.0001
    assert len(hist) == it + 1


def test_oracle_x0_and_zero_rhs():
    m, rp, ci, A, b = _system(*SYSTEMS["tet"])
    x0 = np.linspace(-1.0, 1.0, m.nnode)
    x, it, status, _ = O.bicgstab(rp, ci, A, b, x0=x0, tol=1e-9)
    xs, its, info = _scipy(rp, ci, A, b, 1e-9, True, x0=x0)
    assert status == 0 and it - its in (0, 1) and O.rel_diff(x, xs) < 1e-12
    z, it0, st0, h0 = O.bicgstab(rp, ci, A, np.zeros(m.nnode))
    assert it0 == 0 and st0 == 0 and not z.any()


# ---------------------------------------------------------------- device
@pytest.fixture(scope="module")
def P(cuda_ok):
    import paper_2107_11541_b200 as P

    return P


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(SYSTEMS))
@pytest.mark.parametrize("jacobi", [True, False])
def test_device_matches_oracle(P, name, jacobi):
    m, rp, ci, A, b = _system(*SYSTEMS[name])
    pat = P.CsrMatrix(m.nnode, rp, ci, A)
    x, st = P.bicgstab_solve(pat, b, tol=1e-10, jacobi=jacobi)
    xo, ito, so, ho = O.bicgstab(rp, ci, A, b, tol=1e-10, jacobi=jacobi)
    assert st.converged and so == 0
    assert abs(st.iterations - ito) <= 1
    assert len(st.residual_history) == st.iterations + 1
    n = min(len(ho), len(st.residual_history), 6)
    np.testing.assert_allclose(st.residual_history[:n], ho[:n], rtol=1e-8)
    assert O.rel_diff(x, xo) < 1e-8
    assert st.true_residual < 1e-10 * 1.01


@pytest.mark.gpu
def test_device_torch_in_torch_out_and_x0(P):
    import torch

    m, rp, ci, A, b = _system(*SYSTEMS["tet"])
    pat = P.CsrMatrix(m.nnode, rp, ci, A)
    x0 = np.linspace(-1.0, 1.0, m.nnode)
    xt, st = P.bicgstab_solve(pat, torch.as_tensor(b, device="cuda"), x0=torch.as_tensor(x0, device="cuda"),
                              tol=1e-9)
    assert isinstance(xt, torch.Tensor) and xt.is_cuda
    xo, ito, so, _ = O.bicgstab(rp, ci, A, b, x0=x0, tol=1e-9)
    assert abs(st.iterations - ito) <= 1 and O.rel_diff(xt.cpu().numpy(), xo) < 1e-8
    x2, st2 = P.bicgstab_solve(pat, torch.as_tensor(b, device="cuda"), x0=torch.as_tensor(x0, device="cuda"),
                               tol=1e-9)
    assert torch.equal(xt, x2)  # deterministic reductions: bitwise reproducible
    z, stz = P.bicgstab_solve(pat, np.zeros(m.nnode))
    assert stz.iterations == 0 and not z.any()


@pytest.mark.gpu
def test_device_iteration_cap_and_graph_batches(P):
    m, rp, ci, A, b = _system(O.TET04, (10, 9, 8))
    pat = P.CsrMatrix(m.nnode, rp, ci, A)
    xo, ito, so, ho = O.bicgstab(rp, ci, A, b, tol=1e-11, jacobi=True)
    # small batches exercise the CUDA-graph replay path
    x, st = P.bicgstab_solve(pat, b, tol=1e-11, batch=3)
    assert st.converged and abs(st.iterations - ito) <= 2 and O.rel_diff(x, xo) < 1e-8
    xc, stc = P.bicgstab_solve(pat, b, tol=1e-14, max_iter=4, batch=3)
    assert stc.iterations == 4 and not stc.converged
    xo4, it4, s4, _ = O.bicgstab(rp, ci, A, b, tol=1e-14, max_iter=4)
    assert s4 == -1 and O.rel_diff(xc, xo4) < 1e-9


@pytest.mark.gpu
def test_device_zero_diagonal_raises(P):
    m, rp, ci, A, b = _system(*SYSTEMS["tet"])
    A2 = A.copy()
    rows = np.repeat(np.arange(m.nnode), np.diff(rp))
    A2[(rows == ci) & (rows == 3)] = 0.0
    with pytest.raises(P.SolverBreakdownError):
        P.bicgstab_solve(P.CsrMatrix(m.nnode, rp, ci, A2), b)
