"""Solver vector kernels and PCG on the B200 vs the reference goldens."""

import math

import numpy as np
import pytest

from conftest import load_golden
from oracle import fempack_np as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=["tet_6", "hex_8", "mixed_8", "tet_c1"])
def case(request, cuda_ok):
    import paper_2107_11541_b200 as P
    from gpu_cases import CASES

    return request.param, P.AssemblyContext.build(CASES[request.param](), 8), load_golden(request.param)


def test_spmv_axpy_dot(case):
    import paper_2107_11541_b200 as P

    name, ctx, g = case
    M = ctx.assemble_matrix(P.KernelKind.MASS)
    y = P.spmv(M, g["spmv_x"])
    assert O.rel_diff(y, g["spmv_y"]) < 1e-12  # own MASS values: parity 1e-12
    assert P.spmv(M, g["spmv_x"]).tobytes() == y.tobytes()  # deterministic
    out = P.axpy(2.5, g["bench_scalar0"], g["bench_scalar1"])
    assert out.tobytes() == g["axpy_out"].tobytes()  # one rounding per entry, as the reference
    x, yy = g["bench_scalar0"], g["bench_scalar1"]
    d = P.dot(x, yy)
    assert abs(d - math.fsum(x * yy)) <= 1e-12 * float(np.abs(x * yy).sum())
    assert P.dot(x, yy) == d  # bitwise reproducible
    assert P.norm2(x) == pytest.approx(float(g["norm2"]), rel=1e-13)


def test_sell_spmv_bitwise_reference(case):
    """The solver-side SELL-32 SpMV sums every row in the reference's order
    with separately rounded products (sparse.py:80-84): bit-identical to the
    reference's spmv on the reference's own MASS values."""
    import torch

    from paper_2107_11541_b200 import sparse

    name, ctx, g = case
    M = ctx.pattern.with_vals(g["mat_mass"])
    sc = sparse.SellCopy(M)
    y = sc.spmv_d(torch.as_tensor(g["spmv_x"], device="cuda")).cpu().numpy()
    assert y.tobytes() == g["spmv_y"].tobytes()


@pytest.mark.parametrize("idx16", [True, False])
def test_sell_spmv_ragged(cuda_ok, monkeypatch, idx16):
    """Empty rows, a partial last slice, rows of 1..70 entries: SELL equals
    a sequential per-row sum exactly (16-bit column offsets and int32
    columns); refresh follows value changes."""
    import torch

    from paper_2107_11541_b200 import sparse

    monkeypatch.setattr(sparse, "SELL_IDX16", idx16)

    rng = np.random.default_rng(5)
    n = 1000
    lens = rng.integers(0, 71, n)
    lens[rng.choice(n, 40, replace=False)] = 0
    rowptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    colind = np.concatenate([np.sort(rng.choice(n, k, replace=False)) for k in lens]).astype(np.int64)
    vals = rng.standard_normal(rowptr[-1])
    x = rng.standard_normal(n)

    def ref(v):
        y = np.zeros(n)
        for i in range(n):
            acc = 0.0
            for k in range(rowptr[i], rowptr[i + 1]):
                acc += v[k] * x[colind[k]]
            y[i] = acc
        return y

    A = sparse.CsrMatrix(n, rowptr, colind, vals)
    assert sparse.sell_copy(A) is None  # ~2x padding: public paths keep CSR
    sc = sparse.SellCopy(A, max_padding=float("inf"))
    assert sc.total % 32 == 0 and sc.total >= rowptr[-1]
    assert sc.idx16 == idx16 and sc.col.element_size() == (2 if idx16 else 4)
    xd = torch.as_tensor(x, device="cuda")
    assert sc.spmv_d(xd).cpu().numpy().tobytes() == ref(vals).tobytes()
    A.vals_d.mul_(-0.5)  # torch-visible change -> refresh picks it up
    y2 = sc.refresh(A).spmv_d(xd).cpu().numpy()
    assert y2.tobytes() == ref(vals * -0.5).tobytes()


def test_pcg_matches_reference(case):
    import paper_2107_11541_b200 as P

    name, ctx, g = case
    if "cg_b" not in g:
        pytest.skip("no PCG fixture")
    A = ctx.pattern.with_vals(g["cg_vals"])
    x, st = P.pcg_solve(A, g["cg_b"], tol=1e-8)
    it_ref = int(g["cg_iterations"])
    assert st.converged
    assert abs(st.iterations - it_ref) <= 1
    assert len(st.residual_history) == st.iterations + 1
    n = min(len(st.residual_history), len(g["cg_history"]))
    np.testing.assert_allclose(st.residual_history[: n - 1], g["cg_history"][: n - 1], rtol=1e-6)
    # same solution to the solver tolerance
    assert O.rel_diff(x, g["cg_x"]) < 1e-6
    assert st.true_residual <= 1e-8 * 1.01 or st.true_residual == pytest.approx(float(g["cg_true_residual"]), rel=1e-3)


def _csr(D):
    import paper_2107_11541_b200 as P

    n = D.shape[0]
    rowptr = np.zeros(n + 1, dtype=np.int64)
    cols, vals = [], []
    for i in range(n):
        nz = np.nonzero(D[i])[0]
        rowptr[i + 1] = rowptr[i] + nz.size
        cols.append(nz)
        vals.append(D[i, nz])
    return P.CsrMatrix(n, rowptr, np.concatenate(cols), np.concatenate(vals))


def test_pcg_known_answers(cuda_ok):
    """krylov known answers (test_krylov.py:16-110)."""
    import paper_2107_11541_b200 as P

    x, st = P.pcg_solve(_csr(np.eye(6)), np.arange(1.0, 7.0), tol=1e-12)
    np.testing.assert_allclose(x, np.arange(1.0, 7.0), atol=1e-15)
    assert st.iterations == 1 and st.converged and st.residual_history[0] == 1.0
    x, st = P.pcg_solve(_csr(np.array([[4.0, 1.0], [1.0, 3.0]])), np.array([1.0, 2.0]), tol=1e-14)
    np.testing.assert_allclose(x, [1 / 11, 7 / 11], atol=1e-13)
    rng = np.random.default_rng(21)
    B = rng.standard_normal((50, 50))
    x, st = P.pcg_solve(_csr(B @ B.T + 50 * np.eye(50)), rng.standard_normal(50), tol=1e-10)
    assert st.converged and st.iterations <= 55 and st.true_residual <= 2e-10
    with pytest.raises(P.SolverBreakdownError, match="curvature"):
        P.pcg_solve(_csr(np.array([[1.0, 2.0], [2.0, 1.0]])), np.array([1.0, -1.0]), tol=1e-12)
    with pytest.raises(P.SolverBreakdownError, match="diagonal"):
        P.pcg_solve(_csr(np.array([[1.0, 0.5], [0.5, -2.0]])), np.ones(2))
    x, st = P.pcg_solve(_csr(np.eye(4) * 3.0), np.zeros(4))
    assert not x.any() and st.converged and st.iterations == 0 and st.residual_history == [0.0]
    x, st = P.pcg_solve(_csr(np.diag([2.0, 4.0])), np.array([2.0, 8.0]), x0=np.array([1.0, 2.0]), tol=1e-12)
    assert st.iterations == 0 and st.converged
    rng = np.random.default_rng(24)
    B = rng.standard_normal((30, 30))
    x, st = P.pcg_solve(_csr(B @ B.T + 1e-2 * np.eye(30)), rng.standard_normal(30), tol=1e-14, max_iter=3)
    assert not st.converged and st.iterations == 3 and len(st.residual_history) == 4


def test_spmv_sell_cache_follows_writes(cuda_ok):
    """Public spmv runs on the SELL copy (bit-identical to the reference
    order); assembling new values into the same buffer (kernel write) and
    torch in-place edits are seen by the cached copy."""
    import torch

    import paper_2107_11541_b200 as P
    from paper_2107_11541_b200 import sparse
    from gpu_cases import CASES

    ctx = P.AssemblyContext.build(CASES["tet_6"](), 8)
    n = ctx.mesh.nnode
    vel = torch.as_tensor(np.random.default_rng(3).standard_normal((n, 3)), device="cuda")
    out = torch.empty(ctx.pattern.nnz, dtype=torch.float64, device="cuda")
    A = ctx.pattern.with_vals(out)
    x = torch.as_tensor(np.random.default_rng(4).standard_normal(n), device="cuda")

    def seq(vals):
        rp, ci, v, xx = A.rowptr, A.colind, vals.cpu().numpy(), x.cpu().numpy()
        y = np.zeros(n)
        for i in range(n):
            acc = 0.0
            for k in range(rp[i], rp[i + 1]):
                acc += v[k] * xx[ci[k]]
            y[i] = acc
        return y

    ctx.assemble_matrix_d(P.KernelKind.MASS, None, out)
    y1 = sparse.spmv_d(A, x).cpu().numpy()  # SELL copy built
    y2 = sparse.spmv_d(A, x).cpu().numpy()  # reused
    assert getattr(A, "_sell", None) is not None
    assert y1.tobytes() == y2.tobytes() == seq(out).tobytes()
    ctx.assemble_matrix_d(P.KernelKind.CONVECTION, vel, out)  # kernel write, same buffer
    y3 = sparse.spmv_d(A, x).cpu().numpy()
    assert y3.tobytes() == seq(out).tobytes()
    out.mul_(2.0)  # torch in-place edit
    y4 = sparse.spmv_d(A, x).cpu().numpy()
    assert np.abs(y4 - 2.0 * y3).max() <= 1e-14 * np.abs(y3).max()
