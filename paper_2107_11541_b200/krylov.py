"""Jacobi-preconditioned CG with every vector and scalar in HBM
(krylov.py:27-89).

The recurrence, stopping rule (||r|| / ||b|| <= tol), breakdown test
(p^T A p <= 0), iteration cap, history (initial entry included) and the
true-residual evaluation at exit are the reference's.  Each iteration is
three fused kernels (q = A p with p.q; x/r/z update with r.r and r.z; p
update); convergence is decided on the device, and iterations after it are
no-ops, so the host only synchronises once per batch of iterations.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .errors import SolverBreakdownError
from .sparse import CsrMatrix, axpy_d, dot_d, dot_work, sell_copy, spmv_d, to_device, to_host

S_RZ, S_BNORM, S_TOL, S_STATUS, S_IT, S_RELRES, S_PQ, S_BETA = range(8)

# Solver workspaces (vectors, device state, history ring, the operator's
# SELL-32 copy, captured CUDA graph of one full batch), keyed by the
# operator's device arrays and the batch size: repeated solves with the same
# matrix reuse the buffers, so the batch graph is captured once and replayed
# by every later solve.
#
# The fused SpMVs run on a SELL-32 copy of the operator (sparse.SellCopy:
# one thread per row, coalesced loads, the reference's per-row summation
# order) unless its slice padding is excessive (sparse.SELL_MAX_PADDING);
# its values are re-copied at every solve start (inside the solve, ~one
# SpMV of traffic; profiles/r01o_sell).
_WS: dict = {}
_WS_MAX = 8


def _workspace(kind: str, A: CsrMatrix, nvec: int, nstate: int, cap: int, jacobi: bool) -> dict:
    key = (kind, torch.cuda.current_device(), _lib.stream(), A.rowptr_d.data_ptr(), A.colind_d.data_ptr(),
           A.vals_d.data_ptr(), A.n, cap, jacobi)
    ws = _WS.pop(key, None)
    if ws is None:
        dev = A.vals_d.device
        ws = {"v": [torch.empty(A.n, dtype=torch.float64, device=dev) for _ in range(nvec)],
              "d": torch.empty(A.n, dtype=torch.float64, device=dev),
              "state": torch.zeros(nstate, dtype=torch.float64, device=dev),
              "hist": torch.zeros(cap, dtype=torch.float64, device=dev), "graph": None,
              "sell": sell_copy(A)}
        while len(_WS) >= _WS_MAX:
            _WS.pop(next(iter(_WS)))
    _WS[key] = ws  # most recently used last
    return ws


def _sell_args(ws: dict, A: CsrMatrix) -> tuple:
    """(sell_ptr, scol, sval, idx16) for the solver kernels, values
    refreshed from A; (None, None, None, 0) = CSR kernels."""
    sc = ws["sell"]
    if sc is None:
        return None, None, None, 0
    if not sc.same_pattern(A):  # another pattern at recycled addresses
        sc = ws["sell"] = sell_copy(A)
        ws["graph"] = None
        if sc is None:
            return None, None, None, 0
    sc.refresh(A, force=True)
    A._sell = sc  # the exit residual's spmv_d reuses this copy
    return sc.args()


def _batch(ws: dict, graph: bool, full: bool, launch) -> None:
    """Run one batch of iterations: replay the captured graph for full
    batches after the first, launch directly otherwise."""
    if graph and full:
        if ws["graph"] is None:
            g = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.graph(g, stream=side):
                launch(_lib.stream())
            torch.cuda.current_stream().wait_stream(side)
            ws["graph"] = g
        ws["graph"].replay()
    else:
        launch(_lib.stream())


@dataclass
class SolverStats:
    iterations: int
    converged: bool
    residual_history: list = field(default_factory=list)
    true_residual: float = 0.0


def pcg_solve(A: CsrMatrix, b, x0=None, tol: float = 1e-8, max_iter: int | None = None,
              jacobi: bool = True, batch: int = 32, graph: bool = True):
    """Solve A x = b; returns (x, SolverStats).  numpy b -> numpy x."""
    bd, host = to_device(b)
    n = A.n
    dev = bd.device
    if max_iter is None:
        max_iter = 10 * n
    cap = max(1, min(batch, max_iter))
    ws = _workspace("pcg", A, 5, 8, cap, jacobi)
    d = ws["d"]
    if jacobi:
        _lib.call("fpb_diagonal", n, A.rowptr_d.data_ptr(), A.colind_d.data_ptr(), A.vals_d.data_ptr(),
                  d.data_ptr(), _lib.stream())
        if bool((d <= 0.0).any()):
            raise SolverBreakdownError("Jacobi preconditioner needs a positive diagonal")
    else:
        d.fill_(1.0)
    x0d = to_device(x0)[0] if x0 is not None else None
    x, r, p, q, z = ws["v"]
    state = ws["state"]
    hist_d = ws["hist"]  # hist[it % cap]
    work = dot_work()
    s = _lib.stream()
    rp, ci, va = A.rowptr_d.data_ptr(), A.colind_d.data_ptr(), A.vals_d.data_ptr()
    sell = _sell_args(ws, A)
    _lib.call("fpb_pcg_init", n, A.nnz, rp, ci, va, *sell, bd.data_ptr(), x0d.data_ptr() if x0d is not None else None,
              x.data_ptr(), r.data_ptr(), p.data_ptr(), z.data_ptr(), d.data_ptr(), state.data_ptr(),
              hist_d.data_ptr(), float(tol), work.data_ptr(), s)
    st = state.cpu().numpy()
    out = to_host if host else (lambda t: t)
    if st[S_BNORM] == 0.0:
        return out(torch.zeros(n, dtype=torch.float64, device=dev)), SolverStats(0, True, [0.0], 0.0)
    history = [float(hist_d[0].item())]
    if st[S_STATUS] == 1.0:
        return out(x.clone()), SolverStats(0, True, history, history[0])
    args = (n, A.nnz, rp, ci, va, *sell, x.data_ptr(), r.data_ptr(), p.data_ptr(), q.data_ptr(), z.data_ptr(),
            d.data_ptr(), state.data_ptr(), hist_d.data_ptr(), cap)
    done = 0
    while done < max_iter:
        k = min(cap, max_iter - done)
        # every full batch launches identical arguments: captured once per
        # workspace and replayed (3 kernels x cap iterations per replay)
        _batch(ws, graph, k == cap, lambda st, k=k: _lib.call("fpb_pcg_iterate", *args, k, work.data_ptr(), st))
        st = state.cpu().numpy()
        it = int(st[S_IT])
        if it > done:
            h = hist_d.cpu().numpy()
            history.extend(float(h[i % cap]) for i in range(done + 1, it + 1))
        done = it
        if st[S_STATUS] == 2.0:
            raise SolverBreakdownError(f"non-positive curvature p^T A p = {st[S_PQ]:.6e}")
        if st[S_STATUS] == 1.0:
            break
    converged = bool(st[S_STATUS] == 1.0)
    res = axpy_d(-1.0, spmv_d(A, x), bd)
    bnorm = float(st[S_BNORM])
    true_residual = float(np.sqrt(dot_d(res, res).item())) / bnorm
    return out(x.clone()), SolverStats(done, converged, history, true_residual)


# --------------------------------------------------------------------------
# BiCGSTAB (BASELINE config 5).  Not in the reference: the recurrence is the
# published van der Vorst algorithm as scipy.sparse.linalg.bicgstab states it
# (see include/fempack_b200.h); parity is pinned per vector op and against
# scipy through the oracle's restatement (tests/test_bicgstab.py).
# --------------------------------------------------------------------------

B_RHO, B_RHO_PREV, B_ALPHA, B_OMEGA, B_BNORM, B_ATOL, B_STATUS, B_IT, B_RELRES = range(9)
_BICG_BREAKDOWN = {2.0: "rho = (r~, r) vanished", 3.0: "(r~, A p^) vanished", 4.0: "omega vanished"}


def bicgstab_solve(A: CsrMatrix, b, x0=None, tol: float = 1e-8, max_iter: int | None = None,
                   jacobi: bool = True, batch: int = 32, graph: bool = True):
    """Solve A x = b for a general (non-symmetric) A; returns (x, SolverStats).

    Same calling convention as pcg_solve: numpy b -> numpy x, CUDA tensor b
    -> CUDA tensor x.  Breakdowns raise SolverBreakdownError like the PCG's
    curvature test (krylov.py:46-49).  history[i] = ||r_i|| / ||b||.
    """
    bd, host = to_device(b)
    n = A.n
    dev = bd.device
    if max_iter is None:
        max_iter = 10 * n
    cap = max(1, min(batch, max_iter))
    lib = _lib.load()
    ws = _workspace("bicgstab", A, 9, int(lib.fpb_bicgstab_state_size()), cap, jacobi)
    d = None
    if jacobi:
        d = ws["d"]
        _lib.call("fpb_diagonal", n, A.rowptr_d.data_ptr(), A.colind_d.data_ptr(), A.vals_d.data_ptr(),
                  d.data_ptr(), _lib.stream())
        if bool((d == 0.0).any()):
            raise SolverBreakdownError("Jacobi preconditioner needs a nonzero diagonal")
    x0d = to_device(x0)[0] if x0 is not None else None
    x, r, rt, p, ph, v, sv, sh, t = ws["v"]
    state = ws["state"]
    state.zero_()
    hist_d = ws["hist"]
    work = dot_work()
    s = _lib.stream()
    rp, ci, va = A.rowptr_d.data_ptr(), A.colind_d.data_ptr(), A.vals_d.data_ptr()
    nnz = A.nnz
    sell = _sell_args(ws, A)
    _lib.call("fpb_bicgstab_init", n, nnz, rp, ci, va, *sell, bd.data_ptr(),
              x0d.data_ptr() if x0d is not None else None, x.data_ptr(), r.data_ptr(), rt.data_ptr(),
              p.data_ptr(), v.data_ptr(), state.data_ptr(), hist_d.data_ptr(), float(tol), 0, n, 0,
              work.data_ptr(), s)
    st = state.cpu().numpy()
    out = to_host if host else (lambda q: q)
    if st[B_BNORM] == 0.0:
        return out(torch.zeros(n, dtype=torch.float64, device=dev)), SolverStats(0, True, [0.0], 0.0)
    history = [float(hist_d[0].item())]
    if st[B_STATUS] == 1.0:
        return out(x.clone()), SolverStats(0, True, history, history[0])
    if st[B_STATUS] in _BICG_BREAKDOWN:
        raise SolverBreakdownError(f"BiCGSTAB breakdown: {_BICG_BREAKDOWN[st[B_STATUS]]}")
    args = (n, nnz, rp, ci, va, *sell, d.data_ptr() if d is not None else None, x.data_ptr(), r.data_ptr(),
            rt.data_ptr(), p.data_ptr(), ph.data_ptr(), v.data_ptr(), sv.data_ptr(), sh.data_ptr(),
            t.data_ptr(), state.data_ptr(), hist_d.data_ptr(), cap)
    done = 0
    while done < max_iter:
        k = min(cap, max_iter - done)
        _batch(ws, graph, k == cap,
               lambda st, k=k: _lib.call("fpb_bicgstab_iterate", *args, k, work.data_ptr(), st))
        st = state.cpu().numpy()
        it = int(st[B_IT])
        if it > done:
            h = hist_d.cpu().numpy()
            history.extend(float(h[i % cap]) for i in range(done + 1, it + 1))
        done = it
        if st[B_STATUS] in _BICG_BREAKDOWN:
            raise SolverBreakdownError(f"BiCGSTAB breakdown: {_BICG_BREAKDOWN[st[B_STATUS]]}")
        if st[B_STATUS] == 1.0:
            break
    converged = bool(st[B_STATUS] == 1.0)
    res = axpy_d(-1.0, spmv_d(A, x), bd)
    true_residual = float(np.sqrt(dot_d(res, res).item())) / float(st[B_BNORM])
    return out(x.clone()), SolverStats(done, converged, history, true_residual)
