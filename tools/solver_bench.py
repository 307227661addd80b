"""Solver vector kernels vs the HBM roofline (development aid; bench.py
reports the same numbers in its "solver" block).

    python tools/solver_bench.py [--nx 94 --ny 94 --nz 95] [--vec-n 16974593]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_11541_b200 as P  # noqa: E402
from paper_2107_11541_b200 import _lib  # noqa: E402
from paper_2107_11541_b200 import sparse as S  # noqa: E402


def timed(fn, reps, flush):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def solver_metrics(ctx, vec_n, reps=20, hbm=6541.1):
    dev = ctx.mesh.coords_d.device
    flush = torch.empty(128 << 20, dtype=torch.float32, device=dev)
    n, nnz = ctx.pattern.n, ctx.pattern.nnz
    M = ctx.assemble_matrix(P.KernelKind.MASS)
    x = torch.randn(n, dtype=torch.float64, device=dev)
    y = torch.empty_like(x)
    out = {}
    # public sparse.spmv path: short rows run on the matrix's SELL-32 copy
    # (built once per matrix; its value copy is timed separately)
    by = 12 * nnz + 4 * (n + 1) + 16 * n
    ms = timed(lambda: S.spmv_d(M, x, y), reps, flush)
    sc = M._sell
    ms_b = timed(lambda: sc.refresh(M, force=True), reps, flush)
    out["spmv"] = {"n": n, "nnz": nnz, "padded": sc.total, "ms": ms, "GB_s": by / ms / 1e6,
                   "frac_hbm": by / ms / 1e6 / hbm, "value_copy_ms": ms_b,
                   "kernel": "SELL-32, thread per row, the reference's row-sum order (sparse.spmv)"}
    ms = timed(lambda: _lib.call("fpb_spmv", n, nnz, M.rowptr_d.data_ptr(), M.colind_d.data_ptr(),
                                 M.vals_d.data_ptr(), x.data_ptr(), y.data_ptr(), _lib.stream()), reps, flush)
    out["spmv_csr"] = {"n": n, "nnz": nnz, "ms": ms, "GB_s": by / ms / 1e6, "frac_hbm": by / ms / 1e6 / hbm,
                       "kernel": "CSR, lanes per row (fpb_spmv; long-row operators)"}
    a = torch.randn(vec_n, dtype=torch.float64, device=dev)
    b = torch.randn(vec_n, dtype=torch.float64, device=dev)
    c = torch.empty_like(a)
    ms = timed(lambda: S.axpy_d(2.5, a, b, c), reps, flush)
    out["axpy"] = {"n": vec_n, "ms": ms, "GB_s": 24 * vec_n / ms / 1e6, "frac_hbm": 24 * vec_n / ms / 1e6 / hbm}
    r = torch.empty((), dtype=torch.float64, device=dev)
    ms = timed(lambda: S.dot_d(a, b, r), reps, flush)
    out["dot"] = {"n": vec_n, "ms": ms, "GB_s": 16 * vec_n / ms / 1e6, "frac_hbm": 16 * vec_n / ms / 1e6 / hbm}
    # PCG on the pinned LAPLACIAN (bench.py:240-256 of the reference)
    L = ctx.assemble_matrix(P.KernelKind.LAPLACIAN)
    vals = L.vals_d.clone()
    rp, ci = L.rowptr_d.long(), L.colind_d.long()
    rows = torch.repeat_interleave(torch.arange(n, device=dev), rp[1:] - rp[:-1])
    hit = (rows == 0) | (ci == 0)
    vals[hit] = 0.0
    vals[(rows == 0) & (ci == 0)] = 1.0
    A = L.with_vals(vals)
    bvec = torch.as_tensor(np.random.default_rng(0).standard_normal(n), device=dev)
    bvec[0] = 0.0
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    P.pcg_solve(A, bvec, tol=1e-8)  # warm
    e0.record()
    xs, st = P.pcg_solve(A, bvec, tol=1e-8)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    it_by = 12 * nnz + 4 * (n + 1) + 8 * n * 12  # spmv + ~12 vector passes per iteration
    out["pcg"] = {"n": n, "iterations": st.iterations, "converged": st.converged, "ms": ms,
                  "ms_per_iter": ms / max(st.iterations, 1),
                  "GB_s_equiv": it_by * st.iterations / ms / 1e6, "true_residual": st.true_residual}
    # BiCGSTAB (config 5's solver) on the non-symmetric advection-diffusion
    # operator M + dt (C(u) + kappa L), dt = 0.05, kappa = 1e-2
    vel = torch.as_tensor(np.random.default_rng(0).standard_normal((n, 3)), device=dev)
    C = ctx.assemble_matrix(P.KernelKind.CONVECTION, velocity=vel)
    Ab = M.with_vals(M.vals_d + 0.05 * (C.vals_d + 1e-2 * L.vals_d))
    bb = torch.as_tensor(np.random.default_rng(1).standard_normal(n), device=dev)
    P.bicgstab_solve(Ab, bb, tol=1e-8)  # warm (graph capture)
    torch.cuda.synchronize()
    e0.record()
    xb, stb = P.bicgstab_solve(Ab, bb, tol=1e-8)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    it_by = 2 * (12 * nnz + 4 * (n + 1) + 8 * n) + 23 * 8 * n  # 2 spmv + 23 vector passes / iteration
    out["bicgstab"] = {"n": n, "iterations": stb.iterations, "converged": stb.converged, "ms": ms,
                       "ms_per_iter": ms / max(stb.iterations, 1),
                       "GB_s_equiv": it_by * stb.iterations / ms / 1e6, "true_residual": stb.true_residual}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nx", type=int, default=94)
    ap.add_argument("--ny", type=int, default=94)
    ap.add_argument("--nz", type=int, default=95)
    ap.add_argument("--vec-n", type=int, default=16_974_593)
    args = ap.parse_args()
    mesh = P.generate_box_mesh(P.ElementType.TET04, args.nx, args.ny, args.nz)
    ctx = P.AssemblyContext.build(mesh, 8)
    print(json.dumps(solver_metrics(ctx, args.vec_n), indent=1))


if __name__ == "__main__":
    main()
