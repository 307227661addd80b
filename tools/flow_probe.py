"""FlowSolver pressure-operator SpMV / PCG formats (development aid).

    python tools/flow_probe.py [--max-mean-row 32]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_11541_b200 as P  # noqa: E402
from paper_2107_11541_b200 import _lib, sparse  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-padding", type=float, default=None, help="0 forces the CSR kernels")
    args = ap.parse_args()
    if args.max_padding is not None:
        sparse.SELL_MAX_PADDING = args.max_padding
    mesh = P.generate_box_mesh(P.ElementType.TET04, 94, 94, 95)
    solver = P.FlowSolver(mesh, P.TimeConfig(dt=5e-4, tol=1e-8), robin_alpha=1.0, robin_beta=0.1)
    L = solver.laplacian
    n, nnz = L.n, L.nnz
    dev = L.vals_d.device
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    x = torch.as_tensor(np.random.default_rng(0).standard_normal(n), device=dev)
    y = torch.empty_like(x)

    def timeit(fn, reps=20):
        for _ in range(3):
            fn()
        ts = []
        for _ in range(reps):
            flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return float(np.median(ts))

    by = 12 * nnz + 20 * n
    out = {"n": n, "nnz": nnz, "mean_row": nnz / n}
    t = timeit(lambda: _lib.call("fpb_spmv", n, nnz, L.rowptr_d.data_ptr(), L.colind_d.data_ptr(),
                                 L.vals_d.data_ptr(), x.data_ptr(), y.data_ptr(), _lib.stream()))
    out["csr_ms"], out["csr_GBs"] = t, by / t / 1e6
    sc = sparse.sell_copy(L)
    if sc is not None:
        t = timeit(lambda: sc.spmv_d(x, y))
        out["sell_ms"], out["sell_GBs"], out["sell_padded"] = t, by / t / 1e6, sc.total
    b = torch.as_tensor(np.random.default_rng(1).standard_normal(n), device=dev)
    P.pcg_solve(L, b, tol=0.0, max_iter=64)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _, st = P.pcg_solve(L, b, tol=0.0, max_iter=64)
    e1.record()
    torch.cuda.synchronize()
    out["pcg_us_per_iter"] = e0.elapsed_time(e1) / st.iterations * 1e3
    print(json.dumps(out))


if __name__ == "__main__":
    main()
