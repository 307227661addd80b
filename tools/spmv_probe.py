"""SpMV formats on the bench meshes (development aid).

    python tools/spmv_probe.py [--reps 20]

CSR kernel (fpb_spmv, lanes per row) vs the SELL-32 copy (fpb_spmv_sell,
thread per row) on MASS matrices of the config-2 (TET04 94x94x95),
config-5 (TET04 256^3) and config-4 (HEX08 272^3) meshes; median of reps,
L2 flushed; GB/s over the algorithmic bytes 12 nnz + 20 n.
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
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--meshes", default="TET04:94:94:95,TET04:256:256:256,HEX08:272:272:272")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))["hbm_gbs"]

    def timeit(fn):
        for _ in range(3):
            fn()
        ts = []
        for _ in range(args.reps):
            flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return float(np.median(ts))

    out = {}
    for spec in args.meshes.split(","):
        et, nx, ny, nz = spec.split(":")
        mesh = P.generate_box_mesh(getattr(P.ElementType, et), int(nx), int(ny), int(nz))
        ctx = P.AssemblyContext.build(mesh, vector_size=8)
        A = ctx.assemble_matrix(P.KernelKind.MASS, "packed")
        n, nnz = A.n, A.nnz
        x = torch.as_tensor(np.random.default_rng(0).standard_normal(n), device=dev)
        y1 = torch.empty(n, dtype=torch.float64, device=dev)
        y2 = torch.empty_like(y1)
        torch.cuda.synchronize()
        sc = sparse.SellCopy(A)
        byt = 12 * nnz + 20 * n
        t_csr = timeit(lambda: _lib.call("fpb_spmv", n, nnz, A.rowptr_d.data_ptr(), A.colind_d.data_ptr(),
                                         A.vals_d.data_ptr(), x.data_ptr(), y1.data_ptr(), _lib.stream()))
        t_sell = timeit(lambda: sc.spmv_d(x, y2))
        t_build = timeit(lambda: sparse.SellCopy(A))
        torch.cuda.synchronize()
        rel = float((y1 - y2).abs().max() / y1.abs().max())
        out[spec] = {"n": n, "nnz": nnz, "padded": sc.total, "csr_ms": t_csr, "sell_ms": t_sell,
                     "csr_frac": byt / (t_csr * 1e-3) / 1e9 / peak, "sell_frac": byt / (t_sell * 1e-3) / 1e9 / peak,
                     "sell_build_ms": t_build, "max_rel_diff": rel}
        print(spec, json.dumps(out[spec]), flush=True)
        del ctx, A, sc, mesh
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
