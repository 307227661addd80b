"""Per-kernel device timings on the config-2 mesh (development aid).

    python tools/kbench.py [--nx 94 --ny 94 --nz 95] [--reps 20]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_11541_b200 as P  # noqa: E402


def timeit(fn, reps, flush):
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nx", type=int, default=94)
    ap.add_argument("--ny", type=int, default=94)
    ap.add_argument("--nz", type=int, default=95)
    ap.add_argument("--etype", default="TET04")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--scatters", default="auto,rows,atomic")
    ap.add_argument("--tune", default="", help="name=value[,name=value] passed to fpb_set_tuning")
    args = ap.parse_args()
    from paper_2107_11541_b200 import _lib
    for kv in filter(None, args.tune.split(",")):
        name, val = kv.split("=")
        _lib.check(_lib.load().fpb_set_tuning(name.encode(), int(val)))
    et = P.ElementType[args.etype]
    mesh = P.generate_box_mesh(et, args.nx, args.ny, args.nz)
    n, ne = mesh.nnode, mesh.nelem
    rng = np.random.default_rng(0)
    vel = torch.as_tensor(rng.standard_normal((n, mesh.dim)), device="cuda")
    phi = torch.as_tensor(rng.standard_normal(n), device="cuda")
    flush = torch.empty(128 << 20, dtype=torch.float32, device="cuda")
    res = {"nelem": ne, "nnode": n}
    for sc in args.scatters.split(","):
        ctx = P.AssemblyContext.build(mesh, 8, scatter=sc)
        ctx.refresh_geometry("packed", need_grad=False)
        nnz = ctx.pattern.nnz
        rhs3 = torch.empty((n, mesh.dim), dtype=torch.float64, device="cuda")
        rhs1 = torch.empty(n, dtype=torch.float64, device="cuda")
        mat = torch.empty(nnz, dtype=torch.float64, device="cuda")
        mats = torch.empty(mesh.dim * nnz, dtype=torch.float64, device="cuda")
        K = P.KernelKind
        cases = {
            "momentum_rhs": lambda: ctx.assemble_rhs_d(K.MOMENTUM_RHS, vel, None, 1.0, 1e-2, 0.0, rhs3),
            "scalar_rhs": lambda: ctx.assemble_rhs_d(K.SCALAR_RHS, vel, phi, 1.0, 0.0, 1e-2, rhs1),
            "gradient_xyz": lambda: ctx.assemble_gradients_d(mats),
            "mass": lambda: ctx.assemble_matrix_d(K.MASS, None, mat),
            "laplacian": lambda: ctx.assemble_matrix_d(K.LAPLACIAN, None, mat),
            "convection": lambda: ctx.assemble_matrix_d(K.CONVECTION, vel, mat),
        }
        for name, fn in cases.items():
            ms = timeit(fn, args.reps, flush)
            res[f"{sc}/{name}"] = {"ms": round(ms, 4), "Gelem_s": round(ne / ms / 1e6, 2)}
        del ctx
        torch.cuda.empty_cache()
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
