"""Development aid: BiCGSTAB / PCG / SpMV per-iteration time on the config-5 mesh (256^3 tets) on one GPU."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_11541_b200 as P  # noqa: E402
from paper_2107_11541_b200 import sparse as S  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
mesh = P.generate_box_mesh(P.ElementType.TET04, n, n, n)
ctx = P.AssemblyContext.build(mesh, 8)
nn, nnz = mesh.nnode, ctx.pattern.nnz
vel = torch.as_tensor(np.random.default_rng(0).standard_normal((nn, 3)), device="cuda")
M = ctx.assemble_matrix(P.KernelKind.MASS)
C = ctx.assemble_matrix(P.KernelKind.CONVECTION, velocity=vel)
L = ctx.assemble_matrix(P.KernelKind.LAPLACIAN)
A = M.with_vals(M.vals_d + 0.05 * (C.vals_d + 1e-2 * L.vals_d))
b = torch.as_tensor(np.random.default_rng(1).standard_normal(nn), device="cuda")
out = {}
for name, fn in (("bicgstab", lambda it: P.bicgstab_solve(A, b, tol=0.0, max_iter=it)),
                 ("pcg_mass", lambda it: P.pcg_solve(M, b, tol=0.0, max_iter=it))):
    fn(40)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    x, st = fn(40)
    e1.record()
    torch.cuda.synchronize()
    out[name] = round(e0.elapsed_time(e1) / max(st.iterations, 1), 4)
y = torch.empty_like(b)
S.spmv_d(A, b, y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    S.spmv_d(A, b, y)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
out["spmv_ms"] = round(ms, 4)
out["spmv_frac_hbm"] = round((12 * nnz + 4 * (nn + 1) + 16 * nn) / ms / 1e6 / 6549.4, 3)
print(json.dumps(out))
