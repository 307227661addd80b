"""Development aid: launch each hot kernel once at its bench size so one
`ncu --set full` pass can capture them all (profiles/r01k_kernels)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_11541_b200 as P  # noqa: E402
from paper_2107_11541_b200 import sparse as S  # noqa: E402

K = P.KernelKind
mesh = P.generate_box_mesh(P.ElementType.TET04, 94, 94, 95)
ctx = P.AssemblyContext.build(mesh, 8)
n, nnz = mesh.nnode, ctx.pattern.nnz
rng = np.random.default_rng(0)
vel = torch.as_tensor(rng.standard_normal((n, 3)), device="cuda")
phi = torch.as_tensor(rng.standard_normal(n), device="cuda")
out1 = torch.empty(n, dtype=torch.float64, device="cuda")
for _ in range(2):  # second pass is the one ncu captures (-s skips the first)
    ctx.assemble_rhs_d(K.SCALAR_RHS, vel, phi, 1.0, 0.0, 1e-2, out1)
    M = ctx.assemble_matrix(K.MASS)
    y = S.spmv_d(M, phi)
    a = torch.randn(16_974_593, dtype=torch.float64, device="cuda")
    b = torch.randn_like(a)
    S.axpy_d(2.5, a, b, torch.empty_like(a))
    S.dot_d(a, b)
torch.cuda.synchronize()
del a, b
hmesh = P.generate_box_mesh(P.ElementType.HEX08, 272, 272, 272)
hctx = P.AssemblyContext.build(hmesh, 8)
hn, hnnz = hmesh.nnode, hctx.pattern.nnz
hvel = torch.as_tensor(rng.standard_normal((hn, 3)), device="cuda")
hr = torch.empty((hn, 3), dtype=torch.float64, device="cuda")
hm = torch.empty(3 * hnnz, dtype=torch.float64, device="cuda")
for _ in range(2):
    hctx.assemble_rhs_d(K.MOMENTUM_RHS, hvel, None, 1.0, 1e-2, 0.0, hr)
    hctx.assemble_gradients_d(hm)
torch.cuda.synchronize()
print("done")
