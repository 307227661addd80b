"""Development aid: the round-1 solver / fused-scalar kernels once each at
their bench sizes for one `ncu --set full` pass (profiles/r01t_kernels):
SELL SpMV (config-2 MASS, 16-bit columns; config-5 MASS, int32 columns),
the fused PCG SpMV on the pinned config-2 LAPLACIAN, the fused three-scalar
RHS (config 3) and the hex momentum / scalar RHS (config 4)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_11541_b200 as P  # noqa: E402
from paper_2107_11541_b200 import sparse as S  # noqa: E402

K = P.KernelKind
rng = np.random.default_rng(0)
mesh = P.generate_box_mesh(P.ElementType.TET04, 94, 94, 95)
ctx = P.AssemblyContext.build(mesh, 8)
n = mesh.nnode
vel = torch.as_tensor(rng.standard_normal((n, 3)), device="cuda")
phi3 = torch.as_tensor(rng.standard_normal((3, n)), device="cuda")
out3 = torch.empty((3, n), dtype=torch.float64, device="cuda")
M = ctx.assemble_matrix(K.MASS)
L = ctx.assemble_matrix(K.LAPLACIAN)
x = torch.as_tensor(rng.standard_normal(n), device="cuda")
for _ in range(2):
    ctx.assemble_scalar_rhs3_d(vel, phi3, (1e-2, 1e-2, 1e-2), out3)
    S.spmv_d(M, x)
P.pcg_solve(M, x, tol=0.0, max_iter=2)
torch.cuda.synchronize()
del ctx
big = P.generate_box_mesh(P.ElementType.TET04, 256, 256, 256)
bctx = P.AssemblyContext.build(big, 8)
BM = bctx.assemble_matrix(K.MASS)
bx = torch.as_tensor(rng.standard_normal(big.nnode), device="cuda")
for _ in range(2):
    S.spmv_d(BM, bx)
torch.cuda.synchronize()
del bctx, BM
hmesh = P.generate_box_mesh(P.ElementType.HEX08, 272, 272, 272)
hctx = P.AssemblyContext.build(hmesh, 8)
hn = hmesh.nnode
hvel = torch.as_tensor(rng.standard_normal((hn, 3)), device="cuda")
hphi3 = torch.as_tensor(rng.standard_normal((3, hn)), device="cuda")
hr = torch.empty((hn, 3), dtype=torch.float64, device="cuda")
hs = torch.empty((3, hn), dtype=torch.float64, device="cuda")
for _ in range(2):
    hctx.assemble_rhs_d(K.MOMENTUM_RHS, hvel, None, 1.0, 1e-2, 0.0, hr)
    hctx.assemble_scalar_rhs3_d(hvel, hphi3, (1e-2, 1e-2, 1e-2), hs)
torch.cuda.synchronize()
