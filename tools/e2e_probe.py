"""Where does the end-to-end (host-buffer) step time go? (development aid)"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_11541_b200 as P  # noqa: E402
from paper_2107_11541_b200.sparse import to_host  # noqa: E402


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    return round(float(np.median(ts)), 3)


mesh = P.generate_box_mesh(P.ElementType.TET04, 94, 94, 95)
ctx = P.AssemblyContext.build(mesh, 8)
n, nnz = mesh.nnode, ctx.pattern.nnz
vel = np.random.default_rng(0).standard_normal((n, 3))
dvel = torch.as_tensor(vel, device="cuda")
big = torch.empty(nnz, dtype=torch.float64, device="cuda")
pin = torch.empty(nnz, dtype=torch.float64, pin_memory=True)
res = {
    "h2d_vel_pageable": t(lambda: torch.from_numpy(vel).to("cuda")),
    "h2d_vel_pinned_copy": t(lambda: torch.from_numpy(vel).pin_memory().to("cuda", non_blocking=True)),
    "d2h_102MB_pageable": t(lambda: big.cpu()),
    "d2h_102MB_to_host": t(lambda: to_host(big)),
    "d2h_102MB_prepinned": t(lambda: pin.copy_(big, non_blocking=True)),
    "pinned_alloc_102MB": t(lambda: torch.empty(nnz, dtype=torch.float64, pin_memory=True)),
    "rhs_api": t(lambda: ctx.assemble_rhs(P.KernelKind.MOMENTUM_RHS, "packed", vel, None, 1.0, 1e-2, 0.0)),
    "grad_api_nohost": t(lambda: P.gradient_matrices(ctx)),
    "grad_api_vals": t(lambda: [B.vals for B in P.gradient_matrices(ctx)]),
}
print(res)
