"""Time the pieces of the e2e step (development aid)."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_11541_b200 as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
mesh = P.generate_box_mesh(P.ElementType.TET04, n, n, n)
ctx = P.AssemblyContext.build(mesh, 8)
vel_h = torch.empty((mesh.nnode, 3), dtype=torch.float64, pin_memory=True).numpy()
vel_h[:] = np.random.default_rng(0).standard_normal((mesh.nnode, 3))
def t(f, label):
    torch.cuda.synchronize(); t0 = time.perf_counter(); r = f(); torch.cuda.synchronize()
    print(f"{label}: {1e3*(time.perf_counter()-t0):.1f} ms", flush=True); return r
for rep in range(3):
    r = t(lambda: ctx.assemble_rhs(P.KernelKind.MOMENTUM_RHS, "packed", vel_h, None, 1.0, 1e-2, 0.0), "assemble_rhs")
    g = t(lambda: P.gradient_matrices(ctx), "gradient_matrices")
    v = t(lambda: [B.vals for B in g], ".vals x3")
    t(lambda: [B.vals_d.cpu() for B in g], ".vals_d.cpu() x3 (pageable)")
    from paper_2107_11541_b200.sparse import to_host
    t(lambda: [to_host(B.vals_d) for B in g], "to_host x3 (pinned)")
    del r, g, v
