import sys, os
sys.path.insert(0, os.getcwd())
import torch, paper_2107_11541_b200 as P
mesh = P.generate_box_mesh(P.ElementType.TET04, 94, 94, 95)
ctx = P.AssemblyContext.build(mesh, 8)
mats = torch.empty(3 * ctx.pattern.nnz, dtype=torch.float64, device="cuda")
for _ in range(2): ctx.assemble_gradients_d(mats)
torch.cuda.synchronize()
