cat > /tmp/pp.py <<'PY'
import sys, json, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2107_11541_b200 as P
from paper_2107_11541_b200 import assembly
mesh = P.generate_box_mesh(P.ElementType.TET04, 94, 94, 95)
ctx = P.AssemblyContext.build(mesh, 8)
nnz = ctx.pattern.nnz
mats = torch.empty(3 * nnz, dtype=torch.float64, device="cuda")
ref = torch.empty_like(mats)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
def timeit(fn, reps=20):
    for _ in range(3): fn()
    ts = []
    for _ in range(reps):
        flush.fill_(1); a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return float(np.median(ts))
assembly.GRADIENT_PAIRS = False
t_nb = timeit(lambda: ctx.assemble_gradients_d(ref))
assembly.GRADIENT_PAIRS = True
t_p = timeit(lambda: ctx.assemble_gradients_d(mats))
d = (mats - ref).abs().max().item() / ref.abs().max().item()
print(json.dumps({"rows_nb_ms": t_nb, "pairs_ms": t_p, "max_rel_diff": d}))
PY
for v in "" build_variants/*/libfempack_b200.so; do echo "== $v"; FPB_LIB_PATH=$v timeout 600 python /tmp/pp.py 2>&1 | tail -1; done
