"""Print the canonical TET04 continuity pair stream (pairs.cu) detected on
box meshes (development aid: the compile-time Kuhn table in pairs.cu was
generated with this and is checked against the detected stream at run time)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_11541_b200 as P  # noqa: E402

for n in (40, 64):
    ctx = P.AssemblyContext.build(P.generate_box_mesh(P.ElementType.TET04, n, n, n), 8)
    out = torch.empty(3 * ctx.pattern.nnz, dtype=torch.float64, device="cuda")
    ctx.assemble_gradients_d(out)
    r = ctx.groups[0].rows
    pc = r.pair_canon
    cw = pc["words"]
    if pc["kuhn"]:
        print(n, "len", cw.size, "kuhn rows", pc["rows"].numel(), "of", r.n, "generic rows", pc["other"].numel())
    else:
        print(n, "len", cw.size, "canonical slices", pc["cslices"].numel(), "other", pc["oslices"].numel())
    print("words", ",".join(f"0x{int(w):04x}" for w in cw))
