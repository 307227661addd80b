"""Config-4 HEX08 B_x,B_y,B_z: element-once kernels (hexblock.cu) vs per-row kernel
(rowsq.cu), device time with L2 flushed (development aid).

    python tools/hexprobe.py [--n 272] [--reps 10]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_11541_b200 as P  # noqa: E402
from paper_2107_11541_b200 import assembly as A  # noqa: E402


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
    ap.add_argument("--n", type=int, default=272)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--rows", action="store_true", help="also time the per-row kernel")
    ap.add_argument("--canon-rows", type=int, default=0, help="fpb_set_tuning hex_canon_rows (32 | 64)")
    args = ap.parse_args()
    if args.canon_rows:
        from paper_2107_11541_b200 import _lib
        _lib.check(_lib.load().fpb_set_tuning(b"hex_canon_rows", args.canon_rows), "tuning")
    n = args.n
    mesh = P.generate_box_mesh(P.ElementType.HEX08, n, n, n)
    ctx = P.AssemblyContext.build(mesh, 8)
    nnz = ctx.pattern.nnz
    out = torch.empty(3 * nnz, dtype=torch.float64, device="cuda")
    flush = torch.empty(64 << 20, dtype=torch.float64, device="cuda")
    t0 = time.time()
    ctx.assemble_gradients_d(out)
    torch.cuda.synchronize()
    plan = ctx.groups[0].hexrows
    res = {"nelem": mesh.nelem, "nnz": nnz, "plan_s": time.time() - t0, "maxinc": plan.maxinc,
           "canonical_rows": plan.ncanon, "generic_blocks": plan.ngblocks}
    res["once_ms"] = timeit(lambda: ctx.assemble_gradients_d(out), args.reps, flush)
    if args.rows:
        ref = out.clone()
        A.HEX_ONCE = False
        res["rows_ms"] = timeit(lambda: ctx.assemble_gradients_d(out), args.reps, flush)
        A.HEX_ONCE = True
        d = (out - ref).abs().max().item() / ref.abs().max().item()
        res["rel_diff_once_vs_rows"] = d
    print(json.dumps(res))


if __name__ == "__main__":
    main()
