"""Config-4 HEX08 box RHS timings: cell pencils (kmom.cu KIND 2/3) vs element
blocks, L2 flushed (development aid).  python tools/hexbox_probe.py [--n 272]"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_11541_b200 as P  # noqa: E402
import paper_2107_11541_b200.assembly as A  # noqa: E402


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
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    n = args.n
    mesh = P.generate_box_mesh(P.ElementType.HEX08, n, n, n)
    ctx = P.AssemblyContext.build(mesh, 8)
    nn = mesh.nnode
    g = torch.Generator(device="cuda").manual_seed(0)
    vel = torch.randn((nn, 3), dtype=torch.float64, device="cuda", generator=g)
    phi3 = torch.randn((3, nn), dtype=torch.float64, device="cuda", generator=g)
    out = torch.empty((nn, 3), dtype=torch.float64, device="cuda")
    out3 = torch.empty((3, nn), dtype=torch.float64, device="cuda")
    flush = torch.empty(64 << 20, dtype=torch.float64, device="cuda")
    res = {"kchunk": ctx.groups[0].kuhn.kchunk if ctx.groups[0].kuhn else None}
    for label, on in (("pencils", True), ("blocks", False)):
        A.KUHN_MOMENTUM = on
        res[f"{label}/momentum_ms"] = timeit(
            lambda: ctx.assemble_rhs_d(P.KernelKind.MOMENTUM_RHS, vel, None, 1.0, 1e-2, 0.0, out), args.reps, flush)
        res[f"{label}/scalar3_ms"] = timeit(
            lambda: ctx.assemble_scalar_rhs3_d(vel, phi3, (1e-2, 1e-2, 1e-2), out3), args.reps, flush)
    A.KUHN_MOMENTUM = True
    print(json.dumps(res))


if __name__ == "__main__":
    main()
