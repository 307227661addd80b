"""Config-5 NS step on two streams: when does each kernel finish?  Events on
the launching streams, relative to a start event, L2 flushed (development
aid for the co-residency tuning of assemble_ns_d).

    python tools/ns_timeline.py [--n 256] [--reps 10]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_11541_b200 as P  # noqa: E402
from paper_2107_11541_b200 import KernelKind  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    n = args.n
    mesh = P.generate_box_mesh(P.ElementType.TET04, n, n, n)
    ctx = P.AssemblyContext.build(mesh, vector_size=8)
    g = torch.Generator(device="cuda").manual_seed(0)
    vel = torch.randn((mesh.nnode, 3), dtype=torch.float64, device="cuda", generator=g)
    rhs = torch.empty_like(vel)
    mats = torch.empty(3 * ctx.pattern.nnz, dtype=torch.float64, device="cuda")
    flush = torch.empty(128 << 20, dtype=torch.float32, device="cuda")
    main_s = torch.cuda.current_stream()
    side = torch.cuda.Stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    rows = []
    for it in range(args.reps + 3):
        flush.fill_(1.0)
        e0, em, el, eb = ev(), ev(), ev(), ev()
        e0.record()
        side.wait_stream(main_s)
        with torch.cuda.stream(side):
            ctx.assemble_rhs_d(KernelKind.MOMENTUM_RHS, vel, None, 1.0, 1e-2, 0.0, rhs)
            em.record()
        ctx.assemble_gradients_d(mats, window={"kuhn_part": "lines"})
        el.record()
        ctx.assemble_gradients_d(mats, window={"kuhn_part": "surface"})
        eb.record()
        main_s.wait_stream(side)
        torch.cuda.synchronize()
        if it >= 3:
            rows.append((e0.elapsed_time(em), e0.elapsed_time(el), e0.elapsed_time(eb)))
    r = np.median(np.array(rows), axis=0)
    print(f"momentum(+fixup) done {r[0]:.3f} ms, lines done {r[1]:.3f} ms, surface done {r[2]:.3f} ms")
    # each alone
    for name, fn in (("momentum", lambda: ctx.assemble_rhs_d(KernelKind.MOMENTUM_RHS, vel, None, 1.0, 1e-2, 0.0, rhs)),
                     ("lines", lambda: ctx.assemble_gradients_d(mats, window={"kuhn_part": "lines"})),
                     ("surface", lambda: ctx.assemble_gradients_d(mats, window={"kuhn_part": "surface"}))):
        ts = []
        for it in range(args.reps + 3):
            flush.fill_(1.0)
            a, b = ev(), ev()
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            if it >= 3:
                ts.append(a.elapsed_time(b))
        print(f"{name} alone {np.median(ts):.3f} ms")


if __name__ == "__main__":
    main()
