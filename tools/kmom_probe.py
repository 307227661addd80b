"""Momentum RHS timings: Kuhn cell-line kernel (kmom.cu) vs element blocks
(blocks.cu) on the config-2 and config-5 meshes, L2 flushed between reps.

    python tools/kmom_probe.py [--sizes 94x94x95,256x256x256] [--reps 10]
"""
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
    ap.add_argument("--sizes", default="94x94x95,256x256x256")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--kchunks", default="0")
    ap.add_argument("--blocks", type=int, default=1)
    ap.add_argument("--grad", type=int, default=0, help="also time B_x,B_y,B_z (Kuhn box vs colind path)")
    ap.add_argument("--s3", type=int, default=0, help="also time the three-scalar RHS (Kuhn vs element blocks)")
    ap.add_argument("--overlap", default="", help="kmom_smem_kb values: time momentum + B_xyz sequential vs on two streams")
    ap.add_argument("--tune", default="", help="name=value[,name=value] passed to fpb_set_tuning")
    args = ap.parse_args()
    from paper_2107_11541_b200 import _lib
    for kv in filter(None, args.tune.split(",")):
        name, val = kv.split("=")
        _lib.check(_lib.load().fpb_set_tuning(name.encode(), int(val)))
    flush = torch.empty(128 << 20, dtype=torch.float32, device="cuda")
    res = {}
    for sz in args.sizes.split(","):
        nx, ny, nz = (int(v) for v in sz.split("x"))
        mesh = P.generate_box_mesh(P.ElementType.TET04, nx, ny, nz)
        n, ne = mesh.nnode, mesh.nelem
        g = torch.Generator(device="cuda").manual_seed(0)
        vel = torch.randn((n, 3), dtype=torch.float64, device="cuda", generator=g)
        out = torch.empty((n, 3), dtype=torch.float64, device="cuda")
        ref = torch.empty_like(out)
        for kc in (int(v) for v in args.kchunks.split(",")):
            A.KUHN_KCHUNK = kc
            ctx = P.AssemblyContext.build(mesh, vector_size=8)
            kb = ctx.groups[0].kuhn
            fn = lambda: ctx.assemble_rhs_d(P.KernelKind.MOMENTUM_RHS, vel, None, 1.0, 1e-2, 0.0, out)  # noqa: E731
            ms = timeit(fn, args.reps, flush)
            res[f"{sz}/kuhn/kchunk{kb.kchunk if kb else None}"] = {"ms": round(ms, 4), "Gelem_s": round(ne / ms / 1e6, 2)}
            if args.blocks:
                A.KUHN_MOMENTUM = False
                ctx.assemble_rhs_d(P.KernelKind.MOMENTUM_RHS, vel, None, 1.0, 1e-2, 0.0, ref)
                msb = timeit(lambda: ctx.assemble_rhs_d(P.KernelKind.MOMENTUM_RHS, vel, None, 1.0, 1e-2, 0.0, ref),
                             args.reps, flush)
                A.KUHN_MOMENTUM = True
                fn()
                torch.cuda.synchronize()
                d = float((out - ref).abs().max() / ref.abs().max())
                res[f"{sz}/blocks"] = {"ms": round(msb, 4), "Gelem_s": round(ne / msb / 1e6, 2), "rel_diff": d}
            if args.grad:
                nnz = ctx.pattern.nnz
                ga = torch.empty(3 * nnz, dtype=torch.float64, device="cuda")
                gb = torch.empty_like(ga)
                msg = timeit(lambda: ctx.assemble_gradients_d(ga), args.reps, flush)
                A.KUHN_BOX_GRADIENT = False
                msc = timeit(lambda: ctx.assemble_gradients_d(gb), args.reps, flush)
                A.KUHN_BOX_GRADIENT = True
                res[f"{sz}/grad_box"] = {"ms": round(msg, 4), "Gelem_s": round(ne / msg / 1e6, 2),
                                         "bitwise_equal": bool(torch.equal(ga, gb))}
                res[f"{sz}/grad_colind"] = {"ms": round(msc, 4), "Gelem_s": round(ne / msc / 1e6, 2)}
                del ga, gb
            if args.s3:
                phi3 = torch.randn((3, n), dtype=torch.float64, device="cuda", generator=g)
                o3 = torch.empty((3, n), dtype=torch.float64, device="cuda")
                r3 = torch.empty_like(o3)
                f3 = lambda: ctx.assemble_scalar_rhs3_d(vel, phi3, (1e-2, 1e-2, 1e-2), o3)  # noqa: E731
                ms3 = timeit(f3, args.reps, flush)
                A.KUHN_MOMENTUM = False
                msb3 = timeit(lambda: ctx.assemble_scalar_rhs3_d(vel, phi3, (1e-2, 1e-2, 1e-2), r3), args.reps, flush)
                A.KUHN_MOMENTUM = True
                f3()
                torch.cuda.synchronize()
                res[f"{sz}/s3_kuhn"] = {"ms": round(ms3, 4), "rel_diff": float((o3 - r3).abs().max() / r3.abs().max())}
                res[f"{sz}/s3_blocks"] = {"ms": round(msb3, 4)}
                del phi3, o3, r3
            if args.overlap:
                from paper_2107_11541_b200 import _lib
                nnz = ctx.pattern.nnz
                ga = torch.empty(3 * nnz, dtype=torch.float64, device="cuda")
                side = torch.cuda.Stream()
                main = torch.cuda.current_stream()

                def seq():
                    ctx.assemble_rhs_d(P.KernelKind.MOMENTUM_RHS, vel, None, 1.0, 1e-2, 0.0, out)
                    ctx.assemble_gradients_d(ga)

                def par():
                    side.wait_stream(main)
                    with torch.cuda.stream(side):
                        ctx.assemble_gradients_d(ga)
                    ctx.assemble_rhs_d(P.KernelKind.MOMENTUM_RHS, vel, None, 1.0, 1e-2, 0.0, out)
                    main.wait_stream(side)

                def par2():  # gradients first, momentum on the side stream
                    side.wait_stream(main)
                    with torch.cuda.stream(side):
                        ctx.assemble_rhs_d(P.KernelKind.MOMENTUM_RHS, vel, None, 1.0, 1e-2, 0.0, out)
                    ctx.assemble_gradients_d(ga)
                    main.wait_stream(side)

                for kbv in (int(v) for v in args.overlap.split(",")):
                    _lib.check(_lib.load().fpb_set_tuning(b"kmom_smem_kb", kbv))
                    res[f"{sz}/seq/smem{kbv}"] = {"ms": round(timeit(seq, args.reps, flush), 4)}
                    res[f"{sz}/par_grad_side/smem{kbv}"] = {"ms": round(timeit(par, args.reps, flush), 4)}
                    res[f"{sz}/par_mom_side/smem{kbv}"] = {"ms": round(timeit(par2, args.reps, flush), 4)}
                _lib.check(_lib.load().fpb_set_tuning(b"kmom_smem_kb", 0))
                del ga
            del ctx
            torch.cuda.empty_cache()
        del mesh, vel, out, ref
        torch.cuda.empty_cache()
    for k, v in res.items():
        print(k, json.dumps(v))


if __name__ == "__main__":
    main()
