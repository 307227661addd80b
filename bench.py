"""Headline bench: assembled elements/s for BASELINE.json config 2 —
NS momentum RHS + continuity (B_x, B_y, B_z) assembly on the 5,036,520-tet
box mesh (94 x 94 x 95 cells, unit cube), SIMD-packed layout, one B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

One step = MOMENTUM_RHS (rho=1, mu=1e-2, velocity
= default_rng(0).standard_normal((nnode, 3)), bench.py:196-207 of the
reference) and the fused gradient/continuity matrices B_k over every element.
`value` = elements assembled per second (each element contributes its
momentum block and all three B_k blocks) with inputs resident in HBM, timed
with CUDA events per step, L2 flushed (512 MiB write) between steps.
`e2e` = the same step through the public API with host (numpy) inputs and
outputs: velocity H2D in, RHS + three matrices' values D2H out.

Multi-GPU (torchrun, N > 1): weak scaling — rank r assembles z-slab r of an
(94, 94, 95 N) mesh; interface-plane RHS/matrix contributions are summed by
an NCCL halo exchange that runs on a side stream while the interior rows are
assembled (interface windows first, paper_2107_11541_b200/distributed.py).

`--impl reference`: the reference's CPU algorithm (C restatement of the
packed kernels, oracle/fempack_ref.c, all host threads) on a bounded sample of
the same workload; prints the same JSON line with "impl": "reference".
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "assembled elements/s (Melem/s) & FP64/HBM roofline fraction at 1/2/4/8 B200"
UNIT = "Melem/s"
# measured DFMA rate on this pool's B200 (tools/microbench/peaks.cu,
# profiles/r01_microbench.txt); MEASURED_PEAKS.json carries no FP64 figure
FP64_PEAK_TFLOPS = 34.1
HBM_FALLBACK_GBS = 6650.0
# SURVEY 8(d) algorithmic work per TET04 element (flops, compulsory bytes)
WORK = {"momentum_rhs": (1492.0, 28.0), "gradient_xyz": (676.0, 145.0)}
# SURVEY 8(d) per-element work for the config-3 / config-4 kernels: F =
# G_min + K + S (instrumented reference flop counts), B = compulsory HBM
# bytes (int32 conn, f64 node data at rho_n = nnode/nelem, CSR values at
# rho_z = nnz/nelem plus the int32 element->CSR map for matrices).  TET04
# values are SURVEY's (config-2 mesh); HEX08 F from SURVEY's bounds at
# 37.2 TF/s nominal, B from the same formula at config 4 (rho_n 1.011,
# rho_z 27.10).
WORK_C = {
    ("TET04", "scalar_rhs"): (592.0, 27.0),
    ("HEX08", "momentum_rhs"): (7328.0, 105.0),
    ("HEX08", "scalar_rhs"): (4248.0, 97.0),
    ("HEX08", "gradient_xyz"): (6169.0, 962.0),
}
L2_FLUSH_BYTES = 512 << 20


def hbm_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def _roof(F, B, ms, nelem, hbm):
    """Roofline of one kernel at F flops / B bytes per element."""
    t = ms / 1e3
    fl, by = F * nelem / t / 1e12, B * nelem / t / 1e9
    if F / B > FP64_PEAK_TFLOPS * 1e3 / hbm:
        return {"bound": "fp64", "achieved": fl, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": fl / FP64_PEAK_TFLOPS}
    return {"bound": "hbm", "achieved": by, "peak": hbm, "unit": "GB/s", "frac": by / hbm}


def _time_ms(fn, reps, flush):
    import torch

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
    return statistics.median(ts)


def config3_block(ctx, vel, flush, hbm, reps=10):
    """Config 3: scalar transport (enthalpy + 2 species) on the config-2 mesh;
    the solver vector ops are in the "solver" block."""
    import torch

    import paper_2107_11541_b200 as P

    n, ne = ctx.mesh.nnode, ctx.mesh.nelem
    rng = np.random.default_rng(0)
    rng.standard_normal((n, 3))
    phi3 = torch.as_tensor(np.stack([rng.standard_normal(n) for _ in range(3)]), device=vel.device)
    out3 = torch.empty((3, n), dtype=torch.float64, device=vel.device)
    kap = (1e-2, 1e-2, 1e-2)  # kappa, D, D (timeloop.py:76-79)

    def fused():  # one element-block pass for the three fields (fpb_assemble_blocks_scalar3)
        ctx.assemble_scalar_rhs3_d(vel, phi3, kap, out3)

    def three():
        for f in range(3):
            ctx.assemble_rhs_d(P.KernelKind.SCALAR_RHS, vel, phi3[f], 1.0, 0.0, kap[f], out3[f])

    ms = _time_ms(fused, reps, flush)
    ms_three = _time_ms(three, reps, flush)
    F, B = WORK_C[("TET04", "scalar_rhs")]
    return {"workload": "config 3: TET04 94x94x95, SCALAR_RHS x3 (heat kappa, 2 species D), velocity + scalars "
                        "default_rng(0) draws; one fused element-block pass", "elements": ne, "ms_per_step": ms,
            "ms_three_separate_passes": ms_three,
            "value": 3 * ne / (ms / 1e3) / 1e6, "unit": "Melem/s (element-scalar assemblies)",
            "roofline": dict(_roof(F, B, ms / 3, ne, hbm), kernel="scalar_rhs3 (fused)",
                             work_per_element={"flops": F, "bytes": B},
                             note="F is the reference's per-element work for ONE scalar (geometry included); "
                                  "the fused pass shares geometry, velocity moments and node staging across the "
                                  "three fields, so this reference-flop rate can exceed the FP64 peak")}


def config4_block(flush, hbm, n=272, reps=5):
    """Config 4: 20,123,648-element HEX08 (Q1, 8 Gauss points) box, full NS +
    scalar assembly: momentum RHS, continuity B_x,B_y,B_z and three scalar
    RHS per step."""
    import torch

    import paper_2107_11541_b200 as P

    mesh = P.generate_box_mesh(P.ElementType.HEX08, n, n, n)
    ctx = P.AssemblyContext.build(mesh, vector_size=8)
    ctx.refresh_geometry("packed", need_grad=False)
    nn_, ne, nnz = mesh.nnode, mesh.nelem, ctx.pattern.nnz
    dev = flush.device
    rng = np.random.default_rng(0)
    vel = torch.as_tensor(rng.standard_normal((nn_, 3)), device=dev)
    phi3 = torch.as_tensor(np.stack([rng.standard_normal(nn_) for _ in range(3)]), device=dev)
    rhs = torch.empty((nn_, 3), dtype=torch.float64, device=dev)
    srhs3 = torch.empty((3, nn_), dtype=torch.float64, device=dev)
    mats = torch.empty(3 * nnz, dtype=torch.float64, device=dev)
    K = P.KernelKind
    parts = {
        "momentum_rhs": lambda: ctx.assemble_rhs_d(K.MOMENTUM_RHS, vel, None, 1.0, 1e-2, 0.0, rhs),
        "gradient_xyz": lambda: ctx.assemble_gradients_d(mats),
        # the three scalars in one fused element-block pass
        "scalar_rhs": lambda: ctx.assemble_scalar_rhs3_d(vel, phi3, (1e-2, 1e-2, 1e-2), srhs3),
    }
    ms = {k: _time_ms(f, reps, flush) for k, f in parts.items()}
    roof = {}
    for k, t in ms.items():
        F, B = WORK_C[("HEX08", k)]
        per = t / (3 if k == "scalar_rhs" else 1)
        roof[k] = dict(_roof(F, B, per, ne, hbm), ms=per)
    roof["scalar_rhs"]["note"] = ("per scalar of the fused three-field pass (shared staging); F is the "
                                  "reference's one-scalar work")
    total = sum(ms.values())
    del ctx, mats
    torch.cuda.empty_cache()
    return {"workload": f"config 4: HEX08 box {n}^3 ({ne} elements, {nn_} nodes, nnz {nnz}), momentum RHS + "
                        "B_x,B_y,B_z + 3 scalar RHS", "elements": ne, "ms_per_step": total,
            "value": ne / (total / 1e3) / 1e6, "unit": "Melem/s", "kernels": roof}


def dist_bicgstab_block(sub, vel, dev, dist, iters=60):
    """Config 5's solver leg at N > 1: Jacobi-BiCGSTAB on the slab-decomposed
    advection-diffusion operator M + dt (C(u) + kappa L) — per iteration the
    fused device kernels with owned-row reductions, four 2-double NCCL
    allreduces and two ghost-plane exchanges.  A fixed iteration count
    (tol 0) is timed with CUDA events between barriers, max over ranks."""
    import torch

    import paper_2107_11541_b200 as P
    from paper_2107_11541_b200.distributed import bicgstab_slab

    ctx = sub.ctx
    nnz = ctx.pattern.nnz
    mats = []
    for kind, v in ((P.KernelKind.MASS, None), (P.KernelKind.CONVECTION, vel), (P.KernelKind.LAPLACIAN, None)):
        m = torch.empty(nnz, dtype=torch.float64, device=dev)
        ctx.assemble_matrix_d(kind, v, m)
        sub.halo_sum_matrix(m)
        mats.append(m)
    A = ctx.pattern.with_vals(mats[0] + 0.05 * (mats[1] + 1e-2 * mats[2]))
    L = sub.layout
    nglob = (L.nx + 1) * (L.ny + 1) * (L.nz + 1)
    b = torch.as_tensor(np.random.default_rng(1).standard_normal(nglob)[L.node_offset:L.node_offset + L.nnode],
                        device=dev)
    bicgstab_slab(L, A, b, tol=0.0, max_iter=8, check_every=8)  # warm
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    x, st = bicgstab_slab(L, A, b, tol=0.0, max_iter=iters, check_every=iters)
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    return {"workload": "slab BiCGSTAB on M + 0.05 (C(u) + 1e-2 L), local 94x94x95 cells per GPU",
            "iterations": st.iterations, "ms": ms, "ms_per_iter": ms / max(st.iterations, 1),
            "rows_per_rank": L.owned_rows[1] - L.owned_rows[0], "relres": st.residual_history[-1]}


def config5_block(flush, hbm, n=256, reps=5, iters=40):
    """Config 5's mesh (100,663,296 tets, 256^3 cells) on ONE B200: the
    headline step (momentum RHS + B_x,B_y,B_z) and Jacobi-BiCGSTAB iterations
    on M + 0.05 (C(u) + 1e-2 L) — the single-GPU reference point of the
    2/4/8-GPU decomposition."""
    import torch

    import paper_2107_11541_b200 as P

    t0 = time.perf_counter()
    mesh = P.generate_box_mesh(P.ElementType.TET04, n, n, n)
    ctx = P.AssemblyContext.build(mesh, vector_size=8)
    ctx.refresh_geometry("packed", need_grad=False)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    nn_, ne, nnz = mesh.nnode, mesh.nelem, ctx.pattern.nnz
    dev = flush.device
    vel = torch.as_tensor(np.random.default_rng(0).standard_normal((nn_, 3)), device=dev)
    rhs = torch.empty((nn_, 3), dtype=torch.float64, device=dev)
    mats = torch.empty(3 * nnz, dtype=torch.float64, device=dev)
    K = P.KernelKind
    ms_mom = _time_ms(lambda: ctx.assemble_rhs_d(K.MOMENTUM_RHS, vel, None, 1.0, 1e-2, 0.0, rhs), reps, flush)
    ms_grad = _time_ms(lambda: ctx.assemble_gradients_d(mats), reps, flush)
    del mats
    M = ctx.assemble_matrix(K.MASS)
    C = ctx.assemble_matrix(K.CONVECTION, velocity=vel)
    L = ctx.assemble_matrix(K.LAPLACIAN)
    A = M.with_vals(M.vals_d + 0.05 * (C.vals_d + 1e-2 * L.vals_d))
    del C, L
    b = torch.as_tensor(np.random.default_rng(1).standard_normal(nn_), device=dev)
    P.bicgstab_solve(A, b, tol=0.0, max_iter=iters)  # warm: same workspace + batch graph as the timed solve
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    x, st = P.bicgstab_solve(A, b, tol=0.0, max_iter=iters)
    e1.record()
    torch.cuda.synchronize()
    ms_bicg = e0.elapsed_time(e1)
    F, B = WORK["gradient_xyz"]
    out = {"workload": f"config 5 mesh on one GPU: TET04 box {n}^3 ({ne} elements, {nn_} nodes, nnz {nnz})",
           "setup_s": setup_s, "ms_per_step": ms_mom + ms_grad, "value": ne / ((ms_mom + ms_grad) / 1e3) / 1e6,
           "unit": UNIT, "kernels_ms": {"momentum_rhs": ms_mom, "gradient_xyz": ms_grad},
           "gradient_roofline": _roof(F, B, ms_grad, ne, hbm),
           "bicgstab": {"iterations": st.iterations, "ms_per_iter": ms_bicg / max(st.iterations, 1),
                        "GB_s_equiv": (2 * (12 * nnz + 4 * (nn_ + 1) + 8 * nn_) + 23 * 8 * nn_) * st.iterations
                        / ms_bicg / 1e6}}
    del ctx, A, M
    torch.cuda.empty_cache()
    return out


def flow_block(nx, ny, nz, steps=2):
    """FlowSolver.step on the device on the config-2
    mesh: a Table-1-style profile — CUDA-event time per (category, equation)
    of a full fractional step (3 RK3 stages of momentum + 3 scalar RHS,
    pressure Poisson PCG on the pinned B^T M_L^-1 B operator, correction)."""
    import torch

    import paper_2107_11541_b200 as P
    from paper_2107_11541_b200.timeloop import DeviceState

    mesh = P.generate_box_mesh(P.ElementType.TET04, nx, ny, nz)
    t0 = time.perf_counter()
    solver = P.FlowSolver(mesh, P.TimeConfig(dt=5e-4, tol=1e-8), robin_alpha=1.0, robin_beta=0.1)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    x, y, z = (solver.mesh.coords_d[:, k] for k in range(3))
    pi = np.pi
    vel = torch.stack([torch.sin(pi * x) * torch.cos(pi * y), -torch.cos(pi * x) * torch.sin(pi * y),
                       0.1 * torch.sin(pi * z)], dim=1).contiguous()
    n = mesh.nnode
    zeros = torch.zeros(n, dtype=torch.float64, device=vel.device)
    st = DeviceState(vel, zeros.clone(), (torch.cos(pi * x) * torch.cos(pi * z)).contiguous(),
                     torch.stack([x * y, z * (1.0 - z)]).contiguous(), 1.0, 1e-2, 1e-2, 1e-2)
    st, _ = solver.step_d(st)  # warm (graph capture, workspaces)
    cells: dict = {}
    its, ms = [], []
    for _ in range(steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        st, diag = solver.step_d(st)
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
        its.append(diag.solver.iterations)
        for k, v in diag.timings.items():
            cells[" / ".join(k)] = cells.get(" / ".join(k), 0.0) + v * 1e3 / steps
    return {"workload": f"FlowSolver.step, TET04 box {nx}x{ny}x{nz} ({mesh.nelem} elements, {n} nodes), "
                        "Robin alpha 1 beta 0.1, dt 5e-4, PCG tol 1e-8", "setup_s": setup_s,
            "ms_per_step": statistics.mean(ms), "pcg_iterations": its, "ms_by_cell": cells,
            "pressure_operator_nnz": solver.laplacian.nnz}


def cpu_baseline(nx, ny, nz_sample, steps=30, warmup=2):
    from oracle import cport
    from oracle.baseline import CpuWorkload

    threads = cport.max_threads()
    wl = CpuWorkload(nx, ny, nz_sample, nthreads=threads)
    ts = wl.time_steps(steps, warmup)
    t = statistics.median(ts)
    whole = "the whole config-2 mesh" if nz_sample == 95 else "a slab of the config-2 mesh"
    return {"value": wl.nelem / t / 1e6, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"TET04 {nx}x{ny}x{nz_sample} box, {whole} ({wl.nelem} elements), momentum RHS + "
                      f"3x CONVECTION(e_k) + scatters, reference packed kernels (oracle/fempack_ref.c, vs=8, "
                      f"geometry cached as in the reference bench), median of {steps} steps "
                      f"({sum(ts):.1f} s of timed CPU work)"}


def run_reference(args, rank, world):
    """--impl reference: reference CPU algorithm on the host cores (rank 0)."""
    if rank != 0:
        return
    from oracle import cport
    from oracle.baseline import CpuWorkload

    threads = cport.max_threads()
    wl = CpuWorkload(args.nx, args.ny, args.cpu_nz, nthreads=threads)
    ts = wl.time_steps(args.steps, args.warmup)
    t = statistics.mean(ts)
    value = wl.nelem / t / 1e6
    whole = "the whole config-2 mesh" if args.cpu_nz == 95 else "a slab of the config-2 mesh"
    sample = (f"TET04 {args.nx}x{args.ny}x{args.cpu_nz} box, {whole} ({wl.nelem} elements) per step, "
              f"reference packed kernels in C (oracle/fempack_ref.c), {threads} threads")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": "config 2: TET04 94x94x95 box (5,036,520 elements), NS momentum RHS + "
                               "continuity B_x,B_y,B_z, packed layout", "sample_elements": wl.nelem},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--nx", type=int, default=94)
    ap.add_argument("--ny", type=int, default=94)
    ap.add_argument("--nz", type=int, default=95)
    ap.add_argument("--cpu-nz", type=int, default=95,
                    help="z-layers of the CPU baseline / reference-arm workload (95 = the whole config-2 mesh)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--scatter", default="auto", choices=["auto", "rows", "atomic"],
                    help="global-assembly strategy (AssemblyContext.build)")
    ap.add_argument("--no-solver", action="store_true", help="skip the solver vector-kernel block")
    ap.add_argument("--no-configs", action="store_true", help="skip the config-3 / config-4 blocks")
    ap.add_argument("--soak", type=float, default=1.0, help="untimed seconds under load before timing")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch

    # one GPU per rank; FPB_DIST_BACKEND=gloo lets several ranks share a GPU
    # (functional check of the N > 1 path on a one-GPU box, not a timing)
    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        backend = os.environ.get("FPB_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    import paper_2107_11541_b200 as P

    dev = torch.device("cuda", local)
    if world > 1:
        from paper_2107_11541_b200 import distributed as D

        sub = D.SlabDomain.build(args.nx, args.ny, args.nz * world, rank, world)
        mesh, ctx = sub.mesh, sub.ctx
    else:
        sub = None
        mesh = P.generate_box_mesh(P.ElementType.TET04, args.nx, args.ny, args.nz)
        ctx = P.AssemblyContext.build(mesh, vector_size=8, scatter=args.scatter)
    ctx.refresh_geometry("packed", need_grad=False)
    nelem, nnode, nnz = mesh.nelem, mesh.nnode, ctx.pattern.nnz
    rng = np.random.default_rng(0)
    # host inputs live in pinned memory (the e2e contract: H2D from pinned
    # host buffers); the numpy view is what a reference user passes
    vel_h = torch.empty((nnode, 3), dtype=torch.float64, pin_memory=True).numpy()
    vel_h[:] = rng.standard_normal((nnode, 3))
    vel = torch.as_tensor(vel_h, device=dev)
    rhs = torch.zeros((nnode, 3), dtype=torch.float64, device=dev)
    mats = torch.zeros(3 * nnz, dtype=torch.float64, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()

    side = torch.cuda.Stream() if sub is not None else None
    launches_per_step = 3
    if sub is not None:  # windowed schedule: one launch per non-empty window
        from paper_2107_11541_b200.distributed import _step_windows

        w = _step_windows(sub)
        nonempty = lambda r: r[1] > r[0]  # noqa: E731
        launches_per_step = (sum(map(nonempty, w["blocks_A"])) + sum(map(nonempty, w["nodes_A"]))
                             + sum(map(nonempty, w["rows_A"])) + nonempty(w["blocks_B"])
                             + sum(map(nonempty, w["nodes_B"])) + nonempty(w["rows_B"]))

    def kernels(ev=None):
        if ev:
            ev[0].record(stream)
        ctx.assemble_rhs_d(P.KernelKind.MOMENTUM_RHS, vel, None, 1.0, 1e-2, 0.0, rhs)
        if ev:
            ev[1].record(stream)
        ctx.assemble_gradients_d(mats)
        if ev:
            ev[2].record(stream)

    def step(ev=None):
        if sub is None:
            kernels(ev)
        else:
            # interface rows first, NCCL halo on a side stream overlapping the
            # interior (distributed.assemble_step)
            sub.assemble_step(vel, rhs, mats, 1.0, 1e-2, overlap=True, side=side)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    # soak (untimed) so the clock sampler sees the loaded state; every rank
    # must run the same number of steps (each step has halo exchanges), so
    # rank 0's clock decides and the decision is shared
    t_end = time.perf_counter() + args.soak
    flag = torch.zeros(1, dtype=torch.float64, device=dev)
    while True:
        go = time.perf_counter() < t_end
        if dist:
            flag.fill_(1.0 if (go and rank == 0) else 0.0)
            dist.all_reduce(flag, op=dist.ReduceOp.MAX)
            go = bool(flag.item() > 0.0)
        if not go:
            break
        step()
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms, k_mom, k_grad = [], [], []
    for _ in range(args.steps):
        flush.fill_(1.0)  # L2 flush outside the timed window
        e_start, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e_start.record(stream)
        step(ev)
        e_end.record(stream)
        torch.cuda.synchronize()
        step_ms.append(e_start.elapsed_time(e_end))
        if sub is None:
            k_mom.append(ev[0].elapsed_time(ev[1]))
            k_grad.append(ev[1].elapsed_time(ev[2]))
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    if sub is not None:  # per-kernel times of this rank's slab, outside the timed region
        for _ in range(5):
            flush.fill_(1.0)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            kernels(ev)
            torch.cuda.synchronize()
            k_mom.append(ev[0].elapsed_time(ev[1]))
            k_grad.append(ev[1].elapsed_time(ev[2]))
    total_ms = sum(step_ms)
    if dist:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    total_elems = nelem * world
    value = total_elems / (ms_per_step / 1e3) / 1e6

    # roofline of the dominant kernel (mean launch duration on its stream)
    kern = {"momentum_rhs": statistics.mean(k_mom), "gradient_xyz": statistics.mean(k_grad)}
    dom = max(kern, key=kern.get)
    F, B = WORK[dom]
    t_s = kern[dom] / 1e3
    flops_rate = F * nelem / t_s / 1e12
    bytes_rate = B * nelem / t_s / 1e9
    hbm, hbm_src = hbm_peak()
    if F / B > FP64_PEAK_TFLOPS * 1e3 / hbm:  # compute-bound by the ridge point
        roof = {"bound": "fp64", "achieved": flops_rate, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": flops_rate / FP64_PEAK_TFLOPS,
                "peak_source": "measured DFMA microbenchmark (profiles/r01_microbench.txt)"}
    else:
        roof = {"bound": "hbm", "achieved": bytes_rate, "peak": hbm, "unit": "GB/s",
                "frac": bytes_rate / hbm, "peak_source": hbm_src}
    traffic, ncu = None, None
    try:  # measured DRAM bytes per launch of this kernel (ncu --set full, profiles/traffic.json)
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            entry = json.load(fh)[dom]
        traffic, ncu = entry["bytes"], entry.get("ncu")
    except Exception:
        traffic = None
    roof.update({"kernel": dom, "traffic": traffic, "traffic_unit": "bytes per launch",
                 "algorithmic_bytes": B * nelem,
                 "work_per_element": {"flops": F, "bytes": B, "source": "SURVEY.md 8(d)"}})
    if ncu:
        roof["ncu"] = ncu  # pipe / L1 utilisation of the same kernel (profiles/traffic.json source)
    if roof["bound"] == "fp64":
        roof["note"] = ("achieved = SURVEY 8(d)'s reference-algorithm flops per element / kernel time; the "
                        "closed-form kernel executes fewer FP64 operations than that count, so the algorithmic "
                        "rate can exceed the FP64 peak — the executed FP64 pipe utilisation is roofline.ncu")

    # the whole step against its own roofline: per element, SURVEY 8(d)'s
    # work of each kernel at the binding one of its two roofs, summed
    def _kernel_ns(k):
        Fk, Bk = WORK[k]
        return max(Fk / (FP64_PEAK_TFLOPS * 1e3), Bk / hbm)  # ns per element
    bound_ns = sum(_kernel_ns(k) for k in kern)
    step_roof = {"bound_Gelem_s": 1.0 / bound_ns, "achieved_Gelem_s": nelem / (ms_per_step * 1e6),
                 "frac": (nelem / (ms_per_step * 1e6)) * bound_ns,
                 "per_kernel_bound": {k: ("fp64" if WORK[k][0] / (FP64_PEAK_TFLOPS * 1e3) > WORK[k][1] / hbm
                                          else "hbm") for k in kern},
                 "note": "time-sum of each kernel's roofline bound (momentum FP64, B_xyz HBM) per element"}

    # e2e through the public API with host buffers
    e2e = None
    if args.e2e_steps > 0:
        grads = None
        e2e_ms = []
        e2e_warm = 3  # pinned staging blocks are allocated once, then recycled
        for i in range(args.e2e_steps + e2e_warm):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = ctx.assemble_rhs(P.KernelKind.MOMENTUM_RHS, "packed", vel_h, None, 1.0, 1e-2, 0.0)
            grads = P.gradient_matrices(ctx)
            vals = [B.vals for B in grads]
            torch.cuda.synchronize()
            if i >= e2e_warm:
                e2e_ms.append((time.perf_counter() - t0) * 1e3)
        assert r.shape == (nnode, 3) and all(v.shape == (nnz,) for v in vals)
        t = statistics.mean(e2e_ms)
        if dist:
            tt = torch.tensor([t], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t = float(tt.item())
        e2e = {"value": total_elems / (t / 1e3) / 1e6, "unit": UNIT, "ms_per_step": t,
               "h2d_bytes_per_step": int(vel_h.nbytes),
               "d2h_bytes_per_step": int(r.nbytes + sum(v.nbytes for v in vals)),
               "api": "AssemblyContext.assemble_rhs(MOMENTUM_RHS, numpy) + gradient_matrices(ctx) + .vals"}

    dist_solver = None
    if world > 1 and not args.no_solver:
        dist_solver = dist_bicgstab_block(sub, vel, dev, dist)

    solver = None
    if rank == 0 and world == 1 and not args.no_solver:
        # config 3 companions: SpMV on the MASS matrix, axpy / dot on vectors
        # larger than L2 (C5's node count), Jacobi-PCG on the pinned LAPLACIAN
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        from solver_bench import solver_metrics

        solver = solver_metrics(ctx, 16_974_593, hbm=hbm)

    configs = None
    if rank == 0 and world == 1 and not args.no_configs:
        configs = {"c3": config3_block(ctx, vel, flush, hbm)}
        del mats
        torch.cuda.empty_cache()
        configs["c4"] = config4_block(flush, hbm)
        torch.cuda.empty_cache()
        configs["c5_one_gpu"] = config5_block(flush, hbm)
        configs["flow"] = flow_block(args.nx, args.ny, args.nz)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(args.nx, args.ny, args.cpu_nz)
        except Exception as exc:  # reported, not fatal
            cpu = {"error": repr(exc)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"config 2: TET04 box {args.nx}x{args.ny}x{args.nz} per GPU "
                                   f"({nelem} elements, {nnode} nodes, nnz {nnz}), NS momentum RHS + "
                                   "continuity B_x,B_y,B_z, SIMD-packed (32-lane) layout",
                       "elements_per_step": total_elems, "l2": "flushed (512 MiB write) between steps", "scatter": args.scatter,
                       "parallelism": f"z-slab domain decomposition x{world}" if world > 1 else "single GPU"},
            "roofline": roof,
            "step_roofline": step_roof,
            "kernels_ms": kern,
            # per step: element-block momentum RHS (integrate + partial
            # gather; velocity read in place) and row-owned B_x,B_y,B_z — 3
            # launches (ncu launch list under profiles/); the halo (N > 1) is NCCL
            "gpu_launches": args.steps * launches_per_step,
            "clocks": clk,
            "e2e": e2e,
            "solver": solver,
            "dist_solver": dist_solver,
            "configs": configs,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
