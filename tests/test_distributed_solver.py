"""Distributed solver plumbing: ghost-plane refresh, owned-
row reductions and the slab BiCGSTAB.

CPU (gloo, world 2 and 3): the host logic on torch CPU tensors — after
refresh_ghosts every local entry equals the global vector's, the owned-row
partials of all ranks sum to the global dot, allreduce_sum_ is a sum.
GPU (gloo through the host, 2 ranks sharing the box's one B200): the real
slab BiCGSTAB (device kernels, owned-row reductions, deferred scalar
finishes) reproduces the single-domain device solve."""

import datetime
import os
import tempfile
import traceback

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import fempack_np as O
from paper_2107_11541_b200.distributed import (SlabLayout, allreduce_sum_, ghost_planes, refresh_ghosts)

NX, NY, NZ = 4, 3, 7


def _run(world, target, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with tempfile.TemporaryDirectory() as d:
        initfile = os.path.join(d, "init")
        procs = [ctx.Process(target=target, args=(r, world, initfile, q) + args) for r in range(world)]
        for p in procs:
            p.start()
        out = q.get(timeout=240)
        for p in procs:
            p.join(timeout=60)
            if p.exitcode is None:
                p.kill()
        if isinstance(out, str):
            raise AssertionError(out)
        for p in procs:
            assert p.exitcode == 0
    return out


def _plumbing_worker(rank, world, initfile, q):
    dist.init_process_group("gloo", init_method=f"file://{initfile}", rank=rank, world_size=world)
    try:
        L = SlabLayout.make(NX, NY, NZ, rank, world)
        nglob = (NX + 1) * (NY + 1) * (NZ + 1)
        g = torch.as_tensor(np.random.default_rng(7).standard_normal(nglob))
        loc = g[L.node_offset:L.node_offset + L.nnode].clone()
        for _, _, kg in ghost_planes(L):  # poison the ghost planes
            lo, hi = L.plane_rows(kg)
            loc[lo:hi] = float("nan")
        refresh_ghosts(L, loc)
        ok_refresh = bool(torch.equal(loc, g[L.node_offset:L.node_offset + L.nnode]))
        lo, hi = L.owned_rows
        part = torch.tensor([float((loc[lo:hi] * loc[lo:hi]).sum()), float(rank + 1)], dtype=torch.float64)
        allreduce_sum_(part)
        res = {"refresh": ok_refresh, "dot": float(part[0]), "ranks": float(part[1]),
               "want": float((g * g).sum())}
        gathered = [None] * world
        dist.all_gather_object(gathered, res)
        if rank == 0:
            q.put(gathered)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ghost_refresh_and_owned_reductions(world):
    parts = _run(world, _plumbing_worker)
    for p in parts:
        assert p["refresh"]
        assert p["ranks"] == world * (world + 1) / 2
        assert p["dot"] == pytest.approx(p["want"], rel=1e-13)


def test_ghost_plan_covers_neighbours():
    for world in (2, 3, 4):
        for r in range(world):
            L = SlabLayout.make(NX, NY, NZ, r, world)
            plan = ghost_planes(L)
            assert len(plan) == (r > 0) + (r < world - 1)
            for peer, ks, kg in plan:
                P = SlabLayout.make(NX, NY, NZ, peer, world)
                # what the peer sends is what I receive: its plane ks is my ghost plane kg
                (_, ks2, kg2), = [t for t in ghost_planes(P) if t[0] == r]
                assert ks2 == kg and kg2 == ks
                # and the sent plane lies in the sender's exactly computed range
                assert L.k0 <= ks <= L.k1


# ------------------------------------------------------------------ device
def _system_slab(P, dom, vel_g, b_g, dt=0.05, kappa=0.01):
    L = dom.layout
    ctx = dom.ctx
    v = torch.as_tensor(vel_g[L.node_offset:L.node_offset + L.nnode], device="cuda")
    nnz = ctx.pattern.nnz
    mats = []
    for kind, vel in ((P.KernelKind.MASS, None), (P.KernelKind.CONVECTION, v), (P.KernelKind.LAPLACIAN, None)):
        m = torch.empty(nnz, dtype=torch.float64, device="cuda")
        ctx.assemble_matrix_d(kind, vel, m)
        dom.halo_sum_matrix(m)
        mats.append(m)
    vals = mats[0] + dt * (mats[1] + kappa * mats[2])
    A = ctx.pattern.with_vals(vals)
    b = torch.as_tensor(b_g[L.node_offset:L.node_offset + L.nnode], device="cuda")
    return A, b


def _solver_worker(rank, world, initfile, q, dims):
    import paper_2107_11541_b200 as P
    from paper_2107_11541_b200.distributed import SlabDomain, bicgstab_slab

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"file://{initfile}", rank=rank, world_size=world,
                            timeout=datetime.timedelta(seconds=120))
    try:
        nx, ny, nz = dims
        nglob = (nx + 1) * (ny + 1) * (nz + 1)
        vel_g, sc = O.bench_fields(nglob, 3)
        dom = SlabDomain.build(nx, ny, nz, rank, world)
        A, b = _system_slab(P, dom, vel_g, sc[0])
        x, st = bicgstab_slab(dom.layout, A, b, tol=1e-10, check_every=4)
        L = dom.layout
        x0 = torch.as_tensor(np.linspace(-1.0, 1.0, nglob)[L.node_offset:L.node_offset + L.nnode], device="cuda")
        x2, st2 = bicgstab_slab(L, A, b, x0=x0, tol=1e-10, check_every=4)
        lo, hi = L.owned_rows
        res = {"x": x[lo:hi].cpu().numpy(), "it": st.iterations, "conv": st.converged,
               "hist": st.residual_history, "tr": st.true_residual,
               "consistent": bool(torch.isfinite(x).all()),
               "x2": x2[lo:hi].cpu().numpy(), "it2": st2.iterations, "conv2": st2.converged}
        gathered = [None] * world
        dist.all_gather_object(gathered, res)
        if rank == 0:
            q.put(gathered)
    except Exception:
        q.put(f"rank {rank}: " + traceback.format_exc())
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_slab_bicgstab_reproduces_single_domain(cuda_ok, world):
    import paper_2107_11541_b200 as P

    dims = (9, 8, 11)
    parts = _run(world, _solver_worker, dims)
    nx, ny, nz = dims
    full = P.AssemblyContext.build(P.generate_box_mesh(P.ElementType.TET04, nx, ny, nz), 8)
    n = full.mesh.nnode
    vel_g, sc = O.bench_fields(n, 3)
    M = full.assemble_matrix(P.KernelKind.MASS)
    C = full.assemble_matrix(P.KernelKind.CONVECTION, velocity=vel_g)
    Lp = full.assemble_matrix(P.KernelKind.LAPLACIAN)
    A = M.with_vals(M.vals_d + 0.05 * (C.vals_d + 0.01 * Lp.vals_d))
    x, st = P.bicgstab_solve(A, sc[0], tol=1e-10)
    got = np.concatenate([p["x"] for p in parts])
    assert got.shape == x.shape
    for p in parts:
        assert p["conv"] and p["consistent"]
        assert abs(p["it"] - st.iterations) <= 1
        assert p["tr"] < 1.01e-10
        k = min(len(p["hist"]), len(st.residual_history), 6)
        np.testing.assert_allclose(p["hist"][:k], st.residual_history[:k], rtol=1e-9)
    assert O.rel_diff(got, x) < 1e-8
    xb, stb = P.bicgstab_solve(A, sc[0], x0=np.linspace(-1.0, 1.0, n), tol=1e-10)
    for p in parts:
        assert p["conv2"] and abs(p["it2"] - stb.iterations) <= 1
    assert O.rel_diff(np.concatenate([p["x2"] for p in parts]), xb) < 1e-8


def _step_worker(rank, world, initfile, q, dims):
    import paper_2107_11541_b200 as P  # noqa: F401
    from paper_2107_11541_b200.distributed import SlabDomain

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"file://{initfile}", rank=rank, world_size=world,
                            timeout=datetime.timedelta(seconds=120))
    try:
        nx, ny, nz = dims
        nglob = (nx + 1) * (ny + 1) * (nz + 1)
        vel_g, _ = O.bench_fields(nglob, 3)
        dom = SlabDomain.build(nx, ny, nz, rank, world)
        L = dom.layout
        vel = torch.as_tensor(vel_g[L.node_offset:L.node_offset + L.nnode], device="cuda")
        nnz = dom.ctx.pattern.nnz
        out = {}
        for ov in (False, True):
            rhs = torch.full((L.nnode, 3), float("nan"), dtype=torch.float64, device="cuda")
            mats = torch.full((3 * nnz,), float("nan"), dtype=torch.float64, device="cuda")
            dom.assemble_step(vel, rhs, mats, overlap=ov)
            torch.cuda.synchronize()
            out[ov] = (rhs.cpu().numpy(), mats.cpu().numpy())
        # CUDA-graph replay (gloo: two captured phases, eager halo between)
        from paper_2107_11541_b200.distributed import SlabStepGraph

        rhs = torch.full((L.nnode, 3), float("nan"), dtype=torch.float64, device="cuda")
        mats = torch.full((3 * nnz,), float("nan"), dtype=torch.float64, device="cuda")
        sg = SlabStepGraph(dom, vel, rhs, mats)
        rhs.fill_(float("nan"))
        mats.fill_(float("nan"))
        sg.replay()
        sg.replay()  # idempotent: every row overwritten, halo re-summed from fresh partials
        torch.cuda.synchronize()
        graph_same = bool(np.array_equal(rhs.cpu().numpy(), out[False][0]) and
                          np.array_equal(mats.cpu().numpy(), out[False][1]))
        lo, hi = L.owned_rows
        res = {"same": bool(np.array_equal(out[False][0], out[True][0]) and
                            np.array_equal(out[False][1], out[True][1])) and graph_same,
               "finite": bool(np.isfinite(out[True][0]).all() and np.isfinite(out[True][1]).all()),
               "rhs": out[True][0][lo:hi],
               "kuhn": dom.ctx.groups[0].kuhn is not None}
        rp = dom.ctx.pattern.rowptr_d.cpu().numpy()
        a, b = int(rp[lo]), int(rp[hi])
        res["mats"] = np.concatenate([out[True][1][m * nnz + a:m * nnz + b] for m in range(3)])
        res["mat_rows"] = (lo + L.node_offset, hi + L.node_offset)
        gathered = [None] * world
        dist.all_gather_object(gathered, res)
        if rank == 0:
            q.put(gathered)
    except Exception:
        q.put(f"rank {rank}: " + traceback.format_exc())
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_interface_first_step_matches_plain_step(cuda_ok, world):
    """The overlapped schedule (interface windows, halo on a side stream,
    interior windows) and its CUDA-graph replay (SlabStepGraph) write every
    row and equal the plain sequence bit for bit; owned RHS rows equal the
    single-domain assembly."""
    import paper_2107_11541_b200 as P

    dims = (9, 8, 11)
    parts = _run(world, _step_worker, dims)
    for p in parts:
        assert p["same"] and p["finite"]
    nx, ny, nz = dims
    full = P.AssemblyContext.build(P.generate_box_mesh(P.ElementType.TET04, nx, ny, nz), 8)
    vel_g, _ = O.bench_fields(full.mesh.nnode, 3)
    want = full.assemble_rhs(P.KernelKind.MOMENTUM_RHS, "packed", vel_g, None, 1.0, 1e-2, 0.0)
    assert O.rel_diff(np.concatenate([p["rhs"] for p in parts]), want) < 1e-13
    # owned CSR rows of B_x, B_y, B_z (interface rows halo-summed) = the single domain's
    import torch as _t

    g = _t.empty(3 * full.pattern.nnz, dtype=_t.float64, device="cuda")
    full.assemble_gradients_d(g)
    g = g.cpu().numpy()
    rpg = full.pattern.rowptr_d.cpu().numpy()
    nnzg = full.pattern.nnz
    for p in parts:
        r0, r1 = p["mat_rows"]
        a, b = int(rpg[r0]), int(rpg[r1])
        wantm = np.concatenate([g[m * nnzg + a:m * nnzg + b] for m in range(3)])
        assert p["mats"].shape == wantm.shape
        assert O.rel_diff(p["mats"], wantm) < 1e-13
    assert all(p["kuhn"] for p in parts)  # the slab step ran the Kuhn-box kernels


def _fake_domain(nx, ny, nz, rank, world, be=256):
    from types import SimpleNamespace

    L = SlabLayout.make(nx, ny, nz, rank, world)
    ne = (L.k1 - L.k0) * L.elems_per_layer
    blocks = SimpleNamespace(block_elems=be, nblocks=-(-ne // be))
    ctx = SimpleNamespace(groups=[SimpleNamespace(blocks=blocks)], mesh=SimpleNamespace(nnode=L.nnode))
    return SimpleNamespace(layout=L, ctx=ctx), ne


@pytest.mark.parametrize("world", [2, 3, 5])
@pytest.mark.parametrize("dims", [(9, 8, 11), (94, 94, 95), (4, 3, 7)])
def test_step_windows_partition_the_work(world, dims):
    """Interface-first windows (distributed._step_windows): row windows start
    on 32-row slices and tile [0, n); the interface planes lie in the
    phase-A rows and nodes; node and block windows tile their ranges; the
    phase-A blocks contain every element of the first / last own layer."""
    from paper_2107_11541_b200.distributed import _step_windows

    nx, ny, nz = dims
    if nz < world:
        pytest.skip("fewer layers than ranks")
    for r in range(world):
        dom, ne = _fake_domain(nx, ny, nz * world if nz < 20 else nz, r, world)
        L, n = dom.layout, dom.ctx.mesh.nnode
        w = _step_windows(dom)
        rows = sorted([x for x in w["rows_A"] if x[1] > x[0]] + ([w["rows_B"]] if w["rows_B"][1] > w["rows_B"][0] else []))
        assert rows[0][0] == 0 and rows[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
        assert all(x[0] % 32 == 0 for x in rows)
        for _, k in L.interfaces():
            lo, hi = L.plane_rows(k)
            assert any(a <= lo and hi <= b for a, b in w["rows_A"])
            assert (lo, hi) in w["nodes_A"]
        nodes = sorted(w["nodes_A"] + w["nodes_B"])
        assert nodes[0][0] == 0 and nodes[-1][1] == n and all(a[1] == b[0] for a, b in zip(nodes, nodes[1:]))
        nb, be = dom.ctx.groups[0].blocks.nblocks, dom.ctx.groups[0].blocks.block_elems
        blk = sorted([x for x in w["blocks_A"] if x[1] > x[0]] + ([w["blocks_B"]] if w["blocks_B"][1] > w["blocks_B"][0] else []))
        assert blk[0][0] == 0 and blk[-1][1] == nb and all(a[1] == b[0] for a, b in zip(blk, blk[1:]))
        covered = set()
        for a, b in w["blocks_A"]:
            covered.update(range(a * be, min(b * be, ne)))
        epl, nlay = L.elems_per_layer, L.k1 - L.k0
        if r > 0:
            assert covered.issuperset(range(0, epl))
        if r < world - 1:
            assert covered.issuperset(range((nlay - 1) * epl, nlay * epl))
