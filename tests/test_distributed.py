"""Z-slab domain decomposition (paper_2107_11541_b200/distributed.py) on CPU
with the gloo backend, world size 2 and 3.

Each rank builds its slab (own cell layers + ghost layers) with the CPU
oracle, assembles its own elements (oracle kernels = the reference packed
arithmetic), runs the package's halo sums over gloo, and the owned rows of
all ranks must reproduce the single-domain assembly: CSR graph rows and
element ranges bit-exact, values within 1e-13 (only the order of the
interface sums differs)."""

import os
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import fempack_np as O
from paper_2107_11541_b200.distributed import (SlabLayout, halo_sum_nodes, halo_sum_rows,
                                               slab_ranges)
from paper_2107_11541_b200.elements import ElementType

NX, NY, NZ = 4, 3, 7


def test_slab_ranges_restated():
    """Partition pinned by its NumPy restatement (np.array_split)."""
    for nz in (1, 5, 7, 95, 256):
        for world in (1, 2, 3, 4, 8):
            if world > nz:
                continue
            want = [(int(c[0]), int(c[-1]) + 1) for c in np.array_split(np.arange(nz), world)]
            assert slab_ranges(nz, world) == want


def test_layout_covers_mesh_exactly():
    """Owned elements tile the global element range; owned node rows tile
    the global node range (interface plane to the lower rank)."""
    for et, per in ((ElementType.TET04, 6), (ElementType.HEX08, 1)):
        for world in (1, 2, 3, 4):
            elems, rows = [], []
            for r in range(world):
                L = SlabLayout.make(NX, NY, NZ, r, world, et)
                e0, e1 = L.own_elems
                g0 = L.global_elem_offset
                elems.append((g0, g0 + e1 - e0))
                lo, hi = L.owned_rows
                rows.append((lo + L.node_offset, hi + L.node_offset))
            assert elems[0][0] == 0 and elems[-1][1] == NX * NY * NZ * per
            assert all(a[1] == b[0] for a, b in zip(elems, elems[1:]))
            assert rows[0][0] == 0 and rows[-1][1] == (NX + 1) * (NY + 1) * (NZ + 1)
            assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))


def _slab_oracle(L):
    """Local (extended) slab built by the oracle: coords rows of planes
    kA..kB of the global grid, connectivity of kB-kA cell layers."""
    gcoords = O.grid_coords(NX, NY, NZ, (1.0, 1.0, 1.0), 3)
    coords = gcoords[L.node_offset:L.node_offset + L.nnode]
    _, _, groups = O.generate_box_mesh(O.TET04, NX, NY, L.kB - L.kA)
    conn_ext = groups[0][1]
    e0, e1 = L.own_elems
    return coords, conn_ext, conn_ext[e0:e1]


def _worker(rank, world, initfile, out):
    dist.init_process_group("gloo", init_method=f"file://{initfile}", rank=rank, world_size=world)
    try:
        L = SlabLayout.make(NX, NY, NZ, rank, world)
        coords, conn_ext, conn_own = _slab_oracle(L)
        n = L.nnode
        rowptr, colind = O.build_node_pattern(n, [conn_ext])
        gvel, gsc = O.bench_fields((NX + 1) * (NY + 1) * (NZ + 1), 3)
        vel = gvel[L.node_offset:L.node_offset + n]
        mesh = O.OracleMesh(3, coords, [(O.TET04, conn_own)])
        # local assembly of own elements
        rhs = O.assemble_rhs(mesh, "momentum_rhs", vel, None, 1.0, 1e-2, 0.0)
        mats = []
        for k in range(3):
            unit = np.zeros((n, 3))
            unit[:, k] = 1.0
            mats.append(O.assemble_matrix(mesh, "convection", unit, pattern=(rowptr, colind))[2])
        rhs_t = torch.from_numpy(rhs.copy())
        halo_sum_nodes(L, rhs_t)
        vals_t = torch.from_numpy(np.concatenate(mats))
        halo_sum_rows(L, torch.from_numpy(rowptr), vals_t, nmat=3)
        lo, hi = L.owned_rows
        nnz = colind.size
        vals = vals_t.numpy().reshape(3, nnz)
        own = {
            "rows": (lo + L.node_offset, hi + L.node_offset),
            "rhs": rhs_t.numpy()[lo:hi],
            "rowlen": np.diff(rowptr)[lo:hi],
            "cols": colind[rowptr[lo]:rowptr[hi]] + L.node_offset,
            "vals": vals[:, rowptr[lo]:rowptr[hi]],
            # both copies of an interface row must be bitwise equal after the sum
            "iface": [(k, rhs_t.numpy()[slice(*L.plane_rows(k))].tobytes()) for _, k in L.interfaces()],
        }
        gathered = [None] * world
        dist.all_gather_object(gathered, own)
        if rank == 0:
            out.put(gathered)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_halo_sum_reproduces_single_domain(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with tempfile.TemporaryDirectory() as d:
        initfile = os.path.join(d, "init")
        procs = [ctx.Process(target=_worker, args=(r, world, initfile, q)) for r in range(world)]
        for p in procs:
            p.start()
        parts = q.get(timeout=300)
        for p in procs:
            p.join(timeout=60)
            assert p.exitcode == 0
    # single-domain reference
    m = O.box(O.TET04, NX, NY, NZ)
    (et, conn), = m.groups
    rowptr, colind = O.build_node_pattern(m.nnode, [conn])
    vel, _ = O.bench_fields(m.nnode, 3)
    rhs = O.assemble_rhs(m, "momentum_rhs", vel, None, 1.0, 1e-2, 0.0)
    mats = []
    for k in range(3):
        unit = np.zeros((m.nnode, 3))
        unit[:, k] = 1.0
        mats.append(O.assemble_matrix(m, "convection", unit)[2])
    got_rhs = np.concatenate([p["rhs"] for p in parts])
    assert O.rel_diff(got_rhs, rhs) < 1e-13
    # CSR graph rows bit-exact
    np.testing.assert_array_equal(np.concatenate([p["rowlen"] for p in parts]), np.diff(rowptr))
    np.testing.assert_array_equal(np.concatenate([p["cols"] for p in parts]), colind)
    for k in range(3):
        got = np.concatenate([p["vals"][k] for p in parts])
        assert O.rel_diff(got, mats[k]) < 1e-13
    # interface copies agree bit for bit on both sides
    faces = {}
    for p in parts:
        for k, b in p["iface"]:
            faces.setdefault(k, []).append(b)
    assert faces and all(len(v) == 2 and v[0] == v[1] for v in faces.values())


def _timeout_worker(rank, world, initfile, out, done):
    import time

    from paper_2107_11541_b200.distributed import init_process_group

    init_process_group("gloo", timeout_s=3.0, init_method=f"file://{initfile}", rank=rank, world_size=world)
    if rank == 0:
        t = torch.ones(4)
        t0 = time.perf_counter()
        try:
            dist.all_reduce(t)  # rank 1 never joins: a dead neighbour
            out.put(("returned", time.perf_counter() - t0))
        except RuntimeError as e:
            out.put(("raised", time.perf_counter() - t0, type(e).__name__))
        done.set()
    else:
        done.wait(60)


def test_collective_timeout_detects_missing_rank():
    """Failure detection: with the bounded timeout of
    distributed.init_process_group, a collective whose peer never arrives
    raises on the waiting rank within seconds instead of hanging."""
    ctx = mp.get_context("spawn")
    q, done = ctx.Queue(), ctx.Event()
    with tempfile.TemporaryDirectory() as d:
        initfile = os.path.join(d, "init")
        procs = [ctx.Process(target=_timeout_worker, args=(r, 2, initfile, q, done)) for r in range(2)]
        for p in procs:
            p.start()
        res = q.get(timeout=120)
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    assert res[0] == "raised", res
    assert 2.0 < res[1] < 30.0, res


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_device_slabs_reproduce_single_domain(cuda_ok, world):
    """The device slab builder (fpb_grid_coords_slab, ghost-layer CSR graph,
    own-element contexts) on one GPU: W slabs assembled separately, interface
    planes summed pairwise (what the NCCL halo does across GPUs), owned rows
    equal to the single-domain device assembly and to the oracle."""
    import paper_2107_11541_b200 as P
    from paper_2107_11541_b200.distributed import SlabDomain

    nx, ny, nz = 9, 8, 11
    full = P.AssemblyContext.build(P.generate_box_mesh(P.ElementType.TET04, nx, ny, nz), 8)
    vel_g, _ = O.bench_fields(full.mesh.nnode, 3)
    vel_gd = torch.as_tensor(vel_g, device="cuda")
    doms = [SlabDomain.build(nx, ny, nz, r, world) for r in range(world)]
    rhs, mats = [], []
    for d in doms:
        L = d.layout
        v = vel_gd[L.node_offset:L.node_offset + L.nnode]
        r = torch.empty((L.nnode, 3), dtype=torch.float64, device="cuda")
        d.ctx.assemble_rhs_d(P.KernelKind.MOMENTUM_RHS, v, None, 1.0, 1e-2, 0.0, r)
        m = torch.empty(3 * d.ctx.pattern.nnz, dtype=torch.float64, device="cuda")
        d.ctx.assemble_gradients_d(m)
        rhs.append(r)
        mats.append(m)
    # pairwise interface sums (rank r top plane <-> rank r+1 bottom plane)
    for r in range(world - 1):
        a, b = doms[r].layout, doms[r + 1].layout
        k = a.k1
        sa, sb = slice(*a.plane_rows(k)), slice(*b.plane_rows(k))
        tot = rhs[r][sa] + rhs[r + 1][sb]
        rhs[r][sa] = tot
        rhs[r + 1][sb] = tot
        (_, pa0, pa1), = [s for s in doms[r].segs if s[0] == r + 1]
        (_, pb0, pb1), = [s for s in doms[r + 1].segs if s[0] == r]
        na, nb = doms[r].ctx.pattern.nnz, doms[r + 1].ctx.pattern.nnz
        for mm in range(3):
            t = mats[r][mm * na + pa0:mm * na + pa1] + mats[r + 1][mm * nb + pb0:mm * nb + pb1]
            mats[r][mm * na + pa0:mm * na + pa1] = t
            mats[r + 1][mm * nb + pb0:mm * nb + pb1] = t
    got_rhs = torch.cat([rhs[r][slice(*doms[r].layout.owned_rows)] for r in range(world)]).cpu().numpy()
    want = full.assemble_rhs(P.KernelKind.MOMENTUM_RHS, "packed", vel_g, None, 1.0, 1e-2, 0.0)
    assert O.rel_diff(got_rhs, want) < 1e-13
    grads = P.gradient_matrices(full)
    for mm in range(3):
        parts = []
        for r, d in enumerate(doms):
            lo, hi = d.layout.owned_rows
            rp = d.ctx.pattern.rowptr
            nnz = d.ctx.pattern.nnz
            parts.append(mats[r][mm * nnz + rp[lo]:mm * nnz + rp[hi]].cpu().numpy())
            # owned rows carry the global column lists
            cols = d.ctx.pattern.colind[rp[lo]:rp[hi]] + d.layout.node_offset
            g0, g1 = lo + d.layout.node_offset, hi + d.layout.node_offset
            np.testing.assert_array_equal(cols, full.pattern.colind[full.pattern.rowptr[g0]:full.pattern.rowptr[g1]])
        assert O.rel_diff(np.concatenate(parts), grads[mm].vals) < 1e-13
    # slab coordinates are the full grid's rows, bit for bit
    for d in doms:
        L = d.layout
        assert d.mesh.coords.tobytes() == full.mesh.coords[L.node_offset:L.node_offset + L.nnode].tobytes()
