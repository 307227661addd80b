"""Z-slab domain decomposition of the synthetic box meshes across GPUs.

The reference has no partitioner; this module defines one
 and is pinned by its own restatement in the tests:

* Cells are visited k-major (mesh.py:220-224) and nodes are numbered
  i + (nx+1)(j + (ny+1)k) (mesh.py:183-184), so a contiguous range of cell
  layers [k0, k1) is a contiguous range of elements and its node planes
  k0..k1 a contiguous range of nodes.  Rank r owns layers
  [k0_r, k1_r) = balanced split of nz (first ranks take the remainder).
* Every rank keeps one ghost cell layer on each side that has a neighbour.
  Ghost elements are never integrated; they only shape the local CSR graph,
  so the rows of an interface plane have the same global column set on both
  sides and their values can be summed entry by entry.
* Halo sum: after local assembly, each interface plane's RHS rows / CSR row
  segments are exchanged with the neighbour (one grouped send/recv pair per
  interface — NCCL over NVLink on GPUs, gloo on CPU) and added, so both
  copies hold the global value (a + b == b + a bit for bit).
* Ownership for gathering a global result: rank r owns node planes
  [k0_r + (r > 0), k1_r] — interface plane k1_r belongs to the lower rank.

Everything here is device-agnostic torch code except `SlabDomain.build`,
which generates the local mesh with the CUDA setup kernels.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from .elements import ElementType

# slab domains assemble with the Kuhn-box kernels (no interface-first
# windows: the halo follows the whole-slab kernels); False = windowed
# element-block / row kernels with the halo overlapped
SLAB_KUHN = True


def init_process_group(backend: str = "nccl", device: torch.device | None = None,
                       timeout_s: float | None = None, **kw) -> None:
    """`dist.init_process_group` with the failure detection the slab path relies on.

    * A bounded collective timeout (FPB_DIST_TIMEOUT_S, default 300 s): a rank
      that dies or hangs mid-halo turns into an exception on its peers
      instead of an indefinite wait.
    * NCCL async error handling on (TORCH_NCCL_ASYNC_ERROR_HANDLING=1 unless
      the caller set it): the watchdog aborts the communicator on a timeout or
      a remote failure, so the process exits non-zero.
    * The NCCL group is bound to this rank's device (eager init, the
      communicator exists before the first halo).
    """
    import datetime
    import os

    if timeout_s is None:
        timeout_s = float(os.environ.get("FPB_DIST_TIMEOUT_S", "300"))
    if backend == "nccl":
        os.environ.setdefault("TORCH_NCCL_ASYNC_ERROR_HANDLING", "1")
        if device is not None:
            kw.setdefault("device_id", device)
    dist.init_process_group(backend, timeout=datetime.timedelta(seconds=timeout_s), **kw)


def slab_ranges(nz: int, world: int) -> list[tuple[int, int]]:
    """Balanced cell-layer ranges [k0, k1) per rank."""
    if world < 1 or nz < world:
        raise ValueError(f"cannot split {nz} cell layers over {world} ranks")
    base, rem = divmod(nz, world)
    out, k = [], 0
    for r in range(world):
        n = base + (1 if r < rem else 0)
        out.append((k, k + n))
        k += n
    return out


@dataclass(frozen=True)
class SlabLayout:
    """Index bookkeeping of one rank's slab (all counts in the box grid)."""

    nx: int
    ny: int
    nz: int
    rank: int
    world: int
    k0: int  # first owned cell layer
    k1: int  # one past the last owned cell layer
    kA: int  # first local node plane (k0 - 1 with a lower neighbour)
    kB: int  # last local node plane (k1 + 1 with an upper neighbour)
    cells_per_layer: int
    elems_per_cell: int

    @classmethod
    def make(cls, nx, ny, nz, rank, world, etype: ElementType = ElementType.TET04) -> "SlabLayout":
        k0, k1 = slab_ranges(nz, world)[rank]
        kA = k0 - (1 if rank > 0 else 0)
        kB = k1 + (1 if rank < world - 1 else 0)
        per = {ElementType.TET04: 6, ElementType.HEX08: 1}[etype]
        return cls(nx, ny, nz, rank, world, k0, k1, kA, kB, nx * ny, per)

    @property
    def plane(self) -> int:
        return (self.nx + 1) * (self.ny + 1)

    @property
    def nplanes(self) -> int:
        return self.kB - self.kA + 1

    @property
    def nnode(self) -> int:
        return self.plane * self.nplanes

    @property
    def node_offset(self) -> int:
        """global node id = local node id + node_offset."""
        return self.plane * self.kA

    @property
    def elems_per_layer(self) -> int:
        return self.cells_per_layer * self.elems_per_cell

    @property
    def own_elems(self) -> tuple[int, int]:
        """Own elements as a local element range of the extended slab."""
        return ((self.k0 - self.kA) * self.elems_per_layer, (self.k1 - self.kA) * self.elems_per_layer)

    @property
    def global_elem_offset(self) -> int:
        return self.k0 * self.elems_per_layer

    def plane_rows(self, k: int) -> tuple[int, int]:
        """Local node range of global node plane k."""
        lo = (k - self.kA) * self.plane
        return lo, lo + self.plane

    @property
    def owned_rows(self) -> tuple[int, int]:
        first = self.k0 + (1 if self.rank > 0 else 0)
        return (first - self.kA) * self.plane, (self.k1 - self.kA + 1) * self.plane

    def interfaces(self) -> list[tuple[int, int]]:
        """(neighbour rank, global plane) for each interface of this rank."""
        out = []
        if self.rank > 0:
            out.append((self.rank - 1, self.k0))
        if self.rank < self.world - 1:
            out.append((self.rank + 1, self.k1))
        return out


def _exchange(sends: list[tuple[int, torch.Tensor]], group=None) -> list[torch.Tensor]:
    """Grouped point-to-point exchange; returns one received buffer per send
    (on the send buffers' device).  NCCL moves device memory directly; gloo
    (CPU tests, or several ranks sharing one GPU) is staged through the host."""
    if not sends:
        return []
    dev = sends[0][1].device
    staged = dev.type == "cuda" and dist.get_backend(group) != "nccl"
    if staged:
        sends = [(peer, t.cpu()) for peer, t in sends]
    recvs = [torch.empty_like(t) for _, t in sends]
    ops = []
    for (peer, t), r in zip(sends, recvs):
        ops.append(dist.P2POp(dist.isend, t, peer, group))
        ops.append(dist.P2POp(dist.irecv, r, peer, group))
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    return [r.to(dev) for r in recvs] if staged else recvs


class NativeComm:
    """The compiled NCCL path (halo.cu): one NCCL communicator per rank made
    through the C ABI (fpb_nccl_unique_id on rank 0, broadcast over the
    process group, fpb_nccl_comm_init), then fpb_halo_exchange /
    fpb_allreduce_sum on the current stream.  Used whenever the process
    group runs NCCL (FPB_NATIVE_HALO=0 selects torch.distributed instead);
    every call is CUDA-graph capturable, and scratch buffers are allocated
    once and reused, so captured graphs stay valid."""

    def __init__(self, group=None):
        import ctypes

        from . import _lib

        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        uid = (ctypes.c_ubyte * 128)()
        if self.rank == 0:
            _lib.call("fpb_nccl_unique_id", ctypes.addressof(uid))
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        self._uid = (ctypes.c_ubyte * 128).from_buffer_copy(obj[0])
        self.ptr = ctypes.c_void_p()
        _lib.call("fpb_nccl_comm_init", self.world, self.rank, ctypes.addressof(self._uid),
                  torch.cuda.current_device(), ctypes.byref(self.ptr))
        self._scratch: torch.Tensor | None = None

    def _scratch_for(self, n: int, dev) -> torch.Tensor:
        if self._scratch is None or self._scratch.numel() < n:
            self._scratch = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
        return self._scratch

    def exchange(self, segs, x: torch.Tensor, add: bool) -> torch.Tensor:
        """segs: [(peer, send offset, receive offset, count)] in elements of
        x's flat storage; add = sum into place, else copy into place."""
        import numpy as np

        from . import _lib

        if not segs:
            return x
        peers = np.array([p for p, _, _, _ in segs], dtype=np.int32)
        so = np.array([a for _, a, _, _ in segs], dtype=np.int64)
        ro = np.array([b for _, _, b, _ in segs], dtype=np.int64)
        cnt = np.array([c for _, _, _, c in segs], dtype=np.int64)
        scratch = self._scratch_for(int(cnt.sum()), x.device) if add else None
        _lib.call("fpb_halo_exchange", self.ptr, len(segs), peers.ctypes.data, so.ctypes.data, ro.ctypes.data,
                  cnt.ctypes.data, int(add), x.data_ptr(), _lib.ptr(scratch), _lib.stream())
        return x

    def allreduce(self, t: torch.Tensor) -> torch.Tensor:
        from . import _lib

        _lib.call("fpb_allreduce_sum", self.ptr, t.data_ptr(), t.numel(), _lib.stream())
        return t

    def close(self) -> None:
        """Destroy the communicator (free any CUDA graph that captured its
        work first: NCCL waits for it)."""
        from . import _lib

        if self.ptr:
            _lib.call("fpb_nccl_comm_destroy", self.ptr)
            self.ptr = None


def native_comm(group=None):
    """NativeComm for an NCCL process group (None for gloo, or when
    FPB_NATIVE_HALO=0)."""
    import os

    if not dist.is_available() or not dist.is_initialized():
        return None  # domains built outside a process group (single-process tests)
    if dist.get_backend(group) != "nccl" or os.environ.get("FPB_NATIVE_HALO", "1") == "0":
        return None
    return NativeComm(group)


def halo_sum_nodes(layout: SlabLayout, x: torch.Tensor, group=None, native: NativeComm | None = None) -> torch.Tensor:
    """Sum a node-major field (x[n] or x[n, c]) across every interface plane,
    in place: both copies of an interface row end up with mine + theirs."""
    segs = [(peer, layout.plane_rows(k)) for peer, k in layout.interfaces()]
    if native is not None:
        c = x[0].numel() if x.dim() > 1 else 1
        return native.exchange([(p, lo * c, lo * c, (hi - lo) * c) for p, (lo, hi) in segs], x, True)
    sends = [(peer, x[lo:hi].contiguous()) for peer, (lo, hi) in segs]
    recvs = _exchange(sends, group)
    for (peer, (lo, hi)), r in zip(segs, recvs):
        x[lo:hi] += r
    return x


def interface_segments(layout: SlabLayout, rowptr) -> list[tuple[int, int, int]]:
    """(peer, first entry, end entry) of each interface plane's CSR rows."""
    segs = []
    for peer, k in layout.interfaces():
        lo, hi = layout.plane_rows(k)
        segs.append((peer, int(rowptr[lo]), int(rowptr[hi])))
    return segs


def halo_sum_rows(layout: SlabLayout, rowptr: torch.Tensor, vals: torch.Tensor, nmat: int = 1,
                  nnz: int | None = None, group=None, segs=None, native: NativeComm | None = None) -> torch.Tensor:
    """Sum the CSR values of every interface-plane row across the interface,
    in place.  vals holds nmat matrices back to back (vals[m*nnz + k]); the
    interface rows are contiguous, and have identical global column lists on
    both sides (ghost layers), so the segments line up entry for entry."""
    if nnz is None:
        nnz = vals.numel() // nmat
    if segs is None:
        segs = interface_segments(layout, rowptr)
    if native is not None:
        return native.exchange([(p, m * nnz + a, m * nnz + a, b - a) for p, a, b in segs for m in range(nmat)],
                               vals, True)
    sends = []
    for peer, a, b in segs:
        parts = [vals[m * nnz + a:m * nnz + b] for m in range(nmat)]
        sends.append((peer, torch.cat(parts) if nmat > 1 else parts[0].contiguous()))
    recvs = _exchange(sends, group)
    for (peer, a, b), r in zip(segs, recvs):
        w = b - a
        for m in range(nmat):
            vals[m * nnz + a:m * nnz + b] += r[m * w:(m + 1) * w]
    return vals


class SlabDomain:
    """One rank's slab of an (nx, ny, nz) box mesh on its GPU: local mesh
    (own + ghost layers), CSR graph of the extended slab, an assembly
    context integrating own elements only, and the halo sums."""

    def __init__(self, layout: SlabLayout, mesh, ctx, group=None):
        self.layout, self.mesh, self.ctx, self.group = layout, mesh, ctx, group
        self.segs = interface_segments(layout, ctx.pattern.rowptr)  # host copy, once
        self.native = native_comm(group) if layout.world > 1 else None

    @classmethod
    def build(cls, nx: int, ny: int, nz: int, rank: int, world: int,
              etype: ElementType = ElementType.TET04, vector_size: int = 8, group=None,
              lengths=(1.0, 1.0, 1.0)) -> "SlabDomain":
        from . import _lib
        from .assembly import AssemblyContext
        from .elements import ETYPE_ID, NNODES
        from .mesh import ElementGroup, Mesh
        from .sparse import build_node_pattern

        L = SlabLayout.make(nx, ny, nz, rank, world, etype)
        dev = _lib.device()
        coords = torch.empty((L.nnode, 3), dtype=torch.float64, device=dev)
        _lib.call("fpb_grid_coords_slab", nx, ny, nz, L.kA, L.nplanes, float(lengths[0]),
                  float(lengths[1]), float(lengths[2]), coords.data_ptr(), _lib.stream())
        nlay = L.kB - L.kA
        conn = torch.empty((nlay * L.elems_per_layer, NNODES[etype]), dtype=torch.int32, device=dev)
        _lib.call("fpb_box_conn", ETYPE_ID[etype], nx, ny, nlay, conn.data_ptr(), _lib.stream())
        e0, e1 = L.own_elems
        ext = Mesh(3, coords, [ElementGroup(etype, conn)])
        pattern = build_node_pattern(ext)  # own + ghost elements
        own = Mesh(3, coords, [ElementGroup(etype, conn[e0:e1].contiguous())])
        ctx = AssemblyContext.build(own, vector_size, pattern=pattern, block_order="natural")  # windows = block ranges
        from . import assembly as _asm

        if etype is ElementType.TET04 and _asm.KUHN_MOMENTUM and SLAB_KUHN:
            # the extended slab is the generator's box (nx, ny, nlay) by
            # construction, its CSR graph the box's own: Kuhn-box kernels over
            # the own cell layers (interface planes partial, ghost planes 0)
            ctx.groups[0].kuhn = _asm.KuhnBox(nx, ny, nlay, dev, kc0=L.k0 - L.kA, kc1=L.k1 - L.kA, pattern_ok=True)
        return cls(L, own, ctx, group)

    def halo_sum_rhs(self, rhs: torch.Tensor) -> torch.Tensor:
        return halo_sum_nodes(self.layout, rhs, self.group, self.native)

    def halo_sum_matrix(self, vals: torch.Tensor, nmat: int = 1) -> torch.Tensor:
        return halo_sum_rows(self.layout, self.ctx.pattern.rowptr_d, vals, nmat, self.ctx.pattern.nnz,
                             self.group, self.segs, self.native)

    def assemble_step(self, vel, rhs, mats, rho: float = 1.0, mu: float = 1e-2, overlap: bool = True, side=None,
                      events: dict | None = None):
        return assemble_step(self, vel, rhs, mats, rho, mu, overlap, side, events)


# --------------------------------------------------------------------------
# Distributed solver plumbing ("Solver: x-halo of one plane
# per interface per SpMV, plus an allreduce of 1-3 doubles per dot")
# --------------------------------------------------------------------------

def _staged(t: torch.Tensor, group=None) -> bool:
    """gloo moves host memory: CUDA tensors are staged through the host."""
    return t.is_cuda and dist.get_backend(group) != "nccl"


def allreduce_sum_(t: torch.Tensor, group=None, native: NativeComm | None = None) -> torch.Tensor:
    """In-place SUM over ranks (NCCL on device; gloo through the host)."""
    if dist.get_world_size(group) == 1:
        return t
    if native is not None:
        return native.allreduce(t)
    if _staged(t, group):
        h = t.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def ghost_planes(layout: SlabLayout) -> list[tuple[int, int, int]]:
    """(peer, plane to send, ghost plane to receive) per neighbour: the lower
    neighbour gets my plane k0 + 1 for its ghost plane k1' + 1, the upper one
    my plane k1 - 1 for its ghost plane k0' - 1 (both are planes the sender
    computes exactly — owned rows or the shared interface)."""
    out = []
    if layout.rank > 0:
        out.append((layout.rank - 1, layout.k0 + 1, layout.kA))
    if layout.rank < layout.world - 1:
        out.append((layout.rank + 1, layout.k1 - 1, layout.kB))
    return out


def refresh_ghosts(layout: SlabLayout, x: torch.Tensor, group=None, native: NativeComm | None = None) -> torch.Tensor:
    """Overwrite the ghost node planes of a node vector with the neighbours'
    values, so every local entry holds its global value again."""
    plan = ghost_planes(layout)
    if not plan:
        return x
    if native is not None:
        segs = []
        for peer, ks, kg in plan:
            (lo, hi), (glo, _) = layout.plane_rows(ks), layout.plane_rows(kg)
            segs.append((peer, lo, glo, hi - lo))
        return native.exchange(segs, x, False)
    sends = []
    for peer, ks, _ in plan:
        lo, hi = layout.plane_rows(ks)
        sends.append((peer, x[lo:hi].contiguous()))
    recvs = _exchange(sends, group)
    for (peer, _, kg), r in zip(plan, recvs):
        lo, hi = layout.plane_rows(kg)
        x[lo:hi].copy_(r)
    return x


def bicgstab_slab(layout: SlabLayout, A, b: torch.Tensor, x0=None, tol: float = 1e-8,
                  max_iter: int | None = None, jacobi: bool = True, group=None, check_every: int = 8,
                  native: NativeComm | None = None, graph: bool = True, ws: dict | None = None):
    """Jacobi-BiCGSTAB over the z-slab decomposition (config 5).

    A is this rank's extended-slab CSR with halo-summed values (rows of
    planes k0..k1 are global rows), b a node vector consistent on every local
    plane.  Every iteration runs the one-GPU fused kernels with reductions
    restricted to the owned rows, allreduces the partial sums three times
    (||s|| rides on the (t, s), (t, t) reduction) and refreshes the ghost
    planes of v = A phat and t = A shat.
    Returns (x, SolverStats) with x consistent on every local plane; the
    iterates are those of krylov.bicgstab_solve on the global system up to
    the order of the cross-rank sums.  With the compiled NCCL path (native,
    see NativeComm) each batch of check_every iterations — kernels, ghost
    refreshes and allreduces — is captured once in a CUDA graph and
    replayed; with gloo the iterations run eagerly (host-staged exchanges
    cannot be captured).  ws (optional dict) keeps the vectors and the
    captured graph for repeated solves with the same operator object.
    """
    import numpy as np

    from . import _lib
    from .errors import SolverBreakdownError
    from .krylov import _BICG_BREAKDOWN, B_BNORM, B_IT, B_STATUS, SolverStats
    from .sparse import axpy_d, dot_d, dot_work, sell_copy, spmv_d

    n, nnz = A.n, A.nnz
    dev = b.device
    own_lo, own_hi = layout.owned_rows
    if max_iter is None:  # 10 x the global unknown count, identical on every rank
        nglob = torch.tensor([float(own_hi - own_lo)], dtype=torch.float64, device=dev)
        max_iter = 10 * int(allreduce_sum_(nglob, group, native).item())
    d = None
    if jacobi:
        # ghost-plane rows are partial locally: their diagonal comes from the
        # neighbour, so phat = p / d and shat = s / d are global on every plane
        d = refresh_ghosts(layout, A.diagonal_d(), group, native)
        own_zero = (d[own_lo:own_hi] == 0.0).any().to(torch.float64).reshape(1)
        if allreduce_sum_(own_zero, group, native).item() > 0:
            raise SolverBreakdownError("Jacobi preconditioner needs a nonzero diagonal")
    lib = _lib.load()
    cap = max(1, min(64, max_iter))
    key = (id(A), n, cap, check_every, jacobi)
    if ws is not None and ws.get("key") == key:
        # reuse the vectors (and the captured graph, which names them)
        x, r, rt, p, ph, v, sv, sh, t = ws["vecs"]
        state, hist_d = ws["state"], ws["hist"]
        state.zero_()
        hist_d.zero_()
        if d is not None:
            ws["d"].copy_(d)
            d = ws["d"]
    else:
        x, r, rt, p, ph, v, sv, sh, t = (torch.empty(n, dtype=torch.float64, device=dev) for _ in range(9))
        state = torch.zeros(int(lib.fpb_bicgstab_state_size()), dtype=torch.float64, device=dev)
        hist_d = torch.zeros(cap, dtype=torch.float64, device=dev)
        if ws is not None:
            ws.clear()
            ws.update(key=key, vecs=(x, r, rt, p, ph, v, sv, sh, t), state=state, hist=hist_d, d=d, graph=None)
    red = state[16:18]
    red3 = state[16:19]  # after K4: (t, s), (t, t) and the deferred ||s||^2
    work = dot_work()
    s = _lib.stream()
    rp, ci, va = A.rowptr_d.data_ptr(), A.colind_d.data_ptr(), A.vals_d.data_ptr()
    # the fused SpMVs on the local operator's SELL-32 copy (krylov.py)
    sell = (None, None, None, 0)
    sc = sell_copy(A)
    if sc is not None:
        A._sell = sc
        sell = sc.args()
    x0p = x0.data_ptr() if x0 is not None else None
    _lib.call("fpb_bicgstab_init", n, nnz, rp, ci, va, *sell, b.data_ptr(), x0p, x.data_ptr(), r.data_ptr(),
              rt.data_ptr(), p.data_ptr(), v.data_ptr(), state.data_ptr(), hist_d.data_ptr(), float(tol),
              own_lo, own_hi, 1, work.data_ptr(), s)
    if x0 is not None:  # r = b - A x0 is exact on computed rows only
        refresh_ghosts(layout, r, group, native)
        rt.copy_(r)
    allreduce_sum_(red, group, native)
    _lib.call("fpb_bicgstab_finish", 0, state.data_ptr(), hist_d.data_ptr(), 1, float(tol), s)
    st = state.cpu().numpy()
    if st[B_BNORM] == 0.0:
        return torch.zeros(n, dtype=torch.float64, device=dev), SolverStats(0, True, [0.0], 0.0)
    history = [float(hist_d[0].item())]
    if st[B_STATUS] == 1.0:
        return x, SolverStats(0, True, history, history[0])
    if st[B_STATUS] in _BICG_BREAKDOWN:
        raise SolverBreakdownError(f"BiCGSTAB breakdown: {_BICG_BREAKDOWN[st[B_STATUS]]}")
    args = (n, nnz, rp, ci, va, *sell, d.data_ptr() if d is not None else None, x.data_ptr(),
            r.data_ptr(), rt.data_ptr(), p.data_ptr(), ph.data_ptr(), v.data_ptr(), sv.data_ptr(), sh.data_ptr(),
            t.data_ptr(), state.data_ptr(), hist_d.data_ptr(), cap, own_lo, own_hi, 1, work.data_ptr(), s)

    def iterations(k: int) -> None:
        for _ in range(k):
            # three cross-rank reductions per iteration: K2's (r~, v); K3's
            # ||s||^2 together with K4's (t, s), (t, t); K5's ||r||^2, (r~, r)
            st_ = _lib.stream()
            a_ = args[:-1] + (st_,)
            _lib.call("fpb_bicgstab_step", 1, *a_)
            refresh_ghosts(layout, v, group, native)
            allreduce_sum_(red, group, native)
            _lib.call("fpb_bicgstab_finish", 1, state.data_ptr(), hist_d.data_ptr(), cap, 0.0, st_)
            _lib.call("fpb_bicgstab_step", 2, *a_)
            _lib.call("fpb_bicgstab_step", 3, *a_)
            refresh_ghosts(layout, t, group, native)
            allreduce_sum_(red3, group, native)
            _lib.call("fpb_bicgstab_finish", 2, state.data_ptr(), hist_d.data_ptr(), cap, 0.0, st_)
            _lib.call("fpb_bicgstab_finish", 3, state.data_ptr(), hist_d.data_ptr(), cap, 0.0, st_)
            _lib.call("fpb_bicgstab_step", 4, *a_)
            allreduce_sum_(red, group, native)
            _lib.call("fpb_bicgstab_finish", 4, state.data_ptr(), hist_d.data_ptr(), cap, 0.0, st_)

    captured = ws.get("graph") if ws is not None else None
    done = 0
    while done < max_iter:
        k = min(check_every, max_iter - done)
        if native is not None and graph and k == check_every:
            if captured is None:
                captured = torch.cuda.CUDAGraph()
                side = torch.cuda.Stream()
                side.wait_stream(torch.cuda.current_stream())
                with torch.cuda.graph(captured, stream=side):
                    iterations(k)
                torch.cuda.current_stream().wait_stream(side)
                if ws is not None:
                    ws["graph"] = captured
            captured.replay()
        else:
            iterations(k)
        st = state.cpu().numpy()
        it = int(st[B_IT])
        if it > done:
            h = hist_d.cpu().numpy()
            history.extend(float(h[i % cap]) for i in range(done + 1, it + 1))
        progressed = it > done
        done = it
        if st[B_STATUS] in _BICG_BREAKDOWN:
            raise SolverBreakdownError(f"BiCGSTAB breakdown: {_BICG_BREAKDOWN[st[B_STATUS]]}")
        if st[B_STATUS] == 1.0 or not progressed:
            break
    converged = bool(st[B_STATUS] == 1.0)
    # true residual over the owned rows, summed across ranks
    refresh_ghosts(layout, x, group, native)
    res = axpy_d(-1.0, spmv_d(A, x), b)
    rr = dot_d(res[own_lo:own_hi].contiguous(), res[own_lo:own_hi].contiguous()).reshape(1).clone()
    allreduce_sum_(rr, group, native)
    true_residual = float(np.sqrt(rr.item())) / float(st[B_BNORM])
    return x, SolverStats(done, converged, history, true_residual)


# --------------------------------------------------------------------------
# Interface-first step with the halo on a side stream (SURVEY.md 8(e):
# "assemble interface-layer elements first, launch the NCCL halo on a side
# stream, then assemble interior elements").
# --------------------------------------------------------------------------

def _step_windows(dom: "SlabDomain") -> dict:
    """Work windows of one rank's step: element blocks and nodes touching an
    interface plane (phase A) and the rest (phase B); row windows start on
    32-row slices and partition [0, n)."""
    L, g = dom.layout, dom.ctx.groups[0]
    bp = g.blocks
    n = dom.ctx.mesh.nnode
    epl, nlay = L.elems_per_layer, L.k1 - L.k0
    be, nb = bp.block_elems, bp.nblocks
    lo_b = -(-epl // be) if L.rank > 0 else 0
    hi_b = ((nlay - 1) * epl) // be if L.rank < L.world - 1 else nb
    if lo_b > hi_b:  # thin slab: everything touches an interface
        lo_b = hi_b = nb
    planes = [L.plane_rows(k) for _, k in L.interfaces()]
    A = ((L.plane_rows(L.k0)[1] + 31) // 32) * 32 if L.rank > 0 else 0
    B = (L.plane_rows(L.k1)[0] // 32) * 32 if L.rank < L.world - 1 else n
    A, B = min(A, n), max(min(B, n), 0)
    if A > B:
        A = B = n if L.rank > 0 else 0
    # nodes outside the interface planes, as contiguous windows
    cuts = sorted(planes)
    rest, at = [], 0
    for lo, hi in cuts:
        if lo > at:
            rest.append((at, lo))
        at = max(at, hi)
    if at < n:
        rest.append((at, n))
    return {"blocks_A": [(0, lo_b), (hi_b, nb)], "blocks_B": (lo_b, hi_b),
            "nodes_A": planes, "nodes_B": rest,
            "rows_A": [(0, A), (B, n)], "rows_B": (A, B)}


def assemble_step(dom: "SlabDomain", vel: torch.Tensor, rhs: torch.Tensor, mats: torch.Tensor,
                  rho: float = 1.0, mu: float = 1e-2, overlap: bool = True, side: torch.cuda.Stream | None = None,
                  events: dict | None = None):
    """One decomposed NS step: momentum RHS into rhs[n][dim] and B_x, B_y, B_z
    into mats[3 nnz], interface rows summed across ranks.  overlap = True runs
    the interface windows first and the halo exchange on `side` while the
    interior is assembled; False is the plain sequence (reference for
    tests).  Results are bitwise identical either way (owner-writes kernels,
    fixed per-row / per-node summation order).  events (optional dict) gets
    CUDA events "start", "interface_done", "halo_start", "halo_done" and
    "interior_done" for per-phase times (overlap=True only)."""
    from .assembly import KernelKind

    ctx = dom.ctx
    K = KernelKind.MOMENTUM_RHS
    if overlap and dom.layout.world > 1 and ctx.groups[0].kuhn is not None:
        return _kuhn_slab_step(dom, vel, rhs, mats, rho, mu, side, events)
    if not overlap or dom.layout.world == 1 or ctx.groups[0].kuhn is not None:
        # plain sequence (per-phase events with an empty interior phase)
        ev = None
        if events is not None:
            ev = {k: torch.cuda.Event(enable_timing=True)
                  for k in ("start", "interface_done", "halo_start", "halo_done", "interior_done")}
            events.update(ev)
            ev["start"].record()
        ctx.assemble_rhs_d(K, vel, None, rho, mu, 0.0, rhs)
        ctx.assemble_gradients_d(mats)
        if ev:
            ev["interface_done"].record()
            ev["halo_start"].record()
        dom.halo_sum_rhs(rhs)
        dom.halo_sum_matrix(mats, dom.ctx.mesh.dim)
        if ev:
            ev["halo_done"].record()
            ev["interior_done"].record()
        return rhs, mats
    w = _step_windows(dom)
    none = (0, 0)
    ev = None
    if events is not None:
        ev = {k: torch.cuda.Event(enable_timing=True)
              for k in ("start", "interface_done", "halo_start", "halo_done", "interior_done")}
        events.update(ev)
        ev["start"].record()
    # phase A: everything an interface row depends on
    for b in w["blocks_A"]:
        if b[1] > b[0]:
            ctx.assemble_rhs_d(K, vel, None, rho, mu, 0.0, rhs, {"blocks": b, "nodes": none})
    for nd in w["nodes_A"]:
        ctx.assemble_rhs_d(K, vel, None, rho, mu, 0.0, rhs, {"blocks": none, "nodes": nd})
    for r in w["rows_A"]:
        if r[1] > r[0]:
            ctx.assemble_gradients_d(mats, {"rows": r})
    # halo on the side stream, overlapping phase B
    main = torch.cuda.current_stream()
    if ev:
        ev["interface_done"].record(main)
    side = side or torch.cuda.Stream()
    side.wait_stream(main)
    with torch.cuda.stream(side):
        if ev:
            ev["halo_start"].record(side)
        dom.halo_sum_rhs(rhs)
        dom.halo_sum_matrix(mats, dom.ctx.mesh.dim)
        if ev:
            ev["halo_done"].record(side)
    # phase B: interior
    ctx.assemble_rhs_d(K, vel, None, rho, mu, 0.0, rhs, {"blocks": w["blocks_B"], "nodes": none})
    for nd in w["nodes_B"]:
        ctx.assemble_rhs_d(K, vel, None, rho, mu, 0.0, rhs, {"blocks": none, "nodes": nd})
    if w["rows_B"][1] > w["rows_B"][0]:
        ctx.assemble_gradients_d(mats, {"rows": w["rows_B"]})
    if ev:
        ev["interior_done"].record(main)
    main.wait_stream(side)
    return rhs, mats


def _kuhn_slab_step(dom, vel, rhs, mats, rho, mu, side=None, events=None):
    """Kuhn-box slab step: momentum (whole slab), the B_xyz surface rows
    (which hold the interface planes), then the halo sums on a side stream
    while the interior lines run.  Bitwise the plain sequence's result (the
    halo touches interface rows only, the lines kernel never does)."""
    from .assembly import KernelKind

    ctx = dom.ctx
    main = torch.cuda.current_stream()
    ev = None
    if events is not None:
        ev = {k: torch.cuda.Event(enable_timing=True)
              for k in ("start", "interface_done", "halo_start", "halo_done", "interior_done")}
        events.update(ev)
        ev["start"].record(main)
    # momentum on its own stream (its last wave overlaps the B_xyz kernels)
    mom = getattr(dom, "_mom_stream", None)
    if mom is None:
        mom = dom._mom_stream = torch.cuda.Stream()
    mom.wait_stream(main)
    with torch.cuda.stream(mom):
        ctx.assemble_rhs_d(KernelKind.MOMENTUM_RHS, vel, None, rho, mu, 0.0, rhs)
    ctx.assemble_gradients_d(mats, {"kuhn_part": "surface"})
    side = side or torch.cuda.Stream()
    side.wait_stream(main)
    side.wait_stream(mom)
    with torch.cuda.stream(side):
        if ev:
            ev["interface_done"].record(side)
            ev["halo_start"].record(side)
        dom.halo_sum_rhs(rhs)
        dom.halo_sum_matrix(mats, ctx.mesh.dim)
        if ev:
            ev["halo_done"].record(side)
    ctx.assemble_gradients_d(mats, {"kuhn_part": "lines"})
    if ev:
        ev["interior_done"].record(main)
    main.wait_stream(side)
    main.wait_stream(mom)
    return rhs, mats


class SlabStepGraph:
    """One decomposed NS step (assemble_step) replayed from CUDA graphs.

    With the compiled NCCL path (dom.native) the whole overlapped step —
    interface windows, the halo on the side stream, interior windows — is
    one graph (NCCL send/recv are capturable), so a step costs one launch.
    With gloo (CPU-staged exchanges, several ranks sharing a GPU) the device
    work is captured in two graphs (interface windows, interior windows) and
    the halo runs eagerly between them.  Inputs and outputs are the tensors
    given here (replay reads vel and overwrites rhs / mats in place).
    Results are bitwise those of assemble_step(overlap=False)."""

    def __init__(self, dom: "SlabDomain", vel: torch.Tensor, rhs: torch.Tensor, mats: torch.Tensor,
                 rho: float = 1.0, mu: float = 1e-2):
        from .assembly import KernelKind

        self.dom, self.vel, self.rhs, self.mats = dom, vel, rhs, mats
        self.side = torch.cuda.Stream()
        # eager warm-up: plans, scratch buffers, geometry check
        assemble_step(dom, vel, rhs, mats, rho, mu, overlap=True, side=self.side)
        torch.cuda.synchronize()
        cap = torch.cuda.Stream()
        cap.wait_stream(torch.cuda.current_stream())
        ctx, K, none = dom.ctx, KernelKind.MOMENTUM_RHS, (0, 0)
        self.whole = self.phase_a = self.phase_b = None
        if dom.native is not None or dom.layout.world == 1:
            self.whole = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.whole, stream=cap):
                assemble_step(dom, vel, rhs, mats, rho, mu, overlap=True, side=self.side)
        elif ctx.groups[0].kuhn is not None:  # Kuhn-box slab: momentum + surface rows, eager halo, lines
            self.phase_a, self.phase_b = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.phase_a, stream=cap):
                ctx.assemble_rhs_d(K, vel, None, rho, mu, 0.0, rhs)
                ctx.assemble_gradients_d(mats, {"kuhn_part": "surface"})
            with torch.cuda.graph(self.phase_b, stream=cap):
                ctx.assemble_gradients_d(mats, {"kuhn_part": "lines"})
        else:
            w = _step_windows(dom)
            self.phase_a, self.phase_b = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.phase_a, stream=cap):
                for b in w["blocks_A"]:
                    if b[1] > b[0]:
                        ctx.assemble_rhs_d(K, vel, None, rho, mu, 0.0, rhs, {"blocks": b, "nodes": none})
                for nd in w["nodes_A"]:
                    ctx.assemble_rhs_d(K, vel, None, rho, mu, 0.0, rhs, {"blocks": none, "nodes": nd})
                for r in w["rows_A"]:
                    if r[1] > r[0]:
                        ctx.assemble_gradients_d(mats, {"rows": r})
            with torch.cuda.graph(self.phase_b, stream=cap):
                ctx.assemble_rhs_d(K, vel, None, rho, mu, 0.0, rhs, {"blocks": w["blocks_B"], "nodes": none})
                for nd in w["nodes_B"]:
                    ctx.assemble_rhs_d(K, vel, None, rho, mu, 0.0, rhs, {"blocks": none, "nodes": nd})
                if w["rows_B"][1] > w["rows_B"][0]:
                    ctx.assemble_gradients_d(mats, {"rows": w["rows_B"]})
        torch.cuda.current_stream().wait_stream(cap)

    @property
    def single_graph(self) -> bool:
        return self.whole is not None

    def replay(self):
        if self.whole is not None:
            self.whole.replay()
        else:
            self.phase_a.replay()
            self.dom.halo_sum_rhs(self.rhs)
            self.dom.halo_sum_matrix(self.mats, self.dom.ctx.mesh.dim)
            if self.phase_b is not None:
                self.phase_b.replay()
        return self.rhs, self.mats
