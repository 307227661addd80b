"""Global assembly on the device — drop-in for the reference's
`AssemblyContext` (assembly.py:73-270).

Same methods, arguments, return types and exceptions as the reference:

    ctx = AssemblyContext.build(mesh, vector_size=8)
    A = ctx.assemble_matrix(KernelKind.CONVECTION, "packed", velocity=u)
    r = ctx.assemble_rhs(KernelKind.MOMENTUM_RHS, "packed", u, None, rho, mu)

Both layouts ("scalar", "packed") run the same device kernels (one warp per
32-lane pack); the layout only selects which reference summation order the
result is compared against, and the reference itself holds the two to 1e-12.
numpy inputs are copied to HBM and numpy results returned; torch CUDA inputs
give CUDA results with no host round trip (the bench's and a device time
loop's fast path).  The element->CSR map, pattern, packs and geometry checks
are built once per context on the device.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from enum import Enum

import numpy as np
import torch

from . import _lib
from .elements import (ETYPE_ID, ElementType, ReferenceElement, compute_geometry, face_rule, reference_element,
                       upload_tables)
from .errors import ConfigurationError, InvertedElementError, ScatterPatternError
from .mesh import Mesh, as_device_mesh
from .packing import KERNEL_LANES, PackConfig, PackSet, pack_lanes
from .sparse import CsrMatrix, build_node_pattern, mark_written, to_device, to_host

LAYOUTS = ("scalar", "packed")


class KernelKind(Enum):
    MASS = "mass"
    LAPLACIAN = "laplacian"
    CONVECTION = "convection"
    MOMENTUM_RHS = "momentum_rhs"
    SCALAR_RHS = "scalar_rhs"

    @property
    def is_matrix(self) -> bool:
        return self in (KernelKind.MASS, KernelKind.LAPLACIAN, KernelKind.CONVECTION)


KIND_ID = {KernelKind.MASS: 0, KernelKind.LAPLACIAN: 1, KernelKind.CONVECTION: 2,
           KernelKind.MOMENTUM_RHS: 3, KernelKind.SCALAR_RHS: 4}
GRADIENT_XYZ = 5  # fused continuity kind (include/fempack_b200.h)


def positions_d(conn_d: torch.Tensor, pattern: CsrMatrix, layout: int, vs: int) -> torch.Tensor:
    """Element->CSR map on the device (assembly.py:44-52): layout 0 =
    pos[e][i][j], layout 1 = packed pos[p][i][j][vs]."""
    ne, nn = conn_d.shape
    if layout == 0:
        shape = (ne, nn, nn)
    else:
        shape = (-(-ne // vs), nn, nn, vs)
    pos = torch.empty(shape, dtype=torch.int32, device=conn_d.device)
    _lib.call("fpb_matrix_positions", ne, nn, conn_d.data_ptr(), pattern.n,
              pattern.rowptr_d.data_ptr(), pattern.colind_d.data_ptr(), layout, vs,
              pos.data_ptr(), _lib.stream())
    return pos


def matrix_positions(conn, pattern: CsrMatrix) -> np.ndarray:
    """Index into pattern.vals for every (i, j) node pair of every element;
    raises ScatterPatternError when a pair is missing (assembly.py:44-52)."""
    conn_np = np.asarray(conn)
    lead = conn_np.shape[:-1]
    flat = conn_np.reshape(-1, conn_np.shape[-1])
    cd = torch.from_numpy(np.ascontiguousarray(flat, dtype=np.int32)).to(_lib.device())
    pos = positions_d(cd, pattern, 0, 1)
    return pos.cpu().numpy().astype(np.int64).reshape(lead + pos.shape[1:])


ROW_OWNED = ("TRI03", "TET04")  # affine simplices: row-owned kernels (rows.cu)
ROW_OWNED_GAUSS = ("QUAD04", "PYR05", "HEX08")  # Gauss-loop elements: row-owned matrices (rowsq.cu)


# TET04 continuity matrices by column pairs (pairs.cu) instead of the
# incidence-accumulating row kernel; module switch for A/B measurements
GRADIENT_PAIRS = True
# TET04 continuity: slices whose rows share one pair stream read it from
# constant memory (pairs.cu); False = every slice streams its own words
PAIR_CANON = True
KUHN_STREAM = True  # ... and the Kuhn box's stream compiled in (pairs.cu k_rows_pairs_kuhn)
_PAIR_CANON_LOADED = None  # the canonical stream currently in constant memory
# HEX08 continuity with element geometry evaluated once (hexblock.cu);
# False = the per-row kernel (rowsq.cu)
HEX_ONCE = os.environ.get("FPB_HEX_ONCE", "1") != "0"
HEX_BAND = int(os.environ.get("FPB_HEX_BAND", "32"))
HEX_BOX_IDS = os.environ.get("FPB_HEX_BOX_IDS", "1") != "0"
HEX_BOX_RHS = os.environ.get("FPB_HEX_BOX_RHS", "1") != "0"  # HEX08 box: RHS kinds by z-marching cell pencils  # hex box: canonical rows' element ids computed
# element blocks of the RHS kernels over Morton-ordered elements (BlockPlan);
# slab domains keep natural order (their interface windows are block ranges)
# TET04 momentum RHS on a Kuhn box mesh by z-marching cell lines (kmom.cu)
KUHN_MOMENTUM = os.environ.get("FPB_KUHN_MOM", "1") != "0"
KUHN_KCHUNK = int(os.environ.get("FPB_KUHN_KCHUNK", "0"))  # 0 = from the grid size
# TET04 continuity on a Kuhn box: neighbour ids by offset instead of colind (pairs.cu)
KUHN_BOX_GRADIENT = os.environ.get("FPB_KUHN_BOX_GRAD", "1") != "0"
KUHN_BOX_BOUNDARY = os.environ.get("FPB_KUHN_BOX_BOUNDARY", "1") != "0"  # ... and its boundary rows
BLOCK_MORTON = os.environ.get("FPB_BLOCK_MORTON", "0") != "0"  # measured slower (profiles/r02e_mom)  # y-band of canonical hex rows (0 = natural order)


def _pair_canon(n: int, ptr: torch.Tensor, words: torch.Tensor, rowptr=None, colind=None, chunk: int = 1 << 14):
    """Find the canonical pair stream (pairs.cu): the most frequent row
    stream (64-bit polynomial hash over every row's words, then an exact
    word-by-word check of each row).  Returns a dict (setup only):
      words     the canonical stream (uint16 numpy, even length)
      kuhn      it is pairs.cu's compile-time Kuhn table and every canonical
                row has 15 entries with the diagonal at CSR offset 7: then
      rows      the canonical rows (int32, natural order) for the register
                kernel, and
      other     every other row (int32), for the row-list stream kernel;
    otherwise (constant-memory stream, whole slices only)
      cslices / oslices  fully canonical / other slices.
    None when no row stream repeats."""
    dev = ptr.device
    nsl = ptr.numel() - 1
    if nsl == 0 or n == 0:
        return None
    width = (ptr[1:] - ptr[:-1]).to(torch.int64)
    W = int(width.max())
    if W == 0:
        return None
    w16 = words.view(torch.int16)
    k = torch.arange(W, device=dev, dtype=torch.int64)
    lane = torch.arange(32, device=dev, dtype=torch.int64)
    coef = torch.randint(1, 1 << 62, (W,), generator=torch.Generator().manual_seed(1), dtype=torch.int64).to(dev)

    def streams(s0, s1):  # [s1 - s0, 32, W] int64 words of the slices' rows (0 past each slice's width)
        sl = torch.arange(s0, s1, device=dev)
        base = (ptr[sl] // 2)[:, None, None]
        kk = torch.minimum(k, (width[sl] - 1).clamp(min=0)[:, None])[:, None, :]
        idx = ((base + kk // 2) * 32 + lane[None, :, None]) * 2 + (kk & 1)
        v = w16[idx].to(torch.int64) & 0xffff
        return torch.where(k[None, None, :] < width[sl][:, None, None], v, torch.zeros_like(v))

    h = torch.cat([(streams(c, min(c + chunk, nsl)) * coef).sum(dim=2) for c in range(0, nsl, chunk)]).flatten()
    h = h[:n]
    hv, hc = torch.unique(h, return_counts=True)
    if int(hc.max()) < 2:
        return None
    top = int(torch.nonzero(h == hv[torch.argmax(hc)])[0])
    canon = streams(top // 32, top // 32 + 1)[0, top % 32]
    nz = torch.nonzero(canon).flatten()
    K = (int(nz[-1]) + 2) & ~1 if nz.numel() else 0
    if K == 0 or K > 512:
        return None
    canon_k = canon[:K]
    is_c = torch.cat([(streams(c, min(c + chunk, nsl)) == torch.cat(
        [canon_k, torch.zeros(W - K, dtype=torch.int64, device=dev)])[None, None, :]).all(dim=2).flatten()
        for c in range(0, nsl, chunk)])[:n]
    cw = canon_k.cpu().numpy().astype(np.uint16)
    out = {"words": cw, "kuhn": False}
    if rowptr is not None and KUHN_STREAM:
        tab = np.zeros(512, dtype=np.uint16)
        nk = int(_lib.load().fpb_pair_kuhn_table(tab.ctypes.data))
        if cw.size == nk and np.array_equal(cw, tab[:nk]):
            rp = rowptr.to(torch.int64)
            rows = torch.arange(n, device=dev)
            ok = (rp[1:] - rp[:-1]) == 15
            ok &= colind[(rp[:-1] + 7).clamp(max=max(int(rp[-1]) - 1, 0))].to(torch.int64) == rows
            is_c &= ok
            crow = torch.nonzero(is_c).flatten()
            grow = torch.nonzero(~is_c).flatten()
            # (precomputed row starts / neighbour lists, fpb_assemble_gradient_pairs_kuhn's
            # rlos / nbr, measured 2.21 vs 2.16 ms on config 5: the kernel reads colind)
            out.update(kuhn=True, rows=crow.to(torch.int32).contiguous(), other=grow.to(torch.int32).contiguous())
            return out
    full = torch.ones(nsl * 32, dtype=torch.bool, device=dev)
    full[:n] = is_c
    allc = full.view(nsl, 32).all(dim=1) & (torch.arange(nsl, device=dev) < n // 32)
    out.update(cslices=torch.nonzero(allc).flatten().to(torch.int32).contiguous(),
               oslices=torch.nonzero(~allc).flatten().to(torch.int32).contiguous())
    return out


class RowPlan:
    """SELL-32 node->element incidence of one affine group, plus (for
    matrices) the row-local column offsets of every incidence (rows.cu)."""

    def __init__(self, conn_d: torch.Tensor, n: int, gauss: bool = False):
        nn = int(conn_d.shape[1])
        nsl = -(-n // 32)
        self.n, self.nn, self.gauss = n, nn, gauss
        self.slice_ptr = torch.empty(nsl + 1, dtype=torch.int32, device=conn_d.device)
        ncols = np.zeros(1, dtype=np.int64)
        lib = _lib.load()
        pn = ncols.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
        args = (n, int(conn_d.shape[0]), nn, conn_d.data_ptr(), self.slice_ptr.data_ptr())
        _lib.check(lib.fpb_incidence_build(*args, None, pn, _lib.stream()), "fpb_incidence_build")
        self.ncols = int(ncols[0])
        self.inc = torch.empty(max(self.ncols, 1) * 32, dtype=torch.int32, device=conn_d.device)
        _lib.check(lib.fpb_incidence_build(*args, self.inc.data_ptr(), pn, _lib.stream()),
                   "fpb_incidence_build")
        self.incn = None
        if not gauss:
            # inline node ids per entry (int4), rotated so the row's node is
            # local node 0: one dependent load level less in the hot loop
            # (profiles/r01_rows_variants.txt) and no per-element node search
            self.incn = torch.empty(max(self.ncols, 1) * 32 * 4, dtype=torch.int32, device=conn_d.device)
            _lib.check(lib.fpb_incidence_nodes(n, self.ncols, nn, self.slice_ptr.data_ptr(),
                                               self.inc.data_ptr(), conn_d.data_ptr(), self.incn.data_ptr(),
                                               _lib.stream()), "fpb_incidence_nodes")
        self.slots = None
        self.rowcap = 0
        self.pairs = None  # TET04 continuity pair stream (pairs.cu); False = not eligible
        self.pair_canon = None  # (canonical words, canonical slices, other slices), see _pair_canon

    def ensure_pairs(self, pattern: "CsrMatrix"):
        """(pair_ptr, words) of the TET04 continuity pair stream (pairs.cu),
        built on first use; None when the rows are too long for it."""
        if self.pairs is None:
            lib = _lib.load()
            dev = self.slice_ptr.device
            ptr = torch.empty(self.slice_ptr.numel(), dtype=torch.int64, device=dev)
            total = ctypes.c_int64(0)
            rc = lib.fpb_pair_stream_build(self.n, self.slice_ptr.data_ptr(), self.slots.data_ptr(),
                                           pattern.rowptr_d.data_ptr(), ptr.data_ptr(), None,
                                           ctypes.byref(total), _lib.stream())
            words = None
            if rc == _lib.FPB_OK and self.rowcap <= 129:
                words = torch.empty(max(total.value, 2) * 32, dtype=torch.int16, device=dev)
                rc = lib.fpb_pair_stream_build(self.n, self.slice_ptr.data_ptr(), self.slots.data_ptr(),
                                               pattern.rowptr_d.data_ptr(), ptr.data_ptr(), words.data_ptr(),
                                               ctypes.byref(total), _lib.stream())
            self.pairs = (ptr, words) if rc == _lib.FPB_OK and words is not None else False
            if self.pairs and PAIR_CANON:
                self.pair_canon = _pair_canon(self.n, ptr, words, pattern.rowptr_d, pattern.colind_d)
        return self.pairs if self.pairs is not False else None

    def ensure_slots(self, conn_d: torch.Tensor, pattern: "CsrMatrix") -> None:
        if self.slots is not None:
            return
        words = 2 if self.gauss else 1  # uint2 per entry for up to 8 nodes
        slots = torch.empty(max(self.ncols, 1) * 32 * words, dtype=torch.int32, device=conn_d.device)
        cap = np.zeros(1, dtype=np.int32)
        fn = "fpb_incidence_slots8" if self.gauss else "fpb_incidence_slots"
        _lib.check(getattr(_lib.load(), fn)(
            self.n, self.nn, self.ncols, self.slice_ptr.data_ptr(), self.inc.data_ptr(),
            conn_d.data_ptr(), pattern.rowptr_d.data_ptr(), pattern.colind_d.data_ptr(),
            slots.data_ptr(), cap.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), _lib.stream()), fn)
        self.slots, self.rowcap = slots, int(cap[0])


class HexRowPlan:
    """Row lists for the HEX08 continuity kernels (hexblock.cu): the element
    pass writes each hex's 72-double H record once; the row pass reads them.
    Rows whose incidences and slot bytes equal the interior box pattern
    (hexblock.cu hb_canon_slot) go to the register kernel, with their 8
    element ids; all other rows to the generic kernel, in blocks of 32 with
    per-incidence element ids and relative-corner slot bytes (byte 0 = sign
    bits p(a) of the row's own corner, byte d = off-diagonal slot of corner
    p(a) ^ d).  Built on the device once per mesh (setup)."""

    GEN_ROWS = 32

    def __init__(self, rows: RowPlan, nelem: int, rowcap: int, coords_d: torch.Tensor | None = None):
        lib = _lib.load()
        dev = rows.slice_ptr.device
        n = rows.n
        self.nelem, self.rowcap = nelem, rowcap
        # incidences per row (dense [n, maxinc]) from the SELL-32 arrays
        slc = torch.arange(n, device=dev, dtype=torch.int64)
        sp = rows.slice_ptr.to(torch.int64)
        m0 = sp[slc >> 5]
        ln = sp[(slc >> 5) + 1] - m0
        maxinc = int(ln.max()) if n else 0
        self.maxinc = maxinc
        j = torch.arange(maxinc, device=dev, dtype=torch.int64)
        idx = (m0[:, None] + j[None, :]) * 32 + (slc & 31)[:, None]
        valid = j[None, :] < ln[:, None]
        idx = torch.where(valid, idx, torch.zeros_like(idx))
        inc = torch.where(valid, rows.inc.to(torch.int64)[idx], torch.full_like(idx, -1))
        by = rows.slots.view(torch.int64)[idx].view(torch.uint8).view(n, maxinc, 8).to(torch.int64)
        a = torch.argmax((by == 0xff).to(torch.int64), dim=2)
        pa = a ^ ((a >> 1) & 1)  # corner sign bits, elements.py corner order
        rel = torch.empty_like(by)
        rel[..., 0] = pa
        for d in range(1, 8):
            pb = pa ^ d
            rel[..., d] = torch.gather(by, 2, (pb ^ ((pb >> 1) & 1)).unsqueeze(-1)).squeeze(-1)
        words = rel.to(torch.uint8).view(torch.int64).view(n, maxinc)
        canon = torch.zeros(n, dtype=torch.bool, device=dev)
        if maxinc == 8 and os.environ.get("FPB_HEX_CANON", "1") != "0":
            tab = np.zeros(64, dtype=np.int32)
            _lib.check(lib.fpb_hex_canon_slots(tab.ctypes.data), "fpb_hex_canon_slots")
            tab = tab.reshape(8, 8)
            want = np.zeros((8, 8), dtype=np.uint8)
            for m in range(8):
                want[m, 0] = m ^ 7
                for d in range(1, 8):
                    want[m, d] = tab[m, d] - (tab[m, d] > 13)  # off-diagonal index (diagonal = 13)
            want_w = torch.as_tensor(want.view(np.int64).reshape(8), device=dev)
            canon = valid.all(dim=1) & (words == want_w[None, :]).all(dim=1)
        # row order: x-lines stay whole (a warp's lanes read consecutive
        # elements' H, one 256-byte run per plane, and a CTA's rows are mostly
        # one contiguous CSR range — Morton bricks measured 1.7x slower,
        # profiles/r02c_hex), but lines are visited in y-bands of HEX_BAND
        # lines, z inside the band: each element's 8 rows (2 lines x 2
        # planes) then fall within a few lines of each other instead of a
        # whole node plane apart, so H is read ~once from HBM, not ~1.6x
        crow = torch.nonzero(canon).flatten()
        if coords_d is not None and HEX_BAND > 0 and crow.numel():
            rk = [torch.unique(coords_d[:, d], return_inverse=True)[1].to(torch.int64) for d in range(3)]
            rx, ry, rz = (r[crow] for r in rk)
            nzr = int(rk[2].max()) + 1
            nxr = int(rk[0].max()) + 1
            key = (((ry // HEX_BAND) * nzr + rz) * HEX_BAND + ry % HEX_BAND) * nxr + rx
            crow = crow[torch.argsort(key, stable=True)]
        self.ncanon = int(crow.numel())
        self.canon_rows = crow.to(torch.int32).contiguous()
        self.canon_inc8 = inc[crow].t().contiguous().to(torch.int32) if self.ncanon else \
            torch.empty(8, dtype=torch.int32, device=dev)
        # the generator's hex box: every canonical row's 8 element ids are
        # (i-1+mx) + nx ((j-1+my) + ny (k-1+mz)) of its node (i, j, k) —
        # verified here for every canonical row; then the kernel computes
        # them instead of reading canon_inc8
        self.box = (0, 0)
        if self.ncanon and HEX_BOX_IDS:
            c8 = self.canon_inc8.to(torch.int64)
            bnx = int(c8[2, 0] - c8[0, 0])
            nxny = int(c8[4, 0] - c8[0, 0])
            if bnx >= 1 and nxny % bnx == 0 and nxny // bnx >= 1:
                bny = nxny // bnx
                r64 = crow.to(torch.int64)
                ii, jj, kk = r64 % (bnx + 1), (r64 // (bnx + 1)) % (bny + 1), r64 // ((bnx + 1) * (bny + 1))
                m = torch.arange(8, device=dev, dtype=torch.int64)[:, None]
                want = (ii - 1 + (m & 1)) + bnx * ((jj - 1 + ((m >> 1) & 1)) + bny * (kk - 1 + (m >> 2)))
                if torch.equal(want, c8):
                    self.box = (bnx, bny)
        grow = torch.nonzero(~canon).flatten()
        R = self.GEN_ROWS
        self.ngblocks = -(-int(grow.numel()) // R)
        blk = torch.full((self.ngblocks * R,), -1, dtype=torch.int64, device=dev)
        blk[: grow.numel()] = grow
        safe = blk.clamp(min=0)
        ginc = torch.where((blk >= 0)[:, None], inc[safe], torch.full_like(inc[safe], -1))
        self.gblk_rows = blk.to(torch.int32).contiguous()
        self.ginc = ginc.view(self.ngblocks, R, maxinc).permute(0, 2, 1).contiguous().to(torch.int32)
        self.gslot = words[safe].view(self.ngblocks, R, maxinc).permute(0, 2, 1).contiguous()
        self.H = None

    def run(self, conn_d, xyz4, pattern, accumulate: int, out: torch.Tensor) -> None:
        if self.H is None:  # HBM scratch, 72 planes of nelem doubles (once per mesh)
            self.H = torch.empty(max(self.nelem, 1) * 72, dtype=torch.float64, device=out.device)
        s = _lib.stream()
        _lib.call("fpb_hex_gradient_h", self.nelem, conn_d.data_ptr(), xyz4.data_ptr(), self.H.data_ptr(), s)
        _lib.call("fpb_hex_gradient_rows", self.ncanon, self.canon_rows.data_ptr(), self.canon_inc8.data_ptr(),
                  self.ngblocks, self.maxinc, self.rowcap, self.gblk_rows.data_ptr(), self.ginc.data_ptr(),
                  self.gslot.data_ptr(), self.H.data_ptr(), self.nelem, pattern.rowptr_d.data_ptr(),
                  pattern.colind_d.data_ptr(), pattern.nnz, accumulate, out.data_ptr(), self.box[0],
                  self.box[1], s)


def _centroid_morton(conn_d: torch.Tensor, coords_d: torch.Tensor) -> torch.Tensor:
    """Element permutation in Morton order of the centroids (quantised to
    2^20 levels per axis over the bounding box); setup only."""
    dim = coords_d.shape[1]
    c = coords_d.index_select(0, conn_d.reshape(-1).to(torch.int64)).reshape(conn_d.shape[0], conn_d.shape[1], dim)
    c = c.mean(dim=1)
    lo, hi = c.min(dim=0).values, c.max(dim=0).values
    q = ((c - lo) / torch.clamp(hi - lo, min=1e-300) * ((1 << 20) - 1)).to(torch.int64)
    key = torch.zeros(c.shape[0], dtype=torch.int64, device=c.device)
    for bit in range(20):
        for d in range(dim):
            key |= ((q[:, d] >> bit) & 1) << (dim * bit + d)
    return torch.argsort(key, stable=True)


class KuhnBox:
    """A TET04 group whose connectivity is exactly generate_box_mesh(TET04,
    nx, ny, nz)'s (mesh.py:258-282, cell-major, the six Kuhn tets per cell in
    permutation order) — checked element by element against the device
    generator at setup (or, for a z-slab, the extended slab box generated by
    fpb_box_conn with the own cell layers [kc0, kc1)).  Node coordinates are
    NOT assumed: the kernels read them.  The momentum RHS then runs as
    z-marching cell pencils (kmom.cu) and, when the context's CSR pattern is
    the box's own (pattern_ok), B_x, B_y, B_z as z-marching interior lines
    plus box-masked boundary rows (pairs.cu) — no per-element metadata."""

    def __init__(self, nx: int, ny: int, nz: int, dev, kc0: int = 0, kc1: int | None = None,
                 pattern_ok: bool = True, etype: "ElementType | None" = None):
        self.nx, self.ny, self.nz = nx, ny, nz
        self.etype = etype or ElementType.TET04  # TET04: Kuhn box; HEX08: one Q1 hex per cell
        self.kc0, self.kc1 = kc0, nz if kc1 is None else kc1
        self.pattern_ok = pattern_ok
        # CTAs are 32 x 8 cell pencils, one per SM; the z-chunk minimises
        # waves x layers per CTA (a chunk re-integrates one halo layer)
        pencils = -(-nx // 32) * -(-ny // 8)
        nl = self.kc1 - self.kc0

        def cost(k):
            return -(-(-(-nl // k) * pencils) // 148) * (k + (1 if k < nl else 0))

        kc = min(range(min(8, nl), min(64, nl) + 1), key=lambda k: (cost(k), k)) if nl > 0 else 1
        self.kchunk = max(1, min(KUHN_KCHUNK or kc, nl))
        self._scratch = None
        self._brows = None
        self._zero = None

    def scratch(self, dev) -> torch.Tensor:
        if self._scratch is None:  # CTA boundary partials (kmom.cu Px / Py), once
            m = int(_lib.load().fpb_kuhn_mom_scratch_len(self.nx, self.ny, self.nz))
            self._scratch = torch.empty(max(m, 1), dtype=torch.float64, device=dev)
        return self._scratch

    def boundary_rows(self, dev) -> torch.Tensor:
        """Rows the interior-line kernel does not cover: node planes kc0 and
        kc1 whole, and the x / y boundary ring of the planes between."""
        if self._brows is None:
            nx, ny = self.nx, self.ny
            plane = (nx + 1) * (ny + 1)
            ij = torch.arange(plane, device=dev, dtype=torch.int64)
            i, j = ij % (nx + 1), ij // (nx + 1)
            ring = ij[(i == 0) | (i == nx) | (j == 0) | (j == ny)]
            mid = torch.arange(self.kc0 + 1, self.kc1, device=dev, dtype=torch.int64)
            parts = [ij + plane * self.kc0]
            if mid.numel():
                parts.append((ring[None, :] + plane * mid[:, None]).reshape(-1))
            if self.kc1 > self.kc0:
                parts.append(ij + plane * self.kc1)
            self._brows = torch.cat(parts).to(torch.int32).contiguous()
        return self._brows

    def zero_ranges(self, rowptr_d: torch.Tensor) -> list:
        """CSR value ranges of the node planes outside [kc0, kc1] (a slab's
        ghost planes): no integrated cell touches them."""
        if self._zero is None:
            plane = (self.nx + 1) * (self.ny + 1)
            out = []
            if self.kc0 > 0:
                out.append((0, int(rowptr_d[plane * self.kc0])))
            if self.kc1 < self.nz:
                out.append((int(rowptr_d[plane * (self.kc1 + 1)]), int(rowptr_d[-1])))
            self._zero = out
        return self._zero

    @staticmethod
    def detect_hex(conn_d: torch.Tensor, nnode: int) -> "KuhnBox | None":
        """generate_box_mesh(HEX08, nx, ny, nz)'s connectivity (mesh.py:265-267,
        corner order (0,0,0) (1,0,0) (1,1,0) (0,1,0) then z + 1), checked element
        by element against the device generator."""
        ne = int(conn_d.shape[0])
        if ne == 0 or conn_d.ndim != 2 or conn_d.shape[1] != 8:
            return None
        c0 = [int(v) for v in conn_d[0].tolist()]
        nx = c0[3] - 1
        if nx < 1 or c0[0] != 0 or c0[1] != 1 or c0[4] % (nx + 1):
            return None
        ny = c0[4] // (nx + 1) - 1
        if ny < 1 or ne % (nx * ny):
            return None
        nz = ne // (nx * ny)
        if (nx + 1) * (ny + 1) * (nz + 1) != nnode:
            return None
        ref = torch.empty_like(conn_d)
        _lib.call("fpb_box_conn", ETYPE_ID[ElementType.HEX08], nx, ny, nz, ref.data_ptr(), _lib.stream())
        if not torch.equal(ref, conn_d):
            return None
        return KuhnBox(nx, ny, nz, conn_d.device, etype=ElementType.HEX08)

    @staticmethod
    def detect(conn_d: torch.Tensor, nnode: int) -> "KuhnBox | None":
        ne = int(conn_d.shape[0])
        if ne == 0 or conn_d.ndim != 2 or conn_d.shape[1] != 4:
            return None
        c0 = [int(v) for v in conn_d[0].tolist()]
        if c0[0] != 0 or c0[1] != 1:
            return None
        nx = c0[2] - 2
        if nx < 1 or (c0[3] - c0[2]) % (nx + 1):
            return None
        ny = (c0[3] - c0[2]) // (nx + 1) - 1
        if ny < 1 or ne % (6 * nx * ny):
            return None
        nz = ne // (6 * nx * ny)
        if (nx + 1) * (ny + 1) * (nz + 1) != nnode:
            return None
        ref = torch.empty_like(conn_d)
        _lib.call("fpb_box_conn", ETYPE_ID[ElementType.TET04], nx, ny, nz, ref.data_ptr(), _lib.stream())
        if not torch.equal(ref, conn_d):
            return None
        return KuhnBox(nx, ny, nz, conn_d.device)


class BlockPlan:
    """Element blocks of one group for the deterministic two-phase RHS
    assembly (blocks.cu): per-block distinct nodes + sorted gather slots,
    and per-node lists of block partials."""

    def __init__(self, conn_d: torch.Tensor, n: int, etype_id: int, coords_d: torch.Tensor | None = None):
        lib = _lib.load()
        ne, nn = int(conn_d.shape[0]), int(conn_d.shape[1])
        if coords_d is not None and ne > 0:
            # blocks of Morton-consecutive elements (by centroid): a block is
            # a compact 3-D brick instead of a run of cells along x, so it
            # touches fewer distinct nodes (staging) and leaves fewer
            # per-(block, node) partials (the HBM round trip of phase 2).
            # Only the blocks change — each element is still integrated once
            # and every sum runs in a fixed order (bitwise reproducible).
            conn_d = conn_d.index_select(0, _centroid_morton(conn_d, coords_d)).contiguous()
        be = int(lib.fpb_block_elems(etype_id))
        nblocks = -(-ne // be)
        dev = conn_d.device
        self.n, self.nelem = n, ne
        self.block_elems, self.nblocks = be, nblocks
        self.blk_ptr = torch.empty(nblocks + 1, dtype=torch.int32, device=dev)
        P = np.zeros(1, dtype=np.int64)
        mx = np.zeros(1, dtype=np.int32)
        pp = P.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
        pm = mx.ctypes.data_as(ctypes.POINTER(ctypes.c_int))
        s = _lib.stream()
        _lib.check(lib.fpb_blocks_build(etype_id, ne, conn_d.data_ptr(), n, self.blk_ptr.data_ptr(), None, None,
                                        None, None, None, None, pp, pm, s), "fpb_blocks_build")
        self.npartial, self.maxnu = int(P[0]), int(mx[0])
        self.blk_nodes = torch.empty(max(self.npartial, 1), dtype=torch.int32, device=dev)
        self.blk_gptr = torch.empty(self.npartial + nblocks + 1, dtype=torch.int16, device=dev)
        self.blk_gslot = torch.empty(max(nblocks * be * nn, 1), dtype=torch.int16, device=dev)
        self.blk_lidx = torch.empty(max(nblocks * be * nn, 4), dtype=torch.int16, device=dev)
        self.node_pptr = torch.empty(n + 1, dtype=torch.int32, device=dev)
        self.node_plist = torch.empty(max(self.npartial, 1), dtype=torch.int32, device=dev)
        _lib.check(lib.fpb_blocks_build(etype_id, ne, conn_d.data_ptr(), n, self.blk_ptr.data_ptr(),
                                        self.blk_nodes.data_ptr(), self.blk_gptr.data_ptr(),
                                        self.blk_gslot.data_ptr(), self.blk_lidx.data_ptr(),
                                        self.node_pptr.data_ptr(), self.node_plist.data_ptr(), pp, pm, s),
                   "fpb_blocks_build")
        self._partial: dict = {}

    def partial(self, nv: int, dev) -> torch.Tensor:
        buf = self._partial.get(nv)
        if buf is None:
            buf = self._partial[nv] = torch.empty(max(self.npartial, 1) * nv, dtype=torch.float64, device=dev)
        return buf


@dataclass
class GroupData:
    """Per element-type device state (assembly.py:55-70)."""

    ref: ReferenceElement
    conn_d: torch.Tensor
    offset: int
    packset: PackSet          # packs at the context's vector_size (parity view)
    lane_conn32: torch.Tensor  # kernel packs, 32 lanes
    pattern: CsrMatrix
    rows: RowPlan | None = None
    blocks: BlockPlan | None = None
    kuhn: "KuhnBox | None" = None  # TET04 Kuhn box (momentum RHS by cell lines)
    hexrows: "HexRowPlan | None" = None  # built on first B_xyz use
    _pos32: torch.Tensor | None = None
    _cache: dict = field(default_factory=dict)

    @property
    def nelem(self) -> int:
        return int(self.conn_d.shape[0])

    @property
    def etype_id(self) -> int:
        return ETYPE_ID[self.ref.etype]

    @property
    def conn(self) -> np.ndarray:
        if "conn" not in self._cache:
            self._cache["conn"] = self.conn_d.cpu().numpy().astype(np.int64)
        return self._cache["conn"]

    @property
    def pos32(self) -> torch.Tensor:
        """Kernel scatter map pos[p][i][j][32] (int32, built on first matrix use)."""
        if self._pos32 is None:
            self._pos32 = positions_d(self.conn_d, self.pattern, 1, KERNEL_LANES)
        return self._pos32

    @property
    def pos_scalar(self) -> np.ndarray:
        if "pos_scalar" not in self._cache:
            self._cache["pos_scalar"] = positions_d(self.conn_d, self.pattern, 0, 1).cpu().numpy().astype(np.int64)
        return self._cache["pos_scalar"]

    @property
    def pos_packed(self) -> np.ndarray:
        if "pos_packed" not in self._cache:
            vs = self.packset.vector_size
            self._cache["pos_packed"] = positions_d(self.conn_d, self.pattern, 1, vs).cpu().numpy().astype(np.int64)
        return self._cache["pos_packed"]


class AssemblyContext:
    """Mesh-bound device assembly state (assembly.py:73-270)."""

    def __init__(self, mesh: Mesh, pattern: CsrMatrix, groups: list, vector_size: int):
        self.mesh = mesh
        self.pattern = pattern
        self.groups = groups
        self.vector_size = vector_size
        # 32-byte node records for the owner-writes kernels (256-bit loads)
        n = mesh.nnode
        self.xyz4 = torch.empty((n, 4), dtype=torch.float64, device=mesh.coords_d.device)
        _lib.call("fpb_pack4", n, mesh.dim, mesh.coords_d.data_ptr(), None, self.xyz4.data_ptr(), _lib.stream())
        self._uvw4 = torch.empty((n, 4), dtype=torch.float64, device=mesh.coords_d.device)
        self._vals: dict = {}
        self._geometry: dict = {}
        self._checked = False

    @classmethod
    def build(cls, mesh, vector_size: int = 8, scatter: str = "auto",
              pattern: CsrMatrix | None = None, block_order: str = "morton") -> "AssemblyContext":
        """scatter selects the global-assembly strategy (scatter):
        "auto"   — matrices of affine simplices (TRI03, TET04): row-owned
                   kernels; RHS of every type: element blocks; matrices of
                   PYR05/HEX08/QUAD04: element kernels + FP64 reductions;
        "rows"   — row-owned kernels for every affine kind (RHS included);
        "atomic" — element kernels + FP64 reductions for everything.
        block_order: "morton" (default) builds the RHS element blocks over
            Morton-ordered elements; "natural" keeps the mesh order (slab
            domains, whose interface-first windows are block ranges).
        pattern: an externally built CSR graph that contains every element
        node pair (e.g. a slab's graph including ghost elements,
        distributed.py); default: the mesh's own node graph."""
        if scatter not in ("auto", "rows", "atomic"):
            raise ConfigurationError(f"scatter must be 'auto', 'rows' or 'atomic', got {scatter!r}")
        cfg = PackConfig(vector_size)  # validates like the reference
        mesh = as_device_mesh(mesh)
        if not mesh.is_grouped_by_type():
            raise ConfigurationError("mesh has repeated element-type blocks; renumber_by_type first")
        own_pattern = pattern is None
        if pattern is None:
            pattern = build_node_pattern(mesh)
        elif pattern.n != mesh.nnode:
            raise ConfigurationError("pattern size does not match the mesh node count")
        groups, offset = [], 0
        for g in mesh.groups:
            if not g.nelem:
                continue
            upload_tables(g.etype)
            ps = PackSet(g.etype, cfg.vector_size, g.nelem, offset, pack_lanes(g.conn_d, cfg.vector_size))
            lane32 = ps.lane_conn_d if cfg.vector_size == KERNEL_LANES else pack_lanes(g.conn_d, KERNEL_LANES)
            gd = GroupData(reference_element(g.etype), g.conn_d, offset, ps, lane32, pattern)
            if scatter == "auto":
                gd.blocks = BlockPlan(g.conn_d, mesh.nnode, ETYPE_ID[g.etype],
                                      mesh.coords_d if (block_order == "morton" and BLOCK_MORTON) else None)
                if g.etype is ElementType.TET04 and KUHN_MOMENTUM and len(mesh.groups) == 1:
                    gd.kuhn = KuhnBox.detect(g.conn_d, mesh.nnode)
                    if gd.kuhn is not None:
                        gd.kuhn.pattern_ok = own_pattern
                elif g.etype is ElementType.HEX08 and HEX_BOX_RHS and len(mesh.groups) == 1:
                    gd.kuhn = KuhnBox.detect_hex(g.conn_d, mesh.nnode)  # RHS kinds only (pencils)
            if scatter in ("auto", "rows") and g.etype.value in ROW_OWNED + ROW_OWNED_GAUSS:
                gd.rows = RowPlan(g.conn_d, mesh.nnode, gauss=g.etype.value in ROW_OWNED_GAUSS)
                gd.rows.ensure_slots(g.conn_d, pattern)  # ScatterPatternError at build time
            else:
                _ = gd.pos32  # ScatterPatternError at build time, as in the reference
            groups.append(gd)
            offset += g.nelem
        return cls(mesh, pattern, groups, cfg.vector_size)

    # -- geometry ---------------------------------------------------------

    def refresh_geometry(self, layout: str, need_grad: bool = True) -> None:
        """Validate every element's Jacobian (and tabulate detJw/gradN in the
        reference's layout) — assembly.py:121-142.  The assembly kernels
        recompute geometry in registers, so this is a check plus a parity
        view, not an input of the hot path."""
        _check_layout(layout)
        coords = self.mesh.coords_d
        for g in self.groups:
            vs = 1 if layout == "scalar" else self.vector_size
            ng, nn, dim = g.ref.ngauss, g.ref.nnodes, g.ref.dim
            npacks = -(-g.nelem // vs)
            detjw = torch.empty((npacks, ng, vs), dtype=torch.float64, device=coords.device)
            gradn = (torch.empty((npacks, dim, nn, ng, vs), dtype=torch.float64, device=coords.device)
                     if need_grad else None)
            bad_e = np.zeros(1, dtype=np.int64)
            bad_g = np.zeros(1, dtype=np.int32)
            rc = _lib.load().fpb_geometry(
                g.etype_id, g.nelem, vs, g.conn_d.data_ptr(), coords.data_ptr(), detjw.data_ptr(),
                gradn.data_ptr() if gradn is not None else None,
                bad_e.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                bad_g.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), _lib.stream())
            if rc == _lib.FPB_EINVERTED:
                _raise_inverted(g, self.mesh.coords, int(bad_e[0]), int(bad_g[0]))
            _lib.check(rc, "fpb_geometry")
            if layout == "scalar":
                detjw = detjw.reshape(g.nelem, ng)
                gradn = gradn.reshape(g.nelem, dim, nn, ng) if gradn is not None else None
            self._geometry[(id(g), layout)] = (detjw, gradn)
        self._checked = True

    def geometry(self, g: GroupData, layout: str):
        """(detJw, gradN) of one group as numpy, reference layout (assembly.py:144-148)."""
        key = (id(g), layout)
        if key not in self._geometry or self._geometry[key][1] is None:
            self.refresh_geometry(layout, need_grad=True)
        d, gr = self._geometry[key]
        return to_host(d), to_host(gr)

    def _ensure_checked(self) -> None:
        if not self._checked:
            self.refresh_geometry("packed", need_grad=False)

    # -- global assembly --------------------------------------------------

    def _vals_buffer(self, layout: str, reuse: bool, nmat: int = 1) -> torch.Tensor:
        nnz = self.pattern.nnz
        dev = self.mesh.coords_d.device
        if not reuse:
            return torch.empty(nmat * nnz, dtype=torch.float64, device=dev)
        key = (layout, nmat)
        buf = self._vals.get(key)
        if buf is None:
            buf = self._vals[key] = torch.empty(nmat * nnz, dtype=torch.float64, device=dev)
        return buf  # overwritten by the next assembly

    def _run(self, kind_id: int, vel, phi, rho: float, mu: float, kappa: float,
             out: torch.Tensor, window: dict | None = None) -> torch.Tensor:
        """Overwrite `out` with one assembly over every group.  window
        (single owner-writes group only) restricts the work: "rows" =
        (row0, row1) for row-owned matrices, "blocks" = (b0, b1) and
        "nodes" = (n0, n1) for the element-block RHS phases."""
        self._ensure_checked()
        matrix = kind_id in (0, 1, 2, GRADIENT_XYZ)
        # owner-writes paths (row-owned matrices, element-block RHS) overwrite
        # their output; anything else accumulates into a zeroed buffer
        owner = [(g.rows is not None) if matrix
                 else (g.blocks is not None or (g.rows is not None and not g.rows.gauss))
                 for g in self.groups]
        single_rows = len(self.groups) == 1 and owner[0]
        if window is not None and not single_rows:
            raise ConfigurationError("assembly windows need a single owner-writes element group")
        if not single_rows:
            out.zero_()
        n = self.mesh.nnode
        r0, r1 = window.get("rows", (0, n)) if window else (0, n)
        n0, n1 = window.get("nodes", (0, n)) if window else (0, n)
        nnz = self.pattern.nnz
        coords = self.mesh.coords_d.data_ptr()
        vp = vel.data_ptr() if vel is not None else None
        pp = phi.data_ptr() if phi is not None else None
        uvw4 = None
        # 32-byte (u, v, w, phi) records for the row-owned kernels; the
        # element-block kernels read the caller's arrays directly
        needs_records = any(own and g.rows is not None and (matrix or g.blocks is None)
                            for g, own in zip(self.groups, owner))
        if vel is not None and needs_records:
            _lib.call("fpb_pack4", self.mesh.nnode, self.mesh.dim, vp, pp, self._uvw4.data_ptr(), _lib.stream())
            uvw4 = self._uvw4.data_ptr()
        xyz4 = self.xyz4.data_ptr()
        for g, own in zip(self.groups, owner):
            if own and single_rows and window is None and g.kuhn is not None \
                    and kind_id == KIND_ID[KernelKind.MOMENTUM_RHS] and KUHN_MOMENTUM:
                kb = g.kuhn
                if kb.etype is ElementType.HEX08:
                    _lib.call("fpb_assemble_rhs_hexbox", KIND_ID[KernelKind.MOMENTUM_RHS], kb.nx, kb.ny, kb.nz,
                              kb.kc0, kb.kc1, kb.kchunk, xyz4, vp, None, 0, float(rho), float(mu), 0.0,
                              kb.scratch(out.device).data_ptr(), out.data_ptr(), _lib.stream())
                else:
                    _lib.call("fpb_assemble_momentum_kuhn", kb.nx, kb.ny, kb.nz, kb.kc0, kb.kc1, kb.kchunk, xyz4,
                              vp, float(rho), float(mu), kb.scratch(out.device).data_ptr(), out.data_ptr(),
                              _lib.stream())
            elif own and single_rows and (window is None or "kuhn_part" in window) and g.kuhn is not None \
                    and g.kuhn.etype is ElementType.TET04 and g.kuhn.pattern_ok and kind_id == GRADIENT_XYZ and KUHN_BOX_GRADIENT and g.kuhn.nx > 1 \
                    and g.kuhn.ny > 1:
                # B_x, B_y, B_z on the Kuhn box: interior lines + the surface rows
                # (boundary ring and the kc0 / kc1 planes; ghost planes zero);
                # window {"kuhn_part": "lines" | "surface"} runs one of the two
                # (the slab step sums the interface planes while the lines run)
                kb = g.kuhn
                part = window.get("kuhn_part") if window else None
                rp_ = self.pattern.rowptr_d.data_ptr()
                if part in (None, "lines"):
                    _lib.call("fpb_assemble_gradient_kuhn_lines", kb.nx, kb.ny, kb.nz, kb.kc0 + 1, kb.kc1 - 1, xyz4,
                              rp_, nnz, 0, out.data_ptr(), _lib.stream())
                if part in (None, "surface"):
                    br = kb.boundary_rows(out.device)
                    _lib.call("fpb_assemble_gradient_kuhn_boundary", int(br.numel()), br.data_ptr(), kb.nx, kb.ny,
                              kb.nz, kb.kc0, kb.kc1, xyz4, rp_, nnz, 0, out.data_ptr(), _lib.stream())
                    for a0, a1 in kb.zero_ranges(self.pattern.rowptr_d):
                        for m in range(3):
                            out[m * nnz + a0:m * nnz + a1].zero_()
            elif own and not matrix and g.blocks is not None:
                bp = g.blocks
                nv = self.mesh.dim if kind_id == KIND_ID[KernelKind.MOMENTUM_RHS] else 1
                b0, b1 = window.get("blocks", (0, bp.nblocks)) if window else (0, bp.nblocks)
                _lib.call("fpb_assemble_blocks", kind_id, g.etype_id, g.nelem, b0, b1, xyz4, uvw4, vp, pp,
                          float(rho), float(mu), float(kappa), bp.blk_ptr.data_ptr(),
                          bp.blk_nodes.data_ptr(), bp.blk_gptr.data_ptr(), bp.blk_gslot.data_ptr(),
                          bp.blk_lidx.data_ptr(), bp.maxnu,
                          bp.partial(nv, out.device).data_ptr(), n, n0, n1, bp.node_pptr.data_ptr(),
                          bp.node_plist.data_ptr(), 0 if single_rows else 1, out.data_ptr(), _lib.stream())
            elif own and g.rows.gauss and kind_id == GRADIENT_XYZ and window is None and HEX_ONCE \
                    and g.etype_id == ETYPE_ID[ElementType.HEX08]:
                self._hexrows(g).run(g.conn_d, self.xyz4, self.pattern, 0 if single_rows else 1, out)
            elif own and g.rows.gauss:
                r = g.rows
                _lib.call("fpb_assemble_rows_gl", kind_id, g.etype_id, r.n, r0, r1, r.slice_ptr.data_ptr(),
                          r.inc.data_ptr(), g.conn_d.data_ptr(), r.slots.data_ptr(), xyz4, uvw4,
                          self.pattern.rowptr_d.data_ptr(), self.pattern.colind_d.data_ptr(), nnz, r.rowcap,
                          0 if single_rows else 1, out.data_ptr(), _lib.stream())
            elif own and kind_id == GRADIENT_XYZ and GRADIENT_PAIRS and g.etype_id == ETYPE_ID[ElementType.TET04] \
                    and g.rows.ensure_pairs(self.pattern) is not None:
                r = g.rows
                acc = 0 if single_rows else 1
                if r.pair_canon is not None and window is None:
                    pc = r.pair_canon
                    rp_, ci_ = self.pattern.rowptr_d.data_ptr(), self.pattern.colind_d.data_ptr()
                    kb_ = g.kuhn
                    box = (pc["kuhn"] and kb_ is not None and KUHN_BOX_GRADIENT and kb_.nx > 1 and kb_.ny > 1
                           and int(pc["rows"].numel()) == (kb_.nx - 1) * (kb_.ny - 1) * (kb_.nz - 1))
                    if box:  # canonical rows = the interior nodes: row and neighbour ids computed
                        _lib.call("fpb_assemble_gradient_pairs_kuhn_box", int(pc["rows"].numel()),
                                  pc["rows"].data_ptr(), g.kuhn.nx, g.kuhn.ny, xyz4, rp_, nnz, acc, out.data_ptr(),
                                  _lib.stream())
                        if KUHN_BOX_BOUNDARY:  # boundary rows: the interior stream masked by the box
                            _lib.call("fpb_assemble_gradient_kuhn_boundary", int(pc["other"].numel()),
                                      pc["other"].data_ptr(), kb_.nx, kb_.ny, kb_.nz, 0, kb_.nz, xyz4, rp_, nnz,
                                      acc, out.data_ptr(), _lib.stream())
                        else:
                            _lib.call("fpb_assemble_gradient_pairs_rows", r.n, int(pc["other"].numel()),
                                      pc["other"].data_ptr(), r.pairs[0].data_ptr(), r.pairs[1].data_ptr(), xyz4,
                                      rp_, ci_, nnz, r.rowcap, acc, out.data_ptr(), _lib.stream())
                    elif pc["kuhn"]:  # compile-time stream, edge vectors in registers; the rest masked
                        _lib.call("fpb_assemble_gradient_pairs_kuhn", int(pc["rows"].numel()), pc["rows"].data_ptr(),
                                  None, None, xyz4, rp_, ci_, nnz, acc, out.data_ptr(), _lib.stream())
                        _lib.call("fpb_assemble_gradient_pairs_rows", r.n, int(pc["other"].numel()),
                                  pc["other"].data_ptr(), r.pairs[0].data_ptr(), r.pairs[1].data_ptr(), xyz4, rp_,
                                  ci_, nnz, r.rowcap, acc, out.data_ptr(), _lib.stream())
                    else:
                        cw = pc["words"]
                        global _PAIR_CANON_LOADED
                        if _PAIR_CANON_LOADED is not cw:  # constant memory: upload when the stream changes
                            torch.cuda.current_stream().synchronize()
                            _lib.call("fpb_pair_canon_set", cw.ctypes.data, int(cw.size))
                            _PAIR_CANON_LOADED = cw
                        for sl, clen in ((pc["cslices"], int(cw.size)), (pc["oslices"], 0)):
                            _lib.call("fpb_assemble_gradient_pairs_slices", r.n, int(sl.numel()), sl.data_ptr(),
                                      clen, r.pairs[0].data_ptr(), r.pairs[1].data_ptr(), xyz4, rp_, ci_, nnz,
                                      r.rowcap, acc, out.data_ptr(), _lib.stream())
                else:
                    _lib.call("fpb_assemble_gradient_pairs", r.n, r0, r1, r.pairs[0].data_ptr(),
                              r.pairs[1].data_ptr(), xyz4, self.pattern.rowptr_d.data_ptr(),
                              self.pattern.colind_d.data_ptr(), nnz, r.rowcap, acc, out.data_ptr(), _lib.stream())
            elif own:
                r = g.rows
                _lib.call("fpb_assemble_rows", kind_id, g.etype_id, r.n, r0, r1, r.slice_ptr.data_ptr(),
                          r.inc.data_ptr(), g.conn_d.data_ptr(),
                          r.incn.data_ptr(),
                          r.slots.data_ptr() if matrix else None, xyz4, uvw4,
                          float(rho), float(mu), float(kappa),
                          self.pattern.rowptr_d.data_ptr(), self.pattern.colind_d.data_ptr(), nnz, r.rowcap,
                          0 if single_rows else 1,
                          out.data_ptr(), _lib.stream())
            else:
                _lib.call("fpb_assemble", kind_id, g.etype_id, g.nelem, g.lane_conn32.data_ptr(),
                          coords, vp, pp, float(rho), float(mu), float(kappa),
                          g.pos32.data_ptr() if matrix else None, nnz, out.data_ptr(), _lib.stream())
        mark_written(out)
        return out

    def _hexrows(self, g: GroupData) -> HexRowPlan:
        if g.hexrows is None:
            g.hexrows = HexRowPlan(g.rows, g.nelem, g.rows.rowcap, self.mesh.coords_d)
        return g.hexrows

    def assemble_matrix_d(self, kind: KernelKind, velocity_d: torch.Tensor | None,
                          out: torch.Tensor) -> torch.Tensor:
        """Device fast path: overwrite out[nnz] with the global `kind` matrix values."""
        vel = velocity_d if kind is KernelKind.CONVECTION else None
        return self._run(KIND_ID[kind], vel, None, 1.0, 0.0, 0.0, out)

    def assemble_gradients_d(self, out: torch.Tensor, window: dict | None = None) -> torch.Tensor:
        """Fused continuity assembly: out[k*nnz:(k+1)*nnz] = B_k, k < dim,
        where B_k = CONVECTION with unit velocity e_k (timeloop.py:159-171)."""
        return self._run(GRADIENT_XYZ, None, None, 1.0, 0.0, 0.0, out, window)

    def assemble_rhs_d(self, kind: KernelKind, velocity_d: torch.Tensor, scalar_d, rho: float,
                       mu: float, kappa: float, out: torch.Tensor, window: dict | None = None) -> torch.Tensor:
        """Device fast path: overwrite out with the global RHS."""
        vel = velocity_d.contiguous() if velocity_d is not None else None
        phi = scalar_d.contiguous() if scalar_d is not None else None
        return self._run(KIND_ID[kind], vel, phi, rho, mu, kappa, out, window)

    def assemble_ns_d(self, velocity_d: torch.Tensor, rho: float, mu: float, rhs: torch.Tensor,
                      mats: torch.Tensor) -> tuple:
        """One NS assembly step on the device: the momentum RHS into rhs
        (n, dim) and the continuity matrices B_x, B_y, B_z into mats (3 nnz),
        the two on separate streams — they share no data, so the momentum
        kernel's last wave overlaps the continuity kernels.  Joined before
        returning (stream-ordered on the current stream); results equal the
        two calls in sequence bitwise."""
        main = torch.cuda.current_stream()
        side = getattr(self, "_ns_side", None)
        if side is None:
            side = self._ns_side = torch.cuda.Stream()
        side.wait_stream(main)
        with torch.cuda.stream(side):
            self.assemble_rhs_d(KernelKind.MOMENTUM_RHS, velocity_d, None, rho, mu, 0.0, rhs)
        self.assemble_gradients_d(mats)
        main.wait_stream(side)
        return rhs, mats

    def assemble_scalar_rhs3_d(self, velocity_d: torch.Tensor, phi3_d: torch.Tensor, kappas, out3: torch.Tensor,
                               window: dict | None = None) -> torch.Tensor:
        """Three SCALAR_RHS sharing one velocity (enthalpy + two species,
        timeloop.py:76-79, :361-363) in one element-block pass:
        out3[f] = assemble_rhs(SCALAR_RHS, velocity, phi3[f], kappa=kappas[f])
        to rounding.  phi3 / out3 are (3, n) CUDA tensors; a mesh that is
        not a single element-block group falls back to three passes."""
        self._ensure_checked()
        vel = velocity_d.contiguous()
        phi3 = phi3_d.contiguous()
        k0, k1, k2 = (float(k) for k in kappas)
        n = self.mesh.nnode
        if phi3.shape != (3, n) or out3.shape != (3, n) or not out3.is_contiguous():
            raise ConfigurationError("phi3 and out3 must be (3, nnode); out3 contiguous")
        g = self.groups[0] if len(self.groups) == 1 else None
        if g is not None and g.kuhn is not None and window is None and KUHN_MOMENTUM:
            kb = g.kuhn  # Kuhn / hex box: z-marching cell pencils (kmom.cu), three fields per node
            if kb.etype is ElementType.HEX08:
                _lib.call("fpb_assemble_rhs_hexbox", 101, kb.nx, kb.ny, kb.nz, kb.kc0, kb.kc1, kb.kchunk,
                          self.xyz4.data_ptr(), vel.data_ptr(), phi3.data_ptr(), n, k0, k1, k2,
                          kb.scratch(out3.device).data_ptr(), out3.data_ptr(), _lib.stream())
            else:
                _lib.call("fpb_assemble_scalar3_kuhn", kb.nx, kb.ny, kb.nz, kb.kc0, kb.kc1, kb.kchunk,
                          self.xyz4.data_ptr(), vel.data_ptr(), phi3.data_ptr(), n, k0, k1, k2,
                          kb.scratch(out3.device).data_ptr(), out3.data_ptr(), _lib.stream())
            mark_written(out3)
            return out3
        if g is None or g.blocks is None:
            if window is not None:
                raise ConfigurationError("assembly windows need a single owner-writes element group")
            for f, kap in enumerate((k0, k1, k2)):
                self._run(KIND_ID[KernelKind.SCALAR_RHS], vel, phi3[f], 1.0, 0.0, kap, out3[f])
            return out3
        bp = g.blocks
        b0, b1 = window.get("blocks", (0, bp.nblocks)) if window else (0, bp.nblocks)
        n0, n1 = window.get("nodes", (0, n)) if window else (0, n)
        _lib.call("fpb_assemble_blocks_scalar3", g.etype_id, g.nelem, b0, b1, self.xyz4.data_ptr(), vel.data_ptr(),
                  phi3.data_ptr(), k0, k1, k2, bp.blk_ptr.data_ptr(), bp.blk_nodes.data_ptr(),
                  bp.blk_gptr.data_ptr(), bp.blk_gslot.data_ptr(), bp.blk_lidx.data_ptr(), bp.maxnu,
                  bp.partial(3, out3.device).data_ptr(), n, n0, n1, bp.node_pptr.data_ptr(),
                  bp.node_plist.data_ptr(), 0, out3.data_ptr(), _lib.stream())
        mark_written(out3)
        return out3

    def assemble_matrix(self, kind: KernelKind, layout: str = "packed", velocity=None,
                        reuse: bool = False) -> CsrMatrix:
        """Global matrix sharing the context pattern (assembly.py:209-233).
        reuse=True returns a context-owned value buffer that the next reusing
        call for the same layout overwrites."""
        if not kind.is_matrix:
            raise ConfigurationError(f"{kind.name} does not assemble a matrix")
        _check_layout(layout)
        _check_fields(kind, velocity, None)
        vel = self._field(velocity, self.mesh.dim) if velocity is not None else None
        vals = self._vals_buffer(layout, reuse)
        self.assemble_matrix_d(kind, vel if kind is KernelKind.CONVECTION else None, vals)
        return self.pattern.with_vals(vals)

    def assemble_rhs(self, kind: KernelKind, layout: str = "packed", velocity=None, scalar=None,
                     rho: float = 1.0, mu: float = 0.0, kappa: float = 0.0):
        """Global RHS (assembly.py:235-270): (nnode, dim) for MOMENTUM_RHS,
        (nnode,) for SCALAR_RHS; numpy in -> numpy out."""
        if kind.is_matrix:
            raise ConfigurationError(f"{kind.name} does not assemble an RHS")
        _check_layout(layout)
        _check_fields(kind, velocity, scalar)
        host = not (isinstance(velocity, torch.Tensor) and velocity.is_cuda)
        n, dim = self.mesh.nnode, self.mesh.dim
        vel = self._field(velocity, dim)
        phi = self._field(scalar, 1) if kind is KernelKind.SCALAR_RHS else None
        shape = (n, dim) if kind is KernelKind.MOMENTUM_RHS else (n,)
        out = torch.empty(shape, dtype=torch.float64, device=vel.device)
        self.assemble_rhs_d(kind, vel, phi, rho, mu, kappa, out)
        return to_host(out) if host else out

    def _field(self, x, width: int) -> torch.Tensor:
        t, _ = to_device(x)
        n = self.mesh.nnode
        want = (n,) if width == 1 else (n, width)
        if tuple(t.shape) != want:
            raise ConfigurationError(f"field shape {tuple(t.shape)} != {want}")
        return t


def _check_layout(layout: str) -> None:
    if layout not in LAYOUTS:
        raise ConfigurationError(f"layout must be one of {LAYOUTS}, got {layout!r}")


def _check_fields(kind, velocity, scalar) -> None:
    if kind is KernelKind.MASS or kind is KernelKind.LAPLACIAN:
        return
    if velocity is None:
        raise ConfigurationError(f"{kind.name} needs a velocity field")
    if kind is KernelKind.SCALAR_RHS and scalar is None:
        raise ConfigurationError("SCALAR_RHS needs a scalar field")


def _raise_inverted(g: GroupData, coords: np.ndarray, elem: int, gauss: int):
    """InvertedElementError with the reference's (element, gauss point, det)
    (assembly.py:278-284); det is re-evaluated on the host for the message."""
    x = coords[g.conn[elem]]
    det = float("nan")
    for ig in range(g.ref.ngauss):
        dj = float(np.linalg.det(x.T @ g.ref.dN[:, :, ig].T))
        if dj <= 0.0:
            gauss, det = ig, dj
            break
    raise InvertedElementError(g.offset + elem, gauss, det)


def _element_local(kind: KernelKind, ref: ReferenceElement, lane_conn_d: torch.Tensor, vs: int, nelem: int,
                   coords, velocity, scalar, rho, mu, kappa) -> np.ndarray:
    """Shared body of assemble_element_scalar / _packed: geometry check
    (first bad (element, gauss) in the reference's scan order), then the
    element-local kernel (`fpb_assemble_elements`) into a zeroed output."""
    _check_fields(kind, velocity, scalar)
    upload_tables(ref.etype)
    dev = _lib.device()
    nn, dim, ng = ref.nnodes, ref.dim, ref.ngauss
    npacks = int(lane_conn_d.shape[0])
    xd, _ = to_device(coords)
    if xd.ndim != 2 or xd.shape[1] != dim:
        raise ConfigurationError(f"coords must have shape (nnode, {dim})")
    conn_e = lane_conn_d.permute(0, 2, 1).reshape(-1, nn)[:nelem].contiguous()
    bad_e = np.zeros(1, dtype=np.int64)
    bad_g = np.zeros(1, dtype=np.int32)
    detjw = torch.empty((max(npacks, 1), ng, vs), dtype=torch.float64, device=dev)
    rc = _lib.load().fpb_geometry(ETYPE_ID[ref.etype], nelem, vs, conn_e.data_ptr(), xd.data_ptr(),
                                  detjw.data_ptr(), None, bad_e.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                  bad_g.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), _lib.stream())
    if rc == _lib.FPB_EINVERTED:
        bad, ig = int(bad_e[0]), int(bad_g[0])
        x = to_host(xd)[to_host(conn_e[bad]).astype(np.int64)]
        try:
            compute_geometry(ref, x)
        except InvertedElementError as err:
            raise InvertedElementError(bad, err.gauss_point, err.det) from None
        raise InvertedElementError(bad, ig, float("nan"))
    _lib.check(rc, "fpb_geometry")
    vel = to_device(velocity)[0] if velocity is not None and kind is not KernelKind.MASS \
        and kind is not KernelKind.LAPLACIAN else None
    phi = to_device(scalar)[0] if kind is KernelKind.SCALAR_RHS else None
    if kind.is_matrix:
        shape = (npacks, nn, nn, vs)
    elif kind is KernelKind.MOMENTUM_RHS:
        shape = (npacks, nn, dim, vs)
    else:
        shape = (npacks, nn, vs)
    out = torch.zeros(shape, dtype=torch.float64, device=dev)
    _lib.call("fpb_assemble_elements", KIND_ID[kind], ETYPE_ID[ref.etype], nelem, vs, lane_conn_d.data_ptr(),
              xd.data_ptr(), _lib.ptr(vel), _lib.ptr(phi), float(rho), float(mu), float(kappa), out.data_ptr(),
              _lib.stream())
    return to_host(out)


def assemble_element_scalar(kind: KernelKind, ref: ReferenceElement, conn, coords, velocity=None, scalar=None,
                            rho: float = 1.0, mu: float = 0.0, kappa: float = 0.0) -> np.ndarray:
    """Element-local contributions of one connectivity block
    (assembly.py:296-339): (nelem, nn, nn) for matrix kinds, (nelem, nn, dim)
    for MOMENTUM_RHS, (nelem, nn) for SCALAR_RHS — one device thread per
    element, no scatter."""
    conn_d = _to_conn_d(conn)
    ne, nn = conn_d.shape
    if nn != ref.nnodes:
        raise ConfigurationError(f"connectivity has {nn} nodes per element, {ref.etype.value} needs {ref.nnodes}")
    out = _element_local(kind, ref, conn_d.reshape(ne, nn, 1), 1, ne, coords, velocity, scalar, rho, mu, kappa)
    return out.reshape(out.shape[:-1])


def assemble_element_packed(kind: KernelKind, ref: ReferenceElement, packset: PackSet, coords, velocity=None,
                            scalar=None, rho: float = 1.0, mu: float = 0.0, kappa: float = 0.0) -> np.ndarray:
    """Lane-major element contributions, lane axis last (assembly.py:342-380);
    padded lanes are exact zeros."""
    return _element_local(kind, ref, packset.lane_conn_d, packset.vector_size, packset.nelem, coords, velocity,
                          scalar, rho, mu, kappa)


def _to_conn_d(conn) -> torch.Tensor:
    if isinstance(conn, torch.Tensor):
        return conn.to(_lib.device(), dtype=torch.int32).contiguous()
    a = np.asarray(conn)
    if a.ndim != 2:
        raise ConfigurationError("connectivity must be (nelem, nn)")
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.int32), device=_lib.device())


def gradient_matrices(ctx: AssemblyContext, layout: str = "packed") -> list[CsrMatrix]:
    """B_k with entries int(N_i dN_j/dx_k), one fused device pass
    (timeloop.py:159-171)."""
    _check_layout(layout)
    dim, nnz = ctx.mesh.dim, ctx.pattern.nnz
    out = torch.empty(dim * nnz, dtype=torch.float64, device=ctx.mesh.coords_d.device)
    ctx.assemble_gradients_d(out)
    return [ctx.pattern.with_vals(out[k * nnz:(k + 1) * nnz]) for k in range(dim)]


def lumped_mass(ctx: AssemblyContext, layout: str = "packed") -> np.ndarray:
    """Row-sum lumped mass (timeloop.py:174-181)."""
    M = ctx.assemble_matrix(KernelKind.MASS, layout)
    lumped = to_host(M.row_sums_d())
    if not (lumped > 0.0).all():
        raise ConfigurationError("lumped mass has non-positive entries")
    return lumped


# --------------------------------------------------------------------------
# Robin boundary assembly (assembly.py:383-411)
# --------------------------------------------------------------------------

def assemble_boundary_d(mesh, pattern: CsrMatrix, alpha: float = 0.0, beta: float = 0.0):
    """Device Robin structures: (vals[nnz], rhs[n]) as CUDA tensors."""
    mesh = as_device_mesh(mesh)
    dev = mesh.coords_d.device
    vals = torch.zeros(pattern.nnz, dtype=torch.float64, device=dev)
    rhs = torch.zeros(pattern.n, dtype=torch.float64, device=dev)
    if alpha == 0.0 and beta == 0.0:
        return vals, rhs
    for fg in mesh.boundary:
        fr = face_rule(fg.nnodes)
        ng = fr.ngauss
        Nd, dNd, wd = (torch.as_tensor(np.array(a, dtype=np.float64), device=dev) for a in (fr.N, fr.dN, fr.weights))
        conn = fg.conn_d.to(torch.int32).contiguous()
        pos = positions_d(conn, pattern, 0, 1) if alpha != 0.0 else None
        _lib.call("fpb_robin", fg.nfaces, fg.nnodes, ng, mesh.dim, conn.data_ptr(), mesh.coords_d.data_ptr(),
                  Nd.data_ptr(), dNd.data_ptr(), wd.data_ptr(), pos.data_ptr() if pos is not None else None,
                  float(alpha), float(beta), vals.data_ptr(), rhs.data_ptr(), _lib.stream())
        mark_written(vals)
        mark_written(rhs)
    return vals, rhs


def assemble_boundary(mesh, pattern: CsrMatrix, alpha: float = 0.0, beta: float = 0.0):
    """alpha * face mass and beta * face load (assembly.py:383-411): returns
    (CsrMatrix sharing the pattern, numpy rhs)."""
    vals, rhs = assemble_boundary_d(mesh, pattern, alpha, beta)
    return pattern.with_vals(vals), to_host(rhs)
