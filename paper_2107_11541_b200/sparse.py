"""CSR matrices and the solver vector kernels on the device (sparse.py:1-130).

Drop-in for the reference's `CsrMatrix`, `build_node_pattern`, `spmv`,
`axpy`, `dot`, `norm2`: numpy arguments are copied to HBM and results come
back as numpy (the reference's return types); torch CUDA tensors stay on the
device and results are returned as CUDA tensors without a host round trip.

Storage: rowptr / colind are int32 in HBM (nnz < 2^31 is enforced), vals
float64.  The numpy views `rowptr` / `colind` are int64 like the
reference's; `vals` is a write-back host mirror of the device values.
"""

from __future__ import annotations

import ctypes
import weakref

import numpy as np
import torch
from torch.autograd.graph import increment_version

from . import _lib
from ._mirror import DeviceArray

_INT32_MAX = np.iinfo(np.int32).max


def to_device(x, dtype=torch.float64) -> tuple[torch.Tensor, bool]:
    """(contiguous CUDA tensor, came_from_host)."""
    if isinstance(x, torch.Tensor):
        if not x.is_cuda:
            return x.to(_lib.device(), dtype=dtype).contiguous(), True
        if x.dtype != dtype:
            x = x.to(dtype)
        return x.contiguous(), False
    arr = np.ascontiguousarray(x, dtype=np.float64 if dtype == torch.float64 else np.int32)
    return torch.from_numpy(arr).to(_lib.device()), True


def to_host(t: torch.Tensor) -> np.ndarray:
    """Device -> numpy through a pinned staging buffer (torch's caching host
    allocator recycles it once the returned array is dropped), so D2H runs
    at PCIe DMA speed instead of the pageable-copy path."""
    out = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    out.copy_(t, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return out.numpy()


def _to_i32(x) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        if x.numel() and int(x.max()) > _INT32_MAX:
            raise ValueError("index exceeds int32")
        return x.to(_lib.device(), dtype=torch.int32).contiguous()
    a = np.asarray(x)
    if a.size and a.max() > _INT32_MAX:
        raise ValueError("index exceeds int32")
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(_lib.device())


_VALS_STORES: dict = {}  # id(tensor) -> (weakref to the tensor, its DeviceArray)


def _vals_store(t: torch.Tensor) -> DeviceArray:
    """One write-back mirror per device value array, shared by every
    CsrMatrix over it, so `reuse=True` aliasing (assembly.py:200-207: the
    matrices returned by reusing calls share one vals array) is observable
    from numpy: `A.vals is B.vals`.  Keyed by identity (a tensor's __eq__ is
    elementwise, so no WeakKeyDictionary) and dropped with the tensor; the
    mirror holds the tensor weakly, the CsrMatrix objects strongly."""
    hit = _VALS_STORES.get(id(t))
    if hit is not None and hit[0]() is t:
        return hit[1]
    st = DeviceArray(t, weak=True)
    key = id(t)
    _VALS_STORES[key] = (weakref.ref(t), st)
    weakref.finalize(t, _VALS_STORES.pop, key, None)
    return st


class CsrMatrix:
    """n x n CSR matrix in HBM (sparse.py:20-56).  `vals` is a write-back
    host mirror (_mirror.py): reference code that edits `A.vals[...]` in
    place reaches the device before the next kernel reads the values."""

    def __init__(self, n, rowptr, colind, vals, _host=None):
        self.n = int(n)
        self.rowptr_d = rowptr if isinstance(rowptr, torch.Tensor) and rowptr.is_cuda and rowptr.dtype == torch.int32 else _to_i32(rowptr)
        self.colind_d = colind if isinstance(colind, torch.Tensor) and colind.is_cuda and colind.dtype == torch.int32 else _to_i32(colind)
        self._vals_t = to_device(vals)[0]  # owns the device values
        self._vals = _vals_store(self._vals_t)
        self._host = _host if _host is not None else {}

    @property
    def vals_d(self) -> torch.Tensor:
        return self._vals.device()

    @vals_d.setter
    def vals_d(self, t: torch.Tensor) -> None:
        self._vals_t = to_device(t)[0]
        self._vals = _vals_store(self._vals_t)

    @property
    def nnz(self) -> int:
        return int(self.colind_d.shape[0])

    @property
    def rowptr(self) -> np.ndarray:
        if "rowptr" not in self._host:
            self._host["rowptr"] = self.rowptr_d.cpu().numpy().astype(np.int64)
        return self._host["rowptr"]

    @property
    def colind(self) -> np.ndarray:
        if "colind" not in self._host:
            self._host["colind"] = self.colind_d.cpu().numpy().astype(np.int64)
        return self._host["colind"]

    @property
    def vals(self) -> np.ndarray:
        return self._vals.host()

    @vals.setter
    def vals(self, value) -> None:
        self._vals_t = to_device(value)[0]
        self._vals = _vals_store(self._vals_t)

    def copy(self) -> "CsrMatrix":
        return CsrMatrix(self.n, self.rowptr_d, self.colind_d, self.vals_d.clone(), self._host)

    def with_vals(self, vals) -> "CsrMatrix":
        return CsrMatrix(self.n, self.rowptr_d, self.colind_d, vals, self._host)

    def row_indices(self) -> np.ndarray:
        return np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.rowptr))

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.n, self.n))
        out[self.row_indices(), self.colind] = self.vals
        return out

    def diagonal_d(self) -> torch.Tensor:
        d = torch.empty(self.n, dtype=torch.float64, device=self.vals_d.device)
        _lib.call("fpb_diagonal", self.n, self.rowptr_d.data_ptr(), self.colind_d.data_ptr(),
                  self.vals_d.data_ptr(), d.data_ptr(), _lib.stream())
        return d

    def diagonal(self) -> np.ndarray:
        return to_host(self.diagonal_d())

    def row_sums_d(self) -> torch.Tensor:
        out = torch.empty(self.n, dtype=torch.float64, device=self.vals_d.device)
        _lib.call("fpb_row_sums", self.n, self.rowptr_d.data_ptr(), self.vals_d.data_ptr(),
                  out.data_ptr(), _lib.stream())
        return out


def build_node_pattern(mesh) -> CsrMatrix:
    """Zero-valued CSR graph of node adjacency plus diagonal (sparse.py:59-75)."""
    from .mesh import as_device_mesh

    mesh = as_device_mesh(mesh)
    n = mesh.nnode
    if n > _INT32_MAX:
        raise ValueError("node count exceeds int32")
    groups = [g for g in mesh.groups if g.nelem]
    ng = len(groups)
    conns = (ctypes.c_void_p * max(ng, 1))(*[g.conn_d.data_ptr() for g in groups])
    nelem = np.array([g.nelem for g in groups] or [0], dtype=np.int64)
    nn = np.array([g.conn_d.shape[1] for g in groups] or [0], dtype=np.int32)
    dev = mesh.coords_d.device
    rowptr = torch.empty(n + 1, dtype=torch.int32, device=dev)
    nnz = np.zeros(1, dtype=np.int64)
    lib = _lib.load()
    nnz_p = nnz.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
    _lib.check(lib.fpb_build_pattern(n, ng, ctypes.cast(conns, ctypes.c_void_p), nelem.ctypes.data,
                                     nn.ctypes.data, rowptr.data_ptr(), None, nnz_p, _lib.stream()),
               "fpb_build_pattern")
    colind = torch.empty(int(nnz[0]), dtype=torch.int32, device=dev)
    _lib.check(lib.fpb_build_pattern(n, ng, ctypes.cast(conns, ctypes.c_void_p), nelem.ctypes.data,
                                     nn.ctypes.data, rowptr.data_ptr(), colind.data_ptr(), nnz_p,
                                     _lib.stream()),
               "fpb_build_pattern")
    vals = torch.zeros(int(nnz[0]), dtype=torch.float64, device=dev)
    return CsrMatrix(n, rowptr, colind, vals)


# ---- vector kernels --------------------------------------------------------

_work: dict = {}


def dot_work() -> torch.Tensor:
    """Per-(device, stream) scratch for the deterministic reductions."""
    key = (torch.cuda.current_device(), _lib.stream())
    w = _work.get(key)
    if w is None:
        size = int(_lib.load().fpb_dot_work_size())
        w = torch.zeros(size, dtype=torch.float64, device=_lib.device())
        _work[key] = w
    return w


# Every operator whose SELL-32 padding stays below this factor of its nnz
# (FE matrices and the pressure operator: < 1.02) gets a SELL-32 copy for
# its SpMVs; only matrices whose row lengths vary wildly inside 32-row
# slices stay on the CSR lanes-per-row kernel (profiles/r01o_sell: SELL
# 71-103 % of HBM vs CSR 34-72 %; pressure operator 88 % vs 49 %).
SELL_MAX_PADDING = 1.5


def mark_written(t: torch.Tensor) -> None:
    """Tell torch (and the SELL copies keyed on its version counter) that a
    kernel wrote `t` in place through its raw pointer."""
    increment_version(t)


# 16-bit column offsets (col - row) when every offset fits: 10 instead of
# 12 bytes per entry streamed by the SpMV
SELL_IDX16 = True


def sell_pattern(A: CsrMatrix, max_padding: float | None = None):
    """(rowptr, colind, slice offsets, SELL column array, padded total,
    idx16) of A's pattern, cached in the pattern's host-side dict; None when
    the padding would exceed max_padding (default SELL_MAX_PADDING) x nnz."""
    limit = SELL_MAX_PADDING if max_padding is None else max_padding
    pat = A._host.get("sell_pattern")
    if pat is not None and pat[0] is A.rowptr_d and pat[1] is A.colind_d:
        if pat[3] is not None and pat[5] == (SELL_IDX16 and pat[6] < 32768):
            return pat
        if pat[3] is None and pat[4] > limit * A.nnz + 32:
            return None
    n, dev = A.n, A.vals_d.device
    ptr = torch.empty((n + 31) // 32 + 1, dtype=torch.int64, device=dev)
    total, maxoff = ctypes.c_int64(0), ctypes.c_int32(0)
    _lib.call("fpb_sell_build", n, A.rowptr_d.data_ptr(), A.colind_d.data_ptr(), None, ptr.data_ptr(), None, 0,
              None, ctypes.byref(total), ctypes.byref(maxoff), _lib.stream())
    if total.value > limit * A.nnz + 32:
        A._host["sell_pattern"] = (A.rowptr_d, A.colind_d, None, None, total.value, False, maxoff.value)
        return None
    idx16 = SELL_IDX16 and maxoff.value < 32768
    col = torch.empty(max(total.value, 1), dtype=torch.int16 if idx16 else torch.int32, device=dev)
    _lib.call("fpb_sell_build", n, A.rowptr_d.data_ptr(), A.colind_d.data_ptr(), None, ptr.data_ptr(),
              col.data_ptr(), int(idx16), None, ctypes.byref(total), None, _lib.stream())
    pat = (A.rowptr_d, A.colind_d, ptr, col, total.value, idx16, maxoff.value)
    A._host["sell_pattern"] = pat
    return pat


def sell_copy(A: CsrMatrix):
    """A new SELL copy of A, or None when its padding is too large."""
    return SellCopy(A) if sell_pattern(A) is not None else None


class SellCopy:
    """SELL-32 copy of a device CsrMatrix for the solver kernels
    (fpb_sell_build, vector.cu): slices of 32 rows, entries column-major
    inside a slice, one thread per row, the reference's per-row summation
    order (sparse.py:80-84) bit for bit.  The slice pattern is shared by
    every matrix on the same CSR pattern (cached in the pattern's host-side
    dict); values are re-copied when the matrix's value tensor is replaced
    or written (torch version counter; kernel writes call mark_written)."""

    def __init__(self, A: CsrMatrix, max_padding: float | None = None):
        pat = sell_pattern(A, max_padding)
        if pat is None:
            raise ValueError("SELL-32 padding too large for this matrix (sparse.sell_pattern)")
        # strong references to the CSR pattern: its addresses cannot be
        # recycled for another pattern while this copy lives
        self.rowptr_d, self.colind_d, self.ptr, self.col, self.total, self.idx16, _ = pat
        self.n = A.n
        self.val = torch.empty(max(self.total, 1), dtype=torch.float64, device=A.vals_d.device)
        self._src, self._ver = None, -1
        self.refresh(A)

    def same_pattern(self, A: CsrMatrix) -> bool:
        return self.rowptr_d is A.rowptr_d and self.colind_d is A.colind_d

    def current(self, A: CsrMatrix) -> bool:
        return self.same_pattern(A) and self._src is A.vals_d and self._ver == A.vals_d._version

    def refresh(self, A: CsrMatrix, force: bool = False) -> "SellCopy":
        """Copy A's values in (skipped when they are current, unless force)."""
        if force or not self.current(A):
            _lib.call("fpb_sell_build", A.n, A.rowptr_d.data_ptr(), A.colind_d.data_ptr(), A.vals_d.data_ptr(),
                      self.ptr.data_ptr(), None, 0, self.val.data_ptr(), ctypes.byref(ctypes.c_int64(0)), None,
                      _lib.stream())
            self._src, self._ver = A.vals_d, A.vals_d._version  # strong ref: the address cannot be recycled
        return self

    def args(self) -> tuple:
        """(sell_ptr, scol, sval, idx16) for the fused solver entry points."""
        return self.ptr.data_ptr(), self.col.data_ptr(), self.val.data_ptr(), int(self.idx16)

    def spmv_d(self, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        y = out if out is not None else torch.empty(self.n, dtype=torch.float64, device=x.device)
        _lib.call("fpb_spmv_sell", self.n, self.ptr.data_ptr(), self.col.data_ptr(), int(self.idx16),
                  self.val.data_ptr(), x.data_ptr(), y.data_ptr(), _lib.stream())
        return y


def _sell_for_spmv(A: CsrMatrix) -> SellCopy | None:
    """A's SELL copy (built on first use, values re-copied when they
    change), None when the padding is too large.  Every SpMV on an eligible
    operator goes through it, so repeated products are bit-identical to
    each other and to the reference's row sums."""
    sc = getattr(A, "_sell", None)
    if sc is None or not sc.same_pattern(A):
        sc = sell_copy(A)
        if sc is None:
            return None
        A._sell = sc
    return sc.refresh(A)


def spmv_d(A: CsrMatrix, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """y = A x on the device: through the SELL-32 copy (bit-identical to
    the reference's sparse.py:80-84), or the CSR lanes-per-row kernel for
    matrices whose SELL padding would be too large."""
    sc = _sell_for_spmv(A)
    if sc is not None:
        return sc.spmv_d(x, out)
    y = out if out is not None else torch.empty(A.n, dtype=torch.float64, device=x.device)
    _lib.call("fpb_spmv", A.n, A.nnz, A.rowptr_d.data_ptr(), A.colind_d.data_ptr(),
              A.vals_d.data_ptr(), x.data_ptr(), y.data_ptr(), _lib.stream())
    return y


def spmv(A: CsrMatrix, x, parallel: bool = False):
    """y = A x (sparse.py:110-116); `parallel` is accepted for API parity —
    the device kernel is always parallel and deterministic."""
    xd, host = to_device(x)
    y = spmv_d(A, xd)
    return to_host(y) if host else y


def axpy_d(alpha: float, x: torch.Tensor, y: torch.Tensor, out: torch.Tensor | None = None):
    o = out if out is not None else torch.empty_like(x)
    _lib.call("fpb_axpy", x.numel(), float(alpha), x.data_ptr(), y.data_ptr(), o.data_ptr(),
              _lib.stream())
    return o


def axpy(alpha: float, x, y):
    """out = alpha x + y, a new array (sparse.py:119-122)."""
    xd, hx = to_device(x)
    yd, hy = to_device(y)
    o = axpy_d(alpha, xd, yd)
    return to_host(o) if (hx or hy) else o


def dot_d(x: torch.Tensor, y: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """Device scalar (0-d tensor) = x . y, no host synchronisation."""
    r = out if out is not None else torch.empty((), dtype=torch.float64, device=x.device)
    _lib.call("fpb_dot", x.numel(), x.data_ptr(), y.data_ptr(), r.data_ptr(),
              dot_work().data_ptr(), _lib.stream())
    return r


def dot(x, y) -> float:
    """x . y (sparse.py:125-126); fixed-order tree, bitwise reproducible."""
    xd, _ = to_device(x)
    yd, _ = to_device(y)
    return float(dot_d(xd, yd).item())


def norm2(x) -> float:
    xd, _ = to_device(x)
    return float(np.sqrt(dot_d(xd, xd).item()))


# --------------------------------------------------------------------------
# Pressure-operator setup on the device (sparse.py:133-254; SURVEY.md 8(f)
# rank 4).  CsrMatrix in, CsrMatrix out; every array stays in HBM.
# --------------------------------------------------------------------------

def _scan_rowptr(counts: torch.Tensor) -> torch.Tensor:
    rowptr = torch.zeros(counts.numel() + 1, dtype=torch.int64, device=counts.device)
    torch.cumsum(counts.to(torch.int64), 0, out=rowptr[1:])
    if int(rowptr[-1]) >= 2**31:
        raise ValueError("result has 2^31 or more entries")
    return rowptr.to(torch.int32)


def transpose_csr(A: CsrMatrix) -> CsrMatrix:
    """A^T; each row lists its entries in ascending original row (sparse.py:133-138)."""
    dev = A.vals_d.device
    trp = torch.empty(A.n + 1, dtype=torch.int32, device=dev)
    tci = torch.empty(A.nnz, dtype=torch.int32, device=dev)
    tv = torch.empty(A.nnz, dtype=torch.float64, device=dev)
    _lib.call("fpb_csr_transpose", A.n, A.nnz, A.rowptr_d.data_ptr(), A.colind_d.data_ptr(), A.vals_d.data_ptr(),
              trp.data_ptr(), tci.data_ptr(), tv.data_ptr(), _lib.stream())
    return CsrMatrix(A.n, trp, tci, tv)


def spgemm(A: CsrMatrix, B: CsrMatrix) -> CsrMatrix:
    """A @ B with sorted columns; values summed in the reference's product
    order, so they are bitwise _spgemm_fill's (sparse.py:141-188)."""
    if A.n != B.n:
        raise ValueError("dimension mismatch")
    dev = A.vals_d.device
    counts = torch.empty(A.n, dtype=torch.int32, device=dev)
    _lib.call("fpb_spgemm_count", A.n, A.rowptr_d.data_ptr(), A.colind_d.data_ptr(), B.rowptr_d.data_ptr(),
              B.colind_d.data_ptr(), counts.data_ptr(), _lib.stream())
    rowptr = _scan_rowptr(counts)
    nnz = int(rowptr[-1])
    colind = torch.empty(nnz, dtype=torch.int32, device=dev)
    vals = torch.empty(nnz, dtype=torch.float64, device=dev)
    _lib.call("fpb_spgemm_fill", A.n, A.rowptr_d.data_ptr(), A.colind_d.data_ptr(), A.vals_d.data_ptr(),
              B.rowptr_d.data_ptr(), B.colind_d.data_ptr(), B.vals_d.data_ptr(), rowptr.data_ptr(),
              colind.data_ptr(), vals.data_ptr(), _lib.stream())
    return CsrMatrix(A.n, rowptr, colind, vals)


def normal_product(A: CsrMatrix, d) -> CsrMatrix:
    """A^T diag(d) A (sparse.py:191-194)."""
    dd = to_device(d)[0]
    scaled = torch.empty_like(A.vals_d)
    _lib.call("fpb_scale_rows", A.n, A.rowptr_d.data_ptr(), A.vals_d.data_ptr(), dd.data_ptr(),
              scaled.data_ptr(), _lib.stream())
    return spgemm(transpose_csr(A), A.with_vals(scaled))


def csr_add(A: CsrMatrix, B: CsrMatrix) -> CsrMatrix:
    """A + B over the union pattern (sparse.py:197-214)."""
    if A.n != B.n:
        raise ValueError("dimension mismatch")
    dev = A.vals_d.device
    counts = torch.empty(A.n, dtype=torch.int32, device=dev)
    _lib.call("fpb_csr_add_count", A.n, A.rowptr_d.data_ptr(), A.colind_d.data_ptr(), B.rowptr_d.data_ptr(),
              B.colind_d.data_ptr(), counts.data_ptr(), _lib.stream())
    rowptr = _scan_rowptr(counts)
    nnz = int(rowptr[-1])
    colind = torch.empty(nnz, dtype=torch.int32, device=dev)
    vals = torch.empty(nnz, dtype=torch.float64, device=dev)
    _lib.call("fpb_csr_add_fill", A.n, A.rowptr_d.data_ptr(), A.colind_d.data_ptr(), A.vals_d.data_ptr(),
              B.rowptr_d.data_ptr(), B.colind_d.data_ptr(), B.vals_d.data_ptr(), rowptr.data_ptr(),
              colind.data_ptr(), vals.data_ptr(), _lib.stream())
    return CsrMatrix(A.n, rowptr, colind, vals)


def apply_dirichlet(A: CsrMatrix, nodes, values=None, b=None):
    """Symmetric elimination of Dirichlet nodes (sparse.py:219-254): returns
    (modified copy, modified b or None); numpy b -> numpy b."""
    dev = A.vals_d.device
    nodes_d = torch.as_tensor(np.asarray(nodes, dtype=np.int64) if not isinstance(nodes, torch.Tensor) else nodes,
                              device=dev).to(torch.int64)
    flag = torch.zeros(A.n, dtype=torch.uint8, device=dev)
    flag[nodes_d] = 1
    out = torch.empty_like(A.vals_d)
    bd, host = (None, False)
    lift = None
    if b is not None:
        bd, host = to_device(b)
        bd = bd.clone()
        lift = torch.zeros(A.n, dtype=torch.float64, device=dev)
        if values is not None:
            lift[nodes_d] = to_device(values)[0]
    _lib.call("fpb_apply_dirichlet", A.n, A.rowptr_d.data_ptr(), A.colind_d.data_ptr(), A.vals_d.data_ptr(),
              flag.data_ptr(), lift.data_ptr() if lift is not None else None, out.data_ptr(),
              bd.data_ptr() if bd is not None else None, _lib.stream())
    res = CsrMatrix(A.n, A.rowptr_d, A.colind_d, out, A._host)
    if bd is None:
        return res, None
    return res, (to_host(bd) if host else bd)


def format_coo(A: CsrMatrix) -> str:
    """Triplet text dump, one `row col value` line per entry (sparse.py:257-263)."""
    rows = A.row_indices()
    return "".join(f"{i} {j} {v:.17g}\n" for i, j, v in zip(rows, A.colind, A.vals))
