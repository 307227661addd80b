"""CPU-only checks: the C-ABI library loads and exports every declared
symbol, the ctypes table matches the header, host-side tables and config
validation behave like the reference."""

import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT, load_golden

HEADER = os.path.join(ROOT, "include", "fempack_b200.h")
LIB = os.path.join(ROOT, "paper_2107_11541_b200", "libfempack_b200.so")


def declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const char\*|int64_t|int)\s+(fpb_\w+)\s*\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "run __graft_entry__.build() first"
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (fpb_\w+)", out))
    missing = [f for f in declared_functions() if f not in exported]
    assert not missing, missing


def test_ctypes_table_covers_header():
    from paper_2107_11541_b200 import _lib

    assert sorted(_lib.SIGNATURES) == declared_functions()
    lib = _lib.load(require_gpu=False)
    assert lib.fpb_version() == 1
    assert lib.fpb_dot_work_size() > 0


def test_ctypes_argument_counts_match_header():
    """Every prototype in include/fempack_b200.h has as many parameters as
    its ctypes argtypes entry (a mismatch would only surface as a crash on
    the GPU box)."""
    from paper_2107_11541_b200 import _lib

    src = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    bad = {}
    for m in re.finditer(r"^\s*(?:const char\*|int64_t|int)\s+(fpb_\w+)\s*\(([^)]*)\)\s*;", src, re.M):
        name, params = m.group(1), m.group(2).strip()
        n = 0 if params in ("", "void") else len([p for p in params.split(",") if p.strip()])
        if len(_lib.SIGNATURES[name][1]) != n:
            bad[name] = (n, len(_lib.SIGNATURES[name][1]))
    assert not bad, bad


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_config_errors_without_gpu():
    from paper_2107_11541_b200 import _lib
    from paper_2107_11541_b200.errors import ConfigurationError

    lib = _lib.load(require_gpu=False)
    # invalid vector size is rejected before touching the device
    rc = lib.fpb_build_packs(10, 4, 3, None, None, None)
    assert rc == _lib.FPB_ECONFIG
    assert "vector_size" in _lib.last_error()
    with pytest.raises(ConfigurationError):
        _lib.check(rc)
    assert lib.fpb_set_reference_element(7, 4, 4, 3, None, None, None) == _lib.FPB_ECONFIG


def test_tables_match_reference_bitwise():
    from paper_2107_11541_b200.elements import ElementType, reference_element

    g = load_golden("elements")
    for et in ElementType:
        r = reference_element(et)
        assert r.N.tobytes() == g[f"{et.value}_N"].tobytes(), et
        assert r.dN.tobytes() == g[f"{et.value}_dN"].tobytes(), et
        assert r.weights.tobytes() == g[f"{et.value}_w"].tobytes(), et


def test_pack_config_validation():
    from paper_2107_11541_b200 import ConfigurationError, PackConfig

    for vs in (1, 2, 4, 8, 16, 32):
        PackConfig(vs)
    with pytest.raises(ConfigurationError):
        PackConfig(3)


def test_no_oracle_import_in_product():
    pkg = os.path.join(ROOT, "paper_2107_11541_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*", "", src).replace('"""', ""), f


def test_write_back_mirror_semantics():
    """_mirror.DeviceArray (CsrMatrix.vals, Mesh.coords, ElementGroup.conn):
    stable identity, host edits reach the device, device writes refresh the
    handed-out array in place (CPU tensors stand in for HBM here)."""
    import torch

    from paper_2107_11541_b200._mirror import DeviceArray

    t = torch.arange(6, dtype=torch.float64)
    m = DeviceArray(t)
    h = m.host()
    assert m.host() is h
    h[2] = 42.0                      # in-place host edit ...
    assert m.device()[2].item() == 42.0  # ... is written back before device use
    t.mul_(2.0)                      # device write (version bump) ...
    assert m.host() is h and h[2] == 84.0  # ... refreshes the same ndarray
    conn = DeviceArray(torch.zeros((2, 3), dtype=torch.int32), np.int64)
    c = conn.host()
    assert c.dtype == np.int64
    c[1, 2] = 7
    assert conn.device().dtype == torch.int32 and int(conn.device()[1, 2]) == 7


def test_large_mirror_is_read_only(monkeypatch):
    """Above WRITE_BACK_MAX the mirror is a read-only pinned download (no
    snapshot): in-place writes raise instead of vanishing."""
    import pytest
    import torch

    from paper_2107_11541_b200 import _mirror

    monkeypatch.setattr(_mirror, "WRITE_BACK_MAX", 64)
    m = _mirror.DeviceArray(torch.zeros(100, dtype=torch.float64))
    h = m.host()
    with pytest.raises(ValueError):
        h[0] = 1.0
    assert m.device().sum().item() == 0.0


def test_vals_store_does_not_keep_tensors_alive():
    """The per-tensor mirror registry (sparse._vals_store) holds its key
    weakly: dropping every CsrMatrix over a value tensor frees it."""
    import gc
    import weakref

    import torch

    from paper_2107_11541_b200 import sparse

    t = torch.zeros(8, dtype=torch.float64)
    st = sparse._vals_store(t)
    assert sparse._vals_store(t) is st
    r = weakref.ref(t)
    del t, st
    gc.collect()
    assert r() is None


@pytest.mark.parametrize("dims,own", [((4, 3, 5), None), ((37, 21, 9), None), ((6, 5, 7), (1, 6)),
                                      ((2, 2, 4), (0, 3))])
def test_kuhn_box_row_split_covers_every_row_once(dims, own):
    """KuhnBox (assembly.py): the interior-line kernel's rows (i, j in the
    interior, node planes kc0+1 .. kc1-1) and boundary_rows() partition the
    node planes kc0 .. kc1 exactly; the z-chunk model stays within the
    integrated layers.  Host logic only (torch on the CPU)."""
    import torch

    from paper_2107_11541_b200.assembly import KuhnBox

    nx, ny, nz = dims
    kc0, kc1 = own if own else (0, nz)
    kb = KuhnBox(nx, ny, nz, "cpu", kc0=kc0, kc1=kc1)
    assert 1 <= kb.kchunk <= kc1 - kc0
    br = kb.boundary_rows(torch.device("cpu")).numpy().astype(np.int64)
    assert np.all(np.diff(br) > 0)  # ascending, no duplicates
    plane = (nx + 1) * (ny + 1)
    i, j = np.arange(plane) % (nx + 1), np.arange(plane) // (nx + 1)
    inner = np.arange(plane)[(i > 0) & (i < nx) & (j > 0) & (j < ny)]
    lines = np.concatenate([inner + plane * k for k in range(kc0 + 1, kc1)]) if kc1 - kc0 > 1 else np.zeros(0, int)
    allrows = np.sort(np.concatenate([br, lines]))
    assert np.array_equal(allrows, np.arange(plane * kc0, plane * (kc1 + 1)))
