"""ctypes binding of the C ABI in include/fempack_b200.h.

The shared library is built in-tree (`libfempack_b200.so` next to this file,
see `__graft_entry__.build()`).  There is no CPU fallback: if the library or a
CUDA device is missing, every compute entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os

import torch

from .errors import ConfigurationError, InvertedElementError, ScatterPatternError

LIB_PATH = os.environ.get("FPB_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "libfempack_b200.so")

FPB_OK, FPB_ECONFIG, FPB_EINVERTED, FPB_EPATTERN, FPB_ECUDA = 0, 1, 2, 3, 4

_i32, _i64, _int, _dbl, _vp = C.c_int32, C.c_int64, C.c_int, C.c_double, C.c_void_p
_pi64, _pint = C.POINTER(C.c_int64), C.POINTER(C.c_int)

# name -> (restype, argtypes); mirrors include/fempack_b200.h
SIGNATURES = {
    "fpb_last_error": (C.c_char_p, []),
    "fpb_version": (_int, []),
    "fpb_set_tuning": (_int, [C.c_char_p, _int]),
    "fpb_set_reference_element": (_int, [_int, _int, _int, _int, _vp, _vp, _vp]),
    "fpb_grid_coords": (_int, [_int, _int, _int, _int, _dbl, _dbl, _dbl, _vp, _vp]),
    "fpb_grid_coords_slab": (_int, [_int, _int, _int, _int, _int, _dbl, _dbl, _dbl, _vp, _vp]),
    "fpb_box_conn": (_int, [_int, _int, _int, _int, _vp, _vp]),
    "fpb_mixed_conn": (_int, [_int, _int, _int, _int, _vp, _vp, _vp, _vp]),
    "fpb_build_packs": (_int, [_i64, _int, _int, _vp, _vp, _vp]),
    "fpb_build_pattern": (_int, [_i32, _int, _vp, _vp, _vp, _vp, _vp, _pi64, _vp]),
    "fpb_matrix_positions": (_int, [_i64, _int, _vp, _i32, _vp, _vp, _int, _int, _vp, _vp]),
    "fpb_geometry": (_int, [_int, _i64, _int, _vp, _vp, _vp, _vp, _pi64, _pint, _vp]),
    "fpb_assemble": (_int, [_int, _int, _i64, _vp, _vp, _vp, _vp, _dbl, _dbl, _dbl, _vp, _i64, _vp, _vp]),
    "fpb_assemble_elements": (_int, [_int, _int, _i64, _int, _vp, _vp, _vp, _vp, _dbl, _dbl, _dbl, _vp, _vp]),
    "fpb_nccl_unique_id": (_int, [_vp]),
    "fpb_nccl_comm_init": (_int, [_int, _int, _vp, _int, _vp]),
    "fpb_nccl_comm_destroy": (_int, [_vp]),
    "fpb_halo_sum": (_int, [_vp, _int, _vp, _vp, _vp, _vp, _vp, _vp]),
    "fpb_halo_exchange": (_int, [_vp, _int, _vp, _vp, _vp, _vp, _int, _vp, _vp, _vp]),
    "fpb_allreduce_sum": (_int, [_vp, _vp, _i64, _vp]),
    "fpb_pair_canon_set": (_int, [_vp, _int]),
    "fpb_kuhn_mom_scratch_len": (_i64, [_int, _int, _int]),
    "fpb_assemble_rhs_hexbox": (_int, [_int, _int, _int, _int, _int, _int, _int, _vp, _vp, _vp, _i64, _dbl, _dbl, _dbl,
                                       _vp, _vp, _vp]),
    "fpb_assemble_scalar3_kuhn": (_int, [_int, _int, _int, _int, _int, _int, _vp, _vp, _vp, _i64, _dbl, _dbl, _dbl, _vp,
                                         _vp, _vp]),
    "fpb_assemble_momentum_kuhn": (_int, [_int, _int, _int, _int, _int, _int, _vp, _vp, _dbl, _dbl, _vp, _vp, _vp]),
    "fpb_pair_kuhn_table": (_int, [_vp]),
    "fpb_assemble_gradient_pairs_kuhn": (_int, [_i32, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _int, _vp, _vp]),
    "fpb_assemble_gradient_pairs_kuhn_box": (_int, [_i32, _vp, _int, _int, _vp, _vp, _i64, _int, _vp, _vp]),
    "fpb_assemble_gradient_kuhn_boundary": (_int, [_i32, _vp, _int, _int, _int, _int, _int, _vp, _vp, _i64, _int, _vp,
                                                    _vp]),
    "fpb_assemble_gradient_kuhn_lines": (_int, [_int, _int, _int, _int, _int, _vp, _vp, _i64, _int, _vp, _vp]),
    "fpb_assemble_gradient_pairs_slices": (_int, [_i32, _i32, _vp, _int, _vp, _vp, _vp, _vp, _vp, _i64, _int, _int,
                                                  _vp, _vp]),
    "fpb_assemble_gradient_pairs_rows": (_int, [_i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _int, _int, _vp, _vp]),
    "fpb_hex_canon_slots": (_int, [_vp]),
    "fpb_hex_gradient_h": (_int, [_i64, _vp, _vp, _vp, _vp]),
    "fpb_hex_gradient_rows": (_int, [_i32, _vp, _vp, _i32, _int, _int, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _i64, _int,
                                     _vp, _int, _int, _vp]),
    "fpb_incidence_build": (_int, [_i32, _i64, _int, _vp, _vp, _vp, _pi64, _vp]),
    "fpb_incidence_slots": (_int, [_i32, _int, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _pint, _vp]),
    "fpb_pack4": (_int, [_i64, _int, _vp, _vp, _vp, _vp]),
    "fpb_incidence_nodes": (_int, [_i32, _i64, _int, _vp, _vp, _vp, _vp, _vp]),
    "fpb_assemble_rows": (_int, [_int, _int, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _dbl, _dbl, _dbl,
                                 _vp, _vp, _i64, _int, _int, _vp, _vp]),
    "fpb_pair_stream_build": (_int, [_i32, _vp, _vp, _vp, _vp, _vp, _pi64, _vp]),
    "fpb_assemble_gradient_pairs": (_int, [_i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _i64, _int, _int, _vp, _vp]),
    "fpb_incidence_slots8": (_int, [_i32, _int, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _pint, _vp]),
    "fpb_assemble_rows_gl": (_int, [_int, _int, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _int, _int,
                                    _vp, _vp]),
    "fpb_csr_transpose": (_int, [_i32, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "fpb_spgemm_count": (_int, [_i32, _vp, _vp, _vp, _vp, _vp, _vp]),
    "fpb_spgemm_fill": (_int, [_i32] + [_vp] * 10),
    "fpb_scale_rows": (_int, [_i32, _vp, _vp, _vp, _vp, _vp]),
    "fpb_csr_add_count": (_int, [_i32, _vp, _vp, _vp, _vp, _vp, _vp]),
    "fpb_csr_add_fill": (_int, [_i32] + [_vp] * 10),
    "fpb_apply_dirichlet": (_int, [_i32] + [_vp] * 8),
    "fpb_robin": (_int, [_i64, _int, _int, _int] + [_vp] * 6 + [_dbl, _dbl, _vp, _vp, _vp]),
    "fpb_stage_momentum": (_int, [_i64, _int, _dbl, _dbl, _dbl] + [_vp] * 9),
    "fpb_stage_scalar": (_int, [_i64, _dbl, _dbl, _dbl] + [_vp] * 6),
    "fpb_set_rows": (_int, [_i64, _int, _vp, _vp, _vp, _vp]),
    "fpb_sub_into": (_int, [_i64, _vp, _vp, _dbl, _vp, _vp]),
    "fpb_correct": (_int, [_i64, _int, _int, _dbl] + [_vp] * 6),
    "fpb_block_elems": (_int, [_int]),
    "fpb_blocks_build": (_int, [_int, _i64, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _pi64, _pint, _vp]),
    "fpb_assemble_blocks": (_int, [_int, _int, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _dbl, _dbl, _dbl, _vp, _vp,
                                   _vp, _vp, _vp, _int, _vp, _i32, _i32, _i32, _vp, _vp, _int, _vp, _vp]),
    "fpb_assemble_blocks_scalar3": (_int, [_int, _i64, _i64, _i64, _vp, _vp, _vp, _dbl, _dbl, _dbl] + [_vp] * 5
                                    + [_int, _vp, _i32, _i32, _i32, _vp, _vp, _int, _vp, _vp]),
    "fpb_spmv": (_int, [_i32, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "fpb_sell_build": (_int, [_i32, _vp, _vp, _vp, _vp, _vp, _int, _vp, _pi64, _vp, _vp]),
    "fpb_spmv_sell": (_int, [_i32, _vp, _vp, _int, _vp, _vp, _vp, _vp]),
    "fpb_axpy": (_int, [_i64, _dbl, _vp, _vp, _vp, _vp]),
    "fpb_dot_work_size": (_i64, []),
    "fpb_dot": (_int, [_i64, _vp, _vp, _vp, _vp, _vp]),
    "fpb_diagonal": (_int, [_i32, _vp, _vp, _vp, _vp, _vp]),
    "fpb_row_sums": (_int, [_i32, _vp, _vp, _vp, _vp]),
    "fpb_pcg_init": (_int, [_i32, _i64] + [_vp] * 6 + [_int] + [_vp] * 9 + [_dbl, _vp, _vp]),
    "fpb_pcg_iterate": (_int, [_i32, _i64] + [_vp] * 6 + [_int] + [_vp] * 8 + [_i64, _int, _vp, _vp]),
    "fpb_bicgstab_state_size": (_int, []),
    "fpb_bicgstab_init": (_int, [_i32, _i64] + [_vp] * 6 + [_int] + [_vp] * 9 + [_dbl, _i64, _i64, _int, _vp, _vp]),
    "fpb_bicgstab_iterate": (_int, [_i32, _i64] + [_vp] * 6 + [_int] + [_vp] * 12 + [_i64, _int, _vp, _vp]),
    "fpb_bicgstab_step": (_int, [_int, _i32, _i64] + [_vp] * 6 + [_int] + [_vp] * 12 + [_i64, _i64, _i64, _int, _vp, _vp]),
    "fpb_bicgstab_finish": (_int, [_int, _vp, _vp, _i64, _dbl, _vp]),
}

_lib = None


def load(require_gpu: bool = True):
    """Load the library once; raise loudly when it or the GPU is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)"
            )
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        # FPB_TUNE_<KNOB>=<int> presets fpb_set_tuning(knob, value) (A/B timing aid)
        for key, val in os.environ.items():
            if key.startswith("FPB_TUNE_"):
                knob = key[len("FPB_TUNE_"):].lower()
                if lib.fpb_set_tuning(knob.encode(), int(val)) != 0:
                    raise RuntimeError(f"{key}: {lib.fpb_last_error().decode()}")
        _lib = lib
    if require_gpu and not torch.cuda.is_available():
        raise RuntimeError("fempack_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    return _lib


def last_error() -> str:
    return load(require_gpu=False).fpb_last_error().decode(errors="replace")


def check(rc: int, what: str = "") -> None:
    if rc == FPB_OK:
        return
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if rc == FPB_ECONFIG:
        raise ConfigurationError(msg)
    if rc == FPB_EPATTERN:
        raise ScatterPatternError(msg)
    if rc == FPB_EINVERTED:
        raise InvertedElementError(-1, -1, float("nan"))
    raise RuntimeError(f"CUDA failure in fempack_b200: {msg}")


def call(name: str, *args) -> None:
    lib = load()
    check(getattr(lib, name)(*args), name)


def ptr(t) -> int | None:
    """Device pointer of a tensor (None for None)."""
    if t is None:
        return None
    return t.data_ptr()


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def device() -> torch.device:
    load()
    return torch.device("cuda", torch.cuda.current_device())
