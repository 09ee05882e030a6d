"""ctypes binding of the C-ABI in include/featlsq_b200.h.

The library is built in-tree (`paper_2506_17626_b200/build.py`) and loaded
from this directory only. There is no fallback: if the .so is missing or
no CUDA device is present, the product path raises.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import (DegenerateSubdomainError, DeviceError, DivergenceError,
                     InvalidInputError, SingularFactorError)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FEATLSQ_LIB") or os.path.join(HERE, "libfeatlsq_b200.so")

FL_OK, FL_ERR_INVALID, FL_ERR_DEGENERATE, FL_ERR_DIVERGENCE, FL_ERR_SINGULAR, FL_ERR_CUDA = \
    0, -1, -2, -3, -4, -5
FL_ROW_TILE, FL_COL_TILE = 256, 32
FL_AS_MAX_K = 96
FL_LSQR_SPLIT_MAX = 4
FL_TBUILD_ROWS = 16

p_d, p_i32, p_i64, p_u32 = (C.POINTER(C.c_double), C.POINTER(C.c_int32),
                            C.POINTER(C.c_int64), C.POINTER(C.c_uint32))


class BlockOp(C.Structure):
    _fields_ = [
        ("nblocks", C.c_int32), ("nrows", C.c_int32), ("ncols_total", C.c_int64),
        ("partial_len", C.c_int64), ("max_rows", C.c_int32), ("max_ncols", C.c_int32),
        ("vals", C.c_void_p), ("off", C.c_void_p), ("ld", C.c_void_p), ("m", C.c_void_p),
        ("ncols", C.c_void_p), ("col_off", C.c_void_p), ("row_off", C.c_void_p),
        ("rows", C.c_void_p), ("gptr", C.c_void_p), ("gsrc", C.c_void_p),
        ("n_row_tiles", C.c_int32), ("row_tiles", C.c_void_p),
        ("n_col_tiles", C.c_int32), ("col_tiles", C.c_void_p),
        ("partial", C.c_void_p), ("red_scratch", C.c_void_p), ("counter", C.c_void_p),
        ("order", C.c_void_p),
    ]


class AssemblyDesc(C.Structure):
    _fields_ = [
        ("dim", C.c_int32), ("nsub", C.c_int32), ("count_per_dim", C.c_int32),
        ("nfeat", C.c_int32), ("activation", C.c_int32), ("ngroups", C.c_int32),
        ("reach", C.c_int32),
        ("centers", C.c_void_p), ("half", C.c_void_p), ("weights", C.c_void_p),
        ("biases", C.c_void_p), ("axes", C.c_void_p), ("axis_off", C.c_void_p),
        ("op_coef", C.c_void_p), ("con_pts", C.c_void_p), ("box", C.c_void_p),
        ("con_ptr", C.c_void_p), ("con_idx", C.c_void_p), ("con_grp", C.c_void_p),
        ("n_tiles", C.c_int32), ("tiles", C.c_void_p),
        ("mask_int", C.c_void_p), ("mask_con", C.c_void_p), ("lattice_stride", C.c_int64 * 3),
    ]


class LsqrState(C.Structure):
    _fields_ = [(n, C.c_double) for n in (
        "alpha", "beta", "rhobar", "phibar", "rho", "c", "s", "phi", "theta", "beta_prev",
        "best", "anorm", "ddnorm", "xxnorm", "z", "cs2", "sn2", "bnorm", "atol", "btol",
        "ctol")] + [
        ("it", C.c_int64), ("best_it", C.c_int64), ("diverged_at", C.c_int64),
        ("done", C.c_int32), ("breakdown", C.c_int32), ("istop", C.c_int32),
        ("use_rule", C.c_int32), ("stride", C.c_int32), ("nonfinite", C.c_int32),
        ("monitor", C.c_int32), ("improved", C.c_int32),
    ]


class LsqrVecs(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("u", "v", "vp", "w", "x", "xbest", "trace", "ub")]


class CgVecs(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("tmp", "p", "q", "r", "z", "x", "xbest", "res_trace",
                                          "rhs", "scratch", "counter")] + [("stride", C.c_int32)]


class BlockPrecond(C.Structure):
    _fields_ = [("nblocks", C.c_int32), ("max_size", C.c_int32), ("idx_off", C.c_void_p),
                ("idx", C.c_void_p), ("val_off", C.c_void_p), ("vals", C.c_void_p)]


class TestMonitor(C.Structure):
    _fields_ = [("T", BlockOp), ("lift", C.c_void_p), ("truth", C.c_void_p), ("spread", C.c_double),
                ("err_trace", C.c_void_p), ("result", C.c_void_p)]


_lib = None


def lib():
    """Load the sm_100a library (built by build.py). Raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DeviceError(
            f"{LIB_PATH} is missing: run `python -m paper_2506_17626_b200.build` "
            "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    sig = {
        "fl_assemble": [C.POINTER(AssemblyDesc), C.POINTER(BlockOp), vp],
        "fl_rrqr": [C.POINTER(BlockOp), C.c_int32, C.c_int32, C.c_double, vp, vp, vp, vp, vp],
        "fl_blockop_apply": [C.POINTER(BlockOp), vp, vp, vp],
        "fl_blockop_apply_t": [C.POINTER(BlockOp), vp, vp, vp],
        "fl_lsqr_init": [C.POINTER(BlockOp), vp, C.POINTER(LsqrVecs), vp, vp],
        "fl_lsqr_iterate": [C.POINTER(BlockOp), C.POINTER(LsqrVecs), vp, C.c_int64,
                            C.c_int64, vp],
        "fl_backsub_scatter": [C.c_int32, C.c_int32, vp, vp, vp, vp, vp, vp, vp, vp],
        "fl_probe_fp64": [C.c_int32, C.c_int32, C.c_int32, vp, vp],
        "fl_probe_read": [vp, C.c_int64, vp, vp],
        "fl_rrqr_blocked": [C.POINTER(BlockOp), C.POINTER(BlockOp), C.c_int32, C.c_int64,
                            C.c_double, vp, vp, vp, vp, vp, vp],
        "fl_dev_wy_apply": [vp, vp, vp, vp, vp, vp, vp, vp, C.c_int64, C.c_int32, C.c_int32,
                            C.c_int32, vp, vp, C.c_int32, vp],
        "fl_dev_qform": [vp, vp, vp, vp, vp, vp, vp, vp, vp, C.c_int32, C.c_int32, vp],
        "fl_error_blocks": [C.POINTER(BlockOp), vp, vp, C.c_int32, C.POINTER(BlockOp), C.c_int32,
                            vp, vp],
        "fl_monitor_error": [C.POINTER(TestMonitor), vp, vp],
        "fl_lsqr_iterate_monitored": [C.POINTER(BlockOp), C.POINTER(LsqrVecs), vp, C.c_int64,
                                      C.c_int64, C.POINTER(TestMonitor), vp],
        "fl_lsqr_monitor_flush": [C.POINTER(BlockOp), C.POINTER(LsqrVecs), vp, vp],
        "fl_cg_init": [C.POINTER(BlockOp), C.POINTER(CgVecs), C.POINTER(BlockPrecond), vp, vp],
        "fl_cg_iterate": [C.POINTER(BlockOp), C.POINTER(CgVecs), C.POINTER(BlockPrecond), vp,
                          C.c_int64, C.c_int64, C.POINTER(TestMonitor), vp],
        "fl_cg_residual": [C.POINTER(BlockOp), C.POINTER(CgVecs), vp, vp],
        "fl_block_precond_apply": [C.POINTER(BlockPrecond), vp, vp, vp],
        "fl_as_setup": [C.POINTER(BlockOp), C.c_double, vp, vp, vp],
    }
    for name, args in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = C.c_int
    L.fl_version.restype = C.c_char_p
    L.fl_version.argtypes = []
    L.fl_last_error.restype = C.c_char_p
    L.fl_last_error.argtypes = []
    L.fl_assemble_tile_rows.restype = C.c_int32
    L.fl_assemble_tile_rows.argtypes = []
    L.fl_rrqr_blocked_workspace.restype = C.c_int64
    L.fl_rrqr_blocked_workspace.argtypes = [C.c_int32, C.c_int32, C.c_int64]
    _lib = L
    return L


EXPORTED = ("fl_assemble", "fl_rrqr", "fl_blockop_apply", "fl_blockop_apply_t", "fl_lsqr_init",
            "fl_lsqr_iterate", "fl_backsub_scatter", "fl_probe_fp64", "fl_dev_wy_apply", "fl_dev_qform",
            "fl_rrqr_blocked", "fl_rrqr_blocked_workspace", "fl_version", "fl_last_error",
            "fl_error_blocks", "fl_monitor_error", "fl_lsqr_iterate_monitored",
            "fl_lsqr_monitor_flush", "fl_cg_init", "fl_cg_iterate", "fl_cg_residual",
            "fl_block_precond_apply", "fl_probe_read", "fl_assemble_tile_rows", "fl_as_setup")


def check(code: int, what: str) -> None:
    if code == FL_OK:
        return
    if code == FL_ERR_INVALID:
        raise InvalidInputError(f"{what}: invalid input")
    if code == FL_ERR_DEGENERATE:
        raise DegenerateSubdomainError(what)
    if code == FL_ERR_DIVERGENCE:
        raise DivergenceError(what)
    if code == FL_ERR_SINGULAR:
        raise SingularFactorError(what)
    detail = lib().fl_last_error().decode(errors="replace")
    raise DeviceError(f"{what}: CUDA error (code {code}): {detail}")
