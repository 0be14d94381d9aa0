"""ctypes binding of the C ABI in ``include/sgap.h`` (``libsgap.so``).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc,
``-gencode arch=compute_100a,code=sm_100a``).  There is no fallback: if the
shared object is missing, every entry point raises ``NativeLibraryError``.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("SGAP_LIB", PKG_DIR / "libsgap.so"))

# sgap_status_t
OK = 0
ERR_ILLEGAL_POINT = 1
ERR_NO_TEMPLATE = 2
ERR_SHAPE = 3
ERR_PRECISION = 4
ERR_CUDA = 5
ERR_ARG = 6
ERR_FAULT = 7
ERR_CONFIG = 8

# sgap_family_t (same order as the header)
FAMILY_IDS = {"nnz-multiple": 0, "row-multiple": 1, "row-reciprocal": 2, "nnz-one": 3}
FAMILY_NAMES = {v: k for k, v in FAMILY_IDS.items()}

F32 = 0
F64 = 1

# amount kinds
AMT_RECIPROCAL, AMT_ONE, AMT_MULTIPLE = 0, 1, 2

EXPORTED = (
    "sgap_abi_version",
    "sgap_status_string",
    "sgap_legality_rule",
    "sgap_build_kernel",
    "sgap_block_starts",
    "sgap_row_ids",
    "sgap_exact_row_length",
    "sgap_long_row_threshold",
    "sgap_plan_workspace_bytes",
    "sgap_plan",
    "sgap_validate_csr",
    "sgap_run",
    "sgap_run_rbpr_grid",
    "sgap_reference_spmm_f64",
    "sgap_seg_reduce_group",
    "sgap_atomic_add_group",
    "sgap_mm_line_flags",
    "sgap_mm_parse",
    "sgap_mm_expand",
    "sgap_mm_sum_runs",
    "sgap_mm_row_ptr",
)


class NativeLibraryError(RuntimeError):
    """libsgap.so is missing or failed to load: no CPU fallback exists."""


class SgapError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(f"{what}: {status_string(status)} (status {status})")


class Point(ctypes.Structure):
    _fields_ = [
        ("data_kind", ctypes.c_int32),
        ("data_amount", ctypes.c_int32),
        ("data_param", ctypes.c_int32),
        ("col_amount", ctypes.c_int32),
        ("col_param", ctypes.c_int32),
        ("r", ctypes.c_int32),
    ]


class Kernel(ctypes.Structure):
    _fields_ = [
        ("family", ctypes.c_int32),
        ("n", ctypes.c_int32),
        ("p", ctypes.c_int32),
        ("g", ctypes.c_int32),
        ("c", ctypes.c_int32),
        ("r", ctypes.c_int32),
        ("chunk", ctypes.c_int64),
        ("grid_size", ctypes.c_int64),
        ("block_size", ctypes.c_int64),
        ("has_block_starts", ctypes.c_int32),
        ("hw_block", ctypes.c_int32),
        ("hw_variant", ctypes.c_int32),
    ]


class Csr(ctypes.Structure):
    _fields_ = [
        ("num_rows", ctypes.c_int64),
        ("num_cols", ctypes.c_int64),
        ("nnz", ctypes.c_int64),
        ("d_row_ptr", ctypes.c_void_p),
        ("d_col_idx", ctypes.c_void_p),
        ("d_vals", ctypes.c_void_p),
    ]


class Aux(ctypes.Structure):
    _fields_ = [
        ("d_block_starts", ctypes.c_void_p),
        ("d_rowid", ctypes.c_void_p),
        ("d_long_rows", ctypes.c_void_p),
        ("d_long_count", ctypes.c_void_p),
        ("d_long_acc", ctypes.c_void_p),
        ("long_capacity", ctypes.c_int64),
        ("long_threshold", ctypes.c_int64),
        ("has_exact_rows", ctypes.c_int32),
        ("d_long_slot", ctypes.c_void_p),
        ("long_chunk", ctypes.c_int64),
        ("d_exact_rows", ctypes.c_void_p),
        ("exact_count", ctypes.c_int32),
        ("d_chunk_rows", ctypes.c_void_p),
        ("d_union_off4", ctypes.c_void_p),
        ("d_union_off8", ctypes.c_void_p),
        ("d_union4", ctypes.c_void_p),
        ("d_union8", ctypes.c_void_p),
        ("d_col_hinted", ctypes.c_void_p),
        ("d_panel_b", ctypes.c_void_p),
        ("panel_lanes", ctypes.c_int32),
    ]


class Plan(ctypes.Structure):
    """sgap_plan_t (include/sgap.h): filled by sgap_plan, read by sgap_run."""

    _fields_ = [
        ("abi", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("kernel", Kernel),
        ("num_rows", ctypes.c_int64),
        ("num_cols", ctypes.c_int64),
        ("nnz", ctypes.c_int64),
        ("d_row_ptr", ctypes.c_void_p),
        ("d_col_idx", ctypes.c_void_p),
        ("longest_row", ctypes.c_int64),
        ("table_rows", ctypes.c_int64),
        ("aux", Aux),
        ("d_workspace", ctypes.c_void_p),
        ("workspace_bytes", ctypes.c_size_t),
    ]


# sgap_plan flags
PLAN_VALIDATE = 1
PLAN_SPLIT_ROWS = 2
PLAN_L2_HINTS = 4
PLAN_PANELS = 8

_lib = None


def lib():
    """Load libsgap.so once; raise loudly if it is not there."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise NativeLibraryError(
            f"{LIB_PATH} not found -- build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    try:
        L = ctypes.CDLL(str(LIB_PATH))
    except OSError as e:  # pragma: no cover - environment failure
        raise NativeLibraryError(f"cannot load {LIB_PATH}: {e}") from e
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    L.sgap_abi_version.restype = ctypes.c_int
    L.sgap_status_string.argtypes = [ctypes.c_int]
    L.sgap_status_string.restype = ctypes.c_char_p
    L.sgap_legality_rule.argtypes = [ctypes.POINTER(Point)]
    L.sgap_legality_rule.restype = ctypes.c_int
    L.sgap_build_kernel.argtypes = [ctypes.POINTER(Point), i32, i32, i64, i64,
                                    ctypes.POINTER(Kernel), ctypes.POINTER(i32)]
    L.sgap_build_kernel.restype = ctypes.c_int
    L.sgap_block_starts.argtypes = [vp, i64, i64, i64, vp, vp]
    L.sgap_block_starts.restype = ctypes.c_int
    L.sgap_row_ids.argtypes = [vp, i64, i64, i64, i64, vp, vp]
    L.sgap_row_ids.restype = ctypes.c_int
    L.sgap_exact_row_length.argtypes = []
    L.sgap_exact_row_length.restype = i64
    L.sgap_long_row_threshold.argtypes = [ctypes.POINTER(Kernel), i32]
    L.sgap_long_row_threshold.restype = i64
    L.sgap_plan_workspace_bytes.argtypes = [ctypes.POINTER(Kernel), ctypes.POINTER(Csr), i32,
                                            ctypes.c_uint32, ctypes.POINTER(ctypes.c_size_t)]
    L.sgap_plan_workspace_bytes.restype = ctypes.c_int
    L.sgap_plan.argtypes = [ctypes.POINTER(Kernel), ctypes.POINTER(Csr), i32, ctypes.c_uint32, vp,
                            ctypes.c_size_t, ctypes.POINTER(Plan), vp]
    L.sgap_plan.restype = ctypes.c_int
    L.sgap_validate_csr.argtypes = [ctypes.POINTER(Csr), vp, ctypes.POINTER(i64), vp]
    L.sgap_validate_csr.restype = ctypes.c_int
    L.sgap_run.argtypes = [ctypes.POINTER(Plan), ctypes.POINTER(Csr), vp, vp, i32, vp, vp]
    L.sgap_run.restype = ctypes.c_int
    L.sgap_run_rbpr_grid.argtypes = [ctypes.POINTER(Plan), ctypes.POINTER(Csr), vp, vp, i32, i32,
                                     ctypes.c_double, i32, vp, vp]
    L.sgap_run_rbpr_grid.restype = ctypes.c_int
    L.sgap_reference_spmm_f64.argtypes = [ctypes.POINTER(Csr), vp, i32, i32, vp, vp]
    L.sgap_reference_spmm_f64.restype = ctypes.c_int
    L.sgap_mm_line_flags.argtypes = [vp, i64, vp, vp, vp]
    L.sgap_mm_parse.argtypes = [vp, i64, vp, i64, i64, i64, vp, vp, vp, vp, vp, vp, vp]
    L.sgap_mm_expand.argtypes = [i64, vp, vp, vp, vp, vp, i32, vp, vp, vp]
    L.sgap_mm_sum_runs.argtypes = [i64, vp, vp, vp, i64, vp, vp, vp, vp]
    L.sgap_mm_row_ptr.argtypes = [vp, i64, i64, vp, vp]
    for name in ("sgap_mm_line_flags", "sgap_mm_parse", "sgap_mm_expand", "sgap_mm_sum_runs",
                 "sgap_mm_row_ptr"):
        getattr(L, name).restype = ctypes.c_int
    for name in ("sgap_seg_reduce_group", "sgap_atomic_add_group"):
        fn = getattr(L, name)
        fn.argtypes = [vp, vp, vp, i64, i32, vp, i64, i32, vp, vp, vp]
        fn.restype = ctypes.c_int
    _lib = L
    return L


def status_string(status: int) -> str:
    try:
        return lib().sgap_status_string(status).decode()
    except NativeLibraryError:
        return "unknown"


def check(status: int, what: str):
    if status != OK:
        raise SgapError(status, what)
