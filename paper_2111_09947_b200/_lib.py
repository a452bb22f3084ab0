"""ctypes binding of the C ABI in include/maskmul_b200.h.

The library is built in-tree (paper_2111_09947_b200/_lib/libmaskmul_b200.so).
There is no fallback: if it cannot be loaded, every call raises.
"""

from __future__ import annotations

import ctypes as C
import os

from .build import LIB_PATH, MMIO_LIB_PATH

MM_ALGO = {"msa": 0, "hash": 1, "mca": 2, "heap": 3, "heapdot": 4, "inner": 5, "auto": 6}
MM_OK, MM_ERR_PLAN, MM_ERR_INPUT, MM_ERR_INTERNAL, MM_ERR_CUDA, MM_ERR_CAPACITY = 0, 1, 2, 3, 4, 5
MM_DTYPE_INT64, MM_DTYPE_FLOAT64 = 0, 1

# every symbol declared in include/maskmul_b200.h
EXPORTS = ("mm_abi_version", "mm_last_error", "mm_create", "mm_destroy", "mm_multiply", "mm_multiply_begin",
           "mm_multiply_end", "mm_symbolic", "mm_row_flops", "mm_exclusive_scan",
           "mm_compact_rows", "mm_reduce_sum", "mm_profile_enable", "mm_profile_read",
           "mm_profile_bins", "mm_set_tuning", "mm_filter_min", "mm_lookup_rows",
           "mm_bc_dependency_weights", "mm_bc_scale_by", "mm_ewise_add_begin", "mm_ewise_add_end",
           "mm_bc_accumulate", "mm_csr_from_coo", "mm_expand_rows", "mm_degree_order", "mm_row_work",
           "mm_workspace_bytes")
MM_COO_SYMMETRIC, MM_COO_NO_DIAG, MM_COO_LOWER, MM_COO_DEDUP = 1, 2, 4, 8


class MatrixT(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64), ("nnz", C.c_int64),
                ("ptr", C.c_void_p), ("idx", C.c_void_p), ("values", C.c_void_p)]


class PlanT(C.Structure):
    _fields_ = [("algorithm", C.c_int32), ("phases", C.c_int32), ("complemented", C.c_int32),
                ("semiring", C.c_int32), ("dtype", C.c_int32), ("n_inspect", C.c_int32)]


class StatsT(C.Structure):
    _fields_ = [("generated_flops", C.c_int64), ("evaluated_multiplies", C.c_int64),
                ("output_nnz", C.c_int64), ("rows_push", C.c_int64), ("rows_pull", C.c_int64),
                ("rows_empty", C.c_int64)]


_lib = None


def load(path: str | None = None):
    """Load the CUDA library (no silent fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("MM_LIB_PATH") or LIB_PATH
    if not os.path.exists(path):
        raise RuntimeError(f"maskmul CUDA library missing at {path}: run __graft_entry__.build()")
    lib = C.CDLL(path)
    P = C.c_void_p
    PM = C.POINTER(MatrixT)
    lib.mm_abi_version.restype = C.c_int
    lib.mm_last_error.restype = C.c_char_p
    lib.mm_create.argtypes = [C.c_int, C.POINTER(P)]
    lib.mm_destroy.argtypes = [P]
    lib.mm_multiply_begin.argtypes = [P, C.POINTER(PlanT), PM, PM, PM, PM, P, C.POINTER(C.c_int64)]
    lib.mm_multiply_end.argtypes = [P, P, P, P, C.POINTER(StatsT)]
    lib.mm_multiply.argtypes = [P, C.POINTER(PlanT), PM, PM, PM, PM, P, P, P, P, C.c_int64, C.POINTER(C.c_int64),
                                C.POINTER(StatsT)]
    lib.mm_symbolic.argtypes = [P, C.POINTER(PlanT), PM, PM, PM, PM, P, P]
    lib.mm_row_flops.argtypes = [PM, PM, P, P, P]
    lib.mm_exclusive_scan.argtypes = [P, C.c_int64, P, P]
    lib.mm_compact_rows.argtypes = [C.c_int64, P, P, P, P, P, P, P, C.c_int, P]
    lib.mm_reduce_sum.argtypes = [P, C.c_int64, C.c_int, P, P]
    lib.mm_profile_enable.argtypes = [P, C.c_int]
    lib.mm_profile_read.argtypes = [P, P, C.c_int, C.POINTER(C.c_int64)]
    lib.mm_profile_bins.argtypes = [P, P, P, C.c_int]
    lib.mm_set_tuning.argtypes = [P, P, C.c_int]
    lib.mm_filter_min.argtypes = [C.POINTER(MatrixT), C.c_int64, P, P, C.POINTER(C.c_int64), P]
    lib.mm_lookup_rows.argtypes = [PM, PM, C.c_int, P, P, P]
    lib.mm_bc_dependency_weights.argtypes = [PM, PM, PM, P, P]
    lib.mm_bc_scale_by.argtypes = [PM, PM, P, P]
    lib.mm_ewise_add_begin.argtypes = [PM, PM, P, C.POINTER(C.c_int64), P]
    lib.mm_ewise_add_end.argtypes = [PM, PM, C.c_int, P, P, P, P]
    lib.mm_bc_accumulate.argtypes = [PM, P, P, P]
    lib.mm_csr_from_coo.argtypes = [C.c_int64, C.c_int64, P, P, C.c_int, C.c_int64, P, C.c_int, P, P, P, P,
                                    C.POINTER(C.c_int64), P]
    lib.mm_expand_rows.argtypes = [C.c_int64, P, P, P]
    lib.mm_degree_order.argtypes = [PM, P, P, P]
    lib.mm_row_work.argtypes = [PM, PM, PM, P, P, P]
    lib.mm_workspace_bytes.argtypes = [C.POINTER(PlanT), PM, PM, PM, C.POINTER(C.c_size_t)]
    for name in EXPORTS:
        getattr(lib, name)
        if name not in ("mm_last_error",):
            getattr(lib, name).restype = C.c_int
    lib.mm_last_error.restype = C.c_char_p
    _lib = lib
    return lib


def last_error() -> str:
    msg = load().mm_last_error()
    return msg.decode() if msg else ""


# every symbol declared in include/maskmul_mmio.h
MMIO_EXPORTS = ("mmx_read_header", "mmx_read_entries")
MMX_OK, MMX_ERR_FORMAT, MMX_ERR_OVERFLOW = 0, 2, 5
MMX_FIELDS = ("real", "integer", "pattern")


class MmxHeaderT(C.Structure):
    _fields_ = [("field", C.c_int32), ("symmetric", C.c_int32), ("nrows", C.c_int64), ("ncols", C.c_int64),
                ("nnz", C.c_int64), ("data_offset", C.c_int64), ("data_line", C.c_int64)]


_mmio = None


def load_mmio(path: str | None = None):
    """Load the host Matrix Market reader (no Python fallback parser)."""
    global _mmio
    if _mmio is not None:
        return _mmio
    path = path or MMIO_LIB_PATH
    if not os.path.exists(path):
        raise RuntimeError(f"Matrix Market reader missing at {path}: run __graft_entry__.build()")
    lib = C.CDLL(path)
    P = C.c_void_p
    lib.mmx_read_header.argtypes = [P, C.c_int64, C.POINTER(MmxHeaderT), C.POINTER(C.c_int64), C.c_char_p,
                                    C.c_int]
    lib.mmx_read_entries.argtypes = [P, C.c_int64, C.POINTER(MmxHeaderT), P, P, P, C.c_int,
                                     C.POINTER(C.c_int64), C.c_char_p, C.c_int]
    for name in MMIO_EXPORTS:
        getattr(lib, name).restype = C.c_int
    _mmio = lib
    return lib
