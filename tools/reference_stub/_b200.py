"""The ctypes stub a `maskmul` maintainer would add as `maskmul/_b200.py`
(option B): the reference's `_Prepared` (multiply.py:175-233)
in, the B200 library's C ABI (include/maskmul_b200.h) underneath, the
reference's row_ptr / col_idx / values / stats out.  Exercised by
tests/test_gpu_integration_stub.py with a `_Prepared` built from the same
field names."""
import ctypes as C
import os

import numpy as np
import torch

_LIB = os.environ.get("MASKMUL_B200_LIB", "libmaskmul_b200.so")
_lib = C.CDLL(_LIB)


class _Mat(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64), ("nnz", C.c_int64),
                ("ptr", C.c_void_p), ("idx", C.c_void_p), ("values", C.c_void_p)]


class _Plan(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("algorithm", "phases", "complemented", "semiring", "dtype", "n_inspect")]


class _Stats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("generated_flops", "evaluated_multiplies", "output_nnz",
                                         "rows_push", "rows_pull", "rows_empty")]


_ALGO = {"msa": 0, "hash": 1, "mca": 2, "heap": 3, "heapdot": 4, "inner": 5}
_P = C.c_void_p
_lib.mm_create.argtypes = [C.c_int, C.POINTER(_P)]
_lib.mm_multiply_begin.argtypes = [_P, C.POINTER(_Plan), C.POINTER(_Mat), C.POINTER(_Mat), C.POINTER(_Mat),
                                   C.POINTER(_Mat), _P, C.POINTER(C.c_int64)]
_lib.mm_multiply_end.argtypes = [_P, _P, _P, _P, C.POINTER(_Stats)]
_lib.mm_last_error.restype = C.c_char_p
_h = _P()
if _lib.mm_create(0, C.byref(_h)):
    raise RuntimeError(_lib.mm_last_error().decode())


def _dev(ptr, idx, vals, nrows, ncols):
    t = [torch.from_numpy(np.ascontiguousarray(ptr, np.int64)).cuda(),
         None if idx is None else torch.from_numpy(np.ascontiguousarray(idx, np.int32)).cuda(),
         None if vals is None else torch.from_numpy(np.ascontiguousarray(vals)).cuda()]
    nnz = 0 if idx is None else len(idx)
    m = _Mat(nrows, ncols, nnz, t[0].data_ptr(), 0 if t[1] is None else t[1].data_ptr(),
             0 if t[2] is None else t[2].data_ptr())
    return m, t                                   # keep t alive during the call


def masked_multiply_b200(p, plan):
    """p: the reference's _Prepared; returns (row_ptr, col_idx, values, stats)."""
    vals = plan.semiring.kernel_id == 0
    ninner = len(p.b_row_lengths)
    M, k1 = _dev(p.m_ptr, p.m_idx, None, p.nrows, p.ncols)
    A, k2 = _dev(p.a_ptr, p.a_idx, p.a_val if vals else None, p.nrows, ninner)
    bt = None
    if plan.algorithm == "inner":
        # _Prepared holds B only as CSC for inner (multiply.py:205-210): B's row
        # pointer (the flops_per_row input) from b_row_lengths, B^T as CSC
        B, k3 = _dev(np.concatenate([[0], np.cumsum(p.b_row_lengths)]), None, None, ninner, p.ncols)
        BT, k4 = _dev(p.bc_ptr, p.bc_row, p.bc_val if vals else None, ninner, p.ncols)
        bt = C.byref(BT)
    else:
        B, k3 = _dev(p.b_ptr, p.b_idx, p.b_val if vals else None, ninner, p.ncols)
    pl = _Plan(_ALGO[plan.algorithm], 2 if plan.phases == "2p" else 1, int(p.comp),
               plan.semiring.kernel_id, 1 if p.dtype.kind == "f" else 0, p.kernel_ninspect)
    s = torch.cuda.current_stream().cuda_stream
    nnz = C.c_int64()
    rc = _lib.mm_multiply_begin(_h, C.byref(pl), C.byref(M), C.byref(A), C.byref(B), bt, C.c_void_p(s),
                                C.byref(nnz))
    if rc:
        raise {1: ValueError, 2: ValueError, 3: AssertionError}.get(rc, RuntimeError)(_lib.mm_last_error().decode())
    ptr = torch.empty(p.nrows + 1, dtype=torch.int64, device="cuda")
    idx = torch.empty(nnz.value, dtype=torch.int32, device="cuda")
    val = torch.empty(nnz.value, dtype=torch.float64 if p.dtype.kind == "f" else torch.int64, device="cuda")
    st = _Stats()
    rc = _lib.mm_multiply_end(_h, ptr.data_ptr(), idx.data_ptr() if nnz.value else None,
                              val.data_ptr() if nnz.value else None, C.byref(st))
    if rc:
        raise AssertionError(_lib.mm_last_error().decode())
    return ptr.cpu().numpy(), idx.cpu().numpy().astype(np.int64), val.cpu().numpy(), st
