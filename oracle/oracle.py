"""ctypes front end of the C oracle (test infrastructure; see __init__.py)."""

from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libmaskmul_oracle.so")

ALGO_IDS = {"msa": 0, "hash": 1, "mca": 2, "heap": 3, "heapdot": 4, "inner": 5}


class _Result(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("nnz", C.c_int64),
                ("row_ptr", C.POINTER(C.c_int64)), ("col_idx", C.POINTER(C.c_int64)),
                ("values", C.c_void_p),
                ("generated_flops", C.c_int64), ("evaluated", C.c_int64),
                ("symbolic_seconds", C.c_double), ("numeric_seconds", C.c_double),
                ("assemble_seconds", C.c_double), ("status", C.c_int)]


_lib = None


def build() -> str:
    """Compile the oracle with its Makefile (gcc -fopenmp)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        build()
    lib = C.CDLL(LIB_PATH)
    P = C.c_void_p
    I64 = C.c_int64
    lib.or_masked_multiply.restype = C.POINTER(_Result)
    lib.or_masked_multiply.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, I64,
                                       I64, I64, P, P, P, P, P, P, P, P, P, C.c_int, I64]
    lib.or_free_result.argtypes = [C.POINTER(_Result)]
    lib.or_free_result.restype = None
    lib.or_symbolic_phase.restype = C.c_int
    lib.or_symbolic_phase.argtypes = [C.c_int, C.c_int, I64, I64, I64, P, P, P, P, P, P, P,
                                      C.c_int, P]
    lib.or_max_threads.restype = C.c_int
    lib.or_set_threads.argtypes = [C.c_int]
    lib.or_set_threads.restype = None
    _lib = lib
    return lib


def max_threads() -> int:
    return int(load().or_max_threads())


def use_all_cores() -> int:
    """Run later oracle calls on every core this process may use (torchrun
    sets OMP_NUM_THREADS=1 per rank); returns the thread count."""
    n = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    load().or_set_threads(n)
    return max_threads()


@dataclass
class OracleResult:
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray
    generated_flops: int
    evaluated_multiplies: int
    numeric_seconds: float
    symbolic_seconds: float
    assemble_seconds: float

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    @property
    def total_seconds(self) -> float:
        return self.numeric_seconds + self.symbolic_seconds + self.assemble_seconds


def _ptr(a):
    return None if a is None else a.ctypes.data


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _ninspect(algorithm, n_inspect):
    if n_inspect is None:
        n_inspect = math.inf if algorithm == "heapdot" else 1
    return -1 if n_inspect == math.inf else int(n_inspect)


def _b_arrays(algorithm, b, dtype):
    """Push reads B as CSR, pull (inner) as CSC (multiply.py:205-216)."""
    from paper_2111_09947_b200.sparse import CscMatrix, to_csc, to_csr
    if algorithm == "inner":
        bc = b if isinstance(b, CscMatrix) else to_csc(b)
        row_len = np.bincount(_i64(bc.row_idx[: bc.nnz]), minlength=bc.nrows).astype(np.int64)
        return _i64(bc.col_ptr), _i64(bc.row_idx[: bc.nnz]), \
            np.ascontiguousarray(bc.values[: bc.nnz].astype(dtype)), row_len
    br = b if not isinstance(b, CscMatrix) else to_csr(b)
    return _i64(br.row_ptr), _i64(br.col_idx[: br.nnz]), \
        np.ascontiguousarray(br.values[: br.nnz].astype(dtype)), None


def masked_multiply(mask, a, b, algorithm="msa", phases="1p", complemented=False,
                    semiring_id=0, dtype=np.int64, n_inspect=None, workers=1,
                    grain=64) -> OracleResult:
    """C = M (.) (A B) on the CPU, same semantics as the reference driver."""
    lib = load()
    dtype = np.dtype(dtype)
    comp = bool(complemented or getattr(mask, "complemented", False))
    if algorithm in ("mca", "inner") and comp:
        raise ValueError(f"{algorithm} does not support complemented masks")
    a_ptr = _i64(a.row_ptr)
    a_idx = _i64(a.col_idx[: a.nnz])
    a_val = np.ascontiguousarray(a.values[: a.nnz].astype(dtype))
    b_ptr, b_idx, b_val, b_row_len = _b_arrays(algorithm, b, dtype)
    m_ptr = _i64(mask.row_ptr)
    m_idx = _i64(mask.col_idx[: mask.nnz])
    r = lib.or_masked_multiply(
        ALGO_IDS[algorithm], 1 if phases == "2p" else 0, int(comp), int(semiring_id),
        1 if dtype.kind == "f" else 0, _ninspect(algorithm, n_inspect),
        int(mask.nrows), int(mask.ncols), _ptr(a_ptr), _ptr(a_idx), _ptr(a_val),
        _ptr(b_ptr), _ptr(b_idx), _ptr(b_val), _ptr(b_row_len), _ptr(m_ptr), _ptr(m_idx),
        int(workers), int(grain))
    try:
        res = r.contents
        if res.status != 0:
            raise AssertionError("oracle: row bound / symbolic count violated")
        n = int(res.nrows)
        nnz = int(res.nnz)
        row_ptr = np.ctypeslib.as_array(res.row_ptr, shape=(n + 1,)).copy()
        col_idx = (np.ctypeslib.as_array(res.col_idx, shape=(nnz,)).copy() if nnz
                   else np.empty(0, dtype=np.int64))
        if nnz:
            buf = (C.c_char * (nnz * 8)).from_address(res.values)
            values = np.frombuffer(buf, dtype=dtype).copy()
        else:
            values = np.empty(0, dtype=dtype)
        return OracleResult(row_ptr, col_idx, values, int(res.generated_flops),
                            int(res.evaluated), float(res.numeric_seconds),
                            float(res.symbolic_seconds), float(res.assemble_seconds))
    finally:
        lib.or_free_result(r)


def symbolic_phase(mask, a, b, algorithm="msa", complemented=False, n_inspect=None,
                   workers=1) -> np.ndarray:
    lib = load()
    comp = bool(complemented or getattr(mask, "complemented", False))
    a_ptr = _i64(a.row_ptr)
    a_idx = _i64(a.col_idx[: a.nnz])
    b_ptr, b_idx, _, b_row_len = _b_arrays(algorithm, b, np.int64)
    m_ptr = _i64(mask.row_ptr)
    m_idx = _i64(mask.col_idx[: mask.nnz])
    counts = np.zeros(max(int(mask.nrows), 1), dtype=np.int64)
    lib.or_symbolic_phase(ALGO_IDS[algorithm], int(comp), _ninspect(algorithm, n_inspect),
                          int(mask.nrows), int(mask.ncols), _ptr(a_ptr), _ptr(a_idx),
                          _ptr(b_ptr), _ptr(b_idx), _ptr(b_row_len), _ptr(m_ptr), _ptr(m_idx),
                          int(workers), _ptr(counts))
    return counts[: int(mask.nrows)]
