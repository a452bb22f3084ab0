"""Device element-wise sparse operations used by the graph drivers.

Mirrors of the reference's helpers, computed by the CUDA kernels of
csrc/graph_ops.cuh through the C ABI:
  * ``ewise_add``   — sparse.py:360-370 (union; values added where both hold
                      an entry)
  * ``lookup_rows`` — _kernels.py:597-612 / graphs._values_at (graphs.py:121-129)
  * ``bc_dependency_weights``, ``bc_scale_by``, ``bc_accumulate`` — the
    fused element-wise steps of betweenness centrality (graphs.py:181-197)
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from .device import DeviceCsr
from .multiply import _raise
from .sparse import SparseError


def _stream(dev):
    return C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _dtype_id(t: torch.Tensor) -> int:
    return _lib.MM_DTYPE_FLOAT64 if t.dtype == torch.float64 else _lib.MM_DTYPE_INT64


def _check(rc: int):
    if rc:
        _raise(rc)


def ewise_add(a: DeviceCsr, b: DeviceCsr) -> DeviceCsr:
    """C = A + B over the union of the patterns (sparse.py:360-370)."""
    if a.shape != b.shape:
        raise SparseError(f"shape mismatch {a.shape} vs {b.shape}")
    if a.values is None or b.values is None:
        raise SparseError("ewise_add needs valued operands")
    dtype = torch.promote_types(a.values.dtype, b.values.dtype)
    av = a.values if a.values.dtype == dtype else a.values.to(dtype)
    bv = b.values if b.values.dtype == dtype else b.values.to(dtype)
    a = DeviceCsr(a.nrows, a.ncols, a.ptr, a.idx, av)
    b = DeviceCsr(b.nrows, b.ncols, b.ptr, b.idx, bv)
    dev = a.idx.device
    lib = _lib.load()
    row_ptr = torch.empty(a.nrows + 1, dtype=torch.int64, device=dev)
    nnz = C.c_int64(0)
    ma, mb = a.mm(), b.mm()
    _check(lib.mm_ewise_add_begin(C.byref(ma), C.byref(mb), row_ptr.data_ptr(), C.byref(nnz), _stream(dev)))
    n = int(nnz.value)
    idx = torch.empty(n, dtype=torch.int32, device=dev)
    val = torch.empty(n, dtype=dtype, device=dev)
    _check(lib.mm_ewise_add_end(C.byref(ma), C.byref(mb), _dtype_id(val), row_ptr.data_ptr(),
                                idx.data_ptr() if n else None, val.data_ptr() if n else None, _stream(dev)))
    return DeviceCsr(a.nrows, a.ncols, row_ptr, idx, val)


def lookup_rows(x: DeviceCsr, y: DeviceCsr):
    """Values of Y at X's stored entries and a found mask (absent -> 0)."""
    if x.shape != y.shape:
        raise SparseError(f"shape mismatch {x.shape} vs {y.shape}")
    if y.values is None:
        raise SparseError("lookup_rows needs a valued Y")
    dev = x.idx.device
    out = torch.zeros(x.nnz, dtype=y.values.dtype, device=dev)
    found = torch.zeros(x.nnz, dtype=torch.uint8, device=dev)
    _check(_lib.load().mm_lookup_rows(C.byref(x.mm()), C.byref(y.mm()), _dtype_id(y.values),
                                      out.data_ptr() if x.nnz else None, found.data_ptr() if x.nnz else None,
                                      _stream(dev)))
    return out, found.bool()


def bc_dependency_weights(sigma_t: DeviceCsr, delta: DeviceCsr, paths: DeviceCsr) -> torch.Tensor:
    """(1 + delta) / paths on sigma_t's pattern (graphs.py:181-184)."""
    dev = sigma_t.idx.device
    w = torch.empty(sigma_t.nnz, dtype=torch.float64, device=dev)
    _check(_lib.load().mm_bc_dependency_weights(C.byref(sigma_t.mm()), C.byref(delta.mm()), C.byref(paths.mm()),
                                                w.data_ptr() if sigma_t.nnz else None, _stream(dev)))
    return w


def bc_scale_by(x: DeviceCsr, paths: DeviceCsr) -> torch.Tensor:
    """x.values * paths on x's pattern (graphs.py:186)."""
    dev = x.idx.device
    out = torch.empty(x.nnz, dtype=torch.float64, device=dev)
    _check(_lib.load().mm_bc_scale_by(C.byref(x.mm()), C.byref(paths.mm()),
                                      out.data_ptr() if x.nnz else None, _stream(dev)))
    return out


def bc_accumulate(delta: DeviceCsr, src_col: torch.Tensor, scores: torch.Tensor) -> None:
    """scores += row sums of delta, minus each source's own entry (graphs.py:188-197)."""
    dev = delta.idx.device
    _check(_lib.load().mm_bc_accumulate(C.byref(delta.mm()), src_col.data_ptr(), scores.data_ptr(),
                                        _stream(dev)))
