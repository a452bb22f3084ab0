"""Device-resident sparse operands (torch CUDA tensors as plain buffers).

HBM layout of one operand:
    ptr     int64[nrows+1]   row offsets (CSR) / column offsets (CSC)
    idx     int32[nnz]       column (CSR) / row (CSC) indices
    values  int64|float64[nnz], or absent for masks and plus-pair operands
Upload converts the reference's int64 column indices to int32 (input
preparation; the reference likewise casts in its untimed _Prepared,
multiply.py:199-216).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .sparse import CscMatrix, CsrMatrix, SparseError


def _dev(device) -> torch.device:
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


def _ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


@dataclass
class DeviceCsr:
    """CSR (or, with ``csc=True``, CSC) matrix in device memory."""
    nrows: int
    ncols: int
    ptr: torch.Tensor
    idx: torch.Tensor
    values: torch.Tensor | None = None
    csc: bool = False

    @property
    def nnz(self) -> int:
        return int(self.idx.numel())

    @property
    def shape(self):
        return (self.nrows, self.ncols)

    def mm(self) -> _lib.MatrixT:
        return _lib.MatrixT(self.nrows, self.ncols, self.nnz, _ptr(self.ptr), _ptr(self.idx),
                            _ptr(self.values))

    @staticmethod
    def from_host(m, dtype=None, device=None, with_values=True, pin=False) -> "DeviceCsr":
        """Upload a CsrMatrix / MaskView / CscMatrix (reference or ours)."""
        dev = _dev(device)
        is_csc = hasattr(m, "col_ptr")
        ptr = np.ascontiguousarray(m.col_ptr if is_csc else m.row_ptr, dtype=np.int64)
        n_major = m.ncols if is_csc else m.nrows
        if ptr.shape[0] != n_major + 1:
            raise SparseError("offset array must have (major dimension + 1) entries")
        nnz = int(ptr[-1])
        idx_src = m.row_idx if is_csc else m.col_idx
        idx = np.ascontiguousarray(idx_src[:nnz], dtype=np.int32)
        vals = None
        if with_values and getattr(m, "values", None) is not None:
            v = np.asarray(m.values[:nnz])
            if dtype is not None:
                v = v.astype(dtype, copy=False)
            vals = torch.from_numpy(np.ascontiguousarray(v))
        t_ptr = torch.from_numpy(ptr)
        t_idx = torch.from_numpy(idx)
        if pin:
            t_ptr, t_idx = t_ptr.pin_memory(), t_idx.pin_memory()
            vals = vals.pin_memory() if vals is not None else None
        return DeviceCsr(int(m.nrows), int(m.ncols), t_ptr.to(dev, non_blocking=pin),
                         t_idx.to(dev, non_blocking=pin),
                         None if vals is None else vals.to(dev, non_blocking=pin), csc=is_csc)

    def to_host(self) -> CsrMatrix:
        ptr = self.ptr.cpu().numpy().astype(np.int64, copy=False)
        idx = self.idx.cpu().numpy().astype(np.int64)
        vals = (self.values.cpu().numpy() if self.values is not None
                else np.ones(self.nnz, dtype=np.int64))
        if self.csc:
            return CscMatrix(self.nrows, self.ncols, ptr, idx, vals)
        return CsrMatrix(self.nrows, self.ncols, ptr, idx, vals)

    def transpose_storage(self) -> "DeviceCsr":
        """CSR -> CSC of the same matrix (to_csc, sparse.py:257-266): stable
        order, so row indices ascend inside every column.  Input preparation
        for the pull path (the reference excludes it from timing,
        multiply.py:205-210); runs on the device (prep.transpose: row scatter
        by column + segmented sort, csrc/graph_prep.cuh)."""
        if self.csc:
            raise SparseError("already column-major")
        from .prep import transpose
        t = transpose(self)
        return DeviceCsr(self.nrows, self.ncols, t.ptr, t.idx, t.values, csc=True)
