"""Device-side input preparation.

The reference canonicalises every input on the host before the multiplies it
times (pkg/src/maskmul/sparse.py): ``from_arrays`` (:223-242),
``simple_undirected_graph`` (:344-357), ``degree_sort_relabel`` +
``permute_symmetric`` (:318-341), ``tril_strict`` (:285-291) and ``to_csc`` /
``transpose`` (:257-283).  Here the same steps run on the GPU through the C
ABI (csrc/graph_prep.cuh: atomic row scatter, segmented bitonic sort per row,
duplicate merge, degree bucketing); results are identical to the host
functions (same canonical CSR, same permutation), checked by
tests/test_gpu_prep.py.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .device import DeviceCsr, _dev
from .multiply import _raise
from .sparse import SparseError


def _stream(dev):
    return C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _as_index(x, dev) -> torch.Tensor:
    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(x))
    x = x.to(dev)
    if x.dtype not in (torch.int32, torch.int64):
        x = x.to(torch.int64)
    return x.contiguous()


def csr_from_coo(nrows: int, ncols: int, rows, cols, values=None, *, map=None, symmetric=False,
                 no_diag=False, lower=False, dedup=False, device=None) -> DeviceCsr:
    """Canonical CSR (rows sorted by column) from COO triples on the device.

    ``map`` relabels both endpoints, ``symmetric`` adds the mirrored entry,
    ``no_diag`` drops r == c, ``lower`` keeps c < r, ``dedup`` merges
    duplicates (pattern only).  ``values`` (8-byte dtype) travel with their
    entries when duplicates are not merged."""
    dev = _dev(device)
    r = _as_index(rows, dev)
    c = _as_index(cols, dev)
    if c.dtype != r.dtype:
        c = c.to(r.dtype)
    if r.numel() != c.numel():
        raise SparseError("rows and cols must have equal length")
    nnz = r.numel()
    if values is not None:
        if dedup:
            raise SparseError("duplicate merging is pattern-only")
        values = (torch.from_numpy(np.ascontiguousarray(values)) if isinstance(values, np.ndarray)
                  else values).to(dev).contiguous()
        if values.element_size() != 8 or values.numel() != nnz:
            raise SparseError("values must be one 8-byte value per entry")
    flags = ((_lib.MM_COO_SYMMETRIC if symmetric else 0) | (_lib.MM_COO_NO_DIAG if no_diag else 0)
             | (_lib.MM_COO_LOWER if lower else 0) | (_lib.MM_COO_DEDUP if dedup else 0))
    cap = max(nnz * (2 if symmetric else 1), 1)
    ptr = torch.empty(nrows + 1, dtype=torch.int64, device=dev)
    idx = torch.empty(cap, dtype=torch.int32, device=dev)
    vals = torch.empty(cap, dtype=values.dtype, device=dev) if values is not None else None
    out = C.c_int64(0)
    m = map.to(dev, torch.int32).contiguous() if map is not None else None
    rc = _lib.load().mm_csr_from_coo(nrows, ncols, r.data_ptr() if nnz else None, c.data_ptr() if nnz else None,
                                     int(r.dtype == torch.int64), nnz, m.data_ptr() if m is not None else None,
                                     flags, values.data_ptr() if values is not None and nnz else None,
                                     ptr.data_ptr(), idx.data_ptr(), vals.data_ptr() if vals is not None else None,
                                     C.byref(out), _stream(dev))
    if rc:
        _raise(rc)
    n = int(out.value)
    return DeviceCsr(nrows, ncols, ptr, idx[:n], vals[:n] if vals is not None else None)


def expand_rows(g: DeviceCsr) -> torch.Tensor:
    dev = g.idx.device
    rows = torch.empty(max(g.nnz, 1), dtype=torch.int32, device=dev)
    rc = _lib.load().mm_expand_rows(g.nrows, g.ptr.data_ptr(), rows.data_ptr(), _stream(dev))
    if rc:
        _raise(rc)
    return rows[: g.nnz]


def simple_undirected_graph(rows, cols, n: int, device=None) -> DeviceCsr:
    """sparse.py:344-357 on a COO edge list: symmetrise, drop self-loops,
    merge duplicates (values are the pattern; the reference sets them to 1)."""
    return csr_from_coo(n, n, rows, cols, symmetric=True, no_diag=True, dedup=True, device=device)


def degree_order(g: DeviceCsr):
    """(perm, new_label) of degree_sort_relabel (sparse.py:328-341):
    perm[new] = old by non-increasing degree, ties by index."""
    if g.nrows != g.ncols:
        raise SparseError("degree_sort_relabel requires a square matrix")
    dev = g.idx.device
    perm = torch.empty(max(g.nrows, 1), dtype=torch.int32, device=dev)
    new_label = torch.empty(max(g.nrows, 1), dtype=torch.int32, device=dev)
    rc = _lib.load().mm_degree_order(C.byref(g.mm()), perm.data_ptr(), new_label.data_ptr(), _stream(dev))
    if rc:
        _raise(rc)
    return perm[: g.nrows], new_label[: g.nrows]


def degree_sort_relabel(g: DeviceCsr):
    """P G P^T and perm (int64) — the device form of sparse.degree_sort_relabel.
    G must be pattern-symmetric, like the reference requires."""
    perm, new_label = degree_order(g)
    rows = expand_rows(g)
    out = csr_from_coo(g.nrows, g.ncols, rows, g.idx, g.values, map=new_label, device=g.idx.device)
    return out, perm.to(torch.int64)


def tril_strict(g: DeviceCsr) -> DeviceCsr:
    """Entries with col < row (sparse.py:285-291)."""
    if g.nrows != g.ncols:
        raise SparseError("tril_strict requires a square matrix")
    rows = expand_rows(g)
    return csr_from_coo(g.nrows, g.ncols, rows, g.idx, g.values, lower=True, device=g.idx.device)


def triangle_lower(g: DeviceCsr) -> DeviceCsr:
    """tril_strict(degree_sort_relabel(g)[0]) in one scatter (graphs.py:91-92)."""
    _, new_label = degree_order(g)
    rows = expand_rows(g)
    return csr_from_coo(g.nrows, g.ncols, rows, g.idx, map=new_label, lower=True, device=g.idx.device)


def transpose(g: DeviceCsr) -> DeviceCsr:
    """A^T as CSR — i.e. A stored column-major, row indices ascending inside
    every column (to_csc / transpose, sparse.py:257-283)."""
    rows = expand_rows(g)
    return csr_from_coo(g.ncols, g.nrows, g.idx, rows, g.values, device=g.idx.device)
