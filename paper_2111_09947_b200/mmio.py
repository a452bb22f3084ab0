"""Matrix Market coordinate reader and writer.

Same surface and behaviour as the reference's ``maskmul.mmio``
(pkg/src/maskmul/mmio.py:1-122): field real / integer / pattern, symmetry
general / symmetric, symmetric files expanded to both triangles (the diagonal
once), pattern entries valued 1, 1-based indices made 0-based, canonical CSR
with duplicates summed; ``MatrixMarketError`` carries the offending line.

The text is parsed by the native reader (csrc/mmio_host.cpp behind
include/maskmul_mmio.h, host threads over line ranges) instead of the
reference's per-line Python loop.  ``read_matrix_market`` returns the host
``CsrMatrix`` exactly as the reference does; ``read_matrix_market_device``
canonicalises on the GPU (``mm_csr_from_coo``) and returns a ``DeviceCsr``
ready for the multiply.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib
from .sparse import CsrMatrix, from_arrays

_FIELDS = {"real", "integer", "pattern"}


class MatrixMarketError(ValueError):
    """Malformed Matrix Market content; carries the offending line number (mmio.py:19-24)."""

    def __init__(self, lineno: int, message: str):
        super().__init__(f"line {lineno}: {message}")
        self.lineno = lineno


def _raise(rc: int, line: C.c_int64, msg) -> None:
    text = msg.value.decode("ascii", "replace")
    if rc == _lib.MMX_ERR_OVERFLOW:
        raise OverflowError(f"line {line.value}: {text}")
    raise MatrixMarketError(int(line.value), text)


def _parse(path, threads: int | None):
    """-> (field, symmetric, nrows, ncols, rows, cols, vals) as the reference holds them
    before canonicalisation (mmio.py:63-100, symmetric expansion included)."""
    lib = _lib.load_mmio()
    text = np.fromfile(os.fspath(path), dtype=np.uint8)
    base = text.ctypes.data if text.size else None
    hdr = _lib.MmxHeaderT()
    line = C.c_int64(0)
    msg = C.create_string_buffer(512)
    rc = lib.mmx_read_header(base, text.size, C.byref(hdr), C.byref(line), msg, len(msg))
    if rc:
        _raise(rc, line, msg)
    field = _lib.MMX_FIELDS[hdr.field]
    nnz = int(hdr.nnz)
    rows = np.empty(nnz, dtype=np.int64)
    cols = np.empty(nnz, dtype=np.int64)
    vals = (np.empty(nnz, dtype=np.float64) if field == "real"
            else np.empty(nnz, dtype=np.int64) if field == "integer"
            else np.ones(nnz, dtype=np.int64))
    rc = lib.mmx_read_entries(base, text.size, C.byref(hdr), rows.ctypes.data, cols.ctypes.data,
                              vals.ctypes.data if field != "pattern" else None,
                              int(threads or os.cpu_count() or 1), C.byref(line), msg, len(msg))
    if rc:
        _raise(rc, line, msg)
    if hdr.symmetric:
        off = rows != cols
        rows, cols, vals = (np.concatenate([rows, cols[off]]), np.concatenate([cols, rows[off]]),
                            np.concatenate([vals, vals[off]]))
    return field, bool(hdr.symmetric), int(hdr.nrows), int(hdr.ncols), rows, cols, vals


def read_matrix_market(path, threads: int | None = None) -> CsrMatrix:
    """mmio.py:27-101: canonical host CSR (int64 values for integer/pattern, float64 for real)."""
    _, _, nrows, ncols, rows, cols, vals = _parse(path, threads)
    return from_arrays(nrows, ncols, rows, cols, vals)


def read_matrix_market_device(path, device=None, with_values: bool | None = None, threads: int | None = None):
    """Matrix Market file -> DeviceCsr, canonicalised on the GPU.

    Same matrix as ``read_matrix_market`` (tests/test_gpu_prep.py checks it).
    Pattern files give a pattern-only operand (masks and plus-pair operands
    never read values, _kernels.py:56) unless ``with_values`` asks for the
    reference's values (ones, or duplicate counts).  Valued entries travel
    with their columns through the device sort; a file that repeats a
    coordinate is summed in file order by the host ``from_arrays`` instead,
    because the device sort does not keep the order of equal keys."""
    from .device import DeviceCsr
    from .prep import csr_from_coo

    field, _, nrows, ncols, rows, cols, vals = _parse(path, threads)
    if max(nrows, ncols) >= 2 ** 31:
        raise ValueError("device operands hold int32 indices: dimensions must be < 2^31")
    if with_values is None:
        with_values = field != "pattern"
    if not with_values:
        return csr_from_coo(nrows, ncols, rows, cols, dedup=True, device=device)
    g = csr_from_coo(nrows, ncols, rows, cols, vals, device=device)
    if g.nnz > 1:
        dup = g.idx[1:] == g.idx[:-1]
        cut = g.ptr[1:-1]
        cut = cut[(cut > 0) & (cut < g.nnz)] - 1
        dup[cut] = False
        if bool(dup.any()):
            return DeviceCsr.from_host(from_arrays(nrows, ncols, rows, cols, vals), device=device)
    return g


def write_matrix_market(path, a: CsrMatrix, field: str | None = None) -> None:
    """mmio.py:104-122: coordinate general form, 1-based; reals as repr (round-trip exact)."""
    if field is None:
        field = "integer" if np.issubdtype(a.values.dtype, np.integer) else "real"
    if field not in _FIELDS:
        raise ValueError(f"unsupported field {field!r}")
    rows, cols, vals = a.triples()
    with open(path, "w", encoding="ascii") as fh:
        fh.write(f"%%MatrixMarket matrix coordinate {field} general\n")
        fh.write(f"{a.nrows} {a.ncols} {a.nnz}\n")
        r1 = (np.asarray(rows, dtype=np.int64) + 1).tolist()
        c1 = (np.asarray(cols, dtype=np.int64) + 1).tolist()
        if field == "pattern":
            body = [f"{i} {j}\n" for i, j in zip(r1, c1)]
        elif field == "integer":
            body = [f"{i} {j} {int(v)}\n" for i, j, v in zip(r1, c1, np.asarray(vals).tolist())]
        else:
            body = [f"{i} {j} {float(v)!r}\n" for i, j, v in zip(r1, c1, np.asarray(vals).tolist())]
        fh.writelines(body)
