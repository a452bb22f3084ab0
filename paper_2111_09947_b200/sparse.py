"""Host-side sparse containers — the data contract of the masked multiply.

Mirrors the reference's L0 types (pkg/src/maskmul/sparse.py:28-187) so code
written against ``maskmul`` can hand its matrices to this package unchanged:

* :class:`CsrMatrix`  (sparse.py:28-99)   canonical = rows strictly sorted, no dups
* :class:`CscMatrix`  (sparse.py:102-130)
* :class:`MaskView`   (sparse.py:133-187) pattern-only CSR + complement flag
* constructors / transforms used to build the benchmark inputs
  (from_arrays :223-242, to_csc :257-266, to_csr :269-276, tril_strict :285-291,
  degree_sort_relabel :328-341, simple_undirected_graph :344-357).

Host arrays are numpy int64 (indices) + the semiring dtype (values), exactly
as the reference stores them.  The device copies used by the CUDA path live
in :mod:`paper_2111_09947_b200.device` (int32 column indices, int64 row
offsets).  The canonicalising constructors here are input preparation — the
reference excludes them from its timings and so do we.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class SparseError(ValueError):
    """Construction or shape error on a sparse matrix operation."""


@dataclass(eq=False)
class CsrMatrix:
    nrows: int
    ncols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray
    sorted: bool = True

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[self.nrows])

    @property
    def shape(self) -> tuple[int, int]:
        return (self.nrows, self.ncols)

    def row(self, i: int):
        lo, hi = int(self.row_ptr[i]), int(self.row_ptr[i + 1])
        return self.col_idx[lo:hi], self.values[lo:hi]

    def row_lengths(self) -> np.ndarray:
        return np.diff(self.row_ptr)

    def pattern(self, complemented: bool = False) -> "MaskView":
        return MaskView(self.nrows, self.ncols, self.row_ptr, self.col_idx,
                        complemented=complemented)

    def astype(self, dtype) -> "CsrMatrix":
        dt = np.dtype(dtype)
        if self.values.dtype == dt:
            return self
        return CsrMatrix(self.nrows, self.ncols, self.row_ptr, self.col_idx,
                         self.values.astype(dt), sorted=self.sorted)

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.nrows, self.ncols), dtype=self.values.dtype)
        rows = np.repeat(np.arange(self.nrows), self.row_lengths())
        out[rows, self.col_idx[: self.nnz]] = self.values[: self.nnz]
        return out

    def triples(self):
        rows = np.repeat(np.arange(self.nrows, dtype=np.int64), self.row_lengths())
        return rows, self.col_idx[: self.nnz].copy(), self.values[: self.nnz].copy()

    def equals(self, other) -> bool:
        """Bitwise equality of the canonical representation (sparse.py:75-83)."""
        n = self.nnz
        return (self.shape == tuple(other.shape)
                and np.array_equal(np.asarray(self.row_ptr, np.int64),
                                   np.asarray(other.row_ptr, np.int64))
                and np.array_equal(np.asarray(self.col_idx[:n], np.int64),
                                   np.asarray(other.col_idx[:n], np.int64))
                and self.values.dtype == other.values.dtype
                and np.array_equal(self.values[:n], other.values[:n]))

    def validate(self) -> None:
        _validate_pattern(self.nrows, self.ncols, self.row_ptr, self.col_idx, self.sorted)
        if self.values.shape[0] < self.nnz:
            raise SparseError("col_idx/values shorter than nnz")


@dataclass(eq=False)
class CscMatrix:
    nrows: int
    ncols: int
    col_ptr: np.ndarray
    row_idx: np.ndarray
    values: np.ndarray
    sorted: bool = True

    @property
    def nnz(self) -> int:
        return int(self.col_ptr[self.ncols])

    @property
    def shape(self) -> tuple[int, int]:
        return (self.nrows, self.ncols)

    def astype(self, dtype) -> "CscMatrix":
        dt = np.dtype(dtype)
        if self.values.dtype == dt:
            return self
        return CscMatrix(self.nrows, self.ncols, self.col_ptr, self.row_idx,
                         self.values.astype(dt), sorted=self.sorted)


@dataclass(eq=False)
class MaskView:
    nrows: int
    ncols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    complemented: bool = False

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[self.nrows])

    @property
    def shape(self) -> tuple[int, int]:
        return (self.nrows, self.ncols)

    def row(self, i: int) -> np.ndarray:
        return self.col_idx[int(self.row_ptr[i]):int(self.row_ptr[i + 1])]

    def row_lengths(self) -> np.ndarray:
        return np.diff(self.row_ptr)

    def complement(self) -> "MaskView":
        return MaskView(self.nrows, self.ncols, self.row_ptr, self.col_idx,
                        complemented=not self.complemented)

    def validate(self) -> None:
        _validate_pattern(self.nrows, self.ncols, self.row_ptr, self.col_idx, True)

    @staticmethod
    def full(nrows: int, ncols: int) -> "MaskView":
        row_ptr = np.arange(nrows + 1, dtype=np.int64) * ncols
        col_idx = np.tile(np.arange(ncols, dtype=np.int64), nrows)
        return MaskView(nrows, ncols, row_ptr, col_idx)


def _validate_pattern(nrows, ncols, row_ptr, col_idx, need_sorted) -> None:
    row_ptr = np.asarray(row_ptr)
    if row_ptr.shape[0] != nrows + 1 or (nrows >= 0 and row_ptr[0] != 0):
        raise SparseError("row_ptr must have nrows+1 entries starting at 0")
    d = np.diff(row_ptr)
    if np.any(d < 0):
        raise SparseError("row_ptr must be non-decreasing")
    nnz = int(row_ptr[nrows])
    if col_idx.shape[0] < nnz:
        raise SparseError("col_idx shorter than nnz")
    cols = np.asarray(col_idx[:nnz], dtype=np.int64)
    if nnz and (cols.min() < 0 or cols.max() >= ncols):
        raise SparseError("column index out of range")
    if need_sorted and nnz > 1:
        # vectorised "strictly increasing inside every row" check
        inc = np.diff(cols) > 0
        row_start = np.zeros(nnz, dtype=bool)
        row_start[row_ptr[:-1][d > 0]] = True
        bad = ~inc & ~row_start[1:]
        if np.any(bad):
            t = int(np.flatnonzero(bad)[0]) + 1
            i = int(np.searchsorted(row_ptr, t, side="right")) - 1
            raise SparseError(f"row {i} not strictly sorted")


# ---------------------------------------------------------------------------
# canonicalising construction (input preparation)
# ---------------------------------------------------------------------------

def _row_ptr_from_rows(nrows: int, rows: np.ndarray) -> np.ndarray:
    row_ptr = np.zeros(nrows + 1, dtype=np.int64)
    if rows.size:
        row_ptr[1:] = np.cumsum(np.bincount(rows, minlength=nrows), dtype=np.int64)
    return row_ptr


def sorted_unique(keys: np.ndarray) -> np.ndarray:
    """np.unique for int64 keys via sort + adjacent-difference (np.unique's
    hash path is orders of magnitude slower on large int64 inputs here)."""
    k = np.sort(np.asarray(keys, dtype=np.int64))
    if k.size == 0:
        return k
    keep = np.empty(k.size, dtype=bool)
    keep[0] = True
    np.not_equal(k[1:], k[:-1], out=keep[1:])
    return k[keep]


def from_arrays(nrows: int, ncols: int, rows, cols, vals, dedup=np.add) -> CsrMatrix:
    """Canonical CSR from coordinate arrays; duplicates combined with ``dedup``.

    Same result as the reference constructor (sparse.py:190-242): entries
    ordered by (row, col), one entry per coordinate, duplicate values added
    with np.add semantics in input order.
    """
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    cols = np.ascontiguousarray(cols, dtype=np.int64)
    vals = np.asarray(vals)
    if not (rows.size == cols.size == vals.size):
        raise SparseError("rows, cols and values must have equal length")
    if rows.size == 0:
        return CsrMatrix(nrows, ncols, np.zeros(nrows + 1, dtype=np.int64),
                         np.empty(0, dtype=np.int64), np.empty(0, dtype=vals.dtype))
    if rows.min() < 0 or rows.max() >= nrows:
        raise SparseError(f"row index out of range [0, {nrows})")
    if cols.min() < 0 or cols.max() >= ncols:
        raise SparseError(f"column index out of range [0, {ncols})")
    # one stable sort on the fused (row, col) key
    key = rows * np.int64(max(ncols, 1)) + cols
    order = np.argsort(key, kind="stable")
    key = key[order]
    vals = vals[order]
    first = np.empty(key.size, dtype=bool)
    first[0] = True
    np.not_equal(key[1:], key[:-1], out=first[1:])
    starts = np.flatnonzero(first)
    ukey = key[starts]
    if starts.size == key.size:
        uvals = vals.copy()
    elif dedup is np.add or dedup is None:
        uvals = np.zeros(starts.size, dtype=vals.dtype)
        np.add.at(uvals, np.cumsum(first) - 1, vals)
    else:
        bounds = np.append(starts, key.size)
        uvals = np.empty(starts.size, dtype=vals.dtype)
        for g in range(starts.size):
            acc = vals[bounds[g]]
            for q in range(bounds[g] + 1, bounds[g + 1]):
                acc = dedup(acc, vals[q])
            uvals[g] = acc
    out_rows = ukey // np.int64(max(ncols, 1))
    out_cols = ukey - out_rows * np.int64(max(ncols, 1))
    return CsrMatrix(nrows, ncols, _row_ptr_from_rows(nrows, out_rows), out_cols, uvals)


def from_triples(nrows: int, ncols: int, triples, dedup=np.add) -> CsrMatrix:
    tl = list(triples)
    if not tl:
        return from_arrays(nrows, ncols, [], [], np.empty(0, dtype=np.float64), dedup)
    return from_arrays(nrows, ncols, [t[0] for t in tl], [t[1] for t in tl],
                       np.asarray([t[2] for t in tl]), dedup)


def _pattern_from_sorted_unique_keys(n_rows: int, n_cols: int, key: np.ndarray, dtype=np.int64):
    rows = key // np.int64(max(n_cols, 1))
    cols = key - rows * np.int64(max(n_cols, 1))
    return CsrMatrix(n_rows, n_cols, _row_ptr_from_rows(n_rows, rows), cols,
                     np.ones(key.size, dtype=dtype))


def to_csc(a: CsrMatrix) -> CscMatrix:
    """Column-major copy; rows ascending inside each column (sparse.py:257-266)."""
    nnz = a.nnz
    cols = np.asarray(a.col_idx[:nnz], dtype=np.int64)
    order = np.argsort(cols, kind="stable")
    rows = np.repeat(np.arange(a.nrows, dtype=np.int64), a.row_lengths())
    col_ptr = _row_ptr_from_rows(a.ncols, cols)
    return CscMatrix(a.nrows, a.ncols, col_ptr, rows[order], a.values[:nnz][order])


def to_csr(a: CscMatrix) -> CsrMatrix:
    nnz = a.nnz
    rows = np.asarray(a.row_idx[:nnz], dtype=np.int64)
    order = np.argsort(rows, kind="stable")
    cols = np.repeat(np.arange(a.ncols, dtype=np.int64), np.diff(a.col_ptr))
    return CsrMatrix(a.nrows, a.ncols, _row_ptr_from_rows(a.nrows, rows), cols[order],
                     a.values[:nnz][order])


def transpose(a: CsrMatrix) -> CsrMatrix:
    c = to_csc(a)
    return CsrMatrix(a.ncols, a.nrows, c.col_ptr, c.row_idx, c.values)


def tril_strict(a: CsrMatrix) -> CsrMatrix:
    """Entries with col < row (sparse.py:285-291); input is canonical so the
    filtered pattern stays canonical without re-sorting."""
    if a.nrows != a.ncols:
        raise SparseError("tril_strict requires a square matrix")
    rows, cols, vals = a.triples()
    keep = cols < rows
    return CsrMatrix(a.nrows, a.ncols, _row_ptr_from_rows(a.nrows, rows[keep]),
                     cols[keep], vals[keep])


def is_pattern_symmetric(a: CsrMatrix) -> bool:
    if a.nrows != a.ncols:
        return False
    t = transpose(a)
    return (np.array_equal(a.row_ptr, t.row_ptr)
            and np.array_equal(a.col_idx[: a.nnz], t.col_idx[: t.nnz]))


def permute_symmetric(a: CsrMatrix, perm: np.ndarray) -> CsrMatrix:
    """P A P^T with perm[new] = old (sparse.py:318-325)."""
    new_label = np.empty(a.nrows, dtype=np.int64)
    new_label[perm] = np.arange(a.nrows, dtype=np.int64)
    rows, cols, vals = a.triples()
    return from_arrays(a.nrows, a.ncols, new_label[rows], new_label[cols], vals)


def degree_sort_relabel(a: CsrMatrix):
    """Non-increasing degree order, ties by ascending index (sparse.py:328-341)."""
    if a.nrows != a.ncols:
        raise SparseError("degree_sort_relabel requires a square matrix")
    deg = a.row_lengths()
    perm = np.lexsort((np.arange(a.nrows), -deg)).astype(np.int64)
    return permute_symmetric(a, perm), perm


def simple_undirected_graph(a: CsrMatrix) -> CsrMatrix:
    """Symmetrise, drop self loops, merge duplicates, unit int64 values
    (sparse.py:344-357)."""
    if a.nrows != a.ncols:
        raise SparseError("a graph adjacency matrix must be square")
    rows, cols, _ = a.triples()
    keep = rows != cols
    rows, cols = rows[keep], cols[keep]
    n = np.int64(max(a.ncols, 1))
    key = np.concatenate([rows * n + cols, cols * n + rows])
    key = sorted_unique(key)
    return _pattern_from_sorted_unique_keys(a.nrows, a.ncols, key)
