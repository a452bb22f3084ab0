"""Batched betweenness centrality on the CPU — TEST INFRASTRUCTURE ONLY.

Restates the reference driver ``betweenness_centrality`` (pkg/src/maskmul/
graphs.py:136-200) with the C oracle's masked multiplies and numpy forms of
``ewise_add`` (sparse.py:360-370, dedup add of the lexsorted concatenation,
sparse.py:190-244) and ``lookup_rows`` (_kernels.py:597-612).  Pinned to the
reference by tests/golden/bc.json (scores frozen bit for bit by running the
reference itself); the GPU driver (paper_2111_09947_b200.graphs) is checked
against the same fixtures.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .oracle import masked_multiply


@dataclass
class _Csr:
    nrows: int
    ncols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def rows(self) -> np.ndarray:
        return np.repeat(np.arange(self.nrows, dtype=np.int64), np.diff(self.row_ptr))


def _from_sorted_unique(nrows, ncols, rows, cols, vals) -> _Csr:
    ptr = np.zeros(nrows + 1, dtype=np.int64)
    np.add.at(ptr, rows + 1, 1)
    return _Csr(nrows, ncols, np.cumsum(ptr), cols.astype(np.int64), vals)


def ewise_add(a: _Csr, b: _Csr) -> _Csr:
    """sparse.py:360-370 — union, coinciding entries added (0 + a + b order
    of np.add.at into zeros, sparse.py:205-208)."""
    r = np.concatenate([a.rows(), b.rows()])
    c = np.concatenate([a.col_idx[: a.nnz], b.col_idx[: b.nnz]])
    v = np.concatenate([a.values[: a.nnz], b.values[: b.nnz]]).astype(np.float64)
    if r.size == 0:
        return _Csr(a.nrows, a.ncols, np.zeros(a.nrows + 1, dtype=np.int64), np.empty(0, np.int64),
                    np.empty(0, np.float64))
    order = np.lexsort((c, r))
    r, c, v = r[order], c[order], v[order]
    new = np.empty(r.size, dtype=bool)
    new[0] = True
    new[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
    starts = np.flatnonzero(new)
    if starts.size == r.size:
        out = v.copy()
    else:
        seg = np.cumsum(new) - 1
        out = np.zeros(starts.size, dtype=np.float64)
        np.add.at(out, seg, v)
    return _from_sorted_unique(a.nrows, a.ncols, r[starts], c[starts], out)


def values_at(ptr, idx, y: _Csr) -> np.ndarray:
    """graphs._values_at / lookup_rows: Y's values at a pattern, 0 if absent."""
    out = np.zeros(idx.shape[0], dtype=np.float64)
    for i in range(ptr.shape[0] - 1):
        s, e = int(ptr[i]), int(ptr[i + 1])
        if s == e:
            continue
        ys, ye = int(y.row_ptr[i]), int(y.row_ptr[i + 1])
        cols = y.col_idx[ys:ye]
        q = np.searchsorted(cols, idx[s:e])
        hit = q < cols.size
        hit[hit] = cols[q[hit]] == idx[s:e][hit]
        out[s:e][hit] = y.values[ys:ye][q[hit]]
    return out


def _mm(mask: _Csr, a: _Csr, b: _Csr, comp: bool, algorithm: str):
    r = masked_multiply(mask, a, b, algorithm=algorithm, complemented=comp, semiring_id=0,
                        dtype=np.float64)
    return _Csr(mask.nrows, mask.ncols, r.row_ptr, r.col_idx, r.values), r


def betweenness_centrality(g, batch_size: int, sources=None, algorithm: str = "msa"):
    """graphs.py:136-200 on the oracle.  Returns (scores, multiplies,
    generated flops, evaluated multiplies)."""
    n = g.nrows
    adj = _Csr(n, n, np.asarray(g.row_ptr, np.int64), np.asarray(g.col_idx[: g.nnz], np.int64),
               np.asarray(g.values[: g.nnz], np.float64))
    # adj^T as CSR: stable transpose (sparse.py:257-283)
    order = np.argsort(adj.col_idx[: adj.nnz], kind="stable")
    t_ptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(t_ptr, adj.col_idx[: adj.nnz] + 1, 1)
    adj_t = _Csr(n, n, np.cumsum(t_ptr), adj.rows()[order], adj.values[order])
    src = np.arange(n, dtype=np.int64) if sources is None else np.asarray(list(sources), np.int64)
    scores = np.zeros(n, dtype=np.float64)
    count = flops = evaluated = 0
    for lo in range(0, src.size, batch_size):
        batch = src[lo: lo + batch_size]
        b = batch.size
        order_b = np.argsort(batch, kind="stable")
        sigma = _from_sorted_unique(n, b, batch[order_b], order_b.astype(np.int64), np.ones(b))
        paths = sigma
        frontiers = [sigma]
        while True:
            nxt, st = _mm(paths, adj_t, frontiers[-1], True, algorithm)
            count += 1
            flops += st.generated_flops
            evaluated += st.evaluated_multiplies
            if nxt.nnz == 0:
                break
            paths = ewise_add(paths, nxt)
            frontiers.append(nxt)
        delta = _Csr(n, b, np.zeros(n + 1, np.int64), np.empty(0, np.int64), np.empty(0, np.float64))
        for t in range(len(frontiers) - 1, 0, -1):
            sig_t, sig_prev = frontiers[t], frontiers[t - 1]
            d_at = values_at(sig_t.row_ptr, sig_t.col_idx, delta)
            p_at = values_at(sig_t.row_ptr, sig_t.col_idx, paths)
            w = _Csr(n, b, sig_t.row_ptr, sig_t.col_idx, (1.0 + d_at) / p_at)
            wq, st = _mm(sig_prev, adj, w, False, algorithm)
            count += 1
            flops += st.generated_flops
            evaluated += st.evaluated_multiplies
            contrib = wq.values[: wq.nnz] * values_at(wq.row_ptr, wq.col_idx, paths)
            delta = ewise_add(delta, _Csr(n, b, wq.row_ptr, wq.col_idx, contrib))
        np.add.at(scores, delta.rows(), delta.values[: delta.nnz])
        own_ptr = np.zeros(n + 1, dtype=np.int64)
        np.add.at(own_ptr, batch + 1, 1)
        np.subtract.at(scores, batch[order_b], values_at(np.cumsum(own_ptr), order_b.astype(np.int64), delta))
    return scores, count, flops, evaluated
