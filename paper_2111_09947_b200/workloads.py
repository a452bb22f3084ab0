"""Seeded synthetic inputs: the generators and the five BASELINE configs.

Host-side input preparation (the reference excludes it from every timing).
The generators restate the reference's published recipes so the GPU box can
rebuild bit-identical inputs without /root/reference:

* R-MAT, one quadrant draw per bit (pkg/src/maskmul/generate.py:52-65,
  Graph500 (a,b,c,d) = (0.57, 0.19, 0.19, 0.05), :16)
* Erdős–Rényi pairs with replacement (generate.py:68-73)
* duplicates merged, unit values (generate.py:76-88)

Config recipes are SURVEY.md §8(d); tests/golden/configs.json pins every
generated input by digest against the reference's own generator output.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .semiring import arithmetic_semiring, plus_pair_semiring
from .sparse import CsrMatrix, from_arrays, sorted_unique

GRAPH500_PARAMS = (0.57, 0.19, 0.19, 0.05)


@dataclass(frozen=True)
class GeneratorSpec:
    kind: str
    scale: int
    avg_degree: float
    rmat_params: tuple = GRAPH500_PARAMS
    seed: int = 0

    def __post_init__(self):
        if self.kind not in ("erdos-renyi", "rmat"):
            raise ValueError(f"unknown generator kind {self.kind!r}")
        if self.scale < 1:
            raise ValueError("scale must be >= 1")
        if not self.avg_degree > 0:
            raise ValueError("avg_degree must be > 0")
        if abs(sum(self.rmat_params) - 1.0) > 1e-9:
            raise ValueError("rmat_params must sum to 1 within 1e-9")

    @property
    def nrows(self) -> int:
        return 1 << self.scale

    @property
    def nedges(self) -> int:
        return int(round(self.avg_degree * self.nrows))


def rmat_edges(spec: GeneratorSpec):
    a, b, c, _ = spec.rmat_params
    cuts = np.array([a, a + b, a + b + c])
    rng = np.random.default_rng(spec.seed)
    m = spec.nedges
    wide = spec.scale > 31
    src = np.zeros(m, dtype=np.int64 if wide else np.uint32)
    dst = np.zeros(m, dtype=np.int64 if wide else np.uint32)
    for bit in range(spec.scale):
        r = rng.random(m)
        # == np.searchsorted(cuts, r, side="right") (generate.py:62): the
        # number of cut points <= r, computed branch-free in uint8
        quad = ((r >= cuts[0]).view(np.uint8) + (r >= cuts[1]).view(np.uint8)
                + (r >= cuts[2]).view(np.uint8))
        src |= (quad >> 1).astype(src.dtype) << src.dtype.type(bit)
        dst |= (quad & 1).astype(dst.dtype) << dst.dtype.type(bit)
    return src.astype(np.int64), dst.astype(np.int64)


def erdos_renyi_edges(spec: GeneratorSpec):
    rng = np.random.default_rng(spec.seed)
    n = spec.nrows
    src = rng.integers(0, n, spec.nedges, dtype=np.int64)
    dst = rng.integers(0, n, spec.nedges, dtype=np.int64)
    return src, dst


def _unique_keys(keys: np.ndarray) -> np.ndarray:
    """Sorted unique int64 keys.  Input preparation only: on a GPU box the
    sort runs on the device through torch (same set, same order)."""
    try:
        import torch
        if torch.cuda.is_available() and keys.size > (1 << 20):
            t = torch.from_numpy(np.ascontiguousarray(keys)).cuda()
            return torch.unique(t, sorted=True).cpu().numpy()
    except Exception:
        pass
    return sorted_unique(keys)


def _csr_from_keys(n_rows: int, n_cols: int, key: np.ndarray) -> CsrMatrix:
    rows = key // n_cols
    cols = key - rows * n_cols
    row_ptr = np.zeros(n_rows + 1, dtype=np.int64)
    row_ptr[1:] = np.cumsum(np.bincount(rows, minlength=n_rows))
    return CsrMatrix(n_rows, n_cols, row_ptr, cols, np.ones(key.size, dtype=np.int64))


def generate(spec: GeneratorSpec) -> CsrMatrix:
    src, dst = rmat_edges(spec) if spec.kind == "rmat" else erdos_renyi_edges(spec)
    n = spec.nrows
    return _csr_from_keys(n, n, _unique_keys(src * np.int64(n) + dst))


def simple_graph_direct(spec: GeneratorSpec) -> CsrMatrix:
    """simple_undirected_graph(generate(spec)) in one pass: dedup of the raw
    edges followed by symmetrise + dedup is the dedup of the symmetrised raw
    edges, so the result is the identical canonical CSR."""
    src, dst = rmat_edges(spec) if spec.kind == "rmat" else erdos_renyi_edges(spec)
    n = np.int64(spec.nrows)
    keep = src != dst
    src, dst = src[keep], dst[keep]
    key = _unique_keys(np.concatenate([src * n + dst, dst * n + src]))
    return _csr_from_keys(spec.nrows, spec.nrows, key)


# ---------------------------------------------------------------------------
# BASELINE.json configs
# ---------------------------------------------------------------------------

@dataclass
class Workload:
    name: str
    mask: object          # MaskView
    a: CsrMatrix
    b: CsrMatrix
    semiring: object
    complemented: bool
    description: str


def cfg1() -> Workload:
    a = generate(GeneratorSpec("erdos-renyi", 12, 8, seed=0)).astype(np.float64)
    a.values[:] = np.random.default_rng(1).random(a.nnz)
    return Workload("cfg1", a.pattern(), a, a, arithmetic_semiring(np.float64), False,
                    "ER n=4096 d8, M=A=B, fp64 U(0,1), plus-times")


def triangle_lower(scale: int = 20, degree: float = 16, seed: int = 0) -> CsrMatrix:
    """tril_strict(degree_sort_relabel(simple_undirected_graph(rmat))[0])
    (graphs.py:91-92) computed on keys: relabel by non-increasing degree
    (ties by index, sparse.py:340) and keep new_col < new_row."""
    g = simple_graph_direct(GeneratorSpec("rmat", scale, degree, seed=seed))
    n = g.nrows
    deg = np.diff(g.row_ptr)
    perm = np.lexsort((np.arange(n), -deg)).astype(np.int64)
    new_label = np.empty(n, dtype=np.int64)
    new_label[perm] = np.arange(n, dtype=np.int64)
    rows = np.repeat(np.arange(n, dtype=np.int64), deg)
    nr = new_label[rows]
    nc = new_label[g.col_idx]
    keep = nc < nr
    key = _unique_keys(nr[keep] * np.int64(n) + nc[keep])
    return _csr_from_keys(n, n, key)


def cfg2(scale: int = 20) -> Workload:
    low = triangle_lower(scale)
    return Workload("cfg2", low.pattern(), low, low, plus_pair_semiring(np.int64), False,
                    f"triangle count R-MAT s{scale} ef16, L=tril(relabel(G)), C=L.(L L) plus-pair")


def cfg3(mask_degree: int) -> Workload:
    a = generate(GeneratorSpec("erdos-renyi", 18, 16, seed=0)).astype(np.float64)
    a.values[:] = np.random.default_rng(100).random(a.nnz)
    b = generate(GeneratorSpec("erdos-renyi", 18, 16, seed=1)).astype(np.float64)
    b.values[:] = np.random.default_rng(101).random(b.nnz)
    m = generate(GeneratorSpec("erdos-renyi", 18, mask_degree, seed=2))
    return Workload(f"cfg3_d{mask_degree}", m.pattern(), a, b, arithmetic_semiring(np.float64),
                    False, f"ER 2^18 d16 fp64, mask d={mask_degree}")


def cfg4() -> Workload:
    g = simple_graph_direct(GeneratorSpec("rmat", 18, 16, seed=0))
    n = g.nrows
    rng = np.random.default_rng(4)
    src = rng.choice(n, 512, replace=False)
    ft = from_arrays(512, n, np.arange(512), src, np.ones(512, dtype=np.int64))
    # V = (rng.random((512, n)) < 0.05), drawn row block by row block to
    # bound host memory; the PCG64 double stream is consumed in the same order
    rows_l, cols_l = [], []
    for r0 in range(0, 512, 64):
        blk = rng.random((64, n)) < 0.05
        r, c = np.nonzero(blk)
        rows_l.append(r + r0)
        cols_l.append(c)
    rows = np.concatenate(rows_l)
    cols = np.concatenate(cols_l)
    row_ptr = np.zeros(513, dtype=np.int64)
    row_ptr[1:] = np.cumsum(np.bincount(rows, minlength=512))
    v = CsrMatrix(512, n, row_ptr, cols.astype(np.int64), np.ones(cols.size, dtype=np.int64))
    return Workload("cfg4", v.pattern(complemented=True), ft, g, arithmetic_semiring(np.int64),
                    True, "BFS step C = not(V) . (F^T A), 512 sources, R-MAT s18, int64")


def cfg5(scale: int = 22) -> Workload:
    g = simple_graph_direct(GeneratorSpec("rmat", scale, 16, seed=0))
    return Workload("cfg5", g.pattern(), g, g, plus_pair_semiring(np.int64), False,
                    f"k-truss support R-MAT s{scale} ef16, C=A.(A A) plus-pair")
