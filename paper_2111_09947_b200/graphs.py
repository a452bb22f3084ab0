"""Graph kernels that drive the masked multiply (callers of the hot path).

triangle_count mirrors pkg/src/maskmul/graphs.py:87-96 (relabel by degree,
strict lower triangle L, C = L (.) (L L) under plus-pair int64, sum(C));
k_truss mirrors graphs.py:99-118 (support = G (.) (G G), prune < k-2, repeat).
Graph preparation stays on the host as in the reference (it is excluded from
the timings there too); every multiply and the final reduction run on the GPU.
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np

from .device import DeviceCsr
from .multiply import MultiplyPlan, multiply_device, reduce_sum
from .semiring import plus_pair_semiring
from .sparse import (CsrMatrix, SparseError, degree_sort_relabel, from_arrays,
                     is_pattern_symmetric, tril_strict)


@dataclass
class KernelResult:
    value: object
    multiply_seconds: float = 0.0
    flops: int = 0
    evaluated: int = 0
    multiplies: int = 0
    per_multiply: list = field(default_factory=list)


def _check_simple_symmetric(g: CsrMatrix, what: str) -> None:
    if g.nrows != g.ncols:
        raise SparseError(f"{what} requires a square adjacency matrix")
    if not is_pattern_symmetric(g):
        raise SparseError(f"{what} requires a pattern-symmetric adjacency matrix; "
                          "normalize with simple_undirected_graph() first")
    rows, cols, _ = g.triples()
    if np.any(rows == cols):
        raise SparseError(f"{what} requires a simple graph (no self-loops); "
                          "normalize with simple_undirected_graph() first")


def triangle_count(g: CsrMatrix, plan: MultiplyPlan, device=None) -> KernelResult:
    _check_simple_symmetric(g, "triangle counting")
    low = tril_strict(degree_sort_relabel(g)[0])
    kplan = replace(plan, semiring=plus_pair_semiring(np.int64), complemented=False)
    dl = DeviceCsr.from_host(low, device=device, with_values=False)
    c, st = multiply_device(dl, dl, dl, kplan,
                            b_csc=dl.transpose_storage() if kplan.algorithm == "inner" else None)
    total = int(reduce_sum(c.values).item()) if c.nnz else 0
    return KernelResult(total, st.total_seconds, st.generated_flops, st.evaluated_multiplies, 1,
                        [(st.total_seconds, st.generated_flops)])


def k_truss(g: CsrMatrix, k: int, plan: MultiplyPlan, device=None) -> KernelResult:
    """Edges with support >= k-2, pruned to a fixed point (graphs.py:99-118).

    The whole loop stays on the device: support = G (.) (G G) under
    plus-pair, then mm_filter_min keeps the entries with support >= k-2 as
    the next (canonical) graph; one nnz readback per iteration decides the
    fixed point.  Only the final graph comes back to the host."""
    import ctypes as C

    import torch

    from . import _lib
    from .multiply import _raise

    if k < 3:
        raise ValueError("k-truss needs k >= 3")
    _check_simple_symmetric(g, "k-truss")
    kplan = replace(plan, semiring=plus_pair_semiring(np.int64), complemented=False)
    res = KernelResult(None)
    cur = DeviceCsr.from_host(g, device=device, with_values=False)
    lib = _lib.load()
    while cur.nnz:
        sup, st = multiply_device(cur, cur, cur, kplan,
                                  b_csc=cur.transpose_storage() if kplan.algorithm == "inner" else None)
        res.multiply_seconds += st.total_seconds
        res.flops += st.generated_flops
        res.evaluated += st.evaluated_multiplies
        res.multiplies += 1
        res.per_multiply.append((st.total_seconds, st.generated_flops))
        dev = sup.idx.device
        ptr = torch.empty(cur.nrows + 1, dtype=torch.int64, device=dev)
        idx = torch.empty(max(sup.nnz, 1), dtype=torch.int32, device=dev)
        nnz = C.c_int64(0)
        rc = lib.mm_filter_min(C.byref(sup.mm()), k - 2, ptr.data_ptr(), idx.data_ptr(), C.byref(nnz),
                               C.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
        if rc:
            _raise(rc)
        if int(nnz.value) == cur.nnz:
            break
        cur = DeviceCsr(cur.nrows, cur.ncols, ptr, idx[: int(nnz.value)].contiguous(), None)
    host = cur.to_host()
    host.values = np.ones(host.nnz, dtype=np.int64)
    res.value = host
    return res
