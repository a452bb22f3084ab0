"""Graph kernels that drive the masked multiply (callers of the hot path).

triangle_count mirrors pkg/src/maskmul/graphs.py:87-96 (relabel by degree,
strict lower triangle L, C = L (.) (L L) under plus-pair int64, sum(C));
k_truss mirrors graphs.py:99-118 (support = G (.) (G G), prune < k-2, repeat);
betweenness_centrality mirrors graphs.py:136-200 (batched Brandes: forward
frontier expansion with a complemented mask, backward dependency
accumulation with a plain mask), every step on the device.
Graph preparation stays on the host as in the reference (it is excluded from
the timings there too); every multiply and the final reduction run on the GPU.
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace
from typing import Sequence

import numpy as np

from .device import DeviceCsr
from .multiply import MultiplyPlan, PlanError, multiply_device, reduce_sum
from .semiring import arithmetic_semiring, plus_pair_semiring
from .sparse import CsrMatrix, SparseError


@dataclass(frozen=True)
class BcConfig:
    """graphs.py:26-38."""
    batch_size: int = 512
    sources: Sequence[int] | None = None  # None: every vertex is a source

    def __post_init__(self):
        if self.batch_size < 1:
            raise ValueError("batch_size must be >= 1")
        if self.sources is not None:
            src = list(self.sources)
            if len(set(src)) != len(src):
                raise ValueError("sources must be distinct")


@dataclass
class KernelResult:
    value: object
    multiply_seconds: float = 0.0
    flops: int = 0
    evaluated: int = 0
    multiplies: int = 0
    per_multiply: list = field(default_factory=list)


def _simple_symmetric_on_device(g: CsrMatrix, what: str, device) -> DeviceCsr:
    """Upload the pattern and run graphs.py:75-84's checks on the device: square,
    pattern-symmetric (equal to its own canonical transpose, built by
    prep.transpose as is_pattern_symmetric does on the host, sparse.py:294-300),
    no self-loops.  Same errors as the reference; the host transpose of a
    scale-22 graph took longer than the whole k-truss on the device."""
    import torch

    from . import prep
    if g.nrows != g.ncols:
        raise SparseError(f"{what} requires a square adjacency matrix")
    dg = DeviceCsr.from_host(g, device=device, with_values=False)
    t = prep.transpose(dg)
    if not (torch.equal(t.ptr, dg.ptr) and torch.equal(t.idx, dg.idx)):
        raise SparseError(f"{what} requires a pattern-symmetric adjacency matrix; "
                          "normalize with simple_undirected_graph() first")
    if dg.nnz and bool((prep.expand_rows(dg) == dg.idx).any()):
        raise SparseError(f"{what} requires a simple graph (no self-loops); "
                          "normalize with simple_undirected_graph() first")
    return dg


def triangle_count(g: CsrMatrix, plan: MultiplyPlan, device=None) -> KernelResult:
    """graphs.py:87-96.  The relabel + strict lower triangle run on the device
    (prep.triangle_lower, identical to the host tril_strict(degree_sort_relabel))."""
    from . import prep
    dg = _simple_symmetric_on_device(g, "triangle counting", device)
    kplan = replace(plan, semiring=plus_pair_semiring(np.int64), complemented=False)
    dl = prep.triangle_lower(dg)
    c, st = multiply_device(dl, dl, dl, kplan,
                            b_csc=dl.transpose_storage() if kplan.algorithm == "inner" else None)
    total = int(reduce_sum(c.values).item()) if c.nnz else 0
    return KernelResult(total, st.total_seconds, st.generated_flops, st.evaluated_multiplies, 1,
                        [(st.total_seconds, st.generated_flops)])


_copy_streams: dict = {}


def triangle_count_lower_streamed(h_ptr, h_idx, plan: MultiplyPlan, device=None, first_fraction=0.2,
                                  buffers=None) -> KernelResult:
    """sum(L (.) (L L)) for a HOST-resident strict lower triangle L, the upload
    pipelined with the multiply (graphs.py:87-96 from the multiply on).

    h_ptr (int64, nrows + 1) and h_idx (int32, nnz) are pinned host tensors of
    L = tril_strict(relabelled graph).  Rows are independent (multiply.py:8-11)
    and every k in L_i is smaller than i, so rows [0, r) of C touch only rows
    [0, r) of B = L: the first ``first_fraction`` of L's entries is uploaded,
    its row block is multiplied while the rest of L is still on the wire, then
    the second block runs.  Same products, same C rows, same count as one
    multiply (tests/test_gpu_graph_ops.py); only the upload overlaps.
    ``first_fraction`` may be a sequence of increasing shares (cut points):
    (0.05, 0.25) uploads and multiplies three row blocks.
    ``buffers`` = (ptr, idx) device tensors to upload into (else allocated).
    (Running the second block from a helper thread on a second stream, so the
    two multiplies overlap, measured 1.5 % faster on average but erratic —
    5.6 to 6.8 ms on cfg2 — and was dropped.)"""
    import torch

    from .distributed import row_block
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    m = int(h_ptr.numel()) - 1
    ptr_np = h_ptr.numpy()
    nnz = int(ptr_np[-1])
    kplan = replace(plan, semiring=plus_pair_semiring(np.int64), complemented=False)
    if buffers is None:
        d_ptr = torch.empty(m + 1, dtype=torch.int64, device=dev)
        d_idx = torch.empty(nnz, dtype=torch.int32, device=dev)
    else:
        d_ptr, d_idx = buffers
    # cut rows: the first row whose offset reaches each requested share of the entries
    shares = [first_fraction] if np.isscalar(first_fraction) else list(first_fraction)
    if kplan.algorithm == "inner":
        shares = []   # the pull path transposes all of B first: nothing to overlap
    cuts = [0]
    for f in shares:
        r = int(np.searchsorted(ptr_np, int(min(max(float(f), 0.0), 1.0) * nnz), side="left"))
        cuts.append(min(max(r, cuts[-1]), m))
    cuts.append(m)
    offs = [int(ptr_np[r]) for r in cuts]
    cur = torch.cuda.current_stream(dev)
    cs = _copy_streams.get(dev.index)
    if cs is None:
        cs = _copy_streams[dev.index] = torch.cuda.Stream(dev)
    cs.wait_stream(cur)
    events = []
    with torch.cuda.stream(cs):
        for q in range(len(cuts) - 1):
            lo, hi, q0, q1 = cuts[q], cuts[q + 1], offs[q], offs[q + 1]
            # a block reads row offsets up to its last row only (its own rows and the B rows above them)
            p_lo = lo + 1 if q else 0
            if hi + 1 > p_lo:
                d_ptr[p_lo: hi + 1].copy_(h_ptr[p_lo: hi + 1], non_blocking=True)
            if q1 > q0:
                d_idx[q0:q1].copy_(h_idx[q0:q1], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cs)
            events.append(ev)
    full = DeviceCsr(m, m, d_ptr, d_idx, None)
    res = KernelResult(0)
    total = None
    for q, ev in enumerate(events):
        lo, hi, q0, q1 = cuts[q], cuts[q + 1], offs[q], offs[q + 1]
        cur.wait_event(ev)
        if hi == lo:
            continue
        blk = row_block(full, lo, hi, q0, q1)
        c, st = multiply_device(blk, blk, full, kplan,
                                b_csc=full.transpose_storage() if kplan.algorithm == "inner" else None)
        if c.nnz:
            t = reduce_sum(c.values)
            total = t if total is None else total + t
        res.multiply_seconds += st.total_seconds
        res.flops += st.generated_flops
        res.evaluated += st.evaluated_multiplies
        res.multiplies += 1
        res.per_multiply.append((st.total_seconds, st.generated_flops))
    res.value = int(total.item()) if total is not None else 0
    cur.wait_stream(cs)
    return res


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
    cur = _simple_symmetric_on_device(g, "k-truss", device)
    kplan = replace(plan, semiring=plus_pair_semiring(np.int64), complemented=False)
    res = KernelResult(None)
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


def _record(res: KernelResult, st) -> None:
    res.multiply_seconds += st.total_seconds
    res.flops += st.generated_flops
    res.evaluated += st.evaluated_multiplies
    res.multiplies += 1
    res.per_multiply.append((st.total_seconds, st.generated_flops))


def betweenness_centrality(g: CsrMatrix, cfg: BcConfig, plan: MultiplyPlan, device=None) -> KernelResult:
    """Batched multi-source Brandes over masked multiplies (graphs.py:136-200).

    Forward: next = not(paths) (.) (A^T frontier) under plus-times float64,
    paths += next, until the frontier is empty.  Backward, level by level:
    w = (1 + delta) / paths on the level's pattern, wq = prev_level (.) (A w),
    delta += wq * paths.  Scores add each batch's delta rows and drop a
    source's own entry.  Everything after the graph upload stays in HBM; one
    nnz readback per multiply / union decides sizes.  Unnormalised, directed
    convention summed over the sources, like the reference.
    """
    import torch

    from . import elementwise as ew

    if plan.algorithm in ("mca", "inner"):
        raise PlanError(f"{plan.algorithm} does not support the complemented "
                        "masked multiplies betweenness centrality needs")
    if g.nrows != g.ncols:
        raise SparseError("betweenness centrality requires a square adjacency matrix")
    n = g.nrows
    sources = (np.arange(n, dtype=np.int64) if cfg.sources is None
               else np.asarray(list(cfg.sources), dtype=np.int64))
    if sources.size and (sources.min() < 0 or sources.max() >= n):
        raise SparseError("source vertex out of range")
    sem = arithmetic_semiring(np.float64)
    fwd_plan = replace(plan, semiring=sem, complemented=True)
    bwd_plan = replace(plan, semiring=sem, complemented=False)
    adj = DeviceCsr.from_host(g, dtype=np.float64, device=device)
    dev = adj.idx.device
    t = adj.transpose_storage()          # A^T as CSR, hoisted once (graphs.py:160)
    adj_t = DeviceCsr(n, n, t.ptr, t.idx, t.values)
    res = KernelResult(None)
    scores = torch.zeros(n, dtype=torch.float64, device=dev)
    src_col = torch.full((n,), -1, dtype=torch.int32, device=dev)
    for lo in range(0, sources.size, cfg.batch_size):
        batch = sources[lo: lo + cfg.batch_size]
        b = int(batch.size)
        order = np.argsort(batch, kind="stable")
        ptr = np.zeros(n + 1, dtype=np.int64)
        np.add.at(ptr, batch + 1, 1)
        sigma = DeviceCsr(n, b, torch.from_numpy(np.cumsum(ptr)).to(dev),
                          torch.from_numpy(order.astype(np.int32)).to(dev),
                          torch.ones(b, dtype=torch.float64, device=dev))
        paths = sigma
        frontiers = [sigma]
        while True:
            nxt, st = multiply_device(paths, adj_t, frontiers[-1], fwd_plan, complemented=True)
            _record(res, st)
            if nxt.nnz == 0:
                break
            paths = ew.ewise_add(paths, nxt)
            frontiers.append(nxt)
        delta = DeviceCsr(n, b, torch.zeros(n + 1, dtype=torch.int64, device=dev),
                          torch.empty(0, dtype=torch.int32, device=dev),
                          torch.empty(0, dtype=torch.float64, device=dev))
        for lvl in range(len(frontiers) - 1, 0, -1):
            sig_t, sig_prev = frontiers[lvl], frontiers[lvl - 1]
            w = DeviceCsr(n, b, sig_t.ptr, sig_t.idx, ew.bc_dependency_weights(sig_t, delta, paths))
            wq, st = multiply_device(sig_prev, adj, w, bwd_plan)
            _record(res, st)
            contrib = DeviceCsr(n, b, wq.ptr, wq.idx, ew.bc_scale_by(wq, paths))
            delta = ew.ewise_add(delta, contrib)
        bt = torch.from_numpy(batch).to(dev)
        src_col[bt] = torch.arange(b, dtype=torch.int32, device=dev)
        ew.bc_accumulate(delta, src_col, scores)
        src_col[bt] = -1
    res.value = scores.cpu().numpy()
    return res
