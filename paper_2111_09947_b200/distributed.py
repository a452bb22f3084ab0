"""Row partitioning of the masked multiply across GPUs (one process per GPU).

Rows of C are independent (the reference computes each output row from A_i,
M_i and the referenced B rows only: multiply.py:8-11), so the multi-GPU form
is a row-block partition:

* A and M are cut into contiguous row blocks of balanced masked work
  (w_i = flops_i + nnz(M_i), prefix-sum cuts — ``balanced_cuts``), then
  re-balanced by the kernels' measured cost: each block's weights are scaled
  by its measured time over its predicted work and the cuts recomputed
  (``refine_cuts``; bench.py does this during warm-up, since search-mode and
  sliced hub rows cost far less / more than their flops);
* B is replicated: rank 0 broadcasts it once over NCCL (NVLink/NVSwitch);
* each rank multiplies its block with no data-path collective;
* C row blocks concatenate (``concat_row_blocks`` / ``gather_to_rank0``),
  and the triangle count is an NCCL all-reduce of the per-rank sums.

The partition logic is pure host/torch code and is exercised on CPU with the
gloo backend (tests/test_distributed_gloo.py).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .device import DeviceCsr


def balanced_cuts(work: np.ndarray, parts: int) -> np.ndarray:
    """Row cut points [0, c1, ..., nrows] splitting sum(work) into `parts`
    contiguous blocks of (nearly) equal weight (integer or float weights)."""
    work = np.asarray(work)
    work = work.astype(np.float64 if work.dtype.kind == "f" else np.int64, copy=False)
    n = work.shape[0]
    if parts <= 1 or n == 0:
        return np.array([0, n], dtype=np.int64)
    cum = np.concatenate([[0], np.cumsum(work)])
    total = cum[-1]
    if total == 0:
        return np.linspace(0, n, parts + 1).astype(np.int64)
    targets = total * np.arange(1, parts, dtype=np.float64) / parts
    inner = np.searchsorted(cum, targets, side="left").astype(np.int64)
    cuts = np.concatenate([[0], np.clip(inner, 0, n), [n]])
    return np.maximum.accumulate(cuts)


def refine_cuts(work: np.ndarray, cuts, block_cost, parts: int | None = None) -> np.ndarray:
    """Cost-aware re-cut: scale the weights of every block [cuts[r],
    cuts[r+1]) by block_cost[r] / sum(work in block) — the measured cost per
    unit of predicted work, piecewise constant per block — and recompute the
    balanced cuts.  Blocks with no predicted work keep their weights."""
    w = np.asarray(work, dtype=np.float64).copy()
    cuts = np.asarray(cuts, dtype=np.int64)
    for r in range(len(cuts) - 1):
        lo, hi = int(cuts[r]), int(cuts[r + 1])
        tot = w[lo:hi].sum()
        if hi > lo and tot > 0:
            w[lo:hi] *= float(block_cost[r]) / tot
    return balanced_cuts(w, parts or len(cuts) - 1)


def imbalance(block_cost) -> float:
    """max / mean of per-block costs (1.0 = perfect balance)."""
    c = np.asarray(block_cost, dtype=np.float64)
    return float(c.max() / c.mean()) if c.size and c.mean() > 0 else 1.0


def row_work(a_row_ptr: np.ndarray, a_col_idx: np.ndarray, b_row_ptr: np.ndarray,
             m_row_ptr: np.ndarray) -> np.ndarray:
    """w_i = flops_i + nnz(M_i) (host numpy; flops_per_row of multiply.py:103-108)."""
    blen = np.diff(b_row_ptr)
    per = blen[a_col_idx[: int(a_row_ptr[-1])]]
    cs = np.zeros(per.size + 1, dtype=np.int64)
    np.cumsum(per, out=cs[1:])
    flops = cs[a_row_ptr[1:]] - cs[a_row_ptr[:-1]]
    return flops + np.diff(m_row_ptr)


def row_block(m: DeviceCsr, lo: int, hi: int, p0: int | None = None, p1: int | None = None) -> DeviceCsr:
    """Rows [lo, hi) of a device CSR as a standalone CSR (views + rebased ptr).
    p0 / p1 = ptr[lo] / ptr[hi] when the caller already knows them (no host
    sync); else they are read back."""
    if p0 is None or p1 is None:
        p0, p1 = (int(x) for x in m.ptr[torch.tensor([lo, hi], device=m.ptr.device)].tolist())
    ptr = m.ptr[lo: hi + 1] - p0
    vals = m.values[p0:p1] if m.values is not None else None
    return DeviceCsr(hi - lo, m.ncols, ptr.contiguous(), m.idx[p0:p1], vals)


def cut_offsets(m: DeviceCsr, cuts) -> list[int]:
    """ptr[c] for every cut c, in one device->host read."""
    idx = torch.as_tensor(np.asarray(cuts, dtype=np.int64), device=m.ptr.device)
    return [int(x) for x in m.ptr[idx].tolist()]


def row_blocks(m: DeviceCsr, cuts, offsets: list[int] | None = None) -> list[DeviceCsr]:
    """Every row block [cuts[r], cuts[r+1]) of m (one host read for all of
    them, none when the offsets are given)."""
    offsets = cut_offsets(m, cuts) if offsets is None else offsets
    return [row_block(m, int(cuts[r]), int(cuts[r + 1]), offsets[r], offsets[r + 1])
            for r in range(len(cuts) - 1)]


def concat_row_blocks(parts: list[DeviceCsr]) -> DeviceCsr:
    """Stack row blocks (in order) into one CSR."""
    offs = [0]
    for p in parts:
        offs.append(offs[-1] + p.nnz)
    ptrs = [parts[0].ptr[:1]] + [p.ptr[1:] + off for p, off in zip(parts, offs[:-1])]
    ptr = torch.cat(ptrs)
    idx = torch.cat([p.idx for p in parts])
    vals = None if parts[0].values is None else torch.cat([p.values for p in parts])
    return DeviceCsr(sum(p.nrows for p in parts), parts[0].ncols, ptr, idx, vals)


def row_work_device(a: DeviceCsr, b: DeviceCsr, m: DeviceCsr) -> torch.Tensor:
    """w_i = flops_i + nnz(M_i) on the device (mm_row_work), the same numbers
    as ``row_work`` without a host round trip of A."""
    import ctypes as C

    from . import _lib
    from .multiply import _raise
    w = torch.empty(max(a.nrows, 1), dtype=torch.int64, device=a.idx.device)
    rc = _lib.load().mm_row_work(C.byref(a.mm()), C.byref(b.mm()), C.byref(m.mm()), None, w.data_ptr(),
                                 C.c_void_p(torch.cuda.current_stream(a.idx.device).cuda_stream))
    if rc:
        _raise(rc)
    return w[: a.nrows]


def broadcast_csr(m: DeviceCsr | None, src: int, device, meta_dtype=None) -> DeviceCsr:
    """Replicate a CSR from rank `src` to every rank (NCCL broadcast on GPU,
    gloo on CPU).  Non-source ranks pass m=None."""
    rank = dist.get_rank()
    meta = torch.zeros(5, dtype=torch.int64, device=device)
    if rank == src:
        meta[0], meta[1], meta[2] = m.nrows, m.ncols, m.nnz
        meta[3] = 0 if m.values is None else (2 if m.values.dtype == torch.float64 else 1)
    dist.broadcast(meta, src)
    nrows, ncols, nnz, vk = (int(x) for x in meta[:4].tolist())
    if rank == src:
        ptr, idx, vals = m.ptr, m.idx, m.values
    else:
        ptr = torch.empty(nrows + 1, dtype=torch.int64, device=device)
        idx = torch.empty(nnz, dtype=torch.int32, device=device)
        vals = (None if vk == 0 else
                torch.empty(nnz, dtype=torch.float64 if vk == 2 else torch.int64, device=device))
    dist.broadcast(ptr, src)
    if nnz:
        dist.broadcast(idx, src)
        if vals is not None:
            dist.broadcast(vals, src)
    return DeviceCsr(nrows, ncols, ptr, idx, vals)


def allreduce_sum_(t: torch.Tensor) -> torch.Tensor:
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t


def gather_to_rank0(part: DeviceCsr, device) -> DeviceCsr | None:
    """Concatenate every rank's C row block on rank 0 (all_gather of sizes,
    then point-to-point transfers of the blocks)."""
    world = dist.get_world_size()
    rank = dist.get_rank()
    meta = torch.tensor([part.nrows, part.nnz], dtype=torch.int64, device=device)
    metas = [torch.zeros_like(meta) for _ in range(world)]
    dist.all_gather(metas, meta)
    if rank != 0:
        dist.send(part.ptr, 0)
        if part.nnz:
            dist.send(part.idx, 0)
            dist.send(part.values, 0)
        return None
    parts = [part]
    for r in range(1, world):
        nr, nz = (int(x) for x in metas[r].tolist())
        ptr = torch.empty(nr + 1, dtype=torch.int64, device=device)
        idx = torch.empty(nz, dtype=torch.int32, device=device)
        vals = torch.empty(nz, dtype=part.values.dtype, device=device)
        dist.recv(ptr, r)
        if nz:
            dist.recv(idx, r)
            dist.recv(vals, r)
        parts.append(DeviceCsr(nr, part.ncols, ptr, idx, vals))
    return concat_row_blocks(parts)


def _bcast_host_list(vals: list[int] | None, n: int, src: int, device) -> list[int]:
    t = torch.zeros(n, dtype=torch.int64, device=device)
    if dist.get_rank() == src:
        t.copy_(torch.as_tensor(vals, dtype=torch.int64))
    dist.broadcast(t, src)
    return [int(x) for x in t.tolist()]


class RowPartition:
    """One rank's share of the row-partitioned multiply (bench.py --gpus N,
    tests/test_distributed_gloo.py).

    B (= the whole operand) is replicated from rank 0; this rank's A and M are
    the row block [cuts[rank], cuts[rank+1]) of their full matrices, taken as
    views with host-known offsets (no host sync per step).  Cuts start
    flop-balanced (``balanced_cuts`` of rank 0's work estimate) and can be
    re-balanced from the per-rank measured cost (``rebalance``)."""

    def __init__(self, b: DeviceCsr, work: np.ndarray | None, device):
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.b = b
        self.device = device
        self.work = work                     # rank 0 only: per-row work estimate
        cuts = balanced_cuts(work, self.world) if self.rank == 0 else None
        self._set_cuts(cuts)
        self.history = []                    # (cuts, per-rank cost) of every rebalance round

    def _set_cuts(self, cuts):
        self.cuts = _bcast_host_list(None if cuts is None else [int(x) for x in cuts], self.world + 1, 0,
                                     self.device)
        self.offsets = cut_offsets(self.b, self.cuts)

    @property
    def lo(self) -> int:
        return self.cuts[self.rank]

    @property
    def hi(self) -> int:
        return self.cuts[self.rank + 1]

    def block(self, m: DeviceCsr | None = None) -> DeviceCsr:
        """This rank's row block of m (default: of B, when A = M = B as in
        cfg2 / cfg5).  m must have B's row pointer for the cached offsets."""
        m = self.b if m is None else m
        r = self.rank
        return row_block(m, self.lo, self.hi, self.offsets[r], self.offsets[r + 1])

    def costs(self, my_cost: float) -> list[float]:
        t = torch.zeros(self.world, dtype=torch.float64, device=self.device)
        t[self.rank] = float(my_cost)
        dist.all_reduce(t)
        return [float(x) for x in t.tolist()]

    def rebalance(self, my_cost: float) -> float:
        """Gather every rank's measured cost of its block, re-cut on rank 0
        (``refine_cuts``), broadcast.  Returns the max/mean imbalance of the
        costs just measured."""
        c = self.costs(my_cost)
        self.history.append((list(self.cuts), c))
        cuts = refine_cuts(self.work, self.cuts, c, self.world) if self.rank == 0 else None
        self._set_cuts(cuts)
        return imbalance(c)

    def use_best(self) -> float:
        """Return to the measured cuts with the smallest maximum cost."""
        if not self.history:
            return 1.0
        cuts, c = min(self.history, key=lambda h: max(h[1]))
        self._set_cuts(cuts if self.rank == 0 else None)
        return imbalance(c)


def replicate_from_host(host: list[torch.Tensor] | None, dev: list[torch.Tensor], src: int = 0):
    """The multi-GPU input path: rank `src` copies its pinned host buffers into
    its device buffers, then every buffer is broadcast to the other ranks
    (NCCL over NVLink on GPUs).  dev: preallocated, same shapes on every rank."""
    if dist.get_rank() == src:
        for h, d in zip(host, dev):
            d.copy_(h, non_blocking=True)
    for d in dev:
        if d.numel():
            dist.broadcast(d, src)
