"""Masked multiply drivers: C = M (.) (A B), plain or complemented — on a B200.

Drop-in mirror of the reference's operator API (pkg/src/maskmul/multiply.py):
``MultiplyPlan`` (:46-81), ``MultiplyStats`` (:84-100), ``PlanError`` (:42),
``masked_multiply_with_stats`` (:349-403), ``masked_multiply`` (:406),
``symbolic_phase`` (:411), ``one_phase_multiply`` / ``two_phase_multiply``
(:422-427), ``inner_product_multiply`` (:430), ``flops_of`` (:111).
Same names, argument meaning and exceptions (PlanError / SparseError /
AssertionError for the reference's internal assertions).

Every multiply runs on the GPU through the C ABI (include/maskmul_b200.h):
host matrices are uploaded (input preparation, like the reference's untimed
_Prepared), the device computes C, and C comes back as a canonical CsrMatrix
with int64 indices.  ``multiply_device`` is the device-resident entry point
(inputs and output stay in HBM).  There is no CPU fallback.

Plan extensions: ``algorithm="auto"`` (per-row push/pull cost model).
``workers`` and ``grain`` are accepted for compatibility and have no effect on
the GPU (the reference guarantees results independent of them).
"""

from __future__ import annotations

import contextlib
import ctypes as C
import math
import threading
import time
from dataclasses import dataclass, field, replace

import numpy as np
import torch

from . import _lib
from .device import DeviceCsr
from .semiring import Semiring, arithmetic_semiring
from .sparse import CscMatrix, CsrMatrix, MaskView, SparseError, to_csr

ALGORITHMS = ("msa", "hash", "mca", "heap", "heapdot", "inner")
# plain masks up to this many entries take the one-call multiply into
# nnz(M)-sized outputs (mm_multiply); larger ones allocate nnz(C) exactly
ONE_CALL_MAX_NNZ = 1 << 22
EXTRA_ALGORITHMS = ("auto",)
PHASES = ("1p", "2p")
_LABELS = {"msa": "MSA", "hash": "Hash", "mca": "MCA", "heap": "Heap",
           "heapdot": "HeapDot", "inner": "Inner", "auto": "Auto"}


class PlanError(ValueError):
    """The requested plan cannot execute this multiply."""


@dataclass(frozen=True)
class MultiplyPlan:
    algorithm: str = "msa"
    phases: str = "1p"
    complemented: bool = False
    semiring: Semiring = field(default_factory=arithmetic_semiring)
    workers: int = 1
    grain: int = 64
    n_inspect: float | None = None

    def __post_init__(self):
        if self.algorithm not in ALGORITHMS + EXTRA_ALGORITHMS:
            raise PlanError(f"unknown algorithm {self.algorithm!r}")
        if self.phases not in PHASES:
            raise PlanError(f"phases must be one of {PHASES}")
        if self.workers < 1:
            raise PlanError("workers must be >= 1")
        if self.grain < 1:
            raise PlanError("grain must be >= 1")
        if self.n_inspect not in (None, 0, 1, math.inf):
            raise PlanError("n_inspect must be 0, 1 or inf")
        if self.algorithm == "mca" and self.complemented:
            raise PlanError("the mask-compressed accumulator does not support complemented masks")
        if self.algorithm == "inner" and self.complemented:
            raise PlanError("the inner-product algorithm does not support complemented masks")

    @property
    def effective_n_inspect(self) -> float:
        if self.n_inspect is not None:
            return self.n_inspect
        return math.inf if self.algorithm == "heapdot" else 1

    def label(self) -> str:
        return f"{_LABELS[self.algorithm]}-{self.phases.upper()}"


@dataclass
class MultiplyStats:
    generated_flops: int = 0
    evaluated_multiplies: int = 0
    symbolic_seconds: float = 0.0
    numeric_seconds: float = 0.0
    assemble_seconds: float = 0.0
    output_nnz: int = 0
    workers: int = 1
    rows_push: int = 0
    rows_pull: int = 0
    rows_empty: int = 0

    @property
    def total_seconds(self) -> float:
        return self.symbolic_seconds + self.numeric_seconds + self.assemble_seconds


# ---------------------------------------------------------------------------
# handles
# ---------------------------------------------------------------------------

_handles: dict[tuple[int, int], int] = {}
_lock = threading.Lock()


def _handle(device_index: int) -> int:
    """One library handle per (device, thread): a handle carries the state
    between mm_multiply_begin and mm_multiply_end, so threads never share one."""
    key = (device_index, threading.get_ident())
    h = _handles.get(key)
    if h is not None:
        return h
    with _lock:
        h = _handles.get(key)
        if h is None:
            lib = _lib.load()
            hp = C.c_void_p()
            rc = lib.mm_create(device_index, C.byref(hp))
            if rc:
                raise RuntimeError(f"mm_create failed: {_lib.last_error()}")
            h = hp.value
            _handles[key] = h
        return h


def _raise(rc: int):
    msg = _lib.last_error()
    if rc == _lib.MM_ERR_PLAN:
        raise PlanError(msg)
    if rc == _lib.MM_ERR_INPUT:
        raise SparseError(msg)
    if rc == _lib.MM_ERR_INTERNAL:
        raise AssertionError(msg)
    raise RuntimeError(f"CUDA error in maskmul: {msg}")


_plan_cache: dict = {}


def _plan_t(plan: MultiplyPlan, comp: bool) -> _lib.PlanT:
    """The C plan struct of (plan, complement flag), built once per distinct plan."""
    key = (plan, comp)
    pt = _plan_cache.get(key)
    if pt is None:
        pt = _plan_cache[key] = _plan_t_build(plan, comp)
    return pt


def _plan_t_build(plan: MultiplyPlan, comp: bool) -> _lib.PlanT:
    ni = plan.effective_n_inspect
    return _lib.PlanT(_lib.MM_ALGO[plan.algorithm], 2 if plan.phases == "2p" else 1, int(comp),
                      int(plan.semiring.kernel_id),
                      _lib.MM_DTYPE_FLOAT64 if np.dtype(plan.semiring.dtype).kind == "f"
                      else _lib.MM_DTYPE_INT64,
                      -1 if ni == math.inf else int(ni))


# ---------------------------------------------------------------------------
# device-resident entry point
# ---------------------------------------------------------------------------

def multiply_device(mask: DeviceCsr, a: DeviceCsr, b: DeviceCsr, plan: MultiplyPlan,
                    complemented: bool | None = None, b_csc: DeviceCsr | None = None,
                    stream: torch.cuda.Stream | None = None):
    """C = M (.) (A B) with every operand and the result in HBM.

    Returns (DeviceCsr C, MultiplyStats).  ``complemented`` defaults to
    ``plan.complemented``.  ``b_csc`` (B stored column-major) is required by
    ``algorithm="inner"`` and enables pull rows under ``"auto"``.
    """
    comp = bool(plan.complemented if complemented is None else (complemented or plan.complemented))
    if comp and plan.algorithm in ("mca", "inner"):
        raise PlanError(f"the {'mask-compressed accumulator' if plan.algorithm == 'mca' else 'inner-product algorithm'}"
                        " does not support complemented masks")
    dev = a.idx.device
    di = dev.index if dev.index is not None else torch.cuda.current_device()
    if stream is None:
        # the current stream's raw handle (torch.cuda.current_stream builds a
        # Python Stream object: several microseconds per multiply)
        raw = torch._C._cuda_getCurrentRawStream(di)
        on_current = True
    else:
        raw = stream.cuda_stream
        on_current = raw == torch._C._cuda_getCurrentRawStream(di)
    lib = _lib.load()
    h = _handle(di)
    pt = _plan_t(plan, comp)
    mm_mask, mm_a, mm_b = mask.mm(), a.mm(), b.mm()
    mm_bt = b_csc.mm() if b_csc is not None else None
    nnz = C.c_int64(0)
    dtype = torch.float64 if pt.dtype == _lib.MM_DTYPE_FLOAT64 else torch.int64
    stats = MultiplyStats()
    st = _lib.StatsT()
    t0 = time.perf_counter()
    # C's arrays come from the caching allocator on the multiply's stream
    ctx = contextlib.nullcontext() if on_current else torch.cuda.stream(stream)
    with ctx:
        if not comp and mask.nnz <= ONE_CALL_MAX_NNZ:
            # plain mask: nnz(C) <= nnz(M) (the one-phase bound, multiply.py:233),
            # so C's arrays are allocated up front and one call does the whole
            # multiply (one host sync, compaction queued right after it)
            cap = mask.nnz
            row_ptr = torch.empty(mask.nrows + 1, dtype=torch.int64, device=dev)
            col_idx = torch.empty(cap, dtype=torch.int32, device=dev)
            values = torch.empty(cap, dtype=dtype, device=dev)
            rc = lib.mm_multiply(h, C.byref(pt), C.byref(mm_mask), C.byref(mm_a), C.byref(mm_b),
                                 C.byref(mm_bt) if mm_bt is not None else None, C.c_void_p(raw),
                                 row_ptr.data_ptr(), col_idx.data_ptr() if cap else None,
                                 values.data_ptr() if cap else None, cap, C.byref(nnz), C.byref(st))
            if rc:
                _raise(rc)
            t1 = time.perf_counter()
            n = int(nnz.value)
            if n < cap:   # shrink in place (the storage stays; no new tensor objects)
                col_idx.resize_(n)
                values.resize_(n)
        else:
            rc = lib.mm_multiply_begin(h, C.byref(pt), C.byref(mm_mask), C.byref(mm_a), C.byref(mm_b),
                                       C.byref(mm_bt) if mm_bt is not None else None,
                                       C.c_void_p(raw), C.byref(nnz))
            if rc:
                _raise(rc)
            t1 = time.perf_counter()
            n = int(nnz.value)
            row_ptr = torch.empty(mask.nrows + 1, dtype=torch.int64, device=dev)
            col_idx = torch.empty(n, dtype=torch.int32, device=dev)
            values = torch.empty(n, dtype=dtype, device=dev)
            rc = lib.mm_multiply_end(h, row_ptr.data_ptr(), col_idx.data_ptr() if n else None,
                                     values.data_ptr() if n else None, C.byref(st))
            if rc:
                _raise(rc)
    t2 = time.perf_counter()
    if plan.phases == "2p":
        stats.symbolic_seconds, stats.numeric_seconds = t1 - t0, t2 - t1
    else:
        stats.numeric_seconds, stats.assemble_seconds = t1 - t0, t2 - t1
    stats.generated_flops = int(st.generated_flops)
    stats.evaluated_multiplies = int(st.evaluated_multiplies)
    stats.output_nnz = int(st.output_nnz)
    stats.rows_push, stats.rows_pull, stats.rows_empty = (int(st.rows_push), int(st.rows_pull),
                                                         int(st.rows_empty))
    stats.workers = plan.workers
    return DeviceCsr(mask.nrows, mask.ncols, row_ptr, col_idx, values), stats


# ---------------------------------------------------------------------------
# host-facing drop-in API
# ---------------------------------------------------------------------------

def _check_a(a):
    if not (hasattr(a, "row_ptr") and hasattr(a, "col_idx") and hasattr(a, "values")):
        raise SparseError("A must be a CsrMatrix")


def _prepare(mask, a, b, plan: MultiplyPlan, device=None):
    """_Prepared (multiply.py:175-233): validation, dtype casts, uploads."""
    _check_a(a)
    comp = bool(plan.complemented or getattr(mask, "complemented", False))
    if plan.algorithm == "mca" and comp:
        raise PlanError("the mask-compressed accumulator does not support complemented masks")
    if plan.algorithm == "inner" and comp:
        raise PlanError("the inner-product algorithm does not support complemented masks")
    b_nrows, b_ncols = b.shape
    if mask.nrows != a.nrows or mask.ncols != b_ncols or a.ncols != b_nrows:
        raise SparseError(f"dimension mismatch: mask {mask.shape}, A {a.shape}, B {b.shape}")
    dt = np.dtype(plan.semiring.dtype)
    need_vals = plan.semiring.kernel_id == 0
    dm = DeviceCsr.from_host(mask, device=device, with_values=False)
    da = DeviceCsr.from_host(a, dtype=dt, device=device, with_values=need_vals)
    is_csc = hasattr(b, "col_ptr")
    b_csr = to_csr(b) if is_csc else b
    db = DeviceCsr.from_host(b_csr, dtype=dt, device=device, with_values=need_vals)
    dbt = None
    ordered = plan.semiring.kernel_id == 0 and dt.kind == "f"
    if plan.algorithm == "inner" or (plan.algorithm == "auto" and (is_csc or (not comp and _pull_pays(mask, a, b_csr, ordered)))):
        dbt = (DeviceCsr.from_host(b, dtype=dt, device=device, with_values=need_vals)
               if is_csc else db.transpose_storage())
    return dm, da, db, dbt, comp


def _pull_pays(mask, a, b, ordered: bool = False) -> bool:
    """auto: build B^T in the (untimed) preparation when the byte model of
    SURVEY §8(d) makes pull clearly cheaper in aggregate — the mask is much
    sparser than the product space (cfg3 d1 / d4).  The per-row choice is
    still made on the device by the analysis kernel."""
    nnz_a = int(a.row_ptr[-1])
    nnz_m = int(mask.row_ptr[-1])
    if nnz_a == 0 or nnz_m == 0:
        return False
    blen = np.diff(np.asarray(b.row_ptr, dtype=np.int64))
    flops = int(blen[np.asarray(a.col_idx[:nnz_a], dtype=np.int64)].sum())
    # pull reads (nnz(A_i) + nnz(B_*j)) per mask entry (i, j)
    na = np.diff(np.asarray(a.row_ptr, dtype=np.int64))
    nm = np.diff(np.asarray(mask.row_ptr, dtype=np.int64))
    nnz_b = int(b.row_ptr[-1])
    col_len = np.bincount(np.asarray(b.col_idx[:nnz_b], dtype=np.int64), minlength=b.shape[1])
    pull = int((na * nm).sum()) + int(col_len[np.asarray(mask.col_idx[:nnz_m], dtype=np.int64)].sum())
    # float64 plus-times rows push through the deferred-hit kernel at a third
    # of the pull path's cost per probe (the device's per-row model weighs the
    # same way, analyze.cuh classify_row)
    return (3 if ordered else 1.5) * pull < flops


def masked_multiply_with_stats(mask, a, b, plan: MultiplyPlan, device=None):
    dm, da, db, dbt, comp = _prepare(mask, a, b, plan, device)
    c, stats = multiply_device(dm, da, db, plan, complemented=comp, b_csc=dbt)
    host = c.to_host()
    host.values = host.values.astype(np.dtype(plan.semiring.dtype), copy=False)
    return host, stats


def masked_multiply(mask, a, b, plan: MultiplyPlan, device=None) -> CsrMatrix:
    c, _ = masked_multiply_with_stats(mask, a, b, plan, device)
    return c


def symbolic_phase(mask, a, b, plan: MultiplyPlan, device=None) -> np.ndarray:
    """Exact per-row output nnz (multiply.py:411-419), computed on the GPU."""
    dm, da, db, dbt, comp = _prepare(mask, a, b, plan, device)
    dev = da.idx.device
    stream = torch.cuda.current_stream(dev)
    counts = torch.zeros(max(mask.nrows, 1), dtype=torch.int64, device=dev)
    lib = _lib.load()
    h = _handle(dev.index)
    pt = _plan_t(plan, comp)
    mm_bt = dbt.mm() if dbt is not None else None
    rc = lib.mm_symbolic(h, C.byref(pt), C.byref(dm.mm()), C.byref(da.mm()), C.byref(db.mm()),
                         C.byref(mm_bt) if mm_bt is not None else None,
                         C.c_void_p(stream.cuda_stream), counts.data_ptr())
    if rc:
        _raise(rc)
    return counts[: mask.nrows].cpu().numpy()


def one_phase_multiply(mask, a, b, plan: MultiplyPlan) -> CsrMatrix:
    return masked_multiply(mask, a, b, replace(plan, phases="1p"))


def two_phase_multiply(mask, a, b, plan: MultiplyPlan) -> CsrMatrix:
    return masked_multiply(mask, a, b, replace(plan, phases="2p"))


def inner_product_multiply(mask, a, b, semiring: Semiring, workers: int = 1) -> CsrMatrix:
    return masked_multiply(mask, a, b, MultiplyPlan(algorithm="inner", semiring=semiring,
                                                    workers=workers))


def flops_of(a, b, device=None) -> int:
    """Classical flops(A B) (multiply.py:111-112), counted on the GPU."""
    _check_a(a)
    b_csr = to_csr(b) if hasattr(b, "col_ptr") else b
    da = DeviceCsr.from_host(a, device=device, with_values=False)
    db = DeviceCsr.from_host(b_csr, device=device, with_values=False)
    dev = da.idx.device
    out = torch.zeros(max(a.nrows, 1), dtype=torch.int64, device=dev)
    tot = torch.zeros(1, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)
    rc = _lib.load().mm_row_flops(C.byref(da.mm()), C.byref(db.mm()), out.data_ptr(),
                                  tot.data_ptr(), C.c_void_p(stream.cuda_stream))
    if rc:
        _raise(rc)
    return int(tot.item())


def last_kernel_rows(device=None) -> dict:
    """Rows per kernel bin of this thread's last multiply on `device` (bin
    names as in DESIGN.md §4: which accumulator computed how many rows)."""
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    nb = 64
    rows = (C.c_int64 * nb)()
    n = _lib.load().mm_profile_bins(_handle(dev.index), rows, None, nb)
    return {BIN_NAMES[b]: int(rows[b]) for b in range(min(n, len(BIN_NAMES))) if rows[b]}


# kernel bins (csrc/analyze.cuh enum Bin), named for last_kernel_rows / bench.py
BIN_NAMES = (["empty"] + [f"hash_{m}_t{t}{c}" for m in ("plain", "ctab", "csrch")
                          for t, c in ((0, "s"), (0, "l"), (1, "s"), (1, "l"), (2, "s"), (2, "l"), (3, "g"))]
             + ["pull"] + [f"{f}_t{t}" for f in ("msa", "mca", "heap") for t in range(4)] + ["single"]
             + [f"msa_sparse_t{t}" for t in range(3)] + [f"msa_dense_t{t}" for t in range(3)]
             + [f"msa_dense_comp_t{t}" for t in range(3)] + ["pull_lane", "f64_defer", "msa_window"])


def reduce_sum(values: torch.Tensor) -> torch.Tensor:
    """Deterministic device sum (the triangle-count reduction, graphs.py:96)."""
    dev = values.device
    out = torch.zeros(1, dtype=values.dtype, device=dev)
    dt = _lib.MM_DTYPE_FLOAT64 if values.dtype == torch.float64 else _lib.MM_DTYPE_INT64
    rc = _lib.load().mm_reduce_sum(values.data_ptr() if values.numel() else None, values.numel(),
                                   dt, out.data_ptr(),
                                   C.c_void_p(torch._C._cuda_getCurrentRawStream(dev.index)))
    if rc:
        _raise(rc)
    return out
