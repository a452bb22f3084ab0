"""One-launch path for the smallest plain one-phase multiplies
(csrc/fused_tail.cuh): the row kernel's last block scans the row counts,
compacts C and writes the counters into mapped host memory.  It must equal the
separate-kernel path and the C oracle bit for bit (C, generated / evaluated
counters, empty rows), fall back to the binned path when a mask row does not
fit the fixed table, and survive a change of stream between multiplies.
Reference semantics: the 1P assembly, multiply.py:381-399."""

import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from golden_util import digest_csr  # noqa: E402
from paper_2111_09947_b200 import (MultiplyPlan, _lib, arithmetic_semiring, from_arrays,  # noqa: E402
                                   masked_multiply_with_stats, plus_pair_semiring)
from paper_2111_09947_b200.device import DeviceCsr  # noqa: E402
from paper_2111_09947_b200.multiply import _handle, multiply_device  # noqa: E402

N_TUNE = 19


@pytest.fixture(autouse=True, scope="module")
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield
    _fused(True)


def _fused(on: bool):
    prm = [-1] * N_TUNE
    prm[17] = (1 << 13) if on else 0
    assert _lib.load().mm_set_tuning(_handle(torch.cuda.current_device()), (C.c_int64 * N_TUNE)(*prm), N_TUNE) == 0


def _problem(seed, m, n, da, dm, dtype, wide_row=None):
    rng = np.random.default_rng(seed)

    def rand(rows, cols, deg, vals=True):
        r = np.repeat(np.arange(rows), rng.integers(0, 2 * deg + 1, rows))
        c = rng.integers(0, cols, r.size)
        v = rng.integers(-4, 5, r.size).astype(dtype) if dtype == np.int64 else rng.standard_normal(r.size)
        return from_arrays(rows, cols, r, c, v)

    a = rand(m, n, da)
    b = rand(n, n, da)
    mr = np.repeat(np.arange(m), rng.integers(0, 2 * dm + 1, m))
    mc = rng.integers(0, n, mr.size)
    if wide_row is not None:   # one mask row over half the fixed table (512 / 256 entries)
        mr = np.concatenate([mr, np.full(700, wide_row)])
        mc = np.concatenate([mc, rng.choice(n, 700, replace=False)])
    mask = from_arrays(m, n, mr, mc, np.ones(mr.size, dtype=np.int64)).pattern()
    return mask, a, b


CASES = [
    # (seed, rows, cols, deg A/B, deg M, semiring, algorithm)
    (1, 4096, 4096, 8, 8, "f64", "auto"),     # direct float64 kernel + tail (cfg1's shape)
    (2, 4096, 4096, 8, 8, "f64", "hash"),     # k_tiny_hash<2> + tail
    (3, 3000, 5000, 6, 12, "i64", "auto"),    # k_tiny_hash<1>
    (4, 3000, 5000, 6, 12, "pair", "hash"),   # k_tiny_hash<0>
    (5, 1, 64, 4, 4, "i64", "auto"),          # one row
    (6, 257, 300, 3, 2, "pair", "auto"),      # rows not a multiple of the tail's 256 threads
    (7, 8192, 2000, 2, 1, "f64", "auto"),     # the row limit, mostly empty output
]


def _dig(c):
    return digest_csr(c.row_ptr, c.col_idx, c.values)


def _sem(kind):
    if kind == "f64":
        return arithmetic_semiring(np.float64), np.float64
    if kind == "i64":
        return arithmetic_semiring(np.int64), np.int64
    return plus_pair_semiring(np.int64), np.int64


@pytest.mark.parametrize("seed,m,n,da,dm,kind,algo", CASES)
def test_fused_equals_separate_and_oracle(seed, m, n, da, dm, kind, algo):
    sem, dt = _sem(kind)
    mask, a, b = _problem(seed, m, n, da, dm, dt)
    plan = MultiplyPlan(algorithm=algo, semiring=sem)
    _fused(True)
    c1, s1 = masked_multiply_with_stats(mask, a, b, plan)
    _fused(False)
    c0, s0 = masked_multiply_with_stats(mask, a, b, plan)
    _fused(True)
    assert _dig(c1) == _dig(c0)
    assert (s1.generated_flops, s1.evaluated_multiplies, s1.output_nnz, s1.rows_empty) == \
           (s0.generated_flops, s0.evaluated_multiplies, s0.output_nnz, s0.rows_empty)
    r = oracle.masked_multiply(mask, a, b, algorithm="msa", dtype=dt,
                               semiring_id=1 if kind == "pair" else 0)
    assert np.array_equal(c1.row_ptr, r.row_ptr)
    assert np.array_equal(c1.col_idx, r.col_idx)
    assert np.array_equal(c1.values, r.values)     # bitwise, float64 included (ascending-k order)
    assert s1.generated_flops == r.generated_flops
    assert s1.evaluated_multiplies == r.evaluated_multiplies


@pytest.mark.parametrize("kind,algo", [("f64", "auto"), ("i64", "hash"), ("pair", "auto")])
def test_fused_overflow_falls_back(kind, algo):
    """A 700-entry mask row does not fit the single-pass tables: the one-launch
    kernel raises overflow and the binned path computes the whole multiply."""
    sem, dt = _sem(kind)
    mask, a, b = _problem(11, 2000, 3000, 8, 6, dt, wide_row=777)
    plan = MultiplyPlan(algorithm=algo, semiring=sem)
    _fused(True)
    c1, s1 = masked_multiply_with_stats(mask, a, b, plan)
    r = oracle.masked_multiply(mask, a, b, algorithm="msa", dtype=dt,
                               semiring_id=1 if kind == "pair" else 0)
    assert np.array_equal(c1.row_ptr, r.row_ptr)
    assert np.array_equal(c1.col_idx, r.col_idx)
    assert np.array_equal(c1.values, r.values)
    assert s1.generated_flops == r.generated_flops
    assert s1.evaluated_multiplies == r.evaluated_multiplies
    # and the next multiply on the same handle takes the one-launch path again
    mask2, a2, b2 = _problem(12, 1000, 1000, 5, 5, dt)
    c2, _ = masked_multiply_with_stats(mask2, a2, b2, plan)
    r2 = oracle.masked_multiply(mask2, a2, b2, algorithm="msa", dtype=dt,
                                semiring_id=1 if kind == "pair" else 0)
    assert np.array_equal(c2.col_idx, r2.col_idx) and np.array_equal(c2.values, r2.values)


def test_fused_repeated_and_across_streams():
    """The host returns on the mapped sequence word, before the kernel retires:
    back-to-back multiplies on one stream, then on other streams, stay exact."""
    sem, dt = _sem("f64")
    mask, a, b = _problem(21, 4096, 4096, 8, 8, dt)
    dev = torch.device("cuda", torch.cuda.current_device())
    dm = DeviceCsr.from_host(mask, device=dev, with_values=False)
    da = DeviceCsr.from_host(a, dtype=dt, device=dev)
    db = DeviceCsr.from_host(b, dtype=dt, device=dev)
    _fused(True)
    ref = None
    streams = [None, torch.cuda.Stream(dev), None, torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
    torch.cuda.synchronize()
    for rep in range(40):
        for algo in ("auto", "hash"):
            plan = MultiplyPlan(algorithm=algo, semiring=sem)
            st = streams[rep % len(streams)]
            if st is not None:
                st.wait_stream(torch.cuda.current_stream(dev))
            c, _ = multiply_device(dm, da, db, plan, stream=st)
            if st is not None:
                torch.cuda.current_stream(dev).wait_stream(st)
            d = _dig(c.to_host())
            if ref is None:
                ref = d
            assert d == ref, (rep, algo)


def test_fused_begin_end_mode():
    """mm_multiply_begin / mm_multiply_end (complement-sized capacity unknown to
    the caller): the tail scans, mm_multiply_end compacts."""
    from paper_2111_09947_b200 import multiply as mul
    sem, dt = _sem("i64")
    mask, a, b = _problem(31, 2048, 2048, 6, 6, dt)
    plan = MultiplyPlan(algorithm="hash", semiring=sem)
    old = mul.ONE_CALL_MAX_NNZ
    try:
        mul.ONE_CALL_MAX_NNZ = -1   # force begin / end
        _fused(True)
        c1, s1 = masked_multiply_with_stats(mask, a, b, plan)
    finally:
        mul.ONE_CALL_MAX_NNZ = old
    r = oracle.masked_multiply(mask, a, b, algorithm="msa", dtype=dt)
    assert np.array_equal(c1.row_ptr, r.row_ptr)
    assert np.array_equal(c1.col_idx, r.col_idx)
    assert np.array_equal(c1.values, r.values)
    assert s1.evaluated_multiplies == r.evaluated_multiplies
