"""Robustness of the C ABI on the GPU: input limits, device selection.

* nnz(A), nnz(B), nnz(M) >= 2^31 are rejected with MM_ERR_INPUT (SparseError)
  before any device work: the product loops count one batch's products in
  32-bit ints, which nnz(B) < 2^31 bounds (product_loop.cuh).
* Every extern "C" entry runs on its handle's / stream's / operands' device
  and restores the caller's current device.
"""

import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from paper_2111_09947_b200 import (MultiplyPlan, SparseError, arithmetic_semiring,  # noqa: E402
                                   masked_multiply, plus_pair_semiring, _lib)
from paper_2111_09947_b200.device import DeviceCsr  # noqa: E402
from paper_2111_09947_b200.multiply import _handle, _plan_t, multiply_device, reduce_sum  # noqa: E402
from paper_2111_09947_b200.workloads import GeneratorSpec, generate  # noqa: E402


@pytest.fixture(autouse=True, scope="module")
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def test_nnz_limit_rejected_before_device_work():
    lib = _lib.load()
    h = _handle(0)
    pt = _plan_t(MultiplyPlan(semiring=plus_pair_semiring(np.int64)), False)
    fake = C.c_void_p(0x1000)     # never dereferenced: validation fails first
    small = _lib.MatrixT(4, 4, 4, fake, fake, None)
    big = _lib.MatrixT(4, 4, 1 << 31, fake, fake, None)
    nnz = C.c_int64(0)
    stream = C.c_void_p(torch.cuda.current_stream(0).cuda_stream)
    for a, b, m in ((small, big, small), (big, small, small), (small, small, big)):
        rc = lib.mm_multiply_begin(h, C.byref(pt), C.byref(m), C.byref(a), C.byref(b), None, stream,
                                   C.byref(nnz))
        assert rc == _lib.MM_ERR_INPUT
        assert "2^31" in _lib.last_error()
    # the handle is still usable afterwards
    g = generate(GeneratorSpec("erdos-renyi", 8, 4, seed=1))
    d = DeviceCsr.from_host(g, device=torch.device("cuda", 0), with_values=False)
    c, _ = multiply_device(d, d, d, MultiplyPlan(semiring=plus_pair_semiring(np.int64)))
    assert c.nnz > 0


def test_current_device_preserved():
    torch.cuda.set_device(0)
    g = generate(GeneratorSpec("erdos-renyi", 8, 4, seed=2)).astype(np.float64)
    masked_multiply(g.pattern(), g, g, MultiplyPlan(semiring=arithmetic_semiring(np.float64)))
    assert torch.cuda.current_device() == 0


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs two GPUs")
def test_operands_on_second_device_while_first_is_current():
    """a multiply (and the free-standing calls: reduce, CSC
    transpose via prep kernels, inner) on cuda:1 while cuda:0 is current,
    then the same thread on cuda:0 again (per-device occupancy caches)."""
    torch.cuda.set_device(0)
    g = generate(GeneratorSpec("erdos-renyi", 10, 8, seed=3)).astype(np.float64)
    g.values[:] = np.random.default_rng(0).random(g.nnz)
    want = None
    for dev in (1, 0, 1):
        d = torch.device("cuda", dev)
        dg = DeviceCsr.from_host(g, dtype=np.float64, device=d)
        dm = DeviceCsr.from_host(g.pattern(), device=d, with_values=False)
        for algo in ("auto", "hash", "inner"):
            c, _ = multiply_device(dm, dg, dg, MultiplyPlan(algorithm=algo, semiring=arithmetic_semiring(np.float64)),
                                   b_csc=dg.transpose_storage() if algo == "inner" else None,
                                   stream=torch.cuda.current_stream(d))
            s = float(reduce_sum(c.values).cpu())
            want = s if want is None else want
            assert s == want
            assert torch.cuda.current_device() == 0


def _rand_rows(rng, rows, cols, lens, dtype):
    import numpy as np
    from paper_2111_09947_b200 import from_arrays
    lens = np.minimum(np.asarray(lens), cols)
    r = np.repeat(np.arange(rows), lens)
    c = np.concatenate([rng.choice(cols, ln, replace=False) for ln in lens]) if lens.sum() else np.empty(0, np.int64)
    v = rng.standard_normal(r.size) if dtype == np.float64 else rng.integers(1, 5, r.size)
    return from_arrays(rows, cols, r, c, v)


def _global_tier_problem():
    rng = np.random.default_rng(5)
    m, k, n = 1000, 50, 300000
    a = _rand_rows(rng, m, k, rng.integers(0, 4, m), np.float64)
    b = _rand_rows(rng, k, n, rng.integers(10, 50, k), np.float64)
    mlen = rng.integers(0, 40, m)
    mlen[[3, 500]] = [29654, 12000]
    mask = _rand_rows(rng, m, n, mlen, np.int64).pattern()
    return mask, a, b


def test_symbolic_pass_of_float64_multiply_with_global_tier_rows():
    """Found by tools/fuzz_gpu.py: a float64 plain multiply whose mask rows need the
    global hash tier (29,654 entries) ran its two-phase symbolic pass (kind 0) as
    sliced rows over tables sized for the global tier and failed; the tier is
    decided by the multiply's kind.  Reference: two-phase driver, multiply.py:358-380."""
    import oracle
    from paper_2111_09947_b200 import masked_multiply_with_stats
    mask, a, b = _global_tier_problem()
    ref = oracle.masked_multiply(mask, a, b, algorithm="msa", dtype=np.float64)
    for algo in ("auto", "hash", "msa"):
        for phases in ("1p", "2p"):
            c, st = masked_multiply_with_stats(mask, a, b, MultiplyPlan(algorithm=algo, phases=phases,
                                                                      semiring=arithmetic_semiring(np.float64)))
            assert np.array_equal(c.row_ptr, ref.row_ptr), (algo, phases)
            assert np.array_equal(c.col_idx[: c.nnz], ref.col_idx), (algo, phases)
            assert np.array_equal(c.values[: c.nnz], ref.values), (algo, phases)
            assert st.evaluated_multiplies == ref.evaluated_multiplies


def test_direct_pass_leaves_leading_rows_to_the_binned_pass():
    """Found by tools/fuzz_gpu.py: the direct float64 pass marks rows it cannot take
    with a count of -1; the scan queued behind it summed those, so the first rows'
    offsets went negative and the early compaction wrote before C.  Counts below
    zero scan as zero (scan_compact.cuh).  The leading rows here all have masks over
    the direct kernel's 128 entries."""
    import numpy as np
    import oracle
    from paper_2111_09947_b200 import MultiplyPlan, arithmetic_semiring, masked_multiply_with_stats
    rng = np.random.default_rng(6)
    m, k, n = 20000, 1, 40000
    a = _rand_rows(rng, m, k, (rng.random(m) < 0.9).astype(np.int64), np.float64)
    b = _rand_rows(rng, k, n, [9], np.float64)
    mlen = rng.integers(20, 80, m)
    mlen[:300] = rng.integers(150, 300, 300)
    mask = _rand_rows(rng, m, n, mlen, np.int64).pattern()
    ref = oracle.masked_multiply(mask, a, b, algorithm="msa", dtype=np.float64)
    for rep in range(3):
        c, st = masked_multiply_with_stats(mask, a, b, MultiplyPlan(algorithm="auto",
                                                                  semiring=arithmetic_semiring(np.float64)))
        assert np.array_equal(c.row_ptr, ref.row_ptr)
        assert np.array_equal(c.col_idx[: c.nnz], ref.col_idx)
        assert np.array_equal(c.values[: c.nnz], ref.values)
        assert (st.generated_flops, st.evaluated_multiplies) == (ref.generated_flops, ref.evaluated_multiplies)


def test_second_thread_does_not_lower_a_kernels_shared_memory_limit():
    """The dynamic shared-memory limit of a kernel belongs to the CUDA context.  The
    library kept its record of it per thread: a second thread running the same
    kernel at a smaller size set the limit down, and the first thread's next launch
    at its own (recorded) size was refused with "invalid argument" (seen in the full
    GPU suite, after the threaded parity test).  The record is process-wide now."""
    import threading
    import oracle
    from paper_2111_09947_b200 import masked_multiply_with_stats
    sem = arithmetic_semiring(np.float64)
    mask, a, b = _global_tier_problem()
    ref = oracle.masked_multiply(mask, a, b, algorithm="msa", dtype=np.float64)
    plans = [MultiplyPlan(algorithm=al, phases=ph, semiring=sem) for al in ("msa", "hash", "mca") for ph in ("1p", "2p")]

    def big():
        for plan in plans:
            c, _ = masked_multiply_with_stats(mask, a, b, plan)
            assert np.array_equal(c.row_ptr, ref.row_ptr), plan.label()
            assert np.array_equal(c.col_idx[: c.nnz], ref.col_idx), plan.label()
            assert np.array_equal(c.values[: c.nnz], ref.values), plan.label()

    errors = []

    def small():
        try:
            rng = np.random.default_rng(7)
            for n in (300, 2000, 20000, 300000):
                sa = _rand_rows(rng, 600, 40, rng.integers(0, 4, 600), np.float64)
                sb = _rand_rows(rng, 40, n, rng.integers(5, 30, 40), np.float64)
                sm = _rand_rows(rng, 600, n, rng.integers(0, 6, 600), np.int64).pattern()
                want = oracle.masked_multiply(sm, sa, sb, algorithm="msa", dtype=np.float64)
                for plan in plans:
                    c, _ = masked_multiply_with_stats(sm, sa, sb, plan)
                    assert np.array_equal(c.row_ptr, want.row_ptr), (n, plan.label())
                    assert np.array_equal(c.values[: c.nnz], want.values), (n, plan.label())
        except BaseException as e:   # noqa: BLE001
            errors.append(e)

    big()
    t = threading.Thread(target=small)
    t.start()
    t.join()
    assert not errors, errors
    big()
