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
