"""Hypothesis properties of the reference re-pointed at the GPU path
(reference tests/test_multiply.py:334-364, pattern containment): for random
small operands (duplicates, empty rows, 1 x 1 shapes) and every plan, C's
pattern lies inside the mask (plain) or outside it (complement) and inside the
generated pattern, and C equals the C oracle bit for bit."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
hypothesis = pytest.importorskip("hypothesis")

from hypothesis import given, settings, strategies as st  # noqa: E402

pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from paper_2111_09947_b200 import (MultiplyPlan, arithmetic_semiring, from_arrays,  # noqa: E402
                                   masked_multiply, plus_pair_semiring)

ALGORITHMS = ("msa", "hash", "mca", "heap", "heapdot", "inner", "auto")


@pytest.fixture(autouse=True, scope="module")
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


@st.composite
def small_multiply(draw):
    m = draw(st.integers(1, 10))
    k = draw(st.integers(1, 10))
    n = draw(st.integers(1, 10))

    def entries(rows, cols):
        return st.lists(st.tuples(st.integers(0, rows - 1), st.integers(0, cols - 1),
                                  st.integers(-4, 4).filter(lambda v: v != 0)), max_size=25)

    return (m, k, n, draw(entries(m, k)), draw(entries(k, n)), draw(entries(m, n)), draw(st.booleans()),
            draw(st.sampled_from(("i64", "f64", "pair"))))


def _from_triples(rows, cols, triples, dtype):
    r = np.array([t[0] for t in triples], dtype=np.int64)
    c = np.array([t[1] for t in triples], dtype=np.int64)
    v = np.array([t[2] for t in triples], dtype=dtype)
    return from_arrays(rows, cols, r, c, v)


def _pattern(c):
    rows = np.repeat(np.arange(c.nrows), np.diff(c.row_ptr))
    return set(zip(rows.tolist(), np.asarray(c.col_idx[: c.nnz]).tolist()))


@given(small_multiply())
@settings(max_examples=60, deadline=None)
def test_pattern_containment_and_oracle(inst):
    m, k, n, ae, be, me, comp, kind = inst
    dt = np.float64 if kind == "f64" else np.int64
    sem = plus_pair_semiring(np.int64) if kind == "pair" else arithmetic_semiring(dt)
    a = _from_triples(m, k, ae, dt)
    b = _from_triples(k, n, be, dt)
    mask = _from_triples(m, n, me, np.int64).pattern()
    mask_set = _pattern(mask)
    generated = _pattern(masked_multiply(from_arrays(m, n, np.repeat(np.arange(m), n), np.tile(np.arange(n), m),
                                                     np.ones(m * n, dtype=np.int64)).pattern(), a, b,
                                         MultiplyPlan(algorithm="msa", semiring=sem)))
    ref = oracle.masked_multiply(mask, a, b, algorithm="msa", complemented=comp, dtype=dt,
                                 semiring_id=sem.kernel_id)
    for algo in ALGORITHMS:
        if comp and algo in ("mca", "inner"):
            continue
        for phases in ("1p", "2p"):
            plan = MultiplyPlan(algorithm=algo, phases=phases, complemented=comp, semiring=sem)
            c = masked_multiply(mask, a, b, plan)
            got = _pattern(c)
            assert got.isdisjoint(mask_set) if comp else got <= mask_set, (algo, phases)
            assert got <= generated, (algo, phases)
            assert np.array_equal(c.row_ptr, ref.row_ptr), (algo, phases)
            assert np.array_equal(c.col_idx[: c.nnz], ref.col_idx), (algo, phases)
            if kind == "f64" and algo in ("heap", "heapdot"):
                np.testing.assert_allclose(c.values[: c.nnz], ref.values, rtol=1e-12, atol=0)
            else:
                assert np.array_equal(c.values[: c.nnz], ref.values), (algo, phases)
