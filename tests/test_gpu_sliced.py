"""Sliced hub rows (plain masks wider than the largest shared hash table):
one-phase rows run as (row, slice) work items on any SM
(csrc/push_hash_items.cuh), two-phase rows slice after slice in one group
(push_hash.cuh hash_row).  Both must equal the C oracle bit for bit — result,
evaluated and generated counters — and each other.  Reference semantics:
hash_numeric (_kernels.py:130-218), output in mask order (:208-216)."""

import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from golden_util import digest_csr  # noqa: E402
from paper_2111_09947_b200 import (MultiplyPlan, _lib, arithmetic_semiring, from_arrays,  # noqa: E402
                                   masked_multiply_with_stats, plus_pair_semiring)
from paper_2111_09947_b200.multiply import _handle, last_kernel_rows  # noqa: E402

N_TUNE = 17


@pytest.fixture(autouse=True, scope="module")
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def _split(on: bool):
    prm = [-1] * N_TUNE
    prm[16] = int(on)
    assert _lib.load().mm_set_tuning(_handle(torch.cuda.current_device()), (C.c_int64 * N_TUNE)(*prm), N_TUNE) == 0


def _hub_problem(seed, rows, n, nm_lo, nm_hi, na, empty_rows=()):
    """Rows with masks of nm_lo..nm_hi columns (several 6144-entry slices),
    A rows of ~na entries over B rows of 1..4000 entries (some hubs), so every
    slice meets a different part of each B row; a few rows without A entries
    or with a mask whose length is an exact multiple of the slice."""
    rng = np.random.default_rng(seed)
    nb = 3000
    lens = np.where(rng.random(nb) < 0.03, rng.integers(2000, 4000, nb), rng.integers(1, 60, nb))
    b_r = np.repeat(np.arange(nb), lens)
    b_c = np.concatenate([rng.choice(n, ln, replace=False) for ln in lens])
    b = from_arrays(nb, n, b_r, b_c, rng.integers(-4, 5, b_c.size))
    a_r, a_c, m_r, m_c = [], [], [], []
    for i in range(rows):
        if i not in empty_rows:
            ks = np.unique(rng.integers(0, nb, na))
            a_r.append(np.full(ks.size, i))
            a_c.append(ks)
        nm = 2 * 6144 if i == 1 else int(rng.integers(nm_lo, nm_hi))
        cols = np.sort(rng.choice(n, nm, replace=False))
        m_r.append(np.full(cols.size, i))
        m_c.append(cols)
    a_r, a_c = np.concatenate(a_r), np.concatenate(a_c)
    a = from_arrays(rows, nb, a_r, a_c, rng.integers(-3, 4, a_c.size))
    m_c = np.concatenate(m_c)
    m = from_arrays(rows, n, np.concatenate(m_r), m_c, np.ones(m_c.size, np.int64))
    return a, b, m


@pytest.mark.parametrize("spec", [(7, 40, 300_000, 6200, 60_000, 400, (3,)),
                                  (8, 300, 120_000, 6145, 20_000, 150, (0, 17))])
def test_sliced_items_match_oracle_and_sequential_slices(spec):
    seed, rows, n, lo, hi, na, empty = spec
    a, b, m = _hub_problem(seed, rows, n, lo, hi, na, empty)
    try:
        for sem in (plus_pair_semiring(np.int64), arithmetic_semiring(np.int64)):
            r = oracle.masked_multiply(m.pattern(), a, b, semiring_id=sem.kernel_id, dtype=sem.dtype)
            want = digest_csr(r.row_ptr, r.col_idx, r.values)
            for algo in ("hash", "auto"):
                for ph in ("1p", "2p"):
                    for split in (True, False):
                        _split(split)
                        plan = MultiplyPlan(algorithm=algo, phases=ph, semiring=sem)
                        c, st = masked_multiply_with_stats(m.pattern(), a, b, plan)
                        got = digest_csr(c.row_ptr, c.col_idx, c.values)
                        assert got == want, (spec, sem.name, algo, ph, split)
                        assert st.evaluated_multiplies == r.evaluated_multiplies
                        assert st.generated_flops == r.generated_flops
                        if algo == "hash":
                            assert last_kernel_rows().get("hash_plain_t3g", 0) > 0
    finally:
        _split(True)
