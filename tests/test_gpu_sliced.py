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


def _tune(**kw):
    """mm_set_tuning by parameter index (-1 = keep)."""
    n = 21
    prm = [-1] * n
    for k, v in kw.items():
        prm[int(k[1:])] = int(v)
    assert _lib.load().mm_set_tuning(_handle(torch.cuda.current_device()), (C.c_int64 * n)(*prm), n) == 0


def _launches_of(fn):
    lib = _lib.load()
    h = _handle(torch.cuda.current_device())
    lib.mm_profile_enable(h, 1)
    try:
        out = fn()
        ms = (C.c_float * 6)()
        n = C.c_int64(0)
        lib.mm_profile_read(h, ms, 6, C.byref(n))
    finally:
        lib.mm_profile_enable(h, 0)
    return out, int(n.value)


def test_kblocked_passes_match_oracle():
    """k-blocked passes of the 16-warp plain hash bins (push_hash.cuh, launch_bins_on):
    when B's index array is larger than the block size, the bin's launch is repeated
    over blocks of B's rows and the partial counts wait in the row's mask-shaped
    output slots.  One-phase plus-pair results (int64 and float64 outputs) must equal
    the C oracle bit for bit at every block size, rows without A entries in some blocks
    and rows cut into slices included; the plans the blocking does not apply to
    (two-phase, plus-times) are unchanged.  Reference semantics: hash_numeric
    (_kernels.py:130-218)."""
    a, b, m = _hub_problem(21, 120, 60_000, 300, 9000, 500, empty_rows=(5,))
    # half of the rows meet only the first third of B's rows: no A entry in the later blocks
    rows_of = np.repeat(np.arange(a.nrows), np.diff(a.row_ptr))
    keep = ~((rows_of % 2 == 1) & (a.col_idx >= 1000))
    a = from_arrays(a.nrows, a.ncols, rows_of[keep], a.col_idx[keep], np.asarray(a.values)[keep])
    b_bytes = 4 * b.nnz
    try:
        for sem in (plus_pair_semiring(np.int64), plus_pair_semiring(np.float64), arithmetic_semiring(np.int64)):
            r = oracle.masked_multiply(m.pattern(), a, b, semiring_id=sem.kernel_id, dtype=sem.dtype)
            want = digest_csr(r.row_ptr, r.col_idx, r.values)
            for algo in ("hash", "auto"):
                for ph in ("1p", "2p"):
                    plan = MultiplyPlan(algorithm=algo, phases=ph, semiring=sem)
                    _tune(p20=0)
                    (c0, st0), n0 = _launches_of(lambda: masked_multiply_with_stats(m.pattern(), a, b, plan))
                    assert digest_csr(c0.row_ptr, c0.col_idx, c0.values) == want
                    for blocks in (2, 3, 7):
                        _tune(p20=b_bytes // blocks + 4)
                        (c, st), n = _launches_of(lambda: masked_multiply_with_stats(m.pattern(), a, b, plan))
                        assert digest_csr(c.row_ptr, c.col_idx, c.values) == want, (sem.name, algo, ph, blocks)
                        assert st.evaluated_multiplies == r.evaluated_multiplies, (sem.name, algo, ph, blocks)
                        assert st.generated_flops == r.generated_flops
                        blocked = ph == "1p" and sem.kernel_id != 0
                        if blocked and algo == "hash":
                            assert last_kernel_rows().get("hash_plain_t2s", 0) + last_kernel_rows().get("hash_plain_t2l", 0) > 0
                            assert n > n0, (sem.name, algo, ph, blocks, n, n0)     # the bin's launch repeated
                        if not blocked:
                            assert n == n0
    finally:
        _tune(p20=0)
