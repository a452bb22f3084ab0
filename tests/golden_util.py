"""Shared helpers for the golden fixtures (digest convention of make_golden.py)."""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def digest_csr(row_ptr, col_idx, values) -> str:
    row_ptr = np.asarray(row_ptr)
    nnz = int(row_ptr[-1])
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(row_ptr, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(np.asarray(col_idx)[:nnz], dtype=np.int64).tobytes())
    v = np.asarray(values)[:nnz]
    v = v.astype(np.float64) if v.dtype.kind == "f" else v.astype(np.int64)
    h.update(np.ascontiguousarray(v).tobytes())
    return h.hexdigest()


def digest_pattern(row_ptr, col_idx) -> str:
    row_ptr = np.asarray(row_ptr)
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(row_ptr, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(np.asarray(col_idx)[: int(row_ptr[-1])],
                                  dtype=np.int64).tobytes())
    return h.hexdigest()


def digest_mat(m) -> str:
    vals = getattr(m, "values", None)
    if vals is None:
        return digest_pattern(m.row_ptr, m.col_idx)
    return digest_csr(m.row_ptr, m.col_idx, vals)


def load_json(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def load_npz(name):
    return np.load(os.path.join(GOLDEN, name))


def random_csr(rng, nrows, ncols, avg_degree, vmax=9):
    """The reference's test fixture (pkg/tests/conftest.py:7-13), restated so
    the same rng stream yields the same matrix."""
    from paper_2111_09947_b200.sparse import from_arrays
    nnz = max(int(avg_degree * nrows), 0)
    rows = rng.integers(0, nrows, nnz) if nrows else np.empty(0, dtype=np.int64)
    cols = rng.integers(0, ncols, nnz) if ncols else np.empty(0, dtype=np.int64)
    vals = rng.integers(1, vmax, max(nnz, 0))
    return from_arrays(nrows, ncols, rows, cols, vals)


def regenerate_random_cases():
    """Rebuild the inputs of random_cases.json from its seed (same draw order
    as make_golden.make_random_cases).  Yields (case, A, B, M, semiring)."""
    from paper_2111_09947_b200.semiring import arithmetic_semiring, plus_pair_semiring
    spec = load_json("random_cases.json")
    rng = np.random.default_rng(spec["seed"])
    for case in spec["cases"]:
        m = int(rng.integers(1, 97))
        k = int(rng.integers(1, 97))
        n = int(rng.integers(1, 97))
        da = int(rng.integers(1, 17))
        db = int(rng.integers(1, 17))
        dm = int(rng.integers(0, 17))
        comp = bool(rng.integers(0, 2))
        assert (m, k, n, da, db, dm, comp) == (case["m"], case["k"], case["n"], case["da"],
                                               case["db"], case["dm"], case["complemented"])
        a = random_csr(rng, m, k, da)
        b = random_csr(rng, k, n, db)
        mm = random_csr(rng, m, n, dm)
        if case["kind"] == "fp64":
            a = a.astype(np.float64)
            a.values[:] = rng.standard_normal(a.nnz)
            b = b.astype(np.float64)
            b.values[:] = rng.standard_normal(b.nnz)
            sem = arithmetic_semiring(np.float64)
        elif case["kind"] == "plus_pair":
            sem = plus_pair_semiring(np.int64)
        else:
            sem = arithmetic_semiring(np.int64)
        yield case, a, b, mm, sem


def acceptance_instance(rng):
    """The reference's acceptance instance (pkg/tests/test_acceptance.py:41-49),
    restated with the same draw order as make_golden.acceptance_instance."""
    n = int(rng.integers(8, 129))
    d_in = int(rng.integers(1, 17))
    d_mask = int(rng.integers(1, 17))
    a = random_csr(rng, n, n, d_in)
    b = random_csr(rng, n, n, d_in)
    m = random_csr(rng, n, n, d_mask)
    comp = bool(rng.integers(0, 2))
    return n, a, b, m, comp
