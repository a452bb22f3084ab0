"""The reference's acceptance properties, re-pointed at the CUDA path.

Fixtures: tests/golden/acceptance.json, written by running the REFERENCE
(tests/golden/make_golden.py --acceptance); the inputs are regenerated here
from the same seeds with the restated generators (tests/golden_util.py) and
pinned by digest.

* C1 (pkg/tests/test_acceptance.py:78-98): 500 random instances, seed 5001,
  every supported plan (heap NInspect 0 / 1 / inf, 1P and 2P, plus ``auto``)
  bitwise equal to the reference's dense-oracle result, one signature per
  instance, with the reference's generated / evaluated counters.
* C10 (:248-272): plain and complemented results partition the full-mask
  product (msa, hash, heap), 100 instances, seed 110.
* Full mask equals the plain product (pkg/tests/test_multiply.py:59-65).
* CSC B accepted by the push plans and inner (test_multiply.py:169-186).
* Signed zero: the first product is stored, never added to +0.0
  (_kernels.py:59, 176, 188, 302, 469, 541).
"""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from golden_util import acceptance_instance, digest_csr, digest_mat, load_json, random_csr  # noqa: E402
from paper_2111_09947_b200 import (ALGORITHMS, MaskView, MultiplyPlan, arithmetic_semiring,  # noqa: E402
                                   from_arrays, masked_multiply, masked_multiply_with_stats)
from paper_2111_09947_b200.sparse import to_csc  # noqa: E402

SR = arithmetic_semiring(np.int64)


@pytest.fixture(autouse=True, scope="module")
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


@pytest.fixture(scope="module")
def fx():
    return load_json("acceptance.json")


def _supported_plans(comp):
    """test_acceptance.py:52-62 plus NInspect = inf and ``auto``."""
    algos = [x for x in ALGORITHMS + ("auto",) if not (comp and x in ("mca", "inner"))]
    plans = [MultiplyPlan(algorithm=x, phases=ph, complemented=comp, semiring=SR)
             for x in algos for ph in ("1p", "2p")]
    plans += [MultiplyPlan(algorithm="heap", phases=ph, complemented=comp, semiring=SR, n_inspect=ni)
              for ph in ("1p", "2p") for ni in (0, math.inf)]
    return plans


def _dg(c):
    return digest_csr(c.row_ptr, c.col_idx, c.values)


def test_c1_oracle_sweep_every_plan(fx):
    rng = np.random.default_rng(fx["c1"]["seed"])
    checked = 0
    for rec in fx["c1"]["instances"]:
        n, a, b, m, comp = acceptance_instance(rng)
        assert (n, comp) == (rec["n"], rec["complemented"])
        assert digest_mat(a) == rec["digest_a"] and digest_mat(m) == rec["digest_m"]
        sigs = set()
        for plan in _supported_plans(comp):
            c, st = masked_multiply_with_stats(m.pattern(), a, b, plan)
            sig = (_dg(c), st.generated_flops, st.evaluated_multiplies)
            assert sig == (rec["digest_c"], rec["generated"], rec["evaluated"]), (
                plan.label(), plan.n_inspect, comp, n)
            sigs.add(sig)
            checked += 1
        assert len(sigs) == 1
    assert checked >= 500 * 12


def test_c10_complement_duality(fx):
    rng = np.random.default_rng(fx["c10"]["seed"])
    for rec in fx["c10"]["instances"]:
        n = int(rng.integers(8, 65))
        assert n == rec["n"]
        a = random_csr(rng, n, n, 4)
        b = random_csr(rng, n, n, 4)
        m = random_csr(rng, n, n, 4)
        for algo in ("msa", "hash", "heap", "auto"):
            plain = masked_multiply(m.pattern(), a, b, MultiplyPlan(algorithm=algo, semiring=SR))
            comp = masked_multiply(m.pattern(complemented=True), a, b, MultiplyPlan(algorithm=algo, semiring=SR))
            whole = masked_multiply(MaskView.full(n, n), a, b, MultiplyPlan(algorithm=algo, semiring=SR))
            assert {"plain": _dg(plain), "comp": _dg(comp), "whole": _dg(whole)} == rec["digests"], algo
            pr, pc, pv = plain.triples()
            cr, cc, cv = comp.triples()
            merged = from_arrays(n, n, np.concatenate([pr, cr]), np.concatenate([pc, cc]),
                                 np.concatenate([pv, cv]))
            assert plain.nnz + comp.nnz == whole.nnz          # disjoint
            assert merged.equals(whole)                       # and covering


def test_full_mask_is_plain_product(fx):
    rng = np.random.default_rng(fx["full_mask"]["seed"])
    a = random_csr(rng, 32, 32, 4)
    b = random_csr(rng, 32, 32, 4)
    want = a.to_dense() @ b.to_dense()
    assert int(want.sum()) == fx["full_mask"]["dense_sum"]
    for plan in _supported_plans(False):
        c = masked_multiply(MaskView.full(32, 32), a, b, plan)
        assert np.array_equal(c.to_dense(), want), plan.label()
        assert _dg(c) == fx["full_mask"]["digest_c"], plan.label()


def test_csc_b_accepted(fx):
    rng = np.random.default_rng(fx["csc_b"]["seed"])
    a = random_csr(rng, 12, 12, 3)
    b = random_csr(rng, 12, 12, 3)
    mask = random_csr(rng, 12, 12, 3).pattern()
    for algo in ("msa", "hash", "mca", "heap", "heapdot", "inner", "auto"):
        for ph in ("1p", "2p"):
            c = masked_multiply(mask, a, to_csc(b), MultiplyPlan(algorithm=algo, phases=ph, semiring=SR))
            assert _dg(c) == fx["csc_b"]["digest_c"], (algo, ph)
        if algo in fx["csc_b"]["per_algorithm"]:
            assert fx["csc_b"]["per_algorithm"][algo] == fx["csc_b"]["digest_c"]


def test_signed_zero_first_product_stored(fx):
    kat = fx["signed_zero"]
    rows = [r for r, _, _ in kat["a"]]
    cols = [c for _, c, _ in kat["a"]]
    a = from_arrays(2, 2, rows, cols, np.array([float.fromhex(v) for _, _, v in kat["a"]]))
    b = from_arrays(2, 2, [r for r, _, _ in kat["b"]], [c for _, c, _ in kat["b"]],
                    np.array([float.fromhex(v) for _, _, v in kat["b"]]))
    f64 = arithmetic_semiring(np.float64)
    algos = ALGORITHMS + ("auto",)
    plans = [MultiplyPlan(algorithm=x, phases=ph, semiring=f64) for x in algos for ph in ("1p", "2p")]
    plans += [MultiplyPlan(algorithm="heap", phases=ph, semiring=f64, n_inspect=0) for ph in ("1p", "2p")]
    want = kat["per_plan"]["MSA-1P"]
    assert want["vals_hex"][0] == "-0x0.0p+0"        # the reference keeps the sign of the first product
    for plan in plans:
        key = plan.label() + ("" if plan.n_inspect is None else f"-ni{plan.n_inspect}")
        ref = kat["per_plan"].get(key, want)
        c = masked_multiply(MaskView.full(2, 2), a, b, plan)
        assert c.col_idx.tolist() == ref["cols"], key
        assert [float(x).hex() for x in c.values] == ref["vals_hex"], key
