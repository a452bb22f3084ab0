"""The reference-side ctypes stub of INTEGRATION.md (tools/reference_stub/_b200.py)
run for real: a `_Prepared` with the reference's field names
(pkg/src/maskmul/multiply.py:175-233) goes through the stub, the result must
equal this package's multiply (pinned to the reference's goldens) bitwise,
for every plan incl. inner (B held as CSC only) and complement."""

import importlib.util
import math
import os
import types

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from golden_util import digest_csr, random_csr  # noqa: E402
from paper_2111_09947_b200 import (MultiplyPlan, arithmetic_semiring, masked_multiply_with_stats,  # noqa: E402
                                   plus_pair_semiring)
from paper_2111_09947_b200.build import LIB_PATH  # noqa: E402
from paper_2111_09947_b200.sparse import to_csc  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def stub():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    os.environ["MASKMUL_B200_LIB"] = LIB_PATH
    spec = importlib.util.spec_from_file_location("maskmul_b200_stub",
                                                  os.path.join(ROOT, "tools", "reference_stub", "_b200.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _prepared(mask, a, b, plan, comp):
    """The reference's _Prepared fields the stub reads (multiply.py:175-233)."""
    p = types.SimpleNamespace()
    dt = np.dtype(plan.semiring.dtype)
    p.comp, p.dtype, p.nrows, p.ncols = comp, dt, mask.nrows, mask.ncols
    p.a_ptr = np.asarray(a.row_ptr, np.int64)
    p.a_idx = np.asarray(a.col_idx[: a.nnz], np.int64)
    p.a_val = np.asarray(a.values[: a.nnz]).astype(dt)
    p.m_ptr = np.asarray(mask.row_ptr, np.int64)
    p.m_idx = np.asarray(mask.col_idx[: mask.nnz], np.int64)
    if plan.algorithm == "inner":
        bc = to_csc(b)
        p.bc_ptr = np.asarray(bc.col_ptr, np.int64)
        p.bc_row = np.asarray(bc.row_idx[: bc.nnz], np.int64)
        p.bc_val = np.asarray(bc.values[: bc.nnz]).astype(dt)
        p.b_row_lengths = np.bincount(p.bc_row, minlength=b.nrows)
    else:
        p.b_ptr = np.asarray(b.row_ptr, np.int64)
        p.b_idx = np.asarray(b.col_idx[: b.nnz], np.int64)
        p.b_val = np.asarray(b.values[: b.nnz]).astype(dt)
        p.b_row_lengths = np.diff(p.b_ptr)
    ni = plan.effective_n_inspect
    p.kernel_ninspect = -1 if ni == math.inf else int(ni)
    return p


def test_stub_matches_package(stub):
    rng = np.random.default_rng(31)
    for _ in range(6):
        n = int(rng.integers(20, 300))
        a, b, m = (random_csr(rng, n, n, int(rng.integers(1, 12))) for _ in range(3))
        for sem in (arithmetic_semiring(np.int64), plus_pair_semiring(np.int64), arithmetic_semiring(np.float64)):
            aa, bb = a, b
            if sem.dtype == np.float64:
                aa = a.astype(np.float64)
                aa.values[:] = rng.standard_normal(aa.nnz)
                bb = b.astype(np.float64)
                bb.values[:] = rng.standard_normal(bb.nnz)
            for comp in (False, True):
                for algo in ("msa", "hash", "mca", "heap", "heapdot", "inner"):
                    if comp and algo in ("mca", "inner"):
                        continue
                    for ph in ("1p", "2p"):
                        plan = MultiplyPlan(algorithm=algo, phases=ph, complemented=comp, semiring=sem)
                        want, st = masked_multiply_with_stats(m.pattern(), aa, bb, plan)
                        ptr, idx, val, sst = stub.masked_multiply_b200(_prepared(m, aa, bb, plan, comp), plan)
                        assert digest_csr(ptr, idx, val) == digest_csr(want.row_ptr, want.col_idx, want.values), (
                            algo, ph, comp, sem.name)
                        assert (sst.generated_flops, sst.evaluated_multiplies) == (st.generated_flops,
                                                                                   st.evaluated_multiplies)
