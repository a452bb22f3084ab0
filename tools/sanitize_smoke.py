"""Small multiplies through every kernel family, for compute-sanitizer runs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from golden_util import random_csr
from paper_2111_09947_b200 import MultiplyPlan, arithmetic_semiring, plus_pair_semiring, masked_multiply
import oracle
rng = np.random.default_rng(3)
n = 3000
checks = 0
for rows, da, dm, db in [(40, 4, 6, 8), (20, 30, 120, 30), (6, 200, 900, 64), (2, 600, 9000, 40)]:
    a = random_csr(rng, rows, 500, da)
    b = random_csr(rng, 500, n, db // 4 + 1)
    m = random_csr(rng, rows, n, dm)
    for sem in (arithmetic_semiring(np.int64), plus_pair_semiring(np.int64), arithmetic_semiring(np.float64)):
        aa, bb = a, b
        if sem.dtype == np.float64:
            aa = a.astype(np.float64); aa.values[:] = rng.standard_normal(aa.nnz)
            bb = b.astype(np.float64); bb.values[:] = rng.standard_normal(bb.nnz)
        for comp in (False, True):
            r = oracle.masked_multiply(m.pattern(), aa, bb, complemented=comp, semiring_id=sem.kernel_id, dtype=sem.dtype)
            for algo in ("hash", "msa", "heap", "auto") + (() if comp else ("mca", "inner")):
                for ph in ("1p", "2p"):
                    c = masked_multiply(m.pattern(), aa, bb, MultiplyPlan(algorithm=algo, phases=ph, complemented=comp, semiring=sem))
                    assert np.array_equal(c.col_idx, r.col_idx) and np.array_equal(c.values, r.values), (algo, ph, comp)
                    checks += 1
print("sanitize smoke ok", checks)
