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

# narrow outputs (complemented dense MSA), heavy rows (column-split ordered float64)
for n2 in (300, 512):
    a = random_csr(rng, 6, 400, 150)
    b = random_csr(rng, 400, n2, 40)
    m = random_csr(rng, 6, n2, 60)
    for sem in (plus_pair_semiring(np.int64), arithmetic_semiring(np.float64)):
        aa, bb = a, b
        if sem.dtype == np.float64:
            aa = a.astype(np.float64); aa.values[:] = rng.standard_normal(aa.nnz)
            bb = b.astype(np.float64); bb.values[:] = rng.standard_normal(bb.nnz)
        for comp in (False, True):
            r = oracle.masked_multiply(m.pattern(), aa, bb, complemented=comp, semiring_id=sem.kernel_id, dtype=sem.dtype)
            for algo in ("msa", "auto", "hash"):
                c = masked_multiply(m.pattern(), aa, bb, MultiplyPlan(algorithm=algo, complemented=comp, semiring=sem))
                assert np.array_equal(c.col_idx, r.col_idx) and np.array_equal(c.values, r.values), (n2, algo, comp)
                checks += 1

# a plain row whose mask exceeds the shared tables: sliced hash rows
a = random_csr(rng, 2, 2000, 400)
b = random_csr(rng, 2000, 60000, 30)
m = random_csr(rng, 2, 60000, 12000)
r = oracle.masked_multiply(m.pattern(), a, b, semiring_id=1, dtype=np.int64)
c = masked_multiply(m.pattern(), a, b, MultiplyPlan(algorithm="hash", semiring=plus_pair_semiring(np.int64)))
assert np.array_equal(c.col_idx, r.col_idx) and np.array_equal(c.values, r.values)
checks += 1

# search mode: hub B rows far longer than the mask rows (1-warp / 4-warp / 16-warp hash rows)
from paper_2111_09947_b200.sparse import from_arrays as _fa
for rows_s, dm_s in ((16, 3), (4, 40), (2, 300)):
    hubs = [np.sort(rng.choice(40000, int(rng.integers(3000, 9000)), replace=False)) for _ in range(6)]
    b_r = np.concatenate([np.full(h.size, q) for q, h in enumerate(hubs)])
    b_s = _fa(6, 40000, b_r, np.concatenate(hubs), rng.integers(-4, 5, b_r.size))
    a_s = _fa(rows_s, 6, np.repeat(np.arange(rows_s), 6), np.tile(np.arange(6), rows_s), rng.integers(-3, 4, rows_s * 6))
    mr = np.repeat(np.arange(rows_s), dm_s)
    mc = np.concatenate([rng.choice(hubs[i % 6], dm_s) for i in range(rows_s)])
    m_s = _fa(rows_s, 40000, mr, mc, np.ones(mr.size, dtype=np.int64))
    for sem in (arithmetic_semiring(np.int64), plus_pair_semiring(np.int64)):
        r = oracle.masked_multiply(m_s.pattern(), a_s, b_s, semiring_id=sem.kernel_id, dtype=sem.dtype)
        c = masked_multiply(m_s.pattern(), a_s, b_s, MultiplyPlan(algorithm="hash", semiring=sem))
        assert np.array_equal(c.col_idx, r.col_idx) and np.array_equal(c.values, r.values)
        checks += 1

# graph drivers and device input preparation
import torch
from paper_2111_09947_b200 import prep
from paper_2111_09947_b200.graphs import BcConfig, betweenness_centrality
from paper_2111_09947_b200.sparse import simple_undirected_graph, from_arrays
from oracle.bc import betweenness_centrality as obc
rr = rng.integers(0, 200, 3000); cc = rng.integers(0, 200, 3000)
rr[:5000 // 2] = 0
g = simple_undirected_graph(from_arrays(200, 200, rr, cc, np.ones(3000, dtype=np.int64)))
res = betweenness_centrality(g, BcConfig(batch_size=64), MultiplyPlan(algorithm="msa"))
want = obc(g, 64, None, "msa")[0]
assert np.array_equal(res.value.view(np.int64), want.view(np.int64))
n3 = 9000
hr = rng.integers(0, n3, 20000); hc = rng.integers(0, n3, 20000)
hr[:6000] = 7                                     # a hub: block / global bitonic paths
dg = prep.simple_undirected_graph(hr, hc, n3)
hg = simple_undirected_graph(from_arrays(n3, n3, hr, hc, np.ones(hr.size, dtype=np.int64)))
assert np.array_equal(dg.ptr.cpu().numpy(), hg.row_ptr) and np.array_equal(dg.idx.cpu().numpy(), hg.col_idx[: hg.nnz])
low = prep.triangle_lower(dg)
checks += 3
torch.cuda.synchronize()
print("sanitize smoke (extended) ok", checks)
