"""Randomised parity fuzz of the device graph-side operations against their host forms:
csr_from_coo / simple_undirected_graph / degree_sort_relabel / tril_strict / transpose
(prep.py vs sparse.py), ewise_add and lookup_rows (elementwise.py vs numpy), triangle_count
(plain and streamed upload) and k_truss (vs a host fixed point on the C oracle)."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from paper_2111_09947_b200 import MultiplyPlan, prep, plus_pair_semiring
from paper_2111_09947_b200.device import DeviceCsr
from paper_2111_09947_b200.elementwise import ewise_add, lookup_rows
from paper_2111_09947_b200.graphs import k_truss, triangle_count, triangle_count_lower_streamed
from paper_2111_09947_b200.sparse import (degree_sort_relabel, from_arrays, simple_undirected_graph, to_csc,
                                          tril_strict)

ap = argparse.ArgumentParser()
ap.add_argument("--seconds", type=float, default=300)
ap.add_argument("--seed", type=int, default=1)
args = ap.parse_args()
rng = np.random.default_rng(args.seed)


def same(dev, host, what, info):
    h = dev.to_host()
    if not (np.array_equal(h.row_ptr, host.row_ptr) and np.array_equal(h.col_idx[: h.nnz], host.col_idx[: host.nnz])):
        print("MISMATCH", what, info, flush=True)
        sys.exit(1)


t_end = time.time() + args.seconds
cases = 0
while time.time() < t_end:
    n = int(rng.choice([1, 2, 17, 300, 5000, 60000]))
    e = int(rng.choice([0, 1, 50, 4000, 200000]))
    r = rng.integers(0, n, e)
    c = rng.integers(0, n, e)
    if e > 100 and rng.random() < 0.4:            # a hub vertex, duplicates
        hub = int(rng.integers(1, e // 2))
        r[:hub] = int(rng.integers(0, n))
    info = dict(case=cases, seed=args.seed, n=n, e=e)
    g = simple_undirected_graph(from_arrays(n, n, r, c, np.ones(e, dtype=np.int64)))
    dg = prep.simple_undirected_graph(r, c, n)
    same(dg, g, "simple_undirected_graph", info)
    rl, perm = degree_sort_relabel(g)
    drl, dperm = prep.degree_sort_relabel(dg)
    if not np.array_equal(dperm.cpu().numpy(), perm):
        print("MISMATCH perm", info, flush=True); sys.exit(1)
    same(drl, rl, "relabel", info)
    low = tril_strict(rl)
    same(prep.tril_strict(drl), low, "tril", info)
    same(prep.triangle_lower(dg), low, "triangle_lower", info)
    # rectangular matrix with values: from_arrays / transpose / ewise_add / lookup_rows
    m2, n2 = int(rng.choice([1, 30, 2000])), int(rng.choice([1, 40, 3000, 100000]))
    def mat(ne):
        rr, cc = rng.integers(0, m2, ne), rng.integers(0, n2, ne)
        return from_arrays(m2, n2, rr, cc, rng.standard_normal(ne))
    x, y = mat(int(rng.choice([0, 5, 3000, 50000]))), mat(int(rng.choice([0, 7, 2000, 80000])))
    dx, dy = DeviceCsr.from_host(x, dtype=np.float64), DeviceCsr.from_host(y, dtype=np.float64)
    t = dx.transpose_storage(); want = to_csc(x)
    if not (np.array_equal(t.ptr.cpu().numpy(), want.col_ptr) and np.array_equal(t.idx.cpu().numpy(), want.row_idx[: want.nnz])
            and np.array_equal(t.values.cpu().numpy(), want.values[: want.nnz])):
        print("MISMATCH transpose", info, (m2, n2, x.nnz), flush=True); sys.exit(1)
    s = ewise_add(dx, dy).to_host()
    dense = {}
    for mtx in (x, y):
        rows = np.repeat(np.arange(m2), np.diff(mtx.row_ptr))
        for i, j, v in zip(rows.tolist(), mtx.col_idx[: mtx.nnz].tolist(), mtx.values[: mtx.nnz].tolist()):
            dense[(i, j)] = dense.get((i, j), 0.0) + v if (i, j) in dense else v
    keys = sorted(dense)
    srows = np.repeat(np.arange(m2), np.diff(s.row_ptr))
    if [(int(a), int(b)) for a, b in zip(srows, s.col_idx[: s.nnz])] != keys or \
            not np.array_equal(np.asarray(s.values[: s.nnz]), np.array([dense[k] for k in keys])):
        print("MISMATCH ewise_add", info, (m2, n2, x.nnz, y.nnz), flush=True); sys.exit(1)
    out, found = lookup_rows(dx, dy)
    out, found = out.cpu().numpy(), found.cpu().numpy().astype(bool)
    xr = np.repeat(np.arange(m2), np.diff(x.row_ptr))
    ydict = {}
    yr = np.repeat(np.arange(m2), np.diff(y.row_ptr))
    for i, j, v in zip(yr.tolist(), y.col_idx[: y.nnz].tolist(), y.values[: y.nnz].tolist()):
        ydict[(i, j)] = v
    wf = np.array([(i, j) in ydict for i, j in zip(xr.tolist(), x.col_idx[: x.nnz].tolist())], dtype=bool)
    wv = np.array([ydict.get((i, j), 0.0) for i, j in zip(xr.tolist(), x.col_idx[: x.nnz].tolist())])
    if not (np.array_equal(found, wf) and np.array_equal(out[wf], wv[wf])):
        print("MISMATCH lookup_rows", info, (m2, n2, x.nnz, y.nnz), flush=True); sys.exit(1)
    # graph kernels on the smaller graphs
    if g.nnz <= 60000:
        plan = MultiplyPlan(algorithm=str(rng.choice(["auto", "hash", "msa"])))
        tri_ref = int(oracle.masked_multiply(low.pattern(), low, low, semiring_id=1).values.sum()) if low.nnz else 0
        if triangle_count(g, plan).value != tri_ref:
            print("MISMATCH triangle_count", info, flush=True); sys.exit(1)
        h_ptr = torch.from_numpy(np.ascontiguousarray(low.row_ptr, dtype=np.int64)).pin_memory()
        h_idx = torch.from_numpy(np.ascontiguousarray(low.col_idx[: low.nnz], dtype=np.int32)).pin_memory()
        if low.nrows and triangle_count_lower_streamed(h_ptr, h_idx, plan, first_fraction=float(rng.random())).value != tri_ref:
            print("MISMATCH streamed triangle_count", info, flush=True); sys.exit(1)
        kk = int(rng.choice([3, 4, 5]))
        cur = g
        while cur.nnz:
            rr = oracle.masked_multiply(cur.pattern(), cur, cur, semiring_id=1)
            keep = rr.values >= kk - 2
            rows = np.repeat(np.arange(cur.nrows), np.diff(rr.row_ptr))
            if int(keep.sum()) == cur.nnz:
                break
            cur = from_arrays(cur.nrows, cur.ncols, rows[keep], rr.col_idx[keep], np.ones(int(keep.sum()), dtype=np.int64))
        got = k_truss(g, kk, plan).value
        if not (np.array_equal(got.row_ptr, cur.row_ptr) and np.array_equal(got.col_idx[: got.nnz], cur.col_idx[: cur.nnz])):
            print("MISMATCH k_truss", info, kk, flush=True); sys.exit(1)
    cases += 1
print("graph fuzz ok:", cases, "cases, seed", args.seed)
