"""Device input preparation against the host functions,
which mirror the reference (sparse.py:223-357): identical canonical CSR and
identical permutation, on random COO lists with duplicates and self-loops, on
R-MAT graphs (cfg2's s20 graph included, pinned by the golden digest), and on
segments long enough for the block / global bitonic paths."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from golden_util import digest_mat, load_json  # noqa: E402
from paper_2111_09947_b200 import prep  # noqa: E402
from paper_2111_09947_b200.device import DeviceCsr  # noqa: E402
from paper_2111_09947_b200.sparse import (degree_sort_relabel, from_arrays, simple_undirected_graph,  # noqa: E402
                                          to_csc, tril_strict)
from paper_2111_09947_b200.workloads import GeneratorSpec, generate, rmat_edges, simple_graph_direct  # noqa: E402


@pytest.fixture(autouse=True, scope="module")
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def _same(dev: DeviceCsr, host):
    h = dev.to_host()
    assert np.array_equal(h.row_ptr, host.row_ptr)
    assert np.array_equal(h.col_idx[: h.nnz], host.col_idx[: host.nnz])


@pytest.mark.parametrize("n,m,hub", [(50, 400, 0), (3000, 40000, 0), (2000, 60000, 9000), (70000, 300000, 80000)])
def test_simple_undirected_graph_matches_host(n, m, hub):
    rng = np.random.default_rng(n + m)
    r = rng.integers(0, n, m)
    c = rng.integers(0, n, m)
    if hub:   # one vertex with a long row: block and global bitonic paths
        r[:hub] = 0
        c[:hub] = rng.integers(0, n, hub)
    want = simple_undirected_graph(from_arrays(n, n, r, c, np.ones(m, dtype=np.int64)))
    got = prep.simple_undirected_graph(r, c, n)
    _same(got, want)


@pytest.mark.parametrize("scale", [8, 12, 16])
def test_relabel_tril_transpose_match_host(scale):
    g = simple_graph_direct(GeneratorSpec("rmat", scale, 16, seed=scale))
    dg = DeviceCsr.from_host(g, with_values=False)
    rl, perm = degree_sort_relabel(g)
    drl, dperm = prep.degree_sort_relabel(dg)
    assert np.array_equal(dperm.cpu().numpy(), perm)
    _same(drl, rl)
    _same(prep.tril_strict(drl), tril_strict(rl))
    _same(prep.triangle_lower(dg), tril_strict(rl))
    # transpose with values (8-byte payload follows its entry)
    a = generate(GeneratorSpec("erdos-renyi", scale, 8, seed=scale)).astype(np.float64)
    a.values[:] = np.random.default_rng(scale).standard_normal(a.nnz)
    da = DeviceCsr.from_host(a, dtype=np.float64)
    t = da.transpose_storage()
    want = to_csc(a)
    assert np.array_equal(t.ptr.cpu().numpy(), want.col_ptr)
    assert np.array_equal(t.idx.cpu().numpy(), want.row_idx[: want.nnz])
    assert np.array_equal(t.values.cpu().numpy(), want.values[: want.nnz])


def test_cfg2_input_pipeline_on_device():
    """R-MAT s20 edges (host generator) -> simple graph -> relabel -> tril on
    the device gives cfg2's L bit for bit (golden input digest)."""
    spec = GeneratorSpec("rmat", 20, 16, seed=0)
    src, dst = rmat_edges(spec)
    g = prep.simple_undirected_graph(src, dst, spec.nrows)
    low = prep.triangle_lower(g).to_host()
    want = load_json("configs.json")["cfg2"]["digest_m"]   # the pattern of L
    low.values = None
    assert digest_mat(low) == want


def test_prep_edge_cases():
    """Empty edge lists, only self-loops, a single vertex, duplicate-only
    input, and an empty graph through relabel / tril / transpose."""
    for n, r, c in ((5, [], []), (4, [0, 1, 2, 3], [0, 1, 2, 3]), (1, [0], [0]), (3, [1, 1, 1], [2, 2, 2])):
        r = np.asarray(r, dtype=np.int64)
        c = np.asarray(c, dtype=np.int64)
        want = simple_undirected_graph(from_arrays(n, n, r, c, np.ones(r.size, dtype=np.int64)))
        got = prep.simple_undirected_graph(r, c, n)
        _same(got, want)
        rl, perm = degree_sort_relabel(want)
        drl, dperm = prep.degree_sort_relabel(got)
        assert np.array_equal(dperm.cpu().numpy(), perm)
        _same(drl, rl)
        _same(prep.tril_strict(drl), tril_strict(rl))
        t = got.transpose_storage()
        assert np.array_equal(t.ptr.cpu().numpy(), to_csc(want).col_ptr)
    # rectangular transpose with an empty row block and int64 values
    a = from_arrays(6, 3, np.array([0, 0, 5]), np.array([2, 0, 1]), np.array([7, 8, 9], dtype=np.int64))
    da = DeviceCsr.from_host(a, dtype=np.int64)
    t = da.transpose_storage()
    want = to_csc(a)
    assert np.array_equal(t.ptr.cpu().numpy(), want.col_ptr)
    assert np.array_equal(t.idx.cpu().numpy(), want.row_idx[: want.nnz])
    assert np.array_equal(t.values.cpu().numpy(), want.values[: want.nnz])


@pytest.mark.parametrize("field,symmetric,dups", [("pattern", True, True), ("pattern", False, False),
                                                  ("real", False, False), ("real", True, False),
                                                  ("integer", False, True)])
def test_matrix_market_device_matches_host(tmp_path, field, symmetric, dups):
    """mmio.read_matrix_market_device == the host reader (which matches the
    reference bitwise, tests/test_mmio.py), for the canonical CSR and values."""
    from paper_2111_09947_b200.mmio import read_matrix_market, read_matrix_market_device
    rng = np.random.default_rng(31 + len(field) + symmetric)
    n, nnz = 20000, 150000
    key = rng.choice(n * n, nnz, replace=dups)
    r, c = key // n, key % n
    if symmetric:
        r, c = np.maximum(r, c), np.minimum(r, c)
        if not dups:   # keep the lower triangle free of repeats after folding
            k2 = np.unique(r * n + c)
            r, c = k2 // n, k2 % n
    lines = [f"%%MatrixMarket matrix coordinate {field} {'symmetric' if symmetric else 'general'}\n",
             f"{n} {n} {r.size}\n"]
    vals = rng.standard_normal(r.size)
    for t in range(r.size):
        v = "" if field == "pattern" else f" {float(vals[t])!r}" if field == "real" else f" {t % 17 - 8}"
        lines.append(f"{r[t] + 1} {c[t] + 1}{v}\n")
    p = tmp_path / "g.mtx"
    p.write_text("".join(lines))
    host = read_matrix_market(p)
    dev = read_matrix_market_device(p, device="cuda:0")
    _same(dev, host)
    if field == "pattern":
        assert dev.values is None
        full = read_matrix_market_device(p, device="cuda:0", with_values=True)
        _same(full, host)
        assert np.array_equal(full.values.cpu().numpy(), host.values)
    else:
        assert np.array_equal(dev.values.cpu().numpy(), host.values)   # bitwise (fp64 sums in file order)
