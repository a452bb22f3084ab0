"""Parity of the CUDA path (through the C ABI) with the reference.

Every comparison is bitwise: sha256 digests of int64 row_ptr / col_idx and the
int64 or float64 values (tests/golden/, produced by running the reference),
or exact array equality against the C oracle (oracle/, itself pinned to the
reference by tests/test_oracle_golden.py).  float64 results are bit-identical
here because every GPU kernel folds products in the reference's ascending-k
order; the north_star tolerance (1e-12 relative) is asserted as well.
"""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from golden_util import (digest_csr, digest_mat, load_json, load_npz,  # noqa: E402
                         random_csr, regenerate_random_cases)
from paper_2111_09947_b200 import (ALGORITHMS, MaskView, MultiplyPlan, PlanError,  # noqa: E402
                                   SparseError, arithmetic_semiring, from_arrays, from_triples,
                                   masked_multiply, masked_multiply_with_stats,
                                   plus_pair_semiring, symbolic_phase, workloads)
from paper_2111_09947_b200.device import DeviceCsr  # noqa: E402
from paper_2111_09947_b200.multiply import multiply_device, reduce_sum  # noqa: E402

SR = arithmetic_semiring(np.int64)
ALL = ALGORITHMS + ("auto",)


@pytest.fixture(autouse=True, scope="module")
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def _plans(comp, sem, phases=("1p", "2p")):
    algos = [a for a in ALL if not (comp and a in ("mca", "inner"))]
    out = [MultiplyPlan(algorithm=a, phases=ph, complemented=comp, semiring=sem)
           for a in algos for ph in phases]
    out += [MultiplyPlan(algorithm="heap", phases=ph, complemented=comp, semiring=sem, n_inspect=0)
            for ph in phases]
    return out


def _digest(c):
    return digest_csr(c.row_ptr, c.col_idx, c.values)


def test_random_cases_against_reference_goldens():
    checked = 0
    for case, a, b, m, sem in regenerate_random_cases():
        comp = case["complemented"]
        want_msa = case["digest_c"]["MSA-1P"]
        for plan in _plans(comp, sem):
            c, st = masked_multiply_with_stats(m.pattern(), a, b, plan)
            key = plan.label() + ("" if plan.n_inspect is None else f"-ni{plan.n_inspect}")
            want = case["digest_c"].get(key, want_msa)
            if case["kind"] == "fp64" and plan.algorithm in ("heap", "heapdot"):
                # the reference's heap sums in heap-pop order; ours in ascending k
                want = want_msa
            assert _digest(c) == want, (case["kind"], key, comp)
            assert st.evaluated_multiplies == case["evaluated"], key
            assert st.generated_flops == case["generated"], key
            assert st.output_nnz == case["nnz"]
            checked += 1
    assert checked > 1500


def test_symbolic_counts_match_oracle():
    for case, a, b, m, sem in list(regenerate_random_cases())[:40]:
        comp = case["complemented"]
        r = oracle.masked_multiply(m.pattern(), a, b, complemented=comp, semiring_id=sem.kernel_id,
                                   dtype=sem.dtype)
        want = np.diff(r.row_ptr)
        for plan in _plans(comp, sem, phases=("1p",)):
            got = symbolic_phase(m.pattern(), a, b, plan)
            assert np.array_equal(got, want), plan.label()


def test_kats():
    k = load_json("kats.json")
    b = from_triples(2, 3, [(0, 0, 1), (0, 2, 3), (1, 1, 4), (1, 2, 5)])
    a = from_triples(1, 2, [(0, 0, 1), (0, 1, 2)])
    m = from_triples(1, 3, [(0, 0, 1), (0, 2, 1)])
    for plan in _plans(False, SR):
        c, st = masked_multiply_with_stats(m.pattern(), a, b, plan)
        assert c.col_idx.tolist() == k["worked_row"]["cols"], plan.label()
        assert c.values.tolist() == k["worked_row"]["vals"], plan.label()
        assert st.evaluated_multiplies == k["worked_row"]["evaluated"]
        assert st.generated_flops == k["worked_row"]["generated"]
    empty = from_triples(1, 3, [])
    for plan in _plans(True, SR):
        c = masked_multiply(empty.pattern(complemented=True), a, b, plan)
        assert c.col_idx.tolist() == k["worked_row_empty_complement"]["cols"]
        assert c.values.tolist() == k["worked_row_empty_complement"]["vals"]
    ac = from_triples(1, 2, [(0, 0, 1), (0, 1, -1)])
    bc = from_triples(2, 1, [(0, 0, 5), (1, 0, 5)])
    for plan in _plans(False, SR):
        c = masked_multiply(MaskView.full(1, 1), ac, bc, plan)
        assert c.nnz == 1 and c.values.tolist() == [0], plan.label()   # cancellation zero stored
    n = 400
    mw = from_triples(1, n, [(0, j, 1) for j in range(0, n, 2)])
    aw = from_triples(1, 1, [(0, 0, 2)])
    bw = from_triples(1, n, [(0, 1, 3)])
    for plan in _plans(True, SR):
        c = masked_multiply(mw.pattern(), aw, bw, plan)
        assert c.col_idx.tolist() == [1] and c.values.tolist() == [6]
    for plan in _plans(False, SR):
        assert masked_multiply(mw.pattern(), aw, bw, plan).nnz == 0
    a1 = from_triples(1, 1, [(0, 0, 2)])
    b1 = from_triples(1, 3, [(0, 0, 3), (0, 1, 4), (0, 2, 5)])
    m1 = from_triples(1, 3, [(0, 0, 1), (0, 2, 1)])
    for algo in ("msa", "hash", "mca", "heapdot", "auto"):
        _, st = masked_multiply_with_stats(m1.pattern(), a1, b1, MultiplyPlan(algorithm=algo, semiring=SR))
        assert (st.generated_flops, st.evaluated_multiplies) == (k["lazy"]["generated"], k["lazy"]["evaluated"])


def test_plan_and_shape_errors():
    a = from_triples(2, 2, [(0, 0, 1)])
    with pytest.raises(PlanError):
        masked_multiply(a.pattern(complemented=True), a, a, MultiplyPlan(algorithm="inner", semiring=SR))
    with pytest.raises(PlanError):
        masked_multiply(a.pattern(complemented=True), a, a, MultiplyPlan(algorithm="mca", semiring=SR))
    with pytest.raises(SparseError):
        masked_multiply(from_triples(2, 2, []).pattern(), from_triples(2, 3, []),
                        from_triples(4, 2, []), MultiplyPlan(semiring=SR))


def test_edge_shapes():
    rng = np.random.default_rng(7)
    # empty mask, empty A, empty B rows, zero-row matrices, single column
    cases = [
        (from_triples(10, 10, []), random_csr(rng, 10, 10, 3), random_csr(rng, 10, 10, 3)),
        (random_csr(rng, 10, 10, 3), from_triples(10, 10, []), random_csr(rng, 10, 10, 3)),
        (random_csr(rng, 10, 10, 3), random_csr(rng, 10, 10, 3), from_triples(10, 10, [])),
        (random_csr(rng, 1, 1, 1), random_csr(rng, 1, 7, 3), random_csr(rng, 7, 1, 1)),
        (random_csr(rng, 5, 300, 60), random_csr(rng, 5, 40, 30), random_csr(rng, 40, 300, 120)),
    ]
    for m, a, b in cases:
        for comp in (False, True):
            r = oracle.masked_multiply(m.pattern(), a, b, complemented=comp)
            for plan in _plans(comp, SR):
                c = masked_multiply(m.pattern(), a, b, plan)
                assert _digest(c) == digest_csr(r.row_ptr, r.col_idx, r.values), plan.label()


@pytest.mark.parametrize("comp", [False, True])
def test_every_tier_against_oracle(comp):
    """Rows sized to land in every kernel tier (warp / 4-warp / 16-warp smem
    tables, global-memory tables, complement search vs table)."""
    rng = np.random.default_rng(11 + comp)
    n = 40000
    specs = [(60, 4, 6, 8), (40, 30, 120, 30), (8, 200, 900, 64), (3, 600, 9000, 40),
             (2, 900, 30000, 200)]
    for rows, da, dm, db in specs:
        a = random_csr(rng, rows, 2000, da)
        b = random_csr(rng, 2000, n, db // 4 + 1)
        m = random_csr(rng, rows, n, dm)
        for sem in (SR, plus_pair_semiring(np.int64), arithmetic_semiring(np.float64)):
            aa, bb = a, b
            if sem.dtype == np.float64:
                aa = a.astype(np.float64)
                aa.values[:] = rng.standard_normal(aa.nnz)
                bb = b.astype(np.float64)
                bb.values[:] = rng.standard_normal(bb.nnz)
            r = oracle.masked_multiply(m.pattern(), aa, bb, complemented=comp,
                                       semiring_id=sem.kernel_id, dtype=sem.dtype)
            want = digest_csr(r.row_ptr, r.col_idx, r.values)
            for algo in ("hash", "msa", "heap") + (() if comp else ("inner", "auto", "mca")):
                plan = MultiplyPlan(algorithm=algo, complemented=comp, semiring=sem)
                c, st = masked_multiply_with_stats(m.pattern(), aa, bb, plan)
                assert _digest(c) == want, (rows, algo, sem.name, str(sem.dtype))
                assert st.evaluated_multiplies == r.evaluated_multiplies


@pytest.mark.parametrize("n", [300, 512, 6000])
def test_narrow_outputs_and_heavy_rows(n):
    """Heavy rows (tens of thousands of products) into narrow and wide
    outputs: the complemented dense MSA (every column in shared memory), the
    column-split ordered float64 groups (4/8/16 warps, bitwise order), 2P."""
    rng = np.random.default_rng(500 + n)
    rows = 24
    blocks = [random_csr(rng, 8, 3000, d) for d in (100, 600, 2500)]   # ~5K / 30K / 100K products per row
    a = from_arrays(rows, 3000,
                    np.concatenate([np.repeat(np.arange(8), np.diff(x.row_ptr)) + 8 * q for q, x in enumerate(blocks)]),
                    np.concatenate([x.col_idx[: x.nnz] for x in blocks]),
                    np.concatenate([x.values[: x.nnz] for x in blocks]))
    b = random_csr(rng, 3000, n, min(n / 6, 60))
    m = random_csr(rng, rows, n, min(n / 4, 150))
    for comp in (False, True):
        for sem in (SR, plus_pair_semiring(np.int64), arithmetic_semiring(np.float64)):
            aa, bb = a, b
            if sem.dtype == np.float64:
                aa = a.astype(np.float64)
                aa.values[:] = rng.standard_normal(aa.nnz)
                bb = b.astype(np.float64)
                bb.values[:] = rng.standard_normal(bb.nnz)
            r = oracle.masked_multiply(m.pattern(), aa, bb, complemented=comp,
                                       semiring_id=sem.kernel_id, dtype=sem.dtype)
            want = digest_csr(r.row_ptr, r.col_idx, r.values)
            for algo in ("msa", "hash", "auto") + (() if comp else ("mca",)):
                for ph in ("1p", "2p"):
                    plan = MultiplyPlan(algorithm=algo, phases=ph, complemented=comp, semiring=sem)
                    c, st = masked_multiply_with_stats(m.pattern(), aa, bb, plan)
                    assert _digest(c) == want, (n, comp, algo, ph, sem.name, str(sem.dtype))
                    assert st.evaluated_multiplies == r.evaluated_multiplies


@pytest.mark.parametrize("spec", [(64, 6, 20_000, 60_000, 200_000), (16, 80, 20_000, 60_000, 200_000),
                                  (4, 400, 30_000, 60_000, 200_000), (2, 7000, 20_000, 60_000, 200_000),
                                  (2, 7000, 600_000, 1_000_000, 4_000_000)])
def test_search_mode_long_b_rows(spec):
    """Hub B rows far longer than the mask rows: the plain hash rows
    binary-search each mask column in B_k instead of scanning it
    (flat_products SEARCH, product_loop.cuh); the result, the evaluated count
    and 1P == 2P must not change.  Hub rows of 20K-60K entries, masks of a
    few to thousands of columns (1-warp, 4-warp, 16-warp and sliced rows; the
    last case searches inside the column slices of sliced rows),
    some hub rows repeated inside one A row's batch, plus short B rows
    mixed in so scan and search share a row."""
    rows, dm, h_lo, h_hi, n = spec
    rng = np.random.default_rng(900 + dm + h_lo)
    hubs = 12
    hub_rows = [np.sort(rng.choice(n, int(rng.integers(h_lo, h_hi)), replace=False)) for _ in range(hubs)]
    short = random_csr(rng, 400, n, 5)
    b_rows = np.concatenate([np.full(h.size, q) for q, h in enumerate(hub_rows)] +
                            [np.repeat(np.arange(400), np.diff(short.row_ptr)) + hubs])
    b_cols = np.concatenate(hub_rows + [short.col_idx[: short.nnz]])
    b = from_arrays(hubs + 400, n, b_rows, b_cols, rng.integers(-5, 6, b_cols.size))
    a_r, a_c = [], []
    for i in range(rows):
        ks = np.unique(np.concatenate([rng.choice(hubs, 3, replace=False), hubs + rng.choice(400, 20)]))
        a_r.append(np.full(ks.size, i))
        a_c.append(ks)
    a = from_arrays(rows, hubs + 400, np.concatenate(a_r), np.concatenate(a_c),
                    rng.integers(-3, 4, sum(x.size for x in a_c)))
    # mask columns: half drawn from hub rows (hits), half anywhere
    m_r, m_c = [], []
    for i in range(rows):
        pool = hub_rows[int(rng.integers(hubs))]
        cols = np.unique(np.concatenate([rng.choice(pool, dm // 2 + 1), rng.choice(n, dm // 2 + 1)]))
        m_r.append(np.full(cols.size, i))
        m_c.append(cols)
    m = from_arrays(rows, n, np.concatenate(m_r), np.concatenate(m_c), np.ones(sum(x.size for x in m_c), np.int64))
    for sem in (SR, plus_pair_semiring(np.int64)):
        r = oracle.masked_multiply(m.pattern(), a, b, semiring_id=sem.kernel_id, dtype=sem.dtype)
        want = digest_csr(r.row_ptr, r.col_idx, r.values)
        for algo in ("hash", "auto"):
            for ph in ("1p", "2p"):
                plan = MultiplyPlan(algorithm=algo, phases=ph, semiring=sem)
                c, st = masked_multiply_with_stats(m.pattern(), a, b, plan)
                assert _digest(c) == want, (rows, dm, algo, ph, sem.name)
                assert st.evaluated_multiplies == r.evaluated_multiplies
                assert st.generated_flops == r.generated_flops


def test_determinism_repeat_and_row_partition():
    w = workloads.cfg1()
    d = [DeviceCsr.from_host(x, dtype=np.float64) for x in (w.a,)]
    da = d[0]
    dm = DeviceCsr.from_host(w.mask, with_values=False)
    plan = MultiplyPlan(semiring=w.semiring)
    c1, _ = multiply_device(dm, da, da, plan)
    c2, _ = multiply_device(dm, da, da, plan)
    assert torch.equal(c1.idx, c2.idx) and torch.equal(c1.values, c2.values)
    # row blocks computed separately concatenate to the same C (multi-GPU contract)
    from paper_2111_09947_b200.distributed import row_block, concat_row_blocks
    cuts = [0, 1000, 1001, 2500, w.a.nrows]
    parts = []
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        pa = row_block(da, lo, hi)
        pm = row_block(dm, lo, hi)
        cp, _ = multiply_device(pm, pa, da, plan)
        parts.append(cp)
    cc = concat_row_blocks(parts)
    assert torch.equal(cc.ptr, c1.ptr) and torch.equal(cc.idx, c1.idx)
    assert torch.equal(cc.values, c1.values)


def test_cfg1_bitwise():
    g = load_json("configs.json")["cfg1"]
    w = workloads.cfg1()
    for algo in ALL:
        for ph in ("1p", "2p"):
            c, st = masked_multiply_with_stats(w.mask, w.a, w.b,
                                               MultiplyPlan(algorithm=algo, phases=ph, semiring=w.semiring))
            if algo in ("heap", "heapdot"):
                assert _digest(c) == g["digest_c"]   # ascending-k order == MSA's
            else:
                assert _digest(c) == g["digest_c"], algo
            assert st.evaluated_multiplies == g["evaluated"]
    gold = load_npz("cfg1_C.npz")
    assert np.allclose(c.values, gold["values"], rtol=1e-12, atol=0)


@pytest.mark.parametrize("d", [1, 4, 16, 64])
def test_cfg3_bitwise(d):
    g = load_json("configs.json")["cfg3"][str(d)]
    w = workloads.cfg3(d)
    assert digest_mat(w.a) == g["digest_a"]
    for algo, ph in (("msa", "1p"), ("hash", "1p"), ("mca", "1p"), ("inner", "1p"), ("auto", "1p"),
                     ("inner", "2p")):     # inner: the lane-per-mask-entry pull kernel (numeric and symbolic)
        c, st = masked_multiply_with_stats(w.mask, w.a, w.b, MultiplyPlan(algorithm=algo, phases=ph,
                                                                          semiring=w.semiring))
        assert _digest(c) == g["digest_c"], (algo, ph)
        assert st.evaluated_multiplies == g["evaluated"]
    gold = load_npz(f"cfg3_d{d}_C.npz")
    rel = np.abs(c.values - gold["values"]) / np.maximum(np.abs(gold["values"]), 1e-300)
    assert rel.max(initial=0) <= 1e-12
    # the heap family and the two-phase push plans on the same inputs: pattern bit-exact,
    # float64 values within the north_star's 1e-12 relative (the heap folds in ascending k,
    # the reference's in heap-pop order, _kernels.py:380-463)
    for algo, ph in (("heap", "1p"), ("heapdot", "1p"), ("heap", "2p"), ("msa", "2p"), ("hash", "2p"), ("auto", "2p")):
        c, st = masked_multiply_with_stats(w.mask, w.a, w.b, MultiplyPlan(algorithm=algo, phases=ph,
                                                                          semiring=w.semiring))
        assert np.array_equal(c.row_ptr, gold["row_ptr"]), (algo, ph)
        assert np.array_equal(c.col_idx[: c.nnz], gold["col_idx"]), (algo, ph)
        rel = np.abs(c.values[: c.nnz] - gold["values"]) / np.maximum(np.abs(gold["values"]), 1e-300)
        assert rel.max(initial=0) <= 1e-12, (algo, ph)
        assert st.generated_flops == g["generated"], (algo, ph)


def test_cfg4_complement_bitwise():
    g = load_json("configs.json")["cfg4"]
    w = workloads.cfg4()
    assert digest_mat(w.mask) == g["digest_m"]
    for algo in ("msa", "hash", "heap", "heapdot", "auto"):
        for ph in ("1p", "2p"):
            c, st = masked_multiply_with_stats(w.mask, w.a, w.b,
                                               MultiplyPlan(algorithm=algo, phases=ph, complemented=True,
                                                            semiring=w.semiring))
            assert _digest(c) == g["digest_c"], algo
            assert st.evaluated_multiplies == g["evaluated"]


def test_cfg2_triangle_count_bitwise():
    g = load_json("configs.json")["cfg2"]
    w = workloads.cfg2()
    assert digest_mat(w.a) == g["digest_a"]
    dl = DeviceCsr.from_host(w.a, with_values=False)
    for algo in ("hash", "msa", "auto"):
        c, st = multiply_device(dl, dl, dl, MultiplyPlan(algorithm=algo, semiring=w.semiring),
                                b_csc=dl.transpose_storage() if algo == "auto" else None)
        assert st.generated_flops == g["generated"]
        assert st.evaluated_multiplies == g["evaluated"]
        assert c.nnz == g["nnz_c"]
        assert int(reduce_sum(c.values).item()) == g["sum_c"] == 423909251
        h = c.to_host()
        assert _digest(h) == g["digest_c"], algo


def test_cfg2_two_phase_and_algorithms():
    g = load_json("configs.json")["cfg2"]
    w = workloads.cfg2()
    dl = DeviceCsr.from_host(w.a, with_values=False)
    for algo, ph in (("msa", "2p"), ("hash", "2p"), ("mca", "1p"), ("auto", "2p")):
        c, st = multiply_device(dl, dl, dl, MultiplyPlan(algorithm=algo, phases=ph, semiring=w.semiring))
        assert st.evaluated_multiplies == g["evaluated"], (algo, ph)
        assert _digest(c.to_host()) == g["digest_c"], (algo, ph)


@pytest.mark.slow
def test_cfg5_ktruss_support_bitwise():
    """R-MAT scale 22 k-truss support C = A (.) (A A): hub rows (163,558-entry
    mask rows, 85M products) run on the global-memory tiers."""
    g = load_json("configs.json").get("cfg5")
    if g is None:
        pytest.skip("cfg5 golden not generated")
    w = workloads.cfg5()
    assert digest_mat(w.a) == g["digest_a"]
    da = DeviceCsr.from_host(w.a, with_values=False)
    c, st = multiply_device(da, da, da, MultiplyPlan(algorithm="auto", semiring=w.semiring))
    assert st.generated_flops == g["generated"]
    assert st.evaluated_multiplies == g["evaluated"]
    assert c.nnz == g["nnz_c"]
    assert int(reduce_sum(c.values).item()) == g["sum_c"]
    assert _digest(c.to_host()) == g["digest_c"]


def test_triangle_count_and_k_truss_graph_kernels():
    from paper_2111_09947_b200.graphs import k_truss, triangle_count
    from paper_2111_09947_b200.sparse import simple_undirected_graph
    from paper_2111_09947_b200.workloads import GeneratorSpec, generate
    k = load_json("kats.json")

    def complete(n):
        return from_triples(n, n, [(i, j, 1) for i in range(n) for j in range(n) if i != j])
    plan = MultiplyPlan(algorithm="auto")
    for n, want in k["tc_complete"].items():
        assert triangle_count(complete(int(n)), plan).value == want
    g = simple_undirected_graph(generate(GeneratorSpec("erdos-renyi", 10, 8, seed=42)))
    assert triangle_count(g, plan).value == k["tc_er10_d8_seed42"]
    assert k_truss(complete(5), 5, plan).value.nnz == 20      # test_graphs.py:72-74
    assert k_truss(complete(4), 5, plan).value.nnz == 0
    # input checks (graphs.py:75-84, test_graphs.py:55-61), now on the device
    directed = from_triples(3, 3, [(0, 1, 1), (1, 2, 1), (2, 0, 1)])
    loop = from_triples(2, 2, [(0, 0, 1), (0, 1, 1), (1, 0, 1)])
    rect = from_triples(2, 3, [(0, 1, 1)])
    empty = from_triples(4, 4, [])
    for fn in (lambda g: triangle_count(g, plan), lambda g: k_truss(g, 3, plan)):
        for bad in (directed, loop, rect):
            with pytest.raises(SparseError):
                fn(bad)
    assert triangle_count(empty, plan).value == 0
    assert k_truss(empty, 3, plan).value.nnz == 0
    # R-MAT scale-8 graphs against a host fixed point built on the oracle
    for seed in range(8):
        g = simple_undirected_graph(generate(GeneratorSpec("rmat", 8, 4, seed=seed)))
        cur = g
        while cur.nnz:
            r = oracle.masked_multiply(cur.pattern(), cur, cur, semiring_id=1)
            keep = r.values >= 3
            rows = np.repeat(np.arange(cur.nrows), np.diff(r.row_ptr))
            if int(keep.sum()) == cur.nnz:
                break
            from paper_2111_09947_b200.sparse import from_arrays
            cur = from_arrays(cur.nrows, cur.ncols, rows[keep], r.col_idx[keep],
                              np.ones(int(keep.sum()), dtype=np.int64))
        got = k_truss(g, 5, MultiplyPlan(algorithm="hash")).value
        assert np.array_equal(got.row_ptr, cur.row_ptr) and np.array_equal(got.col_idx, cur.col_idx[: cur.nnz])


@pytest.mark.parametrize("shape", ["tiny_rows", "skewed", "all_empty_but_one"])
def test_compact_rows_row_search_edges(shape):
    """mm_compact_rows against numpy: many 0/1-entry rows (the 32-ary row
    search with spans of exactly 32 rows), a few huge rows, empty rows."""
    import ctypes as C

    from paper_2111_09947_b200 import _lib

    rng = np.random.default_rng(7)
    n = 200_003
    if shape == "tiny_rows":
        cnt = rng.integers(0, 2, n)
    elif shape == "skewed":
        cnt = rng.integers(0, 3, n)
        cnt[rng.integers(0, n, 20)] = rng.integers(1000, 50_000, 20)
    else:
        cnt = np.zeros(n, np.int64)
        cnt[n // 2] = 70_000
    cnt = cnt.astype(np.int64)
    slack = rng.integers(0, 4, n).astype(np.int64)
    bounds = np.zeros(n + 1, np.int64)
    np.cumsum(cnt + slack, out=bounds[1:])
    out_ptr = np.zeros(n + 1, np.int64)
    np.cumsum(cnt, out=out_ptr[1:])
    tmp_idx = rng.integers(0, 1 << 30, int(bounds[-1])).astype(np.int32)
    tmp_val = rng.integers(-(1 << 40), 1 << 40, int(bounds[-1])).astype(np.int64)
    keep = np.concatenate([np.arange(bounds[i], bounds[i] + cnt[i]) for i in np.nonzero(cnt)[0]]) \
        if cnt.sum() else np.zeros(0, np.int64)
    dev = "cuda"
    t = {k: torch.from_numpy(v).to(dev) for k, v in
         dict(bounds=bounds, cnt=cnt, idx=tmp_idx, val=tmp_val, out_ptr=out_ptr).items()}
    oi = torch.empty(max(int(cnt.sum()), 1), dtype=torch.int32, device=dev)
    ov = torch.empty(max(int(cnt.sum()), 1), dtype=torch.int64, device=dev)
    lib = _lib.load()
    rc = lib.mm_compact_rows(n, t["bounds"].data_ptr(), t["cnt"].data_ptr(), t["idx"].data_ptr(),
                             t["val"].data_ptr(), t["out_ptr"].data_ptr(), oi.data_ptr(), ov.data_ptr(),
                             0, C.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0
    torch.cuda.synchronize()
    m = int(cnt.sum())
    assert np.array_equal(oi[:m].cpu().numpy(), tmp_idx[keep])
    assert np.array_equal(ov[:m].cpu().numpy(), tmp_val[keep])


def test_row_work_and_workspace_estimate():
    """mm_row_work (w_i = flops_i + nnz(M_i), multiply.py:103-108 + mask
    lengths) equals the host row_work; mm_workspace_bytes covers the slab."""
    import ctypes as C
    from paper_2111_09947_b200 import _lib
    from paper_2111_09947_b200.distributed import row_work, row_work_device
    from paper_2111_09947_b200.multiply import _plan_t
    rng = np.random.default_rng(8)
    a = random_csr(rng, 3000, 900, 7)
    b = random_csr(rng, 900, 1200, 9)
    m = random_csr(rng, 3000, 1200, 5)
    da, db = DeviceCsr.from_host(a, with_values=False), DeviceCsr.from_host(b, with_values=False)
    dm = DeviceCsr.from_host(m, with_values=False)
    got = row_work_device(da, db, dm).cpu().numpy()
    want = row_work(a.row_ptr, a.col_idx, b.row_ptr, m.row_ptr)
    assert np.array_equal(got, want)
    nbytes = C.c_size_t(0)
    pt = _plan_t(MultiplyPlan(), False)
    assert _lib.load().mm_workspace_bytes(C.byref(pt), C.byref(dm.mm()), C.byref(da.mm()), C.byref(db.mm()),
                                          C.byref(nbytes)) == 0
    assert nbytes.value >= 3000 * 8 * 3 + m.nnz * 12


def test_concurrent_threads_share_no_handle():
    """Two host threads multiplying at once on one device (each gets its own
    library handle) produce the same C as a single thread."""
    import threading
    w = workloads.cfg1()
    da = DeviceCsr.from_host(w.a, dtype=np.float64)
    dm = DeviceCsr.from_host(w.mask, with_values=False)
    plan = MultiplyPlan(semiring=w.semiring)
    ref, _ = multiply_device(dm, da, da, plan)
    torch.cuda.synchronize()
    out, errs = [], []

    def work():
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(20):
                    c, _ = multiply_device(dm, da, da, plan, stream=s)
                s.synchronize()
                out.append(c)
        except Exception as e:   # pragma: no cover - reported below
            errs.append(e)

    ts = [threading.Thread(target=work) for _ in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for c in out:
        assert torch.equal(c.idx, ref.idx) and torch.equal(c.values, ref.values)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_float64_push_pull_per_row_with_bt(seed):
    """Ordered float64 rows given B^T (auto): the deferred-hit kernel picks
    push or pull per row (push_f64_defer.cuh), both fold in ascending k, so C
    is bitwise the oracle's.  Rows span short / wide masks (pull vs push),
    dense hits (hit-list overflow -> in-order walk), masks over the direct
    path's limit (fallback to the binned path) and 1P / 2P."""
    rng = np.random.default_rng(4242 + seed)
    n = 3000
    blocks = []
    for rows, da, dm in ((200, 8, 1), (200, 8, 4), (200, 16, 64), (50, 30, 300), (20, 60, 3000)):
        blocks.append((random_csr(rng, rows, n, da), random_csr(rng, rows, n, dm)))
    a = from_arrays(sum(x.nrows for x, _ in blocks), n,
                    np.concatenate([np.repeat(np.arange(x.nrows), np.diff(x.row_ptr)) + off
                                    for (x, _), off in zip(blocks, np.cumsum([0] + [x.nrows for x, _ in blocks[:-1]]))]),
                    np.concatenate([x.col_idx[: x.nnz] for x, _ in blocks]),
                    rng.standard_normal(sum(x.nnz for x, _ in blocks)))
    m = from_arrays(a.nrows, n,
                    np.concatenate([np.repeat(np.arange(y.nrows), np.diff(y.row_ptr)) + off
                                    for (_, y), off in zip(blocks, np.cumsum([0] + [y.nrows for _, y in blocks[:-1]]))]),
                    np.concatenate([y.col_idx[: y.nnz] for _, y in blocks]),
                    np.ones(sum(y.nnz for _, y in blocks)))
    b = random_csr(rng, n, n, 6).astype(np.float64)
    b.values[:] = rng.standard_normal(b.nnz)
    sem = arithmetic_semiring(np.float64)
    r = oracle.masked_multiply(m.pattern(), a, b, semiring_id=0, dtype=np.float64)
    want = digest_csr(r.row_ptr, r.col_idx, r.values)
    da = DeviceCsr.from_host(a, dtype=np.float64)
    db = DeviceCsr.from_host(b, dtype=np.float64)
    dm = DeviceCsr.from_host(m.pattern(), with_values=False)
    bt = db.transpose_storage()
    for ph in ("1p", "2p"):
        for algo, csc in (("auto", bt), ("auto", None), ("hash", None), ("inner", bt)):
            c, st = multiply_device(dm, da, db, MultiplyPlan(algorithm=algo, phases=ph, semiring=sem), b_csc=csc)
            assert _digest(c.to_host()) == want, (algo, ph, csc is not None)
            assert st.evaluated_multiplies == r.evaluated_multiplies
            assert st.generated_flops == r.generated_flops


def test_plan_runs_its_accumulator():
    """The plan label names the accumulator that runs: every
    non-empty row of a named plan lands in a kernel of that family.  The one
    documented substitution: complemented MSA rows whose output is too wide
    for a state per column in shared memory run the hash complement kernels
    (DESIGN.md §4)."""
    from paper_2111_09947_b200.multiply import last_kernel_rows
    rng = np.random.default_rng(77)
    fam = {"msa": ("msa_",), "mca": ("mca_",), "heap": ("heap_",), "heapdot": ("heap_",),
           "hash": ("hash_",), "inner": ("pull",)}
    for rows, da, dm, n in ((200, 4, 6, 500), (40, 30, 120, 40000), (8, 200, 900, 40000), (3, 600, 9000, 40000)):
        a = random_csr(rng, rows, 2000, da)
        b = random_csr(rng, 2000, n, 4)
        m = random_csr(rng, rows, n, dm)
        for sem in (SR, plus_pair_semiring(np.int64), arithmetic_semiring(np.float64)):
            aa, bb = a, b
            if sem.dtype == np.float64:
                aa = a.astype(np.float64)
                bb = b.astype(np.float64)
            for comp in (False, True):
                for algo, prefixes in fam.items():
                    if comp and algo in ("mca", "inner"):
                        continue
                    masked_multiply(m.pattern(), aa, bb, MultiplyPlan(algorithm=algo, complemented=comp, semiring=sem))
                    used = {k: v for k, v in last_kernel_rows().items() if k != "empty"}
                    allowed = prefixes + (("hash_ctab", "hash_csrch") if comp and algo == "msa" else ())
                    bad = [k for k in used if not k.startswith(allowed)]
                    assert not bad, (algo, comp, sem.name, str(sem.dtype), used)


def test_direct_float64_long_a_rows_go_to_the_binned_pass():
    """Direct float64 path (no analysis pass): rows with more than 1024 A
    entries (one warp would walk them alone) and rows with wide masks are left
    to the binned pass; everything still equals the oracle bit for bit, counters
    included (reference order: _kernels.py:48-65)."""
    from paper_2111_09947_b200.multiply import last_kernel_rows
    rng = np.random.default_rng(77)
    m, n = 3000, 3000
    lens = rng.integers(1, 12, m)
    lens[[5, 1700]] = [2500, 1100]          # two hub rows of A
    a_r = np.repeat(np.arange(m), lens)
    a_c = np.concatenate([rng.choice(n, ln, replace=False) for ln in lens])
    a = from_arrays(m, n, a_r, a_c, rng.standard_normal(a_c.size))
    b_r = np.repeat(np.arange(n), rng.integers(1, 10, n))
    b = from_arrays(n, n, b_r, rng.integers(0, n, b_r.size), rng.standard_normal(b_r.size))
    m_len = rng.integers(0, 4, m)
    m_len[[5, 9]] = [40, 300]               # a hub row with a mask, a wide mask row
    m_r = np.repeat(np.arange(m), m_len)
    m_c = np.concatenate([rng.choice(n, ln, replace=False) for ln in m_len])
    mask = from_arrays(m, n, m_r, m_c, np.ones(m_c.size, dtype=np.int64)).pattern()
    sem = arithmetic_semiring(np.float64)
    c, st = masked_multiply_with_stats(mask, a, b, MultiplyPlan(algorithm="auto", semiring=sem))
    rows = last_kernel_rows()
    r = oracle.masked_multiply(mask, a, b, algorithm="msa", dtype=np.float64)
    assert np.array_equal(c.row_ptr, r.row_ptr)
    assert np.array_equal(c.col_idx[: c.nnz], r.col_idx)
    assert np.array_equal(c.values[: c.nnz], r.values)
    assert (st.generated_flops, st.evaluated_multiplies) == (r.generated_flops, r.evaluated_multiplies)
    assert sum(v for k, v in rows.items() if k != "empty") >= 1, rows
