"""Pin the CPU oracle (oracle/) against the reference's own outputs.

The fixtures in tests/golden/ were produced by running the reference package
(tests/golden/make_golden.py); every check here is bitwise (digests of
int64 row_ptr / col_idx and int64 or float64 values) plus the reference's
generated / evaluated counters.
"""

import numpy as np
import pytest

import oracle
from golden_util import (digest_csr, digest_mat, load_json, load_npz,
                         regenerate_random_cases)
from paper_2111_09947_b200 import workloads
from paper_2111_09947_b200.sparse import (MaskView, from_triples, simple_undirected_graph,
                                          to_csc)


def _plan_from_key(key):
    algo, ph = key.split("-")[:2]
    return algo.lower(), ph.lower(), (0 if key.endswith("ni0") else None)


def test_random_cases_every_plan_bitwise():
    n = 0
    for case, a, b, m, sem in regenerate_random_cases():
        assert digest_mat(a) == case["digest_a"]
        assert digest_mat(b) == case["digest_b"]
        assert digest_mat(m) == case["digest_m"]
        for key, want in case["digest_c"].items():
            algo, ph, ni = _plan_from_key(key)
            r = oracle.masked_multiply(m.pattern(), a, b, algorithm=algo, phases=ph,
                                       complemented=case["complemented"],
                                       semiring_id=sem.kernel_id, dtype=sem.dtype,
                                       n_inspect=ni, workers=2)
            assert digest_csr(r.row_ptr, r.col_idx, r.values) == want, (case, key)
            assert r.evaluated_multiplies == case["evaluated"], key
            assert r.generated_flops == case["generated"], key
            n += 1
    assert n > 1000


def test_symbolic_counts_equal_numeric_row_nnz():
    for case, a, b, m, sem in list(regenerate_random_cases())[:30]:
        algos = ["msa", "hash", "heap", "heapdot"] + ([] if case["complemented"] else ["mca", "inner"])
        for algo in algos:
            counts = oracle.symbolic_phase(m.pattern(), a, b, algorithm=algo,
                                           complemented=case["complemented"])
            r = oracle.masked_multiply(m.pattern(), a, b, algorithm=algo,
                                       complemented=case["complemented"],
                                       semiring_id=sem.kernel_id, dtype=sem.dtype)
            assert np.array_equal(counts, np.diff(r.row_ptr)), algo


def test_kats():
    k = load_json("kats.json")
    b = from_triples(2, 3, [(0, 0, 1), (0, 2, 3), (1, 1, 4), (1, 2, 5)])
    a = from_triples(1, 2, [(0, 0, 1), (0, 1, 2)])
    m = from_triples(1, 3, [(0, 0, 1), (0, 2, 1)])
    for algo in ("msa", "hash", "mca", "heap", "heapdot", "inner"):
        r = oracle.masked_multiply(m.pattern(), a, b, algorithm=algo)
        assert r.col_idx.tolist() == k["worked_row"]["cols"]
        assert r.values.tolist() == k["worked_row"]["vals"]
        assert r.evaluated_multiplies == k["worked_row"]["evaluated"]
    empty = from_triples(1, 3, [])
    for algo in ("msa", "hash", "heap"):
        r = oracle.masked_multiply(empty.pattern(), a, b, algorithm=algo, complemented=True)
        assert r.col_idx.tolist() == k["worked_row_empty_complement"]["cols"]
        assert r.values.tolist() == k["worked_row_empty_complement"]["vals"]
    ac = from_triples(1, 2, [(0, 0, 1), (0, 1, -1)])
    bc = from_triples(2, 1, [(0, 0, 5), (1, 0, 5)])
    r = oracle.masked_multiply(MaskView.full(1, 1), ac, bc)
    assert r.nnz == k["cancellation"]["nnz"] and r.values.tolist() == k["cancellation"]["vals"]
    n = 400
    mw = from_triples(1, n, [(0, j, 1) for j in range(0, n, 2)])
    aw = from_triples(1, 1, [(0, 0, 2)])
    bw = from_triples(1, n, [(0, 1, 3)])
    r = oracle.masked_multiply(mw.pattern(), aw, bw, algorithm="hash", complemented=True)
    assert r.col_idx.tolist() == k["hash_complement_wide"]["cols"]
    assert r.values.tolist() == k["hash_complement_wide"]["vals"]


def test_er10_triangle_kat():
    """ER scale 10 deg 8 seed 42 -> 618 triangles (pkg/test_output.txt:14)."""
    k = load_json("kats.json")
    g = simple_undirected_graph(workloads.generate(workloads.GeneratorSpec("erdos-renyi", 10, 8, seed=42)))
    assert digest_mat(g) == k["er10_d8_seed42_graph_digest"]
    from paper_2111_09947_b200.sparse import degree_sort_relabel, tril_strict
    low = tril_strict(degree_sort_relabel(g)[0])
    r = oracle.masked_multiply(low.pattern(), low, low, semiring_id=1)
    assert int(r.values.sum()) == k["tc_er10_d8_seed42"] == 618


def test_cfg1_full_output():
    cfg = load_json("configs.json")["cfg1"]
    w = workloads.cfg1()
    assert digest_mat(w.a) == cfg["digest_a"]
    gold = load_npz("cfg1_C.npz")
    for algo in ("msa", "hash", "mca", "inner"):
        r = oracle.masked_multiply(w.mask, w.a, w.b, algorithm=algo, dtype=np.float64)
        assert digest_csr(r.row_ptr, r.col_idx, r.values) == cfg["digest_c"]
        assert r.evaluated_multiplies == cfg["evaluated"]
    assert np.array_equal(gold["col_idx"], r.col_idx)


@pytest.mark.slow
def test_cfg3_cfg4_inputs_and_outputs():
    cfgs = load_json("configs.json")
    for d in (1, 4):
        w = workloads.cfg3(d)
        g = cfgs["cfg3"][str(d)]
        assert digest_mat(w.a) == g["digest_a"] and digest_mat(w.b) == g["digest_b"]
        r = oracle.masked_multiply(w.mask, w.a, w.b, algorithm="msa", dtype=np.float64,
                                   workers=oracle.max_threads())
        assert digest_csr(r.row_ptr, r.col_idx, r.values) == g["digest_c"]
    w = workloads.cfg4()
    g = cfgs["cfg4"]
    assert digest_mat(w.a) == g["digest_a"] and digest_mat(w.b) == g["digest_b"]
    assert digest_mat(w.mask) == g["digest_m"]
    r = oracle.masked_multiply(w.mask, w.a, w.b, algorithm="heap", complemented=True,
                               workers=oracle.max_threads())
    assert digest_csr(r.row_ptr, r.col_idx, r.values) == g["digest_c"]
    assert r.evaluated_multiplies == g["evaluated"]


def test_bc_oracle_matches_reference_scores_bitwise():
    """oracle/bc.py (graphs.py:136-200 restated) against the reference's own
    betweenness scores (tests/golden/bc.json), bit for bit, plus the reference's
    multiply count, generated flops and evaluated products."""
    from bc_cases import bc_cases, scores
    from oracle.bc import betweenness_centrality as oracle_bc
    n_checked = 0
    for spec, g in bc_cases():
        for algo, want in spec["results"].items():
            got, count, flops, evaluated = oracle_bc(g, spec["batch"], spec["sources"], algorithm=algo)
            ref = scores(want["scores_hex"])
            assert (count, flops, evaluated) == (want["multiplies"], want["flops"], want["evaluated"]), spec
            if algo == "heap":
                # the reference's heap folds fp64 in tie order: same to 1e-12
                np.testing.assert_allclose(got, ref, rtol=1e-12, atol=0)
            else:
                assert np.array_equal(got.view(np.int64), ref.view(np.int64)), (spec["graph"], algo)
            n_checked += 1
    assert n_checked >= 15


def test_acceptance_fixtures_oracle():
    """The oracle against the reference's acceptance fixtures (acceptance.json:
    C1 seed-5001 sweep and C10 complement duality, test_acceptance.py:78-98,
    248-272; signed-zero KAT, _kernels.py:59)."""
    from golden_util import acceptance_instance, random_csr
    fx = load_json("acceptance.json")
    rng = np.random.default_rng(fx["c1"]["seed"])
    for rec in fx["c1"]["instances"]:
        n, a, b, m, comp = acceptance_instance(rng)
        assert digest_mat(a) == rec["digest_a"] and digest_mat(m) == rec["digest_m"]
        algos = ["msa", "hash", "heap"] + ([] if comp else ["mca", "inner"])
        for algo in algos:
            r = oracle.masked_multiply(m.pattern(), a, b, algorithm=algo, complemented=comp)
            assert digest_csr(r.row_ptr, r.col_idx, r.values) == rec["digest_c"], algo
            assert (r.generated_flops, r.evaluated_multiplies) == (rec["generated"], rec["evaluated"])
    rng = np.random.default_rng(fx["c10"]["seed"])
    for rec in fx["c10"]["instances"]:
        n = int(rng.integers(8, 65))
        a, b, m = (random_csr(rng, n, n, 4) for _ in range(3))
        got = {}
        for key, mask, comp in (("plain", m.pattern(), False), ("comp", m.pattern(), True),
                                ("whole", MaskView.full(n, n), False)):
            r = oracle.masked_multiply(mask, a, b, algorithm="msa", complemented=comp)
            got[key] = digest_csr(r.row_ptr, r.col_idx, r.values)
        assert got == rec["digests"]
    kat = fx["signed_zero"]
    from paper_2111_09947_b200.sparse import from_arrays
    a = from_arrays(2, 2, [0, 1, 1], [0, 0, 1], np.array([float.fromhex(v) for _, _, v in kat["a"]]))
    b = from_arrays(2, 2, [0, 0, 1], [0, 1, 0], np.array([float.fromhex(v) for _, _, v in kat["b"]]))
    for algo in ("msa", "hash", "mca", "inner"):
        r = oracle.masked_multiply(MaskView.full(2, 2), a, b, algorithm=algo, dtype=np.float64)
        assert [float(x).hex() for x in r.values] == kat["per_plan"]["MSA-1P"]["vals_hex"], algo
