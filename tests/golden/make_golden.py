"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

This script is test infrastructure.  It imports the read-only reference package
``maskmul`` from /root/reference/pkg/src (available only in the build
container, never on the GPU box) and freezes its outputs as small JSON / npz
fixtures that the oracle and the CUDA path are pinned against.

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py            # KATs, random cases, cfg1-4
    ... make_golden.py --cfg2                          # R-MAT s20 triangle count (~1 min)
    ... make_golden.py --cfg5                          # R-MAT s22 k-truss support (~8 min)
    ... make_golden.py --bc                            # betweenness centrality scores
    ... make_golden.py --acceptance                    # the reference's acceptance properties

Digest convention (shared with tests/golden_util.py): sha256 over the
little-endian bytes of int64 row_ptr, then int64 col_idx[:nnz], then the values
(int64 or float64) [:nnz].

Input recipes follow SURVEY.md §8(d) exactly; random instances follow the
reference's own ``random_csr`` fixture (pkg/tests/conftest.py:7-13) and
acceptance-instance shape (pkg/tests/test_acceptance.py:41-49).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import sys
import time

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import maskmul  # noqa: E402
from maskmul import (GeneratorSpec, MaskView, MultiplyPlan, arithmetic_semiring,  # noqa: E402
                     degree_sort_relabel, from_arrays, from_triples, generate,
                     masked_multiply_with_stats, plus_pair_semiring,
                     simple_undirected_graph, symbolic_phase, tril_strict,
                     triangle_count)
from maskmul.multiply import ALGORITHMS  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def digest_csr(row_ptr, col_idx, values) -> str:
    nnz = int(row_ptr[-1])
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(row_ptr, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(col_idx[:nnz], dtype=np.int64).tobytes())
    v = np.asarray(values[:nnz])
    if v.dtype.kind == "f":
        v = v.astype(np.float64)
    else:
        v = v.astype(np.int64)
    h.update(np.ascontiguousarray(v).tobytes())
    return h.hexdigest()


def digest_mat(m) -> str:
    vals = getattr(m, "values", None)
    if vals is None:
        vals = np.zeros(0, dtype=np.int64)
        h = hashlib.sha256()
        h.update(np.ascontiguousarray(m.row_ptr, dtype=np.int64).tobytes())
        h.update(np.ascontiguousarray(m.col_idx[: m.nnz], dtype=np.int64).tobytes())
        return h.hexdigest()
    return digest_csr(m.row_ptr, m.col_idx, vals)


def random_csr(rng, nrows, ncols, avg_degree, vmax=9):
    # restated from pkg/tests/conftest.py:7-13 so the stream is identical
    nnz = max(int(avg_degree * nrows), 0)
    rows = rng.integers(0, nrows, nnz) if nrows else np.empty(0, dtype=np.int64)
    cols = rng.integers(0, ncols, nnz) if ncols else np.empty(0, dtype=np.int64)
    vals = rng.integers(1, vmax, max(nnz, 0))
    return from_arrays(nrows, ncols, rows, cols, vals)


def all_plans(comp, sem):
    algos = [a for a in ALGORITHMS if not (comp and a in ("mca", "inner"))]
    plans = [MultiplyPlan(algorithm=a, phases=ph, complemented=comp, semiring=sem)
             for a in algos for ph in ("1p", "2p")]
    plans += [MultiplyPlan(algorithm="heap", phases=ph, complemented=comp, semiring=sem,
                           n_inspect=0) for ph in ("1p", "2p")]
    return plans


# ---------------------------------------------------------------------------
# known-answer tests
# ---------------------------------------------------------------------------

def make_kats():
    sr = arithmetic_semiring(np.int64)
    out = {}
    # worked row example (pkg/tests/test_accumulators.py:35-39,142-148) as a 1-row multiply
    b = from_triples(2, 3, [(0, 0, 1), (0, 2, 3), (1, 1, 4), (1, 2, 5)])
    a = from_triples(1, 2, [(0, 0, 1), (0, 1, 2)])
    m = from_triples(1, 3, [(0, 0, 1), (0, 2, 1)])
    c, st = masked_multiply_with_stats(m.pattern(), a, b, MultiplyPlan(semiring=sr))
    out["worked_row"] = {"cols": c.col_idx.tolist(), "vals": c.values.tolist(),
                         "generated": st.generated_flops, "evaluated": st.evaluated_multiplies}
    # complemented empty mask (test_accumulators.py:176-182)
    empty = from_triples(1, 3, [])
    c, _ = masked_multiply_with_stats(empty.pattern(complemented=True), a, b,
                                      MultiplyPlan(semiring=sr))
    out["worked_row_empty_complement"] = {"cols": c.col_idx.tolist(), "vals": c.values.tolist()}

    def cg(n):
        return from_triples(n, n, [(i, j, 1) for i in range(n) for j in range(n) if i != j])
    out["tc_complete"] = {str(n): triangle_count(cg(n), MultiplyPlan()).value for n in (3, 4, 5)}
    g = simple_undirected_graph(generate(GeneratorSpec("erdos-renyi", 10, 8, seed=42)))
    out["tc_er10_d8_seed42"] = triangle_count(g, MultiplyPlan()).value
    out["er10_d8_seed42_graph_digest"] = digest_mat(g)
    k4 = cg(4)
    c, _ = masked_multiply_with_stats(k4.pattern(), k4, k4, MultiplyPlan(semiring=sr))
    out["k4_masked_square_nnz"] = c.nnz
    # lazy evaluation instance (test_acceptance.py:168-174)
    a1 = from_triples(1, 1, [(0, 0, 2)])
    b1 = from_triples(1, 3, [(0, 0, 3), (0, 1, 4), (0, 2, 5)])
    m1 = from_triples(1, 3, [(0, 0, 1), (0, 2, 1)])
    _, st = masked_multiply_with_stats(m1.pattern(), a1, b1, MultiplyPlan(semiring=sr))
    out["lazy"] = {"generated": st.generated_flops, "evaluated": st.evaluated_multiplies}
    # hash complement wide mask (test_multiply.py:148-158)
    n = 400
    mw = from_triples(1, n, [(0, j, 1) for j in range(0, n, 2)])
    aw = from_triples(1, 1, [(0, 0, 2)])
    bw = from_triples(1, n, [(0, 1, 3)])
    c, _ = masked_multiply_with_stats(mw.pattern(complemented=True), aw, bw,
                                      MultiplyPlan(algorithm="hash", semiring=sr))
    out["hash_complement_wide"] = {"cols": c.col_idx.tolist(), "vals": c.values.tolist()}
    # cancellation zero stored (test_multiply.py:76-83)
    ac = from_triples(1, 2, [(0, 0, 1), (0, 1, -1)])
    bc = from_triples(2, 1, [(0, 0, 5), (1, 0, 5)])
    c, _ = masked_multiply_with_stats(MaskView.full(1, 1), ac, bc, MultiplyPlan(semiring=sr))
    out["cancellation"] = {"nnz": c.nnz, "vals": c.values.tolist()}
    # symbolic identity (test_multiply.py:190-194)
    eye = from_triples(4, 4, [(i, i, 1) for i in range(4)])
    out["symbolic_identity"] = symbolic_phase(MaskView.full(4, 4), eye, eye,
                                              MultiplyPlan(semiring=sr)).tolist()
    return out


# ---------------------------------------------------------------------------
# random instances (int64 arithmetic, plus-pair, fp64)
# ---------------------------------------------------------------------------

def make_random_cases(n_int=80, n_fp=24, n_pp=16, seed=20261020):
    rng = np.random.default_rng(seed)
    cases = []
    for idx in range(n_int + n_fp + n_pp):
        kind = "int" if idx < n_int else ("fp64" if idx < n_int + n_fp else "plus_pair")
        m = int(rng.integers(1, 97))
        k = int(rng.integers(1, 97))
        n = int(rng.integers(1, 97))
        da = int(rng.integers(1, 17))
        db = int(rng.integers(1, 17))
        dm = int(rng.integers(0, 17))
        comp = bool(rng.integers(0, 2))
        a = random_csr(rng, m, k, da)
        b = random_csr(rng, k, n, db)
        mm = random_csr(rng, m, n, dm)
        if kind == "fp64":
            a = a.astype(np.float64)
            a.values[:] = rng.standard_normal(a.nnz)
            b = b.astype(np.float64)
            b.values[:] = rng.standard_normal(b.nnz)
            sem = arithmetic_semiring(np.float64)
        elif kind == "plus_pair":
            sem = plus_pair_semiring(np.int64)
        else:
            sem = arithmetic_semiring(np.int64)
        per_plan = {}
        stats = None
        for plan in all_plans(comp, sem):
            c, st = masked_multiply_with_stats(mm.pattern(), a, b, plan)
            key = plan.label() + ("" if plan.n_inspect is None else f"-ni{plan.n_inspect}")
            per_plan[key] = digest_csr(c.row_ptr, c.col_idx, c.values)
            if stats is None:
                stats = (st.generated_flops, st.evaluated_multiplies, c.nnz)
            assert stats[:2] == (st.generated_flops, st.evaluated_multiplies), key
        cases.append({
            "kind": kind, "m": m, "k": k, "n": n, "da": da, "db": db, "dm": dm,
            "complemented": comp,
            "digest_a": digest_mat(a), "digest_b": digest_mat(b), "digest_m": digest_mat(mm),
            "generated": stats[0], "evaluated": stats[1], "nnz": stats[2],
            "digest_c": per_plan,
        })
    return {"seed": seed, "recipe": "see make_random_cases in make_golden.py", "cases": cases}


# ---------------------------------------------------------------------------
# BASELINE configs (SURVEY.md §8(d) recipes)
# ---------------------------------------------------------------------------

def run_cfg(name, mask, a, b, plan, save_full=False, workers=8):
    plan = MultiplyPlan(algorithm=plan.algorithm, phases=plan.phases,
                        complemented=plan.complemented, semiring=plan.semiring,
                        workers=workers)
    t0 = time.perf_counter()
    c, st = masked_multiply_with_stats(mask, a, b, plan)
    dt = time.perf_counter() - t0
    rec = {
        "digest_a": digest_mat(a), "digest_b": digest_mat(b),
        "digest_m": digest_mat(mask),
        "nnz_a": a.nnz, "nnz_b": b.nnz, "nnz_m": mask.nnz,
        "nrows": a.nrows, "ncols": b.ncols,
        "generated": st.generated_flops, "evaluated": st.evaluated_multiplies,
        "nnz_c": c.nnz, "digest_c": digest_csr(c.row_ptr, c.col_idx, c.values),
        "sum_c": (float(c.values[: c.nnz].sum()) if c.values.dtype.kind == "f"
                  else int(c.values[: c.nnz].sum())),
        "plan": plan.label(), "reference_seconds_8w": st.total_seconds,
        "wall_seconds": dt,
    }
    if save_full:
        np.savez_compressed(os.path.join(HERE, f"{name}_C.npz"),
                            row_ptr=c.row_ptr, col_idx=c.col_idx[: c.nnz],
                            values=c.values[: c.nnz])
    print(name, {k: v for k, v in rec.items() if not k.startswith("digest")}, flush=True)
    return rec


def cfg1():
    a = generate(GeneratorSpec("erdos-renyi", 12, 8, seed=0)).astype(np.float64)
    a.values[:] = np.random.default_rng(1).random(a.nnz)
    return run_cfg("cfg1", a.pattern(), a, a,
                   MultiplyPlan(semiring=arithmetic_semiring(np.float64)), save_full=True)


def cfg2():
    g = simple_undirected_graph(generate(GeneratorSpec("rmat", 20, 16, seed=0)))
    low = tril_strict(degree_sort_relabel(g)[0])
    rec = run_cfg("cfg2", low.pattern(), low, low,
                  MultiplyPlan(semiring=plus_pair_semiring(np.int64)))
    rec["digest_graph"] = digest_mat(g)
    return rec


def cfg3():
    a = generate(GeneratorSpec("erdos-renyi", 18, 16, seed=0)).astype(np.float64)
    a.values[:] = np.random.default_rng(100).random(a.nnz)
    b = generate(GeneratorSpec("erdos-renyi", 18, 16, seed=1)).astype(np.float64)
    b.values[:] = np.random.default_rng(101).random(b.nnz)
    out = {}
    for d in (1, 4, 16, 64):
        m = generate(GeneratorSpec("erdos-renyi", 18, d, seed=2))
        out[str(d)] = run_cfg(f"cfg3_d{d}", m.pattern(), a, b,
                              MultiplyPlan(semiring=arithmetic_semiring(np.float64)),
                              save_full=True)
    return out


def cfg4():
    g = simple_undirected_graph(generate(GeneratorSpec("rmat", 18, 16, seed=0)))
    n = g.nrows
    rng = np.random.default_rng(4)
    src = rng.choice(n, 512, replace=False)
    ft = from_arrays(512, n, np.arange(512), src, np.ones(512, dtype=np.int64))
    dense = rng.random((512, n)) < 0.05
    r, c = np.nonzero(dense)
    v = from_arrays(512, n, r, c, np.ones(r.size, dtype=np.int64))
    rec = run_cfg("cfg4", v.pattern(), ft, g,
                  MultiplyPlan(complemented=True, semiring=arithmetic_semiring(np.int64)),
                  save_full=True)
    rec["digest_graph"] = digest_mat(g)
    rec["src_first8"] = [int(x) for x in src[:8]]
    return rec


def cfg5():
    g = simple_undirected_graph(generate(GeneratorSpec("rmat", 22, 16, seed=0)))
    return run_cfg("cfg5", g.pattern(), g, g,
                   MultiplyPlan(semiring=plus_pair_semiring(np.int64)))



# ---------------------------------------------------------------------------
# Betweenness centrality (graphs.py:136-200), SURVEY §8(f) row 2
# ---------------------------------------------------------------------------

def _bc_graph(spec):
    """Graph recipes of the reference's BC tests (pkg/tests/test_graphs.py:110-170,
    test_acceptance.py:139-152) and two larger R-MAT instances."""
    from maskmul.graphs import BcConfig  # noqa: F401
    kind = spec["graph"]
    if kind == "path":
        edges = []
        for i in range(spec["n"] - 1):
            edges += [(i, i + 1, 1), (i + 1, i, 1)]
        return from_triples(spec["n"], spec["n"], edges)
    if kind == "star":
        edges = []
        for i in range(1, spec["leaves"] + 1):
            edges += [(0, i, 1), (i, 0, 1)]
        return from_triples(spec["leaves"] + 1, spec["leaves"] + 1, edges)
    if kind == "disconnected":
        return from_triples(4, 4, [(0, 1, 1), (1, 0, 1), (2, 3, 1), (3, 2, 1)])
    if kind == "random":   # test_graphs.random_graph with the rng fixture (conftest.py:48-49)
        rng = np.random.default_rng(spec["seed"])
        return simple_undirected_graph(random_csr(rng, spec["n"], spec["n"], spec["degree"]))
    if kind == "rmat":
        return simple_undirected_graph(generate(GeneratorSpec("rmat", spec["scale"], spec["ef"],
                                                              seed=spec["seed"])))
    raise ValueError(kind)


BC_CASES = [
    {"graph": "path", "n": 3, "batch": 2, "plans": ["msa"]},
    {"graph": "path", "n": 4, "batch": 2, "plans": ["heap"]},
    {"graph": "star", "leaves": 4, "batch": 3, "plans": ["msa"]},
    {"graph": "star", "leaves": 4, "batch": 4, "plans": ["msa"]},
    {"graph": "disconnected", "batch": 4, "plans": ["msa"]},
    {"graph": "rmat", "scale": 6, "ef": 4, "seed": 5, "batch": 16, "plans": ["msa", "hash", "heap"]},
    {"graph": "random", "n": 24, "degree": 3, "seed": 20240811, "batch": 3, "sources": [0, 3, 7, 11],
     "plans": ["msa"]},
    {"graph": "random", "n": 20, "degree": 3, "seed": 20240811, "batch": 1, "plans": ["msa"]},
    {"graph": "random", "n": 20, "degree": 3, "seed": 20240811, "batch": 20, "plans": ["msa"]},
    {"graph": "random", "n": 30, "degree": 4, "seed": 20240811, "batch": 8, "plans": ["hash"]},
    {"graph": "rmat", "scale": 8, "ef": 4, "seed": 11, "batch": 64, "plans": ["msa"]},
    {"graph": "rmat", "scale": 10, "ef": 8, "seed": 3, "batch": 128, "n_sources": 256, "source_seed": 7,
     "plans": ["msa", "hash"]},
]


def make_bc():
    from maskmul.graphs import BcConfig, betweenness_centrality
    out = []
    for spec in BC_CASES:
        g = _bc_graph(spec)
        sources = spec.get("sources")
        if "n_sources" in spec:
            sources = [int(x) for x in np.random.default_rng(spec["source_seed"]).choice(
                g.nrows, spec["n_sources"], replace=False)]
        rec = dict(spec)
        rec["sources"] = sources
        rec["digest_graph"] = digest_mat(g)
        rec["results"] = {}
        for algo in spec["plans"]:
            t0 = time.perf_counter()
            res = betweenness_centrality(g, BcConfig(batch_size=spec["batch"], sources=sources),
                                         MultiplyPlan(algorithm=algo))
            rec["results"][algo] = {
                "scores_hex": [float(x).hex() for x in res.value],
                "multiplies": res.multiplies, "flops": int(res.flops), "evaluated": int(res.evaluated),
                "wall_seconds": time.perf_counter() - t0,
            }
        print("bc", {k: v for k, v in rec.items() if k != "results"},
              {a: (r["multiplies"], r["flops"]) for a, r in rec["results"].items()}, flush=True)
        out.append(rec)
    return out


# ---------------------------------------------------------------------------
# the reference's own acceptance properties, frozen for the GPU path
# ---------------------------------------------------------------------------

def acceptance_instance(rng):
    """pkg/tests/test_acceptance.py:41-49 (_random_instance), same draw order."""
    n = int(rng.integers(8, 129))
    d_in = int(rng.integers(1, 17))
    d_mask = int(rng.integers(1, 17))
    a = random_csr(rng, n, n, d_in)
    b = random_csr(rng, n, n, d_in)
    m = random_csr(rng, n, n, d_mask)
    comp = bool(rng.integers(0, 2))
    return n, a, b, m, comp


def make_acceptance():
    """C1 (test_acceptance.py:78-98: 500 instances, seed 5001, every plan incl.
    heap NInspect 0/1/inf, exact vs the dense oracle), C10 (:248-272:
    complement duality, seed 110, 100 instances, msa/hash/heap), the full-mask
    and CSC-B properties of test_multiply.py (:59-65, :169-186, rng fixture
    seed 20240811) and a signed-zero KAT (_kernels.py:59: the first product is
    stored, not added to +0.0).  Every expected output is the reference's own,
    and C1's is also checked here against the reference's dense oracle."""
    sys.path.insert(0, "/root/reference/pkg/tests")
    from oracles import dense_masked_product
    from maskmul.sparse import to_csc
    sr = arithmetic_semiring(np.int64)
    out = {}
    rng = np.random.default_rng(5001)
    c1 = []
    for _ in range(500):
        n, a, b, m, comp = acceptance_instance(rng)
        keep, values = dense_masked_product(m.to_dense() != 0, a.to_dense(), b.to_dense(), comp)
        rows, cols = np.nonzero(keep)
        want = from_arrays(a.nrows, b.ncols, rows, cols, values[rows, cols])
        sig = None
        for plan in all_plans(comp, sr) + [MultiplyPlan(algorithm="heap", phases=ph, complemented=comp,
                                                        semiring=sr, n_inspect=math.inf)
                                           for ph in ("1p", "2p")]:
            c, st = masked_multiply_with_stats(m.pattern(), a, b, plan)
            assert c.equals(want), plan.label()
            s2 = (digest_csr(c.row_ptr, c.col_idx, c.values), st.generated_flops, st.evaluated_multiplies)
            assert sig is None or s2 == sig
            sig = s2
        c1.append({"n": n, "complemented": comp, "digest_c": sig[0], "generated": sig[1],
                   "evaluated": sig[2], "nnz": want.nnz, "digest_a": digest_mat(a), "digest_m": digest_mat(m)})
    out["c1"] = {"seed": 5001, "instances": c1}
    rng = np.random.default_rng(110)
    c10 = []
    for _ in range(100):
        n = int(rng.integers(8, 65))
        a = random_csr(rng, n, n, 4)
        b = random_csr(rng, n, n, 4)
        m = random_csr(rng, n, n, 4)
        rec = {"n": n}
        for algo in ("msa", "hash", "heap"):
            plain = masked_multiply_with_stats(m.pattern(), a, b, MultiplyPlan(algorithm=algo, semiring=sr))[0]
            comp = masked_multiply_with_stats(m.pattern(complemented=True), a, b,
                                              MultiplyPlan(algorithm=algo, semiring=sr))[0]
            whole = masked_multiply_with_stats(MaskView.full(n, n), a, b,
                                               MultiplyPlan(algorithm=algo, semiring=sr))[0]
            assert plain.nnz + comp.nnz == whole.nnz
            d = {k: digest_csr(x.row_ptr, x.col_idx, x.values)
                 for k, x in (("plain", plain), ("comp", comp), ("whole", whole))}
            assert rec.get("digests", d) == d
            rec["digests"] = d
        c10.append(rec)
    out["c10"] = {"seed": 110, "instances": c10}
    rng = np.random.default_rng(20240811)          # the reference's rng fixture
    a = random_csr(rng, 32, 32, 4)
    b = random_csr(rng, 32, 32, 4)
    whole = masked_multiply_with_stats(MaskView.full(32, 32), a, b, MultiplyPlan(semiring=sr))[0]
    dense = a.to_dense() @ b.to_dense()
    assert np.array_equal(whole.to_dense(), dense)
    out["full_mask"] = {"seed": 20240811, "digest_c": digest_csr(whole.row_ptr, whole.col_idx, whole.values),
                        "dense_sum": int(dense.sum())}
    rng = np.random.default_rng(20240811)
    a = random_csr(rng, 12, 12, 3)
    b = random_csr(rng, 12, 12, 3)
    mask = random_csr(rng, 12, 12, 3).pattern()
    want = masked_multiply_with_stats(mask, a, b, MultiplyPlan(semiring=sr))[0]
    csc = {}
    for algo in ("msa", "hash", "mca", "heap", "heapdot", "inner"):
        c = masked_multiply_with_stats(mask, a, to_csc(b), MultiplyPlan(algorithm=algo, semiring=sr))[0]
        assert c.equals(want), algo
        csc[algo] = digest_csr(c.row_ptr, c.col_idx, c.values)
    out["csc_b"] = {"seed": 20240811, "digest_c": digest_csr(want.row_ptr, want.col_idx, want.values),
                    "per_algorithm": csc}
    # signed zero: (-1.0) * 0.0 = -0.0 is stored as the slot's first product;
    # a second product -0.0 keeps it -0.0; +0.0 + (-0.0) would give +0.0
    f64 = arithmetic_semiring(np.float64)
    a = from_triples(2, 2, [(0, 0, -1.0), (1, 0, -1.0), (1, 1, 2.0)]).astype(np.float64)
    b = from_triples(2, 2, [(0, 0, 0.0), (0, 1, 3.0), (1, 0, -0.0)]).astype(np.float64)
    a.values[:] = [-1.0, -1.0, 2.0]
    b.values[:] = [0.0, 3.0, -0.0]
    kat = {}
    for plan in all_plans(False, f64):
        c = masked_multiply_with_stats(MaskView.full(2, 2), a, b, plan)[0]
        kat[plan.label() + ("" if plan.n_inspect is None else f"-ni{plan.n_inspect}")] = {
            "cols": c.col_idx.tolist(), "vals_hex": [float(x).hex() for x in c.values]}
    out["signed_zero"] = {"a": [[0, 0, "-0x1.0000000000000p+0"], [1, 0, "-0x1.0000000000000p+0"],
                                [1, 1, "0x1.0000000000000p+1"]],
                          "b": [[0, 0, "0x0.0p+0"], [0, 1, "0x1.8000000000000p+1"], [1, 0, "-0x0.0p+0"]],
                          "per_plan": kat}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg2", action="store_true")
    ap.add_argument("--cfg5", action="store_true")
    ap.add_argument("--small", action="store_true")
    ap.add_argument("--bc", action="store_true")
    ap.add_argument("--acceptance", action="store_true")
    args = ap.parse_args()
    meta = {"numpy": np.__version__, "reference": "maskmul " + maskmul.__version__,
            "python": sys.version.split()[0]}
    try:
        import numba
        meta["numba"] = numba.__version__
    except ImportError:
        pass
    path = os.path.join(HERE, "configs.json")
    cfgs = json.load(open(path)) if os.path.exists(path) else {}
    cfgs["_meta"] = meta
    if args.small:
        with open(os.path.join(HERE, "kats.json"), "w") as f:
            json.dump(make_kats(), f, indent=1)
        with open(os.path.join(HERE, "random_cases.json"), "w") as f:
            json.dump(make_random_cases(), f)
        cfgs["cfg1"] = cfg1()
        cfgs["cfg3"] = cfg3()
        cfgs["cfg4"] = cfg4()
    if args.bc:
        with open(os.path.join(HERE, "bc.json"), "w") as f:
            json.dump({"meta": meta, "cases": make_bc()}, f)
    if args.acceptance:
        with open(os.path.join(HERE, "acceptance.json"), "w") as f:
            json.dump({"meta": meta, **make_acceptance()}, f)
    if args.cfg2:
        cfgs["cfg2"] = cfg2()
    if args.cfg5:
        cfgs["cfg5"] = cfg5()
    with open(path, "w") as f:
        json.dump(cfgs, f, indent=1)


if __name__ == "__main__":
    main()
