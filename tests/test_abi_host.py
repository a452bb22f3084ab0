"""CPU-only checks: the C-ABI library loads and exports every declared symbol,
and the host-side mirror of the reference API behaves like the reference."""

import ctypes
import math
import os
import re

import numpy as np
import pytest

from golden_util import digest_mat, load_json
from paper_2111_09947_b200 import (MaskView, MultiplyPlan, PlanError, SparseError, from_arrays,
                                   from_triples, plus_pair_semiring, to_csc, to_csr, transpose,
                                   tril_strict)
from paper_2111_09947_b200 import _lib, build
from paper_2111_09947_b200.distributed import balanced_cuts, row_work

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "maskmul_b200.h")


def _declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mm_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    if not os.path.exists(build.LIB_PATH):
        build.build()
    lib = ctypes.CDLL(build.LIB_PATH)
    declared = _declared_functions()
    assert declared, "no functions parsed from the header"
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(_lib.EXPORTS) == declared
    lib.mm_abi_version.restype = ctypes.c_int
    assert lib.mm_abi_version() == 1


def test_abi_struct_layouts_match_header():
    assert ctypes.sizeof(_lib.MatrixT) == 48
    assert ctypes.sizeof(_lib.PlanT) == 24
    assert ctypes.sizeof(_lib.StatsT) == 48


def test_plan_validation_and_labels():
    with pytest.raises(PlanError):
        MultiplyPlan(algorithm="spa")
    with pytest.raises(PlanError):
        MultiplyPlan(phases="3p")
    with pytest.raises(PlanError):
        MultiplyPlan(workers=0)
    with pytest.raises(PlanError):
        MultiplyPlan(n_inspect=2)
    with pytest.raises(PlanError):
        MultiplyPlan(algorithm="mca", complemented=True)
    with pytest.raises(PlanError):
        MultiplyPlan(algorithm="inner", complemented=True)
    assert MultiplyPlan(algorithm="msa").label() == "MSA-1P"
    assert MultiplyPlan(algorithm="heapdot", phases="2p").label() == "HeapDot-2P"
    assert MultiplyPlan(algorithm="heap").effective_n_inspect == 1
    assert MultiplyPlan(algorithm="heapdot").effective_n_inspect == math.inf
    assert MultiplyPlan(algorithm="auto").label() == "Auto-1P"


def test_sparse_constructors_canonical():
    m = from_triples(3, 4, [(2, 1, 5), (0, 3, 1), (0, 3, 2), (0, 0, 7)])
    assert m.row_ptr.tolist() == [0, 2, 2, 3]
    assert m.col_idx.tolist() == [0, 3, 1]
    assert m.values.tolist() == [7, 3, 5]
    c = to_csc(m)
    assert c.col_ptr.tolist() == [0, 1, 2, 2, 3]
    assert c.row_idx.tolist() == [0, 2, 0]
    back = to_csr(c)
    assert back.equals(m)
    t = transpose(transpose(m))
    assert t.equals(m)
    full = MaskView.full(2, 3)
    assert full.row_ptr.tolist() == [0, 3, 6]
    with pytest.raises(SparseError):
        from_arrays(2, 2, [0, 2], [0, 0], [1, 1])


def test_generators_match_reference_digests():
    from paper_2111_09947_b200 import workloads
    k = load_json("kats.json")
    from paper_2111_09947_b200.sparse import simple_undirected_graph
    g = simple_undirected_graph(
        workloads.generate(workloads.GeneratorSpec("erdos-renyi", 10, 8, seed=42)))
    assert digest_mat(workloads.simple_graph_direct(
        workloads.GeneratorSpec("erdos-renyi", 10, 8, seed=42))) == k["er10_d8_seed42_graph_digest"]
    assert digest_mat(g) == k["er10_d8_seed42_graph_digest"]
    cfg1 = load_json("configs.json")["cfg1"]
    assert digest_mat(workloads.cfg1().a) == cfg1["digest_a"]


def test_balanced_cuts():
    w = np.array([5, 0, 0, 5, 10, 0, 20, 1, 1, 1], dtype=np.int64)
    for parts in (1, 2, 3, 4, 8):
        cuts = balanced_cuts(w, parts)
        assert cuts[0] == 0 and cuts[-1] == w.size and len(cuts) == parts + 1
        assert np.all(np.diff(cuts) >= 0)
    cuts = balanced_cuts(w, 2)
    halves = [w[cuts[0]:cuts[1]].sum(), w[cuts[1]:cuts[2]].sum()]
    assert max(halves) <= 0.5 * w.sum() + w.max()
    low = tril_strict(from_triples(4, 4, [(1, 0, 1), (2, 0, 1), (2, 1, 1), (3, 2, 1)]))
    rw = row_work(low.row_ptr, low.col_idx, low.row_ptr, low.row_ptr)
    assert rw.tolist() == [0, 0 + 1, 1 + 2, 2 + 1]


def test_product_path_has_no_oracle_or_cpu_fallback():
    """The package must never import the oracle (it is test infrastructure)."""
    pkg = os.path.join(ROOT, "paper_2111_09947_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(RuntimeError):
        _lib.load(str(tmp_path / "nope.so"))
