"""Rebuild the inputs of tests/golden/bc.json (make_golden.make_bc) without
the reference: graphs from the restated generators, pinned by digest."""

from __future__ import annotations

import numpy as np

from golden_util import digest_mat, load_json, random_csr


def bc_graph(spec):
    from paper_2111_09947_b200.sparse import from_triples, simple_undirected_graph
    from paper_2111_09947_b200.workloads import GeneratorSpec, generate
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
    if kind == "random":
        rng = np.random.default_rng(spec["seed"])
        return simple_undirected_graph(random_csr(rng, spec["n"], spec["n"], spec["degree"]))
    if kind == "rmat":
        return simple_undirected_graph(generate(GeneratorSpec("rmat", spec["scale"], spec["ef"],
                                                              seed=spec["seed"])))
    raise ValueError(kind)


def bc_cases():
    """Yields (spec, graph) with the graph checked against the golden digest."""
    for spec in load_json("bc.json")["cases"]:
        g = bc_graph(spec)
        assert digest_mat(g) == spec["digest_graph"], spec
        yield spec, g


def scores(hexes) -> np.ndarray:
    return np.array([float.fromhex(h) for h in hexes], dtype=np.float64)
