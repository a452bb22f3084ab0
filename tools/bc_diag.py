"""Per-multiply breakdown of the BC benchmark (which bins / kernels are slow)."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2111_09947_b200 import MultiplyPlan, _lib
from paper_2111_09947_b200.graphs import BcConfig, betweenness_centrality
from paper_2111_09947_b200.multiply import _handle
from paper_2111_09947_b200.workloads import GeneratorSpec, simple_graph_direct
import paper_2111_09947_b200.graphs as G

algo = sys.argv[1] if len(sys.argv) > 1 else "auto"
g = simple_graph_direct(GeneratorSpec("rmat", 18, 16, seed=0))
src = np.random.default_rng(4).choice(g.nrows, 512, replace=False)
cfg = BcConfig(batch_size=512, sources=[int(x) for x in src])
lib = _lib.load(); h = _handle(0); lib.mm_profile_enable(h, 1)
orig = G.multiply_device
def wrapped(*a, **k):
    c, st = orig(*a, **k)
    ms = (C.c_float * 6)(); L = C.c_int64()
    lib.mm_profile_read(h, ms, 6, C.byref(L))
    rows = (C.c_int64 * 64)(); fl = (C.c_int64 * 64)()
    nb = lib.mm_profile_bins(h, rows, fl, 64)
    bins = {b: (rows[b], fl[b]) for b in range(nb) if rows[b]}
    print(f"comp={k.get('complemented', False)} nnzC={c.nnz} gen={st.generated_flops} eval={st.evaluated_multiplies} "
          f"ms={[round(x,3) for x in ms]} bins={bins}", flush=True)
    return c, st
G.multiply_device = wrapped
betweenness_centrality(g, cfg, MultiplyPlan(algorithm=algo))
