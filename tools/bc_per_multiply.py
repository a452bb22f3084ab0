"""Per-multiply device time inside batched BC (diagnosis), direct path on/off."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2111_09947_b200 import MultiplyPlan, _lib
from paper_2111_09947_b200 import multiply as mul
from paper_2111_09947_b200 import graphs
from paper_2111_09947_b200.graphs import BcConfig, betweenness_centrality
from paper_2111_09947_b200.workloads import GeneratorSpec, simple_graph_direct

g = simple_graph_direct(GeneratorSpec("rmat", 18, 16, seed=0))
src = np.random.default_rng(4).choice(g.nrows, 512, replace=False)
cfg = BcConfig(batch_size=512, sources=[int(x) for x in src])
plan = MultiplyPlan(algorithm="auto")
lib = _lib.load()
h = mul._handle(0)
orig = mul.multiply_device
log = []
def timed(mask, a, b, plan, complemented=None, b_csc=None, stream=None):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    c, st = orig(mask, a, b, plan, complemented=complemented, b_csc=b_csc, stream=stream)
    torch.cuda.synchronize()
    log.append((time.perf_counter() - t0, mask.nrows, mask.nnz, a.nnz, b.nnz, bool(plan.complemented or complemented),
                str(plan.semiring.dtype), mul.last_kernel_rows()))
    return c, st
graphs.multiply_device = timed
for direct in (True, False):
    prm = [0] * 14 + [1 if direct else 0]
    prm[7] = -1; prm[8] = prm[9] = prm[10] = -1; prm[12] = prm[13] = -1
    lib.mm_set_tuning(h, (C.c_int64 * len(prm))(*prm), len(prm))
    betweenness_centrality(g, cfg, plan)
    log.clear()
    betweenness_centrality(g, cfg, plan)
    print("direct", direct)
    for r in log:
        print(f"  {r[0]*1e3:8.3f} ms rows {r[1]} nnzM {r[2]} nnzA {r[3]} nnzB {r[4]} comp {r[5]} {r[6]} {r[7]}")
