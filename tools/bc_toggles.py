"""BC wall time under host-path toggles (diagnosis): direct path on/off,
one-call multiply on/off, per-multiply timing of the BC loop."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2111_09947_b200 import MultiplyPlan, _lib
from paper_2111_09947_b200 import multiply as mul
from paper_2111_09947_b200.graphs import BcConfig, betweenness_centrality
from paper_2111_09947_b200.workloads import GeneratorSpec, simple_graph_direct

g = simple_graph_direct(GeneratorSpec("rmat", 18, 16, seed=0))
src = np.random.default_rng(4).choice(g.nrows, 512, replace=False)
cfg = BcConfig(batch_size=512, sources=[int(x) for x in src])
plan = MultiplyPlan(algorithm="auto")
lib = _lib.load()
h = mul._handle(0)
def tune(direct):
    prm = [0] * 14 + [1 if direct else 0]
    prm[7] = -1; prm[8] = prm[9] = prm[10] = -1; prm[12] = prm[13] = -1
    lib.mm_set_tuning(h, (C.c_int64 * len(prm))(*prm), len(prm))
orig = mul.ONE_CALL_MAX_NNZ
for direct in (True, False):
    for onecall in (True, False):
        tune(direct)
        mul.ONE_CALL_MAX_NNZ = orig if onecall else -1
        betweenness_centrality(g, cfg, plan)
        best = 1e9
        for _ in range(3):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            res = betweenness_centrality(g, cfg, plan)
            torch.cuda.synchronize(); best = min(best, time.perf_counter() - t0)
        print(f"direct={direct} onecall={onecall} wall {best:.3f} s multiply {res.multiply_seconds:.3f} s", flush=True)
