"""Full batched betweenness centrality (graphs.py:136-200) on the device vs the
CPU oracle restatement (oracle/bc.py), on cfg4's graph and sources: R-MAT
scale 18 edge factor 16 (simple undirected), 512 sources drawn with
default_rng(4).choice (workloads.cfg4), one batch of 512.  Prints one JSON line."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2111_09947_b200 import MultiplyPlan
from paper_2111_09947_b200.graphs import BcConfig, betweenness_centrality
from paper_2111_09947_b200.workloads import GeneratorSpec, simple_graph_direct

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=18)
ap.add_argument("--sources", type=int, default=512)
ap.add_argument("--batch", type=int, default=512)
ap.add_argument("--algo", default="auto")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--cpu", action="store_true")
args = ap.parse_args()
g = simple_graph_direct(GeneratorSpec("rmat", args.scale, 16, seed=0))
src = np.random.default_rng(4).choice(g.nrows, args.sources, replace=False)
cfg = BcConfig(batch_size=args.batch, sources=[int(x) for x in src])
plan = MultiplyPlan(algorithm=args.algo)
betweenness_centrality(g, cfg, plan)          # warm-up (pool, caches)
best = None
for _ in range(args.reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = betweenness_centrality(g, cfg, plan)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    best = dt if best is None else min(best, dt)
out = {"workload": f"BC R-MAT s{args.scale} ef16, {args.sources} sources, batch {args.batch}",
       "algorithm": args.algo, "gpu_seconds_wall": best, "multiply_seconds": res.multiply_seconds,
       "multiplies": res.multiplies, "generated_flops": res.flops, "useful_products": res.evaluated,
       "useful_gprod_per_s": res.evaluated / best / 1e9, "score_sum": float(res.value.sum())}
if args.cpu:
    import oracle
    from oracle.bc import betweenness_centrality as obc
    t0 = time.perf_counter()
    sc, cnt, fl, ev = obc(g, args.batch, [int(x) for x in src], algorithm="msa")
    out["cpu_seconds"] = time.perf_counter() - t0
    out["cpu_threads"] = oracle.max_threads()
    out["bitwise_equal_to_oracle"] = bool(np.array_equal(sc.view(np.int64), res.value.view(np.int64)))
    out["counters_equal"] = (cnt, fl, ev) == (res.multiplies, res.flops, res.evaluated)
print(json.dumps(out), flush=True)
