"""Full k-truss (graphs.py:99-118) on the device: support
multiply G (.) (G G) under plus-pair, prune support < k-2 with mm_filter_min,
repeat to the fixed point; cfg5's graph (R-MAT scale 22, edge factor 16,
simple undirected) by default, k = 5 (the reference CLI default, cli.py:341).
With --cpu the same fixed point is computed by the C oracle restatement
(multithreaded) and compared edge for edge.  Prints one JSON line."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2111_09947_b200 import MultiplyPlan
from paper_2111_09947_b200.graphs import k_truss
from paper_2111_09947_b200.workloads import GeneratorSpec, simple_graph_direct

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=22)
ap.add_argument("--k", type=int, default=5)
ap.add_argument("--algo", default="auto")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--cpu", action="store_true")
args = ap.parse_args()
t0 = time.perf_counter()
g = simple_graph_direct(GeneratorSpec("rmat", args.scale, 16, seed=0))
gen_s = time.perf_counter() - t0
plan = MultiplyPlan(algorithm=args.algo)
k_truss(g, args.k, plan)                      # warm-up (pool, caches)
best = None
for _ in range(args.reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = k_truss(g, args.k, plan)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    best = dt if best is None else min(best, dt)
out = {"workload": f"k-truss k={args.k} R-MAT s{args.scale} ef16 (simple undirected, nnz {g.nnz})",
       "algorithm": args.algo, "gpu_seconds_wall": best, "multiply_seconds": res.multiply_seconds,
       "iterations": res.multiplies, "generated_flops": res.flops, "useful_products": res.evaluated,
       "useful_gprod_per_s": res.evaluated / best / 1e9, "truss_edges_directed": int(res.value.nnz),
       "per_multiply_ms": [round(s * 1e3, 3) for s, _ in res.per_multiply], "input_gen_s": gen_s}
if args.cpu:
    import oracle
    from paper_2111_09947_b200.sparse import from_arrays
    t0 = time.perf_counter()
    cur, iters = g, 0
    while cur.nnz:
        r = oracle.masked_multiply(cur.pattern(), cur, cur, semiring_id=1, workers=oracle.max_threads())
        iters += 1
        keep = r.values >= args.k - 2
        if int(keep.sum()) == cur.nnz:
            break
        rows = np.repeat(np.arange(cur.nrows), np.diff(r.row_ptr))
        cur = from_arrays(cur.nrows, cur.ncols, rows[keep], r.col_idx[keep],
                          np.ones(int(keep.sum()), dtype=np.int64))
    out["cpu_seconds"] = time.perf_counter() - t0
    out["cpu_threads"] = oracle.max_threads()
    out["cpu_iterations"] = iters
    out["equal_to_oracle"] = bool(np.array_equal(cur.row_ptr, res.value.row_ptr)
                                  and np.array_equal(cur.col_idx[: cur.nnz], res.value.col_idx[: res.value.nnz]))
print(json.dumps(out), flush=True)
