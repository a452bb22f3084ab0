"""Threaded parity fuzz: T host threads, each with its own handle (multiply.py keeps one
per device and thread) and its own random stream, multiply small random problems at the
same time — every plan x 1P/2P x plain/complement x int64 / plus-pair / float64 — and check
each result against the C oracle.  ctypes drops the GIL inside the library, so the
launches, the workspace pools and the process-wide shared-memory-limit record really run
concurrently.  Prints the first mismatch / exception and exits 1."""
import argparse, os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
from paper_2111_09947_b200 import (MultiplyPlan, arithmetic_semiring, from_arrays, masked_multiply_with_stats,
                                   plus_pair_semiring)

ap = argparse.ArgumentParser()
ap.add_argument("--seconds", type=float, default=120)
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--threads", type=int, default=4)
args = ap.parse_args()


def rand_matrix(rng, rows, cols, avg, hub_frac, hub_len, dtype, empty_frac):
    lens = rng.poisson(avg, rows)
    lens[rng.random(rows) < empty_frac] = 0
    hubs = rng.random(rows) < hub_frac
    lens[hubs] = rng.integers(hub_len // 2 + 1, hub_len + 1, hubs.sum())
    lens = np.minimum(lens, cols)
    r = np.repeat(np.arange(rows), lens)
    c = np.concatenate([rng.choice(cols, ln, replace=False) for ln in lens]) if lens.sum() else np.empty(0, np.int64)
    v = rng.integers(-3, 4, r.size).astype(np.int64) if dtype == np.int64 else rng.standard_normal(r.size)
    if dtype == np.int64:
        v[v == 0] = 1
    return from_arrays(rows, cols, r, c, v)


failures = []
counts = [0] * args.threads
t_end = time.time() + args.seconds


def worker(tid):
    rng = np.random.default_rng([args.seed, tid])
    try:
        while time.time() < t_end and not failures:
            m = int(rng.choice([1, 7, 100, 1000, 4000]))
            k = int(rng.choice([1, 50, 1000]))
            n = int(rng.choice([1, 64, 3000, 40000, 300000]))
            kind = rng.choice(["i64", "pair", "f64"])
            dt = np.float64 if kind == "f64" else np.int64
            sem = plus_pair_semiring(np.int64) if kind == "pair" else arithmetic_semiring(dt)
            a = rand_matrix(rng, m, k, rng.choice([1, 4, 20]), rng.choice([0, 0.01]), min(k, int(rng.choice([50, 800]))), dt, 0.1)
            b = rand_matrix(rng, k, n, rng.choice([1, 8, 40]), rng.choice([0, 0.02]), min(n, int(rng.choice([200, 8000]))), dt, 0.1)
            mk = rand_matrix(rng, m, n, rng.choice([1, 6, 60]), rng.choice([0, 0.01]),
                             min(n, int(rng.choice([300, 9000, 30000]))), np.int64, 0.2).pattern()
            comp = bool(rng.random() < 0.35) and n <= 40000
            ref = oracle.masked_multiply(mk, a, b, algorithm="msa", complemented=comp, dtype=dt,
                                         semiring_id=sem.kernel_id, workers=2)
            algos = ["auto", "hash", "msa", "heap"] + ([] if comp else ["mca", "inner"])
            for algo in algos:
                for phases in ("1p", "2p"):
                    if rng.random() < 0.5 and algo != "auto":
                        continue
                    plan = MultiplyPlan(algorithm=algo, phases=phases, complemented=comp, semiring=sem)
                    c, st = masked_multiply_with_stats(mk, a, b, plan)
                    ok = (np.array_equal(c.row_ptr, ref.row_ptr) and np.array_equal(c.col_idx[: c.nnz], ref.col_idx)
                          and st.generated_flops == ref.generated_flops)
                    if ok:
                        if kind == "f64" and algo == "heap":
                            ok = np.allclose(c.values[: c.nnz], ref.values, rtol=1e-12, atol=0)
                        else:
                            ok = np.array_equal(c.values[: c.nnz], ref.values)
                    counts[tid] += 1
                    if not ok:
                        failures.append(("MISMATCH", tid, dict(m=m, k=k, n=n, kind=str(kind), comp=comp, algo=algo,
                                                               phases=phases, seed=args.seed)))
                        return
    except BaseException as e:   # noqa: BLE001
        failures.append(("EXCEPTION", tid, repr(e)[:300]))


ths = [threading.Thread(target=worker, args=(t,)) for t in range(args.threads)]
for t in ths:
    t.start()
for t in ths:
    t.join()
if failures:
    print(failures[0], flush=True)
    sys.exit(1)
print(f"threaded fuzz ok: {args.threads} threads, {sum(counts)} multiplies {counts}, seed {args.seed}")
