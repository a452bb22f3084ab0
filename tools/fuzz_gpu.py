"""Randomised parity fuzz of the GPU path against the C oracle: random shapes, skewed
rows (hubs in A, B and the mask), empty rows, every plan x 1P/2P x plain/complement x
int64 / plus-pair / float64, for a time budget.  Prints the first mismatch and exits 1."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
from paper_2111_09947_b200 import (MultiplyPlan, arithmetic_semiring, from_arrays, masked_multiply_with_stats,
                                   plus_pair_semiring)

ap = argparse.ArgumentParser()
ap.add_argument("--seconds", type=float, default=300)
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--only-case", type=int, default=-1, help="replay one case of the seed's stream (same random draws)")
ap.add_argument("--from-case", type=int, default=-1, help="with --only-case N: run cases from-case..N")
args = ap.parse_args()
rng = np.random.default_rng(args.seed)


def rand_matrix(rows, cols, avg, hub_frac, hub_len, dtype, empty_frac):
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


t_end = time.time() + args.seconds
cases = checks = 0
while time.time() < t_end:
    m = int(rng.choice([1, 7, 100, 1000, 5000, 20000]))
    k = int(rng.choice([1, 50, 1000, 8000]))
    n = int(rng.choice([1, 64, 3000, 40000, 300000]))
    kind = rng.choice(["i64", "pair", "f64"])
    dt = np.float64 if kind == "f64" else np.int64
    sem = plus_pair_semiring(np.int64) if kind == "pair" else arithmetic_semiring(dt)
    a = rand_matrix(m, k, rng.choice([1, 4, 20]), rng.choice([0, 0.01]), min(k, int(rng.choice([50, 3000]))), dt, 0.1)
    b = rand_matrix(k, n, rng.choice([1, 8, 40]), rng.choice([0, 0.02]), min(n, int(rng.choice([200, 20000]))), dt, 0.1)
    mk = rand_matrix(m, n, rng.choice([1, 6, 60]), rng.choice([0, 0.01]), min(n, int(rng.choice([300, 9000, 30000]))),
                     np.int64, 0.2).pattern()
    comp = bool(rng.random() < 0.35) and n <= 40000
    replay_skip = args.only_case >= 0 and not ((args.from_case if args.from_case >= 0 else args.only_case) <= cases <= args.only_case)
    ref = None if replay_skip else oracle.masked_multiply(mk, a, b, algorithm="msa", complemented=comp, dtype=dt,
                                                          semiring_id=sem.kernel_id, workers=8)
    algos = ["auto", "hash", "msa", "heap", "heapdot"] + ([] if comp else ["mca", "inner"])
    for algo in algos:
        for phases in ("1p", "2p"):
            if rng.random() < 0.5 and algo != "auto":
                continue
            if replay_skip:
                continue
            plan = MultiplyPlan(algorithm=algo, phases=phases, complemented=comp, semiring=sem)
            print("run", cases, algo, phases, kind, comp, (m, k, n), flush=True) if args.only_case >= 0 else None
            try:
                c, st = masked_multiply_with_stats(mk, a, b, plan)
            except Exception as e:
                print("EXCEPTION", repr(e)[:200], dict(m=m, k=k, n=n, kind=kind, comp=comp, algo=algo, phases=phases,
                                                       case=cases, seed=args.seed, nnz=(a.nnz, b.nnz, mk.nnz),
                                                       max_mask_row=int(np.diff(mk.row_ptr).max()),
                                                       max_a_row=int(np.diff(a.row_ptr).max()),
                                                       max_b_row=int(np.diff(b.row_ptr).max())), flush=True)
                sys.exit(1)
            ok = (np.array_equal(c.row_ptr, ref.row_ptr) and np.array_equal(c.col_idx[: c.nnz], ref.col_idx)
                  and st.generated_flops == ref.generated_flops)
            if ok:
                if kind == "f64" and algo in ("heap", "heapdot"):
                    ok = np.allclose(c.values[: c.nnz], ref.values, rtol=1e-12, atol=0)
                else:
                    ok = np.array_equal(c.values[: c.nnz], ref.values)
            if ok and algo not in ("heap", "heapdot", "inner"):
                ok = st.evaluated_multiplies == ref.evaluated_multiplies
            checks += 1
            if not ok:
                print("MISMATCH", dict(m=m, k=k, n=n, kind=kind, comp=comp, algo=algo, phases=phases, case=cases,
                                       seed=args.seed, nnz=(a.nnz, b.nnz, mk.nnz), got_nnz=c.nnz, ref_nnz=int(ref.row_ptr[-1]),
                                       ev=(st.evaluated_multiplies, ref.evaluated_multiplies),
                                       gen=(st.generated_flops, ref.generated_flops)), flush=True)
                sys.exit(1)
    if not comp and not replay_skip and rng.random() < 0.3:
        # auto with B^T present: the per-row push / pull model on the device
        from paper_2111_09947_b200.device import DeviceCsr
        from paper_2111_09947_b200.multiply import multiply_device
        vals = sem.kernel_id == 0
        dm = DeviceCsr.from_host(mk, with_values=False)
        da = DeviceCsr.from_host(a, dtype=dt, with_values=vals)
        db = DeviceCsr.from_host(b, dtype=dt, with_values=vals)
        for phases in ("1p", "2p"):
            plan = MultiplyPlan(algorithm="auto", phases=phases, semiring=sem)
            try:
                cd, st = multiply_device(dm, da, db, plan, b_csc=db.transpose_storage())
                c = cd.to_host()
            except Exception as e:
                print("EXCEPTION(bt)", repr(e)[:200], dict(m=m, k=k, n=n, kind=kind, phases=phases, case=cases,
                                                           seed=args.seed), flush=True)
                sys.exit(1)
            ok = (np.array_equal(c.row_ptr, ref.row_ptr) and np.array_equal(c.col_idx[: c.nnz], ref.col_idx)
                  and np.array_equal(np.asarray(c.values[: c.nnz]).astype(dt), ref.values)
                  and st.generated_flops == ref.generated_flops)
            checks += 1
            if not ok:
                print("MISMATCH(bt)", dict(m=m, k=k, n=n, kind=kind, phases=phases, case=cases, seed=args.seed,
                                           got_nnz=c.nnz, ref_nnz=int(ref.row_ptr[-1])), flush=True)
                sys.exit(1)
    cases += 1
    if args.only_case >= 0 and cases > args.only_case:
        break
print("fuzz ok:", cases, "problems,", checks, "multiplies, seed", args.seed)
