"""Matrix Market ingestion: the native reader against the
reference's Python reader (pkg/src/maskmul/mmio.py:27-101) on one seeded
file.  Host reader timed with 1 and all threads; with a GPU, the device reader
(canonicalised by mm_csr_from_coo) too; the reference reader only where
/root/reference exists (the build container).  Prints one JSON line.

    python tools/bench_mmio.py [--nnz 2000000] [--field real|integer|pattern] [--symmetric]
"""
import argparse, json, os, sys, tempfile, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
from paper_2111_09947_b200.mmio import read_matrix_market, read_matrix_market_device, write_matrix_market
from paper_2111_09947_b200.sparse import from_arrays

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 18)
ap.add_argument("--nnz", type=int, default=2_000_000)
ap.add_argument("--field", default="real")
args = ap.parse_args()
rng = np.random.default_rng(1)
vals = rng.random(args.nnz) if args.field == "real" else rng.integers(-9, 10, args.nnz)
a = from_arrays(args.n, args.n, rng.integers(0, args.n, args.nnz), rng.integers(0, args.n, args.nnz), vals)
if args.field == "pattern":
    a.values[:] = 1
path = os.path.join(tempfile.mkdtemp(), "bench.mtx")
write_matrix_market(path, a, field=args.field)
out = {"file_bytes": os.path.getsize(path), "entries": int(a.nnz), "field": args.field,
       "host_cores": len(os.sched_getaffinity(0))}


def best(fn, reps=3):
    t = []
    for _ in range(reps):
        t0 = time.perf_counter()
        r = fn()
        t.append(time.perf_counter() - t0)
    return min(t), r


out["native_1thread_s"], m = best(lambda: read_matrix_market(path, threads=1))
out["native_all_threads_s"], m = best(lambda: read_matrix_market(path))
assert m.equals(a)
try:
    import torch
    if torch.cuda.is_available():
        read_matrix_market_device(path)
        torch.cuda.synchronize()
        out["native_device_s"], d = best(lambda: (read_matrix_market_device(path), torch.cuda.synchronize())[0])
        h = d.to_host()
        out["device_equal"] = bool(np.array_equal(h.row_ptr, a.row_ptr) and np.array_equal(h.col_idx, a.col_idx[: a.nnz]))
except ImportError:
    pass
if os.path.isdir("/root/reference/pkg/src"):
    sys.path.insert(0, "/root/reference/pkg/src")
    sys.dont_write_bytecode = True
    from maskmul.mmio import read_matrix_market as ref_read
    out["reference_s"], r = best(lambda: ref_read(path), reps=1)
    out["reference_equal"] = bool(np.array_equal(r.values, m.values) and np.array_equal(r.col_idx, m.col_idx))
print(json.dumps(out), flush=True)
