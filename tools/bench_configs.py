"""All five BASELINE configs on one B200: GPU time per algorithm, roofline
fraction (SURVEY.md §8(d) byte model) and the CPU oracle beside it.

    python tools/bench_configs.py [--cpu] [--configs cfg1,cfg2,...]

Prints one JSON object per (config, algorithm) line; --out writes them all.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

from paper_2111_09947_b200 import MultiplyPlan, workloads
from paper_2111_09947_b200.device import DeviceCsr
from paper_2111_09947_b200.multiply import multiply_device

PEAK = 6455.9
try:
    PEAK = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:
    pass


def bytes_alg(w, flops, nnz_c):
    """min(push, pull) (push only when complemented)."""
    v = 0 if w.semiring.kernel_id == 1 else 8
    m = w.a.nrows
    push = (8 * (m + 1) + w.a.nnz * (4 + v) + 16 * w.a.nnz + flops * (4 + v)
            + 8 * (m + 1) + 4 * w.mask.nnz + 8 * (m + 1) + 12 * nnz_c)
    if w.complemented:
        return push, "push"
    a_len = np.diff(w.a.row_ptr)
    b_csc_len = np.bincount(np.asarray(w.b.col_idx[: w.b.nnz]), minlength=w.b.ncols)
    rows = np.repeat(np.arange(m), np.diff(w.mask.row_ptr))
    cross = int((a_len[rows] + b_csc_len[np.asarray(w.mask.col_idx[: w.mask.nnz])]).sum())
    pull = (8 * (m + 1) + 4 * w.mask.nnz + 16 * w.mask.nnz + cross * (4 + v)
            + 8 * (m + 1) + 12 * nnz_c)
    return (push, "push") if push <= pull else (pull, "pull")


def time_gpu(w, algo, reps=5):
    dt = np.dtype(w.semiring.dtype)
    vals = w.semiring.kernel_id == 0
    dm = DeviceCsr.from_host(w.mask, with_values=False)
    da = DeviceCsr.from_host(w.a, dtype=dt, with_values=vals)
    db = DeviceCsr.from_host(w.b, dtype=dt, with_values=vals)
    bt = db.transpose_storage() if algo in ("inner", "auto+pull") else None
    plan = MultiplyPlan(algorithm=algo.replace("+pull", ""), complemented=w.complemented, semiring=w.semiring)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    times = []
    for r in range(reps + 2):
        flush.fill_(r)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        c, st = multiply_device(dm, da, db, plan, b_csc=bt)
        e1.record()
        e1.synchronize()
        if r >= 2:
            times.append(e0.elapsed_time(e1))
    return min(times), float(np.median(times)), st, c.nnz


def time_cpu(w, algo):
    import oracle
    r = oracle.masked_multiply(w.mask, w.a, w.b, algorithm=algo, complemented=w.complemented,
                               semiring_id=w.semiring.kernel_id, dtype=w.semiring.dtype,
                               workers=oracle.max_threads())
    best = r.total_seconds
    if best < 5:
        for _ in range(2):
            r = oracle.masked_multiply(w.mask, w.a, w.b, algorithm=algo, complemented=w.complemented,
                                       semiring_id=w.semiring.kernel_id, dtype=w.semiring.dtype,
                                       workers=oracle.max_threads())
            best = min(best, r.total_seconds)
    return best, oracle.max_threads()


CONFIGS = {
    "cfg1": (workloads.cfg1, ["auto", "msa", "hash", "mca", "inner", "heap"], "msa"),
    "cfg2": (workloads.cfg2, ["auto", "msa", "hash", "mca", "heap"], "msa"),
    "cfg3_d1": (lambda: workloads.cfg3(1), ["auto", "auto+pull", "inner", "msa", "hash", "mca"], "inner"),
    "cfg3_d4": (lambda: workloads.cfg3(4), ["auto", "auto+pull", "inner", "msa", "hash", "mca"], "inner"),
    "cfg3_d16": (lambda: workloads.cfg3(16), ["auto", "auto+pull", "inner", "msa", "hash", "mca"], "msa"),
    "cfg3_d64": (lambda: workloads.cfg3(64), ["auto", "auto+pull", "inner", "msa", "hash", "mca"], "msa"),
    "cfg4": (workloads.cfg4, ["auto", "hash", "heap", "msa"], "heap"),
    "cfg5": (workloads.cfg5, ["auto", "hash"], None),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default=",".join(CONFIGS))
    ap.add_argument("--cpu", action="store_true")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    lines = []
    for name in args.configs.split(","):
        make, algos, cpu_algo = CONFIGS[name]
        t0 = time.perf_counter()
        w = make()
        gen = time.perf_counter() - t0
        for algo in algos:
            t_min, t_med, st, nnz_c = time_gpu(w, algo)
            b, model = bytes_alg(w, st.generated_flops, nnz_c)
            line = {"config": name, "algorithm": algo, "gpu_ms_min": t_min, "gpu_ms_median": t_med,
                    "generated_flops": st.generated_flops, "useful_products": st.evaluated_multiplies,
                    "nnz_c": nnz_c, "useful_gflops": st.evaluated_multiplies / t_min / 1e6,
                    "bytes_alg": b, "bytes_model": model,
                    "roofline_frac_measured_peak": b / (t_min * 1e-3) / 1e9 / PEAK,
                    "rows_push": st.rows_push, "rows_pull": st.rows_pull, "input_gen_s": gen}
            print(json.dumps(line), flush=True)
            lines.append(line)
        if args.cpu and cpu_algo:
            t_cpu, cores = time_cpu(w, cpu_algo)
            line = {"config": name, "cpu_oracle_algorithm": cpu_algo, "cpu_seconds": t_cpu, "cores": cores}
            print(json.dumps(line), flush=True)
            lines.append(line)
        del w
    if args.out:
        with open(args.out, "w") as f:
            json.dump(lines, f, indent=1)


if __name__ == "__main__":
    main()
