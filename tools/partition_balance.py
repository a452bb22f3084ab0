"""Load balance of the multi-GPU row partition, measured on ONE GPU.

For cfg2 / cfg5 and P in {2, 4, 8}: the P row blocks of bench.py's cuts are
multiplied one after another on one B200 (each block exactly as rank r runs
it: A = M = block, B = the whole matrix), L2 flushed before each, median of
--reps.  Prints per-block ms and max/mean (a load-balance proxy, NOT a
scaling curve) for the flop-balanced cuts and for --rounds of cost refinement
(distributed.refine_cuts), and checks that the blocks concatenate to the
1-GPU C.

    python tools/partition_balance.py [--configs cfg2,cfg5] [--reps 3] [--rounds 3]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

from paper_2111_09947_b200 import MultiplyPlan, workloads
from paper_2111_09947_b200.device import DeviceCsr
from paper_2111_09947_b200.distributed import (balanced_cuts, concat_row_blocks, cut_offsets, imbalance,
                                               refine_cuts, row_blocks, row_work_device)
from paper_2111_09947_b200.multiply import multiply_device


def time_blocks(dl, plan, cuts, reps, flush):
    blocks = row_blocks(dl, cuts, cut_offsets(dl, cuts))
    ms = []
    parts = []
    for blk in blocks:
        ts = []
        for r in range(reps + 1):
            flush.fill_(r & 0xFF)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            c, _ = multiply_device(blk, blk, dl, plan)
            e1.record()
            e1.synchronize()
            if r:
                ts.append(e0.elapsed_time(e1))
        ms.append(float(np.median(ts)))
        parts.append(c)
    return ms, concat_row_blocks(parts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="cfg2,cfg5")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    out = []
    for name in args.configs.split(","):
        w = workloads.cfg2() if name == "cfg2" else workloads.cfg5()
        dl = DeviceCsr.from_host(w.a, with_values=False)
        plan = MultiplyPlan(algorithm="auto", semiring=w.semiring)
        one, full = time_blocks(dl, plan, [0, dl.nrows], args.reps, flush)
        work = row_work_device(dl, dl, dl).cpu().numpy()
        rec0 = {"config": name, "parts": 1, "block_ms": one}
        print(json.dumps(rec0), flush=True)
        out.append(rec0)
        for parts in (2, 4, 8):
            cuts = balanced_cuts(work, parts)
            for rnd in range(args.rounds + 1):
                ms, cc = time_blocks(dl, plan, cuts, args.reps, flush)
                same = (torch.equal(cc.ptr, full.ptr) and torch.equal(cc.idx, full.idx)
                        and torch.equal(cc.values, full.values))
                rec = {"config": name, "parts": parts, "refine_round": rnd, "cuts": [int(x) for x in cuts],
                       "block_ms": ms, "max_ms": max(ms), "mean_ms": float(np.mean(ms)),
                       "imbalance_max_over_mean": imbalance(ms),
                       "ideal_speedup": one[0] / max(ms), "sum_block_ms_over_1gpu": sum(ms) / one[0],
                       "bitwise_equal_to_1gpu": bool(same)}
                print(json.dumps(rec), flush=True)
                out.append(rec)
                assert same
                cuts = refine_cuts(work, cuts, ms, parts)
        del dl, full
        torch.cuda.empty_cache()
    if args.out:
        with open(args.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
