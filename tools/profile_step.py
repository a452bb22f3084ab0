"""Run the cfg2 masked multiply a few times (for ncu / compute-sanitizer captures)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2111_09947_b200 import MultiplyPlan, plus_pair_semiring, workloads
from paper_2111_09947_b200.device import DeviceCsr
from paper_2111_09947_b200.multiply import multiply_device, reduce_sum

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=20)
ap.add_argument("--algo", default="auto")
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()
low = workloads.triangle_lower(args.scale)
dl = DeviceCsr.from_host(low, with_values=False)
bt = dl.transpose_storage() if args.algo == "inner" else None
plan = MultiplyPlan(algorithm=args.algo, semiring=plus_pair_semiring(np.int64))
for _ in range(args.reps):
    c, st = multiply_device(dl, dl, dl, plan, b_csc=bt)
    tri = int(reduce_sum(c.values).item())
torch.cuda.synchronize()
print("triangles", tri, "rows push/pull/empty", st.rows_push, st.rows_pull, st.rows_empty)
