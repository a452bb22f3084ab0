"""Time every algorithm on cfg2 (numeric phase / whole multiply, L2 flushed)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2111_09947_b200 import MultiplyPlan, plus_pair_semiring, workloads, _lib
from paper_2111_09947_b200.device import DeviceCsr
from paper_2111_09947_b200.multiply import _handle, multiply_device, reduce_sum

low = workloads.triangle_lower(int(os.environ.get("SCALE", "20")))
dl = DeviceCsr.from_host(low, with_values=False)
bt = dl.transpose_storage()
lib = _lib.load()
h = _handle(0)
lib.mm_profile_enable(h, 1)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
algos = os.environ.get("ALGOS", "hash,msa,mca,auto,auto+pull").split(",")
tunings = [[int(x) for x in t.split(":")] for t in os.environ.get("TUNINGS", "").split(",") if t]
for tune in tunings or [None]:
    if tune:
        prm = (C.c_int64 * len(tune))(*tune)
        lib.mm_set_tuning(h, prm, len(tune))
    for algo in algos:
        use_bt = algo in ("inner", "auto+pull")
        plan = MultiplyPlan(algorithm=algo.replace("+pull", ""), semiring=plus_pair_semiring(np.int64))
        ms = (C.c_float * 6)()
        best_n, best_t = 1e9, 1e9
        for rep in range(4):
            flush.fill_(rep)
            c, st = multiply_device(dl, dl, dl, plan, b_csc=bt if use_bt else None)
            lib.mm_profile_read(h, ms, 6, None)
            if rep:
                best_n, best_t = min(best_n, ms[2]), min(best_t, ms[5])
        tri = int(reduce_sum(c.values).item())
        nb = 42
        rows = (C.c_int64 * nb)()
        fl = (C.c_int64 * nb)()
        lib.mm_profile_bins(h, rows, fl, nb)
        bins = {b: (rows[b], fl[b]) for b in range(nb) if rows[b]}
        print(tune, algo, f"numeric {best_n:.3f} ms total {best_t:.3f} ms tri={tri}", bins, flush=True)
