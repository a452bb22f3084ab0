"""A few cfg1 multiplies (for ncu launch lists of the small-problem paths)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2111_09947_b200 import MultiplyPlan, workloads, _lib
from paper_2111_09947_b200.device import DeviceCsr
from paper_2111_09947_b200.multiply import _handle, multiply_device

w = workloads.cfg1()
dt = np.dtype(w.semiring.dtype)
dm = DeviceCsr.from_host(w.mask, with_values=False)
da = DeviceCsr.from_host(w.a, dtype=dt)
if os.environ.get("FUSED") == "0":
    prm = [-1] * 19
    prm[17] = 0
    _lib.load().mm_set_tuning(_handle(0), (C.c_int64 * 19)(*prm), 19)
for algo in ("hash", "auto"):
    plan = MultiplyPlan(algorithm=algo, semiring=w.semiring)
    for _ in range(int(os.environ.get("REPS", 3))):
        c, st = multiply_device(dm, da, da, plan)
torch.cuda.synchronize()
print("nnz", c.nnz)
