"""Fixed per-multiply overhead on a tiny problem (cfg1): phase split + host time."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2111_09947_b200 import MultiplyPlan, workloads, _lib
from paper_2111_09947_b200.device import DeviceCsr
from paper_2111_09947_b200.multiply import _handle, multiply_device
for name, w in (("cfg1", workloads.cfg1()), ("cfg4", workloads.cfg4())):
    dt = np.dtype(w.semiring.dtype)
    dm = DeviceCsr.from_host(w.mask, with_values=False)
    da = DeviceCsr.from_host(w.a, dtype=dt)
    db = DeviceCsr.from_host(w.b, dtype=dt)
    lib = _lib.load(); h = _handle(0); lib.mm_profile_enable(h, 1)
    for algo in ("hash", "msa", "heap"):
        plan = MultiplyPlan(algorithm=algo, semiring=w.semiring, complemented=w.complemented)
        ms = (C.c_float * 6)(); L = C.c_int64()
        for rep in range(6):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            c, st = multiply_device(dm, da, db, plan)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            lib.mm_profile_read(h, ms, 6, C.byref(L))
        print(name, algo, f"host {1e3*(t1-t0):.3f} ms", "phases", [round(x, 3) for x in ms], "launches", L.value, flush=True)
