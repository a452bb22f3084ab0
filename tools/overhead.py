"""Fixed per-multiply overhead on small problems: phase split (device events),
host wall time and launches per multiply."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2111_09947_b200 import MultiplyPlan, workloads, _lib
from paper_2111_09947_b200.device import DeviceCsr
from paper_2111_09947_b200.multiply import _handle, multiply_device

PH = ("analyze+sync", "scatter", "bins", "scan+sync", "compact", "total")
cases = [("cfg1", workloads.cfg1(), ("msa", "hash", "auto")),
         ("cfg4", workloads.cfg4(), ("auto", "hash")),
         ("cfg3_d1", workloads.cfg3(1), ("auto", "inner"))]
lib = _lib.load(); h = _handle(0); lib.mm_profile_enable(h, 1)
for name, w, algos in cases:
    dt = np.dtype(w.semiring.dtype)
    dm = DeviceCsr.from_host(w.mask, with_values=False)
    da = DeviceCsr.from_host(w.a, dtype=dt)
    db = DeviceCsr.from_host(w.b, dtype=dt)
    bt = db.transpose_storage()
    for algo in algos:
        plan = MultiplyPlan(algorithm=algo, semiring=w.semiring, complemented=w.complemented)
        ms = (C.c_float * 6)(); L = C.c_int64()
        host = []
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dev_ms = []
        for rep in range(20):
            torch.cuda.synchronize()
            t0 = time.perf_counter(); ev0.record()
            c, st = multiply_device(dm, da, db, plan, b_csc=bt if algo in ("auto", "inner") else None)
            ev1.record(); torch.cuda.synchronize()
            host.append(time.perf_counter() - t0)
            dev_ms.append(ev0.elapsed_time(ev1))
            lib.mm_profile_read(h, ms, 6, C.byref(L))
        print(f"{name:8s} {algo:6s} host_med {1e3*np.median(host):.3f} ms  events_med {np.median(dev_ms):.3f} ms  "
              + " ".join(f"{k}={v:.3f}" for k, v in zip(PH, ms)) + f"  launches {L.value}", flush=True)
