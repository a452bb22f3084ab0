"""Run one BASELINE config's multiply (for ncu launch lists); prints bins."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2111_09947_b200 import MultiplyPlan, workloads, _lib
from paper_2111_09947_b200.device import DeviceCsr
from paper_2111_09947_b200.multiply import _handle, multiply_device
name = sys.argv[1]; algo = sys.argv[2] if len(sys.argv) > 2 else "auto"; reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
w = {"cfg1": workloads.cfg1, "cfg2": workloads.cfg2, "cfg4": workloads.cfg4, "cfg5": workloads.cfg5,
     "cfg3_d1": lambda: workloads.cfg3(1), "cfg3_d4": lambda: workloads.cfg3(4),
     "cfg3_d16": lambda: workloads.cfg3(16), "cfg3_d64": lambda: workloads.cfg3(64)}[name]()
dt = np.dtype(w.semiring.dtype); vals = w.semiring.kernel_id == 0
dm = DeviceCsr.from_host(w.mask, with_values=False)
da = DeviceCsr.from_host(w.a, dtype=dt, with_values=vals)
db = da if w.b is w.a else DeviceCsr.from_host(w.b, dtype=dt, with_values=vals)
bt = db.transpose_storage() if algo == "inner" else None
lib = _lib.load(); h = _handle(0); lib.mm_profile_enable(h, 1)
if os.environ.get("TUNE"):
    prm = [int(x) for x in os.environ["TUNE"].split(":")]
    lib.mm_set_tuning(h, (C.c_int64 * len(prm))(*prm), len(prm))
plan = MultiplyPlan(algorithm=algo, semiring=w.semiring, complemented=w.complemented)
for _ in range(reps):
    c, st = multiply_device(dm, da, db, plan, b_csc=bt)
ms = (C.c_float * 6)(); lib.mm_profile_read(h, ms, 6, None)
rows = (C.c_int64 * 64)(); fl = (C.c_int64 * 64)(); nb = lib.mm_profile_bins(h, rows, fl, 64)
print(name, algo, os.environ.get("TUNE", ""), [round(x, 3) for x in ms], {b: (rows[b], fl[b]) for b in range(nb) if rows[b]})
