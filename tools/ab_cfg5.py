"""cfg5 (k-truss support, R-MAT s22) with the library at MM_LIB_PATH: min multiply
time over reps, and the output checked against the reference golden
(tests/golden/configs.json: digest, nnz, evaluated).  One JSON line."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import ctypes as C
import numpy as np, torch
from golden_util import digest_csr
from paper_2111_09947_b200 import MultiplyPlan, workloads
from paper_2111_09947_b200.device import DeviceCsr
from paper_2111_09947_b200.multiply import multiply_device
scale = int(os.environ.get("SCALE", "22")); reps = int(os.environ.get("REPS", "3"))
w = workloads.cfg5(scale)
da = DeviceCsr.from_host(w.a, with_values=False)
if os.environ.get("TUNE"):   # mm_set_tuning params, ':'-separated (-1 = keep)
    from paper_2111_09947_b200 import _lib
    from paper_2111_09947_b200.multiply import _handle
    prm = [int(x) for x in os.environ["TUNE"].split(":")]
    _lib.load().mm_set_tuning(_handle(0), (C.c_int64 * len(prm))(*prm), len(prm))
plan = MultiplyPlan(algorithm=os.environ.get("ALGO", "auto"), semiring=w.semiring)
ts = []
for _ in range(reps + 1):
    torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); c, st = multiply_device(da, da, da, plan); e1.record(); e1.synchronize()
    ts.append(e0.elapsed_time(e1))
out = {"lib": os.environ.get("MM_LIB_PATH", "default"), "tune": os.environ.get("TUNE", ""), "scale": scale, "ms_min": min(ts[1:]), "ms_all": ts,
       "evaluated": st.evaluated_multiplies, "nnz_c": c.nnz}
if scale == 22:
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "configs.json")))["cfg5"]
    h = c.to_host()
    out["golden_ok"] = (digest_csr(h.row_ptr, h.col_idx, h.values) == g["digest_c"]
                        and st.evaluated_multiplies == g["evaluated"] and c.nnz == g["nnz_c"])
print(json.dumps(out), flush=True)
