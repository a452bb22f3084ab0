"""cfg5 (k-truss support, R-MAT s22; SCALE to change) with the k-blocked passes of the
16-warp plain hash bins at several block sizes (mm_set_tuning param 20, bytes of B's
index array per block; 0 = off): min multiply time over reps, output checked against the
reference golden (tests/golden/configs.json) at scale 22, else against the unblocked run.
One JSON line per block size."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import ctypes as C
import torch
from golden_util import digest_csr
from paper_2111_09947_b200 import MultiplyPlan, workloads, _lib
from paper_2111_09947_b200.device import DeviceCsr
from paper_2111_09947_b200.multiply import multiply_device, _handle
scale = int(os.environ.get("SCALE", "22")); reps = int(os.environ.get("REPS", "3"))
sizes = [int(x) for x in os.environ.get("KBLOCK_MB", "0,48,64,80,100,128").split(",")]
w = workloads.cfg5(scale)
da = DeviceCsr.from_host(w.a, with_values=False)
plan = MultiplyPlan(algorithm=os.environ.get("ALGO", "auto"), semiring=w.semiring)
gold = json.load(open(os.path.join(ROOT, "tests", "golden", "configs.json")))["cfg5"] if scale == 22 else None
base = None
flops_min = [int(x) for x in os.environ.get("KBLOCK_MIN_FLOPS", "1048576").split(",")]
for mb, fmin in [(mb, f) for mb in sizes for f in (flops_min if mb else flops_min[:1])]:
    prm = [-1] * 20 + [mb << 20, fmin]
    _lib.load().mm_set_tuning(_handle(0), (C.c_int64 * len(prm))(*prm), len(prm))
    ts = []
    for _ in range(reps + 1):
        torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); c, st = multiply_device(da, da, da, plan); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    h = c.to_host()
    dg = digest_csr(h.row_ptr, h.col_idx, h.values)
    out = {"kblock_mb": mb, "min_flops": fmin, "scale": scale, "nnz_b": int(w.a.nnz), "ms_min": min(ts[1:]), "ms_all": ts,
           "evaluated": st.evaluated_multiplies, "nnz_c": c.nnz}
    if gold:
        out["golden_ok"] = dg == gold["digest_c"] and st.evaluated_multiplies == gold["evaluated"] and c.nnz == gold["nnz_c"]
    if base is None:
        base = (dg, st.evaluated_multiplies, c.nnz)
    out["same_as_first"] = (dg, st.evaluated_multiplies, c.nnz) == base
    print(json.dumps(out), flush=True)
    del c, h
