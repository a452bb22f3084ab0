"""Host-side cost split of one small multiply (cfg1, device-resident inputs):
the Python steps of multiply_device timed one by one (perf_counter, median
of 300), the C call alone, and CUDA-event time of the whole call."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2111_09947_b200 import MultiplyPlan, workloads, _lib
from paper_2111_09947_b200.device import DeviceCsr
from paper_2111_09947_b200.multiply import _handle, _plan_t, multiply_device

w = workloads.cfg1()
dt = np.dtype(w.semiring.dtype)
dm = DeviceCsr.from_host(w.mask, with_values=False)
da = DeviceCsr.from_host(w.a, dtype=dt)
plan = MultiplyPlan(algorithm="hash", semiring=w.semiring)
lib = _lib.load()
dev = da.idx.device
for _ in range(20):
    multiply_device(dm, da, da, plan)
torch.cuda.synchronize()
T = {}
def tick(name, t0):
    T.setdefault(name, []).append(time.perf_counter() - t0)
for rep in range(300):
    t0 = time.perf_counter(); h = _handle(dev.index); tick("handle", t0)
    t0 = time.perf_counter(); pt = _plan_t(plan, False); tick("plan_t", t0)
    t0 = time.perf_counter(); mm_mask, mm_a, mm_b = dm.mm(), da.mm(), da.mm(); tick("mm_structs", t0)
    t0 = time.perf_counter(); stream = torch.cuda.current_stream(dev); tick("current_stream", t0)
    t0 = time.perf_counter()
    cap = dm.nnz
    row_ptr = torch.empty(dm.nrows + 1, dtype=torch.int64, device=dev)
    col_idx = torch.empty(cap, dtype=torch.int32, device=dev)
    values = torch.empty(cap, dtype=torch.float64, device=dev)
    tick("3x torch.empty", t0)
    nnz = C.c_int64(0); st = _lib.StatsT()
    t0 = time.perf_counter()
    rc = lib.mm_multiply(h, C.byref(pt), C.byref(mm_mask), C.byref(mm_a), C.byref(mm_b), None,
                         C.c_void_p(stream.cuda_stream), row_ptr.data_ptr(), col_idx.data_ptr(),
                         values.data_ptr(), cap, C.byref(nnz), C.byref(st))
    tick("mm_multiply C call", t0)
    t0 = time.perf_counter(); n = int(nnz.value); a1, a2 = col_idx[:n], values[:n]; tick("2x slice", t0)
    t0 = time.perf_counter(); DeviceCsr(dm.nrows, dm.ncols, row_ptr, a1, a2); tick("DeviceCsr()", t0)
    torch.cuda.synchronize()
    t0 = time.perf_counter(); multiply_device(dm, da, da, plan); tick("multiply_device total", t0)
    torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ms = []
for rep in range(200):
    torch.cuda.synchronize()
    ev0.record(); multiply_device(dm, da, da, plan); ev1.record(); ev1.synchronize()
    ms.append(ev0.elapsed_time(ev1))
for k, v in T.items():
    print(f"{k:24s} {np.median(v) * 1e6:8.1f} us")
print(f"{'events multiply_device':24s} {np.median(ms) * 1e3:8.1f} us")
