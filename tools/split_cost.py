"""cfg2: device time of the row blocks [0, r) and [r, m) (r at a share of L's entries) against the whole multiply."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2111_09947_b200 import MultiplyPlan, plus_pair_semiring, workloads
from paper_2111_09947_b200.device import DeviceCsr
from paper_2111_09947_b200.distributed import row_block
from paper_2111_09947_b200.multiply import multiply_device, reduce_sum

low = workloads.triangle_lower(20)
dl = DeviceCsr.from_host(low, with_values=False)
plan = MultiplyPlan(algorithm="auto", semiring=plus_pair_semiring(np.int64))
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ptr = np.asarray(low.row_ptr)

def timed(a):
    best = 1e9
    for rep in range(6):
        flush.fill_(rep)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        c, st = multiply_device(a, a, dl, plan)
        t = reduce_sum(c.values)
        e1.record(); e1.synchronize()
        if rep: best = min(best, e0.elapsed_time(e1))
    return best, st.generated_flops

whole, f = timed(dl)
print("whole %.3f ms flops %d" % (whole, f))
for frac in (0.1, 0.2, 0.3, 0.5):
    r = int(np.searchsorted(ptr, int(frac * low.nnz)))
    b1 = row_block(dl, 0, r, 0, int(ptr[r])); b2 = row_block(dl, r, low.nrows, int(ptr[r]), low.nnz)
    t1, f1 = timed(b1); t2, f2 = timed(b2)
    print("first %.1f: r=%d  block1 %.3f ms (%.3f of flops)  block2 %.3f ms  sum %.3f (+%.3f)" % (frac, r, t1, f1 / f, t2, t1 + t2, t1 + t2 - whole))
