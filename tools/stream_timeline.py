"""Timeline (CUDA events) of the streamed triangle count's pieces on cfg2: copies, block multiplies."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2111_09947_b200 import MultiplyPlan, plus_pair_semiring, workloads
from paper_2111_09947_b200.device import DeviceCsr
from paper_2111_09947_b200.distributed import row_block
from paper_2111_09947_b200.multiply import multiply_device, reduce_sum

first = float(sys.argv[1]) if len(sys.argv) > 1 else 0.2
low = workloads.triangle_lower(20)
m, nnz = low.nrows, low.nnz
h_ptr = torch.from_numpy(np.ascontiguousarray(low.row_ptr, dtype=np.int64)).pin_memory()
h_idx = torch.from_numpy(np.ascontiguousarray(low.col_idx[:nnz], dtype=np.int32)).pin_memory()
dev = torch.device("cuda", 0)
d_ptr = torch.empty(m + 1, dtype=torch.int64, device=dev); d_idx = torch.empty(nnz, dtype=torch.int32, device=dev)
plan = MultiplyPlan(algorithm="auto", semiring=plus_pair_semiring(np.int64))
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
ptr = h_ptr.numpy(); r = int(np.searchsorted(ptr, int(first * nnz))); p1 = int(ptr[r])
cs = torch.cuda.Stream(dev); cur = torch.cuda.current_stream(dev)
E = lambda: torch.cuda.Event(enable_timing=True)
for rep in range(5):
    flush.fill_(rep); torch.cuda.synchronize()
    t0, c0, c1, c2, b1s, b1e, b2s, b2e = (E() for _ in range(8))
    t0.record(cur); cs.wait_stream(cur)
    with torch.cuda.stream(cs):
        d_ptr.copy_(h_ptr, non_blocking=True); c0.record(cs)
        d_idx[:p1].copy_(h_idx[:p1], non_blocking=True); c1.record(cs)
        d_idx[p1:].copy_(h_idx[p1:], non_blocking=True); c2.record(cs)
    full = DeviceCsr(m, m, d_ptr, d_idx, None)
    cur.wait_event(c1); b1s.record(cur)
    blk = row_block(full, 0, r, 0, p1); c, st = multiply_device(blk, blk, full, plan); t1 = reduce_sum(c.values); b1e.record(cur)
    cur.wait_event(c2); b2s.record(cur)
    blk = row_block(full, r, m, p1, nnz); c, st = multiply_device(blk, blk, full, plan); t2 = reduce_sum(c.values); b2e.record(cur)
    tri = int((t1 + t2).item())
    torch.cuda.synchronize()
    f = lambda e: round(t0.elapsed_time(e), 3)
    print("ptr", f(c0), "idx1", f(c1), "idx2", f(c2), "| blk1", f(b1s), "->", f(b1e), "| blk2", f(b2s), "->", f(b2e), "tri", tri)
