"""Sweep kernel-tier tuning on cfg2 (mm_set_tuning) and print numeric-phase ms."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2111_09947_b200 import MultiplyPlan, plus_pair_semiring, workloads, _lib
from paper_2111_09947_b200.device import DeviceCsr
from paper_2111_09947_b200.multiply import _handle, multiply_device

low = workloads.triangle_lower(int(os.environ.get("SCALE", "20")))
dl = DeviceCsr.from_host(low, with_values=False)
plan = MultiplyPlan(algorithm="hash", semiring=plus_pair_semiring(np.int64))
lib = _lib.load()
h = _handle(0)
lib.mm_profile_enable(h, 1)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
configs = [(4096, 65536, 9, 2), (16384, 65536, 9, 2), (4096, 262144, 9, 2), (16384, 262144, 9, 2),
           (1024, 65536, 9, 2), (4096, 65536, 10, 2), (4096, 65536, 9, 3), (16384, 1 << 40, 9, 2),
           (1 << 40, 1 << 41, 9, 2)]
for cfg in configs:
    prm = (C.c_int64 * 4)(*cfg)
    lib.mm_set_tuning(h, prm, 4)
    ms = (C.c_float * 6)()
    best = 1e9
    for rep in range(4):
        flush.fill_(rep)
        c, st = multiply_device(dl, dl, dl, plan)
        lib.mm_profile_read(h, ms, 6, None)
        if rep:
            best = min(best, ms[2])
    print(cfg, f"numeric {best:.3f} ms  total {ms[5]:.3f} ms", flush=True)
