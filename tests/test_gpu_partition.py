"""The multi-GPU row partition on one GPU: every rank's block multiplied
separately (as rank r would on GPU r) and concatenated must equal the 1-GPU C
bit for bit, for P in {2, 4, 8}, with the cuts bench.py uses — the
flop-balanced cuts and the cost-refined cuts (distributed.refine_cuts) — on
cfg2 (R-MAT s20 triangle count) and cfg5 (R-MAT s22 k-truss support).

Row independence is the reference's own contract (multiply.py:8-11); the
expected C is pinned to the reference's digest (tests/golden/configs.json).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from golden_util import digest_csr, digest_mat, load_json  # noqa: E402
from paper_2111_09947_b200 import MultiplyPlan, workloads  # noqa: E402
from paper_2111_09947_b200.device import DeviceCsr  # noqa: E402
from paper_2111_09947_b200.distributed import (balanced_cuts, concat_row_blocks, cut_offsets,  # noqa: E402
                                               imbalance, refine_cuts, row_blocks, row_work_device)
from paper_2111_09947_b200.multiply import multiply_device, reduce_sum  # noqa: E402


@pytest.fixture(autouse=True, scope="module")
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def _partitioned(dl, plan, cuts):
    offs = cut_offsets(dl, cuts)
    parts, ms, sums = [], [], []
    for blk in row_blocks(dl, cuts, offs):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        c, _ = multiply_device(blk, blk, dl, plan)
        e1.record()
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
        parts.append(c)
        sums.append(int(reduce_sum(c.values).item()) if c.nnz else 0)
    return concat_row_blocks(parts), ms, sums


@pytest.mark.parametrize("cfg", ["cfg2", pytest.param("cfg5", marks=pytest.mark.slow)])
def test_partitioned_multiply_bitwise(cfg):
    g = load_json("configs.json").get(cfg)
    if g is None:
        pytest.skip(f"{cfg} golden not generated")
    w = workloads.cfg2() if cfg == "cfg2" else workloads.cfg5()
    assert digest_mat(w.a) == g["digest_a"]
    dl = DeviceCsr.from_host(w.a, with_values=False)
    plan = MultiplyPlan(algorithm="auto", semiring=w.semiring)
    full, _ = multiply_device(dl, dl, dl, plan)
    h = full.to_host()
    assert digest_csr(h.row_ptr, h.col_idx, h.values) == g["digest_c"]
    del h
    work = row_work_device(dl, dl, dl).cpu().numpy()
    for parts in (2, 4, 8):
        cuts = balanced_cuts(work, parts)
        for rnd in range(2):
            cc, ms, sums = _partitioned(dl, plan, cuts)
            assert torch.equal(cc.ptr, full.ptr), (parts, rnd)
            assert torch.equal(cc.idx, full.idx), (parts, rnd)
            assert torch.equal(cc.values, full.values), (parts, rnd)
            assert sum(sums) == g["sum_c"]          # the all-reduced count
            print(cfg, parts, rnd, "imbalance", round(imbalance(ms), 3), [round(x, 2) for x in ms])
            cuts = refine_cuts(work, cuts, ms, parts)
