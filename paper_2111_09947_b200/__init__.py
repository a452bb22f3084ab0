"""B200-native masked SpGEMM: C = M (.) (A B) and C = (not M) (.) (A B).

Drop-in for the hot path of the reference package ``maskmul``
(arXiv 2111.09947): same operator API (pkg/src/maskmul/__init__.py:17-20),
computed by hand-written sm_100a CUDA kernels behind the C ABI in
include/maskmul_b200.h.
"""

from .multiply import (ALGORITHMS, MultiplyPlan, MultiplyStats, PlanError, flops_of,  # noqa: F401
                       inner_product_multiply, masked_multiply, masked_multiply_with_stats,
                       multiply_device, one_phase_multiply, reduce_sum, symbolic_phase,
                       two_phase_multiply)
from .semiring import (Semiring, arithmetic_semiring, plus_pair_semiring,  # noqa: F401
                       semiring_by_name)
from .sparse import (CscMatrix, CsrMatrix, MaskView, SparseError, degree_sort_relabel,  # noqa: F401
                     from_arrays, from_triples, is_pattern_symmetric, permute_symmetric,
                     simple_undirected_graph, to_csc, to_csr, transpose, tril_strict)

__version__ = "0.1.0"
