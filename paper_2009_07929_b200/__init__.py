"""B200-native Eager K-truss engine (arXiv 2009.07929 hot path).

Public surface mirrors the reference's C++ API (ktruss::compute_supports,
prune_edges, detail::run_fixpoint, ktruss, kmax_search); see truss.py. The
compute path is the sm_100a library libktg.so behind the C ABI in
include/ktg.h -- there is no CPU fallback.
"""
from . import errors, graph
from .graph import (ZeroTerminatedCsr, csr_from_pairs, erdos_renyi, extract_edges, rmat, rmat_cliques,
                    validate_csr)
from .truss import (Engine, KmaxResult, Strategy, SupportArray, SupportWidth, TrussOptions, TrussResult,
                    compute_supports, detail, hardware_threads, intersect_tails, kmax_search, ktruss,
                    prune_edges, reset_supports, run_fixpoint, strategy_from_string, to_string)

__all__ = [
    "errors", "graph", "ZeroTerminatedCsr", "csr_from_pairs", "erdos_renyi", "extract_edges", "rmat", "rmat_cliques",
    "validate_csr", "Engine", "KmaxResult", "Strategy", "SupportArray", "SupportWidth", "TrussOptions",
    "TrussResult", "compute_supports", "detail", "hardware_threads", "intersect_tails", "kmax_search",
    "ktruss", "prune_edges", "reset_supports", "run_fixpoint", "strategy_from_string", "to_string",
]
