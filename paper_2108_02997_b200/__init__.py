"""paper_2108_02997_b200 — B200-native pull power-iteration PageRank.

The hot path of arXiv 2108.02997 ("Adjusting PageRank parameters and
Comparing results"): the reference's pagerank()/error_norm()/build_csr()/
run_sweep() re-built as sm_100a CUDA kernels behind a C ABI
(include/prgpu.h, libprgpu.so).  `pagerank_lab` mirrors the reference API.
"""
from .pagerank_lab import (  # noqa: F401
    BatchedRun, CsrGraph, EdgeList, MtxParseError, NormKind, PageRankConfig, PageRankResult,
    SensitivityFinding, Session, SweepPlan, SweepRecord, all_norms, build_csr, csr_from_arrays,
    default_damping_grid, default_tolerance_grid, detect_sensitivity, error_norm,
    estimate_iterations, format_double, generate_grid, generate_rmat, load_csr_graph,
    load_matrix_market, norm_name, pagerank, pagerank_batched, parse_matrix_market, parse_norm,
    reference_config, reference_error, reference_ranks, run_sweep, sweep_csv_header,
    sweep_csv_row, write_sweep_csv,
)

__version__ = "0.1.0"
