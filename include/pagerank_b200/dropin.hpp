// pagerank_b200/dropin.hpp — makes the B200 implementation visible under the
// reference's namespace, so a caller written against
// <pagerank_lab/pagerank_lab.hpp> (pagerank_lab.hpp:4-10) compiles unchanged:
//
//   -#include <pagerank_lab/pagerank_lab.hpp>
//   +#include <pagerank_b200/dropin.hpp>
//
// Every name of the path (graph.hpp, norms.hpp, pagerank.hpp, sweep.hpp) is
// brought in by a using-declaration.  The reference's host-only reporting
// headers — stats.hpp (the mean-ratio tables), csv.hpp, chart.hpp — keep
// working next to this one: include them as before (their csv helpers
// format_double / csv_escape are theirs; this header's sweep CSV rows use its
// own copies internally, with identical output).  Do not include the
// reference's graph.hpp / pagerank.hpp / sweep.hpp in the same translation
// unit (the names would clash).
#pragma once

#include "pagerank_lab.hpp"

namespace pagerank_lab {
// norms.hpp
using cuda::NormKind;
using cuda::all_norms;
using cuda::norm_name;
using cuda::parse_norm;
using cuda::error_norm;
// graph.hpp
using cuda::MtxParseError;
using cuda::EdgeList;
using cuda::CsrGraph;
using cuda::parse_matrix_market;
using cuda::build_csr;
using cuda::load_matrix_market;
using cuda::load_csr_graph;
// pagerank.hpp
using cuda::RankVector;
using cuda::PageRankConfig;
using cuda::PageRankResult;
using cuda::IterationObserver;
using cuda::pagerank;
using cuda::estimate_iterations;
using cuda::reference_config;
using cuda::reference_ranks;
using cuda::reference_error;
// sweep.hpp
using cuda::SweepPlan;
using cuda::SweepRecord;
using cuda::sweep_csv_header;
using cuda::sweep_csv_row;
using cuda::write_sweep_csv;
using cuda::default_damping_grid;
using cuda::default_tolerance_grid;
using cuda::run_sweep;
using cuda::SensitivityFinding;
using cuda::SensitivityReport;
using cuda::detect_sensitivity;
// B200 additions (no reference counterpart)
using cuda::BatchedRun;
using cuda::pagerank_batched;
} // namespace pagerank_lab
