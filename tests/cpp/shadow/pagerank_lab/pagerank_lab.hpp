// Shadow of the reference's umbrella header (pagerank_lab.hpp:4-10): the
// path's headers (graph, norms, pagerank, sweep) come from the B200 drop-in,
// the host-only reporting headers (chart, csv, stats) from the reference
// include tree, unchanged.
#pragma once
#include <pagerank_b200/dropin.hpp>
#include <pagerank_lab/chart.hpp>
#include <pagerank_lab/csv.hpp>
#include <pagerank_lab/stats.hpp>
