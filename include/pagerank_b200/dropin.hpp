// pagerank_b200/dropin.hpp — makes the B200 implementation visible under the
// reference's namespace, so a caller written against
// <pagerank_lab/pagerank_lab.hpp> (pagerank_lab.hpp:4-10) compiles unchanged:
//
//   -#include <pagerank_lab/pagerank_lab.hpp>
//   +#include <pagerank_b200/dropin.hpp>
//
// Do not include both in one translation unit (the names would clash); the
// reference's host-only stats.hpp / chart.hpp / csv.hpp readers can still be
// used next to this header.
#pragma once

#include "pagerank_lab.hpp"

namespace pagerank_lab {
using namespace pagerank_lab::cuda;
} // namespace pagerank_lab
