// Shadow of the reference's <pagerank_lab/norms.hpp>: the B200 drop-in
// provides every name of it (include/pagerank_b200/dropin.hpp), so the
// reference's own tests compile unmodified against the GPU path
// (tests/cpp/Makefile: this directory comes first on the include path).
#pragma once
#include <pagerank_b200/dropin.hpp>
