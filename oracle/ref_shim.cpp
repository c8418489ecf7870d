// ref_shim.cpp — C-ABI shim over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file against
// /root/reference/proj/include (+ tests/support) with the reference's own
// Release flags (CMakeLists.txt:7-9: -O3 -DNDEBUG, C++20) into
// oracle/_ref/libprref.so.  No reference source is copied into this repo;
// this file only forwards plain pointers to the reference's inline functions:
//   build_csr        graph.hpp:204-234
//   pagerank         pagerank.hpp:70-108  (observer hook :51-52,98 records err)
//   error_norm       norms.hpp:48-78
//   estimate_iterations pagerank.hpp:113-123
//   random_digraph / regular_ring / scale_free_web  tests/support/graph_gen.hpp:21-85
//   dense_pagerank   tests/support/dense_oracle.hpp:24-62
//   parse_matrix_market / load_matrix_market  graph.hpp:111-199,238-247
// Used to pin the oracle/oracle.c restatement, to write tests/golden/, and as
// the CPU baseline ("kind": "reference") in bench.py.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <sstream>
#include <string>
#include <random>
#include <span>
#include <stdexcept>
#include <utility>
#include <vector>

#include <pagerank_lab/graph.hpp>
#include <pagerank_lab/norms.hpp>
#include <pagerank_lab/pagerank.hpp>
#include <support/dense_oracle.hpp>
#include <support/graph_gen.hpp>

using namespace pagerank_lab;

namespace {
NormKind kind_of(int k) { return k == 0 ? NormKind::L1 : (k == 1 ? NormKind::L2 : NormKind::LInf); }

EdgeList edge_list_from(uint32_t n, const uint32_t* pairs, uint64_t m) {
    EdgeList el;
    el.vertex_count = n;
    el.edges.resize(m);
    for (uint64_t i = 0; i < m; ++i) el.edges[i] = {pairs[2 * i], pairs[2 * i + 1]};
    return el;
}
} // namespace

extern "C" {

// ---- CsrGraph --------------------------------------------------------------
void* ref_build_csr(uint32_t n, const uint32_t* pairs, uint64_t m) {
    EdgeList el = edge_list_from(n, pairs, m);
    return new CsrGraph(build_csr(std::move(el))); // by value: always move (graph.hpp:204)
}
void ref_csr_free(void* g) { delete static_cast<CsrGraph*>(g); }
uint32_t ref_csr_vertex_count(void* g) { return static_cast<CsrGraph*>(g)->vertex_count; }
uint64_t ref_csr_edge_count(void* g) { return static_cast<CsrGraph*>(g)->edge_count(); }
uint32_t ref_csr_dangling_count(void* g) {
    return static_cast<uint32_t>(static_cast<CsrGraph*>(g)->dangling.size());
}
void ref_csr_copy(void* gp, uint64_t* off, uint32_t* nbr, uint32_t* deg, uint32_t* dang) {
    const CsrGraph& g = *static_cast<CsrGraph*>(gp);
    if (off) std::memcpy(off, g.in_offsets.data(), g.in_offsets.size() * sizeof(uint64_t));
    if (nbr) std::memcpy(nbr, g.in_neighbors.data(), g.in_neighbors.size() * sizeof(uint32_t));
    if (deg) std::memcpy(deg, g.out_degree.data(), g.out_degree.size() * sizeof(uint32_t));
    if (dang) std::memcpy(dang, g.dangling.data(), g.dangling.size() * sizeof(uint32_t));
}

// ---- engine ----------------------------------------------------------------
// Returns 0 ok, 1 std::invalid_argument, 2 other exception.
int ref_pagerank(void* gp, double alpha, double tol, int norm, int max_iter, double* ranks,
                 int* iterations, int* converged, double* err_trace, double* elapsed_ms) {
    try {
        const CsrGraph& g = *static_cast<CsrGraph*>(gp);
        const PageRankConfig cfg{.alpha = alpha, .tolerance = tol, .norm = kind_of(norm),
                                 .max_iterations = max_iter};
        IterationObserver obs;
        if (err_trace)
            obs = [err_trace](int it, std::span<const double>, double err) {
                err_trace[it - 1] = err;
            };
        const PageRankResult r = pagerank(g, cfg, obs);
        if (ranks) std::memcpy(ranks, r.ranks.data(), r.ranks.size() * sizeof(double));
        *iterations = r.iterations;
        *converged = r.converged ? 1 : 0;
        if (elapsed_ms) *elapsed_ms = r.elapsed.count();
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    } catch (...) {
        return 2;
    }
}

double ref_error_norm(int kind, const double* r, const double* s, uint64_t nr, uint64_t ns,
                      int* status) {
    try {
        *status = 0;
        return error_norm(kind_of(kind), std::span<const double>(r, nr),
                          std::span<const double>(s, ns));
    } catch (const std::invalid_argument&) {
        *status = 1;
        return 0.0;
    }
}

int ref_estimate_iterations(double alpha, double tol) {
    try {
        return estimate_iterations(alpha, tol);
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

// ---- reference test generators (std::mt19937 raw draws) ---------------------
void* ref_rng_new(uint32_t seed) { return new std::mt19937(seed); }
void ref_rng_free(void* r) { delete static_cast<std::mt19937*>(r); }
uint32_t ref_rng_next(void* r) { return static_cast<uint32_t>((*static_cast<std::mt19937*>(r))()); }

void* ref_gen_random_digraph(void* rng, uint32_t n, double p, int force_dangling) {
    return new EdgeList(testing::random_digraph(*static_cast<std::mt19937*>(rng), n, p,
                                                force_dangling != 0));
}
void* ref_gen_regular_ring(uint32_t n, uint32_t k) { return new EdgeList(testing::regular_ring(n, k)); }
void* ref_gen_scale_free_web(void* rng, uint32_t n, uint32_t out_links, double dangling_fraction) {
    return new EdgeList(testing::scale_free_web(*static_cast<std::mt19937*>(rng), n, out_links,
                                                dangling_fraction));
}
uint32_t ref_edges_n(void* e) { return static_cast<EdgeList*>(e)->vertex_count; }
uint64_t ref_edges_m(void* e) { return static_cast<EdgeList*>(e)->edges.size(); }
void ref_edges_copy(void* e, uint32_t* pairs) {
    const auto& ed = static_cast<EdgeList*>(e)->edges;
    for (size_t i = 0; i < ed.size(); ++i) {
        pairs[2 * i] = ed[i].first;
        pairs[2 * i + 1] = ed[i].second;
    }
}
void ref_edges_free(void* e) { delete static_cast<EdgeList*>(e); }

int ref_dense_pagerank(uint32_t n, const uint32_t* pairs, uint64_t m, double alpha, double tol,
                       int norm, int max_iter, double* ranks, int* iterations, int* converged) {
    const EdgeList el = edge_list_from(n, pairs, m);
    const PageRankConfig cfg{.alpha = alpha, .tolerance = tol, .norm = kind_of(norm),
                             .max_iterations = max_iter};
    const auto r = testing::dense_pagerank(el, cfg);
    std::memcpy(ranks, r.ranks.data(), r.ranks.size() * sizeof(double));
    *iterations = r.iterations;
    *converged = r.converged ? 1 : 0;
    return 0;
}

} // extern "C"

extern "C" {
// A reference CsrGraph filled from reference-layout arrays (plain data copy, no
// reference logic): lets the CPU baseline time the reference's pagerank on a
// graph that was generated and built elsewhere.
void* ref_csr_from_arrays(uint32_t n, const uint64_t* off, const uint32_t* nbr,
                          const uint32_t* deg) {
    auto* g = new CsrGraph();
    g->vertex_count = n;
    g->in_offsets.assign(off, off + (size_t)n + 1);
    g->in_neighbors.assign(nbr, nbr + off[n]);
    g->out_degree.assign(deg, deg + n);
    for (uint32_t v = 0; v < n; ++v)
        if (g->out_degree[v] == 0) g->dangling.push_back(v); // graph.hpp:230-231
    return g;
}
}

extern "C" {
// parse_matrix_market (graph.hpp:111-199) on an in-memory stream: the
// EdgeList (free with ref_edges_free), or null with the MtxParseError's line
// and what() in err_line / msg.
void* ref_parse_mtx(const char* text, uint64_t len, uint64_t* err_line, char* msg, int cap) {
    std::istringstream in(std::string(text, len));
    try {
        return new EdgeList(parse_matrix_market(in));
    } catch (const MtxParseError& e) {
        *err_line = e.line();
        std::snprintf(msg, (size_t)cap, "%s", e.what());
        return nullptr;
    }
}
// load_matrix_market (graph.hpp:238-247): errors as runtime_error what()
void* ref_load_mtx(const char* path, char* msg, int cap) {
    try {
        return new EdgeList(load_matrix_market(path));
    } catch (const std::exception& e) {
        std::snprintf(msg, (size_t)cap, "%s", e.what());
        return nullptr;
    }
}
}

#include "csr_inplace.hpp"

extern "C" {
// The RMAT benchmark graph as a reference CsrGraph, built in place on all
// host threads by csr_inplace.hpp (the same arrays as build_csr,
// graph.hpp:204-234, which at scale 28 would need ~55 GB and ~16 min on one
// thread).  The reference arm of bench.py then times the reference's own
// pagerank() on it.
void* ref_csr_rmat(uint32_t scale, uint32_t edge_factor, double a, double b, double c, uint64_t seed) {
    auto* g = new CsrGraph();
    uint64_t raw = 0;
    csr_inplace::build_rmat(*g, scale, edge_factor, a, b, c, seed, &raw);
    return g;
}
}
