// c5_golden.cpp — TEST INFRASTRUCTURE ONLY: the reference's own pagerank()
// (pagerank.hpp:70-108, unmodified, included from /root/reference) run on the
// BASELINE configs[4] graph (RMAT-28, 268M vertices, 4.26B edges), to write
// tests/golden/c5_rmat28.* (oracle/make_c5_golden.py drives it).
//
// The graph is built by csr_inplace.hpp (the same arrays as build_csr,
// graph.hpp:204-234, with ~21 GB instead of ~55 GB); `--check` stops after
// the build and prints the fingerprint, which make_c5_golden.py compares with
// the reference-built C2 / C4 goldens' fingerprints before trusting the
// scale-28 build.
//
// The solve is the reference's pagerank(), one std::thread per alpha
// (pagerank() is reentrant on a shared graph); an observer
// (pagerank.hpp:51-52) records the err trace.  Outputs in OUTDIR:
// fingerprint.json, lane<k>.json, ranks<k>.f64 (raw doubles, N of them).
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>
#include <algorithm>

#include <pagerank_lab/graph.hpp>
#include <pagerank_lab/norms.hpp>
#include <pagerank_lab/pagerank.hpp>

#include "csr_inplace.hpp"
#include "oracle.h"

using namespace pagerank_lab;

namespace {

double secs(std::chrono::steady_clock::time_point t0) { return csr_inplace::secs(t0); }

CsrGraph build(uint32_t scale, uint64_t* raw_edges) {
    CsrGraph g;
    csr_inplace::build_rmat(g, scale, 16, 0.57, 0.19, 0.19, 2108, raw_edges, true);
    return g;
}

void write_fingerprint(const CsrGraph& g, uint64_t raw, const char* path) {
    uint64_t maxin = 0;
    for (uint64_t v = 0; v < g.vertex_count; ++v)
        maxin = std::max(maxin, g.in_offsets[v + 1] - g.in_offsets[v]);
    FILE* f = std::fopen(path, "w");
    std::fprintf(f,
                 "{\"n\": %u, \"e\": %llu, \"ndangling\": %zu, \"h_offsets\": %llu, \"h_neighbors\": %llu, "
                 "\"h_degree\": %llu, \"h_dangling\": %llu, \"max_in_degree\": %llu, \"raw_edges\": %llu}\n",
                 g.vertex_count, (unsigned long long)g.edge_count(), g.dangling.size(),
                 (unsigned long long)orc_hash64(g.in_offsets.data(), g.in_offsets.size() * 8),
                 (unsigned long long)orc_hash64(g.in_neighbors.data(), g.in_neighbors.size() * 4),
                 (unsigned long long)orc_hash64(g.out_degree.data(), g.out_degree.size() * 4),
                 (unsigned long long)orc_hash64(g.dangling.data(), g.dangling.size() * 4),
                 (unsigned long long)maxin, (unsigned long long)raw);
    std::fclose(f);
}

} // namespace

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: c5_golden SCALE OUTDIR [--check] [--norm l1|l2|linf] [--tol T] "
                             "[--max-iter M] [alpha ...]\n");
        return 2;
    }
    const uint32_t scale = (uint32_t)std::atoi(argv[1]);
    const std::string out = argv[2];
    bool check = false;
    NormKind norm = NormKind::L2;
    double tol = 1e-6;
    int max_iter = 500;
    std::vector<double> alphas;
    for (int i = 3; i < argc; ++i) {
        const std::string a = argv[i];
        if (a == "--check") check = true;
        else if (a == "--norm") {
            const std::string k = argv[++i];
            norm = k == "l1" ? NormKind::L1 : (k == "l2" ? NormKind::L2 : NormKind::LInf);
        } else if (a == "--tol") tol = std::atof(argv[++i]);
        else if (a == "--max-iter") max_iter = std::atoi(argv[++i]);
        else alphas.push_back(std::atof(a.c_str()));
    }
    uint64_t raw = 0;
    const CsrGraph g = build(scale, &raw);
    write_fingerprint(g, raw, (out + "/fingerprint.json").c_str());
    if (check) return 0;

    std::vector<std::thread> ts;
    for (size_t k = 0; k < alphas.size(); ++k)
        ts.emplace_back([&, k] {
            std::vector<double> trace;
            const PageRankConfig cfg{.alpha = alphas[k], .tolerance = tol, .norm = norm,
                                     .max_iterations = max_iter};
            const auto t0 = std::chrono::steady_clock::now();
            const PageRankResult r = pagerank(g, cfg, [&](int it, std::span<const double>, double err) {
                trace.push_back(err);
                std::fprintf(stderr, "alpha %.2f it %d err %.17g (%.0fs)\n", alphas[k], it, err, secs(t0));
            });
            FILE* f = std::fopen((out + "/ranks" + std::to_string(k) + ".f64").c_str(), "wb");
            std::fwrite(r.ranks.data(), sizeof(double), r.ranks.size(), f);
            std::fclose(f);
            f = std::fopen((out + "/lane" + std::to_string(k) + ".json").c_str(), "w");
            std::fprintf(f, "{\"alpha\": %.17g, \"tol\": %.17g, \"iterations\": %d, \"converged\": %s, "
                            "\"loop_ms\": %.3f, \"err_trace\": [",
                         alphas[k], tol, r.iterations, r.converged ? "true" : "false", r.elapsed.count());
            for (size_t i = 0; i < trace.size(); ++i) std::fprintf(f, "%s%.17g", i ? ", " : "", trace[i]);
            std::fprintf(f, "]}\n");
            std::fclose(f);
        });
    for (auto& t : ts) t.join();
    return 0;
}
