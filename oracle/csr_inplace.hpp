// csr_inplace.hpp — TEST INFRASTRUCTURE ONLY (oracle/): the reference-layout
// reverse CSR (graph.hpp:47-60) of the counter-based RMAT stream, built in
// place and in parallel instead of by build_csr(EdgeList) (graph.hpp:204-234),
// whose by-value sort of the whole edge list peaks at ~1.6x the raw edge
// bytes (~55 GB at scale 28).  The order (dst, src) is total, so
// any correct sort + unique gives the SAME arrays:
//   pass 1  regenerate the stream (oracle.c orc_rmat_gen, the generator the
//           GPU's is hash-checked against), count raw in-edges per
//           destination                                   graph.hpp:220-221
//   pass 2  regenerate, scatter each source into its destination's raw row
//   rows    sort + unique each row (= the std::sort/std::unique of :209-213
//           restricted to one destination)
//   compact rows left in ascending order, offsets scan     :224
//   degrees out_degree over the deduplicated edges         :222
//   dangling ascending                                     :230-231
// Peak memory ~ the CSR itself (21 GB at scale 28).  Pinned against the
// reference-built C2 / C4 fingerprints (make_c5_golden.py, test_oracle.py).
// G is any struct with the CsrGraph members (vertex_count, in_offsets,
// in_neighbors, out_degree, dangling as std::vector).
#pragma once

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

#include "oracle.h"

namespace csr_inplace {

inline unsigned nthreads() {
    const unsigned h = std::thread::hardware_concurrency();
    return h ? h : 4;
}

template <class F>
void parallel_for(uint64_t n, uint64_t grain, F&& f) {
    std::atomic<uint64_t> next{0};
    std::vector<std::thread> ts;
    for (unsigned t = 0; t < nthreads(); ++t)
        ts.emplace_back([&] {
            for (;;) {
                const uint64_t b = next.fetch_add(grain);
                if (b >= n) break;
                f(b, std::min(n, b + grain));
            }
        });
    for (auto& t : ts) t.join();
}

inline double secs(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

template <class G>
void build_rmat(G& g, uint32_t scale, uint32_t edge_factor, double a, double b, double c, uint64_t seed,
                uint64_t* raw_edges, bool log = false) {
    const auto t0 = std::chrono::steady_clock::now();
    orc_rmat_gen gen;
    orc_rmat_gen_init(&gen, scale, a, b, c, seed);
    const uint64_t n = 1ull << scale, m = (uint64_t)edge_factor << scale;
    std::vector<uint32_t> cnt(n, 0);
    std::atomic<uint64_t> kept{0};
    parallel_for(m, 1u << 20, [&](uint64_t lo, uint64_t hi) {
        uint64_t k = 0;
        for (uint64_t i = lo; i < hi; ++i) {
            uint32_t s, d;
            if (!orc_rmat_gen_edge(&gen, i, &s, &d)) continue;
            std::atomic_ref<uint32_t>(cnt[d]).fetch_add(1, std::memory_order_relaxed);
            ++k;
        }
        kept += k;
    });
    *raw_edges = kept.load();
    if (log) std::fprintf(stderr, "count: %.1fs raw edges %llu\n", secs(t0), (unsigned long long)*raw_edges);

    g.vertex_count = (uint32_t)n;
    g.in_offsets.assign(n + 1, 0);
    for (uint64_t v = 0; v < n; ++v) g.in_offsets[v + 1] = g.in_offsets[v] + cnt[v];
    std::fill(cnt.begin(), cnt.end(), 0u);
    g.in_neighbors.resize(*raw_edges);
    parallel_for(m, 1u << 20, [&](uint64_t lo, uint64_t hi) {
        for (uint64_t i = lo; i < hi; ++i) {
            uint32_t s, d;
            if (!orc_rmat_gen_edge(&gen, i, &s, &d)) continue;
            const uint32_t at = std::atomic_ref<uint32_t>(cnt[d]).fetch_add(1, std::memory_order_relaxed);
            g.in_neighbors[g.in_offsets[d] + at] = s;
        }
    });
    if (log) std::fprintf(stderr, "scatter: %.1fs\n", secs(t0));

    // sort + unique per row; cnt[v] = the row's deduplicated length
    parallel_for(n, 1u << 14, [&](uint64_t lo, uint64_t hi) {
        for (uint64_t v = lo; v < hi; ++v) {
            uint32_t* rl = g.in_neighbors.data() + g.in_offsets[v];
            uint32_t* rh = g.in_neighbors.data() + g.in_offsets[v + 1];
            std::sort(rl, rh);
            cnt[v] = (uint32_t)(std::unique(rl, rh) - rl);
        }
    });
    if (log) std::fprintf(stderr, "row sort: %.1fs\n", secs(t0));
    uint64_t pos = 0;
    for (uint64_t v = 0; v < n; ++v) { // left compaction in ascending row order
        const uint64_t lo = g.in_offsets[v];
        if (pos != lo && cnt[v])
            std::memmove(g.in_neighbors.data() + pos, g.in_neighbors.data() + lo, cnt[v] * sizeof(uint32_t));
        g.in_offsets[v] = pos;
        pos += cnt[v];
    }
    g.in_offsets[n] = pos;
    g.in_neighbors.resize(pos);
    std::vector<uint32_t>().swap(cnt);
    g.out_degree.assign(n, 0);
    parallel_for(pos, 1u << 22, [&](uint64_t lo, uint64_t hi) {
        for (uint64_t i = lo; i < hi; ++i)
            std::atomic_ref<uint32_t>(g.out_degree[g.in_neighbors[i]]).fetch_add(1, std::memory_order_relaxed);
    });
    g.dangling.clear();
    for (uint64_t v = 0; v < n; ++v)
        if (g.out_degree[v] == 0) g.dangling.push_back((uint32_t)v);
    if (log) std::fprintf(stderr, "csr: %.1fs e=%llu\n", secs(t0), (unsigned long long)pos);
}

} // namespace csr_inplace
