// test_dropin.cpp — the C++ drop-in (include/pagerank_b200/dropin.hpp) used
// exactly like the reference's own API: same names under pagerank_lab::, same
// exceptions.  Cases follow the reference's tests (test_pagerank.cpp,
// test_graph.cpp, test_norms.cpp, test_sweep.cpp, acceptance.cpp); the
// checker for random graphs is a dense power iteration written here.
// Built by tests/test_cpp_dropin.py, run on the GPU box (needs libprgpu.so).
#include <pagerank_b200/dropin.hpp>

#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <random>
#include <set>
#include <sstream>
#include <string>
#include <vector>

using namespace pagerank_lab;

static int g_failed = 0, g_checks = 0;
#define CHECK(cond)                                                                   \
    do {                                                                              \
        ++g_checks;                                                                   \
        if (!(cond)) {                                                                \
            ++g_failed;                                                               \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);               \
        }                                                                             \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                                   \
    do {                                                                              \
        bool thrown = false;                                                          \
        try {                                                                         \
            (void)(expr);                                                             \
        } catch (const type&) {                                                       \
            thrown = true;                                                            \
        } catch (...) {                                                               \
        }                                                                             \
        CHECK(thrown);                                                                \
    } while (0)

static bool close(double a, double b, double rel) { return std::fabs(a - b) <= rel * std::max(1.0, std::fabs(b)); }

static EdgeList el_of(std::uint32_t n, std::vector<std::pair<std::uint32_t, std::uint32_t>> e) {
    EdgeList el;
    el.vertex_count = n;
    el.edges = std::move(e);
    return el;
}

// dense power iteration over the raw edge list (same update and stop rule)
struct Dense {
    std::vector<double> ranks;
    int iterations = 0;
};
static Dense dense(const EdgeList& el, double alpha, double tol, NormKind norm, int max_it = 500) {
    const std::uint32_t n = el.vertex_count;
    std::vector<char> adj((size_t)n * n, 0);
    for (auto [s, d] : el.edges) adj[(size_t)s * n + d] = 1;
    std::vector<std::uint32_t> deg(n, 0);
    for (std::uint32_t u = 0; u < n; ++u)
        for (std::uint32_t v = 0; v < n; ++v) deg[u] += adj[(size_t)u * n + v];
    std::vector<double> prev(n, 1.0 / n), next(n);
    int it = 0;
    double err = 0;
    do {
        double dsum = 0;
        for (std::uint32_t u = 0; u < n; ++u)
            if (!deg[u]) dsum += prev[u];
        const double c0 = (1.0 - alpha) / n + alpha * dsum / n;
        for (std::uint32_t v = 0; v < n; ++v) {
            double acc = 0;
            for (std::uint32_t u = 0; u < n; ++u)
                if (adj[(size_t)u * n + v]) acc += prev[u] / deg[u];
            next[v] = c0 + alpha * acc;
        }
        long double s = 0;
        double mx = 0;
        for (std::uint32_t v = 0; v < n; ++v) {
            const double d = next[v] - prev[v];
            if (norm == NormKind::L1) s += std::fabs(d);
            else if (norm == NormKind::L2) s += (long double)d * d;
            else mx = std::max(mx, std::fabs(d));
        }
        err = norm == NormKind::L1 ? (double)s : norm == NormKind::L2 ? (double)std::sqrt(s) : mx;
        ++it;
        prev.swap(next);
    } while (err >= tol && it < max_it);
    return {prev, it};
}

static EdgeList random_graph(std::mt19937& rng, std::uint32_t n, double p, bool drop_some) {
    EdgeList el;
    el.vertex_count = n;
    std::uniform_real_distribution<double> U(0, 1);
    std::vector<char> dead(n, 0);
    if (drop_some)
        for (std::uint32_t i = 0; i < n / 4 + 1; ++i) dead[rng() % n] = 1;
    for (std::uint32_t u = 0; u < n; ++u)
        for (std::uint32_t v = 0; v < n; ++v)
            if (!dead[u] && U(rng) < p) el.edges.emplace_back(u, v);
    return el;
}

int main() {
    // ---- pagerank known answers (test_pagerank.cpp:49-100) ----
    const CsrGraph two = build_csr(el_of(2, {{0, 1}, {1, 0}}));
    for (double a : {0.0, 0.5, 0.85, 1.0}) {
        const auto r = pagerank(two, {.alpha = a, .tolerance = 1e-6});
        CHECK(r.iterations == 1 && r.converged);
        CHECK(close(r.ranks[0], 0.5, 1e-12) && close(r.ranks[1], 0.5, 1e-12));
    }
    {
        const auto r = pagerank(build_csr(el_of(1, {})), {.alpha = 0.85});
        CHECK(r.iterations == 1 && r.converged && close(r.ranks[0], 1.0, 1e-14));
    }
    const CsrGraph star = build_csr(el_of(3, {{1, 0}, {2, 0}}));
    {
        const double c = 1.0 / (3.0 + 2 * 0.85);
        const auto r = pagerank(star, {.alpha = 0.85, .tolerance = 1e-10});
        CHECK(r.converged);
        CHECK(close(r.ranks[0], (1 + 1.7) * c, 1e-6) && close(r.ranks[1], c, 1e-6));
    }
    CHECK_THROWS_AS(pagerank(CsrGraph{}, {}), std::invalid_argument);
    CHECK_THROWS_AS(pagerank(two, {.alpha = 1.5}), std::invalid_argument);
    CHECK_THROWS_AS(pagerank(two, {.alpha = -0.1}), std::invalid_argument);
    CHECK_THROWS_AS(pagerank(two, {.tolerance = 0.0}), std::invalid_argument);
    CHECK_THROWS_AS(pagerank(two, {.max_iterations = 0}), std::invalid_argument);
    CHECK(estimate_iterations(0.85, 1e-6) == 85 && estimate_iterations(0.95, 1e-6) == 269);
    CHECK(estimate_iterations(0.75, 1e-6) == 48 && estimate_iterations(0.85, 1e-9) == 128);
    CHECK(estimate_iterations(0.85, 1e-3) == 43);
    CHECK_THROWS_AS(estimate_iterations(1.0, 1e-6), std::invalid_argument);

    // ---- graph building (test_graph.cpp:106-174) ----
    {
        const CsrGraph g = build_csr(el_of(3, {{0, 1}, {1, 2}}));
        CHECK((g.out_degree == std::vector<std::uint32_t>{1, 1, 0}));
        CHECK((g.dangling == std::vector<std::uint32_t>{2}));
        CHECK(g.in_edges(1).size() == 1 && g.in_edges(1)[0] == 0 && g.in_edges(0).empty());
        const CsrGraph d = build_csr(el_of(2, {{0, 1}, {0, 1}}));
        CHECK(d.edge_count() == 1 && (d.out_degree == std::vector<std::uint32_t>{1, 0}));
        const CsrGraph s = build_csr(el_of(2, {{0, 0}, {0, 1}}));
        CHECK(s.out_degree[0] == 2 && (s.dangling == std::vector<std::uint32_t>{1}));
        const CsrGraph e = build_csr(el_of(1, {}));
        CHECK((e.in_offsets == std::vector<std::uint64_t>{0, 0}));
    }
    std::mt19937 rng(21);
    for (int trial = 0; trial < 40; ++trial) {
        const EdgeList el = random_graph(rng, 1 + rng() % 40, 0.15, trial % 2 == 0);
        std::set<std::pair<std::uint32_t, std::uint32_t>> want(el.edges.begin(), el.edges.end());
        const CsrGraph g = build_csr(el);
        std::set<std::pair<std::uint32_t, std::uint32_t>> got;
        for (std::uint32_t v = 0; v < g.vertex_count; ++v)
            for (std::uint32_t u : g.in_edges(v)) got.emplace(u, v);
        CHECK(got == want);
        CHECK(g.in_offsets.front() == 0 && g.in_offsets.back() == g.in_neighbors.size());
    }

    // ---- parser (test_graph.cpp:82-104) ----
    auto line_of = [](const std::string& text) -> std::size_t {
        std::istringstream in(text);
        try {
            parse_matrix_market(in);
        } catch (const MtxParseError& e) {
            return e.line();
        }
        return 0;
    };
    CHECK(line_of("%%MatrixMarket matrix coordinate pattern\n1 1 0\n") == 1);
    CHECK(line_of("%%MatrixMarket matrix coordinate pattern general\n2 2 x\n") == 2);
    CHECK(line_of("%%MatrixMarket matrix coordinate pattern general\n% c\n2 2 1\n3 1\n") == 4);
    CHECK(line_of("%%MatrixMarket matrix coordinate pattern general\n2 2 2\n1 2\n") == 4);
    CHECK(line_of("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 abc\n") == 3);

    // ---- engine vs dense power iteration on random digraphs ----
    std::mt19937 r2(4242);
    for (int trial = 0; trial < 60; ++trial) {
        const EdgeList el = random_graph(r2, 2 + r2() % 40, 0.1 + 0.4 * (r2() % 100) / 100.0, trial % 2 == 0);
        const double alpha = 0.5 + 0.45 * (r2() % 100) / 100.0;
        const NormKind norm = all_norms[trial % 3];
        const double tol = trial % 3 == 0 ? 1e-8 : 1e-6;
        const auto got = pagerank(build_csr(el), {.alpha = alpha, .tolerance = tol, .norm = norm});
        const auto want = dense(el, alpha, tol, norm);
        CHECK(got.iterations == want.iterations);
        CHECK(error_norm(NormKind::LInf, got.ranks, want.ranks) <= 1e-10);
    }

    // ---- observer: rank conservation every iteration ----
    {
        std::mt19937 r3(11);
        const CsrGraph g = build_csr(random_graph(r3, 30, 0.2, true));
        int seen = 0;
        pagerank(g, {.alpha = 0.85, .tolerance = 1e-9}, [&](int it, std::span<const double> ranks, double) {
            long double s = 0;
            for (double x : ranks) s += x;
            CHECK(std::fabs((double)s - 1.0) <= 1e-9);
            CHECK(it == ++seen);
        });
        CHECK(seen > 1);
    }

    // ---- norms (test_norms.cpp:17-31) ----
    CHECK(close(error_norm(NormKind::L1, std::vector<double>{0.3, 0.7}, std::vector<double>{0.5, 0.5}), 0.4, 1e-12));
    CHECK(close(error_norm(NormKind::LInf, std::vector<double>{0.3, 0.7}, std::vector<double>{0.5, 0.5}), 0.2, 1e-12));
    CHECK_THROWS_AS(error_norm(NormKind::L1, std::vector<double>{0.5, 0.5}, std::vector<double>{1.0}),
                    std::invalid_argument);

    // ---- sweep over fixture files (test_sweep.cpp, acceptance.cpp:190-206, 331-366) ----
    {
        const auto dir = std::filesystem::temp_directory_path() / "prgpu_dropin_test";
        std::filesystem::create_directories(dir);
        const auto write = [&](const std::string& name, const std::string& text) {
            std::ofstream(dir / name) << text;
            return dir / name;
        };
        SweepPlan plan;
        plan.graphs = {write("two_cycle.mtx", "%%MatrixMarket matrix coordinate pattern general\n2 2 2\n1 2\n2 1\n"),
                       write("star.mtx", "%%MatrixMarket matrix coordinate pattern general\n3 3 2\n2 1\n3 1\n")};
        plan.alphas = default_damping_grid();
        plan.tolerances = {1e-3, 1e-6, 1e-9};
        plan.norms = {NormKind::L1, NormKind::L2, NormKind::LInf};
        plan.repeats = 2;
        for (bool fuse : {true, false}) {
            plan.fuse = fuse;
            const auto recs = run_sweep(plan);
            CHECK(recs.size() == 2 * 11 * 3 * 3);
            CHECK(recs.front().graph == "star");
            std::map<std::tuple<std::string, double, double>, std::array<int, 3>> by;
            for (const auto& r : recs) by[{r.graph, r.alpha, r.tolerance}][static_cast<int>(r.norm)] = r.iterations;
            for (const auto& [k, it] : by) CHECK(it[2] <= it[1] && it[1] <= it[0]);
        }
        plan.fuse = true;
        const auto a = run_sweep(plan), b = run_sweep(plan);
        plan.fuse = false;
        const auto c = run_sweep(plan);
        for (std::size_t i = 0; i < a.size(); ++i) {
            CHECK(a[i].iterations == b[i].iterations && a[i].err_vs_ref == b[i].err_vs_ref);
            CHECK(a[i].iterations == c[i].iterations && a[i].converged == c[i].converged);
            CHECK(std::fabs(a[i].err_vs_ref - c[i].err_vs_ref) <= 1e-12);
        }
        std::ostringstream os;
        write_sweep_csv(os, a);
        CHECK(os.str().rfind(std::string(sweep_csv_header), 0) == 0);
    }

    { // B200 addition: batched lanes and the power-series sweep agree
        std::mt19937 rng(5);
        EdgeList el;
        el.vertex_count = 3000;
        std::uniform_int_distribution<std::uint32_t> pick(0, 2999);
        for (int i = 0; i < 30000; ++i) el.edges.emplace_back(pick(rng), pick(rng));
        const CsrGraph g = build_csr(el);
        const std::vector<double> alphas{0.5, 0.85, 0.99};
        const auto a = pagerank_batched(g, alphas, 1e-9, NormKind::L2, 500);
        const auto s = pagerank_batched(g, alphas, 1e-9, NormKind::L2, 500, 0, nullptr, true, /*series=*/true);
        for (std::size_t k = 0; k < alphas.size(); ++k) {
            CHECK(std::abs(a.results[k].iterations - s.results[k].iterations) <= 1);
            double d = 0;
            for (std::size_t v = 0; v < g.vertex_count; ++v)
                d = std::max(d, std::fabs(a.results[k].ranks[v] - s.results[k].ranks[v]));
            CHECK(d <= 1e-10);
        }
    }

    std::printf("%s: %d checks, %d failed\n", g_failed ? "FAIL" : "PASS", g_checks, g_failed);
    return g_failed ? 1 : 0;
}
